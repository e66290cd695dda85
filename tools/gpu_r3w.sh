#!/bin/bash
# r3w: 512-key sample, smem candidate sort, separate prep
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider -k "adversarial or c3_unit or golden or outlier or per_head or vs_oracle or med3x or frozen" > gpurun_out/pytest_r3w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3w.log
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_w.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -s 40 -c 40 --csv --log-file gpurun_out/c3_warm_launches.csv python tools/c3_unit.py 10 > gpurun_out/c3_warm.log 2>&1
echo done
