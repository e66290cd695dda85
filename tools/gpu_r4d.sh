#!/bin/bash
# r4d: median grid sizing (>= 32 chunks / thread) + bins-in-use zero/merge
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/c1_unit.py > gpurun_out/c1_unit_d.log 2>&1
timeout 300 python tools/c3_unit.py 40 > gpurun_out/c3_unit_d.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider -k "adversarial or c3_unit or golden or outlier or per_head or vs_oracle or med3x or frozen" > gpurun_out/pytest_r4d.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4d.log
timeout 600 python tools/fuzz_parity.py --cases 600 --seed 99 > gpurun_out/fuzz_r4d.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -s 60 -c 12 \
   --csv --log-file gpurun_out/c1_warm_launches.csv python tools/c1_unit.py > gpurun_out/c1_warm.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 > gpurun_out/bench_c1_d.json 2> gpurun_out/bench_c1_d.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_d.json 2> gpurun_out/bench_c3_d.err
echo done
