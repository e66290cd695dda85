#!/bin/bash
# r3u: sampled-bracket median, 2048 sample + 32-bit chunk split
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider -k "adversarial or c3_unit or golden or outlier or per_head or vs_oracle or med3x or frozen" > gpurun_out/pytest_r3u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3u.log
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_u.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'median|token_off|encode_warp' -s 10 -c 6 \
   -o gpurun_out/prof_median_u -f python tools/c3_unit.py 3 > gpurun_out/prof_median_u.log 2>&1
echo done
