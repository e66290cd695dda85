#!/bin/bash
# r4b: paged append scatter kernel
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_paged.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider > gpurun_out/pytest_r4b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4b.log
timeout 900 python tools/fuzz_attention.py --cases 80 --seed 31 > gpurun_out/fuzz_attn_r4b.log 2>&1
echo done
