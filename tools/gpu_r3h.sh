#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_fuzz.py -q -x -p no:cacheprovider > gpurun_out/pytest_r3h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3h.log
timeout 900 python tools/fuzz_attention.py --cases 300 --seed 5 > gpurun_out/fuzz_attention.log 2>&1
echo done
