#!/bin/bash
# Med3x serving path bring-up: new tests + attention / paged suites
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py tests/test_gpu_attention_shapes.py tests/test_native_abi.py -q -x -p no:cacheprovider --durations=10 > gpurun_out/pytest_med3x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_med3x.log
echo done
