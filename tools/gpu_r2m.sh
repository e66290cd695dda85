#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/med3x_attn_err.py > gpurun_out/med3x_err.log 2>&1
timeout 900 python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py tests/test_gpu_attention_shapes.py -q -p no:cacheprovider > gpurun_out/pytest_med3x.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_med3x.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_mma' -s 6 -c 1 -o gpurun_out/prof_m3attn -f python tools/med3x_attn_err.py > gpurun_out/prof_m3attn.log 2>&1
echo done
