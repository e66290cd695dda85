#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/attn_cmp.py > gpurun_out/attn_cmp.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attention_shapes.py tests/test_gpu_paged.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "attention or paged or pair" > gpurun_out/pytest_r3b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3b.log
echo done
