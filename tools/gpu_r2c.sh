#!/bin/bash
# pair-kernel bring-up: attention tests, timing, ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention_shapes.py tests/test_gpu_paged.py tests/test_gpu_parity.py -k "attention or paged or pair" -q -x -p no:cacheprovider > gpurun_out/pytest_attn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_attn.log
timeout 120 python tools/attn_cmp.py > gpurun_out/attn_cmp.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'attention_pair' -s 3 -c 1 \
   -o gpurun_out/prof_pair -f python tools/attn_prof.py > gpurun_out/prof_pair.log 2>&1
echo done
