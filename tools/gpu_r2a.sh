#!/bin/bash
# round 2 first pass: GPU tests, C4 attention timing, ncu of the decode-attention kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/attn_cmp.py > gpurun_out/attn_cmp.log 2>&1
timeout 300 python tools/decode_bench.py > gpurun_out/decode_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_mma' -s 3 -c 1 \
   -o gpurun_out/prof_attn -f python tools/attn_prof.py > gpurun_out/prof_attn.log 2>&1
echo done
