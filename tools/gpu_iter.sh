#!/bin/bash
# Iteration pass: parity tests, encode variant sweep, attention split sweep,
# short bench, ncu captures of the attention and decode kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/tune_encode.py ${ENC_VARIANTS:-0 4} > gpurun_out/tune_encode.log 2>&1
timeout 300 python tools/attn_bench.py > gpurun_out/attn_bench.log 2>&1
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_quick.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_mma|decode_fast' -c 2 \
   -o gpurun_out/prof_attn -f python tools/prof_unit.py --reps 1 > gpurun_out/prof_attn.log 2>&1
echo done
