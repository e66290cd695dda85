#!/bin/bash
# r4j: call-free pair-attention loop (global descriptor stays uniform) + 32-bit prologue divisions
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or attn or paged or decode or token_range" > gpurun_out/pytest_r4j.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4j.log
timeout 600 python tools/attn_cmp.py > gpurun_out/attn_cmp_j.log 2>&1
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_j.json 2> gpurun_out/bench_j.err
timeout 900 python tools/fuzz_attention.py --cases 100 --seed 5 > gpurun_out/fuzz_attn_j.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_pair' -s 3 -c 1 \
   -o gpurun_out/prof_attn_pair_j -f python tools/attn_prof.py > gpurun_out/prof_attn_pair_j.log 2>&1
echo done
