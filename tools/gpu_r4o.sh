#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_g.log 2> gpurun_out/bench_g.err
timeout 300 python tools/attn_cmp.py > gpurun_out/attn_cmp_g.log 2>&1
echo done
