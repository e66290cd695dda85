#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_v$i.json 2> gpurun_out/bench_c3_v$i.err; done
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_v.json 2> gpurun_out/bench_c2_v.err
echo done
