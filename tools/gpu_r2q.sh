#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
for st in 6 1; do timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 --streams $st > gpurun_out/bench_c3_s$st.json 2>&1; done
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c2 > gpurun_out/bench_c2_q.json 2>&1
echo done
