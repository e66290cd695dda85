#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --workload c1 > gpurun_out/bench_c1_j.json 2> gpurun_out/bench_c1_j.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 --steps 20 > gpurun_out/bench_c1_j20.json 2> gpurun_out/bench_c1_j20.err
echo done
