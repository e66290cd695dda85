#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_z.json 2> gpurun_out/bench_z.err
timeout 600 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_z3.json 2> gpurun_out/bench_z3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_count.csv python bench.py --no-attn --no-cpu --no-e2e --workload c3 --steps 1 --warmup 1 > /dev/null 2>&1
echo done
