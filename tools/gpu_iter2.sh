#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 --attn-tokens 32768 > gpurun_out/bench_quick.log 2>&1; echo "rc=$?" >> gpurun_out/bench_quick.log
timeout 900 python bench.py --workload c3 --no-cpu --no-e2e --no-attn --steps 3 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3unit.csv \
   python tools/prof_unit.py --reps 2 --outlier --attn-batch 0 > gpurun_out/launches_c3unit.log 2>&1
echo done
