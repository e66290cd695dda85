#!/bin/bash
# round 2 re-entry: full GPU suite, smoke, default bench line + C3 / C5 lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-attn > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c5 --no-attn --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
