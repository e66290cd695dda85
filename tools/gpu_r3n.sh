#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r3n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3n.log
timeout 1200 python tools/fuzz_parity.py --cases 1000 --seed 99 > gpurun_out/fuzz_parity_r3n.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_n.json 2> gpurun_out/bench_c2_n.err
timeout 400 python bench.py --no-attn --no-cpu --no-e2e --workload c5 --steps 2 > gpurun_out/bench_c5_n.json 2> gpurun_out/bench_c5_n.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_n.json 2> gpurun_out/bench_c3_n.err
echo done
