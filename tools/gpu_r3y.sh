#!/bin/bash
# r3y: median cleanup + register bin scan; full GPU suite + fuzz + timings
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r3y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3y.log
timeout 900 python tools/fuzz_parity.py --cases 1000 --seed 4242 > gpurun_out/fuzz_r3y.log 2>&1
for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/c3_unit_y.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -s 40 -c 40 --csv --log-file gpurun_out/c3_warm_launches.csv python tools/c3_unit.py 10 > gpurun_out/c3_warm.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_y.json 2> gpurun_out/bench_c3_y.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 > gpurun_out/bench_c1_y.json 2> gpurun_out/bench_c1_y.err
echo done
