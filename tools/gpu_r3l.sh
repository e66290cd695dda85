#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_r3l.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r3l.log
timeout 900 python tools/fuzz_parity.py --cases 500 --seed 77 > gpurun_out/fuzz_parity_r3l.log 2>&1
timeout 120 python tools/enc_timing.py > gpurun_out/enc_timing.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_c2_l.json 2> gpurun_out/bench_c2_l.err
timeout 400 python bench.py --no-attn --no-cpu --no-e2e --workload c5 --steps 2 > gpurun_out/bench_c5_l.json 2> gpurun_out/bench_c5_l.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'encode_prep|encode_tc' -c 6 python tools/prof_unit.py --reps 3 --attn-batch 0 > gpurun_out/ncu_prep.log 2>&1
echo done
