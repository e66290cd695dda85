#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adversarial.py -q -x -p no:cacheprovider > gpurun_out/pytest_r4s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r4s.log
timeout 900 python tools/fuzz_parity.py --cases 1000 --seed 1618 > gpurun_out/fuzz_r4s.log 2>&1
for i in 1 2; do timeout 300 python bench.py --no-attn --no-cpu --no-e2e > gpurun_out/bench_s_$i.json 2> gpurun_out/bench_s_$i.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:encode_prep -s 4 -c 4 --csv --log-file gpurun_out/prep_launch.csv python tools/prof_unit.py --reps 2 --attn-batch 0 > /dev/null 2>&1
echo done
