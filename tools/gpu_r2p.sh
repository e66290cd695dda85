#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider > gpurun_out/pytest_m3dec.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_m3dec.log
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_m3dec.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'decode_flag' -s 3 -c 1 -o gpurun_out/prof_m3dec -f python tools/prof_unit.py --reps 5 --outlier --attn-batch 0 > gpurun_out/prof_m3dec.log 2>&1
echo done
