#!/bin/bash
# r3r: fused Med3x prep (token offsets + prep in one pass)
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py tests/test_gpu_paged.py -q -x -p no:cacheprovider > gpurun_out/pytest_r3r.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3r.log
timeout 900 python tools/fuzz_parity.py --cases 1000 --seed 123 > gpurun_out/fuzz_r3r.log 2>&1
timeout 300 python tools/c3_unit.py 20 > gpurun_out/c3_unit_r.log 2>&1
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c3 > gpurun_out/bench_c3_r.json 2> gpurun_out/bench_c3_r.err
timeout 300 python bench.py --no-attn --no-cpu --no-e2e --workload c1 > gpurun_out/bench_c1_r.json 2> gpurun_out/bench_c1_r.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'radix|prep_ext' -s 10 -c 5 \
   -o gpurun_out/prof_m3enc_c3r -f python tools/c3_unit.py 3 > gpurun_out/prof_m3enc_c3r.log 2>&1
echo done
