#!/bin/bash
# r3q: branch-free Med3x decode payload substitution
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/m3dec_time.py > gpurun_out/m3dec_time_q.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_med3x_serving.py -q -x -p no:cacheprovider -k "c3_unit or token_ranges or outlier or med3x or golden" > gpurun_out/pytest_r3q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r3q.log
timeout 600 python tools/fuzz_parity.py --cases 300 --seed 7 > gpurun_out/fuzz_r3q.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'decode_flag_tma' -s 60 -c 1 \
   -o gpurun_out/prof_m3dec_c3q -f python tools/m3dec_time.py > gpurun_out/prof_m3dec_c3q.log 2>&1
echo done
