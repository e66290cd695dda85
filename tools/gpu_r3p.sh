#!/bin/bash
# r3p: C3 Med3x decode profile (one unit, ncu full) + step timing
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 300 python tools/m3dec_time.py > gpurun_out/m3dec_time_p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'decode_flag_tma' -s 60 -c 1 \
   -o gpurun_out/prof_m3dec_c3 -f python tools/m3dec_time.py > gpurun_out/prof_m3dec_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'radix|token_off|encode_warp' -s 14 -c 7 \
   -o gpurun_out/prof_m3enc_c3 -f python tools/c3_unit.py 3 > gpurun_out/prof_m3enc_c3.log 2>&1
echo done
