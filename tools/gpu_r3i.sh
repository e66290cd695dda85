#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/fl_sweep.log
for cfg in "64 4" "32 4" "32 8" "16 8" "128 2"; do
  set -- $cfg
  HQMQ_NVCC_EXTRA="-DHQMQ_FL_TOK=$1 -DHQMQ_FL_STAGES=$2" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
  echo "TOK=$1 STAGES=$2" >> gpurun_out/fl_sweep.log
  timeout 300 python tools/m3dec_time.py >> gpurun_out/fl_sweep.log 2>&1
done
python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
echo done
