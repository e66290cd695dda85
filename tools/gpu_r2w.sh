#!/bin/bash
# fast-decode tile / ring-depth sweep (C2 split-pass decode, 64 units back to back)
mkdir -p gpurun_out; rm -f gpurun_out/fd_sweep.log
for cfg in "128 2" "128 3" "128 4" "256 2" "256 1" "64 2"; do
  set -- $cfg
  HQMQ_NVCC_EXTRA="-DHQMQ_FD_TOK=$1 -DHQMQ_FD_STAGES=$2" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
  echo "TOK=$1 STAGES=$2" >> gpurun_out/fd_sweep.log
  timeout 300 python tools/split_diag.py 4 2>&1 | tail -2 >> gpurun_out/fd_sweep.log
done
python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
echo done
