#!/bin/bash
# r4g: small-S FFMA2 search geometry sweep (C1 unit, S=16)
mkdir -p gpurun_out
rm -f gpurun_out/c1_sweep.log
for v in "4 2" "2 4" "4 3" "2 3" "8 2"; do
  set -- $v
  HQMQ_NVCC_EXTRA="-DHQMQ_SMALL_S_WT=$1 -DHQMQ_SMALL_S_MINB=$2" python -m paper_2605_27646_b200.build --force > gpurun_out/build_$1_$2.log 2>&1 || echo "build fail $v" >> gpurun_out/c1_sweep.log
  echo "wt $1 minb $2" >> gpurun_out/c1_sweep.log
  for i in 1 2; do timeout 300 python tools/c1_unit.py >> gpurun_out/c1_sweep.log 2>&1; done
done
python -m paper_2605_27646_b200.build --force > gpurun_out/build.log 2>&1
echo done
