#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/off_batch.log
for c in 8 16 32; do
  HQMQ_NVCC_EXTRA="-DHQMQ_OFF_BATCH=$c" python -m paper_2605_27646_b200.build --force > gpurun_out/build_$c.log 2>&1
  echo "batch $c" >> gpurun_out/off_batch.log
  for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/off_batch.log 2>&1; done
done
python -m paper_2605_27646_b200.build --force > gpurun_out/build.log 2>&1
echo done
