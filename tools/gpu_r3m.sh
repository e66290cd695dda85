#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/margin.log
for d in 1e-5f 3e-6f 1.5e-6f 1e-6f; do
  HQMQ_NVCC_EXTRA="-DHQMQ_DELTA_TC=$d" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
  echo "DELTA_TC=$d" >> gpurun_out/margin.log
  timeout 600 python tools/margin_check.py >> gpurun_out/margin.log 2>&1
  timeout 600 python tools/margin_check.py --c5 >> gpurun_out/margin.log 2>&1
done
python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
echo done
