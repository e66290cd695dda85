#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/attn_expt.log
for ex in "-DHQMQ_PAIR_EXPT=2" "-DHQMQ_DISABLE_PAIR"; do
  HQMQ_NVCC_EXTRA="$ex" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
  echo "EXPT $ex" >> gpurun_out/attn_expt.log
  timeout 120 python tools/attn_cmp.py >> gpurun_out/attn_expt.log 2>&1
done
