#!/bin/bash
# pair attention items-per-cluster sweep (key splits)
mkdir -p gpurun_out
rm -f gpurun_out/items_sweep.log
for d in 4 2 8 6 12; do
  HQMQ_NVCC_EXTRA="-DHQMQ_PAIR_ITEMS=$d" python -m paper_2605_27646_b200.build --force > gpurun_out/build_it$d.log 2>&1
  echo "items $d" >> gpurun_out/items_sweep.log
  timeout 300 python tools/attn_cmp.py 2>&1 | head -2 >> gpurun_out/items_sweep.log
done
python -m paper_2605_27646_b200.build --force > gpurun_out/build.log 2>&1
echo done
