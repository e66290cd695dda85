#!/bin/bash
# pair attention L2 prefetch distance sweep (after the load reordering)
mkdir -p gpurun_out
rm -f gpurun_out/pf_sweep.log
for d in 2 0 1 3 4; do
  HQMQ_NVCC_EXTRA="-DHQMQ_PAIR_PF=$d" python -m paper_2605_27646_b200.build --force > gpurun_out/build_pf$d.log 2>&1
  echo "pf $d" >> gpurun_out/pf_sweep.log
  timeout 300 python tools/attn_cmp.py 2>&1 | head -2 >> gpurun_out/pf_sweep.log
done
python -m paper_2605_27646_b200.build --force > gpurun_out/build.log 2>&1
echo done
