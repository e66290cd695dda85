#!/bin/bash
# A/B: pair attention before / after the page-id prefetch (same box)
mkdir -p gpurun_out
rm -f gpurun_out/ab_pg.log
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
for i in 1 2; do echo "new" >> gpurun_out/ab_pg.log; timeout 300 python tools/attn_cmp.py 2>&1 | head -2 >> gpurun_out/ab_pg.log; done
cp paper_2605_27646_b200/csrc/attention_cluster.cu /tmp/ac_new.cu
cp tools/_ac_before_pg.cu.txt paper_2605_27646_b200/csrc/attention_cluster.cu
python -m paper_2605_27646_b200.build --force > gpurun_out/build_old.log 2>&1
for i in 1 2; do echo "old" >> gpurun_out/ab_pg.log; timeout 300 python tools/attn_cmp.py 2>&1 | head -2 >> gpurun_out/ab_pg.log; done
cp /tmp/ac_new.cu paper_2605_27646_b200/csrc/attention_cluster.cu
echo done
