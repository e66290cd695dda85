#!/bin/bash
# pair kernel: tests + L2 prefetch distance sweep
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_attention_shapes.py tests/test_gpu_paged.py tests/test_gpu_parity.py -k "attention or paged" -q -x -p no:cacheprovider > gpurun_out/pytest_attn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_attn.log
for pf in 16 0 4 32 64; do
  if [ $pf != 16 ]; then HQMQ_NVCC_EXTRA="-DHQMQ_PAIR_PF=$pf" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1; fi
  echo "PF=$pf" >> gpurun_out/attn_sweep.log
  timeout 120 python tools/attn_cmp.py >> gpurun_out/attn_sweep.log 2>&1
done
python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'attention_pair' -s 3 -c 1 \
   -o gpurun_out/prof_pair -f python tools/attn_prof.py > gpurun_out/prof_pair.log 2>&1
echo done
