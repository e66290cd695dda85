#!/bin/bash
# r4e: Med3x decode ring depth sweep (C3 decode step)
mkdir -p gpurun_out
for st in 4 2 3; do
  HQMQ_NVCC_EXTRA="-DHQMQ_FL_STAGES=$st" python -m paper_2605_27646_b200.build --force > gpurun_out/build_$st.log 2>&1
  echo "stages $st" >> gpurun_out/m3dec_sweep.log
  for i in 1 2; do timeout 300 python tools/m3dec_time.py >> gpurun_out/m3dec_sweep.log 2>&1; done
done
python -m paper_2605_27646_b200.build --force > gpurun_out/build.log 2>&1
echo done
