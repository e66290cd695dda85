#!/bin/bash
# median pass grid: CTAs per SM sweep (C3 unit)
mkdir -p gpurun_out
rm -f gpurun_out/med_ctas.log
for c in 4 2 8 3; do
  HQMQ_NVCC_EXTRA="-DHQMQ_MED_CTAS=$c" python -m paper_2605_27646_b200.build --force > gpurun_out/build_$c.log 2>&1
  echo "ctas $c" >> gpurun_out/med_ctas.log
  for i in 1 2; do timeout 300 python tools/c3_unit.py 40 >> gpurun_out/med_ctas.log 2>&1; done
  timeout 300 python tools/c1_unit.py >> gpurun_out/med_ctas.log 2>&1
done
python -m paper_2605_27646_b200.build --force > gpurun_out/build.log 2>&1
echo done
