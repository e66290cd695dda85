#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/hist_sweep.log
for n in 4 2 1 8; do
  HQMQ_NVCC_EXTRA="-DHQMQ_HIST_CTAS_PER_SM=$n" python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
  echo "CTAS_PER_SM=$n" >> gpurun_out/hist_sweep.log
  timeout 120 python tools/c3_unit.py 20 >> gpurun_out/hist_sweep.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches_$n.csv python tools/c3_unit.py 2 > /dev/null 2>&1
done
python -m paper_2605_27646_b200.build --force > /dev/null 2>&1
echo done
