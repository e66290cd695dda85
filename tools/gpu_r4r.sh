#!/bin/bash
# streams sweep of the C2 round trip
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
rm -f gpurun_out/streams_sweep.log
for s in 6 4 8 12 6; do
  timeout 300 python bench.py --no-attn --no-cpu --no-e2e --streams $s > gpurun_out/bench_s$s.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_s$s.json')); print($s, d['value'], d['ms_per_step'])" >> gpurun_out/streams_sweep.log
done
echo done
