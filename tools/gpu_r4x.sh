#!/bin/bash
mkdir -p gpurun_out
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
rm -f gpurun_out/streams2.log
for s in 8 8 7 16 5; do
  timeout 300 python bench.py --no-attn --no-cpu --no-e2e --streams $s > gpurun_out/bench_st.json 2> gpurun_out/bench_st_$s.err
  python -c "import json; d=json.load(open('gpurun_out/bench_st.json')); print($s, d['value'], d['ms_per_step'], d['encode']['ms_per_step'], d['decode']['ms_per_step'])" >> gpurun_out/streams2.log
done
echo done
