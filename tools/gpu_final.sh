#!/bin/bash
# Evidence pass: tests, smoke, benches, launch list, ncu full captures.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
for wl in c1 c3 c5; do
  timeout 900 python bench.py --workload $wl --no-attn --no-cpu --steps 3 > gpurun_out/bench_$wl.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$wl.log
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --attn-tokens 32768 > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'encode_tc|encode_warp|decode_fast|attention_mma' -c 5 \
   -o gpurun_out/prof_main -f python tools/prof_unit.py --reps 1 > gpurun_out/prof_main.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'radix_hist|decode_flag' -c 4 \
   -o gpurun_out/prof_med3x -f python tools/prof_unit.py --reps 1 --outlier --attn-batch 0 > gpurun_out/prof_med3x.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_fa' -c 1 \
   -o gpurun_out/prof_prefill -f python tools/prefill_prof.py > gpurun_out/prof_prefill.log 2>&1
timeout 300 python tools/prefill_bench.py > gpurun_out/prefill.log 2>&1
echo done
