#!/bin/bash
# Round-2 final evidence pass (r02d): GPU tests, smoke, bench lines (all configs
# + reference arm), fuzzers, Med3x / C4 attention timings, launch lists (default
# bench; warm C3 unit chain), ncu --set full captures (codec; C3 median chain +
# prep; C3 Med3x decode; pair attention; Med3x attention), sanitizers.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
for wl in c1 c3 c5; do
  timeout 900 python bench.py --workload $wl --no-attn --no-cpu --steps 3 > gpurun_out/bench_$wl.log 2> gpurun_out/bench_$wl.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 1200 python tools/fuzz_parity.py --cases 2000 --seed 2026 > gpurun_out/fuzz_parity.log 2>&1
timeout 900 python tools/fuzz_attention.py --cases 300 --seed 2026 > gpurun_out/fuzz_attention.log 2>&1
timeout 300 python tools/med3x_attn_err.py > gpurun_out/med3x_attention.log 2>&1
timeout 300 python tools/attn_cmp.py > gpurun_out/attn_cmp.log 2>&1
timeout 300 python tools/m3dec_time.py > gpurun_out/m3dec_time.log 2>&1
timeout 300 python tools/c3_unit.py 40 > gpurun_out/c3_unit.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --attn-tokens 32768 > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --cache-control none -s 40 -c 40 \
   --csv --log-file gpurun_out/c3_warm_launches.csv python tools/c3_unit.py 10 > gpurun_out/c3_warm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'encode_tc|encode_warp|encode_prep|decode_fast' -s 3 -c 3 \
   -o gpurun_out/prof_codec -f python tools/prof_unit.py --reps 2 --attn-batch 0 > gpurun_out/prof_codec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'median|token_off|encode_warp' -s 14 -c 7 \
   -o gpurun_out/prof_med3x -f python tools/c3_unit.py 3 > gpurun_out/prof_med3x.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'decode_flag_tma' -s 60 -c 1 \
   -o gpurun_out/prof_m3dec -f python tools/m3dec_time.py > gpurun_out/prof_m3dec.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_pair' -s 3 -c 1 \
   -o gpurun_out/prof_attn_pair -f python tools/attn_prof.py > gpurun_out/prof_attn_pair.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attention_mma' -s 6 -c 1 \
   -o gpurun_out/prof_attn_med3x -f python tools/med3x_attn_err.py > gpurun_out/prof_attn_med3x.log 2>&1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "frozen or token_local or 1032 or adversarial" \
  > gpurun_out/sanitize_memcheck_med3x.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_med3x.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_med3x_serving.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "1032 or token_local or adversarial" \
  > gpurun_out/sanitize_racecheck_med3x.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck_med3x.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "golden and (frozen or c1_slice or outlier or s64) or token_ranges" \
  > gpurun_out/sanitize_memcheck_codec.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_codec.log
echo done
