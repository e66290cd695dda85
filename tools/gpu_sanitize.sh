#!/bin/bash
# compute-sanitizer passes over a representative subset of the GPU tests.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
# every tensor its own cudaMalloc, so memcheck sees allocation bounds
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
compute-sanitizer --tool memcheck python tools/sanitizer_selfcheck.py > gpurun_out/sanitize_selfcheck.log 2>&1; echo "selfcheck rc=$? (deliberate out-of-bounds decode: errors expected, proves the kernels are instrumented)" >> gpurun_out/sanitize_selfcheck.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "golden and (frozen or c1_slice or outlier or s64) or edge or crc or append or token_ranges" \
  > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "golden and (c1_slice or s64) or attention_golden" \
  > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "golden and s64" \
  > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/sanitize_synccheck.log
# paged decode attention and the tcgen05 prefill kernels (all four, via the variant tests)
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_paged.py tests/test_gpu_prefill_variants.py -x -q -k "not 256" \
  > gpurun_out/sanitize_memcheck_attn.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_attn.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_tensor_core" \
  > gpurun_out/sanitize_racecheck_attn.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck_attn.log
echo done
