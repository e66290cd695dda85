#!/bin/bash
# Closing sanitizer pass (r02f) over the final library: memcheck / racecheck of
# the pair attention (contiguous + paged ragged), the codec and Med3x serving.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
python -m paper_2605_27646_b200.build > gpurun_out/build.log 2>&1
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_attention_shapes.py -x -q -p no:cacheprovider -k "pair" \
  > gpurun_out/sanitize_memcheck_pair.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_pair.log
timeout 1800 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_paged.py tests/test_gpu_med3x_serving.py tests/test_gpu_parity.py -x -q -p no:cacheprovider \
  -k "append or frozen or token_local or adversarial or c3_unit or golden and (frozen or outlier or s64) or token_ranges" \
  > gpurun_out/sanitize_memcheck_codec.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck_codec.log
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "adversarial or c3_unit or golden and s64" \
  > gpurun_out/sanitize_racecheck_codec.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck_codec.log
echo done
