# compute-sanitizer memcheck / racecheck / synccheck over a small-shape subset of
# the GPU parity tests (persistent kernel: TMA + cp.async + mbarrier stages,
# stream-K fix-up, every tile configuration through the forced-config tests).
# Summaries land in gpurun_out/sanitize_<tool>.log.
set -u
SEL_MEM='test_conv_vs_oracle or test_gemm_vs_oracle or (test_stream_k_schedule and not sk-0 and not dp-0) or test_flat8 or test_transposed_orientation_forced or test_tall_tiles or test_strided_dgrad_phase_tma'
SEL_RACE='(test_conv_vs_oracle and mitchell and (fwd or dgrad or wgrad)) or test_flat8_narrow_tile or (test_stream_k_schedule and (sk-2 or sk-4)) or test_strided_dgrad_phase_tma'
for tool in memcheck synccheck racecheck; do
  if [ $tool = racecheck ]; then SEL=$SEL_RACE; EXTRA="--racecheck-report hazard"; else SEL=$SEL_MEM; EXTRA=""; fi
  timeout 3000 compute-sanitizer --tool $tool $EXTRA --print-limit 20 --error-exitcode 99 --target-processes all \
      python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
