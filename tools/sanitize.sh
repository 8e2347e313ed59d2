# compute-sanitizer over the decode workload (tools/sanitize_decode.py) at
# desk scale (SIMT attention, head_dim 4) and paper scale (tensor-core
# attention, TMA halos, tcgen05 GEMMs and the GEMM chains): memcheck
# (out-of-bounds / misaligned global and shared accesses), racecheck
# (shared-memory hazards), synccheck (barrier misuse), initcheck (reads of
# uninitialised global memory). Graphs off (PSWA_NO_GRAPH=1) so every launch
# is instrumented on its own; one more memcheck pass keeps the graphs.
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 200"
for preset in desk paper; do
  for tool in memcheck racecheck synccheck initcheck; do
    SAN_PRESET=$preset PSWA_NO_GRAPH=1 timeout 1500 $CS --tool $tool python tools/sanitize_decode.py > gpurun_out/sanitize_${preset}_$tool.log 2>&1
    echo "$preset $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${preset}_$tool.log | tail -1)"
  done
  SAN_PRESET=$preset timeout 1500 $CS --tool memcheck python tools/sanitize_decode.py > gpurun_out/sanitize_${preset}_memcheck_graphs.log 2>&1
  echo "$preset memcheck (graphs) rc=$? $(grep 'ERROR SUMMARY' gpurun_out/sanitize_${preset}_memcheck_graphs.log | tail -1)"
done
