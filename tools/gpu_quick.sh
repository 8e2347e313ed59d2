mkdir -p gpurun_out
for cfg in "PSWA_ATTN_HPC=2" "PSWA_ATTN_HPC=4" "PSWA_ATTN_HPC=2 PSWA_ATTN_HPC2=1" "PSWA_ATTN_HPC2=1 PSWA_ATTN_DBUF2=1" "PSWA_ATTN_HPC2=2 PSWA_ATTN_DBUF2=1"; do
  env $cfg timeout 300 python tools/probe_ops.py 2>&1 | tail -1
done
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 600 $NCU -k regex:window_attn -c 1 -o gpurun_out/ncu_ctx_attn_t8 python tools/profile_decode.py > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -3 gpurun_out/pytest_gpu.log
