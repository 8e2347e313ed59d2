mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 600 $NCU -k regex:gemm_tc_kernel -s 7 -c 1 -o gpurun_out/ncu_ctx_wo2 python tools/profile_decode.py > /dev/null 2>&1
