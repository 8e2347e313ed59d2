mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 600 $NCU -k regex:decode_phase -s 6 -c 1 -o gpurun_out/ncu_decode_phase python tools/profile_decode.py > /dev/null 2>&1
