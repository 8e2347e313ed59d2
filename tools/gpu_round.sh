# One GPU round: tests, smoke, bench, warm kernel times, launch list and
# ncu --set full captures of the probed kernels (see tools/ncu_traffic.py).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py > gpurun_out/kt.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_decode.py > gpurun_out/ncu_launch.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 600 $NCU -k regex:window_attn -c 1 -o gpurun_out/ncu_ctx_attn python tools/profile_decode.py > /dev/null 2>&1
timeout 600 $NCU -k regex:window_attn -s 66 -c 1 -o gpurun_out/ncu_step_attn python tools/profile_decode.py > /dev/null 2>&1
# gemm launch order of a decode: 0-4 hyper, 5-9 context block 0 (kv, q, wo, gate|up, down), ...,
# 53 = accumulator Q projection of step 0 (M=2040 N=K=512, the step_wq shape)
timeout 600 $NCU -k regex:gemm_tc_kernel -s 8 -c 1 -o gpurun_out/ncu_ctx_ffn_gu python tools/profile_decode.py > /dev/null 2>&1
timeout 600 $NCU -k regex:gemm_tc_kernel -s 53 -c 1 -o gpurun_out/ncu_step_wq python tools/profile_decode.py > /dev/null 2>&1
# phase (t=1, g=1) of the entropy decoder
timeout 600 $NCU -k regex:decode_phase -s 5 -c 1 -o gpurun_out/ncu_decode_phase python tools/profile_decode.py > /dev/null 2>&1
python tools/ncu_traffic.py ${TAG:-r01} > gpurun_out/traffic.log 2>&1
ls gpurun_out
