# scratch GPU call (edited per experiment)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3

for v in "" "PSWA_GEMM_NO_WIDE=1"; do
env $v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['e2e']['ms_per_frame'], d['config2_iframe_1gpu'])"
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
