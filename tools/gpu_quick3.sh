# scratch GPU call (edited per experiment): TMA-stored fp32 epilogue (opt-in) validation
mkdir -p gpurun_out
PSWA_GEMM_TMA_STORE=1 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
PSWA_GEMM_TMA_STORE=1 timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_gemm.py -x -q -k "accumulate or f32 or splitk" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_frame'])"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
