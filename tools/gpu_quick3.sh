# scratch GPU call (edited per experiment): L2 bulk prefetch of residual segments
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
for v in "PSWA_GEMM_NO_L2_PREFETCH=1" "PSWA_X=0" "PSWA_GEMM_NO_L2_PREFETCH=1" "PSWA_X=0"; do
env $v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_rooflines']
print('$v', d['ms_per_step'], d['e2e']['ms_per_frame'], {n: (round(k[n]['us_per_launch'],1), round(k[n]['frac'],3)) for n in ('ctx_wo','ctx_wd','step_wo','step_wd','ch_mix','ch_d')})"
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
