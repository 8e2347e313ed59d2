# scratch GPU call (edited per experiment): CTA-pair tiles per epilogue kind
mkdir -p gpurun_out
for v in "PSWA_GEMM_PAIR_KINDS=0" "PSWA_GEMM_PAIR_KINDS=1" "PSWA_GEMM_PAIR_KINDS=2" "PSWA_GEMM_PAIR_KINDS=4" "PSWA_GEMM_PAIR_KINDS=3" "PSWA_GEMM_PAIR_KINDS=0"; do
env $v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['e2e']['ms_per_frame'])"
done
for v in 0 3; do
PSWA_GEMM_PAIR_KINDS=$v PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py 2>/dev/null | head -14 > gpurun_out/kt_pair$v.txt
done
