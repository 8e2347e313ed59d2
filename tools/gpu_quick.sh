# scratch GPU call (edited per experiment): context residual GEMMs
mkdir -p gpurun_out
for v in "PSWA_GEMM_BIG_F32_BN=0" "PSWA_GEMM_BIG_F32_BN=128" "PSWA_GEMM_BIG_F32_BN=0"; do
env $v timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_rooflines']
print('$v', d['ms_per_step'], d['e2e']['ms_per_frame'], {n: (round(k[n]['us_per_launch'],1), round(k[n]['frac'],3)) for n in ('ctx_wo','ctx_wd','ctx_ffn_gu','ctx_wqkv')})"
done
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 900 $NCU -f -o gpurun_out/ncu_ctx_res python tools/profile_probes.py ctx_wo ctx_wd > gpurun_out/ncu_ctx_res.log 2>&1; echo "ncu rc=$?"
