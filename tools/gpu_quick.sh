mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -5 gpurun_out/pytest_gpu.log
python -c "
import json; d=json.load(open('gpurun_out/parity.json'))
for k,v in d.items():
  if 'laplace' in k: print(k, {a:v[a] for a in ('mu_max_abs','sigma_max_rel','rate_rel_err','frac_within_tol') if a in v})"
