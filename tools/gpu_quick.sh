mkdir -p gpurun_out
PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py 2>&1 | grep -v Warn | grep -E "warm|decode_phase"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print(d['ms_per_frame'], d['e2e']['ms_per_frame'], d['gpu_launches'])"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -3 gpurun_out/pytest_gpu.log
