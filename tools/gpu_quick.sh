mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print(d['ms_per_frame'], d['e2e']['ms_per_frame'], d['config2_iframe_1gpu'])"
