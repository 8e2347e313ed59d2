mkdir -p gpurun_out
timeout 300 python tools/probe_ops.py 2>&1 | tail -1
PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py 2>&1 | grep -v Warn | head -14
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -3 gpurun_out/pytest_gpu.log
