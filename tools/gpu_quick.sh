mkdir -p gpurun_out
timeout 300 python tools/probe_ops.py 2>&1 | tail -1
PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py 2>&1 | grep -E "warm|window"
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_bands.py -x -q 2>&1 | tail -2
