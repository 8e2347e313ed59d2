mkdir -p gpurun_out
PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py 2>&1 | grep -v Warn | grep -E "warm|decode_phase"
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -2 gpurun_out/pytest_gpu.log
