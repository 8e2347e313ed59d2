mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/pytest_bands.log 2>&1; echo "bands rc=$?"
tail -30 gpurun_out/pytest_bands.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu rc=$?"
tail -5 gpurun_out/pytest_gpu.log
