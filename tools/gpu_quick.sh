mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bands.py -x -q > gpurun_out/pytest_bands.log 2>&1; echo "bands rc=$?"
tail -30 gpurun_out/pytest_bands.log
timeout 900 python tools/bench_bands.py > gpurun_out/bench_bands.json 2> gpurun_out/bench_bands.err; echo "bb rc=$?"
cat gpurun_out/bench_bands.json; tail -5 gpurun_out/bench_bands.err
