mkdir -p gpurun_out
timeout 300 python tools/make_golden_container.py
timeout 900 python -m pytest tests/test_gpu_sequence.py -x -q 2>&1 | tail -15
