mkdir -p gpurun_out
timeout 300 python tools/make_golden_container.py
