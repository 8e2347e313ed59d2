"""Standalone tcgen05 GEMM timings over shapes (op ABI, CUDA events, 50
back-to-back launches): separates the per-launch latency floor of the small
step-batch GEMMs from their work."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2605_20977_b200 import lib  # noqa: E402

L = lib()
res = []
for (M, N, K, f32) in [(128, 64, 64, 0), (2040, 512, 512, 0), (2040, 512, 512, 1), (2040, 512, 1408, 1),
                       (4080, 512, 512, 0), (8160, 512, 512, 0), (2040, 2816, 512, 0), (2040, 256, 1024, 1),
                       (32640, 512, 512, 1), (32640, 2816, 512, 0)]:
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    c = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.float16)
    s = torch.cuda.Stream()
    def go():
        rc = L.pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), N, f32,
                                    f32, None, None, 0, 0, s.cuda_stream)
        assert rc == 0
    with torch.cuda.stream(s):
        go()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # replayed: no host launch cost in the timing
    with torch.cuda.graph(g, stream=s):
        for _ in range(50):
            go()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    res.append({"M": M, "N": N, "K": K, "f32_acc": f32, "us": round(us, 2),
                "tflops": round(2 * M * N * K / us / 1e6, 1)})
    print(json.dumps(res[-1]), flush=True)
