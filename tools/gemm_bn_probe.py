"""Per-launch time of the 2040-row step gate|up GEMM (SwiGLU epilogue) at
BN = 256 (176 tiles over 148 SMs) vs BN = 352 (128 tiles, one wave), and of
the other tile widths the planner picks between, in CUDA graphs of 50
back-to-back launches (op ABI, CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2605_20977_b200 import lib  # noqa: E402

L = lib()
for (M, N, K, act, bns) in [(2040, 2816, 512, 2, (256, 352, 128)), (1664, 2816, 512, 2, (256,)),
                            (2040, 1408, 512, 0, (64, 352)), (8160, 2816, 512, 2, (256, 352)),
                            (2040, 1536, 512, 0, (256, 192, 128)), (2040, 1408, 256, 2, (128, 352, 64))]:
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    ncol = N // 2 if act == 2 else N
    for bn in bns:
        c = torch.zeros(M, ncol, device="cuda", dtype=torch.float16)
        s = torch.cuda.Stream()

        def go():
            rc = L.pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), ncol, 0, 0,
                                        None, None, act, bn, s.cuda_stream)
            assert rc == 0
        with torch.cuda.stream(s):
            go()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                go()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.replay()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) / 200 * 1e3
        print(json.dumps({"M": M, "N": N, "K": K, "act": act, "bn": bn, "us": round(us, 2),
                          "tflops": round(2 * M * N * K / us / 1e6, 1)}), flush=True)
