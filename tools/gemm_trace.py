"""Per-CTA phase timeline of one production GEMM launch (PSWA_GEMM_TRACE).

Needs the trace build: make -C paper_2605_20977_b200 clean all TRACE=1
(rebuild without TRACE afterwards).

Decodes the bench frame once, replays a probed op (default step_wq and
ctx_ffn_gu) and prints, over the CTAs, the clock64 offsets from kernel entry
of: setup done, pdl_wait done, first TMA stage landed (MMA warp), all TMA
issued, last MMA committed, accumulator ready (epilogue), epilogue done,
exit; plus the spread of CTA start times (globaltimer)."""
import ctypes as C
import os
import sys

os.environ["PSWA_GEMM_TRACE"] = "1"
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2605_20977_b200 import lib  # noqa: E402
from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

cfg = make_cfg("paper", 68, 120, lanes=8192, hyper_lanes=1024)
blob = gen_weights(cfg, 1)
frames = [synth_latent(cfg, 0, f) for f in range(5)]
enc = GpuCodec(cfg, blob)
for f in frames[:4]:
    enc.push_frame(f)
hyper, main, _ = enc.encode_frame(frames[4], fidx=4)
enc.close()
dec = GpuCodec(cfg, blob)
for f in frames[:4]:
    dec.push_frame(f)
y, _ = dec.decode_frame(hyper, main, fidx=4, advance=False)
assert np.array_equal(y, frames[4])
# GEMM_EXP=1: replays without MMAs, 2: without operand loads (timing only)
EXP = int(os.environ.get("GEMM_EXP", "0"))
lib().pswa_debug_gemm_experiment(EXP)
SLOTS = 16
names = {1: "setup", 2: "pdl_wait", 10: "tma_issued", 3: "first_stage", 4: "mma_done",
         13: "epi_inputs", 5: "acc_ready", 11: "chunk0_ld", 12: "chunk0_done", 6: "epi_done",
         7: "exit"}
for op in sys.argv[1:] or ["step_wq", "ctx_ffn_gu"]:
    buf = np.zeros(SLOTS * 1024, np.uint64)
    lib().pswa_debug_gemm_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)  # clears
    us, _ = dec.bench_op(op, 5)
    lib().pswa_debug_gemm_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), buf.size)
    t = buf.reshape(1024, SLOTS).astype(np.int64)
    ctas = t[t[:, 8] != 0]
    g0 = ctas[:, 8].min()
    print(f"{op}: {len(ctas)} CTAs, bench {us:.2f} us/launch; start spread "
          f"{(ctas[:, 8].max() - g0) / 1e3:.2f} us, last exit {(ctas[:, 9].max() - g0) / 1e3:.2f} us")
    for k in (1, 2, 10, 3, 4, 13, 5, 11, 12, 6, 7):
        d = ctas[:, k] - ctas[:, 0]
        d = d[ctas[:, k] != 0]
        if len(d):
            print(f"  {names[k]:12s} cycles from entry: min {d.min():7d} med {int(np.median(d)):7d} max {d.max():7d}")
