"""Decode the bench frame once, then time the probed production launches
(pswa_gpu_bench_op) and print one JSON line; used for launch-policy sweeps
(PSWA_ATTN_* env overrides are read once per process)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
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
import time
import torch
ts = []
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dec.decode_frame(hyper, main, fidx=4, advance=False)
    ts.append(time.perf_counter() - t0)
res = {k: v for k, v in os.environ.items() if k.startswith("PSWA_")}
res["frame_ms_host"] = 1e3 * sorted(ts)[2]
for name in ("ctx_attn", "step_attn", "ctx_ffn_gu", "step_wq"):
    us, fl = dec.bench_op(name, 30)
    res[name] = round(us, 2)
print(json.dumps(res))
