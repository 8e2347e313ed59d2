"""Warm, in-graph per-kernel GPU times (run with PSWA_NO_PDL=1: with PDL a
kernel's duration includes its wait on the predecessor) of the bench decode (CUPTI via the
torch profiler): N decodes of the 1080p paper-scale P-frame, aggregated by
kernel. Unlike an ncu launch list these are not serialised or cold-cache.
PK=encode profiles the teacher-forced encode of the same frame instead."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

N = int(os.environ.get("PN", 5))
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
for _ in range(3):
    y, _ = dec.decode_frame(hyper, main, fidx=4, advance=False)
assert np.array_equal(y, frames[4])
torch.cuda.synchronize()
MODE = os.environ.get("PK", "decode")
if MODE == "encode":
    enc = GpuCodec(cfg, blob)
    for f in frames[:4]:
        enc.push_frame(f)
    for _ in range(2):
        enc.encode_frame(frames[4], fidx=4)
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(N):
        if MODE == "encode":
            enc.encode_frame(frames[4], fidx=4)
        else:
            dec.decode_frame(hyper, main, fidx=4, advance=False)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type.name != "CUDA":
        continue
    name = ev.name
    if "gemm_tc_kernel" in name:
        name = "gemm_tc_kernel<" + name.split("gemm_tc_kernel<")[1].split(">")[0] + ">"
    else:
        base = name.replace("(anonymous namespace)::", "").replace("void ", "")
        name = base.split("(")[0].split("::")[-1][:40] or base[:40]
    agg[name][0] += 1
    agg[name][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values()) / N
lines = [f"warm in-graph kernel time per frame ({MODE}): {tot/1e3:.3f} ms (sum of kernel durations)"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{t/N/1e3:8.3f} ms {100*t/N/tot:5.1f}%  n={n//N:4d}  avg={t/n:7.1f} us  {k}")
print("\n".join(lines))
os.makedirs("gpurun_out", exist_ok=True)
open("gpurun_out/kernel_times.txt", "w").write("\n".join(lines) + "\n")
