"""Bench probes under ncu: sets up the bench workload (1080p paper-scale
P-frame at GOP index 4, tools/profile_decode.py), decodes it, then replays
each named probe (pswa_gpu_bench_probe, the launches bench.py times for its
kernel rooflines) ONCE inside cudaProfilerStart/Stop. With
`ncu --profile-from-start off` the report holds exactly those launches, in
the order written to gpurun_out/probe_order.json ([name, launches] pairs),
so tools/ncu_traffic.py can attribute every row to its probe.

usage: python tools/profile_probes.py [probe ...]   (default: every probe)"""
import json
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

H, W = int(os.environ.get("PH", 68)), int(os.environ.get("PW", 120))
cfg = make_cfg(os.environ.get("PRESET", "paper"), H, W, lanes=8192, hyper_lanes=1024)
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
for _ in range(2):
    y, _ = dec.decode_frame(hyper, main, fidx=4, advance=False)
assert np.array_equal(y, frames[4])
probes = dec.probes()
# gemm_all replays ~380 launches: too many for --set full (its members are
# captured as the individual GEMM probes)
names = sys.argv[1:] or sorted(n for n in probes if n != "gemm_all")
order = []
for name in names:
    dec.bench_probe(name, 3)  # warm
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    dec.bench_probe(name, 0)  # exactly one replay
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    order.append([name, probes[name][2], probes[name][0], probes[name][1]])
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(order, open(os.path.join(ROOT, "gpurun_out", "probe_order.json"), "w"), indent=0)
print("profiled", len(order), "probes:", " ".join(n for n, *_ in order))
