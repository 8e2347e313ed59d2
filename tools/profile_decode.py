"""Set up the 1080p paper-scale P-frame decode (bench workload) and run N
decodes inside cudaProfilerStart/Stop, for `ncu --profile-from-start off`."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

H, W = int(os.environ.get("PH", 68)), int(os.environ.get("PW", 120))
N = int(os.environ.get("PN", 1))
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
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(N):
    dec.decode_frame(hyper, main, fidx=4, advance=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", N, "decodes; launches/frame", dec.last_launch_count())
