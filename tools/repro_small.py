"""Small paper-scale encode/decode round trip (debug / sanitizer runs)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

H, W = int(os.environ.get("PH", 16)), int(os.environ.get("PW", 16))
cfg = make_cfg("paper", H, W, lanes=32, hyper_lanes=16)
blob = gen_weights(cfg, 1)
y = synth_latent(cfg, 0, 0)
g = GpuCodec(cfg, blob)
h, m, _ = g.encode_frame(y, fidx=0)
g.reset_gop()
yd, _ = g.decode_frame(h, m, fidx=0)
print("exact", np.array_equal(yd, y))
