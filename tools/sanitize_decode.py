"""Workload for compute-sanitizer (tools/sanitize.sh): desk-scale 16x16
encode -> decode of an I-frame and a P-frame, a corrupted and a truncated
payload, forward_params with the mu/sigma + BitStats taps, and the symbol-
level coder ops. Small on purpose: every launch is instrumented."""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2605_20977_b200 import PswaError  # noqa: E402
from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

preset = os.environ.get("SAN_PRESET", "desk")
H, W = int(os.environ.get("SAN_H", 16)), int(os.environ.get("SAN_W", 16))
cfg = make_cfg(preset, H, W, lanes=64, hyper_lanes=16)
blob = gen_weights(cfg, 1)
frames = [synth_latent(cfg, 0, f) for f in range(3)]
enc, dec = GpuCodec(cfg, blob), GpuCodec(cfg, blob)
enc.set_stats(True)
streams = [enc.encode_frame(f, fidx=i) for i, f in enumerate(frames)]
for i, (h, m, _) in enumerate(streams):
    y, _, mu, sg = dec.decode_frame(h, m, fidx=i, params=True)
    assert np.array_equal(y, frames[i])
bs = dec.last_bitstats()
assert abs(bs.sum() - streams[-1][2][1]) < 1e-6 * streams[-1][2][1]
bad = bytearray(streams[0][1])
bad[len(bad) // 2] ^= 0xFF
for payload in (bytes(bad), streams[0][1][:-9]):
    dec.reset_gop()
    try:
        dec.decode_frame(streams[0][0], payload, fidx=0)
    except PswaError:
        pass
z = enc.last_zhat()
fp = GpuCodec(cfg, blob)
fp.push_frame(frames[0])
fp.push_frame(frames[1])
fp.forward_params(frames[2], z, fidx=2)
print("sanitize workload done")
