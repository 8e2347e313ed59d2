"""Writes the golden sequence container (FORMAT.md §5) into gpurun_out/:
3 synthetic desk-preset frames (8x8 latent grid, GOP 2, 8 lanes) coded by
the GPU encoder, plus the latents. Run on a B200, then copy to tests/golden/."""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

cfg = make_cfg("desk", 8, 8, lanes=8, hyper_lanes=4)
blob = gen_weights(cfg, 1)
frames = np.stack([synth_latent(cfg, 3, f) for f in range(3)])
enc = GpuCodec(cfg, blob)
cont = enc.encode_sequence(frames, gop=2, rate=1)
dec = GpuCodec(cfg, blob)
y, st, _ = dec.decode_sequence(cont)
assert np.array_equal(y, frames) and (st == 0).all()
out = os.path.join(ROOT, "gpurun_out")
os.makedirs(out, exist_ok=True)
open(os.path.join(out, "seq_desk_8x8.pswa"), "wb").write(cont)
np.save(os.path.join(out, "seq_desk_8x8_frames.npy"), frames)
print("golden container", len(cont), "bytes")
