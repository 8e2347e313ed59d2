"""4K P-frame (BASELINE config 5): single handle vs n row bands stacked on
one GPU (in-process group), host API end to end (payload H2D and latents D2H
inside the timed region), median of N frames. Checks bit-exactness."""
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2605_20977_b200.codec import BandGroupCodec, GpuCodec, gen_weights, make_cfg, synth_latent  # noqa: E402

H, W = int(os.environ.get("PH", 136)), int(os.environ.get("PW", 240))
NB = int(os.environ.get("NB", 8))
N = int(os.environ.get("PN", 5))
LANES = int(os.environ.get("LANES", 8192))
cfg = make_cfg("paper", H, W, lanes=LANES, hyper_lanes=1024)
cfgb = make_cfg("paper", H, W, lanes=LANES // NB, hyper_lanes=1024)
blob = gen_weights(cfg, 1)
frames = [synth_latent(cfg, 0, f) for f in range(5)]
res = {"grid": [H, W], "bands": NB}


def timed(codec, hyper, main):
    ts = []
    for i in range(N + 2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y, _ = codec.decode_frame(hyper, main, fidx=4, advance=False)
        ts.append(time.perf_counter() - t0)
    assert np.array_equal(y, frames[4])
    return 1e3 * statistics.median(ts[2:])


one = GpuCodec(cfg, blob)
for f in frames[:4]:
    one.push_frame(f)
h, m, _ = one.encode_frame(frames[4], fidx=4)
one.reset_gop()
for f in frames[:4]:
    one.push_frame(f)
res["single_ms"] = timed(one, h, m)
res["single_launches"] = one.last_launch_count()
one.close()
grp = BandGroupCodec(cfgb, blob, [0] * NB)
for f in frames[:4]:
    grp.push_frame(f)
hb, mb, _ = grp.encode_frame(frames[4], fidx=4)
grp.reset_gop()
for f in frames[:4]:
    grp.push_frame(f)
res["banded_ms"] = timed(grp, hb, mb)
res["banded_launches"] = grp.last_launch_count()
res["payload_bytes"] = {"single": len(h) + len(m), "banded": len(hb) + len(mb)}
print(json.dumps(res))
