"""Parity triage: per-stage GPU vs oracle error for one frame (test tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle_api import OracleModel, gen_weights, preset  # noqa: E402
from paper_2605_20977_b200.codec import GpuCodec, cfg_from_dict  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-12)), float(np.abs(a - b).mean() / (np.abs(b).mean() + 1e-12))


def main(paper, H, W, npast):
    c = preset(paper, H, W, lanes=16, hyper_lanes=4)
    blob = gen_weights(c, 1)
    om = OracleModel(c, blob)
    g = GpuCodec(cfg_from_dict(c), blob)
    rng = np.random.default_rng(0)
    b = np.repeat(np.array([8.0, 4.0, 2.0, 1.0]), 48)
    frames = [np.rint(rng.laplace(0, b[:, None, None], size=(192, H, W))).astype(np.int32)
              for _ in range(npast + 1)]
    for f in frames[:-1]:
        g.push_frame(f)
    y = frames[-1]
    _, _, z = om.forward(y, past=frames[:-1])
    mu_g, sg_g, _ = g.forward_params(y, z, fidx=npast)
    st = om.forward_debug(y, z, past=frames[:-1])
    mu_o, sg_o, _ = om.forward(y, past=frames[:-1], zhat=z)
    out = [f"paper={paper} {H}x{W} npast={npast}"]
    for name in ("ctx", "hq", "s1", "a", "s2"):
        gv = g.debug_fetch(name)
        if name == "s1":
            Hp, Wp = (H + 3) // 4 * 4, (W + 3) // 4 * 4
            gv = gv.reshape(Hp, Wp, -1)[:H, :W].reshape(H * W, -1)
        out.append(f"  {name:4s} max_rel={rel(gv, st[name])[0]:.3e} mean_rel={rel(gv, st[name])[1]:.3e}")
    out.append(f"  mu   max_abs={np.abs(mu_g-mu_o).max():.3e} mean_abs={np.abs(mu_g-mu_o).mean():.3e}")
    out.append(f"  sig  max_rel={(np.abs(sg_g-sg_o)/sg_o).max():.3e} mean_rel={(np.abs(sg_g-sg_o)/sg_o).mean():.3e}")
    # per group
    for gi in range(4):
        sl = slice(48 * gi, 48 * gi + 48)
        out.append(f"  group {gi}: mu mean_abs={np.abs(mu_g[sl]-mu_o[sl]).mean():.3e} sig mean_rel={(np.abs(sg_g[sl]-sg_o[sl])/sg_o[sl]).mean():.3e}")
    txt = "\n".join(out)
    print(txt, flush=True)
    return txt


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    res = [main(False, 16, 16, 0), main(False, 16, 16, 2), main(True, 16, 16, 0)]
    open("gpurun_out/triage.txt", "w").write("\n".join(res))
