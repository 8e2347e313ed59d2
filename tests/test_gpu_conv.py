"""The hyper decoder's implicit-GEMM convolutions (tcgen05 GEMM whose A
tiles are gathered from the fp16 NHWC image by TMA in im2col mode,
gemm_plan_conv3x3) against the materialised patch-matrix path
(PSWA_CONV_IM2COL_MATERIALISE=1): the hyper decoder output Hq and the
entropy parameters are bitwise equal -- same fp16 operands, same K order.
Each path runs in its own process (the switch is read once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from oracle_api import gen_weights, preset
from paper_2605_20977_b200.codec import GpuCodec, cfg_from_dict, synth_latent
c = preset(True, {H}, {W}, lanes=64, hyper_lanes=16)
cfg = cfg_from_dict(c); blob = gen_weights(c, 1)
y = synth_latent(cfg, 0, 0)
g = GpuCodec(cfg, blob)
rng = np.random.default_rng(7)
z = rng.integers(-6, 7, size=g.zshape).astype(np.int32)
mu, sg, _ = g.forward_params(y, z, fidx=0)
np.savez({out!r}, hq=g.debug_fetch("hq"), mu=mu, sg=sg)
print("ok")
"""


def run(env_extra, out, H, W):
    env = dict(os.environ, **env_extra)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), out=out, H=H, W=W)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    return np.load(out)


@pytest.mark.parametrize("H,W", [(16, 16), (68, 120), (20, 28)])
def test_implicit_conv_matches_patch_matrix(H, W, tmp_path):
    a = run({}, str(tmp_path / "implicit.npz"), H, W)
    b = run({"PSWA_CONV_IM2COL_MATERIALISE": "1"}, str(tmp_path / "patches.npz"), H, W)
    for k in ("hq", "mu", "sg"):
        assert np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32)), k
