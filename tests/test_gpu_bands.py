"""Row-band decode (BASELINE config 5) on one GPU: the frame is
split into n row bands, one handle per band, halo K/V rows pushed between
neighbours after every layer. The bands share device 0 here (the driver's
GPU tiers have one GPU); the exchange kernels are the same P2P stores a
multi-GPU group issues. Checks, against the single-handle codec on the same
weights and inputs:
  * z_hat and the hyper payload are byte-identical;
  * mu / sigma are BITWISE identical (same kernels, same tile anchors);
  * the banded bitstream decodes to the encoder's latents exactly, and its
    rate equals the single-handle rate (same symbols, same tables);
  * a corrupted / truncated container is rejected."""
import numpy as np
import pytest

from oracle_api import gen_weights, preset
from paper_2605_20977_b200 import PswaError
from paper_2605_20977_b200.codec import BandGroupCodec, GpuCodec, band_rows, cfg_from_dict, synth_latent

pytestmark = pytest.mark.gpu

CASES = [  # (paper preset, H, W, bands, P-frame)
    (False, 16, 16, 2, False),
    (False, 16, 20, 4, True),
    (True, 24, 32, 3, True),
    (True, 20, 16, 2, False),
]


@pytest.mark.parametrize("paper,H,W,n,pframe", CASES)
def test_bands_match_single_handle(paper, H, W, n, pframe):
    c = preset(paper, H, W, lanes=32, hyper_lanes=16)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    fidx = 3 if pframe else 0
    frames = [synth_latent(cfg, 0, f) for f in range(fidx + 1)]
    one = GpuCodec(cfg, blob)
    grp = BandGroupCodec(cfg, blob, [0] * n)
    for f in frames[:fidx]:
        one.push_frame(f)
        grp.push_frame(f)
    y = frames[fidx]
    h1, m1, b1 = one.encode_frame(y, fidx=fidx)
    z1 = one.last_zhat()
    hg, mg, bg = grp.encode_frame(y, fidx=fidx)
    zg = grp.last_zhat()
    assert np.array_equal(z1, zg) and h1 == hg
    assert bg[0] == b1[0]
    assert abs(bg[1] - b1[1]) <= 1e-9 * b1[1]
    assert mg[:4] == b"PSWB"
    # mu / sigma bitwise equal to the single-handle forward
    one.reset_gop()
    grp.reset_gop()
    for f in frames[:fidx]:
        one.push_frame(f)
        grp.push_frame(f)
    mu1, sg1, _ = one.forward_params(y, z1, fidx=fidx)
    mug, sgg, _ = grp.forward_params(y, z1, fidx=fidx)
    assert np.array_equal(mu1.view(np.uint32), mug.view(np.uint32))
    assert np.array_equal(sg1.view(np.uint32), sgg.view(np.uint32))
    # banded decode: bit-exact latents
    dec = BandGroupCodec(cfg, blob, [0] * n)
    for f in frames[:fidx]:
        dec.push_frame(f)
    yd, bd = dec.decode_frame(hg, mg, fidx=fidx, advance=False)
    assert np.array_equal(yd, y)
    assert abs(bd[1] - bg[1]) <= 1e-9 * bg[1]
    assert dec.last_launch_count() > 0
    # corrupt container header / truncated band payload
    with pytest.raises(PswaError):
        dec.decode_frame(hg, b"XXXX" + mg[4:], fidx=fidx, advance=False)
    with pytest.raises(PswaError):
        dec.decode_frame(hg, mg[: len(mg) // 2], fidx=fidx, advance=False)


def test_band_gop_sequence():
    """Three frames of a GOP through a 3-band group (ring advances per band)."""
    c = preset(True, 24, 16, lanes=16, hyper_lanes=8)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    enc = BandGroupCodec(cfg, blob, [0, 0, 0])
    dec = BandGroupCodec(cfg, blob, [0, 0, 0])
    for f in range(3):
        y = synth_latent(cfg, 1, f)
        h, m, _ = enc.encode_frame(y, fidx=f)
        yd, _ = dec.decode_frame(h, m, fidx=f)
        assert np.array_equal(yd, y), f


@pytest.mark.parametrize("preset,H,W,n", [("desk", 16, 16, 2), ("paper", 24, 16, 3)])
def test_bands_cross_process(tmp_path, preset, H, W, n):
    """One process per band (torchrun), all on cuda:0 here: the exchange runs
    through CUDA-IPC mappings and device mailbox flags, as across GPUs."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tools", "band_ranks.py"), "--same-device", "--preset", preset,
           "--height", str(H), "--width", str(W), "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.load(open(out))
    assert res["bit_exact"]
