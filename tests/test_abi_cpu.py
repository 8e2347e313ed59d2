"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host logic (weights, synthetic inputs) matches the
oracle's independent restatement byte for byte. No GPU calls here."""
import re
import os

import numpy as np
import pytest

from oracle_api import gen_weights as oracle_gen_weights, preset
from paper_2605_20977_b200 import _lib
from paper_2605_20977_b200.codec import cfg_from_dict, gen_weights, make_cfg, synth_latent

HEADER = os.path.join(os.path.dirname(__file__), "..", "include", "pswa", "pswa_cuda.h")


def test_library_exports_every_declared_symbol():
    decl = re.findall(r"\b(pswa_[a-z0-9_]+)\s*\(", open(HEADER).read())
    names = sorted(set(decl))
    assert len(names) >= 18
    L = _lib.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


@pytest.mark.parametrize("paper,H,W", [(False, 16, 16), (False, 6, 10), (True, 16, 16)])
def test_product_weights_match_oracle_bytes(paper, H, W):
    c = preset(paper, H, W)
    a = gen_weights(cfg_from_dict(c), 1)
    b = oracle_gen_weights(c, 1)
    assert a == b


def test_cfg_preset_matches_python_preset():
    for paper in (True, False):
        cfg = make_cfg("paper" if paper else "desk", 68, 120)
        ref = preset(paper, 68, 120)
        assert cfg.as_dict() == ref


def test_synth_latent_deterministic_and_shaped():
    cfg = make_cfg("desk", 16, 24)
    a = synth_latent(cfg, 0, 0)
    b = synth_latent(cfg, 0, 0)
    c = synth_latent(cfg, 0, 1)
    assert a.shape == (192, 16, 24) and np.array_equal(a, b)
    assert not np.array_equal(a, c)
    # coarse-to-fine channel groups: b_g = 8, 4, 2, 1
    spread = [np.abs(a[48 * g:48 * (g + 1)]).mean() for g in range(4)]
    assert spread[0] > spread[1] > spread[2] > spread[3]
    big = make_cfg("desk", 68, 120)
    n = sum(int((np.abs(synth_latent(big, g, 0)) == 300).sum()) for g in range(8))
    assert n >= 1  # ~1 forced escape per 10^4 positions (8 x 8160 positions here)


def test_bad_config_rejected():
    from paper_2605_20977_b200 import PswaError
    cfg = make_cfg("desk", 16, 16, win_h=6)
    with pytest.raises(PswaError):
        gen_weights(cfg, 1)


@pytest.mark.parametrize("H,n", [(68, 1), (68, 2), (136, 8), (16, 4), (17, 2), (120, 7)])
def test_band_rows_partition(H, n):
    """Row bands tile the grid, start at multiples of 4 (the hyperprior and
    the s = 4 wavefront pattern) and hold >= 3 rows (the 7x7 halo)."""
    from paper_2605_20977_b200.codec import band_rows
    rows = [band_rows(H, n, b) for b in range(n)]
    assert rows[0][0] == 0 and rows[-1][1] == H
    for (a0, a1), (b0, _) in zip(rows, rows[1:]):
        assert a1 == b0
    for r0, r1 in rows:
        assert r0 % 4 == 0 and r1 - r0 >= 3


def test_band_rows_rejects_too_many_bands():
    from paper_2605_20977_b200 import PswaError
    from paper_2605_20977_b200.codec import band_rows
    with pytest.raises(PswaError):
        band_rows(16, 5, 0)


@pytest.mark.parametrize("paper,H,W", [(False, 8, 12), (True, 16, 16)])
def test_synth_gop_matches_oracle_and_per_frame(paper, H, W):
    """The product's and the oracle's synthetic-input generators are the same
    sequence (the reference arm of bench.py uses the oracle's)."""
    from oracle_api import synth_gop as oracle_synth_gop
    from paper_2605_20977_b200.codec import synth_gop
    c = preset(paper, H, W)
    a = synth_gop(cfg_from_dict(c), 3, 5)
    assert np.array_equal(a, oracle_synth_gop(c, 3, 5))
    for f in range(5):
        assert np.array_equal(a[f], synth_latent(cfg_from_dict(c), 3, f))
