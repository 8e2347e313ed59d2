"""Laplace parameter head (cfg.prior = 1; north_star: "the Gaussian or
Laplace parameter head"). SPEC.md:373-381 and :436-456 define the Gaussian
head; the Laplace family reuses the head (its sigma output is the Laplace
scale b), the 64 scales and the quantisation rule (freq = 1 + floor(p *
65279), deficit to the mode), with p(0) = 1 - exp(-1/(2b)), p(v) =
(exp(-(v-1/2)/b) - exp(-(v+1/2)/b)) / 2 and tail mass exp(-127.5/b) / 2 per
escape. CPU checks: table properties, a float64 restatement, and the
oracle's encode -> wavefront decode round trip."""
import numpy as np
import pytest

from oracle_api import OracleModel, cdf_tables_family, gen_weights, preset, scale_table


def _restated(b: float) -> np.ndarray:
    q = lambda p: 1 + np.floor(max(p, 0.0) * 65279.0)
    f = np.zeros(257)
    f[127] = q(1.0 - np.exp(-0.5 / b))
    for v in range(1, 128):
        p = 0.5 * (np.exp(-(v - 0.5) / b) - np.exp(-(v + 0.5) / b))
        f[127 + v] = f[127 - v] = q(p)
    f[255] = f[256] = q(0.5 * np.exp(-127.5 / b))
    f[127] += 65536 - f.sum()
    return f


def test_laplace_tables_properties_and_restatement():
    lap = cdf_tables_family(1).astype(np.int64)
    gau = cdf_tables_family(0).astype(np.int64)
    sc = scale_table().astype(np.float64)
    for i in range(64):
        c = lap[i]
        assert c[0] == 0 and c[-1] == 65536
        f = np.diff(c)
        assert (f >= 1).all()
        assert np.array_equal(f[:127], f[128:255][::-1])        # symmetric
        assert (np.diff(f[127:255]) <= 0).all()                  # unimodal
        # float64 restatement: equal up to one count where numpy's exp and
        # det::exp round differently across a quantisation step
        assert np.abs(f - _restated(sc[i])).max() <= 1
    # heavier tails than the Gaussian of the same scale
    i = 40  # sigma ~ 5.6
    assert np.diff(lap[i])[127 + 30] > np.diff(gau[i])[127 + 30]


@pytest.mark.parametrize("H,W", [(8, 8), (8, 12)])
def test_laplace_oracle_roundtrip(H, W):
    c = preset(False, H, W, lanes=4, hyper_lanes=2, prior=1)
    blob = gen_weights(c, 1)
    om = OracleModel(c, blob)
    rng = np.random.default_rng(5)
    y = np.rint(rng.laplace(0, 3.0, size=(192, H, W))).astype(np.int32)
    y[7, 2, 3] = 400  # escape path
    hyper, main, bits, z = om.encode(y, fidx=0)
    res = om.decode(hyper, main, fidx=0)
    assert res is not None and np.array_equal(res[0], y)
    assert abs(res[1][1] - bits[1]) <= 1e-9 * bits[1]
    cg = dict(c, prior=0)
    og = OracleModel(cg, blob)
    bits_g = og.encode(y, fidx=0, zhat=z)[2]
    assert bits_g[1] != bits[1] and bits_g[0] == bits[0]  # same hyper, different main family
