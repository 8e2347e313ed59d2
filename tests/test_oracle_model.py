"""Oracle model-level properties (SPEC.md acceptance 1-3, 7): master decode
oracle, exact s*N phase count, causality by exhaustive perturbation, GOP
restart and corruption handling."""
import numpy as np
import pytest

from oracle_api import OracleModel, gen_weights, preset


def laplace_yhat(rng, C, H, W, N=4):
    b = np.repeat(np.array([8.0, 4.0, 2.0, 1.0][:N]), C // N)
    y = rng.laplace(0, b[:, None, None], size=(C, H, W))
    return np.rint(y).astype(np.int32)


def small_cfg(H, W, **over):
    c = preset(False, H, W, lanes=3, hyper_lanes=2)
    c.update(over)
    return c


_models = {}


def model(cfg, seed=1):
    key = (tuple(sorted(cfg.items())), seed)
    if key not in _models:
        _models[key] = OracleModel(cfg, gen_weights(cfg, seed))
    return _models[key]


@pytest.mark.parametrize("H,W,rate,npast", [(4, 4, 0, 0), (8, 4, 2, 1), (8, 8, 3, 4)])
def test_master_oracle_small(H, W, rate, npast):
    """encoder y_hat == serial y_hat == wavefront y_hat."""
    cfg = small_cfg(H, W)
    m = model(cfg)
    rng = np.random.default_rng(H * 31 + W + rate)
    past = [laplace_yhat(rng, 192, H, W) for _ in range(npast)]
    y = laplace_yhat(rng, 192, H, W)
    y[5, 1, 2] = 300  # escape path
    hyper, main, bits, z = m.encode(y, rate=rate, fidx=npast, past=past)
    yw, bw, ph = m.decode(hyper, main, rate=rate, fidx=npast, past=past)
    assert np.array_equal(yw, y)
    assert ph == 16  # s*N phases at every resolution
    assert np.allclose(bw, bits, rtol=0, atol=1e-6)
    if H * W <= 32:
        ys, bs, phs = m.decode(hyper, main, rate=rate, fidx=npast, past=past, serial=True)
        assert np.array_equal(ys, y)
        assert phs == H * W * 4  # raster reference: H*W*N sequential steps


@pytest.mark.parametrize("s,N", [(1, 1), (2, 2), (4, 2), (2, 4)])
def test_master_oracle_schedules(s, N):
    """Other (s, N) schedules: s*N phases, exact round trip."""
    cfg = small_cfg(8, 8, s=s, n_groups=N)
    m = model(cfg)
    rng = np.random.default_rng(s * 10 + N)
    y = laplace_yhat(rng, 192, 8, 8, N=min(N, 4)) if N <= 4 else None
    hyper, main, bits, z = m.encode(y, rate=1, fidx=0)
    yw, bw, ph = m.decode(hyper, main, rate=1, fidx=0)
    assert np.array_equal(yw, y) and ph == s * N


def test_causality_exhaustive_6x6():
    """(mu, sigma) at (p, g) is invariant to y_hat at steps >= step(p) elsewhere,
    to groups >= g at p, and to future frames; C=8."""
    H = W = 6
    cfg = small_cfg(H, W, latent_ch=8)
    m = model(cfg)
    rng = np.random.default_rng(5)
    base = laplace_yhat(rng, 8, H, W)
    past = [laplace_yhat(rng, 8, H, W)]
    mu0, sg0, z0 = m.forward(base, past=past)
    step = (np.arange(H)[:, None] + np.arange(W)[None, :]) % 4
    for py in range(H):
        for px in range(W):
            y2 = base.copy()
            y2[:, py, px] += 7  # perturb every channel at one position
            mu, sg, _ = m.forward(y2, past=past, zhat=z0)
            changed = (mu != mu0) | (sg != sg0)  # [C][H][W]
            sp = step[py, px]
            for qy in range(H):
                for qx in range(W):
                    if (qy, qx) == (py, px):
                        # groups at p: group g sees only groups < g at p
                        assert not changed[0:2, qy, qx].any()
                    elif step[qy, qx] <= sp:
                        assert not changed[:, qy, qx].any(), (py, px, qy, qx)
            # a strictly-later step in the window must react (Fig. 2b semantics)
    # group-level perturbation at p: groups >= g untouched
    for g in range(4):
        y2 = base.copy()
        y2[2 * g:2 * g + 2, 3, 3] += 5
        mu, sg, _ = m.forward(y2, past=past, zhat=z0)
        ch = (mu != mu0) | (sg != sg0)
        assert not ch[: 2 * (g + 1), 3, 3].any()
        if g < 3:
            assert ch[2 * (g + 1):, 3, 3].any()


def test_same_step_sensitivity_pair():
    """S1 self-attention is unmasked for same-step keys, the accumulator masks
    them (Fig. 2b): changing a same-step neighbour's y_hat leaves (mu, sigma)
    at p unchanged, changing a strictly-earlier neighbour changes them."""
    H = W = 8
    cfg = small_cfg(H, W, latent_ch=8)
    m = model(cfg)
    rng = np.random.default_rng(6)
    y = laplace_yhat(rng, 8, H, W)
    mu0, sg0, z0 = m.forward(y)
    # p = (4,4): step 0. earlier-step neighbour of q=(4,5) (step 1) is p.
    y2 = y.copy()
    y2[:, 4, 4] += 9
    mu, sg, _ = m.forward(y2, zhat=z0)
    assert (mu[:, 4, 5] != mu0[:, 4, 5]).any()     # strictly past -> visible
    assert (mu[:, 3, 5] == mu0[:, 3, 5]).all()     # (3,5) is step 0: same step -> invisible


def test_temporal_causality_and_gop_reset():
    H = W = 8
    cfg = small_cfg(H, W, latent_ch=8)
    m = model(cfg)
    rng = np.random.default_rng(7)
    frames = [laplace_yhat(rng, 8, H, W) for _ in range(3)]
    mu_a, sg_a, z = m.forward(frames[2], past=frames[:2])
    f1 = frames[1].copy()
    f1 += 3
    mu_b, _, _ = m.forward(frames[2], past=[frames[0], f1], zhat=z)
    assert (mu_a != mu_b).any()  # past frames matter
    # I-frame: no past -> learned pad only; identical regardless of history
    mu_i1, _, zi = m.forward(frames[0], past=[])
    mu_i2, _, _ = m.forward(frames[0], past=[], zhat=zi)
    assert np.array_equal(mu_i1, mu_i2)


def test_corrupt_payload_detected_or_changes_output():
    """Tampering with a main-payload byte changes some symbol or raises
    truncation; truncation is always detected."""
    H = W = 8
    cfg = small_cfg(H, W)
    m = model(cfg)
    rng = np.random.default_rng(8)
    y = laplace_yhat(rng, 192, H, W)
    hyper, main, _, _ = m.encode(y)
    bad = bytearray(main)
    bad[len(bad) // 2] ^= 0x5A
    r = m.decode(hyper, bytes(bad))
    assert r is None or not np.array_equal(r[0], y)
    assert m.decode(hyper, main[:-7]) is None


def test_weights_deterministic_and_validated():
    cfg = small_cfg(4, 4)
    a, b = gen_weights(cfg, 1), gen_weights(cfg, 1)
    assert a == b and gen_weights(cfg, 2) != a
    with pytest.raises(RuntimeError):
        OracleModel(cfg, a[:-10])
    other = dict(cfg, d_spatial=32)
    with pytest.raises(RuntimeError):
        OracleModel(other, a)
