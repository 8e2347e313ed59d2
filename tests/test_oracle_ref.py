"""Pin the oracle's numerics floor to the reference's OWN code, bit for bit.

oracle/_ref/libpswa_ref.so is compiled from the unmodified reference sources
(proj/src/det_math.cpp, tensor.cpp, threading.cpp; recipe in oracle/Makefile).
Every primitive the oracle restates is compared on random inputs with exact
(bitwise) equality.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_api import oracle, ref, ptr

pytestmark = pytest.mark.skipif(ref() is None, reason="oracle/_ref not built (no reference tree)")


def _bits(a):
    return np.asarray(a).view(np.uint32 if np.asarray(a).dtype == np.float32 else np.uint64)


def test_det_fp64_bitwise():
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-750, 750, 4000), rng.uniform(-5, 5, 4000),
                         rng.uniform(1e-300, 10, 2000), [0.0, -0.0, 1e-310, 709.78, -745.13]])
    for fn in range(4):  # exp, log, erf, normal_cdf
        for x in xs:
            if fn == 1 and x < 0:
                continue
            a, b = oracle().oracle_det(fn, float(x)), ref().ref_det(fn, float(x))
            assert np.float64(a).view(np.uint64) == np.float64(b).view(np.uint64) or (
                np.isnan(a) and np.isnan(b)), (fn, x, a, b)


def test_det_f32_bitwise():
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.uniform(-40, 40, 6000), rng.normal(0, 2, 4000)]).astype(np.float32)
    for fn in range(4):  # exp_f32, silu_f32, tanh_f32, softplus_f32
        for x in xs:
            a, b = oracle().oracle_det_f32(fn, float(x)), ref().ref_det_f32(fn, float(x))
            assert np.float32(a).view(np.uint32) == np.float32(b).view(np.uint32), (fn, x)


def test_rng_and_fnv_bitwise():
    for seed in (0, 1, 12345, 2**63 + 7):
        n = 1000
        o = [np.zeros(n, np.uint64), np.zeros(n, np.float32), np.zeros(n, np.float32)]
        r = [np.zeros(n, np.uint64), np.zeros(n, np.float32), np.zeros(n, np.float32)]
        oracle().oracle_rng(seed, n, *[ptr(a) for a in o])
        ref().ref_rng(seed, n, *[ptr(a) for a in r])
        for a, b in zip(o, r):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    for s in (b"", b"embed.w", b"ctx.b0.wq", bytes(range(256))):
        buf = (C.c_uint8 * max(1, len(s))).from_buffer_copy(s or b"\0")
        assert oracle().oracle_fnv1a(buf, len(s)) == ref().ref_fnv1a(buf, len(s))


def test_init_tensor_bitwise():
    for kind, fan in ((0, 1), (0, 512), (0, 1368), (1, 7), (2, 3)):
        n = 4096
        a, b = np.zeros(n, np.float32), np.zeros(n, np.float32)
        oracle().oracle_init_values(99 + fan, ptr(a), n, kind, fan)
        ref().ref_init_tensor(99 + fan, ptr(b), n, kind, fan)
        assert np.array_equal(_bits(a), _bits(b))


@pytest.mark.parametrize("m,k,p", [(1, 1, 1), (5, 4, 3), (17, 64, 33), (64, 512, 96),
                                   (40, 1368, 70)])
def test_matmul_bitwise(m, k, p):
    rng = np.random.default_rng(m * k * p)
    a = rng.normal(size=(m, k)).astype(np.float32)
    b = rng.normal(size=(k, p)).astype(np.float32)
    c1, c2 = np.zeros((m, p), np.float32), np.zeros((m, p), np.float32)
    oracle().oracle_matmul(ptr(a), ptr(b), ptr(c1), m, k, p)
    ref().ref_matmul(ptr(a), ptr(b), ptr(c2), m, k, p)
    assert np.array_equal(_bits(c1), _bits(c2))


def test_matmul_worker_invariance():
    rng = np.random.default_rng(3)
    a = rng.normal(size=(300, 96)).astype(np.float32)
    b = rng.normal(size=(96, 200)).astype(np.float32)
    outs = []
    for w in (1, 4, 8):
        oracle().oracle_set_threads(w)
        c = np.zeros((300, 200), np.float32)
        oracle().oracle_matmul(ptr(a), ptr(b), ptr(c), 300, 96, 200)
        outs.append(c)
    oracle().oracle_set_threads(1)
    assert all(np.array_equal(_bits(outs[0]), _bits(o)) for o in outs[1:])


def test_softmax_bitwise():
    rng = np.random.default_rng(4)
    sentinel = np.finfo(np.float32).min
    x = rng.normal(0, 3, size=(200, 49)).astype(np.float32)
    x[rng.random(x.shape) < 0.3] = sentinel
    x[7, :] = sentinel  # fully masked row
    y2 = np.zeros_like(x)
    ref().ref_softmax_rows(ptr(x), ptr(y2), 200, 49)
    y1 = x.copy()
    for i in range(200):
        oracle().oracle_softmax_row(y1[i].ctypes.data_as(C.c_void_p), 49)
    assert np.array_equal(_bits(y1), _bits(y2))
    assert not y1[7].any()


def test_rmsnorm_and_ffn_hidden_bitwise():
    rng = np.random.default_rng(5)
    for d in (1, 8, 64, 256, 512):
        x = rng.normal(0, 4, d).astype(np.float32)
        g = rng.normal(1, 0.1, d).astype(np.float32)
        a, b = np.zeros(d, np.float32), np.zeros(d, np.float32)
        oracle().oracle_rmsnorm(ptr(x), ptr(g), d, ptr(a))
        ref().ref_rmsnorm(ptr(x), ptr(g), d, ptr(b))
        assert np.array_equal(_bits(a), _bits(b))
    for d in (1, 2, 3, 32, 64, 128, 256, 512, 1024):
        assert oracle().oracle_ffn_hidden(d) == ref().ref_ffn_hidden_dim(d)


def test_swiglu_matches_reference_per_token():
    """The oracle computes SwiGLU as batched matmuls; per token this must equal
    the reference's swiglu_ffn (tensor.cpp:94-116) bit for bit."""
    rng = np.random.default_rng(6)
    d, f = 64, 168
    x = rng.normal(size=d).astype(np.float32)
    wg, wu = (rng.normal(0, 0.1, (d, f)).astype(np.float32) for _ in range(2))
    wd = rng.normal(0, 0.1, (f, d)).astype(np.float32)
    out_ref = np.zeros(d, np.float32)
    ref().ref_swiglu_ffn(ptr(x), ptr(wg), ptr(wu), ptr(wd), d, f, ptr(out_ref))
    g, u = np.zeros((1, f), np.float32), np.zeros((1, f), np.float32)
    oracle().oracle_matmul(ptr(x), ptr(wg), ptr(g), 1, d, f)
    oracle().oracle_matmul(ptr(x), ptr(wu), ptr(u), 1, d, f)
    h = np.array([oracle().oracle_det_f32(1, float(v)) for v in g[0]], np.float32) * u[0]
    out = np.zeros((1, d), np.float32)
    oracle().oracle_matmul(ptr(h.astype(np.float32)), ptr(wd), ptr(out), 1, f, d)
    assert np.array_equal(_bits(out[0]), _bits(out_ref))


@pytest.mark.parametrize("c,h,w,o,k,stride", [(3, 5, 6, 2, 3, 1), (8, 8, 8, 4, 3, 2),
                                               (4, 7, 9, 5, 1, 1)])
def test_conv2d_upsample_bitwise(c, h, w, o, k, stride):
    rng = np.random.default_rng(c * h * w)
    x = rng.normal(size=(c, h, w)).astype(np.float32)
    kk = rng.normal(size=(o, c, k, k)).astype(np.float32)
    y1 = np.zeros((o, h, w), np.float32)
    y2 = np.zeros((o, h, w), np.float32)
    oh1, ow1, oh2, ow2 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    oracle().oracle_conv2d(ptr(x), c, h, w, ptr(kk), o, k, k, stride, k // 2, ptr(y1),
                           C.byref(oh1), C.byref(ow1))
    ref().ref_conv2d(ptr(x), c, h, w, ptr(kk), o, k, k, stride, k // 2, ptr(y2), C.byref(oh2),
                     C.byref(ow2))
    assert (oh1.value, ow1.value) == (oh2.value, ow2.value)
    n = o * oh1.value * ow1.value
    assert np.array_equal(_bits(y1.ravel()[:n]), _bits(y2.ravel()[:n]))
    u1 = np.zeros((c, 2 * h, 2 * w), np.float32)
    u2 = np.zeros_like(u1)
    oracle().oracle_upsample2(ptr(x), c, h, w, ptr(u1))
    ref().ref_upsample2(ptr(x), c, h, w, ptr(u2))
    assert np.array_equal(u1, u2)
