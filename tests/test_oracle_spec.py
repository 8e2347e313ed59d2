"""SPEC known-answer tests for the oracle (the only golden vectors the
reference defines). Each test cites the SPEC line it pins."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle_api import (bits, cdf_tables, decode_lanes, encode_lanes, oracle, ptr,
                        scale_table)


def mm(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    c = np.zeros((a.shape[0], b.shape[1]), np.float32)
    oracle().oracle_matmul(ptr(a), ptr(b), ptr(c), a.shape[0], a.shape[1], b.shape[1])
    return c


def softmax(row):
    r = np.ascontiguousarray(row, np.float32).copy()
    oracle().oracle_softmax_row(ptr(r), r.size)
    return r


# ------------------------------------------------------------ tensor_core --
def test_matmul_kats():
    x = np.random.default_rng(0).normal(size=(3, 4)).astype(np.float32)
    assert np.array_equal(mm(np.eye(3), x), x)
    assert mm([[2.0]], [[3.0]])[0, 0] == 6.0
    a = np.random.default_rng(1).normal(size=(5, 4)).astype(np.float32)
    b = np.random.default_rng(2).normal(size=(4, 3)).astype(np.float32)
    trip = np.zeros((5, 3), np.float32)
    for i in range(5):
        for j in range(3):
            acc = np.float32(0)
            for k in range(4):
                acc = np.float32(acc + np.float32(a[i, k] * b[k, j]))
            trip[i, j] = acc
    assert np.array_equal(mm(a, b), trip)


def test_softmax_kats():
    assert np.allclose(softmax([0, 0]), [0.5, 0.5], atol=0)
    s = np.finfo(np.float32).min
    assert np.array_equal(softmax([s, s]), [0.0, 0.0])
    assert np.allclose(softmax([0, math.log(3)]), [0.25, 0.75], atol=1e-6)


def test_rmsnorm_kats():
    d = 8
    out = np.zeros(d, np.float32)
    one = np.ones(d, np.float32)
    oracle().oracle_rmsnorm(ptr(one), ptr(one), d, ptr(out))
    assert np.allclose(out, 1 / math.sqrt(1 + 1e-5), atol=1e-7)
    x = np.random.default_rng(3).normal(size=d).astype(np.float32)
    o1, o2 = np.zeros(d, np.float32), np.zeros(d, np.float32)
    oracle().oracle_rmsnorm(ptr(x), ptr(one), d, ptr(o1))
    x5 = (x * 5).astype(np.float32)
    oracle().oracle_rmsnorm(ptr(x5), ptr(one), d, ptr(o2))
    assert np.argmax(o1) == np.argmax(o2)
    hp = x.astype(np.float64) / math.sqrt(np.mean(x.astype(np.float64) ** 2) + 1e-5)
    assert np.allclose(o1, hp, atol=1e-6)


def test_swiglu_zero_and_bounded():
    assert oracle().oracle_det_f32(1, 0.0) == 0.0
    for v in np.linspace(-100, 100, 201):
        assert math.isfinite(oracle().oracle_det_f32(1, float(v)))


def test_conv2d_kats():
    x = np.ones((1, 4, 4), np.float32)
    k = np.ones((1, 1, 3, 3), np.float32)
    y = np.zeros((1, 4, 4), np.float32)
    oh, ow = C.c_int(), C.c_int()
    oracle().oracle_conv2d(ptr(x), 1, 4, 4, ptr(k), 1, 3, 3, 1, 1, ptr(y), C.byref(oh), C.byref(ow))
    assert y[0, 0, 0] == 4 and y[0, 1, 1] == 9
    x = np.random.default_rng(4).normal(size=(1, 5, 5)).astype(np.float32)
    k1 = np.ones((1, 1, 1, 1), np.float32)
    y = np.zeros((1, 5, 5), np.float32)
    oracle().oracle_conv2d(ptr(x), 1, 5, 5, ptr(k1), 1, 1, 1, 1, 0, ptr(y), C.byref(oh), C.byref(ow))
    assert np.array_equal(x, y)


def test_init_kats():
    n = 100000
    a, b = np.zeros(n, np.float32), np.ones(n, np.float32)
    oracle().oracle_init_values(7, ptr(b), n, 1, 1)
    assert not b.any()
    oracle().oracle_init_values(7, ptr(a), n, 0, 1)
    c = np.zeros(n, np.float32)
    oracle().oracle_init_values(7, ptr(c), n, 0, 1)
    assert np.array_equal(a, c)
    assert abs(a.mean()) < 3 * a.std() / math.sqrt(n)


# -------------------------------------------------------------- wavefront --
def positions(H, W, s, t):
    out = np.zeros(H * W, np.int32)
    n = oracle().oracle_positions_of_step(H, W, s, t, ptr(out))
    return [(int(p) // W, int(p) % W) for p in out[:n]]


def test_step_of_and_positions_kats():
    assert positions(1, 1, 4, 0) == [(0, 0)]
    assert all(positions(1, 1, 4, t) == [] for t in (1, 2, 3))
    assert positions(4, 4, 4, 1) == [(0, 1), (1, 0), (2, 3), (3, 2)]
    assert [len(positions(8, 8, 4, t)) for t in range(4)] == [16, 16, 16, 16]
    allp = sorted(p for t in range(4) for p in positions(7, 5, 4, t))
    assert allp == [(y, x) for y in range(7) for x in range(5)]
    assert [len(positions(68, 120, 4, t)) for t in range(4)] == [2040] * 4


def test_channel_mask_kats():
    m = np.zeros(4, np.uint8)
    oracle().oracle_channel_mask(2, 1, ptr(m))
    assert m.reshape(2, 2).tolist() == [[1, 0], [1, 1]]
    m = np.zeros(16, np.uint8)
    oracle().oracle_channel_mask(1, 4, ptr(m))
    assert m.all()


@pytest.mark.parametrize("H,W,s,N,steps", [(8, 8, 4, 4, 16), (16, 16, 4, 4, 16), (64, 64, 4, 4, 16),
                                           (5, 5, 1, 1, 1), (7, 9, 3, 2, 6)])
def test_validate_schedule(H, W, s, N, steps):
    st = C.c_int()
    assert oracle().oracle_validate_schedule(H, W, s, 7, 7, N, C.byref(st)) == 1
    assert st.value == steps


# ------------------------------------------------------------ range coder --
def test_cdf_kats():
    t = cdf_tables()
    freq = np.diff(t.astype(np.int64), axis=1)
    assert (t[:, -1] == 65536).all() and (t[:, 0] == 0).all()
    assert (freq >= 1).all()
    assert np.array_equal(freq[:, :255], freq[:, :255][:, ::-1])  # freq(v) == freq(-v)
    assert (freq[:, 255] == freq[:, 256]).all()
    assert freq[0, 127] / 65536 >= 0.99  # sigma = 0.11: >= 99% on v = 0
    sc = scale_table()
    assert abs(sc[0] - 0.11) < 1e-7 and abs(sc[63] - 64) < 1e-4
    assert (np.diff(sc) > 0).all()
    assert oracle().oracle_scale_index(0.11) == 0
    assert oracle().oracle_scale_index(1000.0) == 63
    for i in (1, 17, 40):
        assert oracle().oracle_scale_index(float(sc[i])) == i
        assert oracle().oracle_scale_index(float(np.nextafter(sc[i - 1], np.float32(1e9)))) == i


def test_coder_empty_stream():
    data = encode_lanes(np.zeros(0), np.zeros(0), 1)
    assert len(data) == 4 + 4 + 4 + 2 + 4  # header(lanes, count, width) + 1 u16 length + 4-byte flush
    assert decode_lanes(data, np.zeros(0, np.int32)).size == 0


def test_coder_exhaustive_4pow6():  # all 4^6 sequences of a 4-symbol alphabet
    alphabet = np.array([-1, 0, 1, 2], np.int32)
    idx = np.full(6, 20, np.int32)
    for code in range(4 ** 6):
        v = alphabet[[(code >> (2 * i)) & 3 for i in range(6)]]
        data = encode_lanes(v, idx, 1)
        assert np.array_equal(decode_lanes(data, idx), v)


@pytest.mark.parametrize("lanes", [1, 3, 64])
def test_coder_random_roundtrip_and_bound(lanes):
    rng = np.random.default_rng(lanes)
    worst = 0.0
    for case in range(300 if lanes == 1 else 60):
        n = int(rng.integers(0, 400))
        idx = rng.integers(0, 64, n).astype(np.int32)
        sig = scale_table()[idx]
        v = np.round(rng.laplace(0, sig * 1.5)).astype(np.int32)
        esc = rng.random(n) < 0.02
        v[esc] = rng.integers(-5000, 5000, esc.sum())
        data = encode_lanes(v, idx, lanes)
        assert np.array_equal(decode_lanes(data, idx), v)
        if lanes == 1:  # header: lanes, count, width + one 2-byte length entry
            payload_bits = 8 * (len(data) - 14)
            worst = max(worst, payload_bits - bits(v, idx))
    if lanes == 1:
        assert worst <= 32.0 + 1e-9, worst


def test_lane_length_entry_width():
    """FORMAT.md §2: 2-byte lane lengths while every lane is under 64 KiB,
    4-byte ones beyond; both decode."""
    rng = np.random.default_rng(11)
    for n, lanes, w in ((2000, 4, 2), (120000, 1, 4)):
        idx = np.full(n, 63, np.int32)
        v = np.rint(rng.laplace(0, 40.0, n)).astype(np.int32)
        data = encode_lanes(v, idx, lanes)
        assert np.frombuffer(data[8:12], np.uint32)[0] == w
        lens = np.frombuffer(data[12:12 + w * lanes], np.uint16 if w == 2 else np.uint32)
        assert 12 + w * lanes + int(lens.astype(np.int64).sum()) == len(data)
        assert np.array_equal(decode_lanes(data, idx), v)
    bad = bytearray(encode_lanes(np.zeros(4, np.int32), np.zeros(4, np.int32), 2))
    bad[8] = 3  # a width other than 2 or 4
    assert decode_lanes(bytes(bad), np.zeros(4, np.int32)) is None


def test_coder_truncation_detected():
    rng = np.random.default_rng(9)
    idx = rng.integers(0, 30, 500).astype(np.int32)
    v = rng.integers(-3, 4, 500).astype(np.int32)
    data = encode_lanes(v, idx, 1)
    assert decode_lanes(data[:-5], idx) is None


def test_estimate_bits_kats():
    t = cdf_tables().astype(np.int64)
    f = t[30, 128] - t[30, 127]
    assert bits([0], [30]) == pytest.approx(16 - math.log2(f))
    f0 = t[0, 128] - t[0, 127]
    assert bits([0], [0]) == pytest.approx(-math.log2(f0 / 65536))
    # every one of the 257 buckets keeps freq >= 1, so the mode tops out at
    # 65536 - 256: the cost of a certain symbol is -log2(65280/65536) ~ 5.6e-3
    assert bits([0], [0]) <= -math.log2(65280 / 65536) + 1e-12
