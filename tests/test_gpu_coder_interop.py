"""The GPU lane coder against the CPU oracle's (lane format
DESIGN.md §3), through pswa_gpu_op_encode_symbols / _decode_symbols, which
run the production kernels (lanes_encode + lanes_pack; lanes_init + the phase
decoder). For the same (value, table index) arrays:
  * the GPU encoder's payload is byte-identical to the oracle's;
  * the GPU decodes oracle payloads and the oracle decodes GPU payloads;
  * both report the same estimate_bits;
for L in {1, 64, 8192}, escapes up to 2^30, the empty stream, and
truncation/corruption."""
import ctypes as C

import numpy as np
import pytest

from oracle_api import bits as oracle_bits, decode_lanes, encode_lanes
from paper_2605_20977_b200 import PswaError, check, lib

pytestmark = pytest.mark.gpu

_D = C.POINTER(C.c_double)


def gpu_encode(v, idx, lanes, laplace=0):
    v = np.ascontiguousarray(v, np.int32)
    idx = np.ascontiguousarray(idx, np.int32)
    n = C.c_size_t()
    b = C.c_double()
    check(lib().pswa_gpu_op_encode_symbols(v.ctypes.data, idx.ctypes.data, v.size, lanes, laplace,
                                           None, 0, C.byref(n), C.byref(b)))
    out = np.zeros(max(1, n.value), np.uint8)
    check(lib().pswa_gpu_op_encode_symbols(v.ctypes.data, idx.ctypes.data, v.size, lanes, laplace,
                                           out.ctypes.data, out.size, C.byref(n), C.byref(b)))
    return bytes(out[:n.value]), b.value


def gpu_decode(data, idx, laplace=0):
    idx = np.ascontiguousarray(idx, np.int32)
    buf = np.frombuffer(data, np.uint8).copy()
    out = np.zeros(max(1, idx.size), np.int32)
    b = C.c_double()
    check(lib().pswa_gpu_op_decode_symbols(buf.ctypes.data, len(data), idx.ctypes.data, idx.size,
                                           laplace, out.ctypes.data, C.byref(b)))
    return out[:idx.size], b.value


def symbols(n, seed, escapes=True):
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, 64, n).astype(np.int32)
    sc = np.exp(np.linspace(np.log(0.11), np.log(64.0), 64))
    v = np.rint(rng.laplace(0, sc[idx])).astype(np.int64)
    if escapes and n:
        k = rng.choice(n, size=max(1, n // 200), replace=False)
        mags = np.array([128, 129, 300, 2049, 70000, 1 << 20, (1 << 30) + 5, -(1 << 30), -131072])
        v[k] = mags[rng.integers(0, mags.size, k.size)] * rng.choice([-1, 1], k.size)
    return np.clip(v, -(2**31 - 129), 2**31 - 129).astype(np.int32), idx


@pytest.mark.parametrize("lanes,n", [(1, 5000), (64, 20000), (8192, 300000), (8192, 5000)])
def test_gpu_and_oracle_lane_streams_interoperate(lanes, n):
    v, idx = symbols(n, lanes + n)
    g, gb = gpu_encode(v, idx, lanes)
    o = encode_lanes(v, idx, lanes)
    assert g == o                                  # byte-identical payloads
    yo = decode_lanes(g, idx)                      # GPU stream -> oracle decoder
    assert yo is not None and np.array_equal(yo, v)
    yg, db = gpu_decode(o, idx)                    # oracle stream -> GPU decoder
    assert np.array_equal(yg, v)
    ob = oracle_bits(v, idx)
    assert abs(gb - ob) <= 1e-9 * ob and abs(db - ob) <= 1e-9 * ob


@pytest.mark.parametrize("lanes", [1, 64, 8192])
def test_empty_stream(lanes):  # a flush-only stream per lane
    v = np.zeros(0, np.int32)
    g, gb = gpu_encode(v, v, lanes)
    assert g == encode_lanes(v, v, lanes) and gb == 0.0
    yg, _ = gpu_decode(g, v)
    assert yg.size == 0


def test_truncated_and_corrupt_payloads_are_rejected():
    v, idx = symbols(4000, 3)
    g, _ = gpu_encode(v, idx, 64)
    with pytest.raises(PswaError) as e:
        gpu_decode(g[:-40], idx)
    assert e.value.code == 2
    bad = bytearray(g)
    bad[4] ^= 1  # symbol count in the header
    with pytest.raises(PswaError):
        gpu_decode(bytes(bad), idx)
    # flipping a lane byte (not in its 4-byte flush, whose low bits are free)
    # either changes symbols or is detected
    assert np.frombuffer(g[8:12], np.uint32)[0] == 2  # 16-bit length entries
    lens = np.frombuffer(g[12:12 + 2 * 64], np.uint16).astype(np.int64)
    starts = 12 + 2 * 64 + np.concatenate([[0], np.cumsum(lens)[:-1]])
    rng = np.random.default_rng(0)
    silent = 0
    for lane in rng.choice(64, 16, replace=False):
        b2 = bytearray(g)
        b2[int(starts[lane] + rng.integers(0, lens[lane] - 4))] ^= 0x5A
        try:
            y, _ = gpu_decode(bytes(b2), idx)
            silent += int(np.array_equal(y, v))
        except PswaError:
            pass
    assert silent <= 1  # a byte read only after the lane's last decision can be free


def test_laplace_family_roundtrip():
    v, idx = symbols(50000, 9)
    g, gb = gpu_encode(v, idx, 256, laplace=1)
    y, db = gpu_decode(g, idx, laplace=1)
    assert np.array_equal(y, v) and db == gb
    g0, _ = gpu_encode(v, idx, 256, laplace=0)
    assert g0 != g  # a different table family codes different bytes


def test_single_stream_bound():
    """L = 1: coded size <= estimate + 32 bits plus the 12 B
    header and the lane's length entry (4 B once the lane passes 64 KiB)."""
    v, idx = symbols(100000, 5, escapes=False)
    g, gb = gpu_encode(v, idx, 1)
    w = int(np.frombuffer(g[8:12], np.uint32)[0])
    assert (w == 4) == (len(g) - 14 >= 65536)
    assert 8 * (len(g) - 12 - w) <= gb + 32


@pytest.mark.parametrize("lanes,n", [(1, 120000), (2, 240000)])
def test_wide_length_entries(lanes, n):
    """Lanes longer than 64 KiB switch the length table to 4-byte entries on
    both sides; the streams stay byte-identical and interchangeable."""
    rng = np.random.default_rng(lanes)
    idx = np.full(n, 63, np.int32)  # the widest table: ~9.6 bits per symbol
    v = np.rint(rng.laplace(0, 40.0, n)).astype(np.int32)
    g, _ = gpu_encode(v, idx, lanes)
    assert np.frombuffer(g[8:12], np.uint32)[0] == 4
    assert g == encode_lanes(v, idx, lanes)
    assert np.array_equal(decode_lanes(g, idx), v)
    assert np.array_equal(gpu_decode(g, idx)[0], v)
