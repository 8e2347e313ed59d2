"""pswa/tensor.h on the device, byte-identical to the reference's own CPU
build (oracle/_ref/libpswa_ref.so: proj/src/tensor.cpp compiled unmodified)
on random inputs, including masked softmax rows and ragged shapes."""
import ctypes as C

import numpy as np
import pytest

from oracle_api import ref
from paper_2605_20977_b200 import PswaError, check, lib

pytestmark = pytest.mark.gpu

P = C.c_void_p


def ptr(a):
    return a.ctypes.data_as(P)


@pytest.fixture(scope="module")
def R():
    r = ref()
    if r is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return r


def rnd(rng, *shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float32)


@pytest.mark.parametrize("m,k,p", [(1, 1, 1), (17, 33, 65), (128, 512, 300), (3, 1368, 7)])
def test_matmul_bitexact(R, m, k, p):
    rng = np.random.default_rng(m * k + p)
    a, b = rnd(rng, m, k), rnd(rng, k, p, scale=0.1)
    c, cr = np.zeros((m, p), np.float32), np.zeros((m, p), np.float32)
    check(lib().pswa_tensor_matmul(ptr(a), ptr(b), ptr(c), m, k, p))
    R.ref_matmul(ptr(a), ptr(b), ptr(cr), m, k, p)
    assert np.array_equal(c.view(np.uint32), cr.view(np.uint32))


def test_matmul_shape_error():
    a = np.zeros(4, np.float32)
    # the C-ABI wrapper builds well-formed tensors; exercise the C++ check via k = 0
    check(lib().pswa_tensor_matmul(ptr(a), ptr(a), ptr(a), 2, 0, 2))
    assert not a.any()


def test_softmax_rows_bitexact_with_masked_rows(R):
    rng = np.random.default_rng(1)
    m, k = 300, 49
    x = rnd(rng, m, k, scale=4.0)
    x[5, :] = np.finfo(np.float32).min       # fully masked row -> zeros
    x[6, ::2] = np.finfo(np.float32).min     # partly masked
    y, yr = np.zeros_like(x), np.zeros_like(x)
    check(lib().pswa_tensor_softmax_rows(ptr(x), ptr(y), m, k))
    R.ref_softmax_rows(ptr(x), ptr(yr), m, k)
    assert np.array_equal(y.view(np.uint32), yr.view(np.uint32))
    assert not y[5].any()


@pytest.mark.parametrize("d", [1, 64, 512, 1000])
def test_rmsnorm_bitexact(R, d):
    rng = np.random.default_rng(d)
    x, g = rnd(rng, d, scale=3.0), rnd(rng, d)
    o, orf = np.zeros(d, np.float32), np.zeros(d, np.float32)
    check(lib().pswa_tensor_rmsnorm(ptr(x), ptr(g), d, ptr(o)))
    R.ref_rmsnorm(ptr(x), ptr(g), d, ptr(orf))
    assert np.array_equal(o.view(np.uint32), orf.view(np.uint32))


@pytest.mark.parametrize("d", [64, 512])
def test_swiglu_ffn_bitexact(R, d):
    f = lib().pswa_tensor_ffn_hidden_dim(d)
    assert f == R.ref_ffn_hidden_dim(d)
    rng = np.random.default_rng(f)
    x = rnd(rng, d)
    wg, wu, wd = rnd(rng, d, f, scale=d ** -0.5), rnd(rng, d, f, scale=d ** -0.5), rnd(rng, f, d, scale=f ** -0.5)
    o, orf = np.zeros(d, np.float32), np.zeros(d, np.float32)
    check(lib().pswa_tensor_swiglu_ffn(ptr(x), ptr(wg), ptr(wu), ptr(wd), d, f, ptr(o)))
    R.ref_swiglu_ffn(ptr(x), ptr(wg), ptr(wu), ptr(wd), d, f, ptr(orf))
    assert np.array_equal(o.view(np.uint32), orf.view(np.uint32))


@pytest.mark.parametrize("c,h,w,o,kh,stride,pad", [(3, 9, 11, 5, 3, 1, 1), (32, 17, 30, 32, 3, 2, 1),
                                                   (4, 8, 8, 2, 5, 1, 0), (1, 1, 1, 1, 1, 1, 0)])
def test_conv2d_bitexact(R, c, h, w, o, kh, stride, pad):
    rng = np.random.default_rng(c * h + o)
    x, k = rnd(rng, c, h, w), rnd(rng, o, c, kh, kh, scale=0.2)
    oh, ow = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kh) // stride + 1
    y, yr = np.zeros((o, oh, ow), np.float32), np.zeros((o, oh, ow), np.float32)
    check(lib().pswa_tensor_conv2d(ptr(x), c, h, w, ptr(k), o, kh, kh, stride, pad, ptr(y)))
    a, b = C.c_int(), C.c_int()
    R.ref_conv2d(ptr(x), c, h, w, ptr(k), o, kh, kh, stride, pad, ptr(yr), C.byref(a), C.byref(b))
    assert (a.value, b.value) == (oh, ow)
    assert np.array_equal(y.view(np.uint32), yr.view(np.uint32))


def test_conv2d_even_kernel_rejected():
    x, k = np.zeros(16, np.float32), np.zeros(16, np.float32)
    y = np.zeros(64, np.float32)
    with pytest.raises(PswaError) as e:
        check(lib().pswa_tensor_conv2d(ptr(x), 1, 4, 4, ptr(k), 1, 2, 2, 1, 0, ptr(y)))
    assert e.value.code == 1


def test_upsample_bitexact(R):
    rng = np.random.default_rng(3)
    x = rnd(rng, 5, 7, 9)
    y, yr = np.zeros((5, 14, 18), np.float32), np.zeros((5, 14, 18), np.float32)
    check(lib().pswa_tensor_upsample2(ptr(x), 5, 7, 9, ptr(y)))
    R.ref_upsample2(ptr(x), 5, 7, 9, ptr(yr))
    assert np.array_equal(y, yr)
