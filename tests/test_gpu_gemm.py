"""tcgen05 GEMM parity vs a torch fp32 reference of the same op."""
import ctypes as C

import pytest
import torch

from paper_2605_20977_b200 import lib, check

pytestmark = pytest.mark.gpu


def _run(M, N, K, out_f32=1, accumulate=0, bias=None, scale=None, act=0, force_bn=0):
    torch.manual_seed(M * 7 + N * 3 + K)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    ref = a.float() @ b.float().t()
    if scale is not None:
        ref = ref * scale
    if bias is not None:
        ref = ref + bias
    if act == 1:
        ref = torch.nn.functional.silu(ref)
    if out_f32:
        c = torch.randn(M, N, device="cuda") if accumulate else torch.zeros(M, N, device="cuda")
        base = c.clone()
    else:
        c = torch.zeros(M, N, device="cuda", dtype=torch.float16)
    check(lib().pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), N,
                                     out_f32, accumulate,
                                     bias.data_ptr() if bias is not None else None,
                                     scale.data_ptr() if scale is not None else None,
                                     act, force_bn, None))
    torch.cuda.synchronize()
    if accumulate:
        ref = ref + base
    return c.float(), ref


@pytest.mark.parametrize("M,N,K,bn", [(128, 64, 64, 64), (256, 128, 128, 128), (300, 256, 512, 256),
                                      (2040, 512, 512, 0), (2040, 1536, 512, 0), (77, 64, 1408, 64),
                                      (32640, 2816, 512, 0)])
def test_gemm_f32(M, N, K, bn):
    c, ref = _run(M, N, K, force_bn=bn)
    err = (c - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


def test_gemm_f16_bias_scale_silu():
    N = 256
    bias = torch.randn(N, device="cuda")
    scale = torch.rand(N, device="cuda") + 0.5
    c, ref = _run(513, N, 256, out_f32=0, bias=bias, scale=scale, act=1)
    assert torch.allclose(c, ref, atol=2e-2, rtol=1e-2)


def test_gemm_accumulate():
    c, ref = _run(640, 512, 1408, accumulate=1)
    assert torch.allclose(c, ref, atol=1e-3, rtol=1e-4)


def test_gemm_deterministic():
    c1, _ = _run(2040, 512, 512)
    c2, _ = _run(2040, 512, 512)
    assert torch.equal(c1, c2)


@pytest.mark.parametrize("M,N,K", [(2040, 1408, 256), (32640, 2816, 512), (100, 128, 64)])
def test_gemm_swiglu(M, N, K):
    torch.manual_seed(M + N)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    c = torch.zeros(M, N // 2, device="cuda", dtype=torch.float16)
    check(lib().pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), N // 2,
                                     0, 0, None, None, 2, 0, None))
    torch.cuda.synchronize()
    acc = a.float() @ b.float().t()
    ref = torch.nn.functional.silu(acc[:, 0::2]) * acc[:, 1::2]
    assert torch.allclose(c.float(), ref, atol=3e-2, rtol=2e-2)


def test_gemm_head_epilogue():
    torch.manual_seed(5)
    M, N, K = 333, 128, 512
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    bias = torch.randn(N, device="cuda") * 0.1
    scale = torch.rand(N, device="cuda") + 0.5
    c = torch.zeros(M, N, device="cuda")
    check(lib().pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), N, 1, 0,
                                     bias.data_ptr(), scale.data_ptr(), 3, 0, None))
    torch.cuda.synchronize()
    acc = a.float() @ b.float().t() + bias
    ref = torch.cat([acc[:, :64] * scale[:64], 0.11 + torch.nn.functional.softplus(acc[:, 64:])], 1)
    assert torch.allclose(c, ref, atol=1e-3, rtol=1e-3)


@pytest.mark.parametrize("M,N,K,acc", [(32640, 2816, 512, 0), (16500, 512, 1408, 1), (32640, 1536, 512, 0)])
def test_pair_gemm_bitwise_equals_single_sm(M, N, K, acc):
    """The CTA-pair (tcgen05 cta_group::2) kernel (force_bn = -1; opt-in for
    the large context GEMMs) gives bitwise the single-SM kernel's results
    (same K order), so the encoder/decoder symmetry does not depend on it."""
    c_pair, ref = _run(M, N, K, accumulate=acc, force_bn=-1)
    c_one, _ = _run(M, N, K, accumulate=acc, force_bn=256)
    assert torch.equal(c_pair, c_one)
    err = (c_pair - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("M,N,K,acc,f32", [(2040, 512, 512, 1, 1), (2040, 512, 1408, 1, 1), (300, 256, 192, 0, 1),
                                          (77, 128, 128, 1, 1), (2040, 512, 512, 0, 0), (8160, 512, 1408, 1, 1)])
def test_splitk_gemm(M, N, K, acc, f32):
    """Split-K CTA pairs (force_bn = -2; the step-batch and channel residual
    GEMMs): within fp32 tolerance of the torch reference, deterministic, and
    the same bits for a row whatever M is (a layer's rows agree between the
    2040-row decoder batches and the 8160-row teacher-forced batch)."""
    c, ref = _run(M, N, K, out_f32=f32, accumulate=acc, force_bn=-2)
    tol = 2e-3 if f32 else 2e-2
    assert (c - ref).abs().max().item() <= tol * max(1.0, ref.abs().max().item())
    c2, _ = _run(M, N, K, out_f32=f32, accumulate=acc, force_bn=-2)
    assert torch.equal(c, c2)


def test_splitk_rows_independent_of_m():
    torch.manual_seed(5)
    K, N = 1408, 512
    a = (torch.randn(8160, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    outs = []
    for M in (8160, 2040):
        c = torch.zeros(M, N, device="cuda")
        check(lib().pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), N, 1, 0,
                                         None, None, 0, -2, None))
        outs.append(c)
    torch.cuda.synchronize()
    assert torch.equal(outs[0][:2040], outs[1])


@pytest.mark.parametrize("M,N,K,kind,bn", [(2040, 2816, 512, "swiglu", 352), (2040, 2816, 512, "f16", 352),
                                           (2040, 1408, 512, "f32acc", 352), (8160, 2816, 512, "swiglu", 352),
                                           (300, 704, 128, "f16", 352), (2040, 1536, 512, "f16", 192),
                                           (8160, 1536, 512, "f32acc", 192)])
def test_wide_tiles_bitwise_equal_bn256(M, N, K, kind, bn):
    """128 x 352 tiles (two N = 176 MMAs per K step, one TMEM accumulator;
    chosen for the 2040-row gate|up GEMMs, which fit one wave of 128 tiles)
    give bitwise the 128 x 256 / 128 x 64 kernels' results: the K order per
    element is the same, so the encoder (8160 rows, BN 256) and the decoder
    (2040 rows, BN 352) stay bitwise symmetric. 8160 rows also runs BN 352
    with several tiles per CTA (single-buffered accumulator). 128 x 192
    tiles (one wave of 128 for the 2040-row Q|K|V GEMMs) likewise."""
    torch.manual_seed(M + N + K)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    b = (torch.randn(N, K, device="cuda") * 0.05).half()
    act = 2 if kind == "swiglu" else 0
    f32 = 1 if kind == "f32acc" else 0
    ncol = N // 2 if kind == "swiglu" else N
    base = torch.randn(M, ncol, device="cuda")
    outs = []
    for bn in (bn, 256 if N % 256 == 0 else 64):
        c = base.clone() if f32 else torch.zeros(M, ncol, device="cuda", dtype=torch.float16)
        check(lib().pswa_gpu_op_gemm_f16(a.data_ptr(), K, M, b.data_ptr(), K, N, K, c.data_ptr(), ncol,
                                         f32, f32, None, None, act, bn, None))
        torch.cuda.synchronize()
        outs.append(c)
    assert torch.equal(outs[0], outs[1])
    acc = a.float() @ b.float().t()
    if kind == "swiglu":
        ref = torch.nn.functional.silu(acc[:, 0::2]) * acc[:, 1::2]
    elif kind == "f32acc":
        ref = acc + base
    else:
        ref = acc
    assert torch.allclose(outs[0].float(), ref, atol=3e-2, rtol=2e-2)
