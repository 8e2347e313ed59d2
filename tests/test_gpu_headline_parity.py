"""Parity at the configuration the bench reports (BASELINE config 3: 1080p =
120x68 latents, paper scale, P-frame at GOP index 4; plus the I-frame of
config 2 and the desk preset at the same grid), on the DECODER's own entropy
parameters:

  (a) y_hat decoded from the GPU bitstream is bit-exact to the encoder input;
  (b) the decoder's mu/sigma (pswa_gpu_decode_frame mu_out/sigma_out) are
      bitwise equal to the teacher-forced encoder program's
      (pswa_gpu_forward_params) -- the two run different launch schedules;
  (c) mu/sigma are within the stated tolerance of the CPU oracle's
      teacher-forced forward (tests/test_gpu_pipeline.py tolerances);
  (d) the estimated rate is within 1e-3 of the oracle's on the oracle's own
      mu/sigma (estimate_bits);
  (e) BitStats sum to the frame estimate, are equal on
      encoder and decoder, equal the oracle's estimate_bits of the coded
      symbols per (position, group), and the main payload carries at most the
      per-lane framing on top of them.
The paper-scale oracle forward of a 1080p frame is ~1.2 TMAC (~20 s on 16
host threads)."""
import os

import numpy as np
import pytest

from oracle_api import OracleModel, bits as oracle_bits, gen_weights, oracle, preset, scale_table
from paper_2605_20977_b200.codec import GpuCodec, cfg_from_dict, synth_latent
from test_gpu_pipeline import compare_params, record

pytestmark = pytest.mark.gpu

H, W = 68, 120
LANES, HYPER_LANES = 8192, 1024


def oracle_symbol_bits(y, mu, sg):
    """Per-symbol estimate of the oracle's own parameters: v = y - rint(mu)
    under table index(sigma) = first i with scale[i] >= sigma."""
    sc = scale_table()
    idx = np.minimum(np.searchsorted(sc, sg.astype(np.float32), side="left"), 63).astype(np.int32)
    v = (y.astype(np.int64) - np.rint(mu).astype(np.int64)).astype(np.int32)
    return v, idx


def per_position_group_bits(v, idx, N):
    """[N][H][W] oracle bits: estimate_bits over each group's channels."""
    C_, H_, W_ = v.shape
    Cg = C_ // N
    out = np.zeros((N, H_, W_))
    for g in range(N):
        vg = np.ascontiguousarray(v[g * Cg:(g + 1) * Cg].transpose(1, 2, 0).reshape(-1, Cg))
        ig = np.ascontiguousarray(idx[g * Cg:(g + 1) * Cg].transpose(1, 2, 0).reshape(-1, Cg))
        for p in range(H_ * W_):
            out[g].flat[p] = oracle_bits(vg[p], ig[p])
    return out


@pytest.mark.parametrize("paper,fidx", [(False, 4), (False, 0), (True, 4), (True, 0)])
def test_headline_decoder_params(paper, fidx):
    oracle().oracle_set_threads(os.cpu_count() or 1)
    c = preset(paper, H, W, lanes=LANES, hyper_lanes=HYPER_LANES)
    blob = gen_weights(c, 1)
    cfg = cfg_from_dict(c)
    frames = [synth_latent(cfg, 0, f) for f in range(fidx + 1)]
    past, y = frames[:fidx], frames[fidx]
    enc = GpuCodec(cfg, blob)
    for f in past:
        enc.push_frame(f, rate=0)
    enc.set_stats(True)
    hyper, main, bits_e = enc.encode_frame(y, rate=0, fidx=fidx)
    bs_e = enc.last_bitstats()
    z = enc.last_zhat()

    dec = GpuCodec(cfg, blob)
    for f in past:
        dec.push_frame(f, rate=0)
    yd, bits_d, mu_d, sg_d = dec.decode_frame(hyper, main, rate=0, fidx=fidx, params=True)
    bs_d = dec.last_bitstats()
    assert np.array_equal(yd, y)                                        # (a)
    assert bits_d[1] == bits_e[1] and bits_d[0] == bits_e[0]

    fp = GpuCodec(cfg, blob)
    for f in past:
        fp.push_frame(f, rate=0)
    mu_f, sg_f, bits_f = fp.forward_params(y, z, rate=0, fidx=fidx)
    assert np.array_equal(mu_d.view(np.uint32), mu_f.view(np.uint32))  # (b)
    assert np.array_equal(sg_d.view(np.uint32), sg_f.view(np.uint32))

    om = OracleModel(c, blob)
    mu_o, sg_o, _ = om.forward(y, rate=0, past=past, zhat=z)
    v_o, idx_o = oracle_symbol_bits(y, mu_o, sg_o)
    main_o = oracle_bits(v_o, idx_o)
    tag = f"headline_{'paper' if paper else 'desk'}_{H}x{W}_f{fidx}"
    compare_params(tag, mu_d, sg_d, mu_o, sg_o, bits_d, [bits_d[0], main_o])  # (c), (d)

    # (e) BitStats
    N = c["n_groups"]
    assert bs_d.shape == (N, H, W)
    assert np.array_equal(bs_d, bs_e)
    assert abs(bs_d.sum() - bits_d[1]) <= 1e-9 * bits_d[1]
    payload_bits = 8.0 * len(main)
    overhead = payload_bits - bs_d.sum()
    assert 0 <= overhead <= 64 + LANES * (32 + 32 + 8), overhead
    if not paper:  # per (position, group); host loops, desk is enough
        # exact: the oracle's estimate_bits of the symbols the decoder coded
        # (its own mu/sigma) -- BitStats add up the right per-symbol costs
        v_d, idx_d = oracle_symbol_bits(y, mu_d, sg_d)
        bs_x = per_position_group_bits(v_d, idx_d, N)
        assert np.allclose(bs_d, bs_x, rtol=1e-12, atol=1e-9)
        # against the oracle's own parameters: equal wherever all Cg symbols of
        # the group land on the same (v, table); close in aggregate
        bs_o = per_position_group_bits(v_o, idx_o, N)
        same = np.abs(bs_d - bs_o) <= 1e-9 * np.maximum(1.0, bs_o)
        rel = np.abs(bs_d - bs_o) / np.maximum(1.0, bs_o)
        record(tag + "_bitstats", frac_equal_to_oracle=float(same.mean()),
               rel_p99=float(np.quantile(rel, 0.99)), rel_max=float(rel.max()))
        assert same.mean() >= 0.9 and np.quantile(rel, 0.99) <= 0.05
    record(tag + "_decoder", mu_bitwise_vs_forward_params=True,
           payload_bits=payload_bits, estimate_bits=float(bits_d[1]),
           framing_overhead_bits=float(overhead), lanes=LANES)


def test_headline_lrp_eps_1080p():
    """The LRP transformer at the headline grid with the paper's 4 blocks
    (SURVEY §8(f)2): decoder eps == encoder eps bitwise, within 0.01 of the
    oracle on >= 99.9% of elements, (-0.5, 0.5) everywhere."""
    oracle().oracle_set_threads(os.cpu_count() or 1)
    c = preset(True, H, W, lanes=LANES, hyper_lanes=HYPER_LANES, lrp_blocks=4)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    frames = [synth_latent(cfg, 1, f) for f in range(5)]
    enc, dec = GpuCodec(cfg, blob), GpuCodec(cfg, blob)
    for f in frames[:4]:
        enc.push_frame(f)
        dec.push_frame(f)
    hyper, main, _ = enc.encode_frame(frames[4], fidx=4)
    eps_e, z = enc.last_eps(), enc.last_zhat()
    yd, _ = dec.decode_frame(hyper, main, fidx=4)
    eps_d = dec.last_eps()
    assert np.array_equal(yd, frames[4])
    assert np.array_equal(eps_e.view(np.uint32), eps_d.view(np.uint32))
    assert (np.abs(eps_d) < 0.5).all()
    eps_o = OracleModel(c, blob).lrp(frames[4], z, past=frames[:4])
    err = np.abs(eps_d - eps_o)
    record("headline_lrp_paper_68x120_f4", eps_max_abs=float(err.max()), eps_mean_abs=float(err.mean()),
           frac_within_0p01=float((err <= 0.01).mean()))
    assert (err <= 0.01).mean() >= 0.999 and err.max() <= 0.05


def test_headline_laplace_head_1080p():
    """The Laplace parameter head (prior = 1, north_star item 3) at the
    headline grid: bit-exact round trip, decoder mu/sigma bitwise equal to the
    encoder program's, within the stated tolerance of the oracle, rate within
    1e-3 (estimate_bits of the oracle's own parameters under its Laplace
    tables)."""
    oracle().oracle_set_threads(os.cpu_count() or 1)
    c = preset(True, H, W, lanes=LANES, hyper_lanes=HYPER_LANES, prior=1)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    y = synth_latent(cfg, 3, 0)
    enc = GpuCodec(cfg, blob)
    hyper, main, bits_e = enc.encode_frame(y, fidx=0)
    z = enc.last_zhat()
    dec = GpuCodec(cfg, blob)
    yd, bits_d, mu_d, sg_d = dec.decode_frame(hyper, main, fidx=0, params=True)
    assert np.array_equal(yd, y) and bits_d[1] == bits_e[1]
    fp = GpuCodec(cfg, blob)
    mu_f, sg_f, _ = fp.forward_params(y, z, fidx=0)
    assert np.array_equal(mu_d.view(np.uint32), mu_f.view(np.uint32))
    om = OracleModel(c, blob)
    mu_o, sg_o, _ = om.forward(y, zhat=z)
    v_o, idx_o = oracle_symbol_bits(y, mu_o, sg_o)
    main_o = oracle_bits(v_o, idx_o + 64)  # the oracle's Laplace tables follow the Gaussian 64
    compare_params("headline_laplace_paper_68x120_f0", mu_d, sg_d, mu_o, sg_o, bits_d,
                   [bits_d[0], main_o])
