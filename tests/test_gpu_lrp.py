"""LRP transformer (A8) on the GPU against the
CPU oracle: eps = 0.5 tanh(head(rmsnorm(x))) after lrp_blocks of 3D SWA over
the T past slots (context-transformer inputs) and the current slot
in_proj(concat(final channel representation, y_hat)).
  * the decoder's eps equals the encoder's eps bitwise (same kernels);
  * eps within |d eps| <= 0.01 of the oracle on >= 99.9% of elements, <= 0.05
    everywhere (fp16 tensor-core operands vs the fp32 no-FMA oracle);
  * eps in (-0.5, 0.5); I-frame and P-frame (GOP index 3)."""
import numpy as np
import pytest

from oracle_api import OracleModel, gen_weights, preset
from paper_2605_20977_b200.codec import GpuCodec, cfg_from_dict, synth_latent

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("paper,lrp,fidx", [(False, 1, 0), (False, 2, 3), (True, 1, 0), (True, 2, 3)])
def test_lrp_eps_matches_oracle(paper, lrp, fidx):
    H, W = 16, 16
    c = preset(paper, H, W, lanes=32, hyper_lanes=8, lrp_blocks=lrp)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    frames = [synth_latent(cfg, 2, f) for f in range(fidx + 1)]
    enc, dec = GpuCodec(cfg, blob), GpuCodec(cfg, blob)
    for f in frames[:fidx]:
        enc.push_frame(f)
        dec.push_frame(f)
    y = frames[fidx]
    hyper, main, _ = enc.encode_frame(y, fidx=fidx)
    eps_e = enc.last_eps()
    z = enc.last_zhat()
    yd, _ = dec.decode_frame(hyper, main, fidx=fidx)
    eps_d = dec.last_eps()
    assert np.array_equal(yd, y)
    assert np.array_equal(eps_e.view(np.uint32), eps_d.view(np.uint32))
    assert (np.abs(eps_d) < 0.5).all()
    om = OracleModel(c, blob)
    eps_o = om.lrp(y, z, past=frames[:fidx])
    err = np.abs(eps_d - eps_o)
    from test_gpu_pipeline import record
    record(f"lrp_{'paper' if paper else 'desk'}_b{lrp}_f{fidx}", eps_max_abs=float(err.max()),
           eps_mean_abs=float(err.mean()), frac_within_0p01=float((err <= 0.01).mean()))
    assert (err <= 0.01).mean() >= 0.999, float(err.max())
    assert err.max() <= 0.05
