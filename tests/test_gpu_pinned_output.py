"""Host-output decode into pinned memory (pswa_gpu_decode_frame): the copies
of finished channel groups overlap the last groups' decoding (engine
run_host_copy); the result must equal the pageable-output decode and the
encoder input, frame after frame (P-frames, advancing state)."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2605_20977_b200 import lib
from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("preset,H,W,lrp", [("desk", 12, 20, 0), ("paper", 16, 16, 0),
                                             ("desk", 12, 20, 2)])
def test_pinned_output_matches(preset, H, W, lrp):
    cfg = make_cfg(preset, H, W, lanes=16, hyper_lanes=4, lrp_blocks=lrp)
    blob = gen_weights(cfg, 1)
    frames = [synth_latent(cfg, 0, f) for f in range(3)]
    enc = GpuCodec(cfg, blob)
    streams = [enc.encode_frame(f, fidx=i)[:2] for i, f in enumerate(frames)]
    pinned, pageable = GpuCodec(cfg, blob), GpuCodec(cfg, blob)
    out = torch.empty(cfg.latent_ch * H * W, dtype=torch.int32).pin_memory()
    bits = np.zeros(2, np.float64)
    for i, (hyper, main) in enumerate(streams):
        out.fill_(-7)
        hb = np.frombuffer(hyper, np.uint8)
        mb = np.frombuffer(main, np.uint8)
        rc = lib().pswa_gpu_decode_frame(pinned.h, hb.ctypes.data, len(hyper), mb.ctypes.data,
                                         len(main), 0, i, 1, out.data_ptr(), None, None,
                                         bits.ctypes.data_as(C.POINTER(C.c_double)))
        assert rc == 0
        y_pin = out.numpy().reshape(cfg.latent_ch, H, W)
        y_page, _ = pageable.decode_frame(hyper, main, fidx=i)
        assert np.array_equal(y_pin, frames[i]) and np.array_equal(y_page, frames[i])
        if lrp:  # the LRP stage after the overlapped copies sees the same y_hat
            assert np.array_equal(pinned.last_eps(), pageable.last_eps())
