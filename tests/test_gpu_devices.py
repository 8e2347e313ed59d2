"""Handles are bound to their device, not to the calling thread's current
device (every pswa_gpu_* entry point makes the handle's device current and
restores the caller's): a handle created on one thread decodes bit-exactly
from another thread, interleaved with a second handle; with two or more GPUs,
a band group spread over devices 0 and 1 equals the single handle."""
import threading

import numpy as np
import pytest
import torch

from oracle_api import gen_weights, preset
from paper_2605_20977_b200.codec import BandGroupCodec, GpuCodec, cfg_from_dict, synth_latent

pytestmark = pytest.mark.gpu


def test_handles_used_from_other_threads():
    c = preset(False, 16, 16, lanes=32, hyper_lanes=16)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    frames = [synth_latent(cfg, g, 0) for g in range(2)]
    encs = [GpuCodec(cfg, blob) for _ in range(2)]
    streams = [e.encode_frame(f, fidx=0)[:2] for e, f in zip(encs, frames)]
    decs = [GpuCodec(cfg, blob) for _ in range(2)]
    out, errs = {}, []

    def work(i):
        try:
            for _ in range(3):  # interleaves with the other thread's handle
                decs[i].reset_gop()
                y, _ = decs[i].decode_frame(*streams[i], fidx=0)
            out[i] = y
        except Exception as e:  # noqa: BLE001 - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(2):
        assert np.array_equal(out[i], frames[i])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_band_group_across_two_devices():
    c = preset(True, 24, 32, lanes=32, hyper_lanes=16)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    frames = [synth_latent(cfg, 0, f) for f in range(3)]
    one = GpuCodec(cfg, blob, device=0)
    grp = BandGroupCodec(cfg, blob, [0, 1])
    for f in frames[:2]:
        one.push_frame(f)
        grp.push_frame(f)
    torch.cuda.set_device(1)  # the caller's current device must not matter
    h, m, _ = grp.encode_frame(frames[2], fidx=2)
    y, _ = grp.decode_frame(h, m, fidx=2, advance=False)
    assert np.array_equal(y, frames[2])
    z = grp.last_zhat()
    mu_b, sg_b, _ = grp.forward_params(frames[2], z, fidx=2)
    mu_1, sg_1, _ = one.forward_params(frames[2], z, fidx=2)
    assert np.array_equal(mu_b.view(np.uint32), mu_1.view(np.uint32))
    assert np.array_equal(sg_b.view(np.uint32), sg_1.view(np.uint32))
