"""encode_sequence / decode_sequence through the C ABI:
bit-exact round trip across GOP resets, the 1-frame sequence equals the
I-frame path, whole-frame decoding of truncated containers, drift-free
restart after a corrupted frame, hash mismatches refused, and the committed
golden container decodes bit-exactly."""
import os

import numpy as np
import pytest

from paper_2605_20977_b200 import PswaError
from paper_2605_20977_b200.codec import GpuCodec, gen_weights, make_cfg, synth_latent

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _setup(H=8, W=8, n=5):
    cfg = make_cfg("desk", H, W, lanes=8, hyper_lanes=4)
    blob = gen_weights(cfg, 1)
    frames = np.stack([synth_latent(cfg, 0, f) for f in range(n)])
    return cfg, blob, frames


def test_sequence_roundtrip_gop_resets():
    cfg, blob, frames = _setup()
    cont = GpuCodec(cfg, blob).encode_sequence(frames, gop=2, rate=0)
    y, st, bits = GpuCodec(cfg, blob).decode_sequence(cont)
    assert np.array_equal(y, frames) and (st == 0).all() and (bits[:, 1] > 0).all()


def test_one_frame_sequence_is_the_iframe_path():
    cfg, blob, frames = _setup(n=1)
    cont = GpuCodec(cfg, blob).encode_sequence(frames, gop=32, rate=2)
    h, m, _ = GpuCodec(cfg, blob).encode_frame(frames[0], rate=2, fidx=0)
    assert cont[64:] == len(h).to_bytes(4, "little") + h + len(m).to_bytes(4, "little") + m


def test_truncation_and_corruption():
    cfg, blob, frames = _setup(n=5)
    cont = GpuCodec(cfg, blob).encode_sequence(frames, gop=2, rate=0)
    dec = GpuCodec(cfg, blob)
    y, st, _ = dec.decode_sequence(cont[:-3])  # frame 4 incomplete
    assert len(y) == 4 and np.array_equal(y, frames[:4]) and (st == 0).all()
    # corrupt frame 1's main payload: frame 0 fine, frame 1 fails, GOP 1 (frames 2, 3) fine
    off = 64
    lens = []
    for _ in range(5):
        hl = int.from_bytes(cont[off:off + 4], "little")
        ml = int.from_bytes(cont[off + 4 + hl:off + 8 + hl], "little")
        lens.append((off, hl, ml))
        off += 8 + hl + ml
    o1, hl1, ml1 = lens[1]
    bad = bytearray(cont)
    bad[o1 + 8 + hl1 + 8:o1 + 8 + hl1 + ml1] = b"\xff" * (ml1 - 8)  # keep L, count
    y, st, _ = dec.decode_sequence(bytes(bad))
    assert st[0] == 0 and np.array_equal(y[0], frames[0])
    assert (st[2:] == 0).all() and np.array_equal(y[2:], frames[2:])
    assert st[1] != 0 or not np.array_equal(y[1], frames[1])


def test_hash_mismatch_refused():
    cfg, blob, frames = _setup(n=2)
    cont = GpuCodec(cfg, blob).encode_sequence(frames, gop=2)
    with pytest.raises(PswaError) as e:
        GpuCodec(cfg, gen_weights(cfg, 2)).decode_sequence(cont)
    assert e.value.code == 3
    cfg2 = make_cfg("desk", 8, 8, lanes=16, hyper_lanes=4)
    with pytest.raises(PswaError):
        GpuCodec(cfg2, blob).decode_sequence(cont)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLD, "seq_desk_8x8.pswa")), reason="no golden")
def test_golden_container_decodes():
    cfg = make_cfg("desk", 8, 8, lanes=8, hyper_lanes=4)
    blob = gen_weights(cfg, 1)
    cont = open(os.path.join(GOLD, "seq_desk_8x8.pswa"), "rb").read()
    frames = np.load(os.path.join(GOLD, "seq_desk_8x8_frames.npy"))
    y, st, _ = GpuCodec(cfg, blob).decode_sequence(cont)
    assert (st == 0).all() and np.array_equal(y, frames)
