"""End-to-end frames: PPM I/O, the toy
DCT transform (device kernels), and a sequence round trip built on the
codec's container API. Reconstruction uses y_hat + eps when the handle has an
LRP transformer (cfg.lrp_blocks > 0)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib
from .codec import GpuCodec

_P = C.c_void_p


def read_ppm(path: str) -> np.ndarray:
    w, h = C.c_int(), C.c_int()
    check(lib().pswa_read_ppm(path.encode(), None, 0, C.byref(w), C.byref(h)))
    a = np.zeros((h.value, w.value, 3), np.uint8)
    check(lib().pswa_read_ppm(path.encode(), a.ctypes.data_as(_P), a.size, C.byref(w), C.byref(h)))
    return a


def write_ppm(path: str, rgb: np.ndarray):
    a = np.ascontiguousarray(rgb, np.uint8)
    check(lib().pswa_write_ppm(path.encode(), a.ctypes.data_as(_P), a.shape[1], a.shape[0]))


def pad8(rgb: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(rgb, np.uint8)
    h8, w8 = C.c_int(), C.c_int()
    check(lib().pswa_pad8(a.ctypes.data_as(_P), a.shape[0], a.shape[1], None, C.byref(h8), C.byref(w8)))
    out = np.zeros((h8.value, w8.value, 3), np.uint8)
    check(lib().pswa_pad8(a.ctypes.data_as(_P), a.shape[0], a.shape[1], out.ctypes.data_as(_P),
                          C.byref(h8), C.byref(w8)))
    return out


def analysis(rgb: np.ndarray, rate: int) -> np.ndarray:
    """[H][W][3] u8 (multiples of 8) -> y [192][H/8][W/8] f32 (device DCT)."""
    a = np.ascontiguousarray(rgb, np.uint8)
    y = np.zeros((192, a.shape[0] // 8, a.shape[1] // 8), np.float32)
    check(lib().pswa_toy_analysis(a.ctypes.data_as(_P), a.shape[0], a.shape[1], rate, y.ctypes.data_as(_P)))
    return y


def synthesis(y: np.ndarray, rate: int) -> np.ndarray:
    a = np.ascontiguousarray(y, np.float32)
    out = np.zeros((a.shape[1] * 8, a.shape[2] * 8, 3), np.uint8)
    check(lib().pswa_toy_synthesis(a.ctypes.data_as(_P), out.shape[0], out.shape[1], rate,
                                   out.ctypes.data_as(_P)))
    return out


def quantize(y: np.ndarray) -> np.ndarray:
    """y_hat = round-half-even(y) (A1)."""
    return np.rint(y).astype(np.int32)


def encode_frames(codec: GpuCodec, frames_rgb, gop: int = 32, rate: int = 0) -> bytes:
    """RGB frames (padded to the codec's grid x 8) -> PSWA container."""
    lat = np.stack([quantize(analysis(pad8(f), rate)) for f in frames_rgb])
    return codec.encode_sequence(lat, gop=gop, rate=rate)


def split_container(container: bytes):
    """(header fields, [(hyper, main) per whole frame]) of a PSWA container."""
    from .codec import container_info
    info = container_info(container)
    frames, off = [], 64
    for _ in range(info["frames_present"]):
        hl = int.from_bytes(container[off:off + 4], "little")
        hyper = container[off + 4:off + 4 + hl]
        ml = int.from_bytes(container[off + 4 + hl:off + 8 + hl], "little")
        frames.append((hyper, container[off + 8 + hl:off + 8 + hl + ml]))
        off += 8 + hl + ml
    return info, frames


def decode_frames(codec: GpuCodec, container: bytes):
    """PSWA container -> (reconstructed RGB frames, decoded y_hat). Frames are
    decoded one by one (GOP resets at f % gop == 0) so that each frame's LRP
    output eps is available: y_rec = y_hat + eps, else y_hat."""
    info, frames = split_container(container)
    lrp = codec.cfg.lrp_blocks > 0
    rgb, ys = [], []
    for f, (hyper, main) in enumerate(frames):
        if f % info["gop"] == 0:
            codec.reset_gop()
        y, _ = codec.decode_frame(hyper, main, rate=info["rate"], fidx=f % info["gop"])
        rec = y.astype(np.float32) + (codec.last_eps() if lrp else 0.0)
        rgb.append(synthesis(rec, info["rate"]))
        ys.append(y)
    return rgb, ys
