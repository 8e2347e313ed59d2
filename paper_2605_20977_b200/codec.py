"""Python mirror of the reference's pipeline API over the C ABI.

``GpuCodec`` exposes encode_frame / decode_frame_wavefront / forward_params
 for one handle of ``libpswa_cuda.so``; every call
goes straight to the sm_100a path — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import PswaCfg, check, lib

_P = C.c_void_p


def make_cfg(preset: str = "paper", height: int = 68, width: int = 120, **over) -> PswaCfg:
    cfg = PswaCfg()
    lib().pswa_cfg_preset(C.byref(cfg), 1 if preset == "paper" else 0, height, width)
    for k, v in over.items():
        setattr(cfg, k, int(v))
    return cfg


def cfg_from_dict(d: dict) -> PswaCfg:
    cfg = PswaCfg()
    for k, v in d.items():
        setattr(cfg, k, int(v))
    return cfg


def gen_weights(cfg: PswaCfg, seed: int = 1) -> bytes:
    n = C.c_size_t()
    check(lib().pswa_gen_weights(C.byref(cfg), seed, None, 0, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    check(lib().pswa_gen_weights(C.byref(cfg), seed, buf, n.value, C.byref(n)))
    return bytes(buf)


def synth_latent(cfg: PswaCfg, gop: int, frame: int) -> np.ndarray:
    y = np.zeros((cfg.latent_ch, cfg.height, cfg.width), np.int32)
    check(lib().pswa_synth_latent(C.byref(cfg), gop, frame, y.ctypes.data_as(_P)))
    return y


def synth_gop(cfg: PswaCfg, gop: int, n_frames: int) -> np.ndarray:
    """Frames 0..n_frames-1 of GOP `gop`, [F][C][H][W] int32, in one pass."""
    y = np.zeros((n_frames, cfg.latent_ch, cfg.height, cfg.width), np.int32)
    check(lib().pswa_synth_gop(C.byref(cfg), gop, n_frames, y.ctypes.data_as(_P)))
    return y


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


class GpuCodec:
    """One device handle: weights, K/V caches, temporal ring, coder lanes."""

    def __init__(self, cfg: PswaCfg, weights: bytes, device: int = 0, band: int = 0,
                 n_bands: int = 1):
        self.cfg = cfg
        self._w = (C.c_uint8 * len(weights)).from_buffer_copy(weights)
        h = C.c_void_p()
        if n_bands == 1:
            check(lib().pswa_gpu_create(device, C.byref(cfg), self._w, len(weights), C.byref(h)))
        else:  # one band of a cross-process group (link it with band_link)
            check(lib().pswa_gpu_create_band(device, C.byref(cfg), self._w, len(weights), band,
                                             n_bands, C.byref(h)))
        self.h = h
        self.band, self.n_bands = band, n_bands

    def band_export(self) -> bytes:
        n = C.c_size_t()
        check(lib().pswa_gpu_band_export(self.h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(lib().pswa_gpu_band_export(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def band_link(self, up: bytes | None, down: bytes | None):
        check(lib().pswa_gpu_band_link(self.h, up, len(up) if up else 0, down,
                                       len(down) if down else 0))

    def close(self):
        if getattr(self, "h", None):
            lib().pswa_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    @property
    def shape(self):
        return (self.cfg.latent_ch, self.cfg.height, self.cfg.width)

    @property
    def zshape(self):
        return (self.cfg.hyper_ch, (self.cfg.height + 3) // 4, (self.cfg.width + 3) // 4)

    def reset_gop(self):
        check(lib().pswa_gpu_reset_gop(self.h))

    def push_frame(self, yhat: np.ndarray, rate: int = 0):
        y = np.ascontiguousarray(yhat, np.int32)
        check(lib().pswa_gpu_push_frame(self.h, _ptr(y), rate))

    def encode_frame(self, yhat: np.ndarray, rate: int = 0, fidx: int = 0):
        y = np.ascontiguousarray(yhat, np.int32)
        cap = 20 * y.size + (1 << 20)
        hb = np.empty(cap, np.uint8)
        mb = np.empty(cap, np.uint8)
        hl, ml = C.c_size_t(), C.c_size_t()
        bits = np.zeros(2, np.float64)
        check(lib().pswa_gpu_encode_frame(self.h, _ptr(y), rate, fidx, _ptr(hb), cap, C.byref(hl),
                                          _ptr(mb), cap, C.byref(ml),
                                          bits.ctypes.data_as(C.POINTER(C.c_double))))
        return bytes(hb[:hl.value]), bytes(mb[:ml.value]), bits

    def last_zhat(self) -> np.ndarray:
        z = np.zeros(self.zshape, np.int32)
        check(lib().pswa_gpu_last_zhat(self.h, _ptr(z)))
        return z

    def last_eps(self) -> np.ndarray:
        """LRP output eps [C][H][W] of the last decoded / encoded frame."""
        e = np.zeros(self.shape, np.float32)
        check(lib().pswa_gpu_last_eps(self.h, _ptr(e)))
        return e

    def decode_frame(self, hyper: bytes, main: bytes, rate: int = 0, fidx: int = 0,
                     advance: bool = True, params: bool = False):
        """-> (y_hat, bits[2]); with params=True -> (y_hat, bits, mu, sigma): the
        entropy parameters the decoder computed itself ([C][H][W] each)."""
        hb = np.frombuffer(hyper, np.uint8)
        mb = np.frombuffer(main, np.uint8)
        y = np.empty(self.shape, np.int32)
        bits = np.zeros(2, np.float64)
        mu = np.empty(self.shape, np.float32) if params else None
        sg = np.empty(self.shape, np.float32) if params else None
        check(lib().pswa_gpu_decode_frame(self.h, _ptr(hb), len(hyper), _ptr(mb), len(main), rate,
                                          fidx, int(advance), _ptr(y),
                                          None if mu is None else _ptr(mu),
                                          None if sg is None else _ptr(sg),
                                          bits.ctypes.data_as(C.POINTER(C.c_double))))
        return (y, bits, mu, sg) if params else (y, bits)

    def set_stats(self, on: bool = True):
        """BitStats for every later frame call."""
        check(lib().pswa_gpu_set_stats(self.h, int(on)))

    def last_bitstats(self) -> np.ndarray:
        """Per-position, per-group estimated bits [N][H][W] of the last frame
        call made with stats on (or with mu/sigma requested)."""
        out = np.zeros((self.cfg.n_groups, self.cfg.height, self.cfg.width), np.float64)
        check(lib().pswa_gpu_last_bitstats(self.h, _ptr(out)))
        return out

    def forward_params(self, yhat: np.ndarray, zhat: np.ndarray, rate: int = 0, fidx: int = 0):
        y = np.ascontiguousarray(yhat, np.int32)
        z = np.ascontiguousarray(zhat, np.int32)
        mu = np.zeros(self.shape, np.float32)
        sg = np.zeros(self.shape, np.float32)
        bits = np.zeros(2, np.float64)
        check(lib().pswa_gpu_forward_params(self.h, _ptr(y), _ptr(z), rate, fidx, _ptr(mu), _ptr(sg),
                                            bits.ctypes.data_as(C.POINTER(C.c_double))))
        return mu, sg, bits

    def encode_sequence(self, frames: np.ndarray, gop: int = 32, rate: int = 0) -> bytes:
        """frames [F][C][H][W] -> PSWA container (FORMAT.md); resets the ring."""
        f = np.ascontiguousarray(frames, np.int32)
        n = C.c_size_t()
        cap = 20 * f.size + (1 << 20) * max(1, f.shape[0])
        buf = np.empty(cap, np.uint8)
        check(lib().pswa_gpu_encode_sequence(self.h, _ptr(f), f.shape[0], gop, rate, _ptr(buf), cap,
                                             C.byref(n)))
        return bytes(buf[:n.value])

    def decode_sequence(self, container: bytes, max_frames: int | None = None):
        """-> (frames [F][C][H][W], status [F] (0 ok, -1 skipped, >0 error), bits [F][2])."""
        info = container_info(container)
        mf = info["frames_present"] if max_frames is None else max_frames
        out = np.zeros((max(mf, 1),) + self.shape, np.int32)
        st = np.zeros(max(mf, 1), np.int32)
        bits = np.zeros((max(mf, 1), 2), np.float64)
        n = C.c_int()
        cb = np.frombuffer(container, np.uint8)
        check(lib().pswa_gpu_decode_sequence(self.h, _ptr(cb), len(container), _ptr(out), mf,
                                             _ptr(st), bits.ctypes.data_as(C.POINTER(C.c_double)),
                                             C.byref(n)))
        return out[:n.value], st[:n.value], bits[:n.value]

    def decode_device(self, d_hyper: int, hyper_len: int, d_main: int, main_len: int, rate: int,
                      fidx: int, advance: bool, d_out: int):
        check(lib().pswa_gpu_decode_frame_device(self.h, d_hyper, hyper_len, d_main, main_len,
                                                 rate, fidx, int(advance), d_out))

    def decode_async(self, d_hyper: int, hyper_len: int, d_main: int, main_len: int, rate: int,
                     fidx: int, d_out: int, advance: bool = False):
        check(lib().pswa_gpu_decode_frame_async(self.h, d_hyper, hyper_len, d_main, main_len,
                                                rate, fidx, int(advance), d_out))

    def finish(self):
        bits = np.zeros(2, np.float64)
        check(lib().pswa_gpu_finish(self.h, bits.ctypes.data_as(C.POINTER(C.c_double))))
        return bits

    def debug_fetch(self, name: str) -> np.ndarray:
        n = C.c_size_t()
        check(lib().pswa_gpu_debug_fetch(self.h, name.encode(), None, 0, C.byref(n)))
        buf = np.zeros(n.value, np.uint8)
        check(lib().pswa_gpu_debug_fetch(self.h, name.encode(), _ptr(buf), n.value, C.byref(n)))
        dt = np.float16 if name in ("ctx", "s1", "s2") else np.float32
        return buf.view(dt).astype(np.float32).reshape(-1, self.cfg.d_spatial)

    def last_launch_count(self) -> int:
        return lib().pswa_gpu_last_launch_count(self.h)

    def bench_op(self, name: str, reps: int = 50) -> tuple[float, float]:
        """(us per launch, algorithmic FLOPs per launch) of one production op."""
        us, fl = C.c_double(), C.c_double()
        check(lib().pswa_gpu_bench_op(self.h, name.encode(), reps, C.byref(us), C.byref(fl)))
        return us.value, fl.value

    def probes(self) -> dict:
        """{name: (flops, bytes, launches)} of every bench probe."""
        n = C.c_size_t()
        check(lib().pswa_gpu_probe_list(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().pswa_gpu_probe_list(self.h, buf, n.value, C.byref(n)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, fl, by, nl = line.split()
            out[name] = (float(fl), float(by), int(nl))
        return out

    def bench_probe(self, name: str, reps: int = 50) -> tuple[float, float, float]:
        """(us per replay, FLOPs, HBM bytes) of one probe."""
        us, fl, by = C.c_double(), C.c_double(), C.c_double()
        check(lib().pswa_gpu_bench_probe(self.h, name.encode(), reps, C.byref(us), C.byref(fl),
                                         C.byref(by)))
        return us.value, fl.value, by.value

    def stream(self) -> int:
        return lib().pswa_gpu_stream(self.h)


def split_banded(main: bytes, n: int) -> list[bytes]:
    """Band payloads of a PSWB container ("PSWB" | u32 n | u64 len[n] | ...)."""
    if len(main) < 8 + 8 * n or main[:4] != b"PSWB":
        raise ValueError("not a banded payload")
    if int.from_bytes(main[4:8], "little") != n:
        raise ValueError("band count differs")
    lens = [int.from_bytes(main[8 + 8 * b:16 + 8 * b], "little") for b in range(n)]
    off, out = 8 + 8 * n, []
    for l in lens:
        if off + l > len(main):
            raise ValueError("truncated banded payload")
        out.append(main[off:off + l])
        off += l
    return out


def container_info(container: bytes) -> dict:
    """Header of a PSWA sequence container (FORMAT.md); host only."""
    v = (C.c_int * 10)()
    cb = np.frombuffer(container, np.uint8)
    check(lib().pswa_container_info(_ptr(cb), len(container), v))
    keys = ("version", "w_px", "h_px", "frames", "gop", "rate", "s", "N", "prior", "frames_present")
    return dict(zip(keys, list(v)))


def band_rows(height: int, n_bands: int, band: int) -> tuple[int, int]:
    """Latent rows [r0, r1) of band `band` of `n_bands` (multiples of 4)."""
    r0, r1 = C.c_int(), C.c_int()
    check(lib().pswa_band_rows(height, n_bands, band, C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


class BandGroupCodec:
    """One frame as row bands: one device handle per band, the
    halo K/V rows pushed between neighbours after every layer. Same frame API
    as GpuCodec; the main payload is the banded container (band-local lanes).
    `devices` lists the device of each band (bands may share a device)."""

    def __init__(self, cfg: PswaCfg, weights: bytes, devices):
        self.cfg = cfg
        self.n = len(devices)
        self._w = (C.c_uint8 * len(weights)).from_buffer_copy(weights)
        devs = (C.c_int * self.n)(*devices)
        h = C.c_void_p()
        check(lib().pswa_group_create(devs, self.n, C.byref(cfg), self._w, len(weights),
                                      C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().pswa_group_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    shape = GpuCodec.shape
    zshape = GpuCodec.zshape

    def reset_gop(self):
        check(lib().pswa_group_reset_gop(self.h))

    def push_frame(self, yhat: np.ndarray, rate: int = 0):
        y = np.ascontiguousarray(yhat, np.int32)
        check(lib().pswa_group_push_frame(self.h, _ptr(y), rate))

    def encode_frame(self, yhat: np.ndarray, rate: int = 0, fidx: int = 0, zhat=None):
        y = np.ascontiguousarray(yhat, np.int32)
        z = None if zhat is None else np.ascontiguousarray(zhat, np.int32)
        cap = 20 * y.size + (1 << 20)
        hb = np.empty(cap, np.uint8)
        mb = np.empty(cap, np.uint8)
        hl, ml = C.c_size_t(), C.c_size_t()
        bits = np.zeros(2, np.float64)
        check(lib().pswa_group_encode_frame(self.h, _ptr(y), None if z is None else _ptr(z), rate,
                                            fidx, _ptr(hb), cap, C.byref(hl), _ptr(mb), cap,
                                            C.byref(ml), bits.ctypes.data_as(C.POINTER(C.c_double))))
        return bytes(hb[:hl.value]), bytes(mb[:ml.value]), bits

    def last_zhat(self) -> np.ndarray:
        z = np.zeros(self.zshape, np.int32)
        check(lib().pswa_group_last_zhat(self.h, _ptr(z)))
        return z

    def decode_frame(self, hyper: bytes, main: bytes, rate: int = 0, fidx: int = 0,
                     advance: bool = True):
        hb = np.frombuffer(hyper, np.uint8)
        mb = np.frombuffer(main, np.uint8)
        y = np.empty(self.shape, np.int32)
        bits = np.zeros(2, np.float64)
        check(lib().pswa_group_decode_frame(self.h, _ptr(hb), len(hyper), _ptr(mb), len(main),
                                            rate, fidx, int(advance), _ptr(y),
                                            bits.ctypes.data_as(C.POINTER(C.c_double))))
        return y, bits

    def forward_params(self, yhat: np.ndarray, zhat: np.ndarray, rate: int = 0, fidx: int = 0):
        y = np.ascontiguousarray(yhat, np.int32)
        z = np.ascontiguousarray(zhat, np.int32)
        mu = np.zeros(self.shape, np.float32)
        sg = np.zeros(self.shape, np.float32)
        bits = np.zeros(2, np.float64)
        check(lib().pswa_group_forward_params(self.h, _ptr(y), _ptr(z), rate, fidx, _ptr(mu),
                                              _ptr(sg), bits.ctypes.data_as(C.POINTER(C.c_double))))
        return mu, sg, bits

    def last_launch_count(self) -> int:
        return lib().pswa_group_last_launch_count(self.h)
