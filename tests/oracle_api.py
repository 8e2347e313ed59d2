"""ctypes access to the CPU oracle (oracle/liboracle.so) and to the reference's
own numerics compiled unmodified (oracle/_ref/libpswa_ref.so).

Test infrastructure only: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpswa_ref.so")

CFG_FIELDS = ("d_spatial", "heads", "ctx_blocks", "s1_blocks", "s2_blocks", "d_channel",
              "ch_blocks", "hyper_ch", "latent_ch", "s", "n_groups", "win_h", "win_w", "win_t",
              "ctx_slots", "rate_points", "height", "width", "lanes", "hyper_lanes", "prior", "lrp_blocks")

_P = C.c_void_p
_fp = C.POINTER(C.c_float)


def preset(paper: bool, H: int, W: int, lanes: int = 1, hyper_lanes: int = 1, **over) -> dict:
    c = dict(d_spatial=512 if paper else 64, heads=16, ctx_blocks=8 if paper else 2,
             s1_blocks=8 if paper else 2, s2_blocks=8 if paper else 2,
             d_channel=1024 if paper else 128, ch_blocks=2, hyper_ch=128 if paper else 32,
             latent_ch=192, s=4, n_groups=4, win_h=7, win_w=7, win_t=5, ctx_slots=4,
             rate_points=4, height=H, width=W, lanes=lanes, hyper_lanes=hyper_lanes, prior=0,
             lrp_blocks=0)
    c.update(over)
    return c


def cfg_array(cfg: dict):
    return (C.c_int * len(CFG_FIELDS))(*[int(cfg[f]) for f in CFG_FIELDS])


def ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        L = C.CDLL(ORACLE_SO)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_det.restype = C.c_double
        L.oracle_det.argtypes = [C.c_int, C.c_double]
        L.oracle_det_f32.restype = C.c_float
        L.oracle_det_f32.argtypes = [C.c_int, C.c_float]
        L.oracle_rng.argtypes = [C.c_uint64, C.c_int, _P, _P, _P]
        L.oracle_fnv1a.restype = C.c_uint64
        L.oracle_fnv1a.argtypes = [_P, C.c_size_t]
        L.oracle_init_values.argtypes = [C.c_uint64, _P, C.c_size_t, C.c_int, C.c_int]
        L.oracle_bits.restype = C.c_double
        L.oracle_bits.argtypes = [_P, _P, C.c_size_t]
        L.oracle_encode_lanes.argtypes = [_P, _P, C.c_size_t, C.c_int, _P, C.c_size_t,
                                          C.POINTER(C.c_size_t)]
        L.oracle_decode_lanes.argtypes = [_P, C.c_size_t, _P, C.c_size_t, _P]
        L.oracle_scale_index.argtypes = [C.c_float]
        L.oracle_model_create.restype = _P
        L.oracle_model_create.argtypes = [_P, _P, C.c_size_t]
        L.oracle_model_destroy.argtypes = [_P]
        L.oracle_gen_weights.argtypes = [_P, C.c_uint64, _P, C.c_size_t, C.POINTER(C.c_size_t)]
        L.oracle_param_count.restype = C.c_int64
        L.oracle_forward.argtypes = [_P, _P, _P, C.c_int, _P, C.c_int, _P, _P, _P, _P]
        L.oracle_forward_debug.argtypes = [_P, _P, _P, C.c_int, _P, C.c_int, _P, _P, _P, _P, _P]
        L.oracle_encode.argtypes = [_P, _P, C.c_int, C.c_int, _P, C.c_int, _P, _P, C.c_size_t,
                                    C.POINTER(C.c_size_t), _P, C.c_size_t, C.POINTER(C.c_size_t),
                                    _P, _P]
        L.oracle_decode.argtypes = [_P, C.c_int, _P, C.c_size_t, _P, C.c_size_t, C.c_int, C.c_int,
                                    _P, C.c_int, _P, _P, _P]
        _oracle = L
    return _oracle


def ref():
    """The reference's own numerics (None when oracle/_ref was not built)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            return None
        L = C.CDLL(REF_SO)
        L.ref_det.restype = C.c_double
        L.ref_det.argtypes = [C.c_int, C.c_double]
        L.ref_det_f32.restype = C.c_float
        L.ref_det_f32.argtypes = [C.c_int, C.c_float]
        L.ref_rng.argtypes = [C.c_ulonglong, C.c_int, _P, _P, _P]
        L.ref_fnv1a.restype = C.c_ulonglong
        L.ref_fnv1a.argtypes = [_P, C.c_ulong]
        L.ref_init_tensor.argtypes = [C.c_ulonglong, _P, C.c_int, C.c_int, C.c_int]
        _ref = L
    return _ref


# ---------------------------------------------------------------- helpers --
def gen_weights(cfg: dict, seed: int = 1) -> bytes:
    L = oracle()
    n = C.c_size_t()
    ca = cfg_array(cfg)
    assert L.oracle_gen_weights(ca, seed, None, 0, C.byref(n)) == 0
    buf = (C.c_uint8 * n.value)()
    assert L.oracle_gen_weights(ca, seed, buf, n.value, C.byref(n)) == 0
    return bytes(buf)


def _past_array(past):
    arr = (C.c_void_p * max(1, len(past)))()
    keep = []
    for i, p in enumerate(past):
        p = np.ascontiguousarray(p, dtype=np.int32)
        keep.append(p)
        arr[i] = p.ctypes.data
    return arr, keep


class OracleModel:
    def __init__(self, cfg: dict, blob: bytes):
        self.cfg = dict(cfg)
        self._blob = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        self.h = oracle().oracle_model_create(cfg_array(cfg), self._blob, len(blob))
        if not self.h:
            raise RuntimeError(oracle().oracle_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            oracle().oracle_model_destroy(self.h)

    @property
    def shape(self):
        return (self.cfg["latent_ch"], self.cfg["height"], self.cfg["width"])

    @property
    def zshape(self):
        return (self.cfg["hyper_ch"], (self.cfg["height"] + 3) // 4, (self.cfg["width"] + 3) // 4)

    def forward(self, yhat, rate=0, past=(), zhat=None):
        y = np.ascontiguousarray(yhat, dtype=np.int32)
        mu = np.zeros(self.shape, np.float32)
        sg = np.zeros(self.shape, np.float32)
        zo = np.zeros(self.zshape, np.int32)
        zi = None if zhat is None else np.ascontiguousarray(zhat, dtype=np.int32)
        pa, keep = _past_array(past)
        rc = oracle().oracle_forward(self.h, ptr(y), None if zi is None else ptr(zi), rate, pa,
                                     len(past), ptr(mu), ptr(sg), ptr(zo), None)
        assert rc == 0, oracle().oracle_last_error()
        return mu, sg, zo

    def lrp(self, yhat, zhat, rate=0, past=()):
        """LRP output eps [C][H][W] of a known frame (teacher forced)."""
        y = np.ascontiguousarray(yhat, dtype=np.int32)
        z = np.ascontiguousarray(zhat, dtype=np.int32)
        eps = np.zeros(self.shape, np.float32)
        pa, keep = _past_array(past)
        rc = oracle().oracle_lrp(self.h, ptr(y), ptr(z), rate, pa, len(past), ptr(eps))
        assert rc == 0, oracle().oracle_last_error()
        return eps

    def forward_debug(self, yhat, zhat, rate=0, past=()):
        """Stage outputs [H*W][d]: ctx, s1, hq, a, s2 (parity triage)."""
        y = np.ascontiguousarray(yhat, dtype=np.int32)
        z = np.ascontiguousarray(zhat, dtype=np.int32)
        hw = self.cfg["height"] * self.cfg["width"]
        outs = [np.zeros((hw, self.cfg["d_spatial"]), np.float32) for _ in range(5)]
        pa, keep = _past_array(past)
        rc = oracle().oracle_forward_debug(self.h, ptr(y), ptr(z), rate, pa, len(past),
                                           *[ptr(o) for o in outs])
        assert rc == 0, oracle().oracle_last_error()
        return dict(zip(("ctx", "s1", "hq", "a", "s2"), outs))

    def encode(self, yhat, rate=0, fidx=0, past=(), zhat=None):
        y = np.ascontiguousarray(yhat, dtype=np.int32)
        pa, keep = _past_array(past)
        zi = None if zhat is None else np.ascontiguousarray(zhat, dtype=np.int32)
        hl, ml = C.c_size_t(), C.c_size_t()
        bits = np.zeros(2, np.float64)
        zo = np.zeros(self.zshape, np.int32)
        cap = 64 * y.size + (1 << 16)
        hb = np.zeros(cap, np.uint8)
        mb = np.zeros(cap, np.uint8)
        rc = oracle().oracle_encode(self.h, ptr(y), rate, fidx, pa, len(past),
                                    None if zi is None else ptr(zi), ptr(hb), cap, C.byref(hl),
                                    ptr(mb), cap, C.byref(ml), ptr(bits), ptr(zo))
        assert rc == 0, oracle().oracle_last_error()
        return bytes(hb[:hl.value]), bytes(mb[:ml.value]), bits, zo

    def decode(self, hyper: bytes, main: bytes, rate=0, fidx=0, past=(), serial=False):
        """Returns (yhat, bits, phases) or None for a corrupt/truncated stream."""
        pa, keep = _past_array(past)
        y = np.zeros(self.shape, np.int32)
        bits = np.zeros(2, np.float64)
        ph = C.c_int()
        hb = np.frombuffer(hyper, np.uint8).copy()
        mb = np.frombuffer(main, np.uint8).copy()
        rc = oracle().oracle_decode(self.h, 1 if serial else 0, ptr(hb), len(hyper), ptr(mb),
                                    len(main), rate, fidx, pa, len(past), ptr(y), ptr(bits),
                                    C.byref(ph))
        if rc == 2:
            return None
        assert rc == 0, oracle().oracle_last_error()
        return y, bits, ph.value


def synth_gop(cfg: dict, gop: int, n_frames: int) -> np.ndarray:
    """The oracle's restatement of the synthetic latent generator (SURVEY
    §8(d)): frames 0..n_frames-1 of GOP `gop`, [F][C][H][W] int32."""
    y = np.zeros((n_frames, cfg["latent_ch"], cfg["height"], cfg["width"]), np.int32)
    assert oracle().oracle_synth_gop(cfg_array(cfg), gop, n_frames, ptr(y)) == 0
    return y


def encode_lanes(v: np.ndarray, idx: np.ndarray, lanes: int) -> bytes:
    v = np.ascontiguousarray(v, np.int32)
    idx = np.ascontiguousarray(idx, np.int32)
    cap = 16 * v.size + 8 * lanes + 64
    out = np.zeros(cap, np.uint8)
    n = C.c_size_t()
    assert oracle().oracle_encode_lanes(ptr(v), ptr(idx), v.size, lanes, ptr(out), cap,
                                        C.byref(n)) == 0
    return bytes(out[:n.value])


def decode_lanes(data: bytes, idx: np.ndarray):
    idx = np.ascontiguousarray(idx, np.int32)
    out = np.zeros(idx.size, np.int32)
    buf = np.frombuffer(data, np.uint8).copy()
    rc = oracle().oracle_decode_lanes(ptr(buf), len(data), ptr(idx), idx.size, ptr(out))
    return out if rc == 0 else None


def bits(v, idx) -> float:
    v = np.ascontiguousarray(v, np.int32)
    idx = np.ascontiguousarray(idx, np.int32)
    return oracle().oracle_bits(ptr(v), ptr(idx), v.size)


def cdf_tables() -> np.ndarray:
    t = np.zeros((64, 258), np.uint32)
    oracle().oracle_cdf_tables(ptr(t))
    return t


def scale_table() -> np.ndarray:
    t = np.zeros(64, np.float32)
    oracle().oracle_scale_table(ptr(t))
    return t


def cdf_tables_family(laplace: int) -> np.ndarray:
    """The 64 cumulative tables of the Gaussian (0) or Laplace (1) head."""
    t = np.zeros((64, 258), np.uint32)
    oracle().oracle_cdf_tables_family(int(laplace), ptr(t))
    return t
