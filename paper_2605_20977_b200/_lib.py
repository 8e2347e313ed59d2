"""ctypes loader for the in-tree C-ABI library ``libpswa_cuda.so``.

The product path has no CPU fallback: if the library is missing this raises.
Declarations mirror ``include/pswa/pswa_cuda.h``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpswa_cuda.so")

PSWA_OK = 0


class PswaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pswa error {code}: {msg}")
        self.code = code


class PswaCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "d_spatial", "heads", "ctx_blocks", "s1_blocks", "s2_blocks", "d_channel",
        "ch_blocks", "hyper_ch", "latent_ch", "s", "n_groups", "win_h", "win_w", "win_t",
        "ctx_slots", "rate_points", "height", "width", "lanes", "hyper_lanes", "prior", "lrp_blocks")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None

_VP, _I, _SZ, _F, _D = C.c_void_p, C.c_int, C.c_size_t, C.POINTER(C.c_float), C.POINTER(C.c_double)

_SIGS = {
    "pswa_gpu_last_error": (C.c_char_p, []),
    "pswa_cfg_preset": (None, [C.POINTER(PswaCfg), _I, _I, _I]),
    "pswa_gen_weights": (_I, [C.POINTER(PswaCfg), C.c_uint64, _VP, _SZ, C.POINTER(_SZ)]),
    "pswa_synth_latent": (_I, [C.POINTER(PswaCfg), _I, _I, _VP]),
    "pswa_synth_gop": (_I, [C.POINTER(PswaCfg), _I, _I, _VP]),
    "pswa_gpu_create": (_I, [_I, C.POINTER(PswaCfg), _VP, _SZ, C.POINTER(_VP)]),
    "pswa_gpu_destroy": (None, [_VP]),
    "pswa_gpu_reset_gop": (_I, [_VP]),
    "pswa_gpu_encode_frame": (_I, [_VP, _VP, _I, _I, _VP, _SZ, C.POINTER(_SZ), _VP, _SZ,
                                   C.POINTER(_SZ), _D]),
    "pswa_gpu_decode_frame": (_I, [_VP, _VP, _SZ, _VP, _SZ, _I, _I, _I, _VP, _VP, _VP, _D]),
    "pswa_gpu_set_stats": (_I, [_VP, _I]),
    "pswa_gpu_last_bitstats": (_I, [_VP, _VP]),
    "pswa_gpu_forward_params": (_I, [_VP, _VP, _VP, _I, _I, _VP, _VP, _D]),
    "pswa_gpu_last_zhat": (_I, [_VP, _VP]),
    "pswa_gpu_last_eps": (_I, [_VP, _VP]),
    "pswa_gpu_push_frame": (_I, [_VP, _VP, _I]),
    "pswa_gpu_decode_frame_device": (_I, [_VP, _VP, _SZ, _VP, _SZ, _I, _I, _I, _VP]),
    "pswa_gpu_debug_fetch": (_I, [_VP, C.c_char_p, _VP, _SZ, C.POINTER(_SZ)]),
    "pswa_gpu_last_launch_count": (_I, [_VP]),
    "pswa_gpu_stream": (_VP, [_VP]),
    "pswa_gpu_bench_op": (_I, [_VP, C.c_char_p, _I, _D, _D]),
    "pswa_gpu_bench_probe": (_I, [_VP, C.c_char_p, _I, _D, _D, _D]),
    "pswa_gpu_probe_list": (_I, [_VP, C.c_char_p, _SZ, C.POINTER(_SZ)]),
    "pswa_gpu_decode_frame_async": (_I, [_VP, _VP, _SZ, _VP, _SZ, _I, _I, _I, _VP]),
    "pswa_gpu_finish": (_I, [_VP, _D]),
    "pswa_gpu_op_gemm_f16": (_I, [_VP, _I, _I, _VP, _I, _I, _I, _VP, _I, _I, _I, _VP, _VP, _I,
                                  _I, _VP]),
    "pswa_gpu_op_rmsnorm": (_I, [_VP, _I, _I, _I, _I, _VP, _VP, _I, _VP]),
    "pswa_gpu_op_window_attn": (_I, [_VP, _I, _VP, _I, _VP, _I, _I, _I, _I, _I, _I, _I, _I, _I,
                                     _I, _I, _VP, _VP, _I, _VP]),
    "pswa_gpu_op_build_cdf": (_I, [_VP, _VP]),
    "pswa_gpu_op_build_cdf_family": (_I, [_VP, _VP, _I]),
    "pswa_gpu_op_encode_symbols": (_I, [_VP, _VP, _SZ, _I, _I, _VP, _SZ, C.POINTER(_SZ), _D]),
    "pswa_gpu_op_decode_symbols": (_I, [_VP, _SZ, _VP, _SZ, _I, _VP, _D]),
    "pswa_validate_schedule": (_I, [_I, _I, _I, _I, _I, _I, C.POINTER(_I), C.POINTER(_I), C.c_char_p, _SZ]),
    "pswa_tensor_matmul": (_I, [_VP, _VP, _VP, _I, _I, _I]),
    "pswa_tensor_softmax_rows": (_I, [_VP, _VP, _I, _I]),
    "pswa_tensor_rmsnorm": (_I, [_VP, _VP, _I, _VP]),
    "pswa_tensor_swiglu_ffn": (_I, [_VP, _VP, _VP, _VP, _I, _I, _VP]),
    "pswa_tensor_conv2d": (_I, [_VP, _I, _I, _I, _VP, _I, _I, _I, _I, _I, _VP]),
    "pswa_tensor_upsample2": (_I, [_VP, _I, _I, _I, _VP]),
    "pswa_tensor_ffn_hidden_dim": (_I, [_I]),
    "pswa_band_rows": (_I, [_I, _I, _I, C.POINTER(_I), C.POINTER(_I)]),
    "pswa_group_create": (_I, [_VP, _I, C.POINTER(PswaCfg), _VP, _SZ, C.POINTER(_VP)]),
    "pswa_group_destroy": (None, [_VP]),
    "pswa_group_reset_gop": (_I, [_VP]),
    "pswa_group_push_frame": (_I, [_VP, _VP, _I]),
    "pswa_group_encode_frame": (_I, [_VP, _VP, _VP, _I, _I, _VP, _SZ, C.POINTER(_SZ), _VP, _SZ,
                                     C.POINTER(_SZ), _D]),
    "pswa_group_decode_frame": (_I, [_VP, _VP, _SZ, _VP, _SZ, _I, _I, _I, _VP, _D]),
    "pswa_group_forward_params": (_I, [_VP, _VP, _VP, _I, _I, _VP, _VP, _D]),
    "pswa_group_last_zhat": (_I, [_VP, _VP]),
    "pswa_group_last_launch_count": (_I, [_VP]),
    "pswa_gpu_encode_sequence": (_I, [_VP, _VP, _I, _I, _I, _VP, _SZ, C.POINTER(_SZ)]),
    "pswa_gpu_decode_sequence": (_I, [_VP, _VP, _SZ, _VP, _I, _VP, _D, C.POINTER(_I)]),
    "pswa_container_info": (_I, [_VP, _SZ, C.POINTER(_I)]),
    "pswa_read_ppm": (_I, [C.c_char_p, _VP, _SZ, C.POINTER(_I), C.POINTER(_I)]),
    "pswa_write_ppm": (_I, [C.c_char_p, _VP, _I, _I]),
    "pswa_pad8": (_I, [_VP, _I, _I, _VP, C.POINTER(_I), C.POINTER(_I)]),
    "pswa_toy_analysis": (_I, [_VP, _I, _I, _I, _VP]),
    "pswa_toy_synthesis": (_I, [_VP, _I, _I, _I, _VP]),
    "pswa_gpu_create_band": (_I, [_I, C.POINTER(PswaCfg), _VP, _SZ, _I, _I, C.POINTER(_VP)]),
    "pswa_gpu_band_export": (_I, [_VP, _VP, _SZ, C.POINTER(_SZ)]),
    "pswa_gpu_band_link": (_I, [_VP, _VP, _SZ, _VP, _SZ]),
}


def lib():
    """Load the library (once). Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int):
    if code != PSWA_OK:
        msg = lib().pswa_gpu_last_error()
        raise PswaError(code, msg.decode() if msg else "")


def exported_symbols():
    return [n for n in _SIGS if hasattr(lib(), n)]
