"""ctypes binding of libdpipe.so (the C ABI declared in include/dpipe.h).

The library is built in-tree by ``make`` (see ``__graft_entry__.build``).
There is no fallback: if the shared object is missing or a call fails, the
caller gets an exception.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DP_LIB_PATH") or os.path.join(_HERE, "libdpipe.so")  # override: A/B kernel experiments

DP_F32 = 0
DP_BF16 = 1
DP_OUT_STORE = 0
DP_OUT_ATOMIC_ADD = 1
DP_ACT_NONE, DP_ACT_GELU, DP_ACT_GELU_TANH, DP_ACT_SILU = 0, 1, 2, 3

c_int, c_i64, c_float, c_void_p = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class DpGemmArgs(ctypes.Structure):
    _fields_ = [
        ("M", c_int), ("N", c_int), ("K", c_int),
        ("batch1", c_int), ("batch2", c_int),
        ("dtype", c_int),
        ("A", c_void_p), ("a_ld", c_i64), ("a_bs1", c_i64), ("a_bs2", c_i64), ("a_mn_major", c_int),
        ("B", c_void_p), ("b_ld", c_i64), ("b_bs1", c_i64), ("b_bs2", c_i64), ("b_mn_major", c_int),
        ("D", c_void_p), ("d_dtype", c_int), ("d_ld", c_i64), ("d_bs1", c_i64), ("d_bs2", c_i64),
        ("out_mode", c_int),
        ("bias", c_void_p),
        ("Res", c_void_p), ("r_ld", c_i64), ("r_bs1", c_i64), ("r_bs2", c_i64),
        ("alpha", c_float),
        ("split_k", c_int),
        ("workspace", c_void_p), ("workspace_bytes", c_i64),
        ("geglu_out", c_void_p), ("geglu_ld", c_i64), ("geglu_mode", c_int),
    ]


class DpConvArgs(ctypes.Structure):
    _fields_ = [
        ("dtype", c_int),
        ("N", c_int), ("H", c_int), ("W", c_int), ("C", c_int),
        ("K", c_int), ("R", c_int), ("S", c_int),
        ("stride", c_int), ("pad_h", c_int), ("pad_w", c_int),
        ("P", c_int), ("Q", c_int),
        ("x", c_void_p), ("w", c_void_p), ("y", c_void_p),
        ("bias", c_void_p), ("Res", c_void_p),
        ("alpha", c_float),
        ("out_mode", c_int),
        ("split_k", c_int),
        ("workspace", c_void_p), ("workspace_bytes", c_i64),
        ("gn_sums", c_void_p), ("gn_groups", c_int),
    ]


class DpAttnArgs(ctypes.Structure):
    _fields_ = [
        ("dtype", c_int), ("B", c_int), ("N", c_int), ("Nk", c_int), ("heads", c_int), ("head_dim", c_int),
        ("q", c_void_p), ("k", c_void_p), ("v", c_void_p), ("o", c_void_p),
        ("q_ld", c_i64), ("q_bs", c_i64), ("kv_ld", c_i64), ("kv_bs", c_i64), ("o_ld", c_i64), ("o_bs", c_i64),
        ("scale", c_float), ("lse", c_void_p), ("causal", c_int),
    ]


class DpFlipJob(ctypes.Structure):
    _fields_ = [("w", c_void_p), ("wt", c_void_p), ("K", c_int), ("R", c_int), ("S", c_int), ("C", c_int)]


# name -> argtypes (restype is always c_int unless listed in _RESTYPES)
_SIGNATURES = {
    "dp_gemm": [ctypes.POINTER(DpGemmArgs), c_void_p],
    "dp_gemm_workspace": [ctypes.POINTER(DpGemmArgs)],
    "dp_conv_fwd_workspace": [ctypes.POINTER(DpConvArgs)],
    "dp_conv_dgrad_workspace": [ctypes.POINTER(DpConvArgs)],
    "dp_conv_fwd": [ctypes.POINTER(DpConvArgs), c_void_p],
    "dp_conv_wgrad": [ctypes.POINTER(DpConvArgs), c_void_p],
    "dp_conv_dgrad": [ctypes.POINTER(DpConvArgs), c_void_p],
    "dp_flash_attn_fwd": [ctypes.POINTER(DpAttnArgs), c_void_p],
    "dp_flash_attn_bwd_workspace": [ctypes.POINTER(DpAttnArgs)],
    "dp_flash_attn_bwd": [ctypes.POINTER(DpAttnArgs), c_void_p, c_i64, c_void_p, c_i64, c_void_p, c_void_p,
                          c_i64, c_void_p, c_void_p],
    "dp_im2col": [c_int, c_void_p, c_void_p] + [c_int] * 11 + [c_void_p],
    "dp_col2im": [c_int, c_void_p, c_void_p] + [c_int] * 11 + [c_void_p],
    "dp_conv_weight_flip": [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
    "dp_dilate": [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p],
    # eltwise.cu
    "dp_act_fwd": [c_int, c_int, c_void_p, c_void_p, c_i64, c_void_p],
    "dp_act_bwd": [c_int, c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_void_p],
    "dp_geglu_fwd": [c_int, c_void_p, c_void_p, c_i64, c_int, c_void_p],
    "dp_geglu_bwd": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_void_p],
    "dp_geglu_bwd_db": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_void_p, c_void_p],
    "dp_axpby": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_float, c_float, c_void_p],
    "dp_gate_residual_fwd": [c_int, c_void_p, c_void_p, c_i64, c_void_p, c_void_p, c_i64, c_int,
                             c_int, c_void_p],
    "dp_gate_residual_bwd": [c_int, c_void_p, c_void_p, c_i64, c_void_p, c_void_p, c_void_p, c_i64,
                             c_int, c_int, c_int, c_void_p],
    "dp_q_sample": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64,
                    c_void_p],
    "dp_pred_x0": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64,
                   c_void_p],
    "dp_mse": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_float, c_void_p],
    "dp_timestep_embed": [c_int, c_void_p, c_void_p, c_int, c_int, c_float, c_void_p],
    "dp_embed": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_int, c_void_p],
    "dp_concat": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_int, c_void_p],
    "dp_split": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_int, c_int, c_int, c_void_p],
    "dp_upsample2x": [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
    "dp_upsample2x_bwd": [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p],
    "dp_row_bias_fwd": [c_int, c_void_p, c_void_p, c_i64, c_void_p, c_i64, c_int, c_int, c_void_p],
    "dp_row_bias_bwd": [c_int, c_void_p, c_void_p, c_i64, c_int, c_int, c_int, c_void_p],
    "dp_row_bias_bwd_db": [c_int, c_void_p, c_void_p, c_i64, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p],
    "dp_space_to_depth": [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p],
    "dp_bias_grad": [c_int, c_void_p, c_void_p, c_i64, c_int, c_void_p],
    "dp_cast": [c_int, c_int, c_void_p, c_void_p, c_i64, c_void_p],
    "dp_adamw": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_float, c_float, c_float,
                 c_float, c_float, c_int, c_float, c_void_p],
    "dp_adamw_advance": [c_void_p, c_float, c_float, c_void_p, c_void_p],
    "dp_adamw_apply": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_float, c_float, c_float,
                       c_float, c_float, c_void_p, c_float, c_int, c_int, c_void_p],
    "dp_adamw_dev": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_float, c_float, c_float,
                     c_float, c_float, c_void_p, c_void_p, c_float, c_void_p],
    # norm.cu
    "dp_group_norm_workspace": [c_int, c_int, c_int],
    "dp_group_norm_fwd": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                          c_int, c_int, c_int, c_float, c_int, c_void_p, c_void_p],
    "dp_group_norm_fwd_sums": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                               c_int, c_int, c_int, c_float, c_int, c_void_p, c_void_p],
    "dp_group_norm_bwd": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                          c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_void_p, c_void_p],
    "dp_layer_norm_fwd": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_int, c_int,
                          c_void_p, c_void_p, c_void_p, c_i64, c_int, c_float, c_void_p],
    "dp_layer_norm_bwd": [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_int, c_int,
                          c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_i64,
                          c_int, c_int, c_void_p],
    "dp_rms_norm_fwd": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_float, c_void_p],
    "dp_softmax_fwd": [c_int, c_void_p, c_void_p, c_i64, c_int, c_int, c_float, c_int, c_int, c_void_p],
    "dp_softmax_bwd": [c_int, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_int, c_float, c_void_p],
    "dp_conv_weight_flip_batch": [ctypes.POINTER(DpFlipJob), c_int, c_void_p],
    # timing.cu
    "dp_timing_events": [c_int],
    "dp_timing_record": [c_int, c_void_p],
    "dp_timing_elapsed": [c_int, c_int],
    "dp_last_error": [],
    "dp_version": [],
}
_RESTYPES = {"dp_last_error": ctypes.c_char_p, "dp_timing_elapsed": c_float, "dp_group_norm_workspace": ctypes.c_size_t,
             "dp_gemm_workspace": c_i64, "dp_flash_attn_bwd_workspace": c_i64, "dp_conv_fwd_workspace": c_i64, "dp_conv_dgrad_workspace": c_i64}

_lib = None


class DpipeError(RuntimeError):
    pass


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def register(name: str, argtypes: list, restype=ctypes.c_int) -> None:
    """Declare an additional C-ABI entry point (used by kernel-family modules)."""
    _SIGNATURES[name] = argtypes
    if restype is not ctypes.c_int:
        _RESTYPES[name] = restype
    if _lib is not None:
        _bind(_lib, name)


def _bind(lib, name):
    fn = getattr(lib, name)
    fn.argtypes = _SIGNATURES[name]
    fn.restype = _RESTYPES.get(name, ctypes.c_int)


_telemetry = None


def _tele():
    global _telemetry
    if _telemetry is None:
        from . import telemetry

        _telemetry = telemetry
    return _telemetry


def lib():
    """Load libdpipe.so once; raise loudly when it is missing. While the bench's kernel timer
    is active, calls go through a proxy that brackets each launch with CUDA events."""
    global _lib
    if _lib is not None:
        telemetry = _tele()
        if telemetry.timer.active:
            return telemetry.TimedLib(_lib)
        return _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DpipeError(
                f"{LIB_PATH} not found: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`)"
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name in _SIGNATURES:
            _bind(handle, name)
        _lib = handle
    return _lib


def check(rc: int, what: str, kernels: int = 1) -> None:
    _tele().count(what, kernels)
    if rc != 0:
        msg = lib().dp_last_error().decode(errors="replace")
        raise DpipeError(f"{what} failed (code {rc}): {msg}")
