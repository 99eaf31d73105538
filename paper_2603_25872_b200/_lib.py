"""ctypes binding of libdrs.so (include/drs.h).

The product path has no CPU fallback: importing a compute entry point without
the built library, or calling one without a CUDA device, raises
`NativeLibraryMissing` / `RuntimeError` immediately.
"""

import ctypes
import os

from . import errors

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdrs.so")

# ---- constants mirrored from include/drs.h -------------------------------
DRS_OK = 0
GEN_PCG64 = 0
GEN_SFC64 = 1
FAMILY_DDIM = 0
GEMM_KB2_DEFAULT = 0          # drs_set_gemm_kb2 default (csrc/gemm_tc.cu gemm_kb2_mode)
FAMILY_DDPM = 1
FAMILY_DDPM_X0 = 2
FAMILY_PRED_X0 = 3
FAMILY_EULER = 4
SRC_X = 0
SRC_CUR = 1
SRC_ANCHOR = 2
OP_SAVE_ANCHOR = 1
ERR_NOISE_WINDOW_BIT = 1
ERR_GM_TIMESTEP_BIT = 2
ERR_GM_SIGMA_BIT = 4             # drs_gm_velocity: sigma <= 0 (NonPositiveSigma)


class NativeLibraryMissing(RuntimeError):
    """libdrs.so is not built; run `python -m paper_2603_25872_b200._build`."""


class DrsKey(ctypes.Structure):
    _fields_ = [
        ("vals", ctypes.c_int64 * 4),
        ("n_vals", ctypes.c_int32),
        ("seed_slot", ctypes.c_int32),
        ("seed_mask", ctypes.c_uint64),
    ]


class DrsOp(ctypes.Structure):
    _fields_ = [
        ("c", ctypes.c_double * 6),
        ("family", ctypes.c_int32),
        ("noisy", ctypes.c_int32),
        ("src", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("eps_f32", ctypes.c_int32),
        ("pad", ctypes.c_int32),
        ("x", ctypes.c_void_p),
        ("eps", ctypes.c_void_p),
        ("z", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("out2", ctypes.c_void_p),
    ]


class DrsGemmArgs(ctypes.Structure):       # include/drs_net.h drs_gemm_args
    _fields_ = [
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int64),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64),
        ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
        ("act", ctypes.c_int), ("out_f32", ctypes.c_int),
        ("alpha", ctypes.c_float),
        ("bias", ctypes.c_void_p),
        ("residual", ctypes.c_void_p), ("ldr", ctypes.c_int64), ("res_f32", ctypes.c_int),
        ("colscale", ctypes.c_void_p), ("cs_group", ctypes.c_int), ("cs_ld", ctypes.c_int64),
        ("rowbias", ctypes.c_void_p), ("rb_group", ctypes.c_int), ("rb_ld", ctypes.c_int64),
        ("bn", ctypes.c_int), ("split", ctypes.c_int),
        ("workspace", ctypes.c_void_p),
        ("conv_N", ctypes.c_int), ("conv_H", ctypes.c_int), ("conv_W", ctypes.c_int), ("conv_C", ctypes.c_int),
        ("cta_pair", ctypes.c_int),
        ("b_img_rows", ctypes.c_int), ("b_img_off", ctypes.c_int), ("hs_valid", ctypes.c_int),
        ("out2", ctypes.c_void_p), ("ldo2", ctypes.c_int64),
        ("conv_stride", ctypes.c_int), ("kbox", ctypes.c_int),
    ]


assert ctypes.sizeof(DrsGemmArgs) == 224
assert ctypes.sizeof(DrsKey) == 48
assert ctypes.sizeof(DrsOp) == 112

_lib = None

_SIGS = {
    "drs_noise_fill": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p]),
    "drs_skip_chain": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p]),
    "drs_gm_eps": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p]),
    "drs_gm_velocity": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p]),
    "drs_gm_x0_mean": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_perturb_keys": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_row_sqnorm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_void_p]),
    "drs_mmd_partials": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "drs_copy_rows": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_void_p]),
    "drs_spin": (ctypes.c_int, [ctypes.c_double, ctypes.c_int, ctypes.c_void_p]),
    "drs_host_log1p": (ctypes.c_double, [ctypes.c_double]),
    "drs_host_exp": (ctypes.c_double, [ctypes.c_double]),
    "drs_host_seedseq": (ctypes.c_int, [ctypes.POINTER(DrsKey), ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_uint32), ctypes.c_int]),
    "drs_version": (ctypes.c_int, []),
    "drs_set_pdl": (ctypes.c_int, [ctypes.c_int]),
    "drs_set_early_weights": (ctypes.c_int, [ctypes.c_int]),
    "drs_set_gemm_kb2": (ctypes.c_int, [ctypes.c_int]),
    "drs_set_chain_vec": (ctypes.c_int, [ctypes.c_int]),
    "drs_set_noise_resolve": (ctypes.c_int, [ctypes.c_int]),
    "drs_set_gn_mode": (ctypes.c_int, [ctypes.c_int]),
    "drs_set_attn_split": (ctypes.c_int, [ctypes.c_int]),
    # include/drs_net.h
    "drs_gemm_bf16": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_float, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]),
    "drs_gemm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "drs_gemm_pick": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int)]),
    "drs_gemm_cost_us": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "drs_layernorm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p]),
    "drs_attention": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_float, ctypes.c_void_p]),
    "drs_attention_tc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_float, ctypes.c_void_p]),
    "drs_gemv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_void_p]),
    "drs_attention_tc_v": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_float, ctypes.c_void_p]),
    "drs_timestep_embedding": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                              ctypes.c_void_p, ctypes.c_void_p]),
    "drs_patchify": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_unpatchify": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_silu_cast": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_cast_f32_bf16": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_im2col": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_void_p, ctypes.c_void_p]),
    "drs_groupnorm_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int]),
    "drs_groupnorm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "drs_latent_to_nhwc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "drs_cfg_combine": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                       ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libdrs.so once; raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise NativeLibraryMissing(
                f"{_LIB_PATH} not built (python -m paper_2603_25872_b200._build); "
                "there is no CPU fallback")
        L = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_STATUS_EXC = {
    1: ValueError,
    2: errors.TimestepOutOfRange,
    3: errors.InvalidSkip,
    4: errors.VarianceTooLarge,
    5: errors.DimensionMismatch,
    6: errors.InvalidPlanParams,
    7: RuntimeError,
    8: RuntimeError,
}


LAUNCHES = [0]     # libdrs entry points called (== kernel launches issued); read by bench.py


def check(status: int, what: str):
    LAUNCHES[0] += 1
    if status != DRS_OK:
        exc = _STATUS_EXC.get(status, RuntimeError)
        raise exc(f"{what} failed with drs status {status}")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
