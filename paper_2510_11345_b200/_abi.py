"""ctypes view of include/rf_offpolicy.h and the loader of librf_offpolicy.so.

The shared library is the product: CUDA kernels for sm_100a behind a C ABI.  It
is built in-tree by ``make -C paper_2510_11345_b200`` (``__graft_entry__.build``)
and loaded from the package directory only — there is no CPU fallback, so a
missing library is a hard ImportError.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# RF_LIB_VARIANT=<name> loads an experiment build librf_offpolicy_<name>.so (e.g. "phase":
# per-phase cycle counters compiled in; see the Makefile's `variant` target).
_VARIANT = os.environ.get("RF_LIB_VARIANT")
LIB_PATH = os.path.join(_HERE, f"librf_offpolicy_{_VARIANT}.so" if _VARIANT else "librf_offpolicy.so")

# enums (rf_offpolicy.h)
RF_PPO, RF_DECOUPLED_PPO, RF_TIS, RF_CISPO, RF_TOPR, RF_GRPO, RF_NAIVE_IS = range(7)
RF_TOKEN_MEAN, RF_SEQUENCE_PRODUCT = 0, 1
RF_NORM_SEQ_THEN_BATCH, RF_NORM_GLOBAL_TOKEN = 0, 1
RF_DTYPE_BF16, RF_DTYPE_F32, RF_DTYPE_F64 = 0, 1, 2
RF_KERNEL_AUTO, RF_KERNEL_RING, RF_KERNEL_GENERIC = 0, 1, 2

RF_OK = 0
RF_ERR_CLIP_EPS = 1
RF_ERR_EPS_LOW_HIGH = 2
RF_ERR_TRUNC_CAP = 3
RF_ERR_KL_WEIGHT = 4
RF_ERR_TOPR_WEIGHTS = 5
RF_ERR_MISMATCH_CAP = 6
RF_ERR_EMPTY_BATCH = 7
RF_ERR_MISSING_PROX = 8
RF_ERR_MISSING_REF = 9
RF_ERR_EMPTY_TRAJECTORY = 10
RF_ERR_MISSING_ENGINE_LOGP = 11
RF_ERR_NONFINITE_RATIO = 12
RF_ERR_GROUP_TOO_SMALL = 13
RF_ERR_UNKNOWN_VARIANT = 14
RF_ERR_INVALID_ARGUMENT = 15
RF_ERR_UNSUPPORTED_LAYOUT = 16
RF_ERR_TOKEN_OUT_OF_RANGE = 17
RF_ERR_WORKSPACE_TOO_SMALL = 18
RF_ERR_CUDA = 19

RF_DEVSTAT_NONFINITE_RATIO = 0x1
RF_DEVSTAT_TOKEN_OUT_OF_RANGE = 0x2
RF_DEVSTAT_GROUP_TOO_SMALL = 0x4
RF_DEVSTAT_EMPTY_TRAJECTORY = 0x8

RF_FLAG_CLIPPED = 0x01
RF_FLAG_TOPR_POS = 0x02
RF_FLAG_MISMATCH_CAPPED = 0x04
RF_FLAG_NONFINITE = 0x08
RF_FLAG_ZERO_COEF = 0x10

RF_SCALAR_LOSS, RF_SCALAR_TOKENS, RF_SCALAR_CLIPPED, RF_SCALAR_NONFINITE = 0, 1, 2, 3
RF_SCALAR_ZERO_COEF, RF_SCALAR_MISMATCH, RF_SCALAR_KL, RF_SCALAR_COEF_ABS = 4, 5, 6, 7
RF_NUM_SCALARS = 8

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class rf_loss_config(ctypes.Structure):
    _fields_ = [
        ("variant", _i32),
        ("aggregation", _i32),
        ("clip_eps", _f64),
        ("eps_low", _f64),
        ("eps_high", _f64),
        ("trunc_cap", _f64),
        ("kl_weight", _f64),
        ("w_plus", _f64),
        ("w_minus", _f64),
        ("engine_mismatch_cap", _f64),
    ]


class rf_batch(ctypes.Structure):
    _fields_ = [
        ("num_tokens", _i64),
        ("num_seqs", _i64),
        ("num_groups", _i64),
        ("vocab", _i32),
        ("logits_dtype", _i32),
        ("logits", _p),
        ("logits_row_stride", _i64),
        ("row_of_token", _p),
        ("token_ids", _p),
        ("seq_of_token", _p),
        ("seq_offsets", _p),
        ("group_offsets", _p),
        ("rewards", _p),
        ("advantages", _p),
        ("logp_dtype", _i32),
        ("normalization", _i32),
        ("behavior_logp", _p),
        ("prox_logp", _p),
        ("engine_logp", _p),
        ("ref_logits", _p),
        ("ref_row_stride", _i64),
        ("global_num_seqs", _i64),
        ("global_num_tokens", _i64),
        ("grad_sign", _f64),
    ]


class rf_outputs(ctypes.Structure):
    _fields_ = [
        ("dlogits", _p),
        ("dlogits_dtype", _i32),
        ("_pad0", _i32),
        ("dlogits_row_stride", _i64),
        ("token_logp", _p),
        ("token_ratio", _p),
        ("token_coef", _p),
        ("token_loss", _p),
        ("token_flags", _p),
        ("advantages_out", _p),
        ("group_degenerate", _p),
        ("scalars", _p),
        ("device_status", _p),
        ("workspace", _p),
        ("workspace_bytes", ctypes.c_size_t),
    ]


EXPORTED_SYMBOLS = (
    "rf_loss_config_default",
    "rf_loss_config_validate",
    "rf_loss_variant_name",
    "rf_loss_variant_from_name",
    "rf_status_string",
    "rf_workspace_bytes",
    "rf_grpo_advantages",
    "rf_zero_scalars",
    "rf_loss_and_grad",
    "rf_loss_and_grad_ex",
    "rf_last_launch_count",
    "rf_loss_and_grad_host",
    "rf_debug_counters",
    "rf_lmhead_lse",
    "rf_lmhead_dlogits",
    "rf_token_loss_from_stats",
    "rf_rows_segment_sum",
)

_lib = None


def require_library(path: str = LIB_PATH) -> None:
    """Raise ImportError if librf_offpolicy.so was not built (no CPU fallback)."""
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C {_HERE}` (or __graft_entry__.build()); "
            "there is no CPU fallback for the off-policy loss path"
        )


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Map librf_offpolicy.so (once per process; raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    require_library(path)
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.rf_loss_config_default.argtypes = [P(rf_loss_config)]
    lib.rf_loss_config_default.restype = None
    lib.rf_loss_config_validate.argtypes = [P(rf_loss_config)]
    lib.rf_loss_config_validate.restype = _i32
    lib.rf_loss_variant_name.argtypes = [_i32]
    lib.rf_loss_variant_name.restype = ctypes.c_char_p
    lib.rf_loss_variant_from_name.argtypes = [ctypes.c_char_p, P(_i32)]
    lib.rf_loss_variant_from_name.restype = _i32
    lib.rf_status_string.argtypes = [_i32]
    lib.rf_status_string.restype = ctypes.c_char_p
    lib.rf_workspace_bytes.argtypes = [P(rf_loss_config), P(rf_batch)]
    lib.rf_workspace_bytes.restype = ctypes.c_size_t
    lib.rf_grpo_advantages.argtypes = [P(rf_batch), P(rf_outputs), _p]
    lib.rf_grpo_advantages.restype = _i32
    lib.rf_zero_scalars.argtypes = [P(rf_outputs), _p]
    lib.rf_zero_scalars.restype = _i32
    lib.rf_loss_and_grad.argtypes = [P(rf_loss_config), P(rf_batch), P(rf_outputs), _p]
    lib.rf_loss_and_grad.restype = _i32
    lib.rf_loss_and_grad_ex.argtypes = [P(rf_loss_config), P(rf_batch), P(rf_outputs), _p, _i32]
    lib.rf_loss_and_grad_ex.restype = _i32
    lib.rf_last_launch_count.argtypes = []
    lib.rf_last_launch_count.restype = _i32
    lib.rf_loss_and_grad_host.argtypes = [P(rf_loss_config), P(rf_batch), P(rf_outputs), _i32, _i64]
    lib.rf_loss_and_grad_host.restype = _i32
    lib.rf_lmhead_lse.argtypes = [_p, _p, _p, _i64, _i32, _i32, _p, _p, _p]
    lib.rf_lmhead_lse.restype = _i32
    lib.rf_lmhead_dlogits.argtypes = [_p, _p, _p, _i64, _i32, _i32, _p, _p, _p, _i64, _p]
    lib.rf_lmhead_dlogits.restype = _i32
    lib.rf_token_loss_from_stats.argtypes = [P(rf_loss_config), P(rf_batch), _p, _p, P(rf_outputs), _p]
    lib.rf_token_loss_from_stats.restype = _i32
    lib.rf_rows_segment_sum.argtypes = [_p, _i32, _i64, _p, _p, _i64, _i32, _p, _i64, _p]
    lib.rf_rows_segment_sum.restype = _i32
    lib.rf_debug_counters.argtypes = [_p, _i32, _i32]
    lib.rf_debug_counters.restype = _i32
    _lib = lib
    return lib
