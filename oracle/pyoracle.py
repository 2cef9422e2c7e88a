"""ctypes bindings of the two CPU checkers (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "_build", "librf_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "librlsim_ref.so")

_P = ctypes.c_void_p
_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double


def build(quiet: bool = True) -> None:
    """make -C oracle (the reference part only when /root/reference exists)."""
    subprocess.run(["make", "-C", _HERE], check=True, capture_output=quiet)


class rfo_config(ctypes.Structure):
    _fields_ = [("variant", _i32), ("aggregation", _i32), ("clip_eps", _f64), ("eps_low", _f64),
                ("eps_high", _f64), ("trunc_cap", _f64), ("kl_weight", _f64), ("w_plus", _f64),
                ("w_minus", _f64), ("engine_mismatch_cap", _f64)]


class rfo_batch(ctypes.Structure):
    _fields_ = [("num_tokens", _i64), ("num_seqs", _i64), ("vocab", _i32), ("normalization", _i32),
                ("logits", _P), ("row_stride", _i64), ("row_of_token", _P), ("ref_logits", _P),
                ("ref_row_stride", _i64), ("token_ids", _P), ("seq_offsets", _P), ("advantages", _P),
                ("behavior_logp", _P), ("prox_logp", _P), ("engine_logp", _P), ("global_num_seqs", _i64),
                ("global_num_tokens", _i64), ("grad_sign", _f64)]


class rfo_outputs(ctypes.Structure):
    _fields_ = [("dlogits", _P), ("dlogits_row_stride", _i64), ("token_logp", _P), ("token_ratio", _P),
                ("token_coef", _P), ("token_loss", _P), ("token_flags", _P), ("value", _P)]


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _oracle = ctypes.CDLL(ORACLE_SO)
        _oracle.rfo_loss_and_grad.restype = _i32
        _oracle.rfo_loss_and_grad.argtypes = [ctypes.POINTER(rfo_config), ctypes.POINTER(rfo_batch),
                                              ctypes.POINTER(rfo_outputs)]
        _oracle.rfo_grpo_advantages.restype = _i32
        _oracle.rfo_grpo_advantages.argtypes = [_P, _P, _i64, _P, _P]
        _oracle.rfo_log_softmax.restype = None
        _oracle.rfo_log_softmax.argtypes = [_P, _i32, _P]
        _oracle.rfo_validate.restype = _i32
        _oracle.rfo_validate.argtypes = [ctypes.POINTER(rfo_config)]
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


GPU_SHIM_SO = os.path.join(os.path.dirname(_HERE), "integration", "_build", "librlsim_gpu.so")
_shim = None


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise OSError("oracle/_ref/librlsim_ref.so not built (reference sources absent)")
        _ref = _bind(ctypes.CDLL(REF_SO))
    return _ref


def gpu_shim_available() -> bool:
    return os.path.exists(GPU_SHIM_SO)


def gpu_shim_lib():
    """The reference's own code (bandit/policy/rng/engine/gradcheck) linked against
    integration/rlsim_gpu_shim.cpp — rlsim's loss API on the GPU (integration/Makefile)."""
    global _shim
    if _shim is None:
        _shim = _bind(ctypes.CDLL(GPU_SHIM_SO))
    return _shim


def _bind(L):
    if True:
        L.ref_grpo_advantages.restype = _i32
        L.ref_grpo_advantages.argtypes = [_P, _i64, _P, _P, ctypes.c_char_p, ctypes.c_int]
        L.ref_variant_from_string.restype = _i32
        L.ref_variant_from_string.argtypes = [ctypes.c_char_p, _P, ctypes.c_char_p, ctypes.c_int]
        L.ref_variant_to_string.restype = ctypes.c_char_p
        L.ref_variant_to_string.argtypes = [_i32]
        L.ref_validate.restype = _i32
        L.ref_validate.argtypes = [_i32, _i32, _P, ctypes.c_char_p, ctypes.c_int]
        L.ref_loss_and_grad.restype = _i32
        L.ref_loss_and_grad.argtypes = [_i32, _i32, _P, _i32, _i32, _P, _P, _P, _i64, _P, _P, _P, _P, _P, _P,
                                        _P, _P, ctypes.c_char_p, ctypes.c_int]
        L.ref_log_probs.restype = _i32
        L.ref_log_probs.argtypes = [_i32, _i32, _P, _i64, _P, _P]
        L.ref_trajectory_ratio.restype = _i32
        L.ref_trajectory_ratio.argtypes = [_i32, _i32, _P, _i32, _i64, _P, _P, _P, _P, ctypes.c_char_p,
                                           ctypes.c_int]
        L.ref_finite_diff.restype = _i32
        L.ref_finite_diff.argtypes = [_i32, _i32, _P, _i32, _i32, _P, _P, _P, _i64, _P, _P, _P, _P, _P, _P, _f64,
                                      _P, _P, _P, ctypes.c_char_p, ctypes.c_int]
        L.ref_build_prox_table.restype = None
        L.ref_build_prox_table.argtypes = [_i32, _i32, _P, _P, _P, _P]
        L.ref_bench_mapping_a.restype = _f64
        L.ref_bench_mapping_a.argtypes = [_i32, _i32, _P, _i32, _i32, _P, _P, _P, _P, _P, _P, _i32, _P]
        L.ref_train_loop.restype = _i32
        L.ref_train_loop.argtypes = [_i32, _i32, _i32, _i32, _i32, _f64, _f64, _i64, ctypes.c_uint64, _i32, _i32,
                                     _P, _P, _P, _P, _P, _P, ctypes.c_char_p, ctypes.c_int]
        L.ref_rng_draws.restype = None
        L.ref_rng_draws.argtypes = [ctypes.c_uint64, ctypes.c_char_p, _i32, _i64, _P]
    return L


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def config_params(cfg) -> np.ndarray:
    """8-double parameter pack [clip_eps, eps_low, eps_high, trunc_cap, kl_weight, w_plus, w_minus, cap]."""
    return np.array([cfg.clip_eps, cfg.eps_low, cfg.eps_high, cfg.trunc_cap, cfg.kl_weight, cfg.w_plus,
                     cfg.w_minus, cfg.engine_mismatch_cap], dtype=np.float64)


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------
def oracle_grpo(rewards, group_offsets):
    r = _c(rewards, np.float64)
    go = _c(group_offsets, np.int64)
    adv = np.zeros_like(r)
    deg = np.zeros(len(go) - 1, dtype=np.uint8)
    st = oracle_lib().rfo_grpo_advantages(_ptr(r), _ptr(go), len(go) - 1, _ptr(adv), _ptr(deg))
    return st, adv, deg


def oracle_log_softmax(row):
    r = _c(row, np.float64)
    out = np.empty_like(r)
    oracle_lib().rfo_log_softmax(_ptr(r), len(r), _ptr(out))
    return out


def oracle_loss_and_grad(cfg, logits, token_ids, seq_offsets, advantages, behavior_logp, *, prox_logp=None,
                         engine_logp=None, row_of_token=None, ref_logits=None, normalization=0,
                         global_num_seqs=None, global_num_tokens=None, grad_sign=1.0, want_dlogits=True,
                         vocab=None):
    """Run rf_oracle.c. logits: [R, >=V] float64 rows.  Returns a dict."""
    lg = _c(logits, np.float64)
    V = int(vocab if vocab is not None else lg.shape[1])
    tok = _c(token_ids, np.int32)
    offs = _c(seq_offsets, np.int64)
    T = len(tok)
    N = len(offs) - 1
    adv = _c(advantages, np.float64)
    beh = _c(behavior_logp, np.float64)
    prox = _c(prox_logp, np.float64)
    eng = _c(engine_logp, np.float64)
    rows = _c(row_of_token, np.int32)
    ref = _c(ref_logits, np.float64)
    c = rfo_config(int(cfg.variant), int(cfg.aggregation), cfg.clip_eps, cfg.eps_low, cfg.eps_high, cfg.trunc_cap,
                   cfg.kl_weight, cfg.w_plus, cfg.w_minus, cfg.engine_mismatch_cap)
    b = rfo_batch()
    b.num_tokens, b.num_seqs, b.vocab, b.normalization = T, N, V, int(normalization)
    b.logits, b.row_stride = _ptr(lg), lg.shape[1]
    b.row_of_token = _ptr(rows)
    b.ref_logits = _ptr(ref)
    b.ref_row_stride = 0 if ref is None else ref.shape[1]
    b.token_ids, b.seq_offsets, b.advantages = _ptr(tok), _ptr(offs), _ptr(adv)
    b.behavior_logp, b.prox_logp, b.engine_logp = _ptr(beh), _ptr(prox), _ptr(eng)
    b.global_num_seqs = N if global_num_seqs is None else global_num_seqs
    b.global_num_tokens = T if global_num_tokens is None else global_num_tokens
    b.grad_sign = grad_sign
    out = {
        "dlogits": np.zeros((T, V), dtype=np.float64) if want_dlogits else None,
        "token_logp": np.zeros(T), "token_ratio": np.zeros(T), "token_coef": np.zeros(T),
        "token_loss": np.zeros(T), "token_flags": np.zeros(T, dtype=np.uint8), "value": np.zeros(1),
    }
    o = rfo_outputs(_ptr(out["dlogits"]), V, _ptr(out["token_logp"]), _ptr(out["token_ratio"]),
                    _ptr(out["token_coef"]), _ptr(out["token_loss"]), _ptr(out["token_flags"]),
                    _ptr(out["value"]))
    out["status"] = oracle_lib().rfo_loss_and_grad(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o))
    out["value"] = float(out["value"][0])
    return out


# ---------------------------------------------------------------------------
# The reference itself (oracle/_ref)
# ---------------------------------------------------------------------------
def _err():
    return ctypes.create_string_buffer(512)


def ref_grpo_advantages(rewards):
    r = _c(rewards, np.float64)
    out = np.zeros_like(r)
    deg = np.zeros(1, dtype=np.uint8)
    e = _err()
    st = ref_lib().ref_grpo_advantages(_ptr(r), len(r), _ptr(out), _ptr(deg), e, 512)
    if st:
        raise ValueError(e.value.decode())
    return out, bool(deg[0])


def ref_variant_from_string(name: str) -> int:
    out = np.zeros(1, dtype=np.int32)
    e = _err()
    if ref_lib().ref_variant_from_string(name.encode(), _ptr(out), e, 512):
        raise ValueError(e.value.decode())
    return int(out[0])


def ref_validate(cfg) -> Optional[str]:
    e = _err()
    p = config_params(cfg)
    if ref_lib().ref_validate(int(cfg.variant), int(cfg.aggregation), _ptr(p), e, 512):
        return e.value.decode()
    return None


def ref_loss_and_grad(cfg, logits, traj_context, traj_offsets, tokens, advantages, behavior_logp, *,
                      prox_logits=None, ref_logits=None, engine_logp=None, want_grad=True, lib=None):
    """rlsim::loss_and_grad over trajectories; logits [C, V] fp64.  Returns (value, grad) or raises."""
    lg = _c(logits, np.float64)
    C, V = lg.shape
    ctx = _c(traj_context, np.int32)
    offs = _c(traj_offsets, np.int64)
    tok = _c(tokens, np.int32)
    adv = _c(advantages, np.float64)
    beh = _c(behavior_logp, np.float64)
    eng = _c(engine_logp, np.float64)
    prox = _c(prox_logits, np.float64)
    ref = _c(ref_logits, np.float64)
    grad = np.zeros((C, V), dtype=np.float64) if want_grad else None
    val = np.zeros(1)
    e = _err()
    p = config_params(cfg)
    st = (lib or ref_lib()).ref_loss_and_grad(int(cfg.variant), int(cfg.aggregation), _ptr(p), C, V, _ptr(lg), _ptr(prox),
                                     _ptr(ref), len(ctx), _ptr(ctx), _ptr(offs), _ptr(tok), _ptr(adv), _ptr(beh),
                                     _ptr(eng), _ptr(val), _ptr(grad), e, 512)
    if st:
        raise ValueError(e.value.decode())
    return float(val[0]), grad


def ref_log_probs(logits, rows):
    lg = _c(logits, np.float64)
    C, V = lg.shape
    r = _c(rows, np.int32)
    out = np.zeros((len(r), V))
    ref_lib().ref_log_probs(C, V, _ptr(lg), len(r), _ptr(r), _ptr(out))
    return out


def ref_trajectory_ratio(logits, context, tokens, behavior_logp):
    lg = _c(logits, np.float64)
    C, V = lg.shape
    tok = _c(tokens, np.int32)
    beh = _c(behavior_logp, np.float64)
    per = np.zeros(len(tok))
    prod = np.zeros(1)
    e = _err()
    if ref_lib().ref_trajectory_ratio(C, V, _ptr(lg), int(context), len(tok), _ptr(tok), _ptr(beh), _ptr(per),
                                      _ptr(prod), e, 512):
        raise ValueError(e.value.decode())
    return per, float(prod[0])


def ref_build_prox_table(logits, tokens, lq):
    """Prox table (one row per token) whose log-softmax at tokens[c] equals lq[c]."""
    lg = _c(logits, np.float64)
    R, V = lg.shape
    tok = _c(tokens, np.int32)
    q = _c(lq, np.float64)
    out = np.empty_like(lg)
    ref_lib().ref_build_prox_table(R, V, _ptr(lg), _ptr(tok), _ptr(q), _ptr(out))
    return out


def ref_bench_mapping_a(cfg, logits, tokens, advantages, behavior_logp, *, prox_logits=None, engine_logp=None,
                        threads=1, reps=1):
    """Wall seconds of `reps` reference loss_and_grad calls over mapping-A rows on `threads` threads."""
    lg = _c(logits, np.float64)
    R, V = lg.shape
    tok = _c(tokens, np.int32)
    adv = _c(advantages, np.float64)
    beh = _c(behavior_logp, np.float64)
    prox = _c(prox_logits, np.float64)
    eng = _c(engine_logp, np.float64)
    val = np.zeros(1)
    p = config_params(cfg)
    secs = ref_lib().ref_bench_mapping_a(int(threads), int(cfg.variant), _ptr(p), R, V, _ptr(lg), _ptr(prox),
                                         _ptr(tok), _ptr(adv), _ptr(beh), _ptr(eng), int(reps), _ptr(val))
    return secs, float(val[0])


def ref_train_loop(cfg, *, contexts=4, arms=10, group_size=8, traj_len=1, steps=200, lr=0.5, reward_noise=0.0,
                   async_lag=0, seed=0, lib=None):
    p = config_params(cfg)
    fr = np.zeros(1)
    gv = np.zeros(1)
    cr = np.zeros(steps)
    cg = np.zeros(steps)
    cs = np.zeros(steps, dtype=np.int64)
    e = _err()
    if (lib or ref_lib()).ref_train_loop(contexts, arms, group_size, traj_len, steps, lr, reward_noise, async_lag, seed,
                                int(cfg.variant), int(cfg.aggregation), _ptr(p), _ptr(fr), _ptr(gv), _ptr(cr),
                                _ptr(cg), _ptr(cs), e, 512):
        raise ValueError(e.value.decode())
    return {"final_reward": float(fr[0]), "grad_norm_variance": float(gv[0]), "reward": cr, "grad_norm": cg,
            "staleness": cs}


def ref_finite_diff(cfg, logits, traj_context, traj_offsets, tokens, advantages, behavior_logp, *, h=1e-5,
                    prox_logits=None, ref_logits=None, engine_logp=None):
    lg = _c(logits, np.float64)
    C, V = lg.shape
    ctx = _c(traj_context, np.int32)
    offs = _c(traj_offsets, np.int64)
    tok = _c(tokens, np.int32)
    adv = _c(advantages, np.float64)
    beh = _c(behavior_logp, np.float64)
    eng = _c(engine_logp, np.float64)
    prox = _c(prox_logits, np.float64)
    ref = _c(ref_logits, np.float64)
    mre = np.zeros(1)
    chk = np.zeros(1, dtype=np.int64)
    flg = np.zeros(1, dtype=np.int64)
    e = _err()
    p = config_params(cfg)
    if ref_lib().ref_finite_diff(int(cfg.variant), int(cfg.aggregation), _ptr(p), C, V, _ptr(lg), _ptr(prox),
                                 _ptr(ref), len(ctx), _ptr(ctx), _ptr(offs), _ptr(tok), _ptr(adv), _ptr(beh),
                                 _ptr(eng), h, _ptr(mre), _ptr(chk), _ptr(flg), e, 512):
        raise ValueError(e.value.decode())
    return float(mre[0]), int(chk[0]), int(flg[0])


def ref_rng_draws(seed: int, name: str, kind: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    ref_lib().ref_rng_draws(seed, name.encode(), kind, n, _ptr(out))
    if kind == 2:
        return out.view(np.uint64)
    return out
