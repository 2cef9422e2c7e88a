"""CPU: the C-ABI library loads, exports every symbol include/rf_offpolicy.h
declares, and its host-side paths (registry, config validation, argument
validation mirroring the reference's throw sites) behave like the reference —
no GPU needed for any of these."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2510_11345_b200 import _abi
from paper_2510_11345_b200 import losses as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rf_offpolicy.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:rf_status|void|size_t|int32_t|const char\*)\s+(rf_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load_library()
    fns = header_functions()
    assert len(fns) >= 12
    for f in fns:
        assert hasattr(lib, f), f
    assert set(fns) == set(_abi.EXPORTED_SYMBOLS)


def test_library_is_sm100a_only():
    so = _abi.LIB_PATH
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_variant_registry_matches_reference():  # losses.cpp:8-30
    names = ["ppo", "decoupled_ppo", "tis", "cispo", "topr", "grpo", "naive_is"]
    for i, n in enumerate(names):
        assert L.to_string(i) == n
        assert L.loss_variant_from_string(n) == i
        if O.ref_available():
            assert O.ref_variant_from_string(n) == i
            assert O.ref_lib().ref_variant_to_string(i).decode() == n
    assert L.to_string(99) == "unknown"
    with pytest.raises(L.InvalidArgument, match="unknown loss variant: bogus"):
        L.loss_variant_from_string("bogus")
    if O.ref_available():
        with pytest.raises(ValueError, match="unknown loss variant: bogus"):
            O.ref_variant_from_string("bogus")


def test_config_defaults_match_reference():  # losses.hpp:28-38
    lib = _abi.load_library()
    c = _abi.rf_loss_config()
    lib.rf_loss_config_default(ctypes.byref(c))
    d = L.LossConfig()
    assert (c.variant, c.aggregation) == (0, 0)
    for f in ["clip_eps", "eps_low", "eps_high", "trunc_cap", "kl_weight", "w_plus", "w_minus",
              "engine_mismatch_cap"]:
        assert getattr(c, f) == getattr(d, f)


@pytest.mark.parametrize("field,val,code", [("clip_eps", 0.0, 1), ("clip_eps", 1.0, 1), ("eps_low", -0.1, 2),
                                            ("eps_high", -1.0, 2), ("trunc_cap", 0.0, 3), ("kl_weight", -0.5, 4),
                                            ("w_plus", -1.0, 5), ("w_minus", -1.0, 5),
                                            ("engine_mismatch_cap", -1.0, 6)])
def test_config_validation_mirrors_reference(field, val, code):  # losses.cpp:32-39
    cfg = L.LossConfig(**{field: val})
    lib = _abi.load_library()
    c = cfg.to_c()
    assert lib.rf_loss_config_validate(ctypes.byref(c)) == code
    with pytest.raises(L.InvalidArgument) as ei:
        cfg.validate()
    if O.ref_available():
        msg = O.ref_validate(cfg)
        assert msg is not None and msg == str(ei.value)


def _host_batch(T=4, N=2, V=16):
    b = _abi.rf_batch()
    b.num_tokens, b.num_seqs, b.vocab = T, N, V
    b.logits_dtype, b.logits_row_stride = _abi.RF_DTYPE_BF16, V
    fake = ctypes.c_void_p(0x1000)
    b.logits = b.token_ids = b.seq_of_token = b.seq_offsets = b.advantages = b.behavior_logp = fake
    b.logp_dtype, b.normalization = _abi.RF_DTYPE_F64, _abi.RF_NORM_SEQ_THEN_BATCH
    b.global_num_seqs, b.global_num_tokens, b.grad_sign = N, T, 1.0
    o = _abi.rf_outputs()
    o.scalars = o.device_status = fake
    return b, o


@pytest.mark.parametrize("mut,variant,code", [
    (lambda b, o: setattr(b, "num_tokens", 0), 0, _abi.RF_ERR_EMPTY_BATCH),
    (lambda b, o: setattr(b, "num_seqs", 0), 0, _abi.RF_ERR_EMPTY_BATCH),
    (lambda b, o: None, 1, _abi.RF_ERR_MISSING_PROX),
    (lambda b, o: setattr(b, "token_ids", None), 0, _abi.RF_ERR_INVALID_ARGUMENT),
    (lambda b, o: setattr(o, "scalars", None), 0, _abi.RF_ERR_INVALID_ARGUMENT),
    (lambda b, o: setattr(b, "logits_dtype", 7), 0, _abi.RF_ERR_INVALID_ARGUMENT),
    (lambda b, o: setattr(b, "global_num_seqs", 0), 0, _abi.RF_ERR_INVALID_ARGUMENT),
    (lambda b, o: None, 0, _abi.RF_ERR_WORKSPACE_TOO_SMALL),
])
def test_host_validation_without_gpu(mut, variant, code):
    lib = _abi.load_library()
    b, o = _host_batch()
    mut(b, o)
    c = L.LossConfig(variant=L.LossVariant(variant)).to_c()
    assert lib.rf_loss_and_grad(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), None) == code


def test_missing_ref_and_engine_codes():
    lib = _abi.load_library()
    b, o = _host_batch()
    c = L.LossConfig(variant=L.LossVariant.grpo, kl_weight=0.3).to_c()
    assert lib.rf_loss_and_grad(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), None) == _abi.RF_ERR_MISSING_REF
    c = L.LossConfig(variant=L.LossVariant.tis, engine_mismatch_cap=2.0).to_c()
    assert lib.rf_loss_and_grad(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), None) == \
        _abi.RF_ERR_MISSING_ENGINE_LOGP


def test_workspace_sizes():
    lib = _abi.load_library()
    b, _ = _host_batch(T=1000, N=10)
    c = L.LossConfig().to_c()
    tm = lib.rf_workspace_bytes(ctypes.byref(c), ctypes.byref(b))
    c2 = L.LossConfig(aggregation=L.RatioAggregation.sequence_product).to_c()
    sp = lib.rf_workspace_bytes(ctypes.byref(c2), ctypes.byref(b))
    assert tm >= 148 * 8 * 8 * 8 and sp >= tm + 5 * 1000 * 8


def test_status_strings_match_reference_messages():
    assert L.status_string(_abi.RF_ERR_CLIP_EPS) == "LossConfig: clip_eps must be in (0,1)"
    assert L.status_string(_abi.RF_ERR_EMPTY_BATCH) == "loss_and_grad: empty batch"
    assert L.status_string(_abi.RF_ERR_NONFINITE_RATIO) == "loss_and_grad: non-finite ratio"
    assert L.status_string(_abi.RF_ERR_GROUP_TOO_SMALL) == "grpo_advantages: group size must be >= 2"


def test_host_api_validation_without_gpu():
    """rf_loss_and_grad_host validates host arrays (empty trajectory, token range) before any CUDA call."""
    lib = _abi.load_library()
    T, N, V = 3, 2, 8
    logits = np.zeros((T, V), dtype=np.uint16)
    tok = np.array([1, 2, 9], dtype=np.int32)  # 9 >= V
    seq = np.array([0, 0, 1], dtype=np.int32)
    offs = np.array([0, 2, 3], dtype=np.int64)
    adv = np.zeros(N)
    beh = np.zeros(T)
    b = _abi.rf_batch()
    b.num_tokens, b.num_seqs, b.vocab = T, N, V
    b.logits_dtype, b.logits, b.logits_row_stride = _abi.RF_DTYPE_BF16, logits.ctypes.data, V
    b.token_ids, b.seq_of_token, b.seq_offsets = tok.ctypes.data, seq.ctypes.data, offs.ctypes.data
    b.advantages, b.behavior_logp = adv.ctypes.data, beh.ctypes.data
    b.logp_dtype, b.global_num_seqs, b.global_num_tokens, b.grad_sign = _abi.RF_DTYPE_F64, N, T, 1.0
    scal = np.zeros(8)
    o = _abi.rf_outputs()
    o.scalars = scal.ctypes.data
    c = L.LossConfig().to_c()
    assert lib.rf_loss_and_grad_host(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), 0, 0) == \
        _abi.RF_ERR_TOKEN_OUT_OF_RANGE
    offs2 = np.array([0, 3, 3], dtype=np.int64)  # empty second trajectory
    tok[2] = 1
    b.seq_offsets = offs2.ctypes.data
    assert lib.rf_loss_and_grad_host(ctypes.byref(c), ctypes.byref(b), ctypes.byref(o), 0, 0) == \
        _abi.RF_ERR_EMPTY_TRAJECTORY
