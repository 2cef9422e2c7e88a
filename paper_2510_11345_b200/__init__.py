"""B200-native off-policy policy-gradient loss + dlogits (ROLL Flash training hot path).

The compute path is ``librf_offpolicy.so`` (hand-written sm_100a CUDA behind
the C ABI of ``include/rf_offpolicy.h``); this package is the host-side mirror
of the reference's loss interface (rlsim::loss_and_grad and friends).
"""
from ._abi import load_library  # noqa: F401  (raises ImportError if the .so is missing)
from .losses import (  # noqa: F401
    InvalidArgument,
    LossConfig,
    LossResult,
    LossVariant,
    Normalization,
    OffPolicyLoss,
    PackedBatch,
    PolicyLossResult,
    RatioAggregation,
    Trajectory,
    grpo_advantages,
    loss_and_grad,
    loss_and_grad_policy,
    loss_variant_from_string,
    seq_of_token_from_offsets,
    status_string,
    to_string,
)

load_library()
