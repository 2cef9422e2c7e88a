"""B200-native off-policy policy-gradient loss + dlogits (ROLL Flash training hot path).

The compute path is ``librf_offpolicy.so`` (hand-written sm_100a CUDA behind
the C ABI of ``include/rf_offpolicy.h``); this package is the host-side mirror
of the reference's loss interface (rlsim::loss_and_grad and friends).

Importing the package checks that the library was built (ImportError
otherwise: there is no CPU fallback) but maps it only on the first call, so a
process that imports only the workload synthesis (``synth``) — e.g. the
reference arm of bench.py — never loads the product library.
"""
from ._abi import require_library
from .batch import PackInfo, Sample, pack_samples  # noqa: F401
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

require_library()
