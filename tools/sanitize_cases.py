"""Small launches of every shipped kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Each case has several rows per CTA / cluster / CTA group so the
row-to-row protocols (TMEM parking, mbarrier phases, DSMEM and L2 exchange slots,
double-buffered stream slots) run more than once; results are checked against the
oracle so a sanitizer-perturbed schedule that computes garbage also fails.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402
from tests.cases import config, make_case, make_pool_case  # noqa: E402
from tests.parity import compare, run_oracle, to_device_batch  # noqa: E402


def lag_qwen3():  # K2 ring_lag_kernel, 2-CTA clusters (DSMEM exchange), ~4 rows per cluster
    case = make_pool_case(201, V=151936, R=32, T_min=300, G=4, max_len=16)
    cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    compare(case, cfg, rf.loss_and_grad(cfg, pb, kernel="ring"), run_oracle(case, cfg, normalization=1),
            check_dlogits=True)


def lag_v32k():  # K2 one CTA per row, ~4 rows per CTA
    case = make_pool_case(202, V=32000, R=64, T_min=600, G=4, max_len=16)
    cfg = config("tis", engine_mismatch_cap=2.0)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    compare(case, cfg, rf.loss_and_grad(cfg, pb, kernel="ring"), run_oracle(case, cfg, normalization=1))


def kl_groups():  # K2kl on cooperative CTA groups exchanging through L2
    case = make_pool_case(203, V=151936, R=16, T_min=160, G=4, max_len=16, kl=True)
    cfg = config("grpo", kl_weight=0.1)
    pb = to_device_batch(case, with_ref=True, normalization=L.Normalization.global_token)
    compare(case, cfg, rf.loss_and_grad(cfg, pb, kernel="ring"), run_oracle(case, cfg, normalization=1))


def streams():  # sequence_product: K2st -> K2s -> K2w, several rows per CTA
    case = make_pool_case(204, V=4099, R=64, T_min=3000, G=4, max_len=40, stale=0.02)
    cfg = config("tis", aggregation="sequence_product")
    pb = to_device_batch(case, normalization=L.Normalization.seq_then_batch)
    compare(case, cfg, rf.loss_and_grad(cfg, pb, kernel="ring"), run_oracle(case, cfg, normalization=0))


def generic():  # K2g (unaligned vocabulary) + K1 + K3
    case = make_case(205, T_seqs=12, G=4, V=1003, max_len=9, mapping="B")
    cfg = config("cispo")
    pb = to_device_batch(case)
    adv, _ = rf.grpo_advantages(pb.rewards, pb.group_offsets)
    compare(case, cfg, rf.loss_and_grad(cfg, pb), run_oracle(case, cfg, normalization=0))


def host_api():  # rf_loss_and_grad_host, 4 double-buffered chunks
    from tests.test_gpu_bench_regime import _host_call

    case = make_pool_case(206, V=32000, R=16, T_min=200, G=4, max_len=16)
    case.row_of_token = (np.arange(case.T) % 16).astype(np.int32)
    _host_call(case, config("ppo"), 64, L.Normalization.global_token)


CASES = {f.__name__: f for f in (lag_qwen3, lag_v32k, kl_groups, streams, generic, host_api)}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        print(f"{n} ok", flush=True)
