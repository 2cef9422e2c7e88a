"""CPU: synthetic-workload RNG (restated rlsim::RngStream) and the data-parallel
sharding logic, including a world_size-2 gloo run of the N>1 path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2510_11345_b200 import dist as D
from paper_2510_11345_b200 import synth as S
from tests.cases import config, make_case

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


def test_rngstream_matches_reference_golden():
    g = np.load(GOLDEN)
    s = S.RngStream(42, "lengths")
    assert np.array_equal(np.array([s.uniform01() for _ in range(64)]), g["rng/uniform"])
    s = S.RngStream(42, "lengths")
    assert np.array_equal(np.array([s.normal() for _ in range(64)]), g["rng/normal"])
    s = S.RngStream(42, "lengths")
    assert np.array_equal(np.array([s.next_u64() for _ in range(64)], dtype=np.uint64), g["rng/u64"])


def test_workload_shapes_long_tail():
    wl = S.WORKLOADS["c2"]
    L = S.sequence_lengths(42, wl.prompts * wl.group, wl.max_len)
    assert L.min() >= 1 and L.max() <= wl.max_len
    assert L.max() / np.median(L) > 20  # the paper's ">20x" long tail
    assert np.array_equal(L, S.sequence_lengths(42, wl.prompts * wl.group, wl.max_len))  # deterministic
    r = S.group_rewards(42, 16, 8)
    assert set(np.unique(r)) <= {0.0, 1.0}


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_lpt_shard_partitions_whole_groups(world):
    rng = np.random.default_rng(world)
    gt = rng.integers(1, 10000, 257)
    sh = D.lpt_shard(gt, world)
    allg = sorted(g for s in sh for g in s)
    assert allg == list(range(257))
    loads = [gt[s].sum() for s in sh]
    assert max(loads) - min(loads) <= gt.max()  # LPT bound


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = make_case(31, T_seqs=16, G=4, V=40, max_len=6, mapping="A", stale=0.2)
    lens = np.diff(case.seq_offsets)
    plan = D.ShardPlan.build(lens, case.group_offsets, rank, world)
    # this rank's shard of the packed batch (whole groups)
    idx = plan.seq_index
    toks = np.concatenate([np.arange(case.seq_offsets[i], case.seq_offsets[i + 1]) for i in idx])
    offs = np.zeros(len(idx) + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lens[idx])
    cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    o = O.oracle_loss_and_grad(cfg, case.logits[toks], case.token_ids[toks], offs, case.advantages[idx],
                               case.behavior_logp[toks], prox_logp=case.prox_logp[toks],
                               engine_logp=case.engine_logp[toks], normalization=1,
                               global_num_tokens=plan.global_tokens, global_num_seqs=plan.global_seqs)
    scal = torch.tensor([o["value"], float(len(toks))], dtype=torch.float64)
    D.allreduce_scalars(scal)
    q.put((rank, float(scal[0]), float(scal[1])))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_shard_allreduce_equals_single():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = make_case(31, T_seqs=16, G=4, V=40, max_len=6, mapping="A", stale=0.2)
    cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    one = O.oracle_loss_and_grad(cfg, case.logits, case.token_ids, case.seq_offsets, case.advantages,
                                 case.behavior_logp, prox_logp=case.prox_logp, engine_logp=case.engine_logp,
                                 normalization=1)
    for _, v, ntok in res:
        assert abs(v - one["value"]) <= 1e-12 * max(1.0, abs(one["value"]))
        assert int(ntok) == case.T
