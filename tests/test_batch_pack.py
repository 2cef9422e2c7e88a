"""Batch assembly (paper_2510_11345_b200.batch.pack_samples): a SampleBuffer::get_batch
result (sample_buffer.cpp:26-41) packed into the C ABI's CSR layout.  CPU: the layout,
grouping, sharding and staleness bookkeeping; GPU: the packed batch through K1 + K2
against the oracle."""
import numpy as np
import pytest
import torch

from paper_2510_11345_b200 import dist as D
from paper_2510_11345_b200.batch import Sample, pack_samples
from paper_2510_11345_b200.losses import InvalidArgument


def _samples(seed=0, prompts=7, group=4, V=50):
    rng = np.random.default_rng(seed)
    out, sid = [], 0
    order = [(p, r) for p in range(prompts) for r in range(group)]
    rng.shuffle(order)  # responses of a prompt arrive interleaved with other prompts (FIFO of completion)
    for p, r in order:
        L = int(rng.integers(1, 9))
        out.append(Sample(prompt=100 + p, tokens=rng.integers(0, V, L).tolist(), reward=float(rng.random() < 0.5),
                          behavior_logp=(-rng.random(L) * 5).tolist(), init_version=int(rng.integers(0, 3)),
                          id=sid, prox_logp=(-rng.random(L) * 5).tolist(), engine_logp=(-rng.random(L) * 5).tolist()))
        sid += 1
    return out


def test_pack_layout_groups_and_staleness():
    smp = _samples()
    pb, info = pack_samples(smp, torch.zeros(1, 50), consumer_version=3, device="cpu")
    # groups in FIFO order of their first response, responses in FIFO order inside a group
    first = []
    for s in smp:
        if s.prompt not in first:
            first.append(s.prompt)
    want = [s for p in first for s in smp if s.prompt == p]
    assert info.sample_ids == [s.id for s in want]
    offs = pb.seq_offsets.numpy()
    assert np.array_equal(np.diff(offs), [len(s.tokens) for s in want])
    assert pb.token_ids.tolist() == [t for s in want for t in s.tokens]
    assert np.allclose(pb.behavior_logp.numpy(), np.concatenate([s.behavior_logp for s in want]).astype(np.float32))
    assert np.allclose(pb.prox_logp.numpy(), np.concatenate([s.prox_logp for s in want]).astype(np.float32))
    assert pb.rewards.tolist() == [s.reward for s in want]
    assert np.array_equal(np.diff(pb.group_offsets.numpy()), [4] * 7)
    assert pb.seq_of_token.tolist() == [i for i, s in enumerate(want) for _ in s.tokens]
    assert info.staleness_histogram == dict(sorted(__import__("collections").Counter(3 - s.init_version
                                                                                        for s in smp).items()))
    assert pb.global_num_tokens == sum(len(s.tokens) for s in smp) and pb.global_num_seqs == len(smp)


@pytest.mark.parametrize("world", [2, 3])
def test_pack_shards_whole_groups_by_lpt(world):
    smp = _samples(1, prompts=9)
    parts = [pack_samples(smp, torch.zeros(1, 50), rank=r, world=world, device="cpu") for r in range(world)]
    ids = sorted(i for _, info in parts for i in info.sample_ids)
    assert ids == sorted(s.id for s in smp)  # a partition
    groups = {}
    for s in smp:
        groups.setdefault(s.prompt, []).append(s)
    gtok = [sum(len(s.tokens) for s in g) for g in groups.values()]
    plan = D.lpt_shard(gtok, world)
    for r, (pb, info) in enumerate(parts):
        assert pb.global_num_tokens == sum(gtok) and pb.global_num_seqs == len(smp)
        assert info.num_groups == len(plan[r])


def test_pack_rejects_reference_throw_sites():
    smp = _samples(2)
    with pytest.raises(InvalidArgument, match="empty batch"):
        pack_samples([], device="cpu", vocab=50)
    bad = list(smp)
    bad[0] = Sample(prompt=bad[0].prompt, tokens=[], reward=0.0, behavior_logp=[])
    with pytest.raises(InvalidArgument, match="empty trajectory"):
        pack_samples(bad, device="cpu", vocab=50)
    with pytest.raises(InvalidArgument, match="group size"):
        pack_samples(smp + [Sample(prompt=999, tokens=[1], reward=1.0, behavior_logp=[-1.0])], device="cpu",
                     vocab=50)


@pytest.mark.gpu
def test_packed_batch_through_the_loss_matches_oracle():
    import paper_2510_11345_b200 as rf
    from tests.cases import config
    from tests.parity import compare, run_oracle
    from tests.cases import Case

    V = 4096
    rng = np.random.default_rng(5)
    smp = _samples(3, prompts=6, group=4, V=V)
    first = []
    for s in smp:
        if s.prompt not in first:
            first.append(s.prompt)
    want = [s for p in first for s in smp if s.prompt == p]
    T = sum(len(s.tokens) for s in want)
    logits = torch.from_numpy(rng.normal(0, 2, (T, V))).to(torch.bfloat16).cuda()
    pb, info = pack_samples(smp, logits, consumer_version=2)
    adv, _ = rf.grpo_advantages(pb.rewards, pb.group_offsets)
    pb.advantages = adv
    cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    gpu = rf.loss_and_grad(cfg, pb)
    f64 = lambda t: t.double().cpu().numpy()  # noqa: E731
    case = Case(logits=f64(logits), token_ids=pb.token_ids.cpu().numpy(), seq_offsets=pb.seq_offsets.cpu().numpy(),
                advantages=f64(adv), behavior_logp=f64(pb.behavior_logp), prox_logp=f64(pb.prox_logp),
                engine_logp=f64(pb.engine_logp))
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)
