"""GPU: the reference's remaining throw sites on the device API, the reference-layout
gradient reduction, and stream-capture safety.

* empty trajectory (losses.cpp:157) and a GRPO group of < 2 (losses.cpp:42) are
  device-detected on the stream-ordered API (RF_DEVSTAT_* bits, no host sync);
* rf_rows_segment_sum (LossResult.grad = per-context sums of dlogits rows,
  LogProbGrad add/flush, losses.cpp:87-115) is the exact in-order fp64 sum;
* the exact-KL CTA-group kernel exchanges partials through L2 sequence words:
  a captured CUDA graph replayed on new data must equal an eager call bit for bit;
* the host-buffer API uses a private memory pool (the default pool's release
  threshold is left alone).
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from tests.cases import config, make_case, make_pool_case
from tests.parity import compare, run_oracle, to_device_batch

pytestmark = pytest.mark.gpu

import paper_2510_11345_b200 as rf  # noqa: E402
from paper_2510_11345_b200 import _abi  # noqa: E402
from paper_2510_11345_b200 import losses as L  # noqa: E402


def _with_empty_sequences(case, where):
    """Insert empty sequences (zero-length CSR segments) before the given sequence indices."""
    offs = list(case.seq_offsets)
    adv = list(case.advantages)
    for i in sorted(where, reverse=True):
        offs.insert(i, offs[i])
        adv.insert(i, 0.0)
    case.seq_offsets = np.array(offs, dtype=np.int64)
    case.advantages = np.array(adv)
    return case


@pytest.mark.parametrize("where", [[3], [0], ["end"], [2, 2, 5]])
def test_empty_trajectory_flagged_on_device(where):
    case = make_case(41, T_seqs=8, G=4, V=4096, max_len=6, mapping="A")
    n = case.N
    case = _with_empty_sequences(case, [n if w == "end" else w for w in where])
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    with pytest.raises(rf.InvalidArgument, match="empty trajectory"):
        rf.loss_and_grad(config("tis"), pb)
    # chunked, stream-ordered: the bit is set by the call whose span contains the empty sequence
    op = rf.OffPolicyLoss(config("tis"), pb, chunk_tokens=5)
    op.zero()
    for t0 in range(0, pb.num_tokens, 5):
        op.run(pb, t0, min(pb.num_tokens, t0 + 5))
    torch.cuda.synchronize()
    assert int(op.status.item()) & _abi.RF_DEVSTAT_EMPTY_TRAJECTORY


def test_no_false_empty_trajectory_flag_when_chunked():
    case = make_case(42, T_seqs=16, G=4, V=4096, max_len=9, mapping="A")
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    for chunk in (1, 3, 7, 64):
        op = rf.OffPolicyLoss(config("ppo"), pb, chunk_tokens=chunk)
        op.zero()
        for t0 in range(0, pb.num_tokens, chunk):
            op.run(pb, t0, min(pb.num_tokens, t0 + chunk))
        torch.cuda.synchronize()
        assert int(op.status.item()) == 0, chunk


def test_grpo_group_too_small_flagged_on_device():
    rng = np.random.default_rng(5)
    sizes = np.array([4, 1, 3, 2, 1, 5])
    go = np.zeros(len(sizes) + 1, dtype=np.int64)
    go[1:] = np.cumsum(sizes)
    rewards = rng.uniform(-1, 1, go[-1])
    dev = "cuda"
    out = (torch.full((go[-1],), 7.0, dtype=torch.float64, device=dev),
           torch.full((len(sizes),), 9, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int32, device=dev))
    rf.grpo_advantages(torch.from_numpy(rewards).to(dev), torch.from_numpy(go).to(dev), out=out, validate=False)
    adv, deg, status = (t.cpu().numpy() for t in out)
    assert status[0] & _abi.RF_DEVSTAT_GROUP_TOO_SMALL
    for g, n in enumerate(sizes):
        seg = slice(go[g], go[g + 1])
        if n < 2:  # zeroed, not left uninitialised
            assert (adv[seg] == 0).all() and deg[g] == 0
        else:
            a, d = O.ref_grpo_advantages(rewards[seg]) if O.ref_available() else (None, None)
            if a is not None:
                assert np.array_equal(adv[seg], a) and deg[g] == int(d)
    with pytest.raises(rf.InvalidArgument, match="group size"):
        rf.grpo_advantages(torch.from_numpy(rewards).to(dev), torch.from_numpy(go).to(dev))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rows_segment_sum_is_the_in_order_fp64_sum(dtype):
    rng = np.random.default_rng(8)
    R, W, stride = 300, 1003, 1008
    rows = torch.from_numpy(rng.normal(0, 1, (R, stride))).to(dtype).cuda()
    segs = [rng.integers(0, R, rng.integers(0, 40)) for _ in range(37)]
    offs = np.zeros(len(segs) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(s) for s in segs])
    idx = np.concatenate(segs).astype(np.int32)
    out = torch.full((len(segs), 1024), 3.0, dtype=torch.float64, device="cuda")
    d_offs, d_idx = torch.from_numpy(offs).cuda(), torch.from_numpy(idx).cuda()  # alive across the launch
    st = _abi.load_library().rf_rows_segment_sum(
        rows.data_ptr(), _abi.RF_DTYPE_BF16 if dtype == torch.bfloat16 else _abi.RF_DTYPE_F32, stride,
        d_offs.data_ptr(), d_idx.data_ptr(), len(segs), W, out.data_ptr(), 1024, torch.cuda.current_stream().cuda_stream)
    assert st == 0
    host = rows.float().double().cpu().numpy()
    got = out.cpu().numpy()
    for s, seg in enumerate(segs):
        want = np.cumsum(host[seg, :W], axis=0)[-1] if len(seg) else np.zeros(W)
        assert np.array_equal(got[s, :W], want), s
    assert (got[:, W:] == 3.0).all()  # nothing written past the width


@pytest.mark.parametrize("path", ["exact_kl", "lag", "seqprod"])
def test_graph_replay_equals_eager(path):
    """the CTA-group exchange slots are guarded by sequence words, and every
    persistent kernel claims its rows from a per-launch counter; captured into a CUDA
    graph and replayed on new logits, every replay must see fresh slots and counters."""
    norm = L.Normalization.global_token
    if path == "exact_kl":
        case = make_pool_case(43, V=151936, R=48, T_min=700, G=4, max_len=48, stale=0.2, kl=True)
        cfg = config("grpo", kl_weight=0.1, engine_mismatch_cap=2.0)
    elif path == "lag":
        case = make_pool_case(44, V=151936, R=48, T_min=700, G=4, max_len=48, stale=0.2)
        cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    else:
        case = make_pool_case(45, V=32000, R=64, T_min=2600, G=4, max_len=96, stale=0.2)
        cfg = config("tis", aggregation="sequence_product")
        norm = L.Normalization.seq_then_batch
    pb = to_device_batch(case, with_ref=(path == "exact_kl"), normalization=norm)
    T = pb.num_tokens
    op = rf.OffPolicyLoss(cfg, pb, kernel="ring")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        op.zero()
        op.run(pb, 0, T)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op.zero()
        op.run(pb, 0, T)
    torch.cuda.synchronize()
    gen = torch.Generator(device="cuda")
    for rep in range(3):
        gen.manual_seed(100 + rep)
        pb.logits.copy_(torch.randn(pb.logits.shape, generator=gen, device="cuda") * 2.0)
        g.replay()
        torch.cuda.synchronize()
        eager = rf.loss_and_grad(cfg, pb, kernel="ring", check=False)
        torch.cuda.synchronize()
        assert torch.equal(op.dlogits, eager.dlogits), rep
        assert torch.equal(op.token_logp, eager.token_logp), rep
        assert torch.equal(op.scalars, eager.scalars), rep
    # and the last replay against the oracle on the replayed logits
    case.logits = pb.logits.double().cpu().numpy()
    compare(case, cfg, op, run_oracle(case, cfg, normalization=int(norm), want_dlogits=False), check_dlogits=False)


def test_host_api_leaves_default_mempool_alone():
    import glob

    libs = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob("/usr/local/cuda/targets/*/lib/libcudart.so*")
    cudart = ctypes.CDLL(sorted(libs)[0])
    pool = ctypes.c_void_p()
    assert cudart.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), 0) == 0
    thr = ctypes.c_uint64(0)
    ATTR_RELEASE_THRESHOLD = 4  # cudaMemPoolAttrReleaseThreshold
    assert cudart.cudaMemPoolGetAttribute(pool, ATTR_RELEASE_THRESHOLD, ctypes.byref(thr)) == 0
    before = thr.value
    case = make_case(44, T_seqs=4, G=2, V=4096, max_len=5, mapping="A")
    from tests.test_gpu_bench_regime import _host_call  # pinned host buffers through rf_loss_and_grad_host

    case.row_of_token = np.arange(case.T, dtype=np.int32)
    _host_call(case, config("tis"), 4, L.Normalization.global_token)
    assert cudart.cudaMemPoolGetAttribute(pool, ATTR_RELEASE_THRESHOLD, ctypes.byref(thr)) == 0
    assert thr.value == before


@pytest.mark.parametrize("V,kernel", [(32000, "ring"), (151936, "ring"), (4099, "generic")])
def test_masked_vocabulary_minus_inf_logits(V, kernel):
    """LLM vocabularies are padded and masked with -inf logits: those entries get p = 0 and a
    zero dlogit, every other output matches the oracle (whose log-softmax handles -inf the
    same way, policy.cpp:21-30)."""
    case = make_case(45, T_seqs=8, G=4, V=V, max_len=6, mapping="A", stale=0.2)
    rng = np.random.default_rng(45)
    masked = rng.random(case.logits.shape) < 0.05
    masked[np.arange(case.T), case.token_ids] = False  # sampled tokens are never masked
    case.logits = np.where(masked, -np.inf, case.logits)
    lsm = case.logits - case.logits.max(1, keepdims=True)
    lp = (lsm - np.log(np.exp(lsm).sum(1, keepdims=True)))[np.arange(case.T), case.token_ids]
    case.behavior_logp = lp - 0.05
    case.prox_logp, case.engine_logp = lp - 0.02, lp - 0.06
    cfg = config("decoupled_ppo", engine_mismatch_cap=2.0)
    pb = to_device_batch(case, normalization=L.Normalization.global_token)
    gpu = rf.loss_and_grad(cfg, pb, kernel=kernel)
    ref = run_oracle(case, cfg, normalization=1)
    compare(case, cfg, gpu, ref)
    d = gpu.dlogits.float().cpu().numpy()
    assert (d[masked] == 0).all() and np.isfinite(d).all()
