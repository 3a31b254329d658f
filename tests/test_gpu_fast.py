"""GPU parity of the FAST (tcgen05) path: draft ids / FR remaps / argmax bit-exact vs the
oracle; probabilities within a stated tolerance (PROB_RTOL) because the softmax denominator
is accumulated from the tensor-core logits; rows that fall back to the exact kernel
(FLAG_RECOMPUTED) must be bit-exact."""
import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api
from paper_2502_14856_b200._lib import FLAG_NONFINITE, FLAG_RECOMPUTED, FLAG_UNCERTIFIED, InvalidArgument

pytestmark = pytest.mark.gpu
PROB_RTOL = 1e-4  # relative tolerance on FAST probabilities (approximate Σexp denominator)


def rmsnorm(x):
    x = x.astype(np.float32)
    ms = (x.astype(np.float64) ** 2).mean(axis=1, keepdims=True)
    return (x * (1.0 / np.sqrt(ms + 1e-5)).astype(np.float32)).astype(np.float32)


def case(seed, n, d, v_sub, V=None):
    rng = np.random.default_rng(seed)
    V = V or v_sub + 1000
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16).float().numpy()
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    h = rmsnorm(rng.standard_normal((n, d)))
    return W, ids, h


def check_fast(ctx, restatement, W, ids, h, k, temperature=1.0):
    head = api.restrict_lm_head(ctx, torch.from_numpy(W).cuda(), api.RankedSubset(W.shape[0], ids), dtype="bf16")
    out = api.draft_head_topk(ctx, torch.from_numpy(h).cuda(), head, k, temperature, mode="fast")
    torch.cuda.synchronize()
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, k, temperature)
    kk = min(k, ids.size)
    flags = out.flags.cpu().numpy()
    assert (flags & FLAG_UNCERTIFIED).sum() == 0
    assert np.array_equal(out.ridx.cpu().numpy()[:, :kk], ref["ridx"][:, :kk])
    assert np.array_equal(out.full.cpu().numpy()[:, :kk], ref["full"][:, :kk])
    assert np.array_equal(out.rowmax.cpu().numpy(), ref["mx"])
    prob = out.prob.cpu().numpy()[:, :kk]
    np.testing.assert_allclose(prob, ref["prob"][:, :kk], rtol=PROB_RTOL, atol=0)
    rec = (flags & FLAG_RECOMPUTED) != 0
    if rec.any():  # fallback rows are the exact path: bit-identical
        assert np.array_equal(prob[rec], ref["prob"][rec, :kk])
    return flags


@pytest.mark.parametrize("n,d,v_sub,k", [
    (4, 512, 8192, 4),        # C1 shape
    (10, 4096, 32768, 10),    # C2 shape
    (1, 4096, 32768, 10),     # level-0 root row
    (16, 256, 3000, 16),
    (7, 1024, 300, 10),       # V_sub smaller than one CTA wave
    (10, 2048, 20000, 32),    # k > 16: 64 recomputed candidates
    (20, 512, 8192, 10),      # 17..32 rows: batched path (NP=32)
    (3, 3584, 32768, 10),     # Qwen-2.5-7B hidden size
    (64, 4096, 32768, 10),    # batched path, one full 64-row pass at the Llama shape
    (100, 1024, 12000, 10),   # batched path, two passes (64 + 36)
    (40, 2048, 5000, 40),     # batched path, k > 32
])
def test_fast_draft_ids_exact(cuda_ctx, restatement, n, d, v_sub, k):
    W, ids, h = case(n * 7 + d + v_sub, n, d, v_sub)
    check_fast(cuda_ctx, restatement, W, ids, h, k)


@pytest.mark.parametrize("temperature", [0.6, 1.8])
def test_fast_temperature(cuda_ctx, restatement, temperature):
    W, ids, h = case(21, 5, 1024, 5000)
    check_fast(cuda_ctx, restatement, W, ids, h, 10, temperature)


def test_fast_exact_ties_and_forced_fallback(cuda_ctx, restatement):
    """Identical slab rows give exactly equal logits (ties by restricted index); a fully flat
    row cannot be certified and must fall back to the exact full-row path."""
    W, ids, h = case(22, 3, 512, 4000)
    W[ids[5]] = W[ids[3000]]           # exact duplicates at both ends of the ranking
    W[ids[7]] = W[ids[2999]]
    h[2] = 0.0                          # all logits 0: every prob ties -> flat row
    flags = check_fast(cuda_ctx, restatement, W, ids, h, 10)
    assert flags[2] & FLAG_RECOMPUTED


def test_fast_nonfinite_flag(cuda_ctx):
    W, ids, h = case(23, 2, 256, 1000)
    h[0, 1] = np.nan
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(W.shape[0], ids), dtype="bf16")
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 4, mode="fast")
    flags = out.flags.cpu().numpy()
    assert flags[0] & FLAG_NONFINITE and not flags[1] & FLAG_NONFINITE


@pytest.mark.parametrize("m,d,V", [(61, 4096, 32000), (8, 4096, 128256), (33, 512, 7000), (5, 3584, 20000)])
def test_fast_verify_argmax_exact(cuda_ctx, restatement, m, d, V):
    rng = np.random.default_rng(m + d)
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16)
    Wn = W.float().numpy()
    h = rmsnorm(rng.standard_normal((m, d)))
    ids, vals, flags = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), W.cuda(), mode="fast")
    rid, rval = restatement.verify_argmax(h, Wn)
    assert np.array_equal(ids.cpu().numpy(), rid)
    assert np.array_equal(vals.cpu().numpy(), rval)


def test_fast_verify_ties_lowest_id(cuda_ctx, restatement):
    rng = np.random.default_rng(31)
    V, d = 5000, 256
    Wf = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
    h = rmsnorm(rng.standard_normal((4, d)))
    best = restatement.verify_argmax(h, torch.from_numpy(Wf).to(torch.bfloat16).float().numpy())[0]
    Wf[4999] = Wf[best[0]]  # duplicate the winner of row 0 at a higher id
    Wf[0] = Wf[best[1]]     # and the winner of row 1 at a lower id
    W = torch.from_numpy(Wf).to(torch.bfloat16)
    ids, _, _ = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), W.cuda(), id_offset=100, mode="fast")
    rid, _ = restatement.verify_argmax(h, W.float().numpy())
    assert np.array_equal(ids.cpu().numpy(), rid + 100)


def test_fast_repeated_calls_stable(cuda_ctx, restatement):
    """Monotonic per-row counters and reused workspaces: many back-to-back calls agree."""
    W, ids, h = case(41, 10, 1024, 8192)
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(W.shape[0], ids), dtype="bf16")
    hd = torch.from_numpy(h).cuda()
    first = api.draft_head_topk(cuda_ctx, hd, head, 10, mode="fast")
    f0 = first.full.clone()
    for _ in range(50):
        o = api.draft_head_topk(cuda_ctx, hd, head, 10, mode="fast", out=first)
    torch.cuda.synchronize()
    assert torch.equal(o.full, f0)


def test_fast_fallback_several_rows_one_call(cuda_ctx, restatement):
    """Two uncertifiable (flat) rows in one call go through the grid-wide exact fallback
    together; the certified rows of the same call are untouched."""
    W, ids, h = case(24, 6, 1024, 9000)
    h[1] = 0.0
    h[4] = 0.0
    flags = check_fast(cuda_ctx, restatement, W, ids, h, 10)
    assert flags[1] & FLAG_RECOMPUTED and flags[4] & FLAG_RECOMPUTED
    assert not flags[0] & FLAG_RECOMPUTED


def test_fast_verify_fallback_flat_rows(cuda_ctx, restatement):
    """A zero hidden row makes every logit 0: argmax must be the lowest id (kernels.cpp:117-121),
    reached through the exact fallback; the queue is empty again afterwards."""
    rng = np.random.default_rng(77)
    V, d = 20000, 512
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16)
    h = rmsnorm(rng.standard_normal((5, d)))
    h[2] = 0.0
    for _ in range(2):
        ids, vals, flags = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), W.cuda(), id_offset=7,
                                                  mode="fast")
        rid, rval = restatement.verify_argmax(h, W.float().numpy())
        assert np.array_equal(ids.cpu().numpy(), rid + 7)
        assert np.array_equal(vals.cpu().numpy(), rval)
        f = flags.cpu().numpy()
        assert f[2] & FLAG_RECOMPUTED and not f[0] & FLAG_RECOMPUTED


def test_fast_certification_rate_c2(cuda_ctx, restatement):
    """At the Llama-3-8B shape almost every row is certified without the fallback; every row,
    certified or not, matches the oracle. Fallback reasons are reported, not hidden."""
    W, ids, _ = case(1234, 1, 4096, 32768, V=40000)
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(W.shape[0], ids), dtype="bf16")
    slab = restatement.restrict(W, ids)
    rng = np.random.default_rng(5)
    total, rec, reasons = 0, 0, {}
    for it in range(8):
        h = rmsnorm(rng.standard_normal((10, 4096)))
        out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 10, mode="fast")
        ref = restatement.draft_level(h, slab, ids, 10)
        assert np.array_equal(out.full.cpu().numpy(), ref["full"])
        f = out.flags.cpu().numpy()
        total += f.size
        rec += int(((f & FLAG_RECOMPUTED) != 0).sum())
        for bit in (0x10, 0x20, 0x40):
            reasons[bit] = reasons.get(bit, 0) + int(((f & bit) != 0).sum())
    print(f"certification: {total - rec}/{total} rows certified; fallback reasons {reasons}")
    assert rec <= max(2, total // 20)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_vocab_parallel_emulated(cuda_ctx, restatement, G):
    """emulate the G-GPU vocab-parallel verify on one GPU — each contiguous
    shard through K3 with its id offset, the pairs stacked as an all-gather would, K5 merges —
    bit-exact with the full-vocabulary argmax, including a tie straddling a shard boundary."""
    rng = np.random.default_rng(40 + G)
    V, d, m = 9001, 512, 13
    Wf = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
    h = rmsnorm(rng.standard_normal((m, d)))
    best = restatement.verify_argmax(h, torch.from_numpy(Wf).to(torch.bfloat16).float().numpy())[0]
    s_last, _ = api.vocab_shard(V, G, G - 1)
    Wf[s_last + 5] = Wf[best[0]]  # the same max in the last shard: the lower id must win
    W = torch.from_numpy(Wf).to(torch.bfloat16).cuda()
    hd = torch.from_numpy(h).cuda()
    vals, ids = [], []
    for r in range(G):
        st, cnt = api.vocab_shard(V, G, r)
        i_, v_, _ = api.verify_head_argmax(cuda_ctx, hd, W[st:st + cnt].contiguous(), id_offset=st, mode="fast")
        vals.append(v_)
        ids.append(i_)
    mv, mi = api.argmax_merge(cuda_ctx, torch.stack(vals), torch.stack(ids))
    rid, rval = restatement.verify_argmax(h, W.float().cpu().numpy())
    assert np.array_equal(mi.cpu().numpy(), rid)
    assert np.array_equal(mv.cpu().numpy(), rval)


def test_vocab_parallel_nccl_world1(cuda_ctx, restatement):
    """The C-ABI vocab-parallel verify (frs_verify_head_argmax_vp: K3 + ncclAllGather + K5) on a
    1-rank NCCL communicator made by the library (the unique id broadcast over a gloo group)."""
    import socket
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comm = api.NcclComm(cuda_ctx)
        rng = np.random.default_rng(3)
        V, d, m = 5000, 256, 7
        W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16)
        h = rmsnorm(rng.standard_normal((m, d)))
        rid, rval = restatement.verify_argmax(h, W.float().numpy())
        for mode in ("fast", "exact"):
            ids, vals, _ = api.verify_head_argmax_vocab_parallel(cuda_ctx, torch.from_numpy(h).cuda(), W.cuda(), V, comm,
                                                                 mode=mode)
            assert np.array_equal(ids.cpu().numpy(), rid), mode
            assert np.array_equal(vals.cpu().numpy(), rval), mode
        with pytest.raises(InvalidArgument):
            api.verify_head_argmax_vocab_parallel(cuda_ctx, torch.from_numpy(h).cuda(), W[:10].cuda(), V, comm)
        comm.close()
    finally:
        dist.destroy_process_group()


def test_fast_verify_many_rows_batched(cuda_ctx, restatement):
    """More than 64 verify rows (batched streams) go through the approximate-logits path."""
    rng = np.random.default_rng(91)
    V, d, m = 6000, 512, 150
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16)
    h = rmsnorm(rng.standard_normal((m, d)))
    h[7] = 0.0  # flat row: lowest id through the exact fallback
    ids, vals, flags = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), W.cuda(), id_offset=11, mode="fast")
    rid, rval = restatement.verify_argmax(h, W.float().numpy())
    assert np.array_equal(ids.cpu().numpy(), rid + 11)
    assert np.array_equal(vals.cpu().numpy(), rval)


@pytest.mark.parametrize("n,pinned", [(10, True), (16, True), (1, True), (10, False), (20, True)])
def test_fast_draft_host_buffers(cuda_ctx, restatement, n, pinned):
    """frs_head_draft_host in FAST mode: pinned rows (n <= 16) are read by k_hsplit over the bus
    and the ids / probabilities land in pinned staging with no copy operations; pageable rows
    and n > 16 take the H2D / D2H path. Same outputs as the device-buffer call and the oracle."""
    W, ids, h = case(31, n, 1024, 8192)
    dh = api.DeviceHead(cuda_ctx, W, api.RankedSubset(W.shape[0], ids), dtype="bf16")
    if pinned:
        t = torch.empty((n, W.shape[1]), dtype=torch.float32, pin_memory=True)
        t.copy_(torch.from_numpy(h))
        h_host = t.numpy()
    else:
        h_host = h.copy()
    for _ in range(2):  # repeated calls reuse the staging buffers
        ridx, full, prob = dh.draft_host(h_host, 10, mode="fast")
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(W.shape[0], ids), dtype="bf16")
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 10, mode="fast")
    assert np.array_equal(ridx, out.ridx.cpu().numpy()) and np.array_equal(full, out.full.cpu().numpy())
    assert np.array_equal(prob, out.prob.cpu().numpy())
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, 10)
    assert np.array_equal(ridx, ref["ridx"]) and np.array_equal(full, ref["full"])
    np.testing.assert_allclose(prob, ref["prob"], rtol=PROB_RTOL, atol=0)


def tiled_image_np(slab_bits: np.ndarray) -> np.ndarray:
    """numpy restatement of frs_slab_tile: blocks [K block][32-row chunk] of 4 KB, each the
    SWIZZLE_128B image (16-byte group q of row r at r * 128 + (q ^ (r & 7)) * 16), zero fill."""
    v, d = slab_bits.shape
    nch, kbs = -(-v // 32), -(-d // 64)
    pad = np.zeros((nch * 32, kbs * 64), np.uint16)
    pad[:v, :d] = slab_bits
    out = np.zeros((kbs, nch, 32, 8, 8), np.uint16)  # [kb][c][r][position][8 elements]
    for q in range(8):
        for r in range(32):
            out[:, :, r, q ^ (r & 7), :] = pad.reshape(nch, 32, kbs, 8, 8)[:, r, :, q, :].transpose(1, 0, 2)
    return out.reshape(-1).view(np.uint8)


@pytest.mark.parametrize("v,d", [(100, 200), (4096, 512), (33, 64)])
def test_slab_tile_image(cuda_ctx, v, d):
    """frs_slab_tile == its numpy restatement (ragged rows and K blocks zero-filled)."""
    rng = np.random.default_rng(v + d)
    W = torch.from_numpy((rng.standard_normal((v, d)) * 0.02).astype(np.float32)).cuda()
    head = api.restrict_lm_head(cuda_ctx, W, api.RankedSubset(v, np.arange(v, dtype=np.int32)), dtype="bf16")
    torch.cuda.synchronize()
    bits = head.slab.view(torch.int16).cpu().numpy().view(np.uint16)
    assert head.tiled is not None and head.tiled.numel() == (-(-v // 32)) * (-(-d // 64)) * 4096
    assert np.array_equal(head.tiled.cpu().numpy(), tiled_image_np(bits))


@pytest.mark.parametrize("n,d,v_sub", [(10, 512, 5000 - 17), (7, 200, 3001), (16, 4096, 32768)])
def test_fast_tiled_equals_row_major(cuda_ctx, restatement, n, d, v_sub):
    """FAST over the tiled image (1-D bulk stage loads) == FAST over the row-major slab (2-D
    tensor loads) == the oracle: a ragged slab height (short last tiles), a hidden size that is
    not a multiple of the 64-column K block (zero-filled image columns), the Llama-3-8B shape."""
    W, ids, h = case(31, n, d, v_sub)
    Wd = torch.from_numpy(W).cuda()
    sub = api.RankedSubset(W.shape[0], ids)
    a = api.restrict_lm_head(cuda_ctx, Wd, sub, dtype="bf16")
    b = api.restrict_lm_head(cuda_ctx, Wd, sub, dtype="bf16", tile=False)
    assert a.tiled is not None and b.tiled is None
    hd = torch.from_numpy(h).cuda()
    oa = api.draft_head_topk(cuda_ctx, hd, a, 10, mode="fast")
    ob = api.draft_head_topk(cuda_ctx, hd, b, 10, mode="fast")
    assert not (oa.flags.cpu().numpy() & FLAG_UNCERTIFIED).any()
    torch.cuda.synchronize()
    assert torch.equal(oa.full, ob.full) and torch.equal(oa.ridx, ob.ridx) and torch.equal(oa.rowmax, ob.rowmax)
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, 10)
    assert np.array_equal(oa.full.cpu().numpy(), ref["full"])


@pytest.mark.parametrize("m", [7, 61, 130])
def test_fast_verify_tiled_equals_row_major(cuda_ctx, restatement, m):
    """frs_verify_head_argmax_tiled (the shard's tiled image) == the 2-D tensor path == the
    oracle's argmax, for list-path (<= 64 rows) and batched (> 64 rows) calls, with an id offset."""
    rng = np.random.default_rng(m)
    V, d = 9000 + 13, 256
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16)
    h = rmsnorm(rng.standard_normal((m, d)))
    Wd, hd = W.cuda(), torch.from_numpy(h).cuda()
    Wt = api.tile_image(cuda_ctx, Wd)
    a, va, _ = api.verify_head_argmax(cuda_ctx, hd, Wd, id_offset=50, mode="fast", W_tiled=Wt)
    b, vb, _ = api.verify_head_argmax(cuda_ctx, hd, Wd, id_offset=50, mode="fast")
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(va, vb)
    rid, _ = restatement.verify_argmax(h, W.float().numpy())
    assert np.array_equal(a.cpu().numpy(), rid + 50)
