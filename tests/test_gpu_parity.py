"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical inputs.

EXACT mode bar (BASELINE.json north_star): logits, probabilities, rowmax, Σ, top-k ids and
FR id remaps bit-identical to the reference arithmetic; argmax / accepted sequences exact.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api
from paper_2502_14856_b200._lib import FLAG_NONFINITE, InvalidArgument

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rmsnorm(x):
    """model.cpp:29-40 semantics (gain 1, eps 1e-5) — only shapes the synthetic inputs."""
    x = x.astype(np.float32)
    ms = (x.astype(np.float64) ** 2).mean(axis=1, keepdims=True)
    return (x * (1.0 / np.sqrt(ms + 1e-5)).astype(np.float32)).astype(np.float32)


def make_case(seed, n, d, v_sub, V=None, bf16=False, permuted=True):
    rng = np.random.default_rng(seed)
    V = V or v_sub * 2
    W = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
    if bf16:  # bf16-representable weights: the oracle sees the exact widened values
        W = torch.from_numpy(W).to(torch.bfloat16).to(torch.float32).numpy()
    ids = (rng.permutation(V)[:v_sub] if permuted else np.arange(v_sub)).astype(np.int32)
    h = rmsnorm(rng.standard_normal((n, d)))
    return W, ids, h


def run_draft(ctx, W, ids, h, k, dtype, temperature=1.0, want_logits=True):
    Wd = torch.from_numpy(W).cuda()
    head = api.restrict_lm_head(ctx, Wd, api.RankedSubset(W.shape[0], ids), dtype=dtype)
    out = api.draft_head_topk(ctx, torch.from_numpy(h).cuda(), head, k, temperature, mode="exact",
                              want_logits=want_logits)
    torch.cuda.synchronize()
    return head, out


def assert_level_equal(out, ref, k_eff):
    assert np.array_equal(out.logits.cpu().numpy(), ref["logits"])
    assert np.array_equal(out.ridx.cpu().numpy()[:, :k_eff], ref["ridx"][:, :k_eff])
    assert np.array_equal(out.full.cpu().numpy()[:, :k_eff], ref["full"][:, :k_eff])
    assert np.array_equal(out.prob.cpu().numpy()[:, :k_eff], ref["prob"][:, :k_eff])
    assert np.array_equal(out.rowmax.cpu().numpy(), ref["mx"])
    assert np.array_equal(out.total.cpu().numpy(), ref["total"])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_slab_build_bitwise(cuda_ctx, restatement, dtype):
    W, ids, _ = make_case(1, 1, 96, 700, V=1000, bf16=(dtype == "bf16"))
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(1000, ids), dtype=dtype)
    got = head.slab.float().cpu().numpy()
    assert np.array_equal(got, restatement.restrict(W, ids))
    bad = ids.copy()
    bad[5] = 1000
    with pytest.raises(InvalidArgument):
        api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(1001, bad), dtype=dtype)


@pytest.mark.parametrize("n,d,v_sub,k,dtype", [
    (4, 512, 8192, 4, "f32"),      # C1 shape
    (4, 512, 8192, 4, "bf16"),
    (1, 512, 8192, 10, "f32"),
    (7, 100, 3000, 10, "f32"),     # d % 8 != 0 exercises the scalar tail
    (3, 13, 500, 5, "bf16"),
    (12, 256, 2048, 16, "f32"),
    (17, 128, 1024, 8, "f32"),     # > 12 rows: multi-pass
    (2, 64, 5, 8, "f32"),          # k > V_sub -> min(width, V_sub)
])
def test_draft_head_exact_bitwise(cuda_ctx, restatement, n, d, v_sub, k, dtype):
    W, ids, h = make_case(n * 1000 + d, n, d, v_sub, bf16=(dtype == "bf16"))
    _, out = run_draft(cuda_ctx, W, ids, h, k, dtype)
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, k, want_logits=True)
    assert_level_equal(out, ref, min(k, v_sub))
    assert (out.flags.cpu().numpy() & FLAG_NONFINITE).sum() == 0


@pytest.mark.parametrize("temperature", [0.5, 1.7])
def test_draft_head_exact_temperature(cuda_ctx, restatement, temperature):
    W, ids, h = make_case(11, 3, 256, 4096)
    _, out = run_draft(cuda_ctx, W, ids, h, 10, "f32", temperature)
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, 10, temperature, want_logits=True)
    assert_level_equal(out, ref, 10)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_draft_head_exact_llama_shape(cuda_ctx, restatement, dtype):
    """C2: d=4096, V=128256, V_sub=32768, n=10 beam rows, k=10 — bit-exact."""
    W, ids, h = make_case(2024, 10, 4096, 32768, V=128256, bf16=(dtype == "bf16"))
    _, out = run_draft(cuda_ctx, W, ids, h, 10, dtype)
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, 10, want_logits=True)
    assert_level_equal(out, ref, 10)


def test_draft_head_ties_by_restricted_index(cuda_ctx, restatement):
    """Duplicate slab rows give equal probabilities; ties resolve to the lower restricted index
    (kernels.cpp:101-104) even when the full ids are in the opposite order."""
    W, ids, h = make_case(5, 2, 64, 300, V=600)
    W[ids[10]] = W[ids[200]]
    W[ids[11]] = W[ids[199]]
    _, out = run_draft(cuda_ctx, W, ids, h, 300, "f32")
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, 300, want_logits=True)
    assert_level_equal(out, ref, 300)


def test_nonfinite_flagged(cuda_ctx):
    W, ids, h = make_case(6, 2, 64, 100)
    h[1, 3] = np.inf
    _, out = run_draft(cuda_ctx, W, ids, h, 4, "f32")
    flags = out.flags.cpu().numpy()
    assert flags[1] & FLAG_NONFINITE and not flags[0] & FLAG_NONFINITE


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_verify_argmax_exact(cuda_ctx, restatement, dtype):
    rng = np.random.default_rng(8)
    V, d, m = 6000, 512, 61
    W = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
    W[4000] = W[17]  # exact tie -> lowest id wins
    if dtype == "bf16":
        W = torch.from_numpy(W).to(torch.bfloat16).to(torch.float32).numpy()
    h = rmsnorm(rng.standard_normal((m, d)))
    h[5] = h[4]
    Wd = torch.from_numpy(W).cuda()
    if dtype == "bf16":
        Wd = Wd.to(torch.bfloat16)
    ids, vals, _ = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), Wd)
    rid, rval = restatement.verify_argmax(h, W)
    assert np.array_equal(ids.cpu().numpy(), rid)
    assert np.array_equal(vals.cpu().numpy(), rval)
    # shard emulation: two contiguous shards + merge == full argmax
    half = V // 2
    a = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), Wd[:half].contiguous(), 0)
    b = api.verify_head_argmax(cuda_ctx, torch.from_numpy(h).cuda(), Wd[half:].contiguous(), half)
    mv, mi = api.argmax_merge(cuda_ctx, torch.stack([a[1], b[1]]), torch.stack([a[0], b[0]]))
    assert np.array_equal(mi.cpu().numpy(), rid)


def test_accept_greedy_matches_oracle(cuda_ctx, restatement):
    rng = np.random.default_rng(9)
    for trial in range(60):
        k = int(rng.integers(1, 65))
        parents = np.array([int(rng.integers(-1, i)) for i in range(k)], np.int32)
        tokens = rng.integers(0, 6, size=k).astype(np.int32)
        argmax_ids = rng.integers(0, 6, size=k + 1).astype(np.int32)
        em, path, cnt = api.accept_greedy(cuda_ctx, torch.from_numpy(argmax_ids).cuda(), torch.from_numpy(tokens).cuda(),
                                          torch.from_numpy(parents).cuda())
        cnt = cnt.cpu().numpy()
        rem, rpath = restatement.verify_greedy_ids(argmax_ids, tokens, parents)
        assert np.array_equal(em.cpu().numpy()[: cnt[0]], rem)
        assert np.array_equal(path.cpu().numpy()[: cnt[1]], rpath)


def test_verify_greedy_host_api(cuda_ctx, restatement):
    rng = np.random.default_rng(10)
    V, d, k = 3000, 256, 20
    W = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
    parents = np.array([-1, -1, 0, 0, 1] + [int(rng.integers(-1, i)) for i in range(5, k)], np.int32)
    h = rmsnorm(rng.standard_normal((k + 1, d)))
    rid, _ = restatement.verify_argmax(h, W)
    tokens = rng.integers(0, V, size=k).astype(np.int32)
    tokens[0] = rid[0]          # root argmax matches node 0 -> accepted
    tokens[2] = rid[1]          # node 0's argmax matches its child node 2
    tree = api.DraftTree(tokens, parents, np.ones(k, np.int32), np.zeros(k))
    out = api.verify_greedy(cuda_ctx, torch.from_numpy(h).cuda(), torch.from_numpy(W).cuda(), tree)
    rem, rpath = restatement.verify_greedy_ids(rid, tokens, parents)
    assert np.array_equal(out.emitted, rem) and np.array_equal(out.accepted_path, rpath)
    assert out.accepted_length() >= 3


@pytest.mark.parametrize("name", ["c1_capture_w4", "c1_capture_w10"])
@pytest.mark.parametrize("dtype", ["f32"])
def test_draft_tree_matches_reference_build_draft_tree(cuda_ctx, reference, name, dtype):
    """C1 end to end: the reference's own hidden states (1-layer draft transformer, patched
    build_draft_tree) through our device head + host beam -> identical tree, log_joints too."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = json.loads(str(z["config"]))
    W = reference.model_lm_head(cfg["V"], cfg["d"], cfg["layers"], cfg["heads"], cfg["seed"])
    assert hashlib.sha256(W.tobytes()).hexdigest() == str(z["lm_head_sha256"])
    subset = api.RankedSubset(cfg["V"], z["ordered"])
    head = api.DeviceHead(cuda_ctx, W, subset, dtype=dtype)
    rows, lev, rtok = z["hidden"], z["row_level"], z["row_token"]

    def provider(level, toks, pars):
        idx = np.where(lev == level)[0]
        if level > 0:
            assert np.array_equal(rtok[idx], toks), "beam diverged from the reference"
        return torch.from_numpy(rows[idx]).cuda()

    params = api.DraftParams(int(z["width"]), int(z["depth"]), int(z["total"]))
    tree = head.build_draft_tree(int(cfg["pending"][-1]), params, mode="exact", provider=provider)
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), z[key]), key


def test_draft_host_e2e_matches_oracle(cuda_ctx, restatement):
    W, ids, h = make_case(12, 10, 512, 8192, V=32000)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(32000, ids), dtype="f32")
    ridx, full, prob = head.draft_host(h, 10)
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, 10)
    assert np.array_equal(ridx, ref["ridx"]) and np.array_equal(full, ref["full"]) and np.array_equal(prob, ref["prob"])


def test_draft_tree_identity_layer_table(cuda_ctx, restatement):
    """Head-path decode loop input: hidden(token) = rmsnorm(E[token]) from a device table."""
    rng = np.random.default_rng(13)
    V, d, v_sub = 4000, 128, 1000
    W = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="f32")
    params = api.DraftParams(10, 6, 60)
    tree = head.build_draft_tree(77, params, hidden_table=torch.from_numpy(E).cuda())

    def provider(level, toks, pars):
        return E[[77]] if level == 0 else E[toks]

    ref = restatement.draft_tree(provider, restatement.restrict(W, ids), ids, 10, 6, 60)
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), ref[key]), key


def test_verify_greedy_table_matches_gathered(cuda_ctx, restatement):
    """frs_verify_greedy_table (device gather of [root, tokens]) == verify_greedy on gathered rows."""
    rng = np.random.default_rng(14)
    V, d = 3000, 128
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    E = rmsnorm(rng.standard_normal((V, d)))
    tree = api.DraftTree(np.array([5, 9, 11, 2], np.int32), np.array([-1, 0, 0, 1], np.int32),
                         np.array([1, 2, 2, 3], np.int32), np.zeros(4))
    Ed, Wd = torch.from_numpy(E).cuda(), torch.from_numpy(W).cuda()
    a = api.verify_greedy_table(cuda_ctx, Ed, 77, Wd, tree)
    rows = np.concatenate([[77], tree.tokens])
    b = api.verify_greedy(cuda_ctx, torch.from_numpy(E[rows]).cuda(), Wd, tree)
    assert np.array_equal(a.emitted, b.emitted) and np.array_equal(a.accepted_path, b.accepted_path)
    ids = restatement.verify_argmax(E[rows], W)[0]
    em, path = restatement.verify_greedy_ids(ids, tree.tokens, tree.parents)
    assert np.array_equal(a.emitted, em) and np.array_equal(a.accepted_path, path)


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("width,depth,total", [(10, 6, 60), (2, 2, 10), (4, 3, 4)])
def test_decode_step_table_matches_two_calls(cuda_ctx, restatement, mode, width, depth, total):
    """frs_decode_step_table (tree -> verify rows -> verify head -> accept on the device, one
    sync) == build_draft_tree + verify_greedy_table, over a chain of iterations. (2, 2, 10):
    the tree holds 6 < total nodes, so the verify rows carry root padding the walk never reads."""
    rng = np.random.default_rng(15)
    V, d, v_sub = 4096, 128, 1024
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    W = torch.from_numpy(W).to(torch.bfloat16).to(torch.float32).numpy()
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="f32")
    Ed, Wb = torch.from_numpy(E).cuda(), torch.from_numpy(W).cuda().to(torch.bfloat16)
    params = api.DraftParams(width, depth, total)
    token = 77
    for _ in range(4):
        tree, out = api.decode_step_table(head, Ed, token, Wb, params, mode=mode)
        ref_tree = head.build_draft_tree(token, params, hidden_table=Ed)
        ref = api.verify_greedy_table(cuda_ctx, Ed, token, Wb, ref_tree, mode=mode)
        for key in ("tokens", "parents", "depths", "log_joint"):
            assert np.array_equal(getattr(tree, key), getattr(ref_tree, key)), key
        assert np.array_equal(out.emitted, ref.emitted) and np.array_equal(out.accepted_path, ref.accepted_path)
        rows = np.concatenate([[token], tree.tokens])
        em, path = restatement.verify_greedy_ids(restatement.verify_argmax(E[rows], W)[0], tree.tokens, tree.parents)
        assert np.array_equal(out.emitted, em) and np.array_equal(out.accepted_path, path)
        token = int(out.emitted[-1])


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("width,depth,total,S", [(10, 6, 60, 7), (2, 2, 10, 3), (4, 3, 4, 9)])
def test_decode_step_table_multi_matches_per_stream(cuda_ctx, restatement, mode, width, depth, total, S):
    """frs_decode_step_table_multi (S streams batched per draft level and in one verify call) ==
    decode_step_table per stream, chained over iterations, and the oracle's verify walk."""
    rng = np.random.default_rng(16)
    V, d, v_sub = 4096, 128, 1024
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    W = torch.from_numpy(W).to(torch.bfloat16).to(torch.float32).numpy()
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="f32")
    Ed, Wb = torch.from_numpy(E).cuda(), torch.from_numpy(W).cuda().to(torch.bfloat16)
    params = api.DraftParams(width, depth, total)
    roots = [int(x) for x in rng.integers(0, V, S)]
    roots[-1] = roots[0]  # two streams at the same token: identical results
    for _ in range(3):
        multi = api.decode_step_table_multi(head, Ed, roots, Wb, params, mode=mode)
        assert len(multi) == S
        for q, (tree, out) in enumerate(multi):
            ref_tree, ref = api.decode_step_table(head, Ed, roots[q], Wb, params, mode=mode)
            for key in ("tokens", "parents", "depths", "log_joint"):
                assert np.array_equal(getattr(tree, key), getattr(ref_tree, key)), (q, key)
            assert np.array_equal(out.emitted, ref.emitted) and np.array_equal(out.accepted_path, ref.accepted_path)
            rows = np.concatenate([[roots[q]], tree.tokens])
            em, path = restatement.verify_greedy_ids(restatement.verify_argmax(E[rows], W)[0], tree.tokens,
                                                     tree.parents)
            assert np.array_equal(out.emitted, em) and np.array_equal(out.accepted_path, path)
        roots = [int(out.emitted[-1]) for _, out in multi]


def test_decode_step_tiled_verify_head(cuda_ctx, restatement):
    """decode_step_table / decode_step_table_multi with the verify head's tiled image (FAST) ==
    without it, chained over iterations."""
    rng = np.random.default_rng(19)
    V, d, v_sub = 4096, 128, 1024
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    W = torch.from_numpy(W).to(torch.bfloat16).to(torch.float32).numpy()
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="f32")
    Ed, Wb = torch.from_numpy(E).cuda(), torch.from_numpy(W).cuda().to(torch.bfloat16)
    Wt = api.tile_image(cuda_ctx, Wb)
    params = api.DraftParams(10, 6, 60)
    token = 77
    for _ in range(3):
        t1, o1 = api.decode_step_table(head, Ed, token, Wb, params, mode="fast", lm_head_tiled=Wt)
        t2, o2 = api.decode_step_table(head, Ed, token, Wb, params, mode="fast")
        assert np.array_equal(t1.tokens, t2.tokens) and np.array_equal(o1.emitted, o2.emitted)
        assert np.array_equal(o1.accepted_path, o2.accepted_path)
        token = int(o1.emitted[-1])
    roots = [5, 77, 1000]
    a = api.decode_step_table_multi(head, Ed, roots, Wb, params, mode="fast", lm_head_tiled=Wt)
    b = api.decode_step_table_multi(head, Ed, roots, Wb, params, mode="fast")
    for (ta, oa), (tb, ob) in zip(a, b):
        assert np.array_equal(ta.tokens, tb.tokens) and np.array_equal(oa.emitted, ob.emitted)


def test_decode_step_table_multi_rejects(cuda_ctx):
    rng = np.random.default_rng(18)
    V, d = 512, 64
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    E = rmsnorm(rng.standard_normal((V, d)))
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, np.arange(256, dtype=np.int32)), dtype="f32")
    Ed, Wd = torch.from_numpy(E).cuda(), torch.from_numpy(W).cuda()
    with pytest.raises(api.InvalidArgument, match="root token outside"):
        api.decode_step_table_multi(head, Ed, [3, V], Wd, api.DraftParams(2, 2, 4))
    with pytest.raises(api.InvalidArgument, match="total_draft_tokens"):
        api.decode_step_table_multi(head, Ed, [3, 4], Wd, api.DraftParams(4, 2, 3))
    with pytest.raises(ValueError, match="at least one stream"):
        api.decode_step_table_multi(head, Ed, [], Wd, api.DraftParams(2, 2, 4))


@pytest.mark.parametrize("v_sub,k,temperature", [(5, 10, 1.0), (100, 16, 1.0), (1000, 3, 0.7), (32768, 10, 1.0),
                                                 (40000, 16, 1.0), (65536, 1, 1.3), (2000, 17, 1.0)])
def test_draft_level_without_total_matches_oracle(cuda_ctx, restatement, v_sub, k, temperature):
    """want_total=False: the cluster softmax + top-k (8 CTAs per row, k <= 16, v_sub <= 65536;
    k = 17 takes the one-CTA kernel) gives the reference's ids, probabilities, row max."""
    W, ids, h = make_case(16, 3, 128, v_sub, V=v_sub + 7, bf16=True)
    h[2] = h[2] * 40.0  # a peaked row: tiny tail probabilities, many e_j = 0 or subnormal
    Wd = torch.from_numpy(W).cuda()
    head = api.restrict_lm_head(cuda_ctx, Wd, api.RankedSubset(W.shape[0], ids), dtype="bf16")
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, k, temperature, mode="exact",
                              want_total=False)
    torch.cuda.synchronize()
    assert out.total is None
    ref = restatement.draft_level(h, restatement.restrict(W, ids), ids, k, temperature)
    kk = min(k, v_sub)
    assert np.array_equal(out.ridx.cpu().numpy()[:, :kk], ref["ridx"][:, :kk])
    assert np.array_equal(out.full.cpu().numpy()[:, :kk], ref["full"][:, :kk])
    assert np.array_equal(out.prob.cpu().numpy()[:, :kk], ref["prob"][:, :kk])
    assert np.array_equal(out.rowmax.cpu().numpy(), ref["mx"])
    if k > v_sub:  # entries past V_sub: -1 / -1 / 0
        assert (out.ridx.cpu().numpy()[:, kk:] == -1).all() and (out.prob.cpu().numpy()[:, kk:] == 0).all()


def test_draft_level_without_total_exact_sum_and_nonfinite(cuda_ctx, restatement):
    """Constant logits (every e_j = 1: the lsb test proves the tree sum exact) and a non-finite
    row through the cluster path."""
    v_sub, d = 3000, 64
    W = np.zeros((v_sub, d), np.float32)
    ids = np.arange(v_sub, dtype=np.int32)
    h = rmsnorm(np.random.default_rng(17).standard_normal((2, d)))
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(v_sub, ids), dtype="f32")
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 12, mode="exact", want_total=False)
    ref = restatement.draft_level(h, W, ids, 12)
    assert np.array_equal(out.ridx.cpu().numpy(), ref["ridx"]) and np.array_equal(out.prob.cpu().numpy(), ref["prob"])
    h[1, 5] = np.nan
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 12, mode="exact", want_total=False)
    flags = out.flags.cpu().numpy()
    assert flags[1] & FLAG_NONFINITE and not flags[0] & FLAG_NONFINITE
