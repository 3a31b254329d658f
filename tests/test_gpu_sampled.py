"""Sampled drafting (drafting.cpp:44-74 with an rng): the device draws
children without replacement from the EXACT probabilities with the reference's
std::mt19937_64 / uniform_real_distribution<double> stream, certifying every draw against the
reference's sequential double sums (k_softmax_sample); the host replays a level otherwise.
Pinned against the compiled reference: its pick_children restatement (ref_pick_sampled, itself
pinned by the sampled capture) and its own build_draft_tree(rng) trees (golden captures)."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api, _lib

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rmsnorm(x):
    x = x.astype(np.float32)
    ms = (x.astype(np.float64) ** 2).mean(axis=1, keepdims=True)
    return (x * (1.0 / np.sqrt(ms + 1e-5)).astype(np.float32)).astype(np.float32)


@pytest.mark.parametrize("scale,width,seed", [(0.02, 10, 3), (0.3, 10, 4), (2.0, 8, 5), (0.05, 64, 6)])
def test_sampled_level_matches_reference(cuda_ctx, reference, scale, width, seed):
    """Per-row draws == the reference's pick_children on the same uniforms (flat, peaked and
    very peaked distributions; width up to 64)."""
    rng = np.random.default_rng(seed)
    V, d, v_sub, n = 6000, 256, 3000, 6
    W = (rng.standard_normal((V, d)) * scale).astype(np.float32)
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    h = rmsnorm(rng.standard_normal((n, d)))
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(V, ids), dtype="f32")
    w = min(width, v_sub)
    u = reference.uniforms(100 + seed, n * w)
    out = api.draft_head_sample(cuda_ctx, torch.from_numpy(h).cuda(), head, width, torch.from_numpy(u.reshape(n, w)))
    ex = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 1, mode="exact", want_logits=True)
    logits = ex.logits.cpu().numpy()
    probs = out.probs.cpu().numpy()
    cnt, fl = out.count.cpu().numpy(), out.flags.cpu().numpy()
    for r in range(n):
        ref_p = reference.softmax(logits[r], 1.0)
        assert np.array_equal(probs[r], ref_p), r  # bit-exact probabilities
        picks, pr = reference.pick_sampled(ref_p, width, 100 + seed, skip=r * w)
        if fl[r] & _lib.FLAG_SAMPLE_UNCERTIFIED:
            continue  # the host replays such rows (covered by the tree tests)
        assert cnt[r] == picks.size
        assert np.array_equal(out.ridx.cpu().numpy()[r, :cnt[r]], picks), r
        assert np.array_equal(out.prob.cpu().numpy()[r, :cnt[r]], pr), r
        assert np.array_equal(out.full.cpu().numpy()[r, :cnt[r]], ids[picks]), r
    assert (fl & _lib.FLAG_SAMPLE_UNCERTIFIED).sum() <= 1


@pytest.mark.parametrize("v_sub,width", [(32768, 10), (40000, 16), (50000, 10), (5, 10)])
def test_sampled_level_large_rows(cuda_ctx, reference, v_sub, width):
    """Against the reference's pick_children at C2 widths: the cluster sampler (8 CTAs per row
    softmax, the leader draws from shared memory; 16 logits per thread above 32768) and, past
    the 160 KB shared draw weights (50000), the one-CTA kernel with global draw weights."""
    rng = np.random.default_rng(77)
    V, d, n = v_sub + 100, 128, 4
    W = (rng.standard_normal((V, d)) * 0.1).astype(np.float32)
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    h = rmsnorm(rng.standard_normal((n, d)))
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(V, ids), dtype="f32")
    w = min(width, v_sub)
    u = reference.uniforms(900, n * w)
    out = api.draft_head_sample(cuda_ctx, torch.from_numpy(h).cuda(), head, width, torch.from_numpy(u.reshape(n, w)))
    ex = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 1, mode="exact", want_logits=True)
    logits, probs = ex.logits.cpu().numpy(), out.probs.cpu().numpy()
    cnt, fl = out.count.cpu().numpy(), out.flags.cpu().numpy()
    for r in range(n):
        ref_p = reference.softmax(logits[r], 1.0)
        assert np.array_equal(probs[r], ref_p), r
        picks, pr = reference.pick_sampled(ref_p, width, 900, skip=r * w)
        if fl[r] & _lib.FLAG_SAMPLE_UNCERTIFIED:
            continue
        assert cnt[r] == picks.size
        assert np.array_equal(out.ridx.cpu().numpy()[r, :cnt[r]], picks), r
        assert np.array_equal(out.prob.cpu().numpy()[r, :cnt[r]], pr), r
    assert (fl & _lib.FLAG_SAMPLE_UNCERTIFIED).sum() <= 1


@pytest.mark.parametrize("name", ["c1_sampled_w4_s11", "c1_sampled_w10_s5"])
def test_sampled_tree_matches_reference_build_draft_tree(cuda_ctx, reference, name):
    """C1 end to end in sampled mode: the reference's hidden states and its build_draft_tree(rng)
    tree; our device head + sampler + host bookkeeping with the same mt19937_64 seed."""
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = json.loads(str(z["config"]))
    W = reference.model_lm_head(cfg["V"], cfg["d"], cfg["layers"], cfg["heads"], cfg["seed"])
    assert hashlib.sha256(W.tobytes()).hexdigest() == str(z["lm_head_sha256"])
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(cfg["V"], z["ordered"]), dtype="f32")
    rows, lev, rtok = z["hidden"], z["row_level"], z["row_token"]

    def provider(level, toks, pars):
        idx = np.where(lev == level)[0]
        if level > 0:
            assert np.array_equal(rtok[idx], toks), "beam diverged from the reference"
        return torch.from_numpy(rows[idx]).cuda()

    params = api.DraftParams(int(z["width"]), int(z["depth"]), int(z["total"]))
    tree = head.build_draft_tree(int(cfg["pending"][-1]), params, mode="exact", provider=provider,
                                 rng=api.Rng(int(z["rng_seed"])))
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), z[key]), key


def test_sampled_tree_table_prefix_closed(cuda_ctx, reference):
    """Hidden rows from a device table: the tree is prefix-closed per parent (the children kept
    are a prefix of the draw order), topological, inside the subset; same seed -> same tree."""
    rng = np.random.default_rng(9)
    V, d, v_sub = 4000, 128, 1200
    W = (rng.standard_normal((V, d)) * 0.3).astype(np.float32)
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    sub = api.RankedSubset(V, ids)
    head = api.DeviceHead(cuda_ctx, W, sub, dtype="f32")
    Ed = torch.from_numpy(E).cuda()
    params = api.DraftParams(6, 4, 30)
    t1 = head.build_draft_tree(int(ids[1]), params, hidden_table=Ed, rng=api.Rng(77))
    t2 = head.build_draft_tree(int(ids[1]), params, hidden_table=Ed, rng=api.Rng(77))
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(t1, key), getattr(t2, key)), key
    K = len(t1)
    assert 1 <= K <= 30
    for i in range(K):
        p = int(t1.parents[i])
        assert -1 <= p < i and sub.contains(int(t1.tokens[i]))
        if p >= 0:
            assert t1.depths[i] == t1.depths[p] + 1
    with pytest.raises(ValueError):
        head.build_draft_tree(int(ids[1]), params, mode="fast", hidden_table=Ed, rng=api.Rng(1))


def _softmax64(x):
    x = x.astype(np.float64)
    e = np.exp(x - x.max())
    return (e / e.sum()).astype(np.float32)


@pytest.mark.parametrize("seed,scale,temperature", [(1, 0.05, 1.0), (2, 0.3, 1.0), (3, 0.3, 0.7), (4, 1.5, 1.0)])
def test_verify_stochastic_matches_reference(cuda_ctx, reference, seed, scale, temperature):
    """verification.cpp:76-178 end to end: exact target probabilities on the device + the
    residual walk; emitted tokens and accepted path == the reference's verify_stochastic on
    the same logits, draft distributions, subset and mt19937_64 seed. Targets correlated with
    the drafts so paths get accepted as well as rejected."""
    rng = np.random.default_rng(seed)
    V, d, v_sub, k = 3000, 128, 900, 20
    W = (rng.standard_normal((V, d)) * scale).astype(np.float32)
    ordered = rng.permutation(V)[:v_sub].astype(np.int32)
    parents = np.array([-1, -1, -1, 0, 0, 1, 3, 3, 4, 6, 6, 2, 2, 11, 9, 9, 14, 7, 7, 17], np.int32)
    # draft distributions over the subset; tokens drawn from them (so q > 0)
    q_root = _softmax64(rng.standard_normal(v_sub) * 3.0)
    q_nodes = np.stack([_softmax64(rng.standard_normal(v_sub) * 3.0) for _ in range(k)])
    has_q = np.zeros(k, np.int32)
    has_q[np.unique(parents[parents >= 0])] = 1
    tokens = np.empty(k, np.int32)
    for i in range(k):
        q = q_root if parents[i] < 0 else q_nodes[parents[i]]
        sib = tokens[:i][parents[:i] == parents[i]]
        order = np.argsort(-q, kind="stable")
        cand = [int(ordered[j]) for j in order[:8] if int(ordered[j]) not in sib]
        tokens[i] = cand[rng.integers(0, 3)]
    h = rmsnorm(rng.standard_normal((1 + k, d)))
    # align about half of the target rows with one of their drafted children (that child then
    # carries most of the target mass: accepted), leave the others random (rejections)
    for row in range(1 + k):
        kids = np.where(parents == row - 1)[0]
        if kids.size and rng.random() < 0.6:
            t = tokens[kids[rng.integers(0, kids.size)]]
            h[row] = (12.0 / (np.linalg.norm(W[t]) + 1e-6)) * W[t] / (np.linalg.norm(W[t]) + 1e-6) * np.float32(
                min(1.0, 1.0 / scale))
    Wd = torch.from_numpy(W).cuda()
    tree = api.DraftTree(tokens, parents, np.ones(k, np.int32), np.zeros(k))
    logits = reference.matmul(h, W)  # the reference's dot_f32 logits
    for rs in (11, 12, 13):
        out = api.verify_stochastic(cuda_ctx, torch.from_numpy(h).cuda(), Wd, tree, q_root, q_nodes, has_q, ordered,
                                    api.Rng(1000 * seed + rs), temperature)
        em, path = reference.verify_stochastic(logits[0], logits[1:], tokens, parents, q_root, q_nodes, has_q,
                                               ordered, temperature, 1000 * seed + rs)
        assert np.array_equal(out.emitted, em) and np.array_equal(out.accepted_path, path), rs
        _LENS.append(int(path.size))


_LENS = []


def test_verify_stochastic_paths_cover_accept_and_reject():
    """The parity cases above covered both outcomes: rejected at the root and accepted paths."""
    if not _LENS:
        pytest.skip("parity cases did not run")
    assert min(_LENS) == 0 and max(_LENS) >= 2, _LENS


@pytest.mark.parametrize("seed,rng_seed,width,depth,total", [(7, 11, 4, 3, 12), (9, 5, 6, 4, 24), (13, 3, 3, 2, 6)])
def test_sampled_tree_keep_probs_then_verify_stochastic(cuda_ctx, reference, seed, rng_seed, width, depth, total):
    """The decode loop's stochastic step end to end through the C ABI: sampled drafting with
    keep_probs on the device draft model (frs_draft_tree_model), its DraftResult distributions fed
    to frs_verify_stochastic with the same engine — tree, root/node distributions, emitted tokens
    and accepted path all equal the reference's build_draft_tree(rng, keep_probs) followed by
    verify_stochastic (drafting.cpp:122-245, verification.cpp:76-178)."""
    V, d, heads, max_seq = 900, 64, 4, 64
    sess = reference.draft_session(V, d, heads, max_seq, seed)
    draft = api.DraftModel(cuda_ctx, sess.weights(), heads, max_seq)
    W = reference.model_lm_head(V, d, 1, heads, seed)
    ordered = np.random.default_rng(seed).permutation(V)[:300].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ordered), dtype="f32")
    g = np.random.default_rng(seed + 1)
    h_t = g.standard_normal((total + 1, d)).astype(np.float32)
    W_t = (g.standard_normal((V, d)) * 0.3).astype(np.float32)
    pending = [5, 17, 42]
    ref = reference.draft_verify_rng(V, d, heads, max_seq, seed, ordered, pending, width, depth, total, rng_seed, h_t,
                                     W_t)
    rng = api.Rng(rng_seed)
    tree = api.build_draft_tree_model(head, draft, pending, api.DraftParams(width, depth, total), rng=rng,
                                      keep_probs=True)
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), ref[key]), key
    assert np.array_equal(tree.root_probs, ref["root_probs"])
    assert np.array_equal(tree.has_probs, ref["has_probs"])
    assert np.array_equal(tree.node_probs, ref["node_probs"])
    K = len(tree)
    out = api.verify_stochastic(cuda_ctx, torch.from_numpy(h_t[:K + 1]).cuda(), torch.from_numpy(W_t).cuda(), tree,
                                tree.root_probs, tree.node_probs, tree.has_probs, ordered, rng)
    assert np.array_equal(out.emitted, ref["emitted"])
    assert np.array_equal(out.accepted_path, ref["path"])
    with pytest.raises(api.NotSupported):
        api.build_draft_tree_model(head, draft, pending, api.DraftParams(width, depth, total), keep_probs=True)
