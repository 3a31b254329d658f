"""GPU property tests:

* draft-tree structure: topological parents, ancestor-closed tree masks, depth = parent + 1,
  every drafted token inside the FR subset, log-joint non-increasing along every path;
* FR remap identity: restricted -> full -> restricted is the identity on every drafted child;
* renormalisation: EXACT probabilities over the whole restricted row sum to 1 (within fp32),
  and the top-k probabilities are sorted and match softmax(logits) element-wise;
* greedy losslessness: head-path speculative decoding with greedy verify emits
  exactly the tokens of plain greedy decoding with the target head (FAST and EXACT modes).
"""
import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api

pytestmark = pytest.mark.gpu


def rmsnorm(x):
    x = x.astype(np.float32)
    ms = (x.astype(np.float64) ** 2).mean(axis=1, keepdims=True)
    return (x * (1.0 / np.sqrt(ms + 1e-5)).astype(np.float32)).astype(np.float32)


def _setup(seed, V=6000, d=256, v_sub=2000):
    rng = np.random.default_rng(seed)
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.05).astype(np.float32)).to(torch.bfloat16).float().numpy()
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    return W, E, ids


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_draft_tree_structure(cuda_ctx, mode, seed):
    W, E, ids = _setup(seed)
    sub = api.RankedSubset(W.shape[0], ids)
    head = api.DeviceHead(cuda_ctx, W, sub, dtype="bf16")
    tree = head.build_draft_tree(int(ids[5]), api.DraftParams(6, 5, 30), mode=mode,
                                 hidden_table=torch.from_numpy(E).cuda())
    K = len(tree)
    assert 1 <= K <= 30
    words = api.build_tree_mask(tree.parents)
    for i in range(K):
        p = int(tree.parents[i])
        assert -1 <= p < i
        assert sub.contains(int(tree.tokens[i]))
        assert sub.full_id(sub.restricted_index(int(tree.tokens[i]))) == int(tree.tokens[i])
        if p < 0:
            assert tree.depths[i] == 1 and words[i] == (1 << i)
        else:
            assert tree.depths[i] == tree.depths[p] + 1
            assert tree.log_joint[i] <= tree.log_joint[p]
            assert (int(words[i]) & int(words[p])) == int(words[p])  # ancestor closure
            assert int(words[i]) == int(words[p]) | (1 << i)
    # siblings carry distinct tokens (top-k over distinct restricted indices, injective remap)
    for p in set(tree.parents.tolist()):
        kids = tree.tokens[tree.parents == p]
        assert len(set(kids.tolist())) == kids.size


def test_renormalisation_identity(cuda_ctx, restatement):
    rng = np.random.default_rng(9)
    V, d, v_sub = 9000, 512, 4096
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.02).astype(np.float32)).to(torch.bfloat16).float().numpy()
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    h = rmsnorm(rng.standard_normal((5, d)))
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(V, ids), dtype="bf16")
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 16, mode="exact", want_logits=True)
    logits = out.logits.cpu().numpy()
    for r in range(5):
        p, mx, tot = restatement.softmax(logits[r])
        assert abs(float(p.astype(np.float64).sum()) - 1.0) < 1e-5
        assert np.array_equal(out.prob.cpu().numpy()[r], p[out.ridx.cpu().numpy()[r]])
        pr = out.prob.cpu().numpy()[r]
        assert np.all(pr[:-1] >= pr[1:])
        assert out.rowmax.cpu().numpy()[r] == mx and out.total.cpu().numpy()[r] == tot
    fast = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 16, mode="fast")
    assert np.array_equal(fast.full.cpu().numpy(), out.full.cpu().numpy())


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_greedy_losslessness(cuda_ctx, restatement, mode):
    """Speculative decoding (head path, identity draft layer) with greedy verify emits the same
    tokens as plain greedy decoding with the target head: t_{s+1} = argmax(W . E[t_s])."""
    rng = np.random.default_rng(31)
    V, d, v_sub = 5000, 256, 1500
    # a peaked target (E rows aligned with W rows) so drafts are often accepted
    Wf = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    nxt = rng.permutation(V)
    E = rmsnorm(Wf[nxt] * 20.0 + rng.standard_normal((V, d)).astype(np.float32))
    W = torch.from_numpy(Wf).to(torch.bfloat16)
    Wn = W.float().numpy()
    counts = np.bincount(nxt[rng.integers(0, V, 200000)], minlength=V).astype(np.uint64)
    sub = api.build_subset(api.FrequencyTable(V, counts, int(counts.sum())), v_sub)
    head = api.DeviceHead(cuda_ctx, Wn, sub, dtype="bf16")
    Ed = torch.from_numpy(E).cuda()
    token, produced = 17, []
    stats = api.AcceptanceStats()
    while len(produced) < 40:
        tree = head.build_draft_tree(token, api.DraftParams(4, 4, 16), mode=mode, hidden_table=Ed)
        rows = np.concatenate([[token], tree.tokens]).astype(np.int64)
        outc = api.verify_greedy(cuda_ctx, Ed[torch.from_numpy(rows).cuda()].contiguous(), W.cuda(), tree, mode=mode)
        stats.add(outc.accepted_length())
        produced.extend(int(t) for t in outc.emitted)
        token = int(outc.emitted[-1])
    vanilla, t = [], 17
    for _ in range(len(produced)):
        t = int(restatement.verify_argmax(E[[t]], Wn)[0][0])
        vanilla.append(t)
    assert produced == vanilla
    assert stats.mean_accepted_length > 1.0  # the drafts do get accepted
