"""The draft transformer layer on the device (model.cpp:208-281):
forward_raw of the reference's 1-layer draft (build_draft truncated) reproduced bit for bit —
the hidden states after a causal context forward and after tree-shaped beam forwards on the
growing KV cache — against the compiled reference running the same calls on its own cache."""
import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api
from paper_2502_14856_b200._lib import CapacityError

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("V,d,heads,seed", [(500, 64, 4, 7), (2000, 128, 8, 11), (3000, 96, 3, 5)])
def test_draft_layer_forward_matches_reference(cuda_ctx, reference, V, d, heads, seed):
    max_seq = 48
    ref = reference.draft_session(V, d, heads, max_seq, seed)
    dev = api.DraftModel(cuda_ctx, ref.weights(), heads, max_seq)
    rng = np.random.default_rng(seed)
    # 1. the pending context, causal (draft_forward without a tree mask)
    ctx_toks = rng.integers(0, V, 6)
    pos = np.arange(6)
    allow = np.tril(np.ones((6, 6), np.uint8))
    h_ref = ref.forward(ctx_toks, pos, allow)
    h_dev = dev.forward(ctx_toks, pos, allow).cpu().numpy()
    assert np.array_equal(h_dev, h_ref)
    # 2. two tree levels: each beam row sees the context, its forwarded ancestors and itself;
    #    positions = anchor + depth (drafting.cpp:180-196)
    base, anchor = 6, 5
    parents_rows = []  # cache row of each forwarded beam row
    beam = [(int(t), -1, 1) for t in rng.integers(0, V, 4)]  # (token, parent cache row, depth)
    for level in range(2):
        n = len(beam)
        m = len(dev) + n
        allow = np.zeros((n, m), np.uint8)
        allow[:, :base] = 1
        for i, (tok, par, depth) in enumerate(beam):
            a = par
            while a >= 0:
                allow[i, a] = 1
                a = parents_rows[a - base] if a - base < len(parents_rows) else -1
            allow[i, len(dev) + i] = 1
        toks = [b[0] for b in beam]
        pos = [anchor + b[2] for b in beam]
        h_ref = ref.forward(toks, pos, allow)
        h_dev = dev.forward(toks, pos, allow).cpu().numpy()
        assert np.array_equal(h_dev, h_ref), level
        first = len(dev) - n
        parents_rows += [b[1] for b in beam]
        beam = [(int(rng.integers(0, V)), first + (i % n), beam[i % n][2] + 1) for i in range(5)]


def test_draft_layer_capacity_and_truncate(cuda_ctx, reference):
    ref = reference.draft_session(300, 32, 2, 8, 3)
    dev = api.DraftModel(cuda_ctx, ref.weights(), 2, 8)
    dev.forward(np.arange(6), np.arange(6), np.tril(np.ones((6, 6), np.uint8)))
    with pytest.raises(CapacityError, match="exceeds max_seq_len 8"):
        dev.forward(np.arange(3), np.arange(6, 9), np.ones((3, 9), np.uint8))
    dev.truncate(2)
    assert len(dev) == 2
    h = dev.forward([7], [2], np.ones((1, 3), np.uint8))
    assert h.shape == (1, 32)
    # a query row that permits no key: the reference's masked_attention rejects it; nothing is
    # appended to the cache
    allow = np.ones((2, 5), np.uint8)
    allow[1] = 0
    with pytest.raises(ValueError, match="permits no keys"):
        dev.forward([1, 2], [3, 4], allow)
    assert len(dev) == 3


@pytest.mark.parametrize("name", ["c1_capture_w4", "c1_capture_w10", "c1_sampled_w4_s11", "c1_sampled_w10_s5"])
def test_model_driven_draft_tree_matches_reference(cuda_ctx, reference, name):
    """The whole C1 drafting step on the GPU — draft transformer layer + FR head + beam
    bookkeeping (greedy and sampled) — against the reference's own build_draft_tree trees."""
    import hashlib
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".npz"))
    cfg = json.loads(str(z["config"]))
    W = reference.model_lm_head(cfg["V"], cfg["d"], cfg["layers"], cfg["heads"], cfg["seed"])
    assert hashlib.sha256(W.tobytes()).hexdigest() == str(z["lm_head_sha256"])
    sess = reference.draft_session(cfg["V"], cfg["d"], cfg["heads"], 64, cfg["seed"])
    draft = api.DraftModel(cuda_ctx, sess.weights(), cfg["heads"], 64)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(cfg["V"], z["ordered"]), dtype="f32")
    params = api.DraftParams(int(z["width"]), int(z["depth"]), int(z["total"]))
    rng = api.Rng(int(z["rng_seed"])) if "rng_seed" in z.files else None
    tree = api.build_draft_tree_model(head, draft, cfg["pending"], params, mode="exact", rng=rng)
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), z[key]), key
    assert len(draft) == len(cfg["pending"])  # cache truncated back to the context (drafting.cpp:225)


def test_exact_logits_wide_inputs(cuda_ctx, restatement):
    """Hidden widths whose rows no longer fit four to a CTA in shared memory (the 4d MLP down
    projection at d = 4096 reads 16384-wide rows) take the global-memory dot_f32 kernel: same
    bits as the reference's matmul."""
    rng = np.random.default_rng(2)
    V, d, n = 300, 16384 + 5, 3  # a dot_f32 tail too
    W = (rng.standard_normal((V, d)) * 0.01).astype(np.float32)
    h = rng.standard_normal((n, d)).astype(np.float32)
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(V, np.arange(V, dtype=np.int32)),
                                dtype="f32")
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, 4, mode="exact", want_logits=True)
    assert np.array_equal(out.logits.cpu().numpy(), restatement.logits(h, W))


def test_model_draft_tree_on_persistent_cache(cuda_ctx, reference):
    """Two drafting steps on the same draft model, the second after the first's context (a
    decode loop's cache): the pending tokens continue at the cache's last position + 1
    (causal_layout, model.cpp:288-297) and both trees equal the reference's build_draft_tree on
    its own persistent cache."""
    V, d, heads, seed, max_seq = 700, 64, 4, 19, 96
    sess = reference.draft_session(V, d, heads, max_seq, seed)
    draft = api.DraftModel(cuda_ctx, sess.weights(), heads, max_seq)
    W = reference.model_lm_head(V, d, 1, heads, seed)
    ordered = np.random.default_rng(seed).permutation(V)[:256].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ordered), dtype="f32")
    params = api.DraftParams(4, 3, 12)
    for step, pending in enumerate(([3, 14, 15, 92], [65, 35], [89])):
        ref = sess.draft_tree(ordered, pending, 4, 3, 12)
        tree = api.build_draft_tree_model(head, draft, pending, params, mode="exact")
        for key in ("tokens", "parents", "depths", "log_joint"):
            assert np.array_equal(getattr(tree, key), ref[key]), (step, key)
        assert len(draft) == len(sess)
        assert [draft.position(r) for r in range(len(draft))] == [sess.position(r) for r in range(len(sess))]


def test_kv_compact_matches_reference(cuda_ctx, reference):
    """KVCache::compact (model.cpp:165-196) on the device cache: the kept rows move down with
    their positions, a later forward sees exactly the reference's cache; the rejections."""
    from paper_2502_14856_b200._lib import InvalidArgument, LogicError
    V, d, heads, seed, max_seq = 400, 64, 4, 23, 40
    sess = reference.draft_session(V, d, heads, max_seq, seed)
    dev = api.DraftModel(cuda_ctx, sess.weights(), heads, max_seq)
    rng = np.random.default_rng(seed)
    toks = rng.integers(0, V, 5)
    allow = np.tril(np.ones((5, 5), np.uint8))
    sess.forward(toks, np.arange(5), allow)
    dev.forward(toks, np.arange(5), allow)
    # a tree level of 4 rows at positions 5, 6, 6, 7 (rows 5..8); accept rows 5 and 7 (offsets 0, 2)
    tree_toks = rng.integers(0, V, 4)
    tpos = np.array([5, 6, 6, 7])
    tallow = np.ones((4, 9), np.uint8)
    sess.forward(tree_toks, tpos, tallow)
    dev.forward(tree_toks, tpos, tallow)
    for bad_from, bad_offs, exc in ((-1, [0], InvalidArgument), (10, [0], InvalidArgument),
                                    (5, [1, 0], InvalidArgument), (5, [4], InvalidArgument)):
        with pytest.raises(exc):
            dev.compact(bad_from, bad_offs)
        with pytest.raises(ValueError):
            sess.compact(bad_from, bad_offs)
    assert len(dev) == 9
    sess.compact(5, [0, 2])
    dev.compact(5, [0, 2])
    assert len(dev) == len(sess) == 7
    assert [dev.position(r) for r in range(7)] == [sess.position(r) for r in range(7)] == list(range(7))
    nxt = rng.integers(0, V, 2)
    h_ref = sess.forward(nxt, [7, 8], np.tril(np.ones((2, 9), np.uint8), 7))
    h_dev = dev.forward(nxt, [7, 8], np.tril(np.ones((2, 9), np.uint8), 7)).cpu().numpy()
    assert np.array_equal(h_dev, h_ref)
    # positions 0..8 then keeping offsets {1} of keep_from 7: position 8 lands at row 7 after 6
    with pytest.raises(LogicError, match="not contiguous"):
        dev.compact(6, [0, 2])
    with pytest.raises(RuntimeError, match="not contiguous"):
        sess.compact(6, [0, 2])
    assert len(dev) == len(sess) == 8


def test_forward_shape_rejections(cuda_ctx, reference):
    from paper_2502_14856_b200._lib import InvalidArgument
    sess = reference.draft_session(300, 32, 2, 8, 3)
    dev = api.DraftModel(cuda_ctx, sess.weights(), 2, 8)
    with pytest.raises(InvalidArgument, match="positions size mismatch"):
        dev.forward([1, 2], [0], np.tril(np.ones((2, 2), np.uint8)))
    with pytest.raises(InvalidArgument, match="visibility mask shape mismatch"):
        dev.forward([1, 2], [0, 1], np.ones((2, 1), np.uint8))
    assert len(dev) == 0
