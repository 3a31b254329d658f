"""CPU: pin the plain-C restatement (oracle/frs_oracle.c) to the compiled reference and the
committed golden vectors (SURVEY.md §4.2 worked examples, §8(c))."""
import ctypes
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _spec():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as fh:
        return json.load(fh)


def test_spec_examples_restatement(restatement):
    R, spec = restatement, _spec()
    f32 = np.float32
    assert R.logits(np.array([[1, 2]], f32), np.array([[3, 4], [5, 6]], f32)).tolist() == spec["matmul"]
    p, _, _ = R.softmax(np.log(np.array([1, 2, 3], f32)))
    assert p.tolist() == spec["softmax_ln123"]
    idx, val = R.topk(np.array([5, 1, 7, 7], f32), 2)
    assert [[int(i), float(v)] for i, v in zip(idx, val)] == spec["topk_5177_k2"]
    assert R.build_subset(np.array([5, 1, 7, 7], np.uint64), 2).tolist() == spec["build_subset_5177_size2"]
    assert R.build_subset(np.array([5, 1, 7, 7], np.uint64), 2, [1]).tolist() == spec["build_subset_5177_size2_forced1"]
    assert [int(w) for w in R.tree_mask([-1, 0, 1, 2])] == spec["tree_mask_chain4"]
    assert R.argmax(np.array([1, 3, 3, 2], f32)) == spec["argmax_ties"]
    em, path = R.verify_greedy_ids([7, 9, 3], [7, 5], [-1, -1])
    assert em.tolist() == spec["verify_accept_then_bonus"]["emitted"]
    assert path.tolist() == spec["verify_accept_then_bonus"]["path"]


def test_softmax_constant_and_shift(restatement):
    p, _, _ = restatement.softmax(np.full(4, 3.25, np.float32))
    assert np.allclose(p, 0.25)
    v = np.random.default_rng(1).standard_normal(100).astype(np.float32)
    assert np.allclose(restatement.softmax(v)[0], restatement.softmax(v + 7)[0], atol=1e-6)


@pytest.mark.parametrize("d", [8, 13, 512, 4096])
def test_dot_and_logits_bitwise_vs_reference(restatement, reference, d):
    rng = np.random.default_rng(d)
    h = rng.standard_normal((3, d)).astype(np.float32)
    W = (rng.standard_normal((257, d)) * 0.02).astype(np.float32)
    assert np.array_equal(restatement.logits(h, W), reference.matmul(h, W))


def test_softmax_topk_bitwise_vs_reference(restatement, reference):
    rng = np.random.default_rng(2)
    for t in (1.0, 0.7, 2.5):
        x = (rng.standard_normal(5000) * 4).astype(np.float32)
        p, _, _ = restatement.softmax(x, t)
        assert np.array_equal(p, reference.softmax(x, t))
    for _ in range(300):
        v = rng.integers(0, 6, size=int(rng.integers(1, 80))).astype(np.float32)
        k = int(rng.integers(1, v.size + 1))
        a, b = restatement.topk(v, k), reference.topk(v, k)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_rejections_match_reference(restatement, reference):
    with pytest.raises(ValueError):
        reference.softmax(np.array([1.0, np.inf], np.float32))
    with pytest.raises(ValueError):
        restatement.softmax(np.array([1.0, np.inf], np.float32))
    with pytest.raises(ValueError):
        reference.topk(np.ones(3, np.float32), 4)
    with pytest.raises(ValueError):
        restatement.topk(np.ones(3, np.float32), 4)
    with pytest.raises(OverflowError):
        reference.tree_mask(np.arange(-1, 64, dtype=np.int32))
    with pytest.raises(OverflowError):
        restatement.tree_mask(np.arange(-1, 64, dtype=np.int32))


def test_expf_port_matches_host_libm_sampled(restatement):
    """the glibc expf port equals host expf on [-104, 0]. Sampled here
    (every 4099th float); both device ports are checked exhaustively against host libm in
    tests/test_gpu_expf_kat.py."""
    libm = ctypes.CDLL("libm.so.6")
    libm.expf.restype, libm.expf.argtypes = ctypes.c_float, [ctypes.c_float]
    lo = np.float32(-104.0).view(np.uint32)
    bits = np.arange(0x80000000, lo + 1, 4099, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    bad = [x for x in xs[::7] if restatement.expf(x) != libm.expf(x)]
    assert bad == []


def test_vocab_restatement_vs_reference(restatement, reference):
    s = reference.zipf_tokens(5000, 1.1, 200_000, 9)
    counts, total = reference.count_frequencies(s, 5000)
    assert total == s.size
    assert np.array_equal(restatement.count_frequencies(s, 5000), counts)
    for size, forced in ((1, []), (100, [0, 4999, 17]), (5000, [3])):
        assert np.array_equal(restatement.build_subset(counts, size, forced), reference.build_subset(counts, size, forced))
    rk = np.random.default_rng(3).permutation(5000).astype(np.int32)
    for size, forced in ((10, [rk[4000], rk[4999]]), (4999, [rk[4999]]), (7, [])):
        assert np.array_equal(restatement.subset_from_ranking(rk, size, 5000, forced),
                              reference.subset_from_ranking(rk, size, 5000, forced))
    W = np.random.default_rng(4).standard_normal((5000, 24)).astype(np.float32)
    ordered = reference.build_subset(counts, 300, [0])
    assert np.array_equal(restatement.restrict(W, ordered), reference.restrict_lm_head(W, ordered))


@pytest.mark.parametrize("name", ["c1_capture_w4", "c1_capture_w10"])
def test_headpath_tree_matches_reference_build_draft_tree(restatement, reference, name):
    """The head-path restatement fed the reference's own per-level hidden states reproduces the
    reference build_draft_tree (patched) tree bit for bit (drafting.cpp:122-245)."""
    import hashlib
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = json.loads(str(z["config"]))
    W = reference.model_lm_head(cfg["V"], cfg["d"], cfg["layers"], cfg["heads"], cfg["seed"])
    assert hashlib.sha256(W.tobytes()).hexdigest() == str(z["lm_head_sha256"])
    slab = restatement.restrict(W, z["ordered"])
    rows, lev, rtok = z["hidden"], z["row_level"], z["row_token"]

    def provider(level, toks, pars):
        idx = np.where(lev == level)[0]
        if level > 0:
            assert np.array_equal(rtok[idx], toks)
        return rows[idx]

    t = restatement.draft_tree(provider, slab, z["ordered"], int(z["width"]), int(z["depth"]), int(z["total"]))
    for k in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(t[k], z[k]), k


@pytest.mark.parametrize("width,depth,total,seed", [(3, 3, 9, 1), (5, 4, 20, 2)])
def test_sampled_capture_matches_reference_build_draft_tree(reference, width, depth, total, seed):
    """The sampled capture loop (pick_children's sampled branch restated in the shim, prefix-closed
    select_top_k) reproduces the reference's own build_draft_tree(rng) — this pins
    ref_pick_sampled, the checker of the device sampler (tests/test_gpu_sampled.py)."""
    rng = np.random.default_rng(seed)
    V, d = 2000, 64
    ordered = rng.permutation(V)[:700].astype(np.int32)
    args = (V, d, 1, 4, 64, 7 + seed, ordered, np.array([5, 17, 300], np.int32), width, depth, total, 900 + seed)
    tree = reference.model_draft_tree_rng(*args)
    cap = reference.model_draft_capture_rng(*args)
    for k in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(tree[k], cap[k]), k


def test_sampled_goldens_consistent(reference):
    """The committed sampled goldens are prefix-closed trees of the stated size."""
    for name in ("c1_sampled_w4_s11", "c1_sampled_w10_s5"):
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        par, dep = z["parents"], z["depths"]
        assert par.size == int(z["total"])
        for i, p in enumerate(par):
            assert -1 <= p < i and (p < 0 or dep[i] == dep[p] + 1)
