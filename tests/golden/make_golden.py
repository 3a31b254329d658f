"""Generates the committed golden fixtures from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py [--sampled]
Outputs:
  spec_examples.json   SPEC.md worked examples evaluated by the reference (SPEC.md:38-67,
                       217-219, 246, 354) — asserted against the SPEC's stated answers.
  c1_capture_w4.npz    C1 (d=512, V=32000, V_sub=8192, width 4, depth 3, K 16): the
  c1_capture_w10.npz   reference's build_draft_tree tree + the hidden state of every
                       forwarded draft row (restated loop around forward_raw), for width 4
                       and for width 10 / depth 6 / K 60 (exercises beam pruning).
  c1_sampled_w4_s11.npz / c1_sampled_w10_s5.npz (--sampled): the same for sampled drafting
                       (build_draft_tree with std::mt19937_64(rng_seed), prefix-closed selection).
The LM head is regenerated from the seed on the GPU box through oracle/_ref and checked
against the stored sha256, so no weights are committed.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference, build  # noqa: E402

C1 = dict(V=32000, d=512, layers=1, heads=8, seed=7, v_sub=8192, zipf_seed=42, zipf_count=1_000_000,
          forced=[0, 1], pending=[5, 17, 300, 2])


def c1_subset(ref: Reference):
    s = ref.zipf_tokens(C1["V"], 1.0, C1["zipf_count"], C1["zipf_seed"])
    counts, _ = ref.count_frequencies(s, C1["V"])
    return ref.build_subset(counts, C1["v_sub"], C1["forced"])


def main():
    build(reference=True)
    ref = Reference()
    f32 = np.float32
    spec = {}
    spec["matmul"] = ref.matmul(np.array([[1, 2]], f32), np.array([[3, 4], [5, 6]], f32)).tolist()
    assert spec["matmul"] == [[11.0, 17.0]]
    spec["softmax_ln123"] = [float(x) for x in ref.softmax(np.log(np.array([1, 2, 3], f32)))]
    assert np.allclose(spec["softmax_ln123"], [1 / 6, 2 / 6, 3 / 6], atol=1e-6)
    idx, val = ref.topk(np.array([5, 1, 7, 7], f32), 2)
    spec["topk_5177_k2"] = [[int(i), float(v)] for i, v in zip(idx, val)]
    assert spec["topk_5177_k2"] == [[2, 7.0], [3, 7.0]]
    spec["build_subset_5177_size2"] = ref.build_subset(np.array([5, 1, 7, 7], np.uint64), 2).tolist()
    assert spec["build_subset_5177_size2"] == [2, 3]
    spec["build_subset_5177_size2_forced1"] = ref.build_subset(np.array([5, 1, 7, 7], np.uint64), 2, [1]).tolist()
    assert sorted(spec["build_subset_5177_size2_forced1"]) == [1, 2]
    spec["tree_mask_chain4"] = [int(w) for w in ref.tree_mask(np.array([-1, 0, 1, 2], np.int32))]
    assert spec["tree_mask_chain4"] == [1, 3, 7, 15]
    spec["argmax_ties"] = ref.argmax(np.array([1, 3, 3, 2], f32))
    assert spec["argmax_ties"] == 1
    # accept-then-bonus: root argmax 7 matches child 0, node 0 argmax 9 matches nothing
    V = 12
    root = np.zeros(V, f32); root[7] = 1
    nodes = np.zeros((2, V), f32); nodes[0, 9] = 1; nodes[1, 3] = 1
    em, path = ref.verify_greedy(root, nodes, np.array([7, 5], np.int32), np.array([-1, -1], np.int32))
    spec["verify_accept_then_bonus"] = dict(emitted=em.tolist(), path=path.tolist())
    assert em.tolist() == [7, 9] and path.tolist() == [0]
    spec["flops_ratio_131072_8192"] = 8192 / 131072
    with open(os.path.join(HERE, "spec_examples.json"), "w") as fh:
        json.dump(spec, fh, indent=1)

    ordered = c1_subset(ref)
    W = ref.model_lm_head(C1["V"], C1["d"], C1["layers"], C1["heads"], C1["seed"])
    digest = hashlib.sha256(W.tobytes()).hexdigest()
    for name, (width, depth, total) in {"c1_capture_w4": (4, 3, 16), "c1_capture_w10": (10, 6, 60)}.items():
        args = (C1["V"], C1["d"], C1["layers"], C1["heads"], 64, C1["seed"], ordered, np.array(C1["pending"], np.int32),
                width, depth, total)
        tree = ref.model_draft_tree(*args)
        cap = ref.model_draft_capture(*args)
        for k in ("tokens", "parents", "depths", "log_joint"):
            assert np.array_equal(tree[k], cap[k]), (name, k)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), hidden=cap["hidden"], row_token=cap["row_token"],
                            row_level=cap["row_level"], tokens=tree["tokens"], parents=tree["parents"],
                            depths=tree["depths"], log_joint=tree["log_joint"], ordered=ordered,
                            lm_head_sha256=np.array(digest), width=width, depth=depth, total=total,
                            config=np.array(json.dumps(C1)))
        print(name, "nodes", tree["tokens"].size, "rows", cap["hidden"].shape)


def sampled():
    """c1_sampled_*.npz: sampled drafting (drafting.cpp:44-74 with std::mt19937_64(rng_seed)):
    the reference's build_draft_tree(rng) tree + the hidden state of every forwarded row from the
    restated capture loop (asserted identical to the reference's tree)."""
    build(reference=True)
    ref = Reference()
    ordered = c1_subset(ref)
    W = ref.model_lm_head(C1["V"], C1["d"], C1["layers"], C1["heads"], C1["seed"])
    digest = hashlib.sha256(W.tobytes()).hexdigest()
    for name, (width, depth, total, rng_seed) in {"c1_sampled_w4_s11": (4, 3, 16, 11),
                                                   "c1_sampled_w10_s5": (10, 6, 60, 5)}.items():
        args = (C1["V"], C1["d"], C1["layers"], C1["heads"], 64, C1["seed"], ordered, np.array(C1["pending"], np.int32),
                width, depth, total, rng_seed)
        tree = ref.model_draft_tree_rng(*args)
        cap = ref.model_draft_capture_rng(*args)
        for k in ("tokens", "parents", "depths", "log_joint"):
            assert np.array_equal(tree[k], cap[k]), (name, k)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), hidden=cap["hidden"], row_token=cap["row_token"],
                            row_level=cap["row_level"], tokens=tree["tokens"], parents=tree["parents"],
                            depths=tree["depths"], log_joint=tree["log_joint"], ordered=ordered,
                            lm_head_sha256=np.array(digest), width=width, depth=depth, total=total,
                            rng_seed=rng_seed, config=np.array(json.dumps(C1)))
        print(name, "nodes", tree["tokens"].size, "rows", cap["hidden"].shape)


if __name__ == "__main__":
    if "--sampled" in sys.argv:
        sampled()
    else:
        main()
