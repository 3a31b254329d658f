"""Device-resident beam bookkeeping (csrc/frs_tree.cu) for the head-path build_draft_tree
(drafting.cpp:122-245, greedy): gather -> K2 -> k_tree_level per level, k_tree_select at the end,
one D2H. The tree (tokens, parents, depths) and the log_joints (recomputed on the host with
std::log) must equal the restatement's / the host bookkeeping's bit for bit."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rmsnorm(x):
    x = x.astype(np.float32)
    ms = (x.astype(np.float64) ** 2).mean(axis=1, keepdims=True)
    return (x * (1.0 / np.sqrt(ms + 1e-5)).astype(np.float32)).astype(np.float32)


@pytest.mark.parametrize("width,depth,total", [(10, 6, 60), (4, 3, 16), (8, 5, 64), (1, 4, 4), (6, 1, 6)])
@pytest.mark.parametrize("seed", [21, 22])
def test_device_tree_matches_restatement(cuda_ctx, restatement, width, depth, total, seed):
    rng = np.random.default_rng(seed)
    V, d, v_sub = 3000, 128, 900
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="f32")
    root = int(ids[3])
    tree = head.build_draft_tree(root, api.DraftParams(width, depth, total), hidden_table=torch.from_numpy(E).cuda())

    def provider(level, toks, pars):
        return E[[root]] if level == 0 else E[toks]

    ref = restatement.draft_tree(provider, restatement.restrict(W, ids), ids, width, depth, total)
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), ref[key]), key


def test_device_tree_ties(cuda_ctx, restatement):
    """Duplicated head rows: sibling probabilities tie exactly; the index decides on both sides."""
    rng = np.random.default_rng(5)
    V, d, v_sub = 2000, 64, 600
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    W[1::2] = W[0::2]  # pairs of identical rows
    E = rmsnorm(rng.standard_normal((V, d)))
    ids = np.arange(v_sub, dtype=np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="f32")
    tree = head.build_draft_tree(11, api.DraftParams(6, 4, 40), hidden_table=torch.from_numpy(E).cuda())

    def provider(level, toks, pars):
        return E[[11]] if level == 0 else E[toks]

    ref = restatement.draft_tree(provider, restatement.restrict(W, ids), ids, 6, 4, 40)
    for key in ("tokens", "parents", "depths", "log_joint"):
        assert np.array_equal(getattr(tree, key), ref[key]), key


_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2502_14856_b200 import api
rng = np.random.default_rng(8)
V, d, v_sub = 20000, 512, 6000
W = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
E = rng.standard_normal((V, d)).astype(np.float32)
E = (E / np.sqrt((E.astype(np.float64) ** 2).mean(1, keepdims=True) + 1e-5)).astype(np.float32)
ids = rng.permutation(V)[:v_sub].astype(np.int32)
ctx = api.Context(0)
head = api.DeviceHead(ctx, torch.from_numpy(W).to(torch.bfloat16).float().numpy(), api.RankedSubset(V, ids), dtype="bf16")
Ed = torch.from_numpy(E).cuda()
out = []
for root in (5, 77, 1234):
    t = head.build_draft_tree(root, api.DraftParams(10, 6, 60), mode="fast", hidden_table=Ed)
    out.append([t.tokens.tolist(), t.parents.tolist(), t.depths.tolist(), t.log_joint.tolist()])
print(json.dumps(out))
"""


def test_device_tree_equals_host_bookkeeping_fast():
    """FAST mode at a C2-like width/depth: the device bookkeeping and the host bookkeeping
    (FRS_HOST_TREE=1, the pre-existing path) produce identical trees."""
    runs = []
    for env_extra in ({}, {"FRS_HOST_TREE": "1"}):
        env = dict(os.environ, **env_extra)
        r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        runs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert runs[0] == runs[1]


def test_c2_trees_match_restatement(cuda_ctx, restatement):
    """50 drafting trees at the Llama-3-8B shape (d 4096, V 128256, V_sub 32768, bf16 slab,
    width 10 / depth 6 / 60 tokens; hidden rows = rmsnorm'd embedding rows, the identity draft
    layer of the decode loop) equal the restatement's build_draft_tree bit for bit: tokens,
    parents, depths and log_joint. Requested in FAST mode — the tree levels run EXACT by design
    (a tree compares log-probabilities across rows, so every row's 1/Σ must be the reference's;
    DESIGN.md §3) — and in EXACT mode for a few roots."""
    V, d, v_sub = 128256, 4096, 32768
    g = torch.Generator(device="cuda").manual_seed(2502)
    W = (torch.randn(V, d, generator=g, device="cuda") * 0.02).to(torch.bfloat16).float()
    E = torch.randn(V, d, generator=g, device="cuda")
    E = (E * torch.rsqrt(E.double().pow(2).mean(1, keepdim=True) + 1e-5).float()).contiguous()
    ids = np.random.default_rng(2502).permutation(V)[:v_sub].astype(np.int32)
    head = api.DeviceHead(cuda_ctx, W, api.RankedSubset(V, ids), dtype="bf16")
    slab = W[torch.from_numpy(ids).long().cuda()].cpu().numpy()
    del W
    roots = [int(r) for r in np.random.default_rng(7).choice(ids[:4096], 53, replace=False)]
    for t, root in enumerate(roots):
        mode = "exact" if t >= 50 else "fast"
        tree = head.build_draft_tree(root, api.DraftParams(10, 6, 60), mode=mode, hidden_table=E)

        def provider(level, toks, pars, root=root):
            return E[[root] if level == 0 else torch.from_numpy(toks).long().cuda()].cpu().numpy()

        ref = restatement.draft_tree(provider, slab, ids, 10, 6, 60)
        for key in ("tokens", "parents", "depths", "log_joint"):
            assert np.array_equal(getattr(tree, key), ref[key]), (root, mode, key)
