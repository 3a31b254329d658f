"""Tree attention (masked_attention kernels.cpp:124-171): bit-exact
with the compiled reference for tree-shaped visibility (context prefix + ancestors, the
reference's tree_layout, model.cpp:302-320) and random masks, head widths with and without
a dot_f32 tail, and its rejection of rows that permit no key."""
import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api
from paper_2502_14856_b200._lib import InvalidArgument

pytestmark = pytest.mark.gpu


def tree_mask(ctx_len, parents):
    k = len(parents)
    allow = np.zeros((k, ctx_len + k), bool)
    for i, p in enumerate(parents):
        allow[i, :ctx_len] = True
        a = i
        while a >= 0:
            allow[i, ctx_len + a] = True
            a = parents[a]
    return allow


@pytest.mark.parametrize("dh,dv,ctx_len,seed", [(64, 64, 200, 1), (128, 128, 517, 2), (100, 72, 63, 3), (8, 16, 1, 4),
                                                 (64, 1000, 300, 7),   # wide values: many 32-column slices
                                                 (32, 48, 7000, 8),    # long key range: chunked value staging
                                                 (130, 33, 90, 9)])    # dh % 8 != 0 (scalar tail), ragged slice
def test_tree_attention_matches_reference(cuda_ctx, reference, dh, dv, ctx_len, seed):
    rng = np.random.default_rng(seed)
    parents = [-1, -1, 0, 0, 1, 2, 2, 5, 6, 6, 9, 3, -1, 12, 13]
    k = len(parents)
    m = ctx_len + k
    q = (rng.standard_normal((k, dh)) * 0.5).astype(np.float32)
    kk = (rng.standard_normal((m, dh)) * 0.5).astype(np.float32)
    v = rng.standard_normal((m, dv)).astype(np.float32)
    allow = tree_mask(ctx_len, parents)
    out = api.masked_attention(cuda_ctx, torch.from_numpy(q).cuda(), torch.from_numpy(kk).cuda(),
                               torch.from_numpy(v).cuda(), allow).cpu().numpy()
    ref = reference.masked_attention(q, kk, v, allow)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("seed", [5, 6])
def test_random_mask_attention_matches_reference(cuda_ctx, reference, seed):
    rng = np.random.default_rng(seed)
    n, m, dh, dv = 33, 300, 96, 40
    q = (rng.standard_normal((n, dh)) * 2.0).astype(np.float32)  # peaked rows too
    kk = rng.standard_normal((m, dh)).astype(np.float32)
    v = rng.standard_normal((m, dv)).astype(np.float32)
    allow = rng.random((n, m)) < 0.3
    allow[np.arange(n), rng.integers(0, m, n)] = True
    out = api.masked_attention(cuda_ctx, torch.from_numpy(q).cuda(), torch.from_numpy(kk).cuda(),
                               torch.from_numpy(v).cuda(), allow).cpu().numpy()
    assert np.array_equal(out, reference.masked_attention(q, kk, v, allow))


def test_attention_row_without_keys_is_rejected(cuda_ctx):
    q = torch.ones((2, 8), device="cuda")
    kv = torch.ones((4, 8), device="cuda")
    allow = np.array([[1, 0, 0, 0], [0, 0, 0, 0]], bool)
    with pytest.raises(InvalidArgument, match="query row 1 permits no keys"):
        api.masked_attention(cuda_ctx, q, kv, kv, allow)
