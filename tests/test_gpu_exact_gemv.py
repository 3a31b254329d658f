"""The staged exact GEMV (k_exact_gemv, csrc/frs_exact.cu) at its edges: K tail chunks (d not a
multiple of the 64 / 128-element chunk), per-CTA row ranges that do not divide into 32-row
warps, fewer W rows than SMs, every register tile (n = 1 .. 61: tiles 2 / 4 / 8 / 16, hidden
groups split unevenly, passes of 32 hidden rows), 16k-wide rows, fp32 and bf16 slabs; matrices
with fewer than 2 x SMs 32-row groups take the row-block kernel (both paths covered). Logits must equal the compiled
reference's dot_f32 matmul (kernels.cpp:13-60) bit for bit."""
import numpy as np
import pytest
import torch

from paper_2502_14856_b200 import api

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n,d,v_sub", [(1, 8, 5), (3, 264, 1000), (16, 1032, 333), (17, 512, 4737), (33, 136, 2049),
                                      (10, 4096, 4096), (5, 520, 149), (32, 72, 3001), (61, 200, 1500),
                                      (7, 16392, 300), (2, 64, 20000),
                                      # >= 2 x SMs 32-row groups: the TMA-boxed register-tile kernel
                                      (10, 264, 40000), (61, 72, 12000), (5, 520, 9500), (32, 4096, 9600)])
def test_exact_logits_match_reference_matmul(cuda_ctx, reference, dtype, n, d, v_sub):
    rng = np.random.default_rng(n * 1000 + d)
    V = v_sub + 7
    W = (rng.standard_normal((V, d)) * 0.05).astype(np.float32)
    if dtype == "bf16":
        W = torch.from_numpy(W).to(torch.bfloat16).float().numpy()  # the values the slab holds
    ids = rng.permutation(V)[:v_sub].astype(np.int32)
    h = rng.standard_normal((n, d)).astype(np.float32)
    head = api.restrict_lm_head(cuda_ctx, torch.from_numpy(W).cuda(), api.RankedSubset(V, ids), dtype=dtype)
    out = api.draft_head_topk(cuda_ctx, torch.from_numpy(h).cuda(), head, min(4, v_sub), mode="exact",
                              want_logits=True)
    got = out.logits.cpu().numpy()
    want = reference.matmul(h, W[ids])
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
