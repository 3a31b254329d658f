#!/usr/bin/env python3
"""Batched drafting probe: a few FAST calls at each row count (run under ncu for a launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402

d, V, v_sub, k = 4096, 128256, 32768, 10
dev = torch.device("cuda", 0)
ctx = api.Context(0)
g = torch.Generator(device=dev).manual_seed(1234)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
head = api.restrict_lm_head(ctx, W, api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1]), dtype="bf16")
del W
rows = [int(x) for x in (sys.argv[1:] or ["32", "64"])]
for n in rows:
    h = torch.randn(n, d, generator=g, device=dev)
    h = (h * torch.rsqrt(h.double().pow(2).mean(dim=1, keepdim=True) + 1e-5).float()).contiguous()
    out = api.draft_head_topk(ctx, h, head, k, mode="fast")
    for _ in range(3):
        api.draft_head_topk(ctx, h, head, k, mode="fast", out=out)
    torch.cuda.synchronize()
    print(n, "flags", np.unique(out.flags.cpu().numpy() & 0xff, return_counts=True))
