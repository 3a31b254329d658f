#!/usr/bin/env python3
"""Head-path build_draft_tree at C2 (width 10, depth 6, 60 tokens, FAST, identity draft layer):
a few trees, for an ncu launch list of the device-resident bookkeeping."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402

d, V, v_sub = 4096, 128256, 32768
dev = torch.device("cuda", 0)
ctx = api.Context(0)
g = torch.Generator(device=dev).manual_seed(1234)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
head = api.DeviceHead(ctx, W, api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1]), dtype="bf16")
del W
E = torch.randn(V, d, generator=g, device=dev)
E = (E * torch.rsqrt(E.double().pow(2).mean(dim=1, keepdim=True) + 1e-5).float()).contiguous()
params = api.DraftParams(10, 6, 60)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for i in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    head.build_draft_tree(1 + i, params, mode="fast", hidden_table=E)
    print("tree ms", round((time.perf_counter() - t0) * 1e3, 3), flush=True)
