"""Back-to-back FAST batched calls in a given order of (rows:iters:sync) configs (probe).
"""
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2502_14856_b200 import api
d, V, v_sub, k = 4096, 128256, 32768, 10
dev = torch.device("cuda", 0); ctx = api.Context(0)
g = torch.Generator(device=dev).manual_seed(1234)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
head = api.restrict_lm_head(ctx, W, api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1]), dtype="bf16")
del W
def rms(x): return (x * torch.rsqrt(x.double().pow(2).mean(dim=1, keepdim=True) + 1e-5).float()).contiguous()
cfgs = [tuple(int(x) for x in c.split(":")) for c in (sys.argv[1:] or ["32:62:0", "64:31:0", "32:31:0"])]
for n, iters, sync in cfgs:
    pool = [rms(torch.randn(n, d, generator=g, device=dev)) for _ in range(4)]
    out = api.draft_head_topk(ctx, pool[0], head, k, mode="fast")
    for i in range(5): api.draft_head_topk(ctx, pool[i % 4], head, k, mode="fast", out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        api.draft_head_topk(ctx, pool[i % 4], head, k, mode="fast", out=out)
        if sync: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    us = round(e0.elapsed_time(e1) * 1000 / iters, 1)
    fl = []
    for x in pool:
        api.draft_head_topk(ctx, x, head, k, mode="fast", out=out)
        f = out.flags.cpu().numpy()
        fl.append([int(((f & b) != 0).sum()) for b in (0x8, 0x10, 0x20, 0x40)] + [int(((f >> 8) & 0xff).max())])
    print(n, iters, sync, us, "flags per pool input [recomputed, tie, bound, overflow, max|S|]:", fl, flush=True)
