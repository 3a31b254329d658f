import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2502_14856_b200 import api
dev = torch.device("cuda", 0); ctx = api.Context(0)
d, V, v_sub = 4096, 128256, 32768
g = torch.Generator(device=dev).manual_seed(1)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
head = api.restrict_lm_head(ctx, W, api.RankedSubset(V, np.arange(v_sub)), dtype="bf16")
del W
h = torch.randn(64, d, generator=g, device=dev)
out = api.draft_head_topk(ctx, h, head, 10, mode="fast")
for _ in range(20):
    api.draft_head_topk(ctx, h, head, 10, mode="fast", out=out)
torch.cuda.synchronize()
