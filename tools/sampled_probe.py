import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2502_14856_b200 import api
d, V, v_sub, w = 4096, 128256, 32768, 10
dev = torch.device("cuda", 0); ctx = api.Context(0)
g = torch.Generator(device=dev).manual_seed(1234)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
sub = api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1])
head = api.restrict_lm_head(ctx, W, sub, dtype="bf16")
def rms(x): return (x * torch.rsqrt(x.double().pow(2).mean(dim=1, keepdim=True) + 1e-5).float()).contiguous()
E = rms(torch.randn(V, d, generator=g, device=dev))
rng = api.Rng(2024)
for trial in range(3):
    toks = torch.randint(0, V, (10,), device=dev)
    h = E[toks].contiguous()
    u = torch.from_numpy(rng.uniforms(10 * w).reshape(10, w)).to(dev)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = api.draft_head_sample(ctx, h, head, w, u)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("level ms", round((t1 - t0) * 1e3, 3), "count", out.count.cpu().numpy().tolist(), "flags", out.flags.cpu().numpy().tolist())
dh = api.DeviceHead(ctx, W, sub, dtype="bf16")
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dh.build_draft_tree(1 + i, api.DraftParams(10, 6, 60), mode="exact", hidden_table=E, rng=rng)
    print("tree ms", round((time.perf_counter() - t0) * 1e3, 2))
