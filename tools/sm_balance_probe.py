import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2502_14856_b200 import api, _lib
n, d, v_sub = 10, 4096, 32768
ctx = api.Context(0); dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
W = (torch.randn(v_sub, d, generator=g, device=dev) * 0.02).float()
head = api.restrict_lm_head(ctx, W, api.RankedSubset(v_sub, np.arange(v_sub)), dtype="bf16")
h = torch.randn(n, d, generator=g, device=dev)
out = api.draft_head_topk(ctx, h, head, 10, mode="fast")
G = ctx.sm_count; L = 4 * G
runs = []
ranges = []
for rep in range(12):
    api.draft_head_topk(ctx, h, head, 10, mode="fast", out=out); torch.cuda.synchronize()
    pm, ps, pth = (np.empty(n * L, np.float32) for _ in range(3))
    pkey = np.empty(n * L * 3 + G * 32 + 64 * 8 * 16 + 16 + 64 * 16, np.uint64); pw2 = np.empty(2 * G, np.float32)
    _lib.check(_lib.lib().frs_debug_fast_partials(ctx.handle, n, d, pm.ctypes.data, ps.ctypes.data, pth.ctypes.data, pkey.ctypes.data, pw2.ctypes.data))
    st = pkey[n*L*3:n*L*3+G*32].reshape(G, 32).astype(np.int64)
    t0 = st[:, 0].min()
    dur = (st[:, 2] - st[:, 0]) / 1000.0   # setup -> all TMA issued
    sm = st[:, 17]
    shift = int(os.environ.get("FRS_RANGE_SHIFT", "0"))
    rng_idx = (np.arange(G) + shift) % G     # the row range each CTA streamed
    bysm = np.zeros(G); bysm[sm] = dur
    byrange = np.zeros(G); byrange[rng_idx] = dur
    runs.append(bysm)
    ranges.append(byrange)
R = np.array(runs[2:])
print("per-SM stream us: mean over runs min/med/max", R.mean(0).min(), np.median(R.mean(0)), R.mean(0).max())
print("run-to-run std per SM (median)", np.median(R.std(0)))
c = np.corrcoef(R)
print("corr between runs (mean off-diag)", (c.sum() - len(c)) / (len(c) ** 2 - len(c)))
order = np.argsort(R.mean(0))
print("slowest SMs", order[-10:], R.mean(0)[order[-10:]].round(2))
print("fastest SMs", order[:10], R.mean(0)[order[:10]].round(2))

np.save(os.environ.get("OUT", "/tmp/sm_probe") + ".npy", np.stack([np.array(runs[2:]).mean(0), np.array(ranges[2:]).mean(0)]))
