#!/usr/bin/env python3
"""Where the e2e draft level's time goes (diagnostic): frs_head_draft_host through the Python
wrapper as bench.py calls it, the raw ctypes call with preallocated outputs, with graph replay,
and the device chain alone (isolated: host sync between calls). p50 over 400 calls, us."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402
from paper_2502_14856_b200._lib import lib  # noqa: E402


def pct(fn, iters=400):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(float(np.median(ts)) * 1e6, 1)


def main():
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    d, V, v_sub, n, k = 4096, 128256, 32768, 10, 10
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    subset = api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1])
    dh = api.DeviceHead(ctx, W, subset, dtype="bf16")
    head = api.restrict_lm_head(ctx, W, subset, dtype="bf16")
    del W
    hd = torch.randn(n, d, generator=g, device=dev)
    pinned = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    pinned.copy_(hd.cpu())
    h_host = pinned.numpy()
    ridx, full, prob = np.empty((n, k), np.int32), np.empty((n, k), np.int32), np.empty((n, k), np.float32)
    res = {"wrapper": pct(lambda: dh.draft_host(h_host, k, mode="fast")),
           "wrapper_out": pct(lambda: dh.draft_host(h_host, k, mode="fast", out=(ridx, full, prob)))}
    f = lib().frs_head_draft_host
    args = (dh.handle, C.c_void_p(h_host.ctypes.data), n, k, 1, C.c_void_p(ridx.ctypes.data),
            C.c_void_p(full.ctypes.data), C.c_void_p(prob.ctypes.data))
    res["raw_ctypes"] = pct(lambda: f(*args))
    ctx.set_graphs(True)
    res["raw_ctypes_graphs"] = pct(lambda: f(*args))
    ctx.set_graphs(False)
    out = api.draft_head_topk(ctx, hd, head, k, mode="fast")

    def chain():
        api.draft_head_topk(ctx, hd, head, k, mode="fast", out=out)
        torch.cuda.synchronize()
    res["device_chain_isolated"] = pct(chain)
    hdev = torch.empty_like(hd)

    def h2d():
        hdev.copy_(pinned, non_blocking=True)
        torch.cuda.synchronize()
    res["h2d_163KB_sync"] = pct(h2d)
    print(res)


if __name__ == "__main__":
    main()
