#!/usr/bin/env python3
"""Per-CTA globaltimer trace of the FAST main kernel (FRS_TRACE=1 must be set before the
library allocates its workspace). Prints, per stamp slot, min/median/max microseconds
relative to the earliest slot-0 stamp across CTAs.

  FRS_TRACE=1 python tools/fast_trace.py [--v-sub 32768] [--rows 10]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api, _lib  # noqa: E402

SLOTS = {28: "main entry", 0: "setup done", 1: "producer: before griddep_wait", 9: "producer: after griddep_wait",
         3: "mma: first stage full", 2: "producer: all TMA issued", 4: "mma: all issued", 8: "norm warps done",
         10: "epi: first tfull wait", 11: "epi: first tile ready", 14: "epi w4: last tile ready",
         13: "epi: loop done", 15: "epi w4: softmax merged", 16: "epi w4: after bar2", 5: "cand published",
         17: "epi w4: after bar1", 18: "epi w4: rows done", 19: "cta: final sync", 7: "cta end",
         20: "loop done w0", 21: "loop done w1", 22: "loop done w2", 23: "loop done w3", 24: "loop done w4",
         25: "loop done w5", 26: "loop done w6", 27: "loop done w7"}
SSLOTS = {0: "sel start", 2: "sel after griddep_wait", 3: "sel pass1 (max)", 4: "sel pass2 (sum, survivors)",
          6: "sel S chosen", 12: "sel round 0 gathered", 10: "sel round 0 dot done (tid 0)",
          11: "sel round 1 gathered", 1: "sel round 1 dot done", 5: "sel recompute done", 13: "certify: entry",
          14: "certify: e-keys", 15: "certify: sorted", 9: "certify: checks passed", 7: "sel certified+written"}
FSLOTS = {0: "fin start", 1: "fin h loaded", 2: "fin after griddep_wait", 3: "fin partials merged",
          4: "fin S selected", 5: "fin recompute done", 6: "fin last: certified?", 7: "fin last: written",
          6: "fin keys+M+eps ready", 11: "fin histogram issued", 10: "fin leader: after cluster wait",
          12: "fin cand rows staged", 13: "certify: entry", 14: "certify: e-keys", 15: "certify: sorted",
          9: "certify: checks passed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--v-sub", type=int, default=32768)
    ap.add_argument("--rows", type=int, default=10)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--verify", action="store_true", help="trace the argmax (verify) chain over a [v_sub x d] shard")
    a = ap.parse_args()
    assert os.environ.get("FRS_TRACE"), "set FRS_TRACE=1"
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    g = torch.Generator(device=dev).manual_seed(1)
    W = (torch.randn(a.v_sub, a.d, generator=g, device=dev) * 0.02).float()
    head = api.restrict_lm_head(ctx, W, api.RankedSubset(a.v_sub, np.arange(a.v_sub)), dtype="bf16")
    h = torch.randn(a.rows, a.d, generator=g, device=dev)
    if a.verify:  # the verify head over a shard: W itself (bf16 values), argmax per row
        Wb = head.slab
        call = lambda: api.verify_head_argmax(ctx, h, Wb, mode="fast")  # noqa: E731
    else:
        call = None
    out = api.draft_head_topk(ctx, h, head, 10, mode="fast") if not a.verify else None
    G = ctx.sm_count
    res = []
    for _ in range(a.reps):
        if call:
            call()
        else:
            api.draft_head_topk(ctx, h, head, 10, mode="fast", out=out)
        torch.cuda.synchronize()
        n = a.rows
        L = 4 * G
        pm, ps, pth = (np.empty(n * L, np.float32) for _ in range(3))
        pkey = np.empty(n * L * 3 + G * 32 + 64 * 8 * 16 + 16 + 64 * 16, np.uint64)
        pw2 = np.empty(2 * G, np.float32)
        _lib.check(_lib.lib().frs_debug_fast_partials(ctx.handle, n, a.d, pm.ctypes.data, ps.ctypes.data,
                                                      pth.ctypes.data, pkey.ctypes.data, pw2.ctypes.data))
        st = pkey[n * L * 3:n * L * 3 + G * 32].reshape(G, 32).astype(np.int64)
        ft = pkey[n * L * 3 + G * 32:n * L * 3 + G * 32 + 64 * 8 * 16].reshape(64 * 8, 16).astype(np.int64)[: n * 8]
        xt = pkey[n * L * 3 + G * 32 + 64 * 8 * 16:n * L * 3 + G * 32 + 64 * 8 * 16 + 16].astype(np.int64)

        t0 = st[:, 0][st[:, 0] > 0].min()  # earliest "setup done" of the main kernel
        row = {}
        cp = pkey[n * L * 3 + G * 32 + 64 * 8 * 16 + 16:].reshape(64, 16).astype(np.int64)[:n]
        for q, name in list(enumerate(["mx (redux)", "e-keys", "sorted", "tie", "bound", "inv", "written"])) + [
                (9, "fin: keys filtered"), (10, "fin: partials merged"), (11, "fin: S selected"),
                (12, "fin: cand rows staged"), (13, "fin: recompute done"), (14, "fin leader: cluster wait done")]:
            v = cp[:, q]
            v = v[v > 0]
            if v.size:
                row[f"C{q} cycles: {name}"] = [int(v.min()), int(np.median(v)), int(v.max())]
        for s_, name in ((6, "publish: softmax done"), (12, "publish: bmax done"), (31, "publish: tournament done"),
                         (29, "publish cycles w0 (half 0)"), (30, "publish cycles w4 (half 1)")):
            v = st[:, s_]
            v = v[v > 0]
            if v.size:
                row[f"M{s_} {name}"] = [int(v.min()), int(np.median(v)), int(v.max())]
        for s, name in SLOTS.items():
            v = st[:, s]
            v = v[v > 0]
            if v.size:
                us = (v - t0) / 1000.0
                row[f"{s:02d} {name}"] = [round(float(us.min()), 2), round(float(np.median(us)), 2),
                                          round(float(us.max()), 2)]
        for s, name in (SSLOTS if n > 16 and not a.verify else FSLOTS).items():
            v = ft[::8, s] if n > 16 and not a.verify else ft[:, s]
            v = v[v > 0]
            if v.size:
                us = (v - t0) / 1000.0
                row[f"F{s} {name}"] = [round(float(us.min()), 2), round(float(np.median(us)), 2),
                                       round(float(us.max()), 2)]
        for s_, name in {0: "hsplit start", 1: "hsplit cta0 end", 2: "fallback start", 3: "fallback exit (empty)",
                        4: "fallback dots done (last CTA)", 5: "fallback end", 8: "fb row0: max pass",
                        9: "fb row0: exp+sum pass", 10: "fb row0: total (seq?)", 11: "fb row0: key lists",
                        12: "fb row0: top-k done"}.items():
            if xt[s_] > 0:
                row[f"X{s_} {name}"] = round(float((xt[s_] - t0) / 1000.0), 2)
        if n > 16 and not a.verify:  # batched path: k_fast_select stamps (row i at [i*8]); slot 8 = |S| | robust << 32
            sel8 = ft[::8, 8][:n]
            row["select |S| (min/med/max)"] = [int((sel8 & 0xffffffff).min()), int(np.median(sel8 & 0xffffffff)),
                                               int((sel8 & 0xffffffff).max())]
            row["select robust rows"] = int(((sel8 >> 32) & 1).sum())
            dc = ft[1::8, 15][:n]
            row["select round-0 dot cycles (min/med/max)"] = [int(dc.min()), int(np.median(dc)), int(dc.max())]
        # clock64 vs globaltimer over the exact-recompute phase (slots 12 -> 5; cycles in 13/14)
        sel = (ft[:, 12] > 0) & (ft[:, 5] > ft[:, 12])
        if sel.any():
            ns_ = (ft[sel, 5] - ft[sel, 12]).astype(np.float64)
            cyc = (ft[sel, 14] - ft[sel, 13]).astype(np.float64)
            row["recompute cycles/ns (SM GHz)"] = [round(float(np.median(cyc / ns_)), 3), round(float(np.median(cyc)), 0),
                                                   round(float(np.median(ns_)), 0)]
        res.append(row)
    for k in res[-1]:
        print(k.ljust(40), res[-1][k])
    print(json.dumps(res[-1]))


if __name__ == "__main__":
    main()
