#!/usr/bin/env python3
"""Secondary measurements on one B200 (JSON lines to stdout), for SURVEY.md §8(d) rows the
headline bench line does not carry:

  draft   : FAST (and EXACT) draft level at the Llama-3-8B shape, V_sub sweep (C3)
  verify  : FAST verify head (argmax over the full vocabulary) at C2 (61 rows, V=128256,
            d=4096) and the C4 Qwen-2.5-7B shape split into 1/2/4/8 contiguous vocabulary
            shards (per-shard device time = what one GPU of a vocab-parallel group spends)
  sampled : sampled drafting (EXACT arithmetic) — one level and a whole sampled tree
  stochastic: verify_stochastic at C2 (exact target probabilities + the residual walk)
  decode  : head-path decode loop: build_draft_tree (6 levels, width 10,
            60 tokens, hidden state = identity draft layer over an embedding table) +
            verify_greedy over the full head, tokens/s and mean accepted length

Device times are CUDA events over K back-to-back calls; slabs smaller than 4x L2 rotate
over enough copies that each call streams from HBM.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402

L2 = 126 * 2 ** 20
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0


def rms(x):
    return (x * torch.rsqrt(x.double().pow(2).mean(dim=1, keepdim=True) + 1e-5).float()).contiguous()


def timed(fn, iters, warm=5):
    for _ in range(warm):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / iters


def draft_sweep(ctx, dev, modes):
    d, V, n, k = 4096, 128256, 10, 10
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    pool = [rms(torch.randn(n, d, generator=g, device=dev)) for _ in range(64)]
    h_in = torch.empty((n, d), device=dev)
    for v_sub in (8192, 16384, 32768, 65536, 128256):
        sub = api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1])
        slab_bytes = v_sub * d * 2
        copies = max(1, -(-4 * L2 // slab_bytes))
        heads = [api.restrict_lm_head(ctx, W, sub, dtype="bf16") for _ in range(copies)]
        for mode in modes:
            out = api.draft_head_topk(ctx, pool[0], heads[0], k, mode=mode)

            def step(i):
                h_in.copy_(pool[i % len(pool)])
                api.draft_head_topk(ctx, h_in, heads[i % copies], k, mode=mode, out=out)

            us = timed(step, 200 if mode == "fast" else 20)
            alg = slab_bytes + n * d * 4 + n * k * 12
            print(json.dumps({"sweep": "draft", "mode": mode, "v_sub": v_sub, "d": d, "rows": n, "k": k,
                              "slab_copies": copies, "us_per_level": us, "alg_bytes": alg,
                              "GBps": alg / us / 1e3, "frac_of_peak": alg / us / 1e3 / PEAK}), flush=True)
        del heads
        torch.cuda.empty_cache()
    del W


def batched_draft(ctx, dev):
    """C5-style batched drafting: many independent streams' beam rows in one call (one slab
    pass per 64 rows); µs per call and aggregate rows/s at the Llama-3-8B shape."""
    d, V, v_sub, k = 4096, 128256, 32768, 10
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    head = api.restrict_lm_head(ctx, W, api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1]), dtype="bf16")
    del W
    for n in (10, 16, 32, 64, 128, 256, 640, 2560):
        pool = [rms(torch.randn(n, d, generator=g, device=dev)) for _ in range(4)]
        out = api.draft_head_topk(ctx, pool[0], head, k, mode="fast")

        def step(i):
            api.draft_head_topk(ctx, pool[i % 4], head, k, mode="fast", out=out)

        iters = max(5, 2000 // n)
        us = timed(step, iters)
        f = out.flags.cpu().numpy()
        print(json.dumps({"sweep": "batched_draft", "rows": n, "streams_x10": n / 10, "v_sub": v_sub, "d": d,
                          "us_per_call": us, "rows_per_s": n / us * 1e6,
                          "rows_recomputed_last_call": int(((f & 0x8) != 0).sum()),
                          "reasons_last_call": [int(((f & b) != 0).sum()) for b in (0x10, 0x20, 0x40)],
                          "slab_passes": -(-n // 64) if n > 16 else 1}), flush=True)
    del head


def verify_sweep(ctx, dev):
    for name, d, V, m in (("C2 Llama-3-8B", 4096, 128256, 61), ("C4 Qwen-2.5-7B", 3584, 152064, 61)):
        g = torch.Generator(device=dev).manual_seed(7)
        W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        hs = [rms(torch.randn(m, d, generator=g, device=dev)) for _ in range(8)]
        shard_list = (1,) if name.startswith("C2") else (1, 2, 4, 8)
        for G in shard_list:
            per = -(-V // G)
            # shard 0 of G (all shards have the same size up to one row): per-GPU device time
            Ws = W[:per].contiguous()
            copies = max(1, -(-4 * L2 // (per * d * 2)))
            shards = [Ws] + [Ws.clone() for _ in range(copies - 1)]

            def step(i):
                api.verify_head_argmax(ctx, hs[i % len(hs)], shards[i % copies], id_offset=0, mode="fast")

            us = timed(step, 50)
            alg = per * d * 2 + m * d * 4
            print(json.dumps({"sweep": "verify", "shape": name, "shards": G, "rows": m, "d": d, "vocab": V,
                              "shard_rows": per, "us_per_shard": us, "alg_bytes": alg, "GBps": alg / us / 1e3,
                              "frac_of_peak": alg / us / 1e3 / PEAK}), flush=True)
            del shards, Ws
            torch.cuda.empty_cache()
        del W


def decode_loop(ctx, dev, iters):
    d, V, v_sub = 4096, 128256, 32768
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    sub = api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1])
    head = api.DeviceHead(ctx, W, sub, dtype="bf16")
    E = rms(torch.randn(V, d, generator=g, device=dev))  # identity draft layer: hidden = rmsnorm(E[token])
    Wb = W.to(torch.bfloat16)
    del W
    params = api.DraftParams(10, 6, 60)
    stats = api.AcceptanceStats()
    token = 1
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    emitted_total = 0
    t_tree = t_ver = 0.0
    for it in range(iters):
        ta = time.perf_counter()
        tree = head.build_draft_tree(token, params, mode="fast", hidden_table=E)
        tb = time.perf_counter()
        outc = api.verify_greedy_table(ctx, E, token, Wb, tree, mode="fast")  # root + 60 rows gathered on device
        tc = time.perf_counter()
        t_tree += tb - ta
        t_ver += tc - tb
        stats.add(outc.accepted_length())
        emitted_total += outc.accepted_length()
        token = int(outc.emitted[-1])
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print(json.dumps({"sweep": "decode", "config": "head path: draft tree depth 6 width 10, 60 draft tokens, "
                      "verify 61 rows over V=128256 (bf16), identity draft layer", "iterations": iters,
                      "tokens_per_s": emitted_total / el, "ms_per_iteration": 1000 * el / iters,
                      "mean_accepted_length": stats.mean_accepted_length,
                      "ms_draft_tree": 1000 * t_tree / iters, "ms_verify": 1000 * t_ver / iters}), flush=True)


def sampled_draft(ctx, dev, iters=20):
    """Sampled drafting (drafting.cpp:44-74, EXACT arithmetic) at C2: one 10-row level of
    k_exact_logits + k_softmax_sample, and a whole sampled tree (6 levels, width 10, 60 tokens)."""
    d, V, v_sub, n, w = 4096, 128256, 32768, 10, 10
    g = torch.Generator(device=dev).manual_seed(1234)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    ranked = np.random.default_rng(1234).permutation(V).astype(np.int32)
    sub = api.subset_from_ranking(ranked, v_sub, V, forced=[0, 1])
    head = api.restrict_lm_head(ctx, W, sub, dtype="bf16")
    dh = api.DeviceHead(ctx, W, sub, dtype="bf16")
    E = rms(torch.randn(V, d, generator=g, device=dev))
    del W
    h = rms(torch.randn(n, d, generator=g, device=dev))
    rng = api.Rng(2024)
    u = torch.from_numpy(rng.uniforms(n * w).reshape(n, w)).to(dev)
    us = timed(lambda i: api.draft_head_sample(ctx, h, head, w, u), iters)
    out = api.draft_head_sample(ctx, h, head, w, u)
    unc = int(((out.flags.cpu().numpy() & 0x80) != 0).sum())
    dh.build_draft_tree(1, api.DraftParams(10, 6, 60), mode="exact", hidden_table=E, rng=rng)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(5):
        dh.build_draft_tree(2 + i, api.DraftParams(10, 6, 60), mode="exact", hidden_table=E, rng=rng)
    ms = (time.perf_counter() - t0) * 1000 / 5
    print(json.dumps({"sweep": "sampled_draft", "v_sub": v_sub, "d": d, "rows": n, "width": w,
                      "us_per_level_exact_sampled": us, "rows_uncertified_last_level": unc,
                      "ms_per_sampled_tree_6x10_60": ms}), flush=True)


def stochastic_verify(ctx, dev, iters=5):
    """verify_stochastic at C2 (verification.cpp:76-178): 61 target rows over V = 128256 (fp32
    head: the exact path's dtype), a synthetic sampled draft (tree of 60 nodes, q over V_sub)."""
    d, V, v_sub, k = 4096, 128256, 32768, 60
    g = torch.Generator(device=dev).manual_seed(99)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16).float()
    rs = np.random.default_rng(99)
    ordered = rs.permutation(V)[:v_sub].astype(np.int32)
    parents = np.array([-1] * 10 + [i // 10 for i in range(50)], np.int32)
    q_root = rs.dirichlet(np.ones(v_sub)).astype(np.float32)
    q_nodes = rs.dirichlet(np.ones(v_sub), size=k).astype(np.float32)
    has_q = np.zeros(k, np.int32)
    has_q[:10] = 1
    tokens = np.empty(k, np.int32)
    for i in range(k):
        q = q_root if parents[i] < 0 else q_nodes[parents[i]]
        top = np.argsort(-q)[:20]
        tokens[i] = ordered[top[i % 10]]
    h = rms(torch.randn(1 + k, d, generator=g, device=dev))
    tree = api.DraftTree(tokens, parents, np.ones(k, np.int32), np.zeros(k))
    rng = api.Rng(5)
    api.verify_stochastic(ctx, h, W, tree, q_root, q_nodes, has_q, ordered, rng)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lens = []
    for _ in range(iters):
        lens.append(len(api.verify_stochastic(ctx, h, W, tree, q_root, q_nodes, has_q, ordered, rng).accepted_path))
    ms = (time.perf_counter() - t0) * 1000 / iters
    print(json.dumps({"sweep": "verify_stochastic", "rows": 1 + k, "d": d, "vocab": V, "v_sub": v_sub,
                      "head_dtype": "f32", "ms_per_call": ms, "accepted_lengths": lens}), flush=True)


def corpus_count(ctx, dev):
    """count_frequencies on the device (vocab.cpp:23-38): 256M-token Zipf-like corpus at the
    Qwen vocabulary (ids rank-ordered, and permuted)."""
    V, n = 152064, 1 << 28
    g = torch.Generator(device=dev).manual_seed(3)
    u = torch.rand(n, generator=g, device=dev)
    ranks = torch.clamp((torch.exp(u * np.log(V)) - 1).to(torch.int32), 0, V - 1)  # ~ Zipf(1) ranks
    perm = torch.from_numpy(np.random.default_rng(3).permutation(V).astype(np.int32)).to(dev)
    for name, toks in (("rank_ordered_ids", ranks), ("permuted_ids", perm[ranks.long()])):
        api.count_frequencies_device(ctx, toks, V)
        torch.cuda.synchronize()
        us = timed(lambda i: api.count_frequencies_device(ctx, toks, V), 5, warm=1)
        print(json.dumps({"sweep": "count_frequencies", "ids": name, "tokens": n, "vocab": V, "us_per_call": us,
                          "GBps": n * 4 / us / 1e3, "tokens_per_s": n / us * 1e6}), flush=True)


def draft_layer(ctx, dev, iters=10):
    """The draft transformer layer (model.cpp:208-281, EXACT arithmetic) at the Llama-3-8B
    shape (d = 4096, 32 heads, 4d MLP; fp32 weights): one 10-row beam forward on a 512-row
    cache, and the whole model-driven sampled-free drafting step (6 levels x 10 rows + head)."""
    d, heads, V = 4096, 32, 128256
    rs = np.random.default_rng(0)
    g = torch.Generator(device=dev).manual_seed(0)
    wt = lambda r, c: (torch.randn(r, c, generator=g, device=dev) * 0.02).cpu().numpy()  # noqa: E731
    weights = {"embedding": wt(V, d), "wq": wt(d, d), "wk": wt(d, d), "wv": wt(d, d), "wo": wt(d, d),
               "w_up": wt(4 * d, d), "w_down": wt(d, 4 * d)}
    model = api.DraftModel(ctx, weights, heads, 1024)
    ctx_len = 512
    model.forward(rs.integers(0, V, ctx_len), np.arange(ctx_len), np.tril(np.ones((ctx_len, ctx_len), np.uint8)))
    n = 10
    allow = np.zeros((n, ctx_len + n), np.uint8)
    allow[:, :ctx_len] = 1
    allow[np.arange(n), ctx_len + np.arange(n)] = 1
    toks = rs.integers(0, V, n)

    def step(i):
        model.truncate(ctx_len)
        model.forward(toks, np.full(n, ctx_len), allow)

    step(0)  # warm-up: lazy module loading of the kernel variants
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(iters):
        step(i)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1000 / iters
    flops = 2 * n * (4 * d * d + 8 * d * d)
    print(json.dumps({"sweep": "draft_layer", "d": d, "heads": heads, "rows": n, "cache_rows": ctx_len,
                      "ms_per_forward": ms, "weight_bytes": 12 * d * d * 4,
                      "GBps_weights": 12 * d * d * 4 / (ms * 1e-3) / 1e9, "GFLOPs": flops / (ms * 1e-3) / 1e9}),
          flush=True)
    # the whole drafting step (build_draft_tree with the draft model as the hidden-state source):
    # pending forward + 5 beam-level forwards + 6 FR-head levels (V_sub 32768) + bookkeeping
    model.truncate(ctx_len)
    lm = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    sub = api.RankedSubset(V, rs.permutation(V)[:32768].astype(np.int32))
    pending = rs.integers(0, V, 4)
    for mode, dtype in (("fast", "bf16"), ("exact", "f32")):
        head = api.DeviceHead(ctx, lm if dtype == "bf16" else lm.float(), sub, dtype=dtype)
        api.build_draft_tree_model(head, model, pending, api.DraftParams(10, 6, 60), mode=mode)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(iters):
            tree = api.build_draft_tree_model(head, model, pending, api.DraftParams(10, 6, 60), mode=mode)
        torch.cuda.synchronize()
        ms_tree = (time.perf_counter() - t0) * 1000 / iters
        print(json.dumps({"sweep": "model_draft_tree", "mode": mode, "head_dtype": dtype, "d": d, "vocab": V,
                          "v_sub": 32768, "context_rows": ctx_len, "pending": int(pending.size),
                          "width_depth_total": [10, 6, 60], "nodes": len(tree), "ms_per_tree": ms_tree}), flush=True)
        del head


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="draft,batched,verify,decode,sampled,stochastic,count,layer")
    ap.add_argument("--exact", action="store_true", help="also time the EXACT draft level")
    ap.add_argument("--decode-iters", type=int, default=100)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = api.Context(0)
    what = a.what.split(",")
    if "draft" in what:
        draft_sweep(ctx, dev, ["fast", "exact"] if a.exact else ["fast"])
    if "batched" in what:
        batched_draft(ctx, dev)
    if "verify" in what:
        verify_sweep(ctx, dev)
    if "decode" in what:
        decode_loop(ctx, dev, a.decode_iters)
    if "sampled" in what:
        sampled_draft(ctx, dev)
    if "stochastic" in what:
        stochastic_verify(ctx, dev)
    if "count" in what:
        corpus_count(ctx, dev)
    if "layer" in what:
        draft_layer(ctx, dev)


if __name__ == "__main__":
    main()
