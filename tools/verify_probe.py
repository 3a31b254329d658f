#!/usr/bin/env python3
"""FAST verify head at C2 (61 rows x V=128256, d=4096, bf16): a few calls (ncu launch list) and
back-to-back timing with rotating head copies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_14856_b200 import api  # noqa: E402

d, V, m = 4096, 128256, int(sys.argv[2]) if len(sys.argv) > 2 else 61
dev = torch.device("cuda", 0)
ctx = api.Context(0)
g = torch.Generator(device=dev).manual_seed(7)
Ws = [(torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16) for _ in range(2)]
hs = []
for _ in range(4):
    x = torch.randn(m, d, generator=g, device=dev)
    hs.append((x * torch.rsqrt(x.double().pow(2).mean(dim=1, keepdim=True) + 1e-5).float()).contiguous())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for i in range(5):
    api.verify_head_argmax(ctx, hs[i % 4], Ws[i % 2], id_offset=0, mode="fast")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(n):
    api.verify_head_argmax(ctx, hs[i % 4], Ws[i % 2], id_offset=0, mode="fast")
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1000 / n
print(f"verify rows={m}: {us:.1f} us/call, {(V * d * 2 + m * d * 4) / us / 1e3:.0f} GB/s")
