"""CPU (gloo, world_size 2) coverage of the vocab-parallel verify plumbing:
contiguous shard ranges, the all-gather of per-shard (value, id) argmax pairs, and the merge
by (value desc, id asc) — checked against the oracle's full-vocabulary argmax, including
ties that straddle the shard boundary. The per-shard argmax here is the oracle's (test-only);
on GPUs the same plumbing runs K3 + ncclAllGather + K5 inside the library
(frs_verify_head_argmax_vp via api.verify_head_argmax_vocab_parallel,
tests/test_gpu_fast.py::test_vocab_parallel_nccl_world1 / ::test_vocab_parallel_emulated)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Restatement
        from paper_2502_14856_b200 import api
        R = Restatement()
        rng = np.random.default_rng(11)
        V, d, m = 1001, 64, 9
        W = (rng.standard_normal((V, d)) * 0.02).astype(np.float32)
        h = rng.standard_normal((m, d)).astype(np.float32)
        # ties across the boundary: row 0's winner duplicated in the other shard
        best0 = int(R.verify_argmax(h, W)[0][0])
        s1, c1 = api.vocab_shard(V, world, 1)
        dup = s1 + 3 if best0 < s1 else 2
        W[dup] = W[best0]
        start, count = api.vocab_shard(V, world, rank)
        ids, vals = R.verify_argmax(h, W[start:start + count])
        ids = ids.astype(np.int32) + start
        gv = [torch.empty(m, dtype=torch.float32) for _ in range(world)]
        gi = [torch.empty(m, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gv, torch.from_numpy(vals.astype(np.float32)))
        dist.all_gather(gi, torch.from_numpy(ids))
        mv, mi = api.argmax_merge_host(torch.stack(gv).numpy(), torch.stack(gi).numpy())
        full_ids, full_vals = R.verify_argmax(h, W)
        ok = bool(np.array_equal(mi, full_ids) and np.array_equal(mv, full_vals))
        result[rank] = int(ok)
    finally:
        dist.destroy_process_group()


def test_vocab_shard_ranges_cover_vocab():
    from paper_2502_14856_b200 import api
    for V in (1, 7, 128256, 152064):
        for world in (1, 2, 3, 4, 8):
            if V < world:
                continue
            spans = [api.vocab_shard(V, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert spans[-1][0] + spans[-1][1] == V
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_argmax_merge_host_rules():
    from paper_2502_14856_b200 import api
    vals = np.array([[1.0, 2.0, -0.0, np.nan], [1.0, 3.0, 0.0, 1.0]], np.float32)
    ids = np.array([[5, 7, 9, 2], [40, 41, 42, 43]], np.int32)
    v, i = api.argmax_merge_host(vals, ids)
    assert i.tolist() == [5, 41, 9, 43]  # tie -> lowest id; -0 == +0 -> lowest id; NaN loses


def test_vocab_parallel_gloo_world2():
    world = 2
    result = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), result), nprocs=world, join=True)
    assert dict(result) == {0: 1, 1: 1}
