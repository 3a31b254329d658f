"""Python mirror of the reference's hot-path API over libfrspec_cuda.so.

Names, argument meaning and errors follow /root/reference/proj:
  FrequencyTable / count_frequencies / build_subset / subset_from_ranking / coverage /
  flops_ratio / RankedSubset / RestrictedHead / restrict_lm_head   (vocab.h:14-77)
  DraftParams / DraftTree / build_draft_tree (head path)           (drafting.h:13-67)
  TreeMask / build_tree_mask / VerifyOutcome / verify_greedy /
  AcceptanceStats                                                  (verification.h:16-62)
plus the device-level kernels draft_head_topk / verify_head_argmax / accept_greedy /
argmax_merge (include/frspec_cuda.h). Device buffers are torch CUDA tensors (PyTorch is
plumbing here: memory, streams); every computation runs in the CUDA library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import (DTYPE_BF16, DTYPE_F32, MODE_EXACT, MODE_FAST, CapacityError, InvalidArgument, NotSupported, check,
                   lib)

_DTYPES = {"f32": DTYPE_F32, "fp32": DTYPE_F32, "float32": DTYPE_F32, "bf16": DTYPE_BF16, "bfloat16": DTYPE_BF16}
_MODES = {"exact": MODE_EXACT, "fast": MODE_FAST}


def _dtype(d) -> int:
    if isinstance(d, int):
        return d
    return _DTYPES[str(d).replace("torch.", "")]


def _mode(m) -> int:
    return m if isinstance(m, int) else _MODES[m]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _stream(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Context:
    """frs_ctx: one per device per host thread (SURVEY.md §8(b) threading)."""

    def __init__(self, device: int = 0):
        self.device = device
        p = C.c_void_p()
        check(lib().frs_ctx_create(device, C.byref(p)), "frs_ctx_create")
        self.handle = p

    @property
    def sm_count(self) -> int:
        return lib().frs_ctx_sm_count(self.handle)

    def reserve(self, max_rows: int, max_vocab: int, d: int) -> None:
        check(lib().frs_ctx_reserve(self.handle, max_rows, max_vocab, d), "frs_ctx_reserve")

    def set_timing(self, enable: bool) -> None:
        """Record CUDA events around each call's dominant kernel (on its launch stream)."""
        check(lib().frs_ctx_set_timing(self.handle, int(enable)), "set_timing")

    def timing_read(self):
        """-> (summed milliseconds, number of timed calls); resets the record."""
        ms, cnt = C.c_double(), C.c_int()
        check(lib().frs_ctx_timing_read(self.handle, C.byref(ms), C.byref(cnt)), "timing_read")
        return ms.value, cnt.value

    def set_graphs(self, enable: bool) -> None:
        """Replay repeated FAST calls as one captured CUDA graph (latency-bound callers)."""
        check(lib().frs_ctx_set_graphs(self.handle, 1 if enable else 0), "set_graphs")

    @property
    def launch_count(self) -> int:
        v = C.c_uint64()
        check(lib().frs_ctx_launch_count(self.handle, C.byref(v)), "launch_count")
        return int(v.value)

    def close(self) -> None:
        if self.handle:
            lib().frs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- vocab (vocab.h:14-77)
@dataclass
class FrequencyTable:
    vocab_size: int
    counts: np.ndarray
    total: int

    def merge(self, other: "FrequencyTable") -> None:  # vocab.cpp:15-21
        if other.vocab_size != self.vocab_size:
            raise InvalidArgument("FrequencyTable::merge: vocab_size mismatch")
        self.counts = self.counts + other.counts
        self.total += other.total


def count_frequencies(stream, vocab_size: int) -> FrequencyTable:
    s = _i32(stream)
    counts = np.zeros(max(vocab_size, 1), np.uint64)
    check(lib().frs_count_frequencies(_np_ptr(s), s.size, vocab_size, _np_ptr(counts)), "count_frequencies")
    return FrequencyTable(vocab_size, counts, int(s.size))


def count_frequencies_device(ctx: "Context", tokens: torch.Tensor, vocab_size: int) -> FrequencyTable:
    """count_frequencies (vocab.cpp:23-38) on the device (int32 CUDA token tensor)."""
    t = tokens.to(torch.int32).contiguous()
    counts = torch.empty(max(vocab_size, 1), dtype=torch.int64, device=t.device)
    check(lib().frs_count_frequencies_device(ctx.handle, _ptr(t), t.numel(), vocab_size, _ptr(counts),
                                             _stream(None)), "count_frequencies")
    return FrequencyTable(vocab_size, counts.cpu().numpy().view(np.uint64), int(t.numel()))


def masked_attention(ctx: "Context", q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, allow) -> torch.Tensor:
    """kernels.cpp:124-171 (the tree attention): allow [n, m] bool/0-1 (numpy or tensor), packed
    here into the reference's BitMask words. Raises InvalidArgument like the reference when a
    query row permits no key."""
    q, k, v = (t.to(torch.float32).contiguous() for t in (q, k, v))
    n, dh = q.shape
    m, dv = v.shape
    if tuple(k.shape) != (m, dh):  # kernels.cpp:124-130
        raise InvalidArgument("masked_attention: q/k width mismatch" if k.shape[1] != dh
                              else "masked_attention: k/v row mismatch")
    a = np.asarray(allow.cpu() if isinstance(allow, torch.Tensor) else allow).astype(bool).reshape(n, m)
    stride = (m + 63) // 64
    bits = np.zeros((n, stride * 64), np.uint8)
    bits[:, :m] = a
    words = np.packbits(bits.reshape(n, stride, 64)[:, :, ::-1], axis=2, bitorder="big").reshape(n, stride, 8)
    words = words[:, :, ::-1].copy().view(np.uint64).reshape(n, stride)  # little-endian u64, bit j = key j
    wd = torch.from_numpy(words.view(np.int64)).to(q.device)
    out = torch.empty((n, dv), dtype=torch.float32, device=q.device)
    flags = torch.empty(n, dtype=torch.int32, device=q.device)
    check(lib().frs_masked_attention(ctx.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(wd), n, m, dh, dv, _ptr(out),
                                     _ptr(flags), _stream(None)), "masked_attention")
    bad = np.nonzero(flags.cpu().numpy() & _lib.FLAG_EMPTY_ROW)[0]
    if bad.size:
        raise InvalidArgument(f"masked_attention: query row {int(bad[0])} permits no keys")
    return out


def _mask_words(allow) -> np.ndarray:
    """[n, m] bool -> the reference's BitMask words [n, ceil(m / 64)] (bit j = column j)."""
    a = np.asarray(allow).astype(bool)
    n, m = a.shape
    stride = (m + 63) // 64
    bits = np.zeros((n, stride * 64), np.uint8)
    bits[:, :m] = a
    w = np.packbits(bits.reshape(n, stride, 64)[:, :, ::-1], axis=2, bitorder="big").reshape(n, stride, 8)
    return np.ascontiguousarray(w[:, :, ::-1]).view(np.uint64).reshape(n, stride)


class DraftModel:
    """The draft model's transformer layer on the device (model.cpp:208-281, forward_raw of a
    1-layer draft) with its KV cache; bit-exact with the reference. weights: host fp32 arrays
    embedding [V, d], wq / wk / wv / wo [d, d], w_up [4d, d], w_down [d, 4d] (x W^T), optional
    attn_norm / mlp_norm / final_norm gains [d]."""

    def __init__(self, ctx: "Context", weights: dict, heads: int, max_seq: int):
        self.ctx = ctx
        self._w = {k: np.ascontiguousarray(v, np.float32) for k, v in weights.items()}
        V, d = self._w["embedding"].shape
        self.V, self.d, self.heads, self.max_seq = V, d, heads, max_seq
        g = lambda k: _np_ptr(self._w[k]) if k in self._w else None  # noqa: E731
        h = C.c_void_p()
        check(lib().frs_draft_model_create(ctx.handle, V, d, heads, max_seq, g("embedding"), g("wq"), g("wk"), g("wv"),
                                           g("wo"), g("w_up"), g("w_down"), g("attn_norm"), g("mlp_norm"),
                                           g("final_norm"), C.byref(h)), "draft_model")
        self.handle = h

    def __len__(self) -> int:
        n = C.c_int()
        check(lib().frs_draft_model_length(self.handle, C.byref(n)), "draft_model")
        return n.value

    def truncate(self, new_len: int) -> None:
        check(lib().frs_draft_model_truncate(self.handle, new_len), "truncate")

    def position(self, row: int) -> int:
        """KVCache::positions[row]: the position a cached row was forwarded at."""
        p = C.c_int()
        check(lib().frs_draft_model_position(self.handle, row, C.byref(p)), "position")
        return p.value

    def compact(self, keep_from: int, kept_offsets) -> None:
        """KVCache::compact (model.cpp:165-196): keep rows keep_from + kept_offsets[i] at
        keep_from + i (K, V and positions); ValueError / RuntimeError (logic_error) as the
        reference."""
        o = _i32(kept_offsets)
        check(lib().frs_draft_model_compact(self.handle, keep_from, _np_ptr(o) if o.size else None, o.size,
                                            _stream(None)), "compact")

    def forward(self, tokens, positions, allow) -> torch.Tensor:
        """forward_raw: allow [n, len + n] (cache rows visible to each token)."""
        t, p = _i32(tokens), _i32(positions)
        n = t.size
        allow = np.asarray(allow)
        if p.size != n:  # model.cpp:216-225
            raise InvalidArgument("forward: positions size mismatch")
        if allow.ndim != 2 or allow.shape != (n, len(self) + n):
            raise InvalidArgument("forward: visibility mask shape mismatch")
        words = _mask_words(allow)
        out = torch.empty((t.size, self.d), dtype=torch.float32, device=torch.device("cuda", self.ctx.device))
        check(lib().frs_draft_model_forward(self.handle, _np_ptr(t), _np_ptr(p), t.size, _np_ptr(words), _ptr(out),
                                            _stream(None)), "forward")
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib._LIB is not None:
                lib().frs_draft_model_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def write_token_stream(path: str, vocab_size: int, tokens) -> None:
    """vocab.cpp:236-245: binary FRTK v1 token stream."""
    t = _i32(tokens)
    check(lib().frs_write_token_stream(path.encode(), vocab_size, _np_ptr(t), t.size), "write_token_stream")


def read_token_stream(path: str):
    """vocab.cpp:247-272 -> (vocab_size, tokens)."""
    v, n = C.c_int(), C.c_int64()
    check(lib().frs_read_token_stream(path.encode(), None, 0, C.byref(v), C.byref(n)), "read_token_stream")
    out = np.empty(n.value, np.int32)
    check(lib().frs_read_token_stream(path.encode(), _np_ptr(out), out.size, C.byref(v), C.byref(n)),
          "read_token_stream")
    return v.value, out


def read_token_stream_text(path: str, vocab_size: int) -> np.ndarray:
    """vocab.cpp:274-286: whitespace-separated ids."""
    n = C.c_int64()
    check(lib().frs_read_token_stream_text(path.encode(), vocab_size, None, 0, C.byref(n)), "read_token_stream_text")
    out = np.empty(n.value, np.int32)
    check(lib().frs_read_token_stream_text(path.encode(), vocab_size, _np_ptr(out), out.size, C.byref(n)),
          "read_token_stream_text")
    return out


def write_ranked_file(path: str, ordered_ids) -> None:
    """vocab.cpp:288-293: one id per line."""
    t = _i32(ordered_ids)
    check(lib().frs_write_ranked_file(path.encode(), _np_ptr(t), t.size), "write_ranked_file")


def read_ranked_file(path: str) -> np.ndarray:
    """vocab.cpp:295-306."""
    n = C.c_int64()
    check(lib().frs_read_ranked_file(path.encode(), None, 0, C.byref(n)), "read_ranked_file")
    out = np.empty(n.value, np.int32)
    check(lib().frs_read_ranked_file(path.encode(), _np_ptr(out), out.size, C.byref(n)), "read_ranked_file")
    return out


@dataclass
class RankedSubset:
    vocab_size: int
    ordered_ids: np.ndarray
    full_to_restricted: np.ndarray = field(default=None)

    def __post_init__(self):
        self.ordered_ids = _i32(self.ordered_ids)
        if self.full_to_restricted is None:
            f2r = np.full(self.vocab_size, -1, np.int32)
            f2r[self.ordered_ids] = np.arange(self.ordered_ids.size, dtype=np.int32)
            self.full_to_restricted = f2r

    def size(self) -> int:
        return int(self.ordered_ids.size)

    def full_id(self, restricted: int) -> int:
        return int(self.ordered_ids[restricted])

    def restricted_index(self, full: int) -> int:
        return int(self.full_to_restricted[full])

    def contains(self, full: int) -> bool:
        return self.full_to_restricted[full] >= 0


def build_subset(table: FrequencyTable, size: int, forced: Sequence[int] = ()) -> RankedSubset:
    f = _i32(list(forced))
    out = np.empty(max(size, 1), np.int32)
    check(lib().frs_build_subset(_np_ptr(np.ascontiguousarray(table.counts, np.uint64)), table.vocab_size, size,
                                 _np_ptr(f), f.size, _np_ptr(out)), "build_subset")
    return RankedSubset(table.vocab_size, out[:size])


def subset_from_ranking(ranked_desc, size: int, vocab_size: int, forced: Sequence[int] = ()) -> RankedSubset:
    r, f = _i32(ranked_desc), _i32(list(forced))
    out = np.empty(max(size, 1), np.int32)
    check(lib().frs_subset_from_ranking(_np_ptr(r), r.size, size, vocab_size, _np_ptr(f), f.size, _np_ptr(out)),
          "subset_from_ranking")
    return RankedSubset(vocab_size, out[:size])


def coverage(table: FrequencyTable, subset: RankedSubset) -> float:
    if subset.vocab_size != table.vocab_size:
        raise InvalidArgument("coverage: subset does not match the table vocabulary")
    out = C.c_double()
    check(lib().frs_coverage(_np_ptr(np.ascontiguousarray(table.counts, np.uint64)), table.vocab_size,
                             _np_ptr(subset.ordered_ids), subset.size(), C.byref(out)), "coverage")
    return out.value


def flops_ratio(full_size: int, restricted_size: int) -> float:
    out = C.c_double()
    check(lib().frs_flops_ratio(full_size, restricted_size, C.byref(out)), "flops_ratio")
    return out.value


# ---------------------------------------------------------------- K1: restrict_lm_head
@dataclass
class RestrictedHead:
    """Device-resident row-gathered LM head slice (vocab.h:49-52). ``slab`` is row-major
    [V_sub x d] in ``dtype``; ``ordered_dev`` is the restricted->full id map on the device;
    ``tiled`` (bf16 slabs) the FAST head's stream-order image of the slab (frs_slab_tile), which
    FAST draft levels stream instead of the row-major slab."""
    slab: torch.Tensor
    ordered_dev: torch.Tensor
    subset: RankedSubset
    dtype: int
    tiled: Optional[torch.Tensor] = None

    @property
    def v_sub(self) -> int:
        return int(self.slab.shape[0])

    @property
    def d(self) -> int:
        return int(self.slab.shape[1])


def restrict_lm_head(ctx: Context, lm_head: torch.Tensor, subset: RankedSubset, dtype="bf16",
                     stream=None, tile: bool = True) -> RestrictedHead:
    """K1 (vocab.cpp:152-168): the FR slab, plus (bf16, tile=True) its FAST stream-order image."""
    if lm_head.dtype != torch.float32 or not lm_head.is_cuda or lm_head.dim() != 2:
        raise InvalidArgument("restrict_lm_head: lm_head must be a CUDA float32 [V x d] tensor")
    lm_head = lm_head.contiguous()
    dt = _dtype(dtype)
    V, d = lm_head.shape
    ordered_dev = torch.from_numpy(subset.ordered_ids).to(lm_head.device)
    slab = torch.empty((subset.size(), d), dtype=torch.bfloat16 if dt == DTYPE_BF16 else torch.float32,
                       device=lm_head.device)
    check(lib().frs_slab_build(ctx.handle, _ptr(lm_head), V, d, _ptr(ordered_dev), subset.size(), dt, _ptr(slab),
                               _stream(stream)), "restrict_lm_head")
    tiled = None
    if dt == DTYPE_BF16 and d % 8 == 0 and tile:
        tiled = torch.empty(int(lib().frs_slab_tile_bytes(subset.size(), d)), dtype=torch.uint8, device=lm_head.device)
        check(lib().frs_slab_tile(ctx.handle, _ptr(slab), subset.size(), d, _ptr(tiled), _stream(stream)),
              "restrict_lm_head")
    return RestrictedHead(slab, ordered_dev, subset, dt, tiled)


# ---------------------------------------------------------------- K2: draft head + top-k
@dataclass
class DraftLevel:
    ridx: torch.Tensor     # [n, k] int32 restricted index
    full: torch.Tensor     # [n, k] int32 full-vocabulary id
    prob: torch.Tensor     # [n, k] float32
    rowmax: torch.Tensor   # [n] float32
    total: torch.Tensor    # [n] float64
    flags: torch.Tensor    # [n] int32 (FRS_FLAG_*)
    logits: Optional[torch.Tensor] = None


def draft_head_topk(ctx: Context, h: torch.Tensor, head: RestrictedHead, k: int, temperature: float = 1.0,
                    mode="exact", want_logits: bool = False, stream=None, out: Optional[DraftLevel] = None,
                    want_total: bool = True) -> DraftLevel:
    """want_total=False: Σ is not returned (out.total None); EXACT mode then pins 1 / Σ by
    bracketing and splits each row over a CTA cluster (the tree levels' path)."""
    if h.dtype != torch.float32 or not h.is_cuda:
        raise InvalidArgument("draft head: h must be a CUDA float32 tensor")
    h = h.contiguous()
    if h.dim() != 2 or h.shape[1] != head.d:  # kernels.cpp:35-37 matmul: inner dimensions differ
        raise InvalidArgument(f"matmul: inner dimensions differ ({tuple(h.shape)} vs head width {head.d})")
    if k < 1:  # drafting.cpp:15; k > V_sub draws min(width, V_sub) (drafting.cpp:37-43)
        raise InvalidArgument("draft params: beam_width must be >= 1")
    n, d = h.shape
    dev = h.device
    if out is None:
        out = DraftLevel(torch.empty((n, k), dtype=torch.int32, device=dev), torch.empty((n, k), dtype=torch.int32, device=dev),
                         torch.empty((n, k), dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.float32, device=dev),
                         torch.empty(n, dtype=torch.float64, device=dev) if want_total else None,
                         torch.zeros(n, dtype=torch.int32, device=dev),
                         torch.empty((n, head.v_sub), dtype=torch.float32, device=dev) if want_logits else None)
    if _mode(mode) == MODE_FAST and head.tiled is not None and out.logits is None:
        check(lib().frs_draft_head_topk_tiled(ctx.handle, _ptr(h), n, d, _ptr(head.slab), _ptr(head.tiled), head.v_sub,
                                              _ptr(head.ordered_dev), k, temperature, _ptr(out.ridx), _ptr(out.full),
                                              _ptr(out.prob), _ptr(out.rowmax), _ptr(out.total), _ptr(out.flags),
                                              _stream(stream)), "draft_head_topk")
        return out
    check(lib().frs_draft_head_topk(ctx.handle, _ptr(h), n, d, _ptr(head.slab), head.v_sub, head.dtype,
                                    _ptr(head.ordered_dev), k, temperature, _mode(mode), _ptr(out.ridx), _ptr(out.full),
                                    _ptr(out.prob), _ptr(out.rowmax), _ptr(out.total), _ptr(out.logits),
                                    _ptr(out.flags), _stream(stream)), "draft_head_topk")
    return out


# ---------------------------------------------------------------- K3/K4/K5
def tile_image(ctx: Context, W: torch.Tensor, stream=None) -> torch.Tensor:
    """The FAST heads' stream-order image of a CUDA bf16 [rows x d] matrix (frs_slab_tile)."""
    if W.dtype != torch.bfloat16 or not W.is_cuda or W.dim() != 2 or not W.is_contiguous():
        raise InvalidArgument("slab tile: W must be a contiguous CUDA bf16 [rows x d] tensor")
    img = torch.empty(int(lib().frs_slab_tile_bytes(W.shape[0], W.shape[1])), dtype=torch.uint8, device=W.device)
    check(lib().frs_slab_tile(ctx.handle, _ptr(W), W.shape[0], W.shape[1], _ptr(img), _stream(stream)), "slab_tile")
    return img


def verify_head_argmax(ctx: Context, h: torch.Tensor, W: torch.Tensor, id_offset: int = 0, mode="exact",
                       stream=None, W_tiled: Optional[torch.Tensor] = None):
    """Per-row argmax of h . W^T with ties to the lowest id; W is a CUDA fp32/bf16 shard. FAST mode
    with W_tiled (tile_image(ctx, W)) streams the shard's tiled image."""
    h = h.contiguous()
    m, d = h.shape
    if W.dim() != 2 or W.shape[1] != d:
        raise InvalidArgument(f"matmul: inner dimensions differ ({tuple(h.shape)} vs {tuple(W.shape)})")
    dt = DTYPE_BF16 if W.dtype == torch.bfloat16 else DTYPE_F32
    ids = torch.empty(m, dtype=torch.int32, device=h.device)
    vals = torch.empty(m, dtype=torch.float32, device=h.device)
    flags = torch.zeros(m, dtype=torch.int32, device=h.device)
    if W_tiled is not None and _mode(mode) == MODE_FAST and dt == DTYPE_BF16:
        check(lib().frs_verify_head_argmax_tiled(ctx.handle, _ptr(h), m, d, _ptr(W), _ptr(W_tiled), W.shape[0],
                                                 id_offset, _ptr(ids), _ptr(vals), _ptr(flags), _stream(stream)),
              "verify_head_argmax")
        return ids, vals, flags
    check(lib().frs_verify_head_argmax(ctx.handle, _ptr(h), m, d, _ptr(W), W.shape[0], dt, id_offset, _mode(mode),
                                       _ptr(ids), _ptr(vals), _ptr(flags), _stream(stream)), "verify_head_argmax")
    return ids, vals, flags


def accept_greedy(ctx: Context, argmax_ids: torch.Tensor, tokens: torch.Tensor, parents: torch.Tensor, stream=None):
    k = int(tokens.numel())
    dev = argmax_ids.device
    emitted = torch.empty(k + 1, dtype=torch.int32, device=dev)
    path = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    counts = torch.empty(2, dtype=torch.int32, device=dev)
    check(lib().frs_accept_greedy(ctx.handle, _ptr(argmax_ids), _ptr(tokens), _ptr(parents), k, _ptr(emitted),
                                  _ptr(path), _ptr(counts), _stream(stream)), "accept_greedy")
    return emitted, path, counts


def argmax_merge(ctx: Context, vals: torch.Tensor, ids: torch.Tensor, stream=None):
    G, m = vals.shape
    ov = torch.empty(m, dtype=torch.float32, device=vals.device)
    oi = torch.empty(m, dtype=torch.int32, device=vals.device)
    check(lib().frs_argmax_merge(ctx.handle, _ptr(vals.contiguous()), _ptr(ids.contiguous()), G, m, _ptr(ov), _ptr(oi),
                                 _stream(stream)), "argmax_merge")
    return ov, oi


# ---------------------------------------------------------------- vocab-parallel verify
def vocab_shard(vocab_size: int, world: int, rank: int):
    """Contiguous vocabulary shard [start, start + count) of `rank` (frs_vocab_shard)."""
    st, cnt = C.c_int64(), C.c_int64()
    check(lib().frs_vocab_shard(vocab_size, world, rank, C.byref(st), C.byref(cnt)), "vocab_shard")
    return int(st.value), int(cnt.value)


def argmax_merge_host(vals: np.ndarray, ids: np.ndarray):
    """Host twin of argmax_merge for host-resident gathered pairs [shards x m]."""
    v = np.ascontiguousarray(vals, np.float32)
    i = np.ascontiguousarray(ids, np.int32)
    G, m = v.shape
    ov, oi = np.empty(m, np.float32), np.empty(m, np.int32)
    check(lib().frs_argmax_merge_host(_np_ptr(v), _np_ptr(i), G, m, _np_ptr(ov), _np_ptr(oi)), "argmax_merge_host")
    return ov, oi


class NcclComm:
    """An NCCL communicator owned by the library (frs_nccl_comm_init): rank 0 makes the
    ncclUniqueId, `group` (any torch.distributed group, gloo or nccl) broadcasts it, every rank
    joins on ctx's device. Used by verify_head_argmax_vocab_parallel."""

    def __init__(self, ctx: Context, group=None):
        import torch.distributed as dist
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (C.c_ubyte * 128)()
        if self.rank == 0:
            check(lib().frs_nccl_get_unique_id(uid), "nccl unique id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        check(lib().frs_nccl_comm_init(ctx.handle, self.world, uid, self.rank, C.byref(h)), "nccl comm init")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            check(lib().frs_nccl_comm_destroy(self.handle), "nccl comm destroy")
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def verify_head_argmax_vocab_parallel(ctx: Context, h: torch.Tensor, W_shard: torch.Tensor, vocab_size: int,
                                      comm: NcclComm, mode="fast", stream=None):
    """Vocab-parallel verify head through the C ABI (frs_verify_head_argmax_vp): this rank holds
    rows [start, start + count) of the LM head (`vocab_shard`); K3 on its shard (id_offset =
    start), ncclAllGather of every rank's (value, id) pairs, K5 merge by (value desc, id asc) —
    argmax's lowest-id rule (kernels.cpp:117-121). Returns (ids, values, this rank's flags)."""
    start, count = vocab_shard(vocab_size, comm.world, comm.rank)
    if W_shard.shape[0] != count:
        raise InvalidArgument(f"verify (vocab-parallel): rank {comm.rank} holds {W_shard.shape[0]} rows, expected {count}")
    h = h.contiguous()
    m, d = h.shape
    if W_shard.dim() != 2 or W_shard.shape[1] != d:
        raise InvalidArgument(f"matmul: inner dimensions differ ({tuple(h.shape)} vs {tuple(W_shard.shape)})")
    dt = DTYPE_BF16 if W_shard.dtype == torch.bfloat16 else DTYPE_F32
    ids = torch.empty(m, dtype=torch.int32, device=h.device)
    vals = torch.empty(m, dtype=torch.float32, device=h.device)
    flags = torch.zeros(m, dtype=torch.int32, device=h.device)
    check(lib().frs_verify_head_argmax_vp(ctx.handle, comm.handle, _ptr(h), m, d, _ptr(W_shard), W_shard.shape[0], dt,
                                          start, _mode(mode), _ptr(ids), _ptr(vals), _ptr(flags), _stream(stream)),
          "verify_head_argmax_vp")
    return ids, vals, flags


def gather_rows(ctx: Context, table: torch.Tensor, tokens: torch.Tensor, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
    n = int(tokens.numel())
    if out is None:
        out = torch.empty((n, table.shape[1]), dtype=torch.float32, device=table.device)
    check(lib().frs_gather_rows(ctx.handle, _ptr(table), table.shape[0], table.shape[1], _ptr(tokens), n, _ptr(out),
                                _stream(stream)), "gather_rows")
    return out


# ---------------------------------------------------------------- drafting / verification
@dataclass
class DraftParams:  # drafting.h:13-17
    beam_width: int = 10
    search_depth: int = 6
    total_draft_tokens: int = 60


@dataclass
class DraftTree:  # drafting.h:21-29 as parallel arrays (+ DraftResult's distributions, drafting.h:31-37)
    tokens: np.ndarray
    parents: np.ndarray
    depths: np.ndarray
    log_joint: np.ndarray
    root_probs: Optional[np.ndarray] = None  # keep_probs: [V_sub] root distribution
    node_probs: Optional[np.ndarray] = None  # keep_probs: [K, V_sub], rows of unexpanded nodes zero
    has_probs: Optional[np.ndarray] = None   # keep_probs: [K] 1 where node_probs[i] was recorded

    def __len__(self) -> int:
        return int(self.tokens.size)


def build_tree_mask(parents) -> np.ndarray:
    """verification.cpp:13-27: words[i] = words[parent] | 1 << i."""
    p = _i32(parents)
    w = np.zeros(max(p.size, 1), np.uint64)
    check(lib().frs_tree_mask(_np_ptr(p), p.size, _np_ptr(w)), "build_tree_mask")
    return w[: p.size]


class DeviceHead:
    """frs_head: a device-resident RestrictedHead owned by the library (host-buffer API)."""

    def __init__(self, ctx: Context, lm_head, subset: RankedSubset, dtype="bf16"):
        self.ctx, self.subset, self.dtype = ctx, subset, _dtype(dtype)
        self._keep = lm_head
        if isinstance(lm_head, torch.Tensor) and lm_head.is_cuda:
            W, on_dev, V, d = _ptr(lm_head.contiguous()), 1, lm_head.shape[0], lm_head.shape[1]
        else:
            arr = np.ascontiguousarray(lm_head, np.float32)
            self._keep = arr
            W, on_dev, (V, d) = _np_ptr(arr), 0, arr.shape
        self.vocab, self.d = int(V), int(d)
        p = C.c_void_p()
        check(lib().frs_head_create(ctx.handle, W, V, d, on_dev, _np_ptr(subset.ordered_ids), subset.size(),
                                    self.dtype, C.byref(p)), "restrict_lm_head")
        self.handle = p
        self._keep = None

    def close(self):
        if self.handle:
            lib().frs_head_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def draft_host(self, h: np.ndarray, k: int, mode="exact", out=None):
        """One level with HOST buffers (the e2e call): h [n x d] float32; returns (ridx, full,
        prob) [n x k], written into `out` when given (three C-contiguous arrays, int32 / int32 /
        float32). Pinned h (e.g. a pin_memory tensor's .numpy()) in FAST mode with n <= 16 is
        read by the device directly, with no copy operation."""
        if not (h.dtype == np.float32 and h.flags.c_contiguous):
            h = np.ascontiguousarray(h, np.float32)
        n = h.shape[0]
        if out is None:
            out = (np.empty((n, k), np.int32), np.empty((n, k), np.int32), np.empty((n, k), np.float32))
        ridx, full, prob = out
        if not all(a.flags.c_contiguous and a.size >= n * k for a in out) or ridx.dtype != np.int32 \
                or full.dtype != np.int32 or prob.dtype != np.float32:
            raise InvalidArgument("draft_host: out must be three C-contiguous [n x k] int32/int32/float32 arrays")
        st = lib().frs_head_draft_host(self.handle, h.ctypes.data, n, k, _mode(mode), ridx.ctypes.data,
                                       full.ctypes.data, prob.ctypes.data)
        if st:
            check(st, "draft_host")
        return ridx, full, prob

    def build_draft_tree(self, root_token: int, params: DraftParams = DraftParams(), mode="exact",
                         provider: Optional[Callable] = None, hidden_table: Optional[torch.Tensor] = None,
                         rng: Optional["Rng"] = None, keep_probs: bool = False) -> DraftTree:
        """Head-path build_draft_tree (drafting.cpp:122-245). provider(level, tokens,
        parent_cands) -> CUDA float32 [n x d] tensor of the forwarded rows' hidden states.
        rng=None: greedy children (top-width); with an Rng: sampled children without
        replacement (drafting.cpp:44-74, EXACT arithmetic) and the prefix-closed selection."""
        if rng is not None and mode != "exact":
            raise ValueError("sampled drafting runs on the exact probabilities: mode must be 'exact'")
        if keep_probs and rng is None:
            raise NotSupported("keep_probs is provided with an rng (sampled drafting)")
        keep = {}

        def cb(_user, level, n, tok_p, par_p, hidden_dev, stream):
            try:
                toks = np.ctypeslib.as_array(tok_p, (n,)).copy()
                pars = np.ctypeslib.as_array(par_p, (n,)).copy()
                hid = provider(level, toks, pars).to(torch.float32).contiguous()
                dst = torch.as_tensor(_DeviceView(hidden_dev, (n, self.d)), device=hid.device)
                dst.copy_(hid)
                torch.cuda.current_stream(hid.device).synchronize()  # library stream reads it next
                return 0
            except Exception as exc:  # surfaced as FRS_ELOGIC by the library
                keep["exc"] = exc
                return 9

        fn = _lib.HIDDEN_FN(cb) if provider is not None else C.cast(None, _lib.HIDDEN_FN)
        total = params.total_draft_tokens
        tok, par, dep = (np.empty(max(total, 1), np.int32) for _ in range(3))
        lj, cnt = np.empty(max(total, 1), np.float64), C.c_int()
        if rng is None:
            st = lib().frs_draft_tree(self.handle, root_token, fn, None, _ptr(hidden_table), params.beam_width,
                                      params.search_depth, total, _mode(mode), _np_ptr(tok), _np_ptr(par),
                                      _np_ptr(dep), _np_ptr(lj), C.byref(cnt))
        else:
            rp, npb, hp = _probs_buffers(keep_probs, total, self.subset.size())
            st = lib().frs_draft_tree_sampled(self.handle, root_token, fn, None, _ptr(hidden_table),
                                              params.beam_width, params.search_depth, total, rng.handle,
                                              _np_ptr(tok), _np_ptr(par), _np_ptr(dep), _np_ptr(lj), C.byref(cnt),
                                              _np_ptr(rp), _np_ptr(npb), _np_ptr(hp))
        if "exc" in keep:
            raise keep["exc"]
        check(st, "build_draft_tree")
        n = cnt.value
        tree = DraftTree(tok[:n].copy(), par[:n].copy(), dep[:n].copy(), lj[:n].copy())
        if rng is not None and keep_probs:
            tree.root_probs, tree.node_probs, tree.has_probs = rp, npb[:n].copy(), hp[:n].copy()
        return tree


class Rng:
    """The reference's ``std::mt19937_64`` (drafting.cpp:44-74, verification.cpp:76-178): one
    engine, advanced by every draw in the reference's order."""

    def __init__(self, seed: int):
        h = C.c_void_p()
        check(lib().frs_rng_create(C.c_uint64(seed), C.byref(h)), "rng")
        self.handle = h

    def uniforms(self, count: int) -> np.ndarray:
        """std::uniform_real_distribution<double>(0, 1) draws (advances the engine)."""
        out = np.empty(count, np.float64)
        check(lib().frs_rng_uniforms(self.handle, count, _np_ptr(out)), "rng")
        return out

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib._LIB is not None:
                lib().frs_rng_destroy(self.handle)
                self.handle = None
        except Exception:  # interpreter shutdown
            pass


@dataclass
class SampledLevel:
    ridx: torch.Tensor   # [n, w] restricted indices, draw order
    full: torch.Tensor   # [n, w] full-vocabulary ids
    prob: torch.Tensor   # [n, w] probabilities of the drawn children
    count: torch.Tensor  # [n] draws made
    flags: torch.Tensor  # [n] FLAG_SAMPLE_UNCERTIFIED: replay the row on the host
    probs: torch.Tensor  # [n, v_sub] exact probabilities


def draft_head_sample(ctx: Context, h: torch.Tensor, head: "RestrictedHead", width: int,
                      uniforms: torch.Tensor) -> SampledLevel:
    """K2 sampled (pick_children's sampled branch, drafting.cpp:44-74) over the EXACT softmax:
    uniforms [n, min(width, v_sub)] float64 on the device, in draw order."""
    h = h.contiguous()
    n, d = h.shape
    w = min(width, head.v_sub)
    dev = h.device
    u = uniforms.to(device=dev, dtype=torch.float64).contiguous()
    out = SampledLevel(torch.empty((n, w), dtype=torch.int32, device=dev), torch.empty((n, w), dtype=torch.int32, device=dev),
                       torch.empty((n, w), dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
                       torch.empty(n, dtype=torch.int32, device=dev),
                       torch.empty((n, head.v_sub), dtype=torch.float32, device=dev))
    check(lib().frs_draft_head_sample(ctx.handle, _ptr(h), n, d, _ptr(head.slab), head.v_sub, head.dtype,
                                      _ptr(head.ordered_dev), width, C.c_float(1.0), _ptr(u), _ptr(out.probs),
                                      _ptr(out.ridx), _ptr(out.full), _ptr(out.prob), _ptr(out.count),
                                      _ptr(out.flags), _stream(None)), "draft_head_sample")
    return out


def _probs_buffers(keep_probs: bool, total: int, v_sub: int):
    if not keep_probs:
        return None, None, None
    return (np.zeros(v_sub, np.float32), np.zeros((max(total, 1), v_sub), np.float32),
            np.zeros(max(total, 1), np.int32))


def build_draft_tree_model(head: "DeviceHead", draft: "DraftModel", pending, params: "DraftParams" = None,
                           mode="exact", rng: Optional["Rng"] = None, keep_probs: bool = False) -> "DraftTree":
    """build_draft_tree (drafting.cpp:122-245) with the device draft model as the hidden-state
    source (the reference's own drafting loop: pending context forward, per-level beam forwards
    with tree visibility, cache truncated back). rng: sampled children (EXACT arithmetic);
    keep_probs (with rng): the DraftResult distributions stochastic verification consumes."""
    params = params or DraftParams()
    if rng is not None and mode != "exact":
        raise ValueError("sampled drafting runs on the exact probabilities: mode must be 'exact'")
    pend = _i32(pending)
    total = params.total_draft_tokens
    tok, par, dep = (np.empty(max(total, 1), np.int32) for _ in range(3))
    lj, cnt = np.empty(max(total, 1), np.float64), C.c_int()
    rp, npb, hp = _probs_buffers(keep_probs, total, head.subset.size())
    check(lib().frs_draft_tree_model(head.handle, draft.handle, _np_ptr(pend), pend.size, params.beam_width,
                                     params.search_depth, total, _mode(mode), None if rng is None else rng.handle,
                                     _np_ptr(tok), _np_ptr(par), _np_ptr(dep), _np_ptr(lj), C.byref(cnt),
                                     _np_ptr(rp), _np_ptr(npb), _np_ptr(hp)),
          "build_draft_tree")
    n = cnt.value
    tree = DraftTree(tok[:n].copy(), par[:n].copy(), dep[:n].copy(), lj[:n].copy())
    if keep_probs:
        tree.root_probs, tree.node_probs, tree.has_probs = rp, npb[:n].copy(), hp[:n].copy()
    return tree


class _DeviceView:
    """__cuda_array_interface__ view of a library-owned float32 device buffer."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


@dataclass
class VerifyOutcome:  # verification.h:25-30
    accepted_path: np.ndarray
    emitted: np.ndarray

    def accepted_length(self) -> int:
        return int(self.emitted.size)


def verify_greedy(ctx: Context, h_dev: torch.Tensor, lm_head: torch.Tensor, tree: DraftTree, mode="exact") -> VerifyOutcome:
    """verification.cpp:42-71 with the target head on the device. h_dev: [1 + K, d] CUDA
    float32 (row 0 = root position, row 1 + i = node i)."""
    k = len(tree)
    dt = DTYPE_BF16 if lm_head.dtype == torch.bfloat16 else DTYPE_F32
    em, path = np.empty(k + 1, np.int32), np.empty(max(k, 1), np.int32)
    ne, npth = C.c_int(), C.c_int()
    tok, par = _i32(tree.tokens), _i32(tree.parents)
    check(lib().frs_verify_greedy(ctx.handle, _ptr(h_dev.contiguous()), _ptr(lm_head), lm_head.shape[0],
                                  lm_head.shape[1], dt, _mode(mode), _np_ptr(tok), _np_ptr(par), k, _np_ptr(em),
                                  C.byref(ne), _np_ptr(path), C.byref(npth)), "verify_greedy")
    return VerifyOutcome(path[: npth.value].copy(), em[: ne.value].copy())


def verify_stochastic(ctx: Context, h_dev: torch.Tensor, lm_head: torch.Tensor, tree: DraftTree, q_root,
                      q_nodes, has_q, ordered, rng: "Rng", temperature: float = 1.0) -> VerifyOutcome:
    """verification.cpp:76-178: exact target probabilities on the device (rows of h_dev: root
    first, then one per node), the reference's residual walk on the host with ``rng``. q_root
    [v_sub] / q_nodes [K, v_sub] / has_q [K]: the draft distributions (DraftResult root_probs /
    node_probs; has_q[i] = 0 where node i was not expanded); ordered: the drafting subset's ids
    (None: the draft head is the full vocabulary)."""
    k = len(tree)
    dt = DTYPE_BF16 if lm_head.dtype == torch.bfloat16 else DTYPE_F32
    qr = np.ascontiguousarray(q_root, np.float32)
    qn = np.ascontiguousarray(q_nodes, np.float32).reshape(k, qr.size) if k else np.zeros((1, qr.size), np.float32)
    hq = _i32(has_q) if k else np.zeros(1, np.int32)
    od = None if ordered is None else _i32(ordered)
    em, path = np.empty(k + 1, np.int32), np.empty(max(k, 1), np.int32)
    ne, npth = C.c_int(), C.c_int()
    tok, par = _i32(tree.tokens), _i32(tree.parents)
    check(lib().frs_verify_stochastic(ctx.handle, _ptr(h_dev.contiguous()), _ptr(lm_head), lm_head.shape[0],
                                      lm_head.shape[1], dt, _np_ptr(tok), _np_ptr(par), k, _np_ptr(qr), qr.size,
                                      _np_ptr(qn), _np_ptr(hq), _np_ptr(od), C.c_float(temperature), rng.handle,
                                      _np_ptr(em), C.byref(ne), _np_ptr(path), C.byref(npth)), "verify_stochastic")
    return VerifyOutcome(path[: npth.value].copy(), em[: ne.value].copy())


def verify_greedy_table(ctx: Context, table: torch.Tensor, root_token: int, lm_head: torch.Tensor, tree: DraftTree,
                        mode="exact") -> VerifyOutcome:
    """verify_greedy with hidden rows gathered on the device from table[V x d] (CUDA float32)
    by [root_token, tree.tokens...] — the head-path decode loop's identity draft/target layer."""
    k = len(tree)
    dt = DTYPE_BF16 if lm_head.dtype == torch.bfloat16 else DTYPE_F32
    em, path = np.empty(k + 1, np.int32), np.empty(max(k, 1), np.int32)
    ne, npth = C.c_int(), C.c_int()
    tok, par = _i32(tree.tokens), _i32(tree.parents)
    check(lib().frs_verify_greedy_table(ctx.handle, _ptr(table), table.shape[0], root_token, _ptr(lm_head),
                                        lm_head.shape[0], lm_head.shape[1], dt, _mode(mode), _np_ptr(tok), _np_ptr(par),
                                        k, _np_ptr(em), C.byref(ne), _np_ptr(path), C.byref(npth)), "verify_greedy")
    return VerifyOutcome(path[: npth.value].copy(), em[: ne.value].copy())


def decode_step_table(head: "DeviceHead", table: torch.Tensor, root_token: int, lm_head: torch.Tensor,
                      params: "DraftParams" = None, mode="exact",
                      lm_head_tiled: Optional[torch.Tensor] = None) -> Tuple[DraftTree, VerifyOutcome]:
    """One head-path decode iteration: build_draft_tree(root_token, hidden_table=table) then
    verify_greedy_table(table, root_token, lm_head, tree) with no host round trip in between
    (frs_decode_step_table). Same results as the two calls."""
    params = params or DraftParams()
    total = params.total_draft_tokens
    tok, par, dep = (np.empty(max(total, 1), np.int32) for _ in range(3))
    lj, cnt = np.empty(max(total, 1), np.float64), C.c_int()
    em, path = np.empty(total + 1, np.int32), np.empty(max(total, 1), np.int32)
    ne, npth = C.c_int(), C.c_int()
    dt = DTYPE_BF16 if lm_head.dtype == torch.bfloat16 else DTYPE_F32
    if table.shape[1] != head.d or lm_head.shape[1] != head.d or table.shape[0] < head.vocab:
        raise ValueError("decode_step: table [>= vocab x d] and verify head [V x d] must match the draft head")
    if lm_head_tiled is not None and dt == DTYPE_BF16:  # the verify head's tiled image (tile_image)
        check(lib().frs_decode_step_table_tiled(head.handle, _ptr(table), root_token, _ptr(lm_head), _ptr(lm_head_tiled),
                                                lm_head.shape[0], _mode(mode), params.beam_width, params.search_depth,
                                                total, _np_ptr(tok), _np_ptr(par), _np_ptr(dep), _np_ptr(lj),
                                                C.byref(cnt), _np_ptr(em), C.byref(ne), _np_ptr(path), C.byref(npth)),
              "decode_step")
    else:
        check(lib().frs_decode_step_table(head.handle, _ptr(table), root_token, _ptr(lm_head), lm_head.shape[0], dt,
                                          _mode(mode), params.beam_width, params.search_depth, total, _np_ptr(tok),
                                          _np_ptr(par), _np_ptr(dep), _np_ptr(lj), C.byref(cnt), _np_ptr(em),
                                          C.byref(ne), _np_ptr(path), C.byref(npth)), "decode_step")
    n = cnt.value
    return (DraftTree(tok[:n].copy(), par[:n].copy(), dep[:n].copy(), lj[:n].copy()),
            VerifyOutcome(path[: npth.value].copy(), em[: ne.value].copy()))


def decode_step_table_multi(head: "DeviceHead", table: torch.Tensor, roots, lm_head: torch.Tensor,
                            params: "DraftParams" = None, mode="fast",
                            lm_head_tiled: Optional[torch.Tensor] = None) -> List[Tuple[DraftTree, VerifyOutcome]]:
    """One head-path decode iteration for each of S independent streams (BASELINE configs[4]),
    batched across streams (frs_decode_step_table_multi): per stream the same results as
    decode_step_table(head, table, roots[q], lm_head, params, mode)."""
    params = params or DraftParams()
    total = params.total_draft_tokens
    r = np.ascontiguousarray(np.asarray(roots, dtype=np.int32).reshape(-1))
    S = int(r.size)
    if S < 1:
        raise ValueError("decode_step: at least one stream")
    if table.shape[1] != head.d or lm_head.shape[1] != head.d or table.shape[0] < head.vocab:
        raise ValueError("decode_step: table [>= vocab x d] and verify head [V x d] must match the draft head")
    tok, par, dep = (np.empty(S * total, np.int32) for _ in range(3))
    lj = np.empty(S * total, np.float64)
    em, path = np.empty(S * (total + 1), np.int32), np.empty(S * total, np.int32)
    cnt, ne, npth = (np.empty(S, np.int32) for _ in range(3))
    dt = DTYPE_BF16 if lm_head.dtype == torch.bfloat16 else DTYPE_F32
    check(lib().frs_decode_step_table_multi(head.handle, _ptr(table), S, _np_ptr(r), _ptr(lm_head),
                                            _ptr(lm_head_tiled) if dt == DTYPE_BF16 else None, lm_head.shape[0],
                                            dt, _mode(mode), params.beam_width, params.search_depth, total,
                                            _np_ptr(tok), _np_ptr(par), _np_ptr(dep), _np_ptr(lj), _np_ptr(cnt),
                                            _np_ptr(em), _np_ptr(ne), _np_ptr(path), _np_ptr(npth)), "decode_step")
    out = []
    for q in range(S):
        n, o = int(cnt[q]), q * total
        tree = DraftTree(tok[o:o + n].copy(), par[o:o + n].copy(), dep[o:o + n].copy(), lj[o:o + n].copy())
        e0 = q * (total + 1)
        out.append((tree, VerifyOutcome(path[o:o + int(npth[q])].copy(), em[e0:e0 + int(ne[q])].copy())))
    return out


class AcceptanceStats:
    """AcceptanceStats (verification.h:52-62, verification.cpp:180-206) over the C ABI
    (frs_acceptance_add / frs_acceptance_merge / frs_accepted_length_stats)."""

    def __init__(self):
        self._c = _lib.AcceptanceStatsC()

    @property
    def iterations(self) -> int:
        return int(self._c.iterations)

    @property
    def emitted(self) -> int:
        return int(self._c.emitted)

    @property
    def mean_accepted_length(self) -> float:
        return float(self._c.mean_accepted_length)

    @property
    def histogram(self) -> list:
        return [int(self._c.histogram[i]) for i in range(self._c.hist_len)]

    def add(self, accepted_length: int) -> None:
        check(lib().frs_acceptance_add(C.byref(self._c), int(accepted_length)), "AcceptanceStats::add")

    def merge(self, other: "AcceptanceStats") -> None:
        check(lib().frs_acceptance_merge(C.byref(self._c), C.byref(other._c)), "AcceptanceStats::merge")


def accepted_length_stats(outcomes: Sequence[VerifyOutcome]) -> AcceptanceStats:
    """verification.cpp:197-206 (raises InvalidArgument on an empty list, as the reference)."""
    lens = np.array([o.accepted_length() for o in outcomes], np.int32)
    s = AcceptanceStats()
    check(lib().frs_accepted_length_stats(_np_ptr(lens) if lens.size else None, int(lens.size), C.byref(s._c)),
          "accepted_length_stats")
    return s


__all__ = [n for n in dir() if not n.startswith("_")] + ["CapacityError"]
