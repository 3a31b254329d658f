"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy/ctypes front end to the two CPU checkers.

* ``Restatement``: the plain-C restatement (oracle/frs_oracle.c -> libfrs_oracle.so).
* ``Reference``: the reference's own sources compiled by oracle/Makefile into
  oracle/_ref/libfrspec_ref.so (patched for the drafting.cpp:200-219 use-after-free).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference arm may
import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "libfrs_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libfrspec_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_ip = C.POINTER(C.c_int)

HIDDEN_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int32),
                        C.POINTER(C.c_int32), C.POINTER(C.c_float))


def build(reference: bool = True) -> None:
    """Compile the restatement (always) and the reference (.so in _ref/) when its sources exist."""
    target = "all" if reference else "restatement"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ci32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Restatement:
    """Plain-C restatement (frs_oracle.h)."""

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            build(reference=False)
        L = self.lib = C.CDLL(path)
        L.frs_o_dot_f32.restype = C.c_float
        L.frs_o_dot_f32.argtypes = [_f32p, _f32p, C.c_int]
        L.frs_o_logits.argtypes = [_f32p, C.c_int, _f32p, C.c_int, C.c_int, _f32p]
        L.frs_o_expf_glibc.restype = C.c_float
        L.frs_o_expf_glibc.argtypes = [C.c_float]
        L.frs_o_libm_expf_range.restype = None
        L.frs_o_libm_expf_range.argtypes = [C.c_uint32, C.c_int64, _f32p]
        L.frs_o_softmax.argtypes = [_f32p, C.c_int, C.c_float, _f32p, C.POINTER(C.c_float),
                                    C.POINTER(C.c_double)]
        L.frs_o_topk.argtypes = [_f32p, C.c_int, C.c_int, _i32p, _f32p]
        L.frs_o_argmax.argtypes = [_f32p, C.c_int]
        L.frs_o_draft_level.argtypes = [_f32p, C.c_int, _f32p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                        C.c_float, _i32p, _i32p, _f32p, _f32p, _f64p, C.c_void_p]
        L.frs_o_verify_argmax.argtypes = [_f32p, C.c_int, _f32p, C.c_int, C.c_int, _i32p, _f32p]
        L.frs_o_verify_greedy_ids.argtypes = [_i32p, _i32p, _i32p, C.c_int, _i32p, _ip, _i32p, _ip]
        L.frs_o_tree_mask.argtypes = [_i32p, C.c_int, _u64p]
        L.frs_o_count_frequencies.argtypes = [_i32p, C.c_int64, C.c_int, _u64p]
        L.frs_o_build_subset.argtypes = [_u64p, C.c_int, C.c_int, _i32p, C.c_int, _i32p]
        L.frs_o_subset_from_ranking.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p]
        L.frs_o_restrict.argtypes = [_f32p, C.c_int, C.c_int, _i32p, C.c_int, _f32p]
        L.frs_o_draft_tree.argtypes = [HIDDEN_FN, C.c_void_p, _f32p, C.c_int, C.c_int, C.c_void_p,
                                       C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _f64p, _ip]

    def dot_f32(self, a, b) -> np.float32:
        a, b = _c32(a), _c32(b)
        return np.float32(self.lib.frs_o_dot_f32(a, b, a.size))

    def libm_expf_range(self, first_bits: int, count: int) -> np.ndarray:
        """The host libm's expf over float bit patterns first_bits + i (not the restatement)."""
        out = np.empty(count, np.float32)
        self.lib.frs_o_libm_expf_range(first_bits, count, out)
        return out

    def logits(self, h, W):
        h, W = _c32(h), _c32(W)
        out = np.empty((h.shape[0], W.shape[0]), np.float32)
        self.lib.frs_o_logits(h, h.shape[0], W, W.shape[0], W.shape[1], out)
        return out

    def expf(self, x: float) -> np.float32:
        return np.float32(self.lib.frs_o_expf_glibc(float(x)))

    def softmax(self, logits, temperature: float = 1.0):
        x = _c32(logits)
        p = np.empty_like(x)
        mx, tot = C.c_float(), C.c_double()
        if self.lib.frs_o_softmax(x, x.size, temperature, p, C.byref(mx), C.byref(tot)):
            raise ValueError("softmax: rejected input")
        return p, np.float32(mx.value), tot.value

    def topk(self, values, k: int):
        v = _c32(values)
        idx, val = np.empty(k, np.int32), np.empty(k, np.float32)
        if self.lib.frs_o_topk(v, v.size, k, idx, val):
            raise ValueError("topk: k out of range")
        return idx, val

    def argmax(self, values) -> int:
        v = _c32(values)
        return int(self.lib.frs_o_argmax(v, v.size))

    def draft_level(self, h, slab, ordered_ids, k: int, temperature: float = 1.0, want_logits=False):
        h, slab = _c32(np.atleast_2d(h)), _c32(slab)
        n, d = h.shape
        v_sub = slab.shape[0]
        ids = None if ordered_ids is None else _ci32(ordered_ids)
        ridx, full = np.zeros((n, k), np.int32), np.zeros((n, k), np.int32)
        prob, mx, tot = np.zeros((n, k), np.float32), np.zeros(n, np.float32), np.zeros(n, np.float64)
        lg = np.empty((n, v_sub), np.float32) if want_logits else None
        rc = self.lib.frs_o_draft_level(h, n, slab, v_sub, d, None if ids is None else ids.ctypes.data,
                                        k, temperature, ridx, full, prob, mx, tot,
                                        None if lg is None else lg.ctypes.data)
        if rc:
            raise ValueError("draft_level: rejected input")
        out = dict(ridx=ridx, full=full, prob=prob, mx=mx, total=tot)
        if want_logits:
            out["logits"] = lg
        return out

    def verify_argmax(self, h, W):
        h, W = _c32(np.atleast_2d(h)), _c32(W)
        ids, vals = np.empty(h.shape[0], np.int32), np.empty(h.shape[0], np.float32)
        self.lib.frs_o_verify_argmax(h, h.shape[0], W, W.shape[0], W.shape[1], ids, vals)
        return ids, vals

    def verify_greedy_ids(self, argmax_ids, tokens, parents):
        a, t, p = _ci32(argmax_ids), _ci32(tokens), _ci32(parents)
        k = t.size
        em, path = np.empty(k + 1, np.int32), np.empty(k + 1, np.int32)
        ne, npth = C.c_int(), C.c_int()
        self.lib.frs_o_verify_greedy_ids(a, t, p, k, em, C.byref(ne), path, C.byref(npth))
        return em[: ne.value].copy(), path[: npth.value].copy()

    def tree_mask(self, parents):
        p = _ci32(parents)
        w = np.zeros(max(p.size, 1), np.uint64)
        rc = self.lib.frs_o_tree_mask(p, p.size, w)
        if rc == 2:
            raise OverflowError("tree exceeds 64 nodes")
        if rc:
            raise ValueError("tree is not topological")
        return w[: p.size]

    def count_frequencies(self, stream, vocab_size: int):
        s = _ci32(stream)
        c = np.zeros(vocab_size, np.uint64)
        if self.lib.frs_o_count_frequencies(s, s.size, vocab_size, c):
            raise ValueError("count_frequencies: id out of range")
        return c

    def build_subset(self, counts, size: int, forced=()):
        c = np.ascontiguousarray(counts, np.uint64)
        f = _ci32(np.array(forced, np.int32))
        out = np.empty(size, np.int32)
        if self.lib.frs_o_build_subset(c, c.size, size, f, f.size, out):
            raise ValueError("build_subset: rejected input")
        return out

    def subset_from_ranking(self, ranked, size: int, vocab_size: int, forced=()):
        r = _ci32(ranked)
        f = _ci32(np.array(forced, np.int32))
        out = np.empty(size, np.int32)
        if self.lib.frs_o_subset_from_ranking(r, r.size, size, vocab_size, f, f.size, out):
            raise ValueError("subset_from_ranking: rejected input")
        return out

    def restrict(self, W, ordered):
        W, o = _c32(W), _ci32(ordered)
        out = np.empty((o.size, W.shape[1]), np.float32)
        if self.lib.frs_o_restrict(W, W.shape[0], W.shape[1], o, o.size, out):
            raise ValueError("restrict: id out of range")
        return out

    def draft_tree(self, provider, slab, ordered_ids, width: int, depth: int, total: int):
        """provider(level, tokens[n], parent_cands[n]) -> hidden [n x d] float32."""
        slab = _c32(slab)
        d = slab.shape[1]
        ids = None if ordered_ids is None else _ci32(ordered_ids)

        def cb(_user, level, n, tok_p, par_p, out_p):
            toks = np.ctypeslib.as_array(tok_p, (n,)).copy()
            pars = np.ctypeslib.as_array(par_p, (n,)).copy()
            try:
                hid = _c32(provider(level, toks, pars)).reshape(n, d)
            except Exception:  # pragma: no cover - surfaced as rc
                return 9
            C.memmove(out_p, hid.ctypes.data, hid.nbytes)
            return 0

        fn = HIDDEN_FN(cb)
        tok, par, dep = (np.empty(64, np.int32) for _ in range(3))
        lj, cnt = np.empty(64, np.float64), C.c_int()
        rc = self.lib.frs_o_draft_tree(fn, None, slab, slab.shape[0], d,
                                       None if ids is None else ids.ctypes.data, width, depth, total,
                                       tok, par, dep, lj, C.byref(cnt))
        if rc:
            raise ValueError(f"draft_tree: rc={rc}")
        n = cnt.value
        return dict(tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(), log_joint=lj[:n].copy())


class Reference:
    """The compiled (patched) reference via oracle/ref_shim.cpp."""

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_dot_f32.restype = C.c_float
        L.ref_dot_f32.argtypes = [_f32p, _f32p, C.c_int]
        L.ref_matmul.argtypes = [_f32p, C.c_int, C.c_int, _f32p, C.c_int, _f32p]
        L.ref_softmax.argtypes = [_f32p, C.c_int, C.c_float, _f32p]
        L.ref_topk.argtypes = [_f32p, C.c_int, C.c_int, _i32p, _f32p]
        L.ref_argmax.argtypes = [_f32p, C.c_int, C.POINTER(C.c_int32)]
        L.ref_count_frequencies.argtypes = [_i32p, C.c_int64, C.c_int, _u64p, C.POINTER(C.c_uint64)]
        L.ref_build_subset.argtypes = [_u64p, C.c_int, C.c_uint64, C.c_int, _i32p, C.c_int, _i32p]
        L.ref_subset_from_ranking.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p]
        L.ref_restrict_lm_head.argtypes = [_f32p, C.c_int, C.c_int, _i32p, C.c_int, _f32p]
        L.ref_zipf_tokens.argtypes = [C.c_int, C.c_double, C.c_int64, C.c_uint64, _i32p]
        L.ref_fill_gaussian.argtypes = [_f32p, C.c_int64, C.c_uint64, C.c_float]
        L.ref_fill_gaussian.restype = None
        L.ref_build_tree_mask.argtypes = [_i32p, C.c_int, _u64p]
        L.ref_verify_greedy.argtypes = [_f32p, C.c_int, _f32p, C.c_int, _i32p, _i32p, _i32p, _ip, _i32p, _ip]
        L.ref_model_lm_head.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _f32p]
        L.ref_head_new.restype = C.c_void_p
        L.ref_head_new.argtypes = [_f32p, C.c_int, C.c_int]
        L.ref_head_free.restype = None
        L.ref_head_free.argtypes = [C.c_void_p]
        L.ref_draft_level.argtypes = [C.c_void_p, _f32p, C.c_int, C.c_int, C.c_int, _i32p, _f32p]
        L.ref_verify_argmax.argtypes = [C.c_void_p, _f32p, C.c_int, C.c_int, _i32p]
        L.ref_model_draft_tree.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_void_p, C.c_int, _i32p, C.c_int,
                                                           C.c_int, C.c_int, C.c_int, _i32p, _i32p, _i32p, _f64p, _ip]
        L.ref_model_draft_capture.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_void_p, C.c_int, _i32p, C.c_int,
                                                              C.c_int, C.c_int, C.c_int, _f32p, _i32p, _i32p, _ip,
                                                              _i32p, _i32p, _i32p, _f64p, _ip]
        L.ref_model_draft_tree_rng.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_void_p, C.c_int, _i32p, C.c_int,
                                                               C.c_int, C.c_int, C.c_int, C.c_uint64, _i32p, _i32p,
                                                               _i32p, _f64p, _ip]
        L.ref_model_draft_capture_rng.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_void_p, C.c_int, _i32p, C.c_int,
                                                                  C.c_int, C.c_int, C.c_int, C.c_uint64, _f32p, _i32p,
                                                                  _i32p, _ip, _i32p, _i32p, _i32p, _f64p, _ip]
        L.ref_pick_sampled.argtypes = [_f32p, C.c_int, C.c_int, C.c_uint64, C.c_int64, _i32p, _f32p, _ip]
        L.ref_uniforms.argtypes = [C.c_uint64, C.c_int64, C.c_int, _f64p]
        L.ref_write_token_stream.argtypes = [C.c_char_p, C.c_int, _i32p, C.c_int64]
        L.ref_draft_session_new.restype = C.c_void_p
        L.ref_draft_session_new.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.ref_draft_session_free.restype = None
        L.ref_draft_session_free.argtypes = [C.c_void_p]
        L.ref_draft_session_weights.argtypes = [C.c_void_p] + [_f32p] * 7
        L.ref_draft_session_forward.argtypes = [C.c_void_p, _i32p, _i32p, C.c_int, C.c_void_p, _f32p]
        L.ref_draft_session_len.argtypes = [C.c_void_p]
        L.ref_draft_session_position.argtypes = [C.c_void_p, C.c_int]
        L.ref_draft_session_compact.argtypes = [C.c_void_p, C.c_int, _i32p, C.c_int]
        L.ref_draft_session_draft_tree.argtypes = [C.c_void_p, C.c_void_p, C.c_int, _i32p, C.c_int, C.c_int, C.c_int,
                                                   C.c_int, _i32p, _i32p, _i32p, _f64p, _ip]
        L.ref_draft_verify_rng.argtypes = [C.c_int] * 4 + [C.c_uint64, C.c_void_p, C.c_int, _i32p, C.c_int, C.c_int,
                                                            C.c_int, C.c_int, C.c_uint64, _f32p, _f32p, C.c_float, _i32p,
                                                            _i32p, _i32p, _f64p, _ip, _f32p, _f32p, _i32p, _i32p, _ip,
                                                            _i32p, _ip]
        L.ref_acceptance_stats.argtypes = [_i32p, C.c_int, _i32p, C.c_int, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                           np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"), C.c_int, _ip]
        L.ref_masked_attention.argtypes = [_f32p, _f32p, _f32p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p]
        L.ref_read_token_stream.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, _ip, C.POINTER(C.c_int64)]
        L.ref_read_token_stream_text.argtypes = [C.c_char_p, C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_write_ranked_file.argtypes = [C.c_char_p, _i32p, C.c_int64]
        L.ref_read_ranked_file.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_verify_stochastic.argtypes = [_f32p, C.c_int, _f32p, C.c_int, _i32p, _i32p, _f32p, C.c_int, _f32p, _i32p,
                                            C.c_void_p, C.c_float, C.c_uint64, _i32p, _ip, _i32p, _ip]

    def _check(self, rc: int, what: str):
        if rc:
            msg = self.lib.ref_last_error().decode()
            exc = {1: ValueError, 2: OverflowError, 3: IOError}.get(rc, RuntimeError)
            raise exc(f"{what}: {msg}")

    def dot_f32(self, a, b):
        a, b = _c32(a), _c32(b)
        return np.float32(self.lib.ref_dot_f32(a, b, a.size))

    def matmul(self, a, bt):
        a, bt = _c32(np.atleast_2d(a)), _c32(np.atleast_2d(bt))
        out = np.empty((a.shape[0], bt.shape[0]), np.float32)
        self._check(self.lib.ref_matmul(a, a.shape[0], a.shape[1], bt, bt.shape[0], out), "matmul")
        return out

    def softmax(self, logits, temperature: float = 1.0):
        x = _c32(logits)
        p = np.empty_like(x)
        self._check(self.lib.ref_softmax(x, x.size, temperature, p), "softmax")
        return p

    def topk(self, values, k: int):
        v = _c32(values)
        idx, val = np.empty(k, np.int32), np.empty(k, np.float32)
        self._check(self.lib.ref_topk(v, v.size, k, idx, val), "topk")
        return idx, val

    def argmax(self, values) -> int:
        v = _c32(values)
        o = C.c_int32()
        self._check(self.lib.ref_argmax(v, v.size, C.byref(o)), "argmax")
        return o.value

    def count_frequencies(self, stream, vocab_size: int):
        s = _ci32(stream)
        c, tot = np.zeros(vocab_size, np.uint64), C.c_uint64()
        self._check(self.lib.ref_count_frequencies(s, s.size, vocab_size, c, C.byref(tot)), "count_frequencies")
        return c, tot.value

    def build_subset(self, counts, size: int, forced=()):
        c = np.ascontiguousarray(counts, np.uint64)
        f = _ci32(np.array(forced, np.int32))
        out = np.empty(size, np.int32)
        self._check(self.lib.ref_build_subset(c, c.size, int(c.sum()), size, f, f.size, out), "build_subset")
        return out

    def subset_from_ranking(self, ranked, size: int, vocab_size: int, forced=()):
        r = _ci32(ranked)
        f = _ci32(np.array(forced, np.int32))
        out = np.empty(size, np.int32)
        self._check(self.lib.ref_subset_from_ranking(r, r.size, size, vocab_size, f, f.size, out),
                    "subset_from_ranking")
        return out

    def restrict_lm_head(self, W, ordered):
        W, o = _c32(W), _ci32(ordered)
        out = np.empty((o.size, W.shape[1]), np.float32)
        self._check(self.lib.ref_restrict_lm_head(W, W.shape[0], W.shape[1], o, o.size, out), "restrict_lm_head")
        return out

    def zipf_tokens(self, vocab_size: int, exponent: float, count: int, seed: int):
        out = np.empty(count, np.int32)
        self._check(self.lib.ref_zipf_tokens(vocab_size, exponent, count, seed, out), "zipf_tokens")
        return out

    def fill_gaussian(self, count: int, seed: int, std: float = 0.02):
        out = np.empty(count, np.float32)
        self.lib.ref_fill_gaussian(out, count, seed, std)
        return out

    def tree_mask(self, parents):
        p = _ci32(parents)
        w = np.zeros(max(p.size, 1), np.uint64)
        self._check(self.lib.ref_build_tree_mask(p, p.size, w), "build_tree_mask")
        return w[: p.size]

    def verify_greedy(self, root_logits, node_logits, tokens, parents):
        r, nl = _c32(root_logits), _c32(node_logits)
        t, p = _ci32(tokens), _ci32(parents)
        k = t.size
        em, path = np.empty(k + 1, np.int32), np.empty(k + 1, np.int32)
        ne, npth = C.c_int(), C.c_int()
        self._check(self.lib.ref_verify_greedy(r, r.size, nl, k, t, p, em, C.byref(ne), path, C.byref(npth)),
                    "verify_greedy")
        return em[: ne.value].copy(), path[: npth.value].copy()

    def head(self, W) -> "RefHead":
        return RefHead(self, W)

    def model_lm_head(self, V, d, layers, heads, seed):
        out = np.empty((V, d), np.float32)
        self._check(self.lib.ref_model_lm_head(V, d, layers, heads, seed, out), "model_lm_head")
        return out

    def model_draft_tree(self, V, d, layers, heads, max_seq, seed, ordered, pending, width, depth, total):
        o = None if ordered is None else _ci32(ordered)
        pend = _ci32(pending)
        tok, par, dep = (np.empty(64, np.int32) for _ in range(3))
        lj, cnt = np.empty(64, np.float64), C.c_int()
        self._check(self.lib.ref_model_draft_tree(V, d, layers, heads, max_seq, seed,
                                                  None if o is None else o.ctypes.data,
                                                  0 if o is None else o.size, pend, pend.size, width, depth,
                                                  total, tok, par, dep, lj, C.byref(cnt)), "build_draft_tree")
        n = cnt.value
        return dict(tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(), log_joint=lj[:n].copy())

    def model_draft_capture(self, V, d, layers, heads, max_seq, seed, ordered, pending, width, depth, total):
        o = None if ordered is None else _ci32(ordered)
        pend = _ci32(pending)
        max_rows = 1 + (depth - 1) * width
        hid = np.empty((max_rows, d), np.float32)
        rtok, rlev, nrows = np.empty(max_rows, np.int32), np.empty(max_rows, np.int32), C.c_int()
        tok, par, dep = (np.empty(64, np.int32) for _ in range(3))
        lj, cnt = np.empty(64, np.float64), C.c_int()
        self._check(self.lib.ref_model_draft_capture(V, d, layers, heads, max_seq, seed,
                                                     None if o is None else o.ctypes.data,
                                                     0 if o is None else o.size, pend, pend.size, width, depth,
                                                     total, hid, rtok, rlev, C.byref(nrows), tok, par, dep, lj,
                                                     C.byref(cnt)), "draft_capture")
        n, r = cnt.value, nrows.value
        return dict(hidden=hid[:r].copy(), row_token=rtok[:r].copy(), row_level=rlev[:r].copy(),
                    tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(),
                    log_joint=lj[:n].copy())


    def model_draft_tree_rng(self, V, d, layers, heads, max_seq, seed, ordered, pending, width, depth, total,
                             rng_seed):
        o = None if ordered is None else _ci32(ordered)
        pend = _ci32(pending)
        tok, par, dep = (np.empty(64, np.int32) for _ in range(3))
        lj, cnt = np.empty(64, np.float64), C.c_int()
        self._check(self.lib.ref_model_draft_tree_rng(V, d, layers, heads, max_seq, seed,
                                                      None if o is None else o.ctypes.data,
                                                      0 if o is None else o.size, pend, pend.size, width, depth,
                                                      total, C.c_uint64(rng_seed), tok, par, dep, lj,
                                                      C.byref(cnt)), "build_draft_tree(rng)")
        n = cnt.value
        return dict(tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(), log_joint=lj[:n].copy())

    def model_draft_capture_rng(self, V, d, layers, heads, max_seq, seed, ordered, pending, width, depth, total,
                                rng_seed):
        o = None if ordered is None else _ci32(ordered)
        pend = _ci32(pending)
        max_rows = 1 + (depth - 1) * width
        hid = np.empty((max_rows, d), np.float32)
        rtok, rlev, nrows = np.empty(max_rows, np.int32), np.empty(max_rows, np.int32), C.c_int()
        tok, par, dep = (np.empty(64, np.int32) for _ in range(3))
        lj, cnt = np.empty(64, np.float64), C.c_int()
        self._check(self.lib.ref_model_draft_capture_rng(V, d, layers, heads, max_seq, seed,
                                                         None if o is None else o.ctypes.data,
                                                         0 if o is None else o.size, pend, pend.size, width, depth,
                                                         total, C.c_uint64(rng_seed), hid, rtok, rlev,
                                                         C.byref(nrows), tok, par, dep, lj, C.byref(cnt)),
                    "draft_capture(rng)")
        n, r = cnt.value, nrows.value
        return dict(hidden=hid[:r].copy(), row_token=rtok[:r].copy(), row_level=rlev[:r].copy(),
                    tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(),
                    log_joint=lj[:n].copy())

    def verify_stochastic(self, root_logits, node_logits, tokens, parents, q_root, q_nodes, has_q, ordered,
                          temperature, rng_seed):
        rl, nl = _c32(root_logits), _c32(node_logits)
        k = nl.shape[0]
        tok, par = _ci32(tokens), _ci32(parents)
        qr, qn, hq = _c32(q_root), _c32(q_nodes), _ci32(has_q)
        o = None if ordered is None else _ci32(ordered)
        em, pa = np.empty(70, np.int32), np.empty(70, np.int32)
        ne, npth = C.c_int(), C.c_int()
        self._check(self.lib.ref_verify_stochastic(rl, rl.size, nl, k, tok, par, qr, qr.size, qn, hq,
                                                   None if o is None else o.ctypes.data, temperature,
                                                   C.c_uint64(rng_seed), em, C.byref(ne), pa, C.byref(npth)),
                    "verify_stochastic")
        return em[:ne.value].copy(), pa[:npth.value].copy()

    def draft_session(self, V, d, heads, max_seq, seed):
        """A reference 1-layer draft model + KV cache (forward_raw parity)."""
        ref = self

        class Session:
            def __init__(self):
                self.h = ref.lib.ref_draft_session_new(V, d, heads, max_seq, seed)
                assert self.h, "ref_draft_session_new failed"

            def weights(self):
                out = [np.empty((V, d), np.float32)] + [np.empty((d, d), np.float32) for _ in range(4)] + \
                      [np.empty((4 * d, d), np.float32), np.empty((d, 4 * d), np.float32)]
                ref._check(ref.lib.ref_draft_session_weights(self.h, *out), "weights")
                return dict(zip(["embedding", "wq", "wk", "wv", "wo", "w_up", "w_down"], out))

            def forward(self, tokens, positions, allow):
                t, p = _ci32(tokens), _ci32(positions)
                a = np.ascontiguousarray(allow, np.uint8)
                out = np.empty((t.size, d), np.float32)
                ref._check(ref.lib.ref_draft_session_forward(self.h, t, p, t.size, a.ctypes.data, out), "forward_raw")
                return out

            def __len__(self):
                return ref.lib.ref_draft_session_len(self.h)

            def position(self, row):
                return ref.lib.ref_draft_session_position(self.h, row)

            def compact(self, keep_from, offsets):
                o = _ci32(offsets)
                ref._check(ref.lib.ref_draft_session_compact(self.h, keep_from, o, o.size), "compact")

            def draft_tree(self, ordered, pending, width, depth, total):
                """build_draft_tree on this session's persistent cache (greedy)."""
                o = None if ordered is None else _ci32(ordered)
                p = _ci32(pending)
                tok, par, dep = (np.empty(total, np.int32) for _ in range(3))
                lj = np.empty(total, np.float64)
                cnt = C.c_int()
                ref._check(ref.lib.ref_draft_session_draft_tree(self.h, None if o is None else o.ctypes.data, 0 if o is None else o.size, p, p.size, width,
                                                                depth, total, tok, par, dep, lj, C.byref(cnt)),
                           "build_draft_tree")
                n = cnt.value
                return dict(tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(),
                            log_joint=lj[:n].copy())

            def __del__(self):
                ref.lib.ref_draft_session_free(self.h)

        return Session()

    def draft_verify_rng(self, V, d, heads, max_seq, seed, ordered, pending, width, depth, total, rng_seed, h_t, W_t,
                         temperature=1.0):
        """Sampled build_draft_tree(keep_probs) then verify_stochastic with the same engine."""
        o = _ci32(ordered)
        p = _ci32(pending)
        hv = o.size
        tok, par, dep = (np.empty(total, np.int32) for _ in range(3))
        lj = np.empty(total, np.float64)
        rp, npb, hp = np.zeros(hv, np.float32), np.zeros((total, hv), np.float32), np.zeros(total, np.int32)
        em, path = np.empty(total + 1, np.int32), np.empty(total + 1, np.int32)
        cnt, ne, npth = C.c_int(), C.c_int(), C.c_int()
        self._check(self.lib.ref_draft_verify_rng(V, d, heads, max_seq, seed, o.ctypes.data, hv, p, p.size, width, depth,
                                                  total, rng_seed, _c32(h_t), _c32(W_t), temperature, tok, par, dep, lj,
                                                  C.byref(cnt), rp, npb, hp, em, C.byref(ne), path, C.byref(npth)),
                    "draft_verify_rng")
        n = cnt.value
        return dict(tokens=tok[:n].copy(), parents=par[:n].copy(), depths=dep[:n].copy(), log_joint=lj[:n].copy(),
                    root_probs=rp, node_probs=npb[:n].copy(), has_probs=hp[:n].copy(), emitted=em[:ne.value].copy(),
                    path=path[:npth.value].copy())

    def acceptance_stats(self, lengths_a, lengths_b=None):
        """accepted_length_stats(a) [.merge(accepted_length_stats(b))] -> (iterations, emitted,
        mean, histogram); lengths_b=[] merges a default (empty) AcceptanceStats."""
        a = _ci32(lengths_a)
        b = _ci32(lengths_b if lengths_b is not None else [])
        it, em, mean, hl = C.c_int64(), C.c_int64(), C.c_double(), C.c_int()
        hist = np.zeros(128, np.int64)
        self._check(self.lib.ref_acceptance_stats(a, a.size, b, -1 if lengths_b is None else b.size, C.byref(it),
                                                  C.byref(em), C.byref(mean), hist, hist.size, C.byref(hl)),
                    "accepted_length_stats")
        return it.value, em.value, mean.value, hist[:hl.value].tolist()

    def masked_attention(self, q, k, v, allow):
        q, k, v = _c32(q), _c32(k), _c32(v)
        a = np.ascontiguousarray(allow, np.uint8)
        out = np.empty((q.shape[0], v.shape[1]), np.float32)
        self._check(self.lib.ref_masked_attention(q, k, v, a.ctypes.data, q.shape[0], k.shape[0], q.shape[1],
                                                  v.shape[1], out), "masked_attention")
        return out

    def write_token_stream(self, path, vocab, tokens):
        t = _ci32(tokens)
        self._check(self.lib.ref_write_token_stream(path.encode(), vocab, t, t.size), "write_token_stream")

    def read_token_stream(self, path):
        v, n = C.c_int(), C.c_int64()
        self._check(self.lib.ref_read_token_stream(path.encode(), None, 0, C.byref(v), C.byref(n)), "read_token_stream")
        out = np.empty(n.value, np.int32)
        self._check(self.lib.ref_read_token_stream(path.encode(), out.ctypes.data, out.size, C.byref(v), C.byref(n)),
                    "read_token_stream")
        return v.value, out

    # (the text / ranked-file readers of the reference parse with iostreams, whose libstdc++
    # differs from the one numpy loads into this process: they are not wrapped here)

    def uniforms(self, seed, count, skip=0):
        out = np.empty(count, np.float64)
        self._check(self.lib.ref_uniforms(C.c_uint64(seed), C.c_int64(skip), count, out), "uniforms")
        return out

    def pick_sampled(self, probs, width, rng_seed, skip=0):
        p = _c32(probs)
        picks, pr, cnt = np.empty(width, np.int32), np.empty(width, np.float32), C.c_int()
        self._check(self.lib.ref_pick_sampled(p, p.size, width, C.c_uint64(rng_seed), C.c_int64(skip), picks, pr,
                                              C.byref(cnt)), "pick_sampled")
        return picks[:cnt.value].copy(), pr[:cnt.value].copy()


class RefHead:
    """A reference ``Matrix`` LM head kept resident, for timing the reference's own draft level
    (model.cpp:278 + drafting.cpp:204, 37-43) and verify head (model.cpp:278 + kernels.cpp:113)."""

    def __init__(self, ref: Reference, W):
        self.ref = ref
        W = _c32(W)
        self.rows, self.d = W.shape
        self.ptr = ref.lib.ref_head_new(W, self.rows, self.d)

    def draft_level(self, h, k: int):
        h = _c32(np.atleast_2d(h))
        n = h.shape[0]
        ridx, prob = np.zeros((n, k), np.int32), np.zeros((n, k), np.float32)
        self.ref._check(self.ref.lib.ref_draft_level(self.ptr, h, n, self.d, k, ridx, prob), "draft_level")
        return ridx, prob

    def verify_argmax(self, h):
        h = _c32(np.atleast_2d(h))
        ids = np.zeros(h.shape[0], np.int32)
        self.ref._check(self.ref.lib.ref_verify_argmax(self.ptr, h, h.shape[0], self.d, ids), "verify_argmax")
        return ids

    def __del__(self):
        if getattr(self, "ptr", None):
            self.ref.lib.ref_head_free(self.ptr)
            self.ptr = None
