"""CPU: the C-ABI library loads, exports every symbol include/frspec_cuda.h declares, and its
host-side FR vocabulary / tree-mask logic matches the oracle (no device compute here)."""
import os
import re

import numpy as np
import pytest

from paper_2502_14856_b200 import api
from paper_2502_14856_b200._lib import LIB_PATH, InvalidArgument, CapacityError, lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "frspec_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(frs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    assert os.path.exists(LIB_PATH)
    L = lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []
    assert L.frs_abi_version() == 1


def test_vocab_matches_oracle(restatement):
    rng = np.random.default_rng(5)
    stream = np.minimum(rng.zipf(1.2, 300_000) - 1, 7999).astype(np.int32)
    t = api.count_frequencies(stream, 8000)
    assert np.array_equal(t.counts, restatement.count_frequencies(stream, 8000))
    for size, forced in ((2048, [0, 1]), (1, []), (8000, [7999])):
        s = api.build_subset(t, size, forced)
        assert np.array_equal(s.ordered_ids, restatement.build_subset(t.counts, size, forced))
        assert all(s.full_id(s.restricted_index(int(x))) == int(x) for x in s.ordered_ids[:50])
    rk = rng.permutation(8000).astype(np.int32)
    s = api.subset_from_ranking(rk, 100, 8000, [rk[7000]])
    assert np.array_equal(s.ordered_ids, restatement.subset_from_ranking(rk, 100, 8000, [rk[7000]]))
    cov = api.coverage(t, api.build_subset(t, 2048))
    assert 0.0 < cov <= 1.0
    assert api.flops_ratio(131072, 8192) == 0.0625


def test_vocab_rejections():
    t = api.count_frequencies(np.array([0, 1, 1], np.int32), 4)
    with pytest.raises(InvalidArgument):
        api.build_subset(t, 5)
    with pytest.raises(InvalidArgument):
        api.build_subset(t, 1, [0, 1])
    with pytest.raises(InvalidArgument):
        api.count_frequencies(np.array([4], np.int32), 4)
    with pytest.raises(InvalidArgument):
        api.subset_from_ranking(np.array([0, 0], np.int32), 1, 4)
    with pytest.raises(InvalidArgument):
        api.flops_ratio(8, 9)


def test_tree_mask(restatement):
    rng = np.random.default_rng(6)
    for _ in range(200):
        k = int(rng.integers(1, 65))
        parents = np.array([int(rng.integers(-1, i)) for i in range(k)], np.int32)
        assert np.array_equal(api.build_tree_mask(parents), restatement.tree_mask(parents))
    with pytest.raises(CapacityError):
        api.build_tree_mask(np.arange(-1, 64, dtype=np.int32))
    with pytest.raises(InvalidArgument):
        api.build_tree_mask(np.array([-1, 1], np.int32))


def test_acceptance_stats_match_reference(reference):
    """AcceptanceStats add / merge / accepted_length_stats through the C ABI against the
    reference's own (verification.cpp:180-206), including the empty-list rejection."""
    from paper_2502_14856_b200 import api
    from paper_2502_14856_b200._lib import InvalidArgument
    rng = np.random.default_rng(4)
    for _ in range(20):
        a = rng.integers(1, 8, rng.integers(1, 40)).tolist()
        b = rng.integers(1, 12, rng.integers(0, 30)).tolist()
        outs = [api.VerifyOutcome(np.zeros(max(x - 1, 0), np.int32), np.zeros(x, np.int32)) for x in a]
        s = api.accepted_length_stats(outs)
        if b:
            s.merge(api.accepted_length_stats([api.VerifyOutcome(np.zeros(0, np.int32), np.zeros(x, np.int32))
                                               for x in b]))
        else:
            s.merge(api.AcceptanceStats())
        it, em, mean, hist = reference.acceptance_stats(a, b)
        assert (s.iterations, s.emitted, s.histogram) == (it, em, hist)
        assert s.mean_accepted_length == mean  # same double division
    with pytest.raises(InvalidArgument, match="empty outcome list"):
        api.accepted_length_stats([])
    with pytest.raises(ValueError, match="empty outcome list"):
        reference.acceptance_stats([])
    s = api.AcceptanceStats()
    s.add(3)
    s.add(0)
    assert s.histogram == [1, 0, 0, 1] and s.iterations == 2 and s.mean_accepted_length == 1.5


def test_nccl_unique_id_through_the_abi():
    """The vocab-parallel boundary resolves NCCL at run time (dlopen): the unique id a rank 0
    broadcasts comes out of the library (no GPU needed for the id itself)."""
    import ctypes as C
    uid = (C.c_ubyte * 128)()
    rc = lib().frs_nccl_get_unique_id(uid)
    if rc != 0:
        pytest.skip("NCCL not loadable here: " + lib().frs_last_error().decode())
    assert any(bytes(uid))
