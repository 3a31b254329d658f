"""Corpus formats and counting (vocab.cpp:15-38, 198-308): the FRTK
binary token stream, the text stream and the ranked-id file, cross-checked with the compiled
reference in both directions (write here / read there and back), including its DataError
rejections; count_frequencies on the device (GPU test) == the reference's on a Zipf corpus."""
import os

import numpy as np
import pytest

from paper_2502_14856_b200 import api
from paper_2502_14856_b200._lib import FrsError


def test_token_stream_roundtrip_both_ways(reference, tmp_path):
    toks = reference.zipf_tokens(5000, 1.0, 20000, 42)
    a, b = str(tmp_path / "ours.frtk"), str(tmp_path / "ref.frtk")
    api.write_token_stream(a, 5000, toks)
    reference.write_token_stream(b, 5000, toks)
    assert open(a, "rb").read() == open(b, "rb").read()  # byte-identical files
    v, t = api.read_token_stream(b)
    assert v == 5000 and np.array_equal(t, toks)
    v2, t2 = reference.read_token_stream(a)
    assert v2 == 5000 and np.array_equal(t2, toks)


def test_token_stream_rejections_match_reference(reference, tmp_path):
    cases = {"bad_magic": b"FRTX" + bytes(16),
             "bad_version": b"FRTK" + (2).to_bytes(4, "little") + bytes(12),
             "truncated": b"FRTK" + (1).to_bytes(4, "little") + (10).to_bytes(4, "little"),
             "bad_vocab": b"FRTK" + (1).to_bytes(4, "little") + (0).to_bytes(4, "little") + (0).to_bytes(8, "little"),
             "out_of_range": b"FRTK" + (1).to_bytes(4, "little") + (10).to_bytes(4, "little") +
                             (2).to_bytes(8, "little") + (3).to_bytes(4, "little") + (10).to_bytes(4, "little"),
             "short_body": b"FRTK" + (1).to_bytes(4, "little") + (10).to_bytes(4, "little") +
                           (3).to_bytes(8, "little") + (3).to_bytes(4, "little")}
    for name, blob in cases.items():
        p = str(tmp_path / (name + ".frtk"))
        with open(p, "wb") as fh:
            fh.write(blob)
        with pytest.raises(Exception) as ref_exc:
            reference.read_token_stream(p)
        with pytest.raises(FrsError) as our_exc:
            api.read_token_stream(p)
        assert str(our_exc.value).split(": ", 1)[1] == str(ref_exc.value).split(": ", 1)[1], name


def test_text_stream_and_ranked_file(tmp_path):
    """Text formats (vocab.cpp:274-306). Checked against their stated layouts: the compiled
    reference's iostream number parsing cannot run inside this numpy-hosting process (its
    libstdc++ differs from the one numpy loads), so these readers are pinned by content."""
    p = str(tmp_path / "t.txt")
    with open(p, "w") as fh:
        fh.write("3 1\n4 1 5\n\n9 2 6\n")
    assert api.read_token_stream_text(p, 10).tolist() == [3, 1, 4, 1, 5, 9, 2, 6]
    with open(p, "w") as fh:
        fh.write("3 1 x\n")
    with pytest.raises(FrsError, match="unparsable token id at offset 2"):
        api.read_token_stream_text(p, 10)
    with open(p, "w") as fh:
        fh.write("3 10\n")
    with pytest.raises(FrsError, match="token id 10 out of range at offset 1"):
        api.read_token_stream_text(p, 10)
    ids = np.random.default_rng(1).permutation(700)[:300].astype(np.int32)
    a = str(tmp_path / "ours.rank")
    api.write_ranked_file(a, ids)
    assert open(a).read() == "".join(f"{i}\n" for i in ids)  # `f << t << '\n'` (vocab.cpp:291)
    assert np.array_equal(api.read_ranked_file(a), ids)
    with open(a, "w") as fh:
        fh.write("5\n-1\n")
    with pytest.raises(FrsError, match="negative token id"):
        api.read_ranked_file(a)
    with open(a, "w") as fh:
        fh.write("5\n7\nz\n")
    with pytest.raises(FrsError, match="unparsable token id at line 3"):
        api.read_ranked_file(a)


@pytest.mark.gpu
@pytest.mark.parametrize("vocab,count,permute", [(32000, 1_000_000, False), (152064, 2_000_000, True), (50, 10, False)])
def test_count_frequencies_device_matches_reference(cuda_ctx, reference, vocab, count, permute):
    import torch
    toks = reference.zipf_tokens(vocab, 1.0, count, 42)
    if permute:  # ids no longer rank-ordered: most counts go through the global atomics
        toks = np.random.default_rng(3).permutation(vocab).astype(np.int32)[toks]
    ref_counts, ref_total = reference.count_frequencies(toks, vocab)
    tab = api.count_frequencies_device(cuda_ctx, torch.from_numpy(toks).cuda(), vocab)
    assert np.array_equal(tab.counts, ref_counts) and tab.total == count


@pytest.mark.gpu
def test_count_frequencies_device_rejects_like_reference(cuda_ctx):
    import torch
    toks = np.arange(1000, dtype=np.int32) % 100
    toks[[700, 300]] = [150, -2]  # the first offending offset is 300
    with pytest.raises(FrsError, match="token id -2 out of range at offset 300"):
        api.count_frequencies_device(cuda_ctx, torch.from_numpy(toks).cuda(), 100)
