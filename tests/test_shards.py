"""FSOMSHRD writer/lister (host side, no GPU): byte-identical to the
reference's write_shards (dataset.hpp:252-275)."""
import os

import numpy as np
import pytest

from paper_2604_26555_b200 import shards


def test_writer_matches_reference(tmp_path):
    from paper_2604_26555_b200 import dropin
    if not dropin.available():
        pytest.skip("libtsom_dropin.so not built")
    x = np.random.default_rng(3).standard_normal((1003, 7)).astype(np.float32)
    mine = shards.write_shards(x, str(tmp_path / "a"), 4)
    dropin.write_shards(x, str(tmp_path / "b"), 4)
    theirs = shards.list_shards(str(tmp_path / "b"))
    assert [os.path.basename(p) for p in mine] == [os.path.basename(p) for p in theirs]
    for a, b in zip(mine, theirs):
        assert open(a, "rb").read() == open(b, "rb").read()


def test_layout_and_listing(tmp_path):
    x = np.arange(30, dtype=np.float32).reshape(10, 3)
    paths = shards.write_shards(x, str(tmp_path), 3)
    raw = open(paths[0], "rb").read()
    assert raw[:8] == b"FSOMSHRD" and len(raw) == 24 + 4 * 3 * 4
    back = np.concatenate([np.frombuffer(open(p, "rb").read()[24:], np.float32) for p in paths])
    np.testing.assert_array_equal(back.reshape(10, 3), x)
    assert shards.list_shards(str(tmp_path)) == sorted(paths)
    empty = tmp_path / "sub"
    empty.mkdir()
    with pytest.raises(RuntimeError, match="no .shard files"):
        shards.list_shards(str(empty))
