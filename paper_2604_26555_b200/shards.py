"""FSOMSHRD shard files (dataset.hpp:171-344), host side.

Format (dataset.hpp:171-183): 8-byte magic ``FSOMSHRD``, u32 version (1), u64
row count, u32 column count, then rows x cols little-endian float32, row-major.
``open_shards`` takes every ``*.shard`` file in a directory sorted by name
(dataset.hpp:277-301).  The engine reads the files itself
(:meth:`Engine.bind_shards`); these helpers only write and list them.
"""
from __future__ import annotations

import os
import struct

import numpy as np

MAGIC = b"FSOMSHRD"
VERSION = 1
HEADER = struct.Struct("<8sIQI")  # 24 bytes


def write_one_shard(path: str, rows: np.ndarray) -> None:
    """detail::write_one_shard (dataset.hpp:235-250)."""
    rows = np.ascontiguousarray(rows, np.float32)
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, VERSION, rows.shape[0], rows.shape[1]))
        rows.tofile(f)  # no host copy of the rows


def write_shards(data: np.ndarray, out_dir: str, n_shards: int) -> list[str]:
    """write_shards (dataset.hpp:252-275): contiguous near-equal row blocks,
    one ``part-NNNNN.shard`` per block."""
    if n_shards < 1:
        raise ValueError("write_shards: n_shards must be >= 1")
    os.makedirs(out_dir, exist_ok=True)
    base, extra = divmod(data.shape[0], n_shards)
    paths, row = [], 0
    for s in range(n_shards):
        cnt = base + (1 if s < extra else 0)
        p = os.path.join(out_dir, f"part-{s:05d}.shard")
        write_one_shard(p, data[row:row + cnt])
        paths.append(p)
        row += cnt
    return paths


def list_shards(directory: str) -> list[str]:
    """The file order open_shards uses (dataset.hpp:277-301)."""
    paths = sorted(os.path.join(directory, e) for e in os.listdir(directory)
                   if e.endswith(".shard"))
    if not paths:
        raise RuntimeError(f"no .shard files in {directory}")
    return paths
