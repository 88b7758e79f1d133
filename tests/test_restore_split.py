"""Restore fetch splitting (host logic, CPU): a stored chunk larger than the device
staging budget, or one that lands contiguously in no target shard, is fetched as
contiguous leading-dimension slabs.  Checked by replaying the pieces against numpy:
each piece's byte range of the stored chunk must be exactly the row-major bytes of its
box, pieces never overlap, and every element some target needs is read exactly once.

Reference behaviour being preserved: ``chunkstore.py:507-593`` assembles any target box
from whole chunks on the host (no size ceiling)."""

from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

from paper_2605_23066_b200 import chunkstore as cs


def _grid_boxes(shape, splits):
    """Target boxes of a grid sharding: dim d split into splits[d] equal parts."""
    per_dim = []
    for g, n in zip(shape, splits):
        step = g // n
        per_dim.append([(i * step, step) for i in range(n)])
    return tuple(itertools.product(*per_dim))


def _replay(shape, w, isz, boxes, max_bytes):
    """Replay the split geometry of a whole-chunk grid; returns (pieces, read mask)."""
    geometry = cs.fetch_geometry(w, w, isz, boxes)
    pieces = cs.split_geometry(geometry, boxes, max_bytes)
    glob = np.arange(math.prod(shape), dtype=np.int64).reshape(shape)
    read = np.zeros(shape, np.int32)
    per_chunk: dict = {}
    for coords, ck, rel, nbytes, origin, pshape, whole, obj in pieces:
        chunk_origin = tuple(c * wi for c, wi in zip(coords, w))
        chunk = glob[tuple(slice(o, o + e) for o, e in zip(chunk_origin, w))]
        raw = np.ascontiguousarray(chunk).view(np.uint8).reshape(-1)
        # isz = 8 (int64 values) in this replay regardless of the planned itemsize
        scale = 8 // isz
        got = raw[rel * scale:(rel + nbytes) * scale].view(np.int64).reshape(pshape)
        want = glob[tuple(slice(o, o + e) for o, e in zip(origin, pshape))]
        assert np.array_equal(got, want), (coords, rel, origin, pshape)
        read[tuple(slice(o, o + e) for o, e in zip(origin, pshape))] += 1
        assert obj == math.prod(w) * isz
        per_chunk.setdefault(ck, []).append((rel, nbytes))
    for spans in per_chunk.values():   # no two pieces of a chunk overlap
        spans.sort()
        for (a, n), (b, _) in zip(spans, spans[1:]):
            assert a + n <= b
    need = np.zeros(shape, bool)
    for box in boxes:
        need[tuple(slice(o, o + e) for o, e in box)] = True
    assert np.array_equal(read[need], np.ones(need.sum(), np.int32))  # needed: read once
    return pieces, read


def test_up_scaling_pieces_land_directly():
    """FSDP-1 chunk restored onto FSDP-4: cut at the targets' row boundaries, each piece
    one contiguous run of exactly one target (direct H2D), nothing staged."""
    shape, w = (64, 16), (64, 16)
    boxes = _grid_boxes(shape, (4, 1))
    pieces, _ = _replay(shape, w, 8, boxes, max_bytes=1 << 30)
    assert [p[4] for p in pieces] == [(0, 0), (16, 0), (32, 0), (48, 0)]
    assert all(p[3] == 16 * 16 * 8 and not p[6] for p in pieces)
    index = cs.BoxIndex(boxes)
    for p in pieces:
        box = tuple(zip(p[4], p[5]))
        assert any(cs._lands_contiguously(box, boxes[i]) for i in index.hits(box))


def test_column_reshard_is_capped_by_budget():
    """(None, 'tp'): no row cut helps; slabs of at most the budget, scattered by the
    unpack kernel into both column halves."""
    shape, w = (64, 16), (64, 16)
    boxes = _grid_boxes(shape, (1, 2))
    budget = 10 * 16 * 8  # 10 rows
    pieces, _ = _replay(shape, w, 8, boxes, max_bytes=budget)
    assert all(p[3] <= budget for p in pieces)
    assert sum(p[3] for p in pieces) == 64 * 16 * 8
    assert len(pieces) == 7


def test_replicated_direct_consumer_keeps_chunk_whole():
    """A chunk some target holds contiguously (replicas of a row shard) stays one fetch
    even above the budget: it lands directly, the replica copy comes from HBM."""
    shape, w = (32, 8), (16, 8)
    boxes = ((( 0, 16), (0, 8)), ((0, 16), (0, 8)), ((16, 16), (0, 8)), ((16, 16), (0, 8)))
    pieces, _ = _replay(shape, w, 8, boxes, max_bytes=64)
    assert len(pieces) == 2 and all(p[6] for p in pieces)


def test_single_row_larger_than_budget_descends():
    shape, w = (2, 1024), (2, 1024)
    boxes = _grid_boxes(shape, (1, 4))
    pieces, _ = _replay(shape, w, 8, boxes, max_bytes=1000)
    assert all(p[3] <= 1000 for p in pieces)
    assert all(p[5][0] == 1 for p in pieces)


@pytest.mark.parametrize("src,dst", [((1, 1), (4, 1)), ((2, 1), (8, 1)), ((1, 1), (1, 4)),
                                     ((4, 1), (2, 2)), ((1, 1), (3, 1)), ((2, 2), (3, 2))])
def test_random_grids_read_each_needed_element_once(src, dst):
    shape = (48, 24)
    w = (shape[0] // src[0], shape[1] // src[1])
    boxes = _grid_boxes(shape, dst)
    for budget in (64, 1000, 1 << 30):
        _replay(shape, w, 8, boxes, budget)


def test_partial_target_does_not_read_unneeded_rows():
    """A target covering part of a chunk: rows nobody needs are not fetched."""
    shape, w = (64, 8), (64, 8)
    boxes = (((8, 16), (0, 8)),)
    pieces, read = _replay(shape, w, 8, boxes, max_bytes=1 << 30)
    assert sum(p[3] for p in pieces) == 16 * 8 * 8
    assert read.sum() == 16 * 8


def test_split_fetch_guard():
    f = cs.Fetch("k", "get", 0, 40 * 4 * 4, (0, 0), (40, 4), True, 40 * 4 * 4)
    parts = cs.split_fetch(f, 100)
    assert all(p.nbytes <= 100 and p.op == "get_range" and not p.whole_file for p in parts)
    assert sum(p.nbytes for p in parts) == f.nbytes
    assert all(p.object_bytes == f.object_bytes for p in parts)
    offs = [p.file_off for p in parts]
    assert offs == sorted(offs) and offs[0] == 0
    assert cs.split_fetch(f, f.nbytes) == [f]
