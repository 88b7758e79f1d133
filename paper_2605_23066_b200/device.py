"""Placing host arrays onto the runtime's GPUs as sharded device arrays.

The reference's leaves are global host arrays; a training job on B200 holds per-device
shards.  ``device_put`` builds that state from a host array (tests, benchmarks, users
migrating from the reference), one H2D copy per addressable mesh device.
"""

from __future__ import annotations

from typing import Any, Mapping

import numpy as np

from . import treemodel
from .dtypes import torch_dtype
from .sharding import Sharding, shards_of
from .treemodel import DenseArray, ShardedArray


def _upload(host: np.ndarray, dtype: str, gpu: int):
    import torch

    host = np.ascontiguousarray(host)
    t = torch.empty(host.shape, dtype=torch_dtype(dtype), device=torch.device("cuda", gpu))
    if host.size:
        src = torch.from_numpy(host.reshape(-1).view(np.uint8))
        t.view(-1).view(torch.uint8).copy_(src)
    return t


def device_put(value: Any, sharding: Sharding | None, runtime, dtype: str | None = None):
    """Host array (numpy or DenseArray) -> ShardedArray on the runtime's GPUs (only the
    devices of addressable processes), or a device DenseArray when ``sharding`` is None
    (placed on process 0's GPU)."""
    if isinstance(value, DenseArray):
        dtype = dtype or value.dtype
        host = value.to_numpy()
    else:
        arr = DenseArray(dtype, value) if dtype else DenseArray.from_numpy(np.asarray(value))
        dtype, host = arr.dtype, arr.data
    if sharding is None:
        gpu = runtime.gpu_of_process(runtime.addressable_processes[0])
        return DenseArray(dtype, _upload(host, dtype, gpu))
    owned = set(runtime.addressable_processes)
    shards = {}
    for s in shards_of(sharding):
        if sharding.mesh.process_of(s.device) not in owned:
            continue
        sel = tuple(slice(o, o + e) for o, e in s.ranges)
        shards[s.device] = _upload(host[sel], dtype, runtime.gpu_of_device(s.device))
    return ShardedArray(dtype, sharding, shards)


def device_put_tree(tree: Any, shardings: Mapping[str, Sharding] | None, runtime):
    """Every array leaf of ``tree`` placed by ``device_put`` with its path's sharding."""
    shardings = dict(shardings or {})
    pairs = []
    for path, leaf in treemodel.flatten(treemodel.as_tree(tree)):
        if isinstance(leaf, DenseArray):
            leaf = device_put(leaf, shardings.get(path), runtime)
        pairs.append((path, leaf))
    structure = treemodel.tree_metadata(treemodel.as_tree(tree))
    return treemodel.unflatten(pairs, structure)
