"""Element types: names, numpy storage types and torch device types.

The reference's table (``dtypes.py:14-21``) is {f32, f64, i32, i64, u8, bool}; this
build adds ``bf16`` because the north-star trees (Llama-3-8B params) are bf16.  On disk a
bf16 element is its 2-byte little-endian bit pattern, so its host (numpy) storage type is
``<u2`` — the same shim the oracle applies to the reference
(``NUMPY_DTYPES["bf16"] = np.dtype("<u2")``).  Chunk bytes never depend on
anything but the item size, so every dtype moves through the same byte kernels.
"""

from __future__ import annotations

import numpy as np

from .errors import TreeError

# name -> little-endian numpy storage dtype (host side, and on-disk byte order)
NUMPY_DTYPES: dict[str, np.dtype] = {
    "f32": np.dtype("<f4"),
    "f64": np.dtype("<f8"),
    "i32": np.dtype("<i4"),
    "i64": np.dtype("<i8"),
    "u8": np.dtype("|u1"),
    "bool": np.dtype("|b1"),
    "bf16": np.dtype("<u2"),
}

FLOAT_DTYPES = frozenset({"f32", "f64", "bf16"})
INT_DTYPES = frozenset({"i32", "i64", "u8"})
NUMERIC_DTYPES = FLOAT_DTYPES | INT_DTYPES

_TORCH_NAMES = {
    "f32": "float32",
    "f64": "float64",
    "i32": "int32",
    "i64": "int64",
    "u8": "uint8",
    "bool": "bool",
    "bf16": "bfloat16",
}


def numpy_dtype(name: str) -> np.dtype:
    dt = NUMPY_DTYPES.get(name)
    if dt is None:
        raise TreeError(f"unsupported dtype {name!r}")
    return dt


def itemsize(name: str) -> int:
    return numpy_dtype(name).itemsize


def dtype_name(dt) -> str:
    """Name of a numpy dtype (matched on kind and width, like the reference) or of a
    torch dtype."""
    torch_name = _torch_dtype_name(dt)
    if torch_name is not None:
        return torch_name
    dt = np.dtype(dt)
    if dt.name == "bfloat16":  # ml_dtypes.bfloat16
        return "bf16"
    for name, candidate in NUMPY_DTYPES.items():
        if candidate.kind == dt.kind and candidate.itemsize == dt.itemsize:
            return name
    raise TreeError(f"unsupported numpy dtype {dt!r}")


def torch_dtype(name: str):
    import torch

    numpy_dtype(name)  # validates the name
    return getattr(torch, _TORCH_NAMES[name])


def _torch_dtype_name(dt) -> str | None:
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is a hard dependency of the data path
        return None
    if not isinstance(dt, torch.dtype):
        return None
    for name, tname in _TORCH_NAMES.items():
        if getattr(torch, tname) == dt:
            return name
    raise TreeError(f"unsupported torch dtype {dt!r}")
