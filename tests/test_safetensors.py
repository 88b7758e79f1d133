"""safetensors input (SPEC acceptance criterion 11; host parser, outside the GPU path):
an independently written container loads value-exact; corrupt containers raise
SafetensorsError (reference load_pipeline.py:643-716)."""

from __future__ import annotations

import json
import struct

import numpy as np
import pytest

import paper_2605_23066_b200 as tv
from paper_2605_23066_b200.errors import SafetensorsError

ST = {np.dtype("float32"): "F32", np.dtype("float64"): "F64", np.dtype("int64"): "I64",
      np.dtype("int32"): "I32", np.dtype("uint8"): "U8", np.dtype("bool"): "BOOL"}


def _write(path, tensors, bf16=()):
    header, blobs, off = {}, [], 0
    for name, arr in tensors.items():
        raw = np.ascontiguousarray(arr).tobytes()
        dt = "BF16" if name in bf16 else ST[arr.dtype]
        header[name] = {"dtype": dt, "shape": list(arr.shape), "data_offsets": [off, off + len(raw)]}
        blobs.append(raw)
        off += len(raw)
    head = json.dumps(header).encode()
    path.write_bytes(struct.pack("<Q", len(head)) + head + b"".join(blobs))
    return path


def test_safetensors_round_trip_and_corruption(tmp_path):
    rng = np.random.default_rng(11)
    tensors = {
        "embed": rng.standard_normal((16, 8)).astype(np.float32),
        "head.bias": rng.standard_normal(8),
        "steps": np.array([1, 2, 3], np.int64),
        "mask": rng.integers(0, 2, (4, 4)).astype(bool),
        "bytes": rng.integers(0, 256, 32).astype(np.uint8),
        "w_bf16": rng.integers(0, 1 << 16, (4, 6)).astype(np.uint16),
    }
    path = _write(tmp_path / "model.safetensors", tensors, bf16=("w_bf16",))
    tree = tv.load_safetensors(str(path))
    assert set(tree) == set(tensors)
    for name, arr in tensors.items():
        assert tree[name].to_numpy().tobytes() == np.ascontiguousarray(arr).tobytes(), name
        assert tree[name].shape == arr.shape
    assert tree["w_bf16"].dtype == "bf16"
    raw = path.read_bytes()
    (tmp_path / "trunc.safetensors").write_bytes(raw[:-16])
    with pytest.raises(SafetensorsError):
        tv.load_safetensors(str(tmp_path / "trunc.safetensors"))
    head = b'{"oops": '
    (tmp_path / "bad.safetensors").write_bytes(struct.pack("<Q", len(head)) + head)
    with pytest.raises(SafetensorsError):
        tv.load_safetensors(str(tmp_path / "bad.safetensors"))
    hdr = {"a": {"dtype": "F32", "shape": [2], "data_offsets": [0, 8]},
           "b": {"dtype": "F32", "shape": [2], "data_offsets": [4, 12]}}
    h = json.dumps(hdr).encode()
    (tmp_path / "overlap.safetensors").write_bytes(struct.pack("<Q", len(h)) + h + b"\0" * 12)
    with pytest.raises(SafetensorsError):
        tv.load_safetensors(str(tmp_path / "overlap.safetensors"))
