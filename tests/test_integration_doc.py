"""INTEGRATION.md's ctypes binding (what a reference maintainer would paste) declares
every function with the arity include/tvgpu.h gives it, and its STATS dtype has the
header's tv_stats fields in order (CPU)."""

from __future__ import annotations

import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _prototypes() -> dict[str, int]:
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "tvgpu.h").read_text(), flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:int|int64_t)\s+(tv_\w+)\s*\(([^)]*)\)\s*;", text):
        params = m.group(2).strip()
        out[m.group(1)] = 0 if params in ("", "void") else len(params.split(","))
    return out


def test_ctypes_stub_matches_header_arity():
    protos = _prototypes()
    doc = (ROOT / "INTEGRATION.md").read_text()
    stubs = re.findall(r"_lib\.(tv_\w+)\.argtypes\s*=\s*\[([^\]]*)\]", doc)
    assert stubs, "no ctypes stub in INTEGRATION.md"
    for name, args in stubs:
        assert name in protos, name
        # split on top-level commas (ctypes.POINTER(x) holds none)
        n = len([a for a in args.split(",") if a.strip()])
        assert n == protos[name], (name, n, protos[name])


def test_stats_dtype_matches_tv_stats():
    header = (ROOT / "include" / "tvgpu.h").read_text()
    body = re.search(r"typedef struct tv_stats \{(.*?)\} tv_stats;", header, flags=re.S).group(1)
    fields = re.findall(r"(?:int64_t|double)\s+(\w+);", body)
    doc = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"STATS = np\.dtype\((.*?)align=True\)", doc, flags=re.S).group(1)
    names = re.findall(r'"(\w+)"', block)
    names = [n for n in names if n not in ("<i8", "<f8")]
    assert names == fields
