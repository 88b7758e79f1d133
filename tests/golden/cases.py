"""Parity cases shared by tests/golden/gen_golden.py (runs the real reference) and the
tests (run the oracle and the GPU path).  Pure numpy + plain Python: no reference and no
product imports, so the same seeded inputs can be rebuilt anywhere.

Tree notation (neutral):
  ("array", dtype, np.ndarray)   dense array (bf16 as uint16 bit patterns)
  ("scalar", dtype, value)       inline scalar
  ("text", str)                  inline text
  dict / list / tuple            containers
Top-level checkpointables: name -> tree | ("json", obj) | ("stateful", index)

Sharding notation: leaf path -> (axes, process_count, replica_axis, spec).
"""

from __future__ import annotations

import numpy as np

NP = {
    "f32": np.dtype("<f4"),
    "f64": np.dtype("<f8"),
    "i32": np.dtype("<i4"),
    "i64": np.dtype("<i8"),
    "u8": np.dtype("|u1"),
    "bool": np.dtype("|b1"),
    "bf16": np.dtype("<u2"),
}


def arr(rng: np.random.Generator, dtype: str, shape) -> tuple:
    shape = tuple(shape)
    if dtype in ("f32", "f64"):
        data = rng.standard_normal(shape).astype(NP[dtype])
    elif dtype == "bf16":
        f = (rng.standard_normal(shape) * 0.02).astype(np.float32)
        bits = f.view(np.uint32).astype(np.uint64)
        data = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16).astype(np.uint16)
    elif dtype == "bool":
        data = rng.integers(0, 2, shape).astype(bool)
    elif dtype == "u8":
        data = rng.integers(0, 256, shape).astype(np.uint8)
    else:
        data = rng.integers(-1000, 1000, shape).astype(NP[dtype])
    return ("array", dtype, np.ascontiguousarray(data))


def llama_like(rng, layers: int, d: int, ffn: int, vocab: int, kv: int) -> dict:
    """Llama-shaped state: bf16 params + f32 Adam mu/nu (SURVEY §8(d) C2 shapes, scaled)."""

    def block(dtype):
        out = {
            "embed": arr(rng, dtype, (vocab, d)),
            "lm_head": arr(rng, dtype, (vocab, d)),
            "final_norm": arr(rng, dtype, (d,)),
            "layers": {},
        }
        for i in range(layers):
            out["layers"][str(i)] = {
                "attn": {
                    "q": arr(rng, dtype, (d, d)),
                    "k": arr(rng, dtype, (kv, d)),
                    "v": arr(rng, dtype, (kv, d)),
                    "o": arr(rng, dtype, (d, d)),
                },
                "mlp": {
                    "gate": arr(rng, dtype, (ffn, d)),
                    "up": arr(rng, dtype, (ffn, d)),
                    "down": arr(rng, dtype, (d, ffn)),
                },
                "norm_in": arr(rng, dtype, (d,)),
                "norm_post": arr(rng, dtype, (d,)),
            }
        return out

    return {"params": block("bf16"), "mu": block("f32"), "nu": block("f32")}


def leaf_paths(tree, prefix=""):
    if isinstance(tree, tuple) and tree and tree[0] in ("array", "scalar", "text"):
        yield prefix, tree
        return
    if isinstance(tree, dict):
        for k in sorted(tree):
            yield from leaf_paths(tree[k], f"{prefix}/{k}" if prefix else k)
    else:
        for i, c in enumerate(tree):
            yield from leaf_paths(c, f"{prefix}/{i}" if prefix else str(i))


def fsdp_shardings(tree, axes, process_count, replica_axis=None, axis="fsdp"):
    out = {}
    for path, leaf in leaf_paths(tree):
        if leaf[0] != "array":
            continue
        out[path] = (axes, process_count, replica_axis, (axis,) + (None,) * (leaf[2].ndim - 1))
    return out


def _c1(rng):
    return {"model": {f"a{i}": arr(rng, "f32", (64, 64)) for i in range(4)}}


def _mixed(rng):
    return {
        "model": {
            "w": arr(rng, "f32", (8, 6)),
            "b": arr(rng, "f64", (8,)),
            "mask": arr(rng, "bool", (4, 3)),
            "bytes": arr(rng, "u8", (5,)),
            "ids": arr(rng, "i64", (2, 3, 4)),
            "i32": arr(rng, "i32", (8, 2)),
            "zero_d": arr(rng, "f32", ()),
            "step": ("scalar", "i64", 7),
            "lr": ("scalar", "f64", 0.25),
            "nan": ("scalar", "f32", float("nan")),
            "tag": ("text", "ünïcode ✓"),
            "empty": {},
            "seq": [arr(rng, "f32", (4,)), ("scalar", "bool", True)],
            "tup": (("text", "x"), arr(rng, "i32", (3,))),
        },
        "config": ("json", {"name": "run", "n": 3, "nested": {"a": [1, 2]}}),
        "iterator": ("stateful", 42),
    }


def _case(name, build, shard_fn, options, P, backend, loads=(), seed=0):
    return {
        "name": name,
        "build": build,
        "shardings": shard_fn,
        "options": options,
        "process_count": P,
        "backend": backend,   # "fs" (rename) | "mem" (indicator) | "mem+rename"
        "loads": list(loads),
        "seed": seed,
    }


def _mesh2(rng_tree, P=4):
    return {"model": fsdp_shardings(rng_tree["model"], [("replica", 2), ("fsdp", 2)], P, "replica")}


def _rp_tree(rng):
    return {"model": llama_like(rng, layers=1, d=32, ffn=48, vocab=40, kv=8)}


def _xy(rng):
    return {"m": {"w": arr(rng, "f32", (16, 8)), "v": arr(rng, "i32", (8, 8, 4))}}


def _xy_shardings(tree):
    return {"m": {
        "w": ([("x", 4), ("y", 2)], 2, None, ("x", "y")),
        "v": ([("x", 4), ("y", 2)], 2, None, ("y", None, "x")),
    }}


CASES = [
    _case("c1_per_leaf", _c1, lambda t: {}, {}, 1, "fs",
          loads=[{"mesh": None}]),
    _case("c1_aggregated", _c1, lambda t: {}, {"layout": "aggregated", "target_file_bytes": 40000},
          1, "fs", loads=[{"mesh": None}]),
    _case("mixed_indicator", _mixed,
          lambda t: {"model": {"w": ([("data", 2)], 2, None, ("data", None)),
                               "i32": ([("data", 2)], 2, None, ("data", None))}},
          {}, 2, "mem", loads=[{"mesh": "saved"}]),
    _case("mixed_rename_agg", _mixed,
          lambda t: {"model": {"w": ([("data", 2)], 2, None, ("data", None))}},
          {"layout": "aggregated", "target_file_bytes": 64}, 2, "mem+rename",
          loads=[{"mesh": "saved"}]),
    _case("fsdp4_per_leaf",
          lambda r: {"state": llama_like(r, layers=2, d=32, ffn=48, vocab=40, kv=8)},
          lambda t: {"state": fsdp_shardings(t["state"], [("fsdp", 4)], 4)},
          {}, 4, "fs",
          loads=[
              {"mesh": "saved"},
              {"mesh": {"axes": [("replica", 2), ("fsdp", 2)], "P": 4, "replica_axis": "replica",
                        "axis": "fsdp"}, "read_once": False},
              {"mesh": {"axes": [("fsdp", 2)], "P": 2, "replica_axis": None, "axis": "fsdp"},
               "read_once": False},
          ]),
    _case("fsdp4_aggregated",
          lambda r: {"state": llama_like(r, layers=2, d=32, ffn=48, vocab=40, kv=8)},
          lambda t: {"state": fsdp_shardings(t["state"], [("fsdp", 4)], 4)},
          {"layout": "aggregated", "target_file_bytes": 8192}, 4, "fs",
          loads=[{"mesh": "saved"}]),
    _case("replica_parallel", _rp_tree, _mesh2, {"replica_parallel": True}, 4, "fs",
          loads=[{"mesh": "saved"},
                 {"mesh": "saved", "broadcast": True, "read_once": False}]),
    _case("single_slice", _rp_tree, _mesh2, {"replica_parallel": False}, 4, "fs",
          loads=[{"mesh": "saved", "read_once": False}]),
    _case("subchunk", _xy, _xy_shardings, {"subchunk_target_bytes": 32}, 2, "fs",
          loads=[{"mesh": "saved", "read_once": False},
                 {"mesh": {"axes": [("z", 8)], "P": 2, "replica_axis": None, "axis": "z"},
                  "read_once": False}]),
    _case("xy_2d", _xy, _xy_shardings, {"layout": "aggregated", "target_file_bytes": 100}, 2, "fs",
          loads=[{"mesh": "saved"}]),
]


def case(name: str) -> dict:
    for c in CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)


def build_inputs(c: dict):
    """(checkpointables, shardings) in neutral notation for case ``c``."""
    rng = np.random.default_rng(1000 + c["seed"])
    tree = c["build"](rng)
    return tree, c["shardings"](tree)


def target_spec(c: dict, load: dict, path: str, leaf) -> tuple | None:
    """Target sharding (neutral) of one array leaf for a load entry."""
    mesh = load["mesh"]
    if mesh is None:
        return None
    if mesh == "saved":
        return "saved"
    ndim = leaf[2].ndim
    if ndim == 0:
        return None
    return (mesh["axes"], mesh["P"], mesh["replica_axis"], (mesh["axis"],) + (None,) * (ndim - 1))


# -- load-time casts ----------------------------------------------------------------------

CAST_DTYPES = ["f32", "f64", "i32", "i64", "u8"]


def cast_input(src: str, dst: str, kind: str, seed: int = 0) -> np.ndarray:
    """Deterministic (64, 48) input for a cast src -> dst.  kind "ok" is castable by the
    reference; "overflow" / "nonfinite" / "nonintegral" trigger its checks."""
    rng = np.random.default_rng(7000 + seed + 31 * CAST_DTYPES.index(src) + CAST_DTYPES.index(dst))
    shape = (64, 48)
    int_dst = dst in ("i32", "i64", "u8")
    if src in ("f32", "f64"):
        if int_dst:
            lo, hi = (0, 255) if dst == "u8" else (-2**20, 2**20)
            x = rng.integers(lo, hi, shape).astype(NP[src])
            if kind == "overflow":
                x[3, 5] = 1e12 if dst != "i64" else 1e19
            elif kind == "nonfinite":
                x[7, 1] = np.inf
            elif kind == "nonintegral":
                x[2, 2] += 0.5
        else:
            x = (rng.standard_normal(shape) * 1e3).astype(NP[src])
            x[0, :4] = [1.0000001, -2.5e-39, 3.4e38, 65504.123]
    else:
        if int_dst:
            lo, hi = {"u8": (0, 256), "i32": (-2**31, 2**31), "i64": (-2**62, 2**62)}[src]
            dlo, dhi = {"u8": (0, 256), "i32": (-2**31, 2**31), "i64": (-2**62, 2**62)}[dst]
            x = rng.integers(max(lo, dlo), min(hi, dhi), shape).astype(NP[src])
            if kind == "overflow":
                x[4, 4] = hi - 1 if hi > dhi else lo
        else:
            lo, hi = {"u8": (0, 256), "i32": (-2**31, 2**31), "i64": (-2**62, 2**62)}[src]
            x = rng.integers(lo, hi, shape).astype(NP[src])
    return np.ascontiguousarray(x)


def cast_cases() -> list[tuple[str, str, str]]:
    out = []
    for s in CAST_DTYPES:
        for d in CAST_DTYPES:
            if s == d:
                continue
            out.append((s, d, "ok"))
            if d in ("i32", "i64", "u8"):
                if s in ("f32", "f64"):
                    out += [(s, d, "overflow"), (s, d, "nonfinite"), (s, d, "nonintegral")]
                elif (s, d) in (("i64", "i32"), ("i64", "u8"), ("i32", "u8")):
                    out.append((s, d, "overflow"))
    return out
