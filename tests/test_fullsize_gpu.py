"""Full BASELINE size on one B200 (C2: Llama-3-8B bf16 params + fp32 Adam mu/nu, 873
leaves, 80,302,612,480 bytes): size-independent properties of the data path.

* async save → restore round trip: every restored shard is bit-identical to the saved
  state (compared on the device);
* stored bytes: every chunk file of the per-leaf layout is exactly the row-major bytes
  of its shard (checked for a spread of leaves: the largest fp32 and bf16 payloads, a
  norm, an MLP matrix), and the committed key set is exactly the expected one;
* the checkpoint's total payload = the tree's bytes (each element written once)."""

from __future__ import annotations

import os
import shutil

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c2_llama3_8b_round_trip_and_stored_bytes():
    import sys

    import torch

    sys.path.insert(0, ROOT)
    import bench
    import paper_2605_23066_b200 as tv

    from paper_2605_23066_b200 import native

    native.release_pool()      # engines (and their device staging) left by earlier tests
    torch.cuda.empty_cache()   # blocks cached by earlier tests in this process
    free, total = torch.cuda.mem_get_info(0)
    if free < 2.03 * bench.TREE_BYTES_C2:
        pytest.skip(f"needs ~170 GB of free HBM (state + snapshot arena), have {free / 1e9:.0f} GB")
    base = "/dev/shm/tv_fullsize_test"
    shutil.rmtree(base, ignore_errors=True)
    try:
        backend = tv.FilesystemBackend(base)
        rt = tv.SimulatedRuntime(1, backend, gpus=[0])
        leaves = bench.llama_leaves(**bench.LLAMA3_8B)
        mesh = tv.Mesh.create([("fsdp", 1)], process_count=1)
        state, shardings = bench.build_state(tv, rt, mesh, leaves)
        tree_bytes = sum(bench.nbytes(s, dt) for _, _, s, dt in leaves)
        assert tree_bytes == bench.TREE_BYTES_C2 and len(leaves) == 873
        tv.save_checkpoint(rt, "ck", state, shardings, tv.SaveOptions(sync=False)).wait()

        # stored layout: one chunk file per leaf (FSDP-1: the shard is the write chunk)
        root = os.path.join(base, "ck", "process_0", "state")
        files = {}
        for dirpath, _, names in os.walk(root):
            for n in names:
                files[os.path.relpath(os.path.join(dirpath, n), root)] = os.path.getsize(os.path.join(dirpath, n))
        expect = {f"{t}/{p}/c.0.0" if len(s) == 2 else f"{t}/{p}/c.0": bench.nbytes(s, dt)
                  for t, p, s, dt in leaves}
        assert files == expect
        assert sum(files.values()) == tree_bytes

        flat = dict(tv.flatten(state["state"]))
        for t, p in (("mu", "embed"), ("params", "lm_head"), ("nu", "layers/31/mlp/down"),
                     ("params", "layers/0/attn/k"), ("mu", "final_norm")):
            leaf = flat[f"{t}/{p}"]
            shard = leaf.shards[0]
            key = f"{t}/{p}/c.0.0" if shard.dim() == 2 else f"{t}/{p}/c.0"
            with open(os.path.join(root, key), "rb") as f:
                on_disk = np.frombuffer(f.read(), np.uint8)
            ints = {2: torch.int16, 4: torch.int32}[shard.element_size()]
            host = shard.view(ints).cpu().numpy().view(np.uint8).reshape(-1)
            assert np.array_equal(on_disk, host), f"stored bytes of {t}/{p}"

        out = tv.load_checkpoint(rt, "ck", None, tv.LoadOptions(), current_mesh=mesh)
        nbytes, bad = bench.verify_restore(tv, state, out)
        assert nbytes == tree_bytes and bad == 0
        del out
    finally:
        shutil.rmtree(base, ignore_errors=True)
        torch.cuda.empty_cache()
