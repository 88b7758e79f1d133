"""Step management and retention (host logic; scalar/text trees never touch the GPU).

Mirrors the reference's tests/test_training_manager.py intent: monotonic steps,
retention enumeration vs an independent oracle, markers deleted first, failure
surfacing; plus this build's parallel bulk delete and background deletion.
"""

from __future__ import annotations

import random

import pytest

import paper_2605_23066_b200 as tv
from paper_2605_23066_b200.errors import GarbageCollectionError, StepError


def retained_oracle(steps, keep_last, keep_period=None):
    ordered = sorted(steps)
    keep = set(ordered[-keep_last:]) if ordered else set()
    if ordered:
        keep.add(ordered[-1])
    if keep_period:
        keep |= {s for s in ordered if s % keep_period == 0}
    return keep


def test_retention_matches_oracle():
    rng = random.Random(3)
    for _ in range(300):
        steps = rng.sample(range(100), rng.randint(0, 20))
        kl, kp = rng.randint(1, 5), rng.choice([None, 2, 3, 10])
        assert tv.RetentionPolicy(kl, kp).retained(steps) == retained_oracle(steps, kl, kp)
    with pytest.raises(StepError):
        tv.RetentionPolicy(keep_last=0)


def test_should_save():
    assert [s for s in range(21) if tv.should_save(s, 5)] == [0, 5, 10, 15, 20]
    with pytest.raises(StepError):
        tv.should_save(1, 0)


@pytest.mark.parametrize("backend_kind", ["mem", "fs"])
@pytest.mark.parametrize("background", [False, True])
def test_scalar_checkpointer_loop(backend_kind, background, tmp_path):
    backend = tv.MemoryBackend() if backend_kind == "mem" else tv.FilesystemBackend(tmp_path)
    rt = tv.SimulatedRuntime(2, backend)
    cp = tv.Checkpointer(rt, "root", tv.RetentionPolicy(keep_last=3),
                         tv.SaveOptions(sync=False), background_delete=background)
    for step in range(10):
        cp.save_step(step, {"m": tv.as_tree({"x": float(step), "tag": f"s{step}"})})
    cp.wait()
    cp.garbage_collect()  # joins any background deletion
    assert cp.all_steps() == [7, 8, 9]
    keys = backend.store().list_keys("root/")
    assert {k.split("/")[1] for k in keys} == {"step_00000007", "step_00000008", "step_00000009"}
    assert cp.load_step()["m"]["x"].value == 9.0
    with pytest.raises(StepError):
        cp.save_step(5, {"m": tv.as_tree({"x": 1.0})})


def test_delete_markers_first_and_bulk(tmp_path):
    backend = tv.FilesystemBackend(tmp_path)
    rt = tv.SimulatedRuntime(1, backend)
    cp = tv.Checkpointer(rt, "root", tv.RetentionPolicy(keep_last=1))
    for step in range(3):
        cp.save_step(step, {"m": tv.as_tree({"x": float(step), "y": {"z": step}})}, options=tv.SaveOptions(sync=True))
    deletes = [k for ident, kind, k in backend.trace() if kind == "delete"]
    first = [k for k in deletes if "step_00000000" in k]
    assert first[0].endswith("global_metadata.json")  # de-finalized before anything else
    assert not (tmp_path / "root" / "step_00000000").exists()  # directories pruned
    assert cp.all_steps() == [2]


def test_gc_failure_keeps_step_and_surfaces(tmp_path):
    backend = tv.MemoryBackend()
    rt = tv.SimulatedRuntime(1, backend)
    cp = tv.Checkpointer(rt, "root", tv.RetentionPolicy(keep_last=1), background_delete=True)
    cp.save_step(0, {"m": tv.as_tree({"x": 0.0})}, options=tv.SaveOptions(sync=True))
    backend.set_fault_plan(tv.FaultPlan(fail_delete_substring="step_00000000/m"))
    cp.save_step(1, {"m": tv.as_tree({"x": 1.0})})
    cp.wait()  # starts background deletion of step 0, which fails
    with pytest.raises(GarbageCollectionError):
        cp.wait()
    assert 0 in cp.all_steps()


def test_bulk_delete_records_ops_and_faults(tmp_path):
    backend = tv.FilesystemBackend(tmp_path)
    store = backend.store("x")
    keys = [f"a/b{i}/c.{j}" for i in range(5) for j in range(4)]
    for k in keys:
        store.put(k, b"12")
    store.delete_many(keys[:10])
    assert backend.counters("x").ops["delete"] == 10
    assert store.list_keys("a/") == sorted(keys[10:])
    backend.set_fault_plan(tv.FaultPlan(fail_delete_substring="b3/c.1"))
    with pytest.raises(tv.errors.InjectedFaultError):
        store.delete_many(keys[10:])
    assert store.list_keys("a/") == sorted(keys[keys.index("a/b3/c.1"):])
