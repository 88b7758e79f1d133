"""Drop-in conformance: the reference's OWN test suite run against this package.

    python tools/conformance.py [--out profiles/r02_conformance] [pytest args...]

The unmodified suite (``/root/reference/pkg/tests``, staged into the git-ignored
``oracle/_ref/tests`` by ``oracle/ref_recipe.py``) is copied to a scratch directory and
run with ``import treevault`` resolving to ``paper_2605_23066_b200`` (every submodule
aliased), with the reference-compatible load defaults (``reference_defaults()``: host
numpy results, the reference's per-process reads).  Array bytes move through libtvgpu on
the GPU, so this runs on the B200 box.  Writes ``<out>.log`` (pytest output),
``<out>.xml`` (junit) and ``<out>.json`` (per-file pass / fail / error counts).
"""

from __future__ import annotations

import importlib
import json
import os
import shutil
import sys
import tempfile
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUBMODULES = ("backend", "chunkstore", "coordination", "docio", "dtypes", "errors", "load_pipeline",
              "save_pipeline", "sharding", "training_manager", "treemodel")


def alias_package() -> None:
    sys.path.insert(0, ROOT)
    import paper_2605_23066_b200 as pkg

    pkg.reference_defaults(True)
    sys.modules["treevault"] = pkg
    for name in SUBMODULES:
        sys.modules[f"treevault.{name}"] = importlib.import_module(f"paper_2605_23066_b200.{name}")


def summarize(xml_path: str) -> dict:
    per_file: dict[str, dict[str, int]] = {}
    failures = []
    for case in ET.parse(xml_path).getroot().iter("testcase"):
        f = (case.get("classname") or "?").split(".")[0]
        rec = per_file.setdefault(f, {"passed": 0, "failed": 0, "error": 0, "skipped": 0})
        kids = {c.tag for c in case}
        if "failure" in kids:
            rec["failed"] += 1
            failures.append(f"{case.get('classname')}::{case.get('name')}")
        elif "error" in kids:
            rec["error"] += 1
            failures.append(f"{case.get('classname')}::{case.get('name')} (error)")
        elif "skipped" in kids:
            rec["skipped"] += 1
        else:
            rec["passed"] += 1
    tot = {k: sum(r[k] for r in per_file.values()) for k in ("passed", "failed", "error", "skipped")}
    ran = tot["passed"] + tot["failed"] + tot["error"]
    return {"totals": tot, "pass_rate": round(tot["passed"] / max(1, ran), 4), "per_file": per_file,
            "not_passed": failures}


def main(argv: list[str]) -> int:
    out = os.path.join(ROOT, "profiles", "conformance")
    if "--out" in argv:
        i = argv.index("--out")
        out = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    src = os.path.join(ROOT, "oracle", "_ref", "tests")
    if not os.path.isdir(src):
        print("oracle/_ref/tests missing: run __graft_entry__.build() in the build container", file=sys.stderr)
        return 2
    alias_package()
    import pytest

    work = tempfile.mkdtemp(prefix="tv_conformance_")
    dst = os.path.join(work, "tests")
    shutil.copytree(src, dst, ignore=shutil.ignore_patterns("__pycache__"))
    xml = out + ".xml"
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    log = open(out + ".log", "w")
    old_out, old_err = sys.stdout, sys.stderr
    sys.stdout = sys.stderr = log
    try:
        rc = pytest.main([dst, "-q", "-rfE", "-p", "no:cacheprovider", f"--junitxml={xml}",
                          "--continue-on-collection-errors",
                          "--rootdir", work, "-o", "junit_family=xunit1", *argv])
    finally:
        sys.stdout, sys.stderr = old_out, old_err
        log.close()
    summary = summarize(xml)
    summary["how"] = ("the reference's pkg/tests, unmodified, with `treevault` aliased to "
                      "paper_2605_23066_b200 (reference_defaults: host results, per-process reads)")
    with open(out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: summary[k] for k in ("totals", "pass_rate")}))
    shutil.rmtree(work, ignore_errors=True)
    return int(rc)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
