"""Drop-in conformance on the GPU box: the reference's own test suite (unmodified,
staged in oracle/_ref/tests by oracle/ref_recipe.py) run against this package imported
as ``treevault`` (tools/conformance.py).  In scope: everything but test_cli.py (the CLI
is out of scope and not built); the one known divergence is BF16 support in
load_safetensors (the reference rejects BF16; this build's north-star tree is bf16)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
KNOWN = {"tests.test_load_pipeline.TestSafetensors::test_unsupported_dtype_rejected"}


def test_reference_suite_passes_against_this_package(tmp_path):
    if not (ROOT / "oracle" / "_ref" / "tests").is_dir():
        pytest.skip("oracle/_ref not staged (run __graft_entry__.build() in the build container)")
    out = tmp_path / "conf"
    subprocess.run([sys.executable, str(ROOT / "tools" / "conformance.py"), "--out", str(out)],
                   capture_output=True, text=True, timeout=1200, cwd=ROOT,
                   env=dict(os.environ, PYTHONPATH=str(ROOT)))
    summary = json.loads((tmp_path / "conf.json").read_text())
    failed = set(summary["not_passed"]) - {"::tests.test_cli (error)"}
    assert failed <= KNOWN, sorted(failed)[:20]
    assert summary["totals"]["passed"] >= 264, summary["totals"]
