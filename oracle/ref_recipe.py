"""Recipe: stage the UNMODIFIED reference (treevault, pure Python + numpy) into the
git-ignored ``oracle/_ref/`` so it travels to the GPU box with the snapshot.

Test / measurement infrastructure only (like the rest of ``oracle/``): the reference is
the checker and the CPU baseline, never part of the product path.  ``/root/reference``
exists only in the build container; ``__graft_entry__.build()`` runs this recipe there,
and the GPU box uses the staged copy.

    oracle/_ref/treevault/   <- /root/reference/pkg/src/treevault   (the package, as is)
    oracle/_ref/tests/       <- /root/reference/pkg/tests           (its own test suite)
    oracle/_ref/STAMP.json   <- file list + sha256 of every staged file

Nothing is edited: the bf16 shim the reference arm needs (the reference's
dtype table has no bf16, so it is registered as its 2-byte bit pattern "<u2") is applied
at import time by ``load_reference()``, not written into the copy.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"
SOURCES = {
    "treevault": Path("/root/reference/pkg/src/treevault"),
    "tests": Path("/root/reference/pkg/tests"),
}


def _digest(root: Path) -> dict[str, str]:
    out = {}
    for p in sorted(root.rglob("*.py")):
        out[str(p.relative_to(REF))] = hashlib.sha256(p.read_bytes()).hexdigest()
    return out


def stage(force: bool = False) -> Path | None:
    """Copy the reference package and tests into oracle/_ref (no-op when the reference is
    absent, e.g. on the GPU box, or already staged from the same sources)."""
    if not all(src.exists() for src in SOURCES.values()):
        return REF if (REF / "treevault").exists() else None
    stamp = REF / "STAMP.json"
    if stamp.exists() and not force:
        old = json.loads(stamp.read_text())
        if old.get("sources") == {k: str(v) for k, v in SOURCES.items()} and all(
            (REF / rel).exists() for rel in old.get("files", {})
        ):
            src_now = {}
            for name, src in SOURCES.items():
                for p in sorted(src.rglob("*.py")):
                    src_now[f"{name}/{p.relative_to(src)}"] = hashlib.sha256(p.read_bytes()).hexdigest()
            if src_now == old["files"]:
                return REF
    tmp = REF.with_name("_ref.tmp")
    shutil.rmtree(tmp, ignore_errors=True)
    tmp.mkdir(parents=True)
    for name, src in SOURCES.items():
        shutil.copytree(src, tmp / name, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    shutil.rmtree(REF, ignore_errors=True)
    os.replace(tmp, REF)
    (REF / "STAMP.json").write_text(json.dumps(
        {"sources": {k: str(v) for k, v in SOURCES.items()}, "files": _digest(REF)}, indent=1, sort_keys=True))
    return REF


def available() -> bool:
    return (REF / "treevault" / "__init__.py").exists()


def load_reference():
    """Import the staged reference package as ``treevault`` (with the bf16 shim)."""
    if not available():
        raise RuntimeError("oracle/_ref is not staged: run __graft_entry__.build() in the build container")
    import numpy as np

    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import treevault
    import treevault.dtypes

    treevault.dtypes.NUMPY_DTYPES["bf16"] = np.dtype("<u2")
    return treevault


if __name__ == "__main__":
    print(stage(force="--force" in sys.argv))
