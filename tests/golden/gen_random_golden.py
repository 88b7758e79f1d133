"""Golden digests of the random save cases (random_cases.py) produced by the REAL
reference in the build container (bf16 through the documented "<u2" shim):

    python tests/golden/gen_random_golden.py     # rewrites tests/golden/random_cases.json

For each case: every stored key -> [length, sha256], and the payload bytes each process
reads when the reference restores it onto random_cases.restore_targets."""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import gen_golden  # noqa: E402
import random_cases  # noqa: E402


def main() -> None:
    tv = gen_golden._import_reference()
    out = {}
    for seed in range(random_cases.N_CASES):
        tree, specs, options, P, _ = random_cases.case(seed)
        leaves = dict(tree["m"])
        shardings = {"m": {p: gen_golden.sharding(tv, s, leaves[p][2].shape) for p, s in specs["m"].items()}}
        with tempfile.TemporaryDirectory() as tmp:
            backend = tv.FilesystemBackend(tmp)
            rt = tv.SimulatedRuntime(P, backend)
            opts = tv.SaveOptions(**options, sync=True)
            tv.save_checkpoint(rt, "ck/run", gen_golden.checkpointables(tv, tree), shardings, opts).wait()
            files = {k: [len(v), gen_golden.sha(v)] for k, v in sorted(backend.dump().items())}
            # restore onto another random sharding: per-process payload bytes the reference reads
            targets = random_cases.restore_targets(seed, tree, P)
            abstract = {"m": {name: tv.AbstractLeaf("array", leaf[2].shape, leaf[1],
                                                    gen_golden.sharding(tv, targets[name], leaf[2].shape))
                              for name, leaf in leaves.items()}}
            before = {i: backend.counters(i) for i in backend.identities()}
            loaded = tv.load_checkpoint(rt, "ck/run", abstract)
            for name, leaf in leaves.items():
                assert loaded["m"][name].data.tobytes() == leaf[2].tobytes(), (seed, name)
            reads = {}
            for ident in backend.identities():
                if not ident.startswith("process_"):
                    continue
                now, prev = backend.counters(ident), before.get(ident)
                reads[ident] = (now.minus(prev) if prev is not None else now).payload_bytes_read
            out[str(seed)] = {"files": files, "load_payload_bytes_read": reads}
    (HERE / "random_cases.json").write_text(json.dumps(out, indent=0, sort_keys=True) + "\n")
    print(f"{len(out)} cases")


if __name__ == "__main__":
    main()
