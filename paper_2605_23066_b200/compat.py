"""Reference-compatible defaults (the drop-in switch for reference-era callers).

``TREEVAULT_COMPAT=1`` in the environment, or ``reference_defaults(True)``, makes the
package behave like the reference where this build's defaults differ for speed:

* ``LoadOptions()`` returns global host numpy arrays (``to_host=True``) and reads
  exactly the reference's per-process chunk ranges (``read_once=False``);
* ``ChunkReader.read_range`` returns a host numpy array (the reference's type,
  ``chunkstore.py:507-593``) instead of a CUDA tensor.

Off by default: a training job wants device shards and read-once restores.
"""

from __future__ import annotations

import os

_ON = [os.environ.get("TREEVAULT_COMPAT", "0") == "1"]


def reference_defaults(on: bool = True) -> None:
    _ON[0] = bool(on)


def enabled() -> bool:
    return _ON[0]
