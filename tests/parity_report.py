"""Parity report writer shared by the GPU parity tests.

When the environment variable ``PSCA_PARITY_REPORT`` names a file, the tests
merge what they measured into that JSON document (per config: max relative
error against the reference, the map-ur tolerance floors, min |score - theta|,
every instance whose bar exceeded 1e-9).  profiles/r02_parity.json is one such
report from a B200 run.  Without the variable nothing is written.
"""

from __future__ import annotations

import json
import os
import pathlib


def record(section: str, key: str, value) -> None:
    path = os.environ.get("PSCA_PARITY_REPORT")
    if not path:
        return
    p = pathlib.Path(path)
    doc = json.loads(p.read_text()) if p.exists() else {}
    doc.setdefault(section, {})[key] = value
    p.parent.mkdir(parents=True, exist_ok=True)
    p.write_text(json.dumps(doc, indent=1, sort_keys=True))
