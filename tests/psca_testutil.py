"""Helpers shared by the test modules (imported by name; tests/ is on sys.path)."""

import numpy as np


def max_rel(a, b):
    """max |a - b| / max |b| (0 for empty arrays); complex-aware."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.size == 0:
        return 0.0
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


def case(g, i):
    """Fields of golden case i (keys 'case{i}_*')."""
    pre = f"case{i}_"
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}
