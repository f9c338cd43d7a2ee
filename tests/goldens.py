"""Loader for the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def group(name: str) -> dict:
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return {k: z[k] for k in z.files}


def cases(name: str):
    g = group(name)
    key = {"tables": "tables__names", "steps": "steps__names", "runs": "runs__names",
           "extract": "extract__names", "tracking": "track__names"}[name]
    return [str(c) for c in g[key]]


def case(name: str, c: str) -> dict:
    g = group(name)
    pre = c + "__"
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}


def big(name: str) -> dict:
    z = np.load(GOLDEN / f"big_{name}.npz", allow_pickle=False)
    return {k: z[k] for k in z.files}
