"""Loader for the reference-generated planner fixtures (tests/golden/make_goldens.py)."""

import functools
import gzip
import json
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden" / "planner_goldens.json.gz"


@functools.lru_cache(maxsize=1)
def goldens() -> dict:
    return json.loads(gzip.decompress(GOLDEN.read_bytes()))


def entries(pairs) -> frozenset:
    return frozenset((int(c), int(d)) for c, d in pairs)
