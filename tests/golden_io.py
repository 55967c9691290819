"""Loader for the committed golden fixtures (tests/golden, made by
oracle/make_golden.py from the real reference)."""
import json
import os
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def manifest():
    """manifest.json (oracle/make_golden.py) merged with the manifest_*.json
    of the other generators (make_golden_gs_direct.py: Gauss-Seidel and
    Direct; make_golden_cfg3_full.py: full-size BASELINE config 3)."""
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        man = json.load(fh)
    for extra in sorted(os.listdir(GOLDEN)):   # manifest_gsd.json, manifest_cfg3_full.json
        if extra.startswith("manifest_") and extra.endswith(".json"):
            with open(os.path.join(GOLDEN, extra)) as fh:
                man["cases"].update(json.load(fh)["cases"])
    return man


def case(name):
    """(arrays, meta) of one golden case."""
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        arrs = {k: z[k] for k in z.files}
    return arrs, manifest()["cases"][name]


def names(prefix):
    return sorted(k for k in manifest()["cases"] if k.startswith(prefix))
