"""Loader of tests/golden/fixtures.{json,bin} (made by gen_golden.cpp, which
replays the reference tests' std::mt19937 streams)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def _load():
    if not _cache:
        with open(os.path.join(HERE, "fixtures.json")) as f:
            _cache["json"] = json.load(f)
        _cache["bin"] = np.fromfile(os.path.join(HERE, "fixtures.bin"), dtype="<f8")
    return _cache["json"], _cache["bin"]


def _arr(spec, blob):
    off, r, c = spec
    return blob[off:off + r * c].reshape(r, c).copy()


def cases(name):
    """List of dicts; array entries ([off, rows, cols]) become numpy arrays."""
    meta, blob = _load()
    out = []
    for case in meta[name]["cases"]:
        d = {}
        for k, v in case.items():
            if k in ("a", "b", "raw", "shuffled", "padded") and isinstance(v, list) and len(v) == 3 \
                    and all(isinstance(x, int) for x in v):
                d[k] = _arr(v, blob)
            else:
                d[k] = v
        out.append(d)
    return out


def case(name, label):
    for c in cases(name):
        if c.get("name") == label:
            return c
    raise KeyError(label)
