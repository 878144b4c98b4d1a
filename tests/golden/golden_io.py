"""Pack/unpack lists of per-case array dicts into one .npz (no pickles)."""
from __future__ import annotations

import numpy as np


def pack(cases: list[dict], path):
    keys = sorted(cases[0].keys())
    out = {"__n": np.array([len(cases)])}
    for k in keys:
        arrs = [np.atleast_1d(np.asarray(c[k])) for c in cases]
        off = np.zeros(len(arrs) + 1, dtype=np.int64)
        np.cumsum([a.size for a in arrs], out=off[1:])
        out[k + "__off"] = off
        out[k] = np.concatenate(arrs) if arrs else np.zeros(0)
    np.savez_compressed(path, **out)


def unpack(path) -> list[dict]:
    z = np.load(path)
    n = int(z["__n"][0])
    keys = [k for k in z.files if not k.endswith("__off") and k != "__n"]
    data = {k: (z[k], z[k + "__off"]) for k in keys}
    cases = []
    for i in range(n):
        cases.append({k: v[o[i]:o[i + 1]] for k, (v, o) in data.items()})
    return cases
