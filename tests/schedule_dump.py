"""Golden-fixture loaders and the canonical per-iteration schedule text.

The canonical line format must stay identical to ``iter_line`` in
tests/golden/gen_golden.py (which produced the fixtures from the reference).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rb") as f:
            return json.loads(f.read())
    with open(path) as f:
        return json.load(f)


def iter_line(it, t0, dur, win0, rows, admitted, fin, moves, moved, t1, after):
    return "|".join([str(it), float(t0).hex(), float(dur).hex(), str(win0),
                     ",".join(map(str, rows)),
                     ";".join(f"{a}@{b}" for a, b in admitted),
                     ",".join(map(str, fin)),
                     ";".join(f"{r}:{a}>{b}:{s}" for r, a, b, s in moves),
                     str(moved), float(t1).hex(), f"{after[0]}+{after[1]}"])


def sha(lines):
    h = hashlib.sha256()
    for ln in lines:
        h.update(ln.encode())
        h.update(b"\n")
    return h.hexdigest()


def decode_cost(d):
    return {k: (float.fromhex(v) if isinstance(v, str) else v) for k, v in d.items()}


def decode_requests(rows):
    """[(rid, batch, input_len, max_out, actual_out, arrival)]"""
    return [(r[0], r[1], r[2], r[3], r[4], float.fromhex(r[5])) for r in rows]
