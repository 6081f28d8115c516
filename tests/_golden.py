"""Loaders for the reference-generated fixtures in tests/golden/ (see make_golden.py)."""

from __future__ import annotations

import hashlib
import json
import pathlib

import numpy as np

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def unhex(lst) -> np.ndarray:
    return np.array([float.fromhex(v) for v in lst], dtype=np.float64)


def small_pairs():
    z = np.load(GOLDEN / "ref_small.npz")

    def unpack(name):
        v, off = z[name], z[name + "_off"]
        return [v[off[i]:off[i + 1]] for i in range(len(off) - 1)]

    cols = {k: unpack(k) for k in ("e", "h", "scatter", "commuted", "direct", "skip")}
    n = len(cols["e"])
    return [dict({k: cols[k][i] for k in cols}, threshold=float(z["threshold"][i]),
                 kind=int(z["kind"][i])) for i in range(n)]


def engine_sessions():
    with open(GOLDEN / "ref_engine.json", encoding="utf-8") as fh:
        return json.load(fh)


def configs_pins():
    return dict(np.load(GOLDEN / "ref_configs.npz"))


def replay(session, make_engine, to_host=np.asarray):
    """Run a recorded session against an engine exposing the reference API
    (process_block/process_sample/swap_ir/swap_ir_at_next_block/flush and the
    state hooks); yields (op, got, expect) per op."""
    eng = make_engine(unhex(session["h"]), session["nb"], float.fromhex(session["threshold"]))
    for op, want in zip(session["ops"], session["expect"]):
        kind = op[0]
        if kind == "block":
            got = to_host(eng.process_block(unhex(op[1])))
        elif kind == "sample":
            got = np.array([eng.process_sample(float.fromhex(op[1]))])
        elif kind == "swap":
            eng.swap_ir(unhex(op[1]))
            got = None
        elif kind == "defer":
            eng.swap_ir_at_next_block(unhex(op[1]))
            got = None
        elif kind == "flush":
            got = to_host(eng.flush())
        elif kind == "state":
            got = eng.state_dict()
        yield kind, got, want
