"""bench.py drives N ranks by itself (`--gpus N` outside torchrun re-launches
as N processes under torch.distributed.run), times each rank and reports the
max over ranks; here on CPU under gloo with the oracle standing in for the
kernel (SC_BENCH_COMPUTE=oracle test mode), checking that the shards cover
the whole output and concatenate to the single-pass result."""

from __future__ import annotations

import json
import os
import pathlib
import subprocess
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent


def _run(gpus: int):
    env = dict(os.environ, SC_BENCH_COMPUTE="oracle", SC_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(gpus), "--steps", "2",
                          "--warmup", "1", "--test-ne", "25000", "--test-nh", "900"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=REPO)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout          # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [1, 2, 3])
def test_bench_spawns_ranks_and_covers_output(gpus):
    line = _run(gpus)
    assert line["n_gpus"] == gpus
    assert line["compute"].startswith("oracle-cpu")
    cov = line["coverage"]
    assert cov["gathered"] == cov["outputs"] == 25000 + 900 - 1
    shards = cov["shards"]
    assert len(shards) == gpus and shards[0][0] == 0 and shards[-1][1] == cov["outputs"]
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))     # contiguous, no overlap
    assert cov["max_abs_err"] == 0.0
    assert line["value"] > 0 and line["ms_per_step"] > 0
