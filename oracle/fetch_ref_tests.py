"""Stage the reference's own test modules for an unchanged run against the drop-in.

TEST INFRASTRUCTURE ONLY.  Copies ``/root/reference/pkg/tests/*.py`` byte for
byte into ``oracle/_ref/ref_tests/`` -- a git-ignored directory (the
reference's sources never enter this repo's history) that is NOT
gpurun-ignored, so the copies travel to the GPU box with the snapshot, like a
compiled ``oracle/_ref`` would.  ``tests/golden/ref_tests_sha256.json`` pins
the sha256 of every module, so the GPU run proves it executes the reference's
files unchanged.  ``tests/ref_alias.py`` (a pytest plugin) makes
``import scatterconv`` resolve to ``paper_2401_01607_b200``;
``tests/test_ref_unchanged_gpu.py`` runs each module under it.

    python oracle/fetch_ref_tests.py          # copy (no-op without /root/reference)
    python oracle/fetch_ref_tests.py --pin    # also rewrite the sha256 pin file
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import shutil
import sys

HERE = pathlib.Path(__file__).resolve().parent
SRC = pathlib.Path("/root/reference/pkg/tests")
DST = HERE / "_ref" / "ref_tests"
PIN = HERE.parent / "tests" / "golden" / "ref_tests_sha256.json"


def sha256(p: pathlib.Path) -> str:
    return hashlib.sha256(p.read_bytes()).hexdigest()


def fetch(pin: bool = False) -> bool:
    if not SRC.is_dir():
        return False
    DST.mkdir(parents=True, exist_ok=True)
    digests = {}
    for f in sorted(SRC.glob("*.py")):
        out = DST / f.name
        if not out.exists() or sha256(out) != sha256(f):
            shutil.copyfile(f, out)
        digests[f.name] = sha256(f)
    # an empty ini so the repo's pytest.ini (testpaths, plugins) stays out of it
    (DST / "pytest.ini").write_text("[pytest]\n")
    if pin:
        PIN.write_text(json.dumps(digests, indent=1, sort_keys=True) + "\n")
    return True


if __name__ == "__main__":
    ok = fetch(pin="--pin" in sys.argv)
    print(f"{'staged' if ok else 'no reference tree; nothing staged'}: {DST}")
