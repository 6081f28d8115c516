"""The reference's own test modules, run UNCHANGED against the drop-in.

``oracle/fetch_ref_tests.py`` (run by ``__graft_entry__.build()`` in the
build container) stages ``/root/reference/pkg/tests/*.py`` byte for byte in
the git-ignored ``oracle/_ref/ref_tests/``; the sha256 of every module is
pinned in ``tests/golden/ref_tests_sha256.json`` and checked here, so what
runs is the reference's file, not a restatement.  Each module runs in its own
pytest process with ``-p ref_alias`` (``import scatterconv`` →
``paper_2401_01607_b200``, tests/ref_alias.py), i.e. exactly as the
reference's CI would run it against a package named ``scatterconv``.

Every collected test must pass.  The only deselection is acceptance
criterion 5 (test_acceptance.py:123-138): a wall-clock r² >= 0.98 gate on a
CPU sweep of 441,000-sample renders that the reference itself fails on this
class of host (r² 0.956 in the survey); the device sweep it
would time is covered by tests/test_sweeps_gpu.py.
"""

from __future__ import annotations

import hashlib
import json
import os
import pathlib
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
STAGE = REPO / "oracle" / "_ref" / "ref_tests"
PIN = json.loads((REPO / "tests" / "golden" / "ref_tests_sha256.json").read_text())

# module -> minimum number of tests it holds (the reference's own counts)
MODULES = {
    "test_core.py": 33,
    "test_engine.py": 34,
    "test_acceptance.py": 9,
    "test_quantize.py": 42,
    "test_wavio.py": 26,
    "test_bench.py": 23,
    "test_cli.py": 32,
}
DESELECT = {
    "test_acceptance.py": ["test_acceptance.py::test_criterion_05_runtime_linearity_ir_sweep"],
}


def _staged() -> bool:
    return all((STAGE / name).is_file() for name in PIN)


def test_staged_modules_are_the_reference_files():
    if not _staged():
        pytest.skip("oracle/_ref/ref_tests not staged (run oracle/fetch_ref_tests.py where /root/reference exists)")
    for name, digest in PIN.items():
        assert hashlib.sha256((STAGE / name).read_bytes()).hexdigest() == digest, f"{name} differs from the reference"


@pytest.mark.gpu
@pytest.mark.parametrize("module", sorted(MODULES))
def test_reference_module_passes_unchanged(module, tmp_path):
    assert _staged(), "oracle/_ref/ref_tests missing: build() stages it from /root/reference"
    test_staged_modules_are_the_reference_files()
    junit = tmp_path / "junit.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REPO / "tests"), str(REPO), env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_alias", "-p", "no:cacheprovider", "-q",
           f"--junitxml={junit}", "--rootdir", str(STAGE), "-c", str(STAGE / "pytest.ini"), module]
    for d in DESELECT.get(module, []):
        cmd += ["--deselect", d]
    res = subprocess.run(cmd, cwd=STAGE, env=env, capture_output=True, text=True, timeout=1800)
    tail = (res.stdout + res.stderr)[-6000:]
    assert junit.exists(), tail
    suite = ET.parse(junit).getroot()
    suite = suite if suite.tag == "testsuite" else suite.find("testsuite")
    n = int(suite.get("tests"))
    bad = int(suite.get("failures")) + int(suite.get("errors"))
    skipped = int(suite.get("skipped"))
    print(f"{module}: {n} collected, {n - bad - skipped} passed, {bad} failed, {skipped} skipped")
    assert bad == 0 and res.returncode == 0, tail
    assert skipped == 0, tail
    assert n >= MODULES[module], f"{module}: only {n} tests collected\n{tail}"
