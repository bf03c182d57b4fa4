"""The reference's OWN test suite running unmodified on the drop-in.

scripts/install_reference.sh installs the unmodified reference package
(`shardsim`) into baseline/_ref and copies its test files next to it (test
infrastructure, git-ignored).  This runner executes those files in a
subprocess with the `shardcu_alias` plugin, which aliases `shardsim.ket` to
`paper_2304_14969_b200.ket` before shardsim is imported — so the reference's
engine, tableau, validate and CLI, and every test, drive libshardcu's device
DenseKet.  The `slow` acceptance ensembles are deselected (minutes of
host-bound Python even on the reference's own NumPy kets).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "shardsim_tests"

pytestmark = pytest.mark.gpu

# Tests of the reference that cannot hold for ANY device-resident DenseKet,
# with the reason (documented deviation):
KNOWN_DEVIATIONS: dict[str, str] = {
    "test_acceptance.py::test_criterion_2_factorized_input_scaling":
        "asserts the NumPy kets' CPU cost model: QFT-on-GHZ wall time must grow >= 1.7x per qubit from 14 to "
        "17 qubits.  On the device these shards (<= 2 MiB) are launch-latency bound, so the time is nearly flat; "
        "its exactness/peak-memory halves are covered by test_engine.py and tests/test_engine_gpu.py",
}


def test_reference_suite_on_device_ket(tmp_path):
    if not (SUITE / "test_ket.py").exists():
        pytest.skip("baseline/_ref not installed (run scripts/install_reference.sh)")
    report = tmp_path / "alias.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "refsuite"), str(ROOT), str(REF),
                                         env.get("PYTHONPATH", "")])
    env["SHARDCU_ALIAS_REPORT"] = str(report)
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-m", "not slow", "-p", "shardcu_alias", "--tb=short",
           "-p", "no:cacheprovider", "--rootdir", str(SUITE), "-o", "addopts=",
           "-W", "ignore::DeprecationWarning"]
    for nodeid in KNOWN_DEVIATIONS:
        cmd += ["--deselect", nodeid]
    r = subprocess.run(cmd, cwd=str(SUITE), env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-120:])
    assert report.exists(), f"alias plugin did not run:\n{tail}"
    rep = json.loads(report.read_text())
    assert rep["engine_binds_device_ket"] and rep["tableau_binds_device_ket"] and rep["validate_binds_device_ket"], rep
    assert rep["device_states_created"] > 1000, rep  # the suite really built device kets
    assert r.returncode == 0, f"reference suite failed on the device DenseKet:\n{tail}"
