"""pytest plugin (loaded with `-p shardcu_alias`): bind the reference
package's `shardsim.ket` to the device module before anything imports
shardsim, exactly as INTEGRATION.md §1 prescribes.  Everything above it —
the reference's engine.py, tableau.py, validate.py, cli.py and its own test
files — then runs unmodified on libshardcu's DenseKet.

At session end it writes a summary (which DenseKet the reference bound, how
many device states were created) to $SHARDCU_ALIAS_REPORT, so the runner in
tests/test_reference_suite.py can prove the device class was the one used.
"""
from __future__ import annotations

import json
import multiprocessing
import os
import sys

import paper_2304_14969_b200.ket as dev_ket

dev_ket.set_default_dtype("c128")  # the reference's precision (ket.py:77,82)
sys.modules["shardsim.ket"] = dev_ket

# The reference's process pool (validate.py:224-229) uses the default start
# method.  CUDA cannot be used in a child forked from a process that already
# holds a CUDA context, so a CUDA-backed shardsim runs its pool from a fork
# server that imported this binding (and no CUDA) first: the workers bind
# the device DenseKet and create their own contexts.  No reference code changes.
multiprocessing.set_forkserver_preload(["shardcu_alias"])
multiprocessing.set_start_method("forkserver", force=True)


def pytest_report_header(config):
    return "shardsim.ket -> paper_2304_14969_b200.ket (device DenseKet, libshardcu, complex128)"


def pytest_sessionfinish(session, exitstatus):
    import shardsim.engine as eng
    import shardsim.tableau as tab
    import shardsim.validate as val

    out = os.environ.get("SHARDCU_ALIAS_REPORT")
    if not out:
        return
    from paper_2304_14969_b200 import _build
    report = {
        "engine_binds_device_ket": eng.DenseKet is dev_ket.DenseKet,
        "tableau_binds_device_ket": tab.DenseKet is dev_ket.DenseKet,
        "validate_binds_device_ket": val.DenseKet is dev_ket.DenseKet,
        "device_states_created": dev_ket.alloc_count,
        "libshardcu": str(_build.LIB),
        "exitstatus": int(exitstatus),
    }
    with open(out, "w") as f:
        json.dump(report, f)
