"""The multi-GPU path behind the drop-in C++ API (include/swe/multigpu.hpp):
swe::run with backend.gpus / backend.comm, the C++ push plan and link
sequence, and rank-local part meshes built from the RawMesh alone
(tests/cpp/multigpu_driver.cpp)."""
import json
import subprocess

import pytest

from conftest import ROOT

EXE = ROOT / "tests" / "cpp" / "multigpu_driver"


def run(*args, timeout=900):
    p = subprocess.run([str(EXE), *args], capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout)


@pytest.mark.skipif(not EXE.exists(), reason="multigpu driver not built")
def test_rank_local_mesh_equals_the_global_slice():
    """build_rank_mesh (owned + ghost triangles, build_mesh on the subset)
    equals build_local_mesh sliced from the global Mesh, array by array."""
    out = run("host")
    assert out["rank_mesh_matches"]


@pytest.mark.gpu
@pytest.mark.skipif(not EXE.exists(), reason="multigpu driver not built")
def test_run_with_gpus_and_comm_matches_one_device():
    """run() over 2 linked parts (backend.gpus, lockstep on one device) and
    over 2 ranks (backend.comm: threads, in-process allgather) are
    bit-identical to the single-domain run(): state, t / dt / max-speed
    series, snapshots, clip ledger; the mass series to 1e-12."""
    out = run()
    assert out["steps"] > 50
    assert out["gpus2_state_bitwise"] and out["gpus2_series_ok"]
    assert out["snapshots"][0] == out["snapshots"][1] >= 3 and out["snap_ok"]
    assert out["ledger_events"][0] == out["ledger_events"][1]
    assert out["comm_ranks_ok"], out["comm_errors"]
