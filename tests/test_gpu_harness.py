"""The reference's own harness (bench.hpp: Stoker convergence study, grid
ladder) compiled unchanged against the drop-in headers (tests/cpp/
harness_driver) runs on the B200 and prints the same study, byte for byte, as
the same driver built on the reference headers alone (oracle/_ref/harness_ref,
CPU) -- SURVEY.md §8(f) row 4 and acceptance criterion 6."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

OURS = ROOT / "tests" / "cpp" / "harness_driver"
REF = ROOT / "oracle" / "_ref" / "harness_ref"


def run(exe, *args, timeout=600):
    p = subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr
    return p.stdout


@pytest.mark.skipif(not (OURS.exists() and REF.exists()), reason="harness drivers not built")
def test_convergence_study_matches_reference_bytes():
    ours = run(OURS, "converge", 100, 10, 3, 40.0)
    assert ours == run(REF, "converge", 100, 10, 3, 40.0)
    rows = [r.split(",") for r in ours.strip().splitlines()[1:]]
    l1 = [float(r[2]) for r in rows]  # acceptance.cpp:231-250 (c6: 151.0, 87.82, 50.10)
    assert [round(x, 2) for x in l1] == [150.99, 87.82, 50.1]
    assert all(r[5] == "yes" for r in rows)


@pytest.mark.skipif(not OURS.exists(), reason="harness driver not built")
def test_ladder_runs_on_the_device():
    out = run(OURS, "ladder", 5, 23, 71)
    rows = [r.split(",") for r in out.strip().splitlines()[1:]]
    assert len(rows) == 2 * 3  # grids x reps (bench.hpp:123-210)
    for r in rows:
        assert int(r[6]) == 5 and float(r[8]) > 0.0
