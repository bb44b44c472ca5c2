"""SURVEY.md §8(f) rows 2 and 4 next to the reference's own io.hpp
(tests/cpp/io_ext_driver): the parallel VTK writer is byte-identical to
write_vtk_snapshot (io.hpp:171-206); backend.gpus / devices ride in the
config text the reference's parse_config (io.hpp:288-420) reads unchanged."""
import json
import subprocess

import pytest

from conftest import ROOT

EXE = ROOT / "tests" / "cpp" / "io_ext_driver"
pytestmark = pytest.mark.skipif(not EXE.exists(), reason="io_ext driver not built (needs the reference)")


def run(*args):
    p = subprocess.run([str(EXE), *args], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout)


@pytest.mark.parametrize("nx,ny", [(1, 1), (13, 7), (120, 50)])
def test_parallel_vtk_writer_is_byte_identical(nx, ny, tmp_path):
    out = run("vtk", str(nx), str(ny), str(tmp_path))
    assert out["vtk_identical"] and out["cells"] == 2 * nx * ny


def test_backend_gpus_in_the_config_text():
    out = run("config")
    assert out["gpus"] == 2 and out["devices"] == 2
    assert out["kind_parallel"] and out["threads"] == 2  # the reference's keys still parsed
    assert out["plain_parser_error"] == "unknown key 'devices' in backend"


@pytest.mark.gpu
def test_config_with_two_gpus_runs_like_one():
    out = run("config-run")
    assert out["steps"] > 10 and out["two_gpu_run_equals_one"]
