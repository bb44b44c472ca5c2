"""build_mesh on the device (swe_dev_build_mesh):
the same Mesh as the host build_mesh (itself pinned to the reference's
mesh.hpp by tests/test_host.py) bit for bit, and the same error texts."""
import numpy as np
import pytest

from conftest import bit_equal
from paper_1807_00672_b200 import api

pytestmark = pytest.mark.gpu

FIELDS = ("cell_nodes", "cell_area", "cx", "cy", "cell_inradius", "cell_edge", "cell_sign",
          "edge_nodes", "edge_left", "edge_right", "nx", "ny", "edge_length")


def same_mesh(a, b):
    assert (a.n_cells, a.n_edges, a.n_boundary_edges) == (b.n_cells, b.n_edges, b.n_boundary_edges)
    for f in FIELDS:
        assert bit_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("case", ["square", "three_mounds", "channel", "sloping"])
def test_device_build_equals_host_build(case):
    if case == "square":
        raw = api.generate_square_mesh(37, 23, 3.0, 2.0)
        bed, man = np.linspace(0, 1, raw.n_cells), np.full(raw.n_cells, 0.02)
    else:
        name = {"three_mounds": "three_mounds_friction", "channel": "channel",
                "sloping": "sloping_wet_dry"}[case]
        sc = api.make_scenario(name, scale=0.05)
        raw, bed, man = sc.raw, sc.bed, sc.manning
    same_mesh(api.build_mesh(raw, bed, man, device=0), api.build_mesh(raw, bed, man))


def _err(fn):
    try:
        fn()
    except api.SweError as e:
        return type(e).__name__, str(e)
    return None


def corrupt_cases():
    base = api.generate_square_mesh(4, 3, 1.0, 1.0)
    nodes, tris = base.nodes.copy(), base.triangles.copy()
    out = {}
    t = tris.copy(); t[5, 1] = 99; out["range"] = (nodes, t)
    t = tris.copy(); t[7, 2] = t[7, 0]; out["degenerate"] = (nodes, t)
    n = np.vstack([nodes, [[0.5, 0.0], [1.0, 0.0]]]); t = np.vstack([tris, [[0, len(n) - 2, len(n) - 1]]])
    out["zero_area"] = (n, t)
    t = np.vstack([tris, tris[3:4]]); out["shared_by_3"] = (nodes, t)
    t = np.vstack([tris, tris[2:3, [0, 2, 1]]]); out["same_direction"] = (nodes, t)
    t = tris.copy(); t[[1, 9]] = t[[9, 1]]; out["ok_permuted"] = (nodes, t)
    return out


@pytest.mark.parametrize("name", sorted(corrupt_cases()))
def test_device_build_errors_match_host(name):
    nodes, tris = corrupt_cases()[name]
    raw = api.RawMesh.from_arrays(nodes, tris)
    z, n = np.zeros(raw.n_cells), np.zeros(raw.n_cells)
    host = _err(lambda: api.build_mesh(raw, z, n))
    dev = _err(lambda: api.build_mesh(raw, z, n, device=0))
    assert host == dev
    assert (host is None) == (name == "ok_permuted"), host
