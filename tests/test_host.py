"""Host side (CPU only): the mesh builder and case producers of the drop-in API
(include/swe/mesh.hpp, include/swe/cases.hpp), the C-ABI library's exports,
and the C++ drop-in driver build.  Mirrors the reference's test_mesh.cpp /
test_cases.cpp cases."""
import subprocess

import numpy as np
import pytest

from conftest import ROOT, bit_equal
from paper_1807_00672_b200 import _lib, api

MESH_KEYS = [("cell_nodes", "cell_nodes"), ("area", "cell_area"), ("cx", "cx"), ("cy", "cy"),
             ("inradius", "cell_inradius"), ("cell_edge", "cell_edge"), ("cell_sign", "cell_sign"),
             ("edge_nodes", "edge_nodes"), ("edge_left", "edge_left"),
             ("edge_right", "edge_right"), ("nx", "nx"), ("ny", "ny"), ("len", "edge_length")]


def flat(raw):
    n = raw.n_cells
    return api.build_mesh(raw, np.zeros(n), np.zeros(n))


def test_library_exports_every_declared_symbol():
    """include/swe_dev.h + include/swe_host.h symbols are exported (no GPU needed)."""
    lib = _lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = set()
    for h in ("swe_dev.h", "swe_host.h"):
        import re
        txt = (ROOT / "include" / h).read_text()
        declared |= set(re.findall(r"SWE_API [^(]*?\b(swe_\w+)\(", txt))
    assert declared and declared <= exported, declared - exported
    assert set(_lib.DECLARED) <= declared
    for name in declared:
        getattr(lib, name)


def test_generator_smallest_mesh():
    """test_mesh.cpp:20-27"""
    raw = api.generate_square_mesh(1, 1, 1.0, 1.0)
    assert raw.nodes.shape == (4, 2) and raw.triangles.shape == (2, 3)
    m = flat(raw)
    assert m.n_edges == 5 and m.n_boundary_edges == 4


def test_generator_2x2_euler():
    """test_mesh.cpp:29-37"""
    raw = api.generate_square_mesh(2, 2, 1.0, 1.0)
    m = flat(raw)
    assert len(raw.nodes) == 9 and m.n_cells == 8 and m.n_edges == 16
    assert len(raw.nodes) - m.n_edges + m.n_cells == 1 and m.n_boundary_edges == 8


def test_generator_1k_rung_and_errors():
    assert api.generate_square_mesh(23, 23, 75.0, 75.0).n_cells == 1058
    for args in ((0, 1, 1.0, 1.0), (1, 1, 0.0, 1.0), (1, 1, 1.0, -2.0)):
        with pytest.raises(api.MeshError):
            api.generate_square_mesh(*args)


@pytest.mark.parametrize("nx,ny,lx,ly", [(1, 1, 1.0, 1.0), (5, 3, 2.5, 7.0), (23, 23, 75.0, 75.0)])
def test_closure_and_unit_normals(nx, ny, lx, ly):
    """test_mesh.cpp:60-80"""
    m = flat(api.generate_square_mesh(nx, ny, lx, ly))
    assert np.all(np.abs(np.hypot(m.nx, m.ny) - 1.0) <= 1e-12)
    s = (m.cell_sign * m.edge_length[m.cell_edge])[..., None] * m.edge_normal[m.cell_edge]
    per = m.edge_length[m.cell_edge].sum(axis=1)
    assert np.all(np.hypot(*s.sum(axis=1).T) <= 1e-10 * per)
    assert np.all(m.cell_area > 0)


def test_build_errors():
    with pytest.raises(api.MeshError, match="degenerate triangle 0"):
        api.build_mesh(api.RawMesh.from_arrays([[0, 0], [1, 0], [0, 1]], [[0, 1, 1]]), [0.0], [0.0])
    with pytest.raises(api.MeshError, match="out of range"):
        api.build_mesh(api.RawMesh.from_arrays([[0, 0], [1, 0], [0, 1]], [[0, 1, 7]]), [0.0], [0.0])
    with pytest.raises(api.MeshError, match="zero area"):
        api.build_mesh(api.RawMesh.from_arrays([[0, 0], [1, 0], [2, 0]], [[0, 1, 2]]), [0.0], [0.0])
    raw = api.RawMesh.from_arrays([[0, 0], [1, 0], [0, 1]], [[0, 1, 2], [0, 1, 2]])
    with pytest.raises(api.MeshError, match="non-manifold"):
        api.build_mesh(raw, [0.0, 0.0], [0.0, 0.0])
    raw = api.generate_square_mesh(1, 1, 1.0, 1.0)
    with pytest.raises(api.MeshError, match="negative Manning coefficient at cell 1"):
        api.build_mesh(raw, [0.0, 0.0], [0.0, -1.0])


@pytest.mark.parametrize("kind", ["square", "unstructured"])
def test_build_matches_c_oracle(coracle, kind):
    raw = (api.generate_square_mesh(31, 17, 75.0, 30.0) if kind == "square"
           else api.generate_unstructured_mesh(31, 17, 75.0, 30.0, seed=3))
    m = flat(raw)
    o = coracle.build_mesh(raw.nodes, raw.triangles)
    for ok, mk in MESH_KEYS:
        assert np.array_equal(np.asarray(o[ok]).view(np.uint8),
                              np.ascontiguousarray(getattr(m, mk)).view(np.uint8)), ok


@pytest.mark.parametrize("kind", ["square", "unstructured"])
def test_build_matches_reference(refo, kind):
    raw = (api.generate_square_mesh(64, 40, 75.0, 30.0) if kind == "square"
           else api.generate_unstructured_mesh(64, 40, 75.0, 30.0, seed=11))
    bed, man, _ = api.init_case("three_mounds", raw)
    m = api.build_mesh(raw, bed, man)
    r = refo.build_mesh(raw.nodes, raw.triangles, bed, man)
    for ok, mk in MESH_KEYS:
        assert np.array_equal(np.asarray(r.a[ok]).view(np.uint8),
                              np.ascontiguousarray(getattr(m, mk)).view(np.uint8)), ok


@pytest.mark.parametrize("case", ["water_drop", "three_mounds", "lake_at_rest", "dam_break_1d"])
def test_cases_match_reference(refo, case):
    spec = api.case_defaults(case)
    raw = api.generate_unstructured_mesh(50, 20, spec["lx"], spec["ly"], seed=4)
    bed, man, st = api.init_case(case, raw)
    r = refo.init_case(case, [spec[k] for k in api.CASE_SPEC_KEYS], raw.nodes, raw.triangles)
    for a, b in zip((bed, man, st.h, st.qx, st.qy), r):
        assert bit_equal(a, b)


def test_case_errors():
    """test_cases.cpp:51-62, :168-171"""
    raw = api.generate_square_mesh(4, 4, 100.0, 100.0)
    with pytest.raises(api.CaseError, match="does not cover"):
        api.init_case("water_drop", raw)
    raw = api.generate_square_mesh(4, 4, 1000.0, 1000.0)
    with pytest.raises(api.CaseError, match="below the bed"):
        api.init_case("water_drop", raw, eta0=-5.0, amplitude=0.1)
    raw = api.generate_square_mesh(4, 4, 400.0, 40.0)
    with pytest.raises(api.CaseError, match="hL > hR"):
        api.init_case("dam_break_1d", raw, h_left=0.1, h_right=1.0)
    with pytest.raises(api.ConfigError):
        api.case_defaults("no_such_case")


@pytest.mark.parametrize("name", ["circular_dam_break", "three_mounds_friction", "channel",
                                  "sloping_wet_dry", "weak_square"])
def test_scenarios_build(name):
    sc = api.make_scenario(name, scale=0.02 if name != "circular_dam_break" else 0.5)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    assert m.n_cells == sc.raw.n_cells and m.n_cells > 0
    assert np.all(sc.state.h >= 0) and np.any(sc.state.h > 0)
    assert len(sc.raw.nodes) - m.n_edges + m.n_cells == 1


def test_unstructured_is_permuted_and_valid():
    raw = api.generate_unstructured_mesh(40, 30, 1.0, 1.0, seed=9)
    m = flat(raw)
    assert len(raw.nodes) - m.n_edges + m.n_cells == 1
    # a random numbering: neighbouring cells are far apart in index
    inter = m.edge_right >= 0
    gap = np.abs(m.edge_left[inter] - m.edge_right[inter])
    assert np.median(gap) > 100
    with pytest.raises(api.MeshError):
        api.generate_unstructured_mesh(4, 4, 1.0, 1.0, jitter=0.3)


def test_cpp_driver_builds():
    from paper_1807_00672_b200 import build
    exe = build.build_api_driver()
    assert exe.exists()
