"""Argument validation of the newer C-ABI entry points (include/swe_dev.h):
they return SWE_INVALID with a message instead of crashing."""
import ctypes as C

import numpy as np
import pytest

from paper_1807_00672_b200 import _lib as L
from paper_1807_00672_b200 import api

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def solver():
    raw = api.generate_square_mesh(8, 6, 8.0, 6.0)
    m = api.build_mesh(raw, np.zeros(raw.n_cells), np.zeros(raw.n_cells))
    s = api.DeviceSolver(m)
    s.set_state(api.FieldState(np.ones(raw.n_cells), np.zeros(raw.n_cells),
                               np.zeros(raw.n_cells)))
    return s


def test_snapshot_slot_and_buffers_are_checked(solver):
    lib = L.load()
    h = np.empty(solver.n_cells)
    assert lib.swe_dev_snapshot_async(solver.ctx, 2, L.ptr(h), L.ptr(h), L.ptr(h)) == L.SWE_INVALID
    assert lib.swe_dev_snapshot_async(solver.ctx, 0, None, L.ptr(h), L.ptr(h)) == L.SWE_INVALID
    assert lib.swe_dev_snapshot_wait(solver.ctx, 5) == L.SWE_INVALID


def test_snapshot_roundtrip_equals_get_state(solver):
    lib = L.load()
    solver.advance(1e30, max_steps=7)
    a = [np.empty(solver.n_cells) for _ in range(3)]
    assert lib.swe_dev_snapshot_async(solver.ctx, 1, *[L.ptr(x) for x in a]) == L.SWE_OK
    assert lib.swe_dev_snapshot_wait(solver.ctx, 1) == L.SWE_OK
    st, _, _ = solver.get_state()
    for x, k in zip(a, ("h", "qx", "qy")):
        assert np.array_equal(x.view(np.int64), getattr(st, k).view(np.int64))


def test_link_arguments_are_checked(solver):
    lib = L.load()
    cells = np.array([solver.n_cells], np.int64)
    rc = lib.swe_dev_link(solver.ctx, 1, 1, None, None, L.ptr(cells), 0, None, None, None, None,
                          None, 1.0)  # rank >= nranks
    assert rc == L.SWE_INVALID
    bad = np.array([solver.n_cells + 1], np.int64)
    rc = lib.swe_dev_link(solver.ctx, 0, 1, (C.c_void_p * 1)(None), None, L.ptr(bad), 0, None,
                          None, None, None, None, 1.0)  # wrong own size
    assert rc == L.SWE_INVALID and b"n_cells" in lib.swe_dev_last_error()
    assert lib.swe_dev_link_phase(solver.ctx, 0, 1.0) == L.SWE_INVALID  # not linked


def test_advance_async_needs_a_graph():
    raw = api.generate_square_mesh(4, 4, 1.0, 1.0)
    m = api.build_mesh(raw, np.zeros(raw.n_cells), np.zeros(raw.n_cells))
    s = api.DeviceSolver(m, graph=False)
    assert L.load().swe_dev_advance_async(s.ctx, 1.0, 5, float("inf"), 16) == L.SWE_INVALID


def test_build_mesh_device_arguments_are_checked():
    lib = L.load()
    out = C.c_void_p()
    err = C.create_string_buffer(256)
    assert lib.swe_dev_build_mesh(0, 3, None, 1, None, C.byref(out), err, 256) == L.SWE_INVALID
    assert lib.swe_dev_build_mesh(0, -1, None, 0, None, C.byref(out), err, 256) == L.SWE_INVALID


def test_cell_skip_matches_info(solver):
    cs = solver.cell_skip()
    assert cs.dtype == np.uint8 and len(cs) == solver.n_cells and set(np.unique(cs)) <= {0, 1}
