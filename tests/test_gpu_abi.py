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


def _hilbert16(x, y):
    """d2xy's inverse on a 65536^2 grid (csrc/swe_prep.cuh hilbert16)"""
    d, s = 0, 1 << 15
    while s > 0:
        rx, ry = (1 if x & s else 0), (1 if y & s else 0)
        d += s * s * ((3 * rx) ^ ry)
        if ry == 0:
            if rx == 1:
                x, y = 65535 - x, 65535 - y
            x, y = y, x
        s >>= 1
    return d


def test_cell_order_is_the_blocked_hilbert_curve():
    """swe_dev_cell_order equals an independent restatement of the blocked-
    Hilbert renumbering (squares of the short side along the long axis, a
    65536^2 Hilbert curve in each, stable sort of 40-bit keys); it is a
    permutation, square after square, and consecutive cells are neighbours
    except where the curve crosses the thin last square."""
    raw = api.generate_square_mesh(64, 16, 4.0, 1.0)  # 4:1 strip, cells of 1/16
    m = api.build_mesh(raw, np.zeros(raw.n_cells), np.zeros(raw.n_cells))
    s = api.DeviceSolver(m)
    order = np.empty(m.n_cells, np.int32)
    assert L.load().swe_dev_cell_order(s.ctx, L.ptr(order)) == L.SWE_OK
    cx, cy = m.cx, m.cy
    x0, x1, y0, y1 = cx.min(), cx.max(), cy.min(), cy.max()
    side = max(min(x1 - x0, y1 - y0), max(x1 - x0, y1 - y0) / 255.0) * (1.0 + 1e-9)
    keys = []
    for c in range(m.n_cells):
        a, b = (cx[c] - x0) / side, (cy[c] - y0) / side
        blk = min(max(np.floor(a), 0.0), 255.0)
        fx, fy = min(max((a - blk) * 65536.0, 0.0), 65535.0), min(max(b * 65536.0, 0.0), 65535.0)
        keys.append((int(blk) << 32) | _hilbert16(int(fx), int(fy)))
    want = np.argsort(np.array(keys, dtype=np.uint64), kind="stable")
    assert np.array_equal(order, want)
    assert np.array_equal(np.sort(order), np.arange(m.n_cells))
    c = np.stack([cx, cy], 1)[order]
    assert np.all(np.diff(np.floor((c[:, 0] - x0) / side)) >= 0)  # square after square
    jumps = np.hypot(*np.diff(c, axis=0).T) * 16
    assert (jumps > 2.0).sum() <= 2 and jumps.max() <= 8.0
