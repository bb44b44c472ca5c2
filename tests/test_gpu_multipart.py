"""Decomposed-domain runs on the device: P part contexts
with ghost cells and halo exchange (include/swe_dev.h multi-device entries),
driven in one process on one GPU, must be bit-identical to the single-domain
run -- the same machinery a multi-GPU run uses with NCCL moving the blocks."""
import numpy as np
import pytest

from conftest import bit_equal
from oracle.pyoracle import COracle, MeshArrays
from paper_1807_00672_b200 import api, dist

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("two_phase", [False, True], ids=["fused", "two_phase"])
def test_parts_on_one_gpu_match_single_domain(P, two_phase):
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, P)
    parts = [dist.PartSolver(dist.local_mesh(m, part, p), two_phase=two_phase) for p in range(P)]
    for p in parts:
        p.set_state(sc.state)
    ex = dist.LocalExchange(parts)
    recs = dist.run_parts(parts, ex, 150)
    got = api.FieldState.zeros(m.n_cells)
    for p in parts:
        t, step = p.gather_owned(got)
        assert step == 150
    ref = COracle().advance(MeshArrays.from_mesh(m), sc.state.h, sc.state.qx, sc.state.qy,
                            nsteps=150)
    assert bit_equal(recs[:, 1], ref["dts"]) and bit_equal(recs[:, 2], ref["max_speeds"])
    for k, a in (("h", got.h), ("qx", got.qx), ("qy", got.qy)):
        assert bit_equal(a, ref[k]), k
    m0 = recs[0, 3]
    assert abs(recs[-1, 3] - m0) <= 1e-12 * m0 + 1e-9


def test_part_error_reports_global_index():
    sc = api.make_scenario("sloping_wet_dry", scale=0.03)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    part = dist.partition(m, 2)
    lm = dist.local_mesh(m, part, 1)
    p = dist.PartSolver(lm)
    st = sc.state.copy()
    bad = int(lm.cells[5])
    st.h[bad] = 1.0
    st.qx[bad] = np.nan
    p.set_state(st)
    with pytest.raises(api.NumericError, match=f"non-finite velocity in cell {bad}$"):
        p.local_cfl()
