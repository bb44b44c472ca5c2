"""Held skipped tiles (skip_code, csrc/swe_step.cuh): a tile that k_tile
skipped at the two previous steps already holds, in the buffer the step
writes, exactly the state it would write, so the write is elided.  The
results must equal the path that writes every skipped tile (SWE_NO_HELD=1)
and the reference bit for bit -- also after set_state restores a different
state under the same step number, when the buffers' stale contents must not
be trusted, and across several advance() launches."""
import os

import numpy as np
import pytest

from conftest import bit_equal
from oracle.pyoracle import COracle, MeshArrays
from paper_1807_00672_b200 import api

pytestmark = pytest.mark.gpu


def _solver(mesh, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return api.DeviceSolver(mesh)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name,scale", [("sloping_wet_dry", 0.05), ("three_mounds_friction", 0.05)])
def test_held_tiles_equal_written_tiles_and_reference(name, scale):
    sc = api.make_scenario(name, scale=scale)
    m = api.build_mesh(sc.raw, sc.bed, sc.manning)
    # the graph loop (k_tile) at any size: SWE_PERSISTENT=0
    a = _solver(m, SWE_PERSISTENT=0)
    b = _solver(m, SWE_PERSISTENT=0, SWE_NO_HELD=1)
    rng = np.random.default_rng(5)
    other = api.FieldState(sc.state.h.copy(), sc.state.qx.copy(), sc.state.qy.copy())
    wet = other.h > 0
    other.h[wet] *= rng.uniform(0.9, 1.1, int(wet.sum()))
    out = []
    for s in (a, b):
        s.set_state(sc.state)
        r1 = np.concatenate([s.advance(1e30, max_steps=k) for k in (40, 200, 360)])
        st1, _, _ = s.get_state()
        s.set_state(other, 0.0, 0)  # a different state under the same step numbers
        r2 = np.concatenate([s.advance(1e30, max_steps=k) for k in (7, 300)])
        st2, _, n2 = s.get_state()
        out.append((r1, st1, r2, st2, n2, s.info()["skipped_tiles"]))
    (ra1, sa1, ra2, sa2, na, ka), (rb1, sb1, rb2, sb2, nb, kb) = out
    assert na == nb == 300 and ka == kb and ka > 0
    assert bit_equal(ra1, rb1) and bit_equal(ra2, rb2)
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(sa1, k), getattr(sb1, k)), k
        assert bit_equal(getattr(sa2, k), getattr(sb2, k)), k
    ref = COracle().advance(MeshArrays.from_mesh(m), other.h, other.qx, other.qy, nsteps=300)
    assert bit_equal(ra2[:, 2], ref["dts"])
    for k in ("h", "qx", "qy"):
        assert bit_equal(getattr(sa2, k), ref[k]), k
