"""The ABI's error contract: invalid configuration and
misuse raise InputError with the reference's messages where it has them
(units.hpp:56-68, lattice.hpp:66-69), instability is a status (never an
error), and every check fires before any device work."""
import numpy as np
import pytest

import cases as K
from paper_2206_01683_b200 import CoupledSession, EnvBatch, InputError, SessionConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kw,msg", [
    (dict(dims=(7, 16, 16)), "dims"),                       # lattice.hpp:66-67
    (dict(nu=0.1, dx=0.02), "tau"),                         # units.hpp:56-68 (tau > 1.5)
    (dict(nu=-1.0), "positive"),
    (dict(dims=(16, 16, 4), z_offset=2, nz_global=32), None),  # ok slab, must not raise
    (dict(dims=(16, 16, 4), z_offset=30, nz_global=32), "slab"),
])
def test_config_validation(kw, msg):
    base = dict(dims=(16, 16, 16), dx=0.01, dt=0.004, precision="fp32")
    base.update(kw)
    if msg is None:
        CoupledSession(SessionConfig(**base)).close()
        return
    with pytest.raises(InputError, match=msg):
        CoupledSession(SessionConfig(**base))


def test_marker_misuse():
    s = CoupledSession(SessionConfig(dims=(16, 16, 16), dx=0.01, dt=0.004, precision="fp32",
                                     max_markers=8))
    pts, nrm, area = K.fib_sphere(0.02, 10, np.zeros(3))
    vel = np.zeros_like(pts)
    with pytest.raises(InputError, match="capacity"):
        s.set_markers(np.array([0, 10]), pts, vel, nrm, area)
    with pytest.raises(InputError, match="offsets"):
        s.set_markers(np.array([1, 8]), pts[:8], vel[:8], nrm[:8], area[:8])
    with pytest.raises(InputError, match="non-decreasing"):
        s.set_markers(np.array([0, 5, 3]), pts[:3], vel[:3], nrm[:3], area[:3])
    with pytest.raises(InputError, match="z-slab"):
        s.halo_begin(0)
    s.close()


def test_slab_misuse():
    s = CoupledSession(SessionConfig(dims=(16, 16, 4), dx=0.01, dt=0.004, precision="fp32",
                                     z_offset=4, nz_global=16))
    with pytest.raises(InputError, match="recenter"):
        s.recenter((1, 0, 0))
    s.close()


def test_instability_is_a_status_not_an_error():
    """solver.hpp:13-20: a blown-up step reports stable() == False."""
    s = CoupledSession(SessionConfig(dims=(16, 16, 16), dx=0.01, dt=0.004, precision="fp32",
                                     boundary="periodic"))
    n = 16 ** 3
    s.initialize(np.ones(n), np.tile([0.9, 0.0, 0.0], n))  # |u| far beyond the lattice limit
    st = None
    for _ in range(5):
        st = s.step()
    assert not st.stable()
    s.close()


def test_batch_session_handles():
    b = EnvBatch(SessionConfig(dims=(16, 16, 16), dx=0.01, dt=0.004, precision="fp32"), 3)
    assert len(b.envs) == 3 and len({int(e.handle.value) for e in b.envs}) == 3
    sts = b.step()
    assert len(sts) == 3 and all(st.stable() for st in sts)
    b.close()
