"""Batched envs (BASELINE config 5; SURVEY.md §8(e) "batched into one launch
per kernel"): E env sessions stepped by one marker launch and one
collide/stream launch give BIT-IDENTICAL distributions, marker forces and
statuses to the same envs stepped one by one -- with different bodies and
frames per env, an env without markers, host- and device-resident markers,
and the collide-only first step."""
import numpy as np
import pytest
import torch

import cases as K
from paper_2206_01683_b200 import CoupledSession, EnvBatch, SessionConfig

pytestmark = pytest.mark.gpu

DT = 0.004
E = 5
NO_MARKERS, DEVICE_MARKERS = 3, 1


def _cfg():
    return SessionConfig(dims=(40, 32, 24), dx=0.01, dt=DT, rho=1000.0, nu=0.00089,
                         frame_mode="translation_yaw", precision="fp32", max_markers=512)


def _env_inputs(e):
    n = 40 * 32 * 24
    r = np.random.default_rng(100 + e)
    rho, u = 1.0 + 0.01 * (r.random(n) - 0.5), 0.02 * (r.random(3 * n) - 0.5)
    pts, nrm, area = K.fib_sphere(0.05 + 0.004 * e, 160 + 30 * e, np.array([0.004 * e, -0.003, 0.002]))
    return rho, u, pts, nrm, area


def _markers(e, k, pts, nrm, area):
    shift = np.array([0.003 * np.sin(0.7 * k + e), 0.002 * np.cos(0.5 * k), 0.0])
    vel = np.tile([0.05 * np.cos(0.7 * k), -0.02, 0.01 * e], (len(area), 1))
    return np.ascontiguousarray(pts + shift), vel, nrm, area


def _drive(sessions, step_all):
    inputs = [_env_inputs(e) for e in range(E)]
    for e, s in enumerate(sessions):
        s.initialize(inputs[e][0], inputs[e][1])
    keep = []
    for k in range(6):
        for e, s in enumerate(sessions):
            s.set_frame(K._fs_to_product(K.frame_at(k + 3 * e, DT)))
            if e == NO_MARKERS:
                continue
            pts, vel, nrm, area = _markers(e, k, *inputs[e][2:])
            off = np.array([0, len(area)], dtype=np.int64)
            if e == DEVICE_MARKERS:
                dev = [torch.tensor(np.ascontiguousarray(a).reshape(-1), device="cuda")
                       for a in (pts, vel, nrm, area)]
                keep.append(dev)
                s.set_markers_device(off, *(t.data_ptr() for t in dev))
            else:
                s.set_markers(off, pts, vel, nrm, area)
        sts = step_all()
    out = []
    for e, s in enumerate(sessions):
        fw = s.marker_forces()[0] if e != NO_MARKERS else np.zeros((0, 3))
        out.append(dict(f=s.get_f(), fw=fw, min_f=sts[e].min_f, oob=sts[e].out_of_bounds_markers,
                        stable=sts[e].stable()))
    return out


def test_batch_bit_identical_to_single_sessions():
    singles = [CoupledSession(_cfg()) for _ in range(E)]
    ref = _drive(singles, lambda: [s.step() for s in singles])
    for s in singles:
        s.close()
    b = EnvBatch(_cfg(), E)
    got = _drive(b.envs, b.step)
    b.close()
    for e in range(E):
        assert ref[e]["stable"] and got[e]["stable"]
        assert np.array_equal(got[e]["f"], ref[e]["f"]), f"env {e}: distributions differ"
        assert np.array_equal(got[e]["fw"], ref[e]["fw"]), f"env {e}: marker forces differ"
        assert got[e]["min_f"] == ref[e]["min_f"] and got[e]["oob"] == ref[e]["oob"]


def test_batch_rejects_bad_configs():
    from paper_2206_01683_b200 import InputError
    with pytest.raises(InputError):
        EnvBatch(SessionConfig(dims=(16, 16, 16), precision="fp64"), 2)
    with pytest.raises(InputError):
        EnvBatch(SessionConfig(dims=(16, 16, 16), precision="fp32"), 0)
