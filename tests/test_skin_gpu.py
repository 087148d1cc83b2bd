"""GPU: skinned bodies on the device against the oracle.

fp64 (parity mode): the device-skinned markers (update_samples), the marker
forces, tau_ext and CouplingStats (session.hpp:129-143) and the fluid state
are bit-identical to the oracle driving the same steps.  fp32 (throughput):
the skinned markers and stencil sets are identical to fp64 (the skinning is
fp64 in both modes), tau_ext and the stats within rel-L2 1e-5 of fp64, and
bit-identical run to run (fixed reduction order)."""
import numpy as np
import pytest

from cases import rel_l2
from skin_cases import init_fluid, run_gpu_skin, run_oracle_skin, skin_scene

pytestmark = pytest.mark.gpu

STEPS = [0, 1, 2, 3]


@pytest.fixture(scope="module")
def one_fish():
    sc = skin_scene()
    return sc, run_oracle_skin(sc, STEPS)


def test_fp64_skinned_step_bit_exact(one_fish):
    sc, (o, fo) = one_fish
    g, fg = run_gpu_skin(sc, STEPS, "fp64")
    for a, b in zip(g, o):
        for k in ("pts", "vel", "nrm", "fw", "tau", "stats"):
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
        assert np.array_equal(a["valid"], b["valid"])
        assert np.array_equal(a["stats_session"], b["stats_session"])
        assert a["min_f"] == b["min_f"]
    assert np.array_equal(fg, fo)


def test_fp64_two_bodies_frame_none():
    sc = skin_scene(dims=(64, 28, 28), frame_mode="none", bodies=2)
    o, fo = run_oracle_skin(sc, [0, 1, 2])
    g, fg = run_gpu_skin(sc, [0, 1, 2], "fp64")
    for a, b in zip(g, o):
        for k in ("pts", "vel", "nrm", "fw", "tau", "stats"):
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    assert np.array_equal(fg, fo)


def test_fp32_skinned_step_within_tolerance(one_fish):
    sc, (o, _) = one_fish
    g64, _ = run_gpu_skin(sc, STEPS, "fp64")
    g, _ = run_gpu_skin(sc, STEPS, "fp32")
    for a, b, c in zip(g, o, g64):
        for k in ("pts", "vel", "nrm"):
            assert np.array_equal(a[k], b[k]), k  # fp64 skinning in both modes
        assert np.array_equal(a["valid"], b["valid"])
        assert np.array_equal(a["stencils"], c["stencils"])
        assert rel_l2(a["fw"], b["fw"]) <= 1e-5
        assert rel_l2(a["tau"], b["tau"]) <= 1e-5
        assert rel_l2(a["stats"], b["stats"]) <= 1e-5


def test_fp32_three_bodies_split_kernels():
    """More than two skinned bodies take the separate skin kernels (k_skin_update,
    k_skin_tau beside K4) instead of the fused marker kernel: same contract."""
    sc = skin_scene(dims=(120, 28, 28), frame_mode="none", bodies=3)
    o, _ = run_oracle_skin(sc, [0, 1, 2])
    g, _ = run_gpu_skin(sc, [0, 1, 2], "fp32")
    g2, _ = run_gpu_skin(sc, [0, 1, 2], "fp32")
    for a, b, c in zip(g, o, g2):
        for k in ("pts", "vel", "nrm"):
            assert np.array_equal(a[k], b[k]), k
        assert rel_l2(a["tau"], b["tau"]) <= 1e-5 and rel_l2(a["stats"], b["stats"]) <= 1e-5
        assert np.array_equal(a["tau"], c["tau"]) and np.array_equal(a["stats"], c["stats"])


def test_fp32_two_bodies_fused():
    sc = skin_scene(dims=(64, 28, 28), frame_mode="none", bodies=2)
    o, _ = run_oracle_skin(sc, [0, 1, 2])
    g, _ = run_gpu_skin(sc, [0, 1, 2], "fp32")
    for a, b in zip(g, o):
        for k in ("pts", "vel", "nrm"):
            assert np.array_equal(a[k], b[k]), k
        assert rel_l2(a["tau"], b["tau"]) <= 1e-5 and rel_l2(a["stats"], b["stats"]) <= 1e-5


def test_fp32_tau_run_to_run_identical():
    sc = skin_scene()
    a, _ = run_gpu_skin(sc, [0, 1, 2], "fp32")
    b, _ = run_gpu_skin(sc, [0, 1, 2], "fp32")
    for x, y in zip(a, b):
        assert np.array_equal(x["tau"], y["tau"]) and np.array_equal(x["stats"], y["stats"])


def test_fp32_virtual_work_identity():
    """test_ib.cpp:215-249 on the device's outputs: tau_ext . v = power_on_body."""
    sc = skin_scene()
    g, _ = run_gpu_skin(sc, [0, 1, 2], "fp32")
    for k, r in zip([0, 1, 2], g):
        _, _, v, _ = sc.joint_state(0, k)
        p = r["stats"][0, 6]
        assert abs(r["tau"] @ v - p) < 1e-9 * max(1.0, abs(p))


def test_skin_api_contract():
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    from paper_2206_01683_b200._abi import FsgError, InputError
    sc = skin_scene()
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
    off, sks, rest, nrest, W, areas = sc.skin()
    with pytest.raises(FsgError):
        s.set_pose(sc.poses(0))  # no skinned bodies yet
    s.set_skin(off, sks, rest, nrest, W, areas)
    with pytest.raises(FsgError):
        s.step()  # no pose yet
    bad = [np.full_like(W[0], 1.0 / W[0].shape[1])]  # 6 nonzero weights per marker
    with pytest.raises(InputError):
        s.set_skin(off, sks, rest, nrest, bad, areas)
    s.set_skin(off, sks, rest, nrest, W, areas)
    s.set_frame(sc.frame(0))
    s.set_pose(sc.poses(0))
    assert s.step().stable()
    # back to host markers: the skinned path is off again
    s.set_markers(off, *sc.markers(1))
    s.step()
    with pytest.raises(FsgError):
        s.body_wrench()
    s.close()


@pytest.mark.parametrize("E", [4, 32])
def test_batched_skinned_envs_match_single_sessions(E):
    """EnvBatch with skinned envs (one fish per env, each its own gait phase)
    plus one env with host markers: distributions, skinned markers and marker
    forces bit-identical to the envs stepped one by one; tau_ext / stats within
    1e-9 (the batch sums each marker's fixed-point terms, a session its warps'
    sums).  E = 32 (20480 markers): more than SKC = 8 markers per warp of the batched
    marker grid, so the warps refill their skin cache chunk by chunk."""
    from paper_2206_01683_b200 import CoupledSession, EnvBatch, SessionConfig
    sc = skin_scene()
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    rho, u = init_fluid(sc)

    def drive(sessions, step_all):
        for s in sessions:
            s.initialize(rho, u)
        for e, s in enumerate(sessions):
            if e == 2:
                continue
            s.set_skin(*sc.skin())
        out = []
        for k in range(4):
            for e, s in enumerate(sessions):
                s.set_frame(sc.frame(k + 5 * e))
                if e == 2:
                    s.set_markers(sc.offsets, *sc.markers(k))
                else:
                    s.set_pose(sc.poses(k + 5 * e))
            step_all()
        for e, s in enumerate(sessions):
            r = dict(f=s.get_f(), fw=s.marker_forces()[0], st=s.last_status())
            if e != 2:
                r["mk"] = s.markers()
                r["tau"], r["stats"] = s.body_wrench()
            out.append(r)
        return out

    singles = [CoupledSession(cfg) for _ in range(E)]
    a = drive(singles, lambda: [s.step() for s in singles])
    batch = EnvBatch(cfg, E)
    b = drive(batch.envs, batch.step)
    for x, y in zip(a, b):
        assert np.array_equal(x["f"], y["f"]) and np.array_equal(x["fw"], y["fw"])
        if "mk" in x:
            for p, q in zip(x["mk"], y["mk"]):
                assert np.array_equal(p, q)
            assert rel_l2(np.concatenate(y["tau"]), np.concatenate(x["tau"])) <= 1e-9
            assert rel_l2(y["stats"], x["stats"]) <= 1e-9
    for s in singles:
        s.close()
    batch.close()


def test_step_skinned_one_call_matches_separate_calls():
    """fsg_step_skinned (frame + pose + step + wrench in one ABI call) gives
    the same step as the separate calls."""
    from paper_2206_01683_b200 import CoupledSession, SessionConfig
    sc = skin_scene()
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    rho, u = init_fluid(sc)
    a, b = CoupledSession(cfg), CoupledSession(cfg)
    for s in (a, b):
        s.initialize(rho, u)
        s.set_skin(*sc.skin())
    for k in range(3):
        a.set_frame(sc.frame(k))
        a.set_pose(sc.poses(k))
        sa = a.step()
        ta, wa = a.body_wrench()
        sb, tb, wb = b.step_skinned(sc.frame(k).packed(), sc.poses(k))
        assert sa.min_f == sb.min_f and np.array_equal(np.concatenate(ta), np.concatenate(tb))
        assert np.array_equal(wa, wb)
    assert np.array_equal(a.get_f(), b.get_f())
    a.close()
    b.close()


def test_batch_step_skinned_one_call_matches_separate_calls():
    from paper_2206_01683_b200 import EnvBatch, SessionConfig
    sc = skin_scene()
    E = 3
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    rho, u = init_fluid(sc)
    A, Bt = EnvBatch(cfg, E), EnvBatch(cfg, E)
    for bt in (A, Bt):
        for s in bt.envs:
            s.initialize(rho, u)
            s.set_skin(*sc.skin())
    for k in range(3):
        for e, s in enumerate(A.envs):
            s.set_frame(sc.frame(k + 5 * e))
            s.set_pose(sc.poses(k + 5 * e))
        sa = A.step()
        frames = np.stack([sc.frame(k + 5 * e).packed() for e in range(E)])
        poses = np.stack([sc.poses(k + 5 * e)[0] for e in range(E)])
        sb, taus, stats = Bt.step_skinned(frames, poses)
        for e in range(E):
            ta, wa = A.envs[e].body_wrench()
            assert sa[e].min_f == sb[e].min_f and sa[e].stable() == sb[e].stable()
            assert np.array_equal(ta[0], taus[e]) and np.array_equal(wa[0], stats[e])
    for e in range(E):
        assert np.array_equal(A.envs[e].get_f(), Bt.envs[e].get_f())
    A.close()
    Bt.close()
