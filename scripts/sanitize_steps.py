"""Drive a few coupled throughput steps for compute-sanitizer (racecheck,
synccheck, memcheck): c2 with device-skinned markers (k_markers_skin ->
k_collide_band as its programmatic dependent), c2 with host markers
(k_markers_fix), c3 with 2 skinned bodies, and one c5 batch round
(k_markers_batch -> k_collide_band_batch).

    compute-sanitizer --tool racecheck python scripts/sanitize_steps.py [steps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2206_01683_b200 import CoupledSession, EnvBatch, SessionConfig  # noqa: E402
from paper_2206_01683_b200.scenes import make_scene  # noqa: E402


def cfg_of(sc):
    return SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                         frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)


def single(name, steps, skinned):
    sc = make_scene(name)
    s = CoupledSession(cfg_of(sc))
    if skinned:
        s.set_skin(*sc.skin())
    for k in range(steps):
        if skinned:
            st = s.step_skinned(sc.frame(k), sc.poses(k))
        else:
            s.set_frame(sc.frame(k))
            s.set_markers(sc.offsets, *sc.markers(k))
            st = s.step()
    print(name, "skinned" if skinned else "host", "ok", st if not skinned else "")
    s.close()


def batch(steps, E=2):
    sc = make_scene("c5")
    b = EnvBatch(cfg_of(sc), E)
    for e in range(E):
        b.envs[e].set_skin(*sc.skin())
    for k in range(steps):
        fr = [sc.frame(k + 37 * e) for e in range(E)]
        po = [sc.poses(k + 37 * e) for e in range(E)]
        b.step_skinned(fr, po)
    print("c5 batch ok")
    b.close()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c2s", "c2h", "c3s", "c5b"]
    if "c2s" in which:
        single("c2", n, True)
    if "c2h" in which:
        single("c2", n, False)
    if "c3s" in which:
        single("c3", n, True)
    if "c5b" in which:
        batch(n)
