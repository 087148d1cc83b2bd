"""Dev probe: where the end-to-end skinned coupled step spends host time.
Per step: set_frame, set_pose (per-link pose), step() (launch + synchronous
status), body_wrench() (tau_ext + stats readback)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

for name in sys.argv[1:] or ["c2"]:
    sc = make_scene(name)
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
    s.set_skin(*sc.skin())
    poses = [sc.poses(k) for k in range(8)]
    frames = [sc.frame(k) for k in range(8)]
    T = dict(set_frame=0.0, set_pose=0.0, step_async=0.0, last_status=0.0, body_wrench=0.0)
    N = 300
    for k in range(N + 20):
        t0 = time.perf_counter(); s.set_frame(frames[k % 8])
        t1 = time.perf_counter(); s.set_pose(poses[k % 8])
        t2 = time.perf_counter(); s.step_async()
        t3 = time.perf_counter(); s.last_status()
        t4 = time.perf_counter(); s.body_wrench()
        t5 = time.perf_counter()
        if k >= 20:
            for key, a, b in (("set_frame", t0, t1), ("set_pose", t1, t2), ("step_async", t2, t3),
                              ("last_status", t3, t4), ("body_wrench", t4, t5)):
                T[key] += b - a
    tot = sum(T.values())
    print(name, " | ".join(f"{k} {v / N * 1e6:.1f} us" for k, v in T.items()),
          f"| total {tot / N * 1e6:.1f} us = {sc.n_cells / (tot / N) / 1e6:.0f} MLUPS")
    s.close()
