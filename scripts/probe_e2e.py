"""Dev probe: where the end-to-end (host API) coupled step spends its time.

Per step, like bench.py's e2e leg: set_frame, set_markers (host arrays),
step() (launch + synchronous status), marker_forces() (pinned readback +
CouplingStats).  Prints the mean wall time of each call."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

for name in sys.argv[1:] or ["c2"]:
    sc = make_scene(name)
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
    mk = [sc.markers(k) for k in range(8)]
    frames = [sc.frame(k) for k in range(8)]
    T = {"set_frame": 0.0, "set_markers": 0.0, "step_async": 0.0, "last_status": 0.0,
         "marker_forces": 0.0}
    N = 200
    for k in range(N + 10):
        t0 = time.perf_counter()
        s.set_frame(frames[k % 8])
        t1 = time.perf_counter()
        s.set_markers(sc.offsets, *mk[k % 8])
        t2 = time.perf_counter()
        s.step_async()
        t25 = time.perf_counter()
        s.last_status()
        t3 = time.perf_counter()
        s.marker_forces()
        t4 = time.perf_counter()
        if k >= 10:
            T["set_frame"] += t1 - t0
            T["set_markers"] += t2 - t1
            T["step_async"] += t25 - t2
            T["last_status"] += t3 - t25
            T["marker_forces"] += t4 - t3
    tot = sum(T.values())
    print(name, " | ".join(f"{k} {v / N * 1e6:.1f} us" for k, v in T.items()),
          f"| total {tot / N * 1e6:.1f} us = {sc.n_cells / (tot / N) / 1e6:.0f} MLUPS")
    # device time of the same steps (events around each step on the session stream)
    s.profile(True)
    for k in range(50):
        s.set_frame(frames[k % 8]); s.set_markers(sc.offsets, *mk[k % 8]); s.step(); s.marker_forces()
    ms, n = s.profile_read()
    print(f"   device time per step (same loop): {ms / n * 1e3:.1f} us")
    s.close()
