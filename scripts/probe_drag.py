"""Dev probe: batched empirical drag (fsg_drag_*) throughput vs the oracle
restatement on one CPU core.  Prints env-steps/s of the surface work."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bind as B
from paper_2206_01683_b200 import DragBatch
from paper_2206_01683_b200.scenes import make_scene

sc = make_scene("c5")
off, sks, rest, nrest, W, areas = sc.skin()
for E in (8, 64, 512):
    d = DragBatch(E, precision="fp32")
    for e in range(E):
        d.set_skin(e, sks[0], rest, nrest, W[0], areas)
    poses = [sc.poses(k)[0] for k in range(8)]
    for e in range(E):
        d.set_pose(e, poses[e % 8])
    d.step()
    N = 200
    t0 = time.perf_counter()
    P = [np.stack([poses[(k + e) % 8] for e in range(E)]) for k in range(8)]
    for k in range(N):
        d.set_poses(P[k % 8])
        d.step()
    dt = (time.perf_counter() - t0) / N
    print(f"E={E}: {dt * 1e6:.1f} us per batched step (poses up, tau + stats down) = {E / dt:.0f} env-steps/s")
    d.close()
t0 = time.perf_counter()
n = 0
while time.perf_counter() - t0 < 2.0:
    B.empirical_step(sks[0], poses[n % 8], rest, nrest, W[0], areas, 40.0)
    n += 1
dt = (time.perf_counter() - t0) / n
print(f"oracle (C restatement, 1 core): {dt * 1e6:.1f} us per env-step = {1 / dt:.0f} env-steps/s ({sc.m} markers)")
