"""Dev probe: per-call wall time of EnvBatch.step_dynamic on the c5 scene
(8 skinned koi envs, robots on the device) vs step_skinned."""
import os, sys, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0] = [R]
import numpy as np
from paper_2206_01683_b200 import EnvBatch, SessionConfig, dynamics as D
from paper_2206_01683_b200.scenes import make_scene
sc = make_scene("c5"); E = 8
cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu, frame_mode=sc.frame_mode,
                    precision="fp32", max_markers=sc.m)
b = EnvBatch(cfg, E)
for s in b.envs:
    s.set_skin(*sc.skin())
robot = D.koi_robot(sc.bodies[0], sc.articulations()[0])
rb = D.RobotBatch(robot, E); rb.set_rest(*D.rest_pose(robot))
nj = robot.n_joints
ts = []
for k in range(60):
    fr = np.stack([sc.frame(k + 37 * e).packed() for e in range(E)])
    po = np.stack([sc.poses(k + 37 * e)[0] for e in range(E)])
    t0 = time.perf_counter(); b.step_skinned(fr, po); t1 = time.perf_counter()
    act = np.array([[0.2 * np.sin(2 * np.pi * 2.0 * k * sc.dt - 0.8 * j + e) for j in range(nj)] for e in range(E)])
    t2 = time.perf_counter(); st, fl, _ = b.step_dynamic(rb, act, fr, sc.rho, (0, 0, -9.81), sc.dt, 4); t3 = time.perf_counter()
    t4 = time.perf_counter(); rb.step(act, None, sc.rho, (0, 0, -9.81), sc.dt, 4); t5 = time.perf_counter()
    ts.append(((t1 - t0) * 1e6, (t3 - t2) * 1e6, (t5 - t4) * 1e6, int(fl.max())))
for k in (0, 1, 2, 10, 30, 59):
    print(k, "skinned %.0f us  dynamic %.0f us  robot-only %.0f us  flags %d" % ts[k])
print("median skinned/dynamic/robot:", np.median([t[0] for t in ts]), np.median([t[1] for t in ts]), np.median([t[2] for t in ts]))
import torch
dev = torch.device("cuda", 0)
fw = torch.empty(1 << 27, dtype=torch.float32, device=dev); fr_ = torch.ones(1 << 27, dtype=torch.float32, device=dev)
sink = torch.zeros(1, device=dev)
for mode in ("back-to-back", "l2-flush"):
    tt = []
    for k in range(40):
        if mode == "l2-flush":
            fw.fill_(1.0); torch.sum(fr_, dim=0, out=sink[0]); torch.cuda.synchronize(dev)
        fr = np.stack([sc.frame(k + 37 * e).packed() for e in range(E)])
        act = np.zeros((E, nj))
        t0 = time.perf_counter(); b.step_dynamic(rb, act, fr, sc.rho, (0, 0, -9.81), sc.dt, 4); tt.append((time.perf_counter() - t0) * 1e6)
    print(mode, "median %.0f us, max %.0f us" % (np.median(tt), max(tt)))
