"""Dev probe: where the coupled step's time goes at one scene (default c3):
device time per step (L2 flushed between steps, as bench.py) for
  fluid      no markers (k_collide_fix)
  oob        the scene's markers moved out of the box (marker kernel exits at
             once; the banded K4 runs phase A over every cell)
  host       the scene's markers as device arrays (k_markers_fix + K4)
  skinned    the bodies skinned on the device (k_markers_skin + K4)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
sc = make_scene(name)
fw_buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
fr_buf = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
sink = torch.zeros(1, dtype=torch.float32, device="cuda")


def run(mode):
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
    keep = []
    if mode in ("host", "oob"):
        pts, vel, nrm, area = sc.markers(0)
        if mode == "oob":
            pts = pts + 1e3
        keep = [torch.tensor(np.ascontiguousarray(a).reshape(-1), device="cuda") for a in (pts, vel, nrm, area)]
        s.set_markers_device(sc.offsets, *(t.data_ptr() for t in keep))
    elif mode == "skinned":
        s.set_skin(*sc.skin())
    stream = torch.cuda.ExternalStream(s.stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        for k in range(10 + K):
            s.set_frame(sc.frame(k))
            if mode == "skinned":
                s.set_pose(sc.poses(k))
            if k >= 10:
                fw_buf.fill_(1.0)
                torch.sum(fr_buf, dim=0, out=sink[0])
                ev[k - 10][0].record(stream)
            s.step_async()
            if k >= 10:
                ev[k - 10][1].record(stream)
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    s.close()
    return np.median(t), np.percentile(t, 10), np.percentile(t, 90)


for mode in ("fluid", "oob", "host", "skinned"):
    m, lo, hi = run(mode)
    print(f"{name} {mode:8s} step {m:7.1f} us  (p10 {lo:6.1f}, p90 {hi:6.1f})  "
          f"{sc.n_cells / m:8.0f} MLUPS", flush=True)
