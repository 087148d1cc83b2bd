"""Dev probe: aggregate throughput of E concurrent env sessions (c5 envs) on
one GPU, each on its own stream, stepped round-robin with device markers."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

sc = make_scene("c5")
for E in [int(v) for v in (sys.argv[1:] or ["1", "2", "4", "8"])]:
    ss, dms = [], []
    for e in range(E):
        s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                         frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
        dm = [torch.tensor(np.ascontiguousarray(a).reshape(-1), device="cuda") for a in sc.markers(e)]
        s.set_markers_device(sc.offsets, *(t.data_ptr() for t in dm))
        ss.append(s); dms.append(dm)
    frames = [sc.frame(k) for k in range(16)]
    for k in range(20):
        for s in ss:
            s.set_frame(frames[k % 16]); s.step_async()
    for s in ss:
        s.last_status()
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:  # every env stream starts after e0
        torch.cuda.ExternalStream(s.stream).wait_event(e0)
    for k in range(n):
        for s in ss:
            s.set_frame(frames[k % 16]); s.step_async()
    for s in ss:
        ev = torch.cuda.Event(); ev.record(torch.cuda.ExternalStream(s.stream))
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{E} envs: {ms / n * 1e3:.1f} us per round, {E * sc.n_cells * n / ms / 1e3:.0f} MLUPS aggregate")
    for s in ss:
        s.close()
