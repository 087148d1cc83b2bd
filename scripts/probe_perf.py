"""Dev probe: time the async coupled step (CUDA events on the session stream)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

def time_steps(s, nsteps, scene=None, warm=5):
    ext = torch.cuda.ExternalStream(s.stream)
    mk = None
    if scene is not None and scene.m:
        mk = [scene.markers(k) for k in range(4)]
    def one(k):
        if scene is not None:
            s.set_frame(scene.frame(k))
            if mk is not None:
                s.set_markers(scene.offsets, *mk[k % 4])
        s.step_async()
    for k in range(warm):
        one(k)
    s.last_status()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for k in range(nsteps):
        one(k)
    e1.record(ext)
    st = s.last_status()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / nsteps, st

for name in sys.argv[1:] or ["c1", "c2", "c3"]:
    sc = make_scene(name)
    for prec in ("fp32",):
        cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                            frame_mode=sc.frame_mode, precision=prec)
        s = CoupledSession(cfg)
        ms, st = time_steps(s, 50, None)
        n = sc.n_cells
        print(f"{name} {prec} pure-LBM step: {ms*1e3:.1f} us  {n/ms/1e3:.0f} MLUPS  status={st}")
        s.close()
        s = CoupledSession(cfg)
        ms, st = time_steps(s, 50, sc)
        print(f"{name} {prec} coupled step (m={sc.m}): {ms*1e3:.1f} us  {n/ms/1e3:.0f} MLUPS  status={st}")
        s.close()
