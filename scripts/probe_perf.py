"""Dev probe: time the async coupled step (CUDA events on the session stream)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

def time_steps(s, nsteps, scene=None, per_step_markers=False, warm=5, device_mk=False):
    ext = torch.cuda.ExternalStream(s.stream)
    mk = [scene.markers(k) for k in range(4)] if scene is not None and scene.m else None
    if mk is not None and device_mk:
        dm = [torch.tensor(np.ascontiguousarray(a, dtype=np.float64).reshape(-1), device="cuda") for a in mk[0]]
        s.set_markers_device(scene.offsets, *(t.data_ptr() for t in dm))
    elif mk is not None and not per_step_markers:
        s.set_markers(scene.offsets, *mk[0])
    def one(k):
        if scene is not None:
            s.set_frame(scene.frame(k))
            if mk is not None and per_step_markers:
                s.set_markers(scene.offsets, *mk[k % 4])
        s.step_async()
    for k in range(warm):
        one(k)
    s.last_status()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(ext)
    for k in range(nsteps):
        one(k)
    e1.record(ext)
    st = s.last_status()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / nsteps
    return e0.elapsed_time(e1) / nsteps, wall * 1e3, st

for name in sys.argv[1:] or ["c1", "c2", "c3"]:
    sc = make_scene(name)
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32")
    n = sc.n_cells
    for label, scene, per, dev in (("pure-LBM", None, False, False), ("coupled device-mk", sc, False, True),
                                   ("coupled static-mk", sc, False, False),
                                   ("coupled host-mk/step", sc, True, False)):
        s = CoupledSession(cfg)
        ms, wall, st = time_steps(s, int(os.environ.get("PROBE_STEPS", "100")), scene, per,
                                  warm=int(os.environ.get("PROBE_WARM", "5")), device_mk=dev)
        print(f"{name} {label}: {ms*1e3:.1f} us/step (host wall {wall*1e3:.1f})  {n/ms/1e3:.0f} MLUPS  stable={st.stable()} min_f={st.min_f:.4f}")
        s.close()
