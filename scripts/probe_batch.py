"""Dev probe: EnvBatch round time (device, async, warm) and host enqueue time."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2206_01683_b200 import EnvBatch, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

sc = make_scene("c5")
for E in [int(v) for v in (sys.argv[1:] or ["1", "4", "8"])]:
    b = EnvBatch(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                               frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m), E)
    dms = []
    for e, s in enumerate(b.envs):
        if os.environ.get("PROBE_NO_MARKERS"):
            s.set_markers_device(np.array([0], dtype=np.int64), 0, 0, 0, 0)
            continue
        dm = [torch.tensor(np.ascontiguousarray(a).reshape(-1), device="cuda") for a in sc.markers(e)]
        s.set_markers_device(sc.offsets, *(t.data_ptr() for t in dm))
        dms.append(dm)
    frames = [sc.frame(k) for k in range(16)]
    ext = torch.cuda.ExternalStream(b.envs[0].stream)
    for k in range(20):
        for s in b.envs:
            s.set_frame(frames[k % 16])
        b.step_async()
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ext):
        torch.cuda._sleep(int(3e6))  # host enqueues ahead of the GPU
    e0.record(ext)
    th = 0.0
    for k in range(n):
        t0 = time.perf_counter()
        for s in b.envs:
            s.set_frame(frames[k % 16])
        b.step_async()
        th += time.perf_counter() - t0
    e1.record(ext)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"E={E}: device {ms*1e3:.1f} us/round = {E*sc.n_cells/ms/1e3:.0f} MLUPS | host enqueue {th/n*1e6:.1f} us/round")
    b.close()
