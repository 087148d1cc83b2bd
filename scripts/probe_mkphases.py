"""Dev probe (libfsg_dbg.so): per-warp phase timestamps of the skinned marker
kernel (first marker of each warp) in the last of a few coupled steps.
Slots: 0 start, 1 staged, 2 stamped, 3 triggered, 4 vel/nrm, 5 finish start,
6 phi, 7 gathered, 8 butterfly, 9 forced, 10 spread, 11 tau, 12 loop end,
13 block tail.  usage: probe_mkphases.py c3"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSG_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2206_01683_b200", "libfsg_dbg.so")
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig, _abi
from paper_2206_01683_b200.scenes import make_scene

lib = ctypes.CDLL(_abi.LIB_PATH)
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
sc = make_scene(name)
s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                 frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
s.set_skin(*sc.skin())
fw = torch.empty(64 << 20, device="cuda"); fr = torch.ones(64 << 20, device="cuda"); sk = torch.zeros(1, device="cuda")
buf = (ctypes.c_ulonglong * (4096 * 16))()
for k in range(12):
    if k == 11:
        lib.fsg_debug_mkt(buf)  # clear-ish: overwritten slots below
        ctypes.memset(buf, 0, ctypes.sizeof(buf))
    fw.fill_(1.0); torch.sum(fr, dim=0, out=sk[0])
    s.set_frame(sc.frame(k)); s.set_pose(sc.poses(k)); s.step_async()
s.last_status()
lib.fsg_debug_mkt(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16).astype(np.float64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
rel = (a - t0) / 1e3
names = ["start", "staged", "stamped", "triggered", "velnrm", "fin0", "phi", "gathered", "bfly",
         "forced", "spread", "tau", "loopend", "tail"]
print(f"{name}: {len(a)} warps; times in us from the first warp start (p10 / p50 / p90)")
prev = None
for j, nm in enumerate(names):
    col = rel[:, j]
    col = col[a[:, j] > 0]
    if len(col) == 0:
        continue
    p = np.percentile(col, [10, 50, 90])
    d = "" if prev is None else f"   step p50 {np.percentile(col - prev[:len(col)], 50) if len(prev) == len(col) else float('nan'):6.2f}"
    print(f"  {j:2d} {nm:10s} {p[0]:7.2f} {p[1]:7.2f} {p[2]:7.2f}{d}")
    prev = col
