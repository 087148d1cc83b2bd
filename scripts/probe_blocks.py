"""Dev probe (libfsg_dbg.so): per-block phase-A timing of the banded K4 in
the last of a few coupled steps -- start, end of phase A, items taken, SM --
to see where the phase-A tail comes from.  usage: probe_blocks.py c3 [--skin|--oob]"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSG_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2206_01683_b200", "libfsg_dbg.so")
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig, _abi
from paper_2206_01683_b200.scenes import make_scene

lib = ctypes.CDLL(_abi.LIB_PATH)
name = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "--skin"
sc = make_scene(name)
s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                 frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
keep = []
if mode == "--skin":
    s.set_skin(*sc.skin())
else:
    mk0 = list(sc.markers(0))
    if mode == "--oob":
        mk0[0] = mk0[0] + 1e3
    keep = [torch.tensor(np.ascontiguousarray(a).reshape(-1), device="cuda") for a in mk0]
    s.set_markers_device(sc.offsets, *(t.data_ptr() for t in keep))
fw = torch.empty(64 << 20, device="cuda"); fr = torch.ones(64 << 20, device="cuda"); sk = torch.zeros(1, device="cuda")
for k in range(12):
    fw.fill_(1.0); torch.sum(fr, dim=0, out=sk[0])
    s.set_frame(sc.frame(k))
    if mode == "--skin":
        s.set_pose(sc.poses(k))
    s.step_async()
s.last_status()
buf = (ctypes.c_ulonglong * (8192 * 4))()
lib.fsg_debug_blocks(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4).astype(np.float64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
st, en, n, sm = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2], a[:, 3]
print(f"{name} {mode}: {len(a)} blocks; start p0/p50/p100 {np.percentile(st, [0, 50, 100]).round(1)}; "
      f"phaseA end p0/p10/p50/p90/p100 {np.percentile(en, [0, 10, 50, 90, 100]).round(1)}")
print("items per block p0/p50/p100", np.percentile(n, [0, 50, 100]))
late = np.argsort(en)[-12:]
for i in late:
    print(f"  block {i:4d} sm {int(sm[i]):3d} start {st[i]:6.1f} end {en[i]:6.1f} items {int(n[i])}")
# per-SM: blocks, total items, last end
for k in np.argsort([en[sm == q].max() if (sm == q).any() else 0 for q in range(148)])[-6:]:
    m = sm == k
    print(f"  SM {k:3d}: blocks {m.sum()} items {int(n[m].sum())} last end {en[m].max():6.1f} first start {st[m].min():6.1f}")
