"""Dev probe: device phase timeline of the coupled throughput step (steady state;\n--flush: L2 flushed between steps as in bench.py).

Needs the instrumented build (make -C paper_2206_01683_b200/csrc dbg ->
libfsg_dbg.so, -DFSG_TIMING).  Slots: 0 marker kernel start, 1 last marker
warp done, 2 K4 start, 3 last block out of phase A, 4 first band start,
5 K4 end; printed in us relative to slot 0, with the gap to the previous step.
"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSG_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2206_01683_b200", "libfsg_dbg.so")
import numpy as np
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig, _abi
from paper_2206_01683_b200.scenes import make_scene

lib = ctypes.CDLL(_abi.LIB_PATH)
FLUSH = "--flush" in sys.argv
SKIN = "--skin" in sys.argv
if SKIN:
    sys.argv.remove("--skin")
OOB = "--oob" in sys.argv  # host markers moved out of the box (no band)
if OOB:
    sys.argv.remove("--oob")
if FLUSH:
    sys.argv.remove("--flush")
    fw_buf = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    fr_buf = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.zeros(1, dtype=torch.float32, device="cuda")
S = 8
buf = (ctypes.c_ulonglong * (64 * S))()
for name in sys.argv[1:] or ["c2"]:
    sc = make_scene(name)
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m)
    s = CoupledSession(cfg)
    if SKIN:  # skinned on the device (fsg_set_skin / fsg_set_pose)
        s.set_skin(*sc.skin())
        poses = [sc.poses(k) for k in range(60)]
    else:
        mk0 = list(sc.markers(0))
        if OOB:
            mk0[0] = mk0[0] + 1e3
        dm = [torch.tensor(np.ascontiguousarray(a).reshape(-1), device="cuda") for a in mk0]
        s.set_markers_device(sc.offsets, *(t.data_ptr() for t in dm))
    for k in range(30):
        s.set_frame(sc.frame(k))
        if SKIN:
            s.set_pose(poses[k])
        s.step_async()
    s.last_status(); lib.fsg_debug_timeline(None)
    frames = [sc.frame(k) for k in range(30, 60)]
    ss = torch.cuda.ExternalStream(s.stream)
    with torch.cuda.stream(ss):
        torch.cuda._sleep(int(2e6))  # queue every step before the GPU starts
        for f in frames:
            if FLUSH:  # as bench.py: write + read 2x L2 between steps
                fw_buf.fill_(1.0)
                torch.sum(fr_buf, dim=0, out=sink[0])
            s.set_frame(f)
            if SKIN:
                s.set_pose(poses[30])
            s.step_async()
    s.last_status(); lib.fsg_debug_timeline(buf)
    t = list(buf)
    rows = sorted([t[S * j: S * j + S] for j in range(64) if t[S * j + 5] not in (0, ~0 & (2**64 - 1))],
                  key=lambda r: r[0])
    prev = None
    for r in rows[5:13]:
        b = r[0]
        f = lambda v: (v - b) / 1e3
        gap = f"{(b - prev) / 1e3:5.1f}" if prev and not FLUSH else "  -  "
        print(f"{name} gap {gap} | markers -> {f(r[1]):6.1f} | K4 {f(r[2]):6.1f} | phaseA out "
              f"{f(r[3]):6.1f} | band {f(r[4]):6.1f} -> {f(r[5]):6.1f}")
        prev = r[5]
    s.close()
