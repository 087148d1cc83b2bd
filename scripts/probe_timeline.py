"""Dev probe: device timeline of the banded coupled step (async steady state).

Needs the instrumented build libfsg_dbg.so (-DFSG_TIMING: per-step globaltimer
stamps indexed by the tile stamp).  Per step: marker kernel first-start /
last-end, K4 first-start / last phase-A end, first phase-B start / last end,
in us relative to the marker start; `gap` = marker start minus the previous
step's K4 end.
"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01683_b200 import _abi
_abi.LIB_PATH = os.path.join(os.path.dirname(_abi.LIB_PATH), "libfsg_dbg.so")
import torch
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

lib = ctypes.CDLL(_abi.LIB_PATH)
buf = (ctypes.c_ulonglong * 512)()
for name in sys.argv[1:] or ["c2"]:
    sc = make_scene(name)
    cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                        frame_mode=sc.frame_mode, precision="fp32")
    s = CoupledSession(cfg)
    s.set_markers(sc.offsets, *sc.markers(0))
    for k in range(30):
        s.set_frame(sc.frame(k)); s.step_async()
    s.last_status(); lib.fsg_debug_timeline(buf)
    frames = [sc.frame(k) for k in range(30, 70)]
    if os.environ.get("PROBE_BLOCK"):  # queue every step before the GPU starts
        with torch.cuda.stream(torch.cuda.ExternalStream(s.stream)):
            torch.cuda._sleep(int(2e6))
    for f in frames:
        s.set_frame(f); s.step_async()
    s.last_status(); lib.fsg_debug_timeline(buf)
    t = list(buf)
    rows = [t[8 * j: 8 * j + 8] for j in range(64) if t[8 * j + 1] != 0]
    rows.sort(key=lambda r: r[0])
    prev_end = None
    for r in rows[5:15]:
        b = r[0]
        f = lambda v: (v - b) / 1e3
        gap = f"{(b - prev_end)/1e3:5.1f}" if prev_end else "  -  "
        print(f"{name} gap {gap} | mk 0.0->{f(r[1]):5.1f} | K4 {f(r[2]):5.1f}->A {f(r[3]):5.1f} | B {f(r[4]):5.1f}->{f(r[5]):5.1f}"
              f" | exit {f(r[7]):5.1f}")
        prev_end = r[7] if r[7] else r[5]
    s.close()
