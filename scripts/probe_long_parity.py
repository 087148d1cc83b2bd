"""Long-horizon fp32 parity probe: run a BASELINE scene N steps in fp32
(throughput) and fp64 (parity) mode on identical prescribed inputs and print
rel-L2 of rho-1, u, marker forces every `every` steps; optionally also the
reference (oracle/_ref) on the host for c1."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import cases as K  # noqa: E402
from paper_2206_01683_b200 import CoupledSession, SessionConfig  # noqa: E402
from paper_2206_01683_b200.scenes import make_scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
every = int(sys.argv[3]) if len(sys.argv) > 3 else 100
sc = make_scene(name)
ss = {}
for prec in ("fp64", "fp32"):
    ss[prec] = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                            frame_mode=sc.frame_mode, precision=prec,
                                            max_markers=sc.m))
t0 = time.time()
for k in range(steps):
    fr = sc.frame(k)
    mk = sc.markers(k)
    for prec, s in ss.items():
        s.set_frame(fr)
        s.set_markers(sc.offsets, *mk)
        st = s.step()
        assert st.stable(), (prec, k)
    if (k + 1) % every == 0:
        r = {}
        for prec, s in ss.items():
            fw, valid, stats = s.marker_forces()
            rho, u = s.macro()
            r[prec] = dict(u=u, rho=rho, fw=fw, valid=valid, st=s.stencils(), F=s.force())
        a, b = r["fp32"], r["fp64"]
        print(f"{name} step {k+1}: stencils_eq={np.array_equal(a['st'], b['st'])} "
              f"valid_eq={np.array_equal(a['valid'], b['valid'])} "
              f"u={K.rel_l2(a['u'], b['u']):.3e} rho-1={K.rel_l2(a['rho']-1, b['rho']-1):.3e} "
              f"fw={K.rel_l2(a['fw'], b['fw']):.3e} F={K.rel_l2(a['F'], b['F']):.3e} "
              f"|u|max={np.abs(b['u']).max():.3e} t={time.time()-t0:.1f}s", flush=True)
