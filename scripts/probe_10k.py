"""First unstable step of a long device-skinned c2 run (cycled vs fresh poses)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01683_b200 import CoupledSession, SessionConfig
from paper_2206_01683_b200.scenes import make_scene

sc = make_scene(sys.argv[1] if len(sys.argv) > 1 else "c2")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
for mode in ("fresh", "cycled"):
    s = CoupledSession(SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu,
                                     frame_mode=sc.frame_mode, precision="fp32", max_markers=sc.m))
    s.set_skin(*sc.skin())
    t0 = time.time()
    bad = None
    for k in range(N):
        kk = k if mode == "fresh" else k % 200
        st, tau, _ = s.step_skinned(sc.frame(kk), sc.poses(kk))
        if not st.stable():
            bad = (k, st)
            break
    print(mode, "first unstable:", bad, "%.1fs" % (time.time() - t0), flush=True)
    s.close()
