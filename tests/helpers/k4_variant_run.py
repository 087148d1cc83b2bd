"""Run a few pure-fluid fp32 steps on three grids and save the distributions
(tests/test_k4_variants_gpu.py runs it once per K4 variant)."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2206_01683_b200 import CoupledSession, FrameState, SessionConfig  # noqa: E402
out = {}
for name, dims, bnd, fm in (("open", (64, 48, 40), "open", "translation_yaw"), ("per", (96, 32, 24), "periodic", "none"),
                            ("wide", (256, 20, 12), "open", "full"),
                            ("per128", (128, 24, 20), "periodic", "translation_yaw")):
    s = CoupledSession(SessionConfig(dims=dims, dx=0.01, dt=0.004, boundary=bnd, frame_mode=fm, precision="fp32", max_markers=1))
    n = int(np.prod(dims)); r = np.random.default_rng(3)
    s.initialize(1.0 + 0.01 * (r.random(n) - 0.5), 0.03 * (r.random(3 * n) - 0.5))
    for k in range(7):
        yaw = 0.2 + 0.1 * k
        s.set_frame(FrameState(p=np.array([0.01 * k, 0, 0]), pd=np.array([0.05, 0, 0.01]), pdd=np.array([0.3, -0.1, 0.2]),
                               q=np.array([math.cos(yaw / 2), 0, 0, math.sin(yaw / 2)]), omega=np.array([0.1, -0.2, 0.5]),
                               alpha=np.array([0.3, 0.1, -1.0])))
        st = s.step()
    out[name] = s.get_f(); out[name + "_min"] = np.array([st.min_f])
    s.close()
np.savez(sys.argv[1], **out)
