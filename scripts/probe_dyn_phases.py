"""Dev probe: per-phase clock64 cycles of the warp-per-env robot kernel
(FSG_LIB=paper_2206_01683_b200/ab/dyntime.so, built with -DFSG_DYN_TIMING)."""
import ctypes as C, os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0] = [R]
import numpy as np
from paper_2206_01683_b200 import dynamics as D, _abi
from paper_2206_01683_b200.scenes import koi_articulation, koi_body
body = koi_body(0.01); robot = D.koi_robot(body, koi_articulation(body))
rb = D.RobotBatch(robot, 8)
L = _abi.lib(); out = (C.c_ulonglong * 8)()
L.fsg_dyn_debug_timing(out, 1)
n = 50
for _ in range(n):
    rb.step(np.zeros((8, robot.n_joints)), None, 1000.0, (0, 0, -9.81), 0.004, 4)
L.fsg_dyn_debug_timing(out, 0)
names = ["load+hydro", "forces", "fk", "crba", "rnea", "llt", "integrate"]
for k, nm in enumerate(names):
    print(f"{nm:12s} {out[k] / n:10.0f} cycles/step ({out[k] / n / 1.9e3:.1f} us)")
