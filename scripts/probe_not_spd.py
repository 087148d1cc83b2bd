"""Dev probe: the robot kernels' NOT_SPD exit (a NaN joint angle makes the
mass matrix NaN, so the Cholesky stops) in the two-warp and one-warp forms
of the warp kernel and in the thread kernel; flags and the other envs'
states must come back (no hang)."""
import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
from paper_2206_01683_b200 import dynamics as D
from paper_2206_01683_b200.scenes import koi_articulation, koi_body
body = koi_body(0.01)
for name, E, wmax in (("two-warp", 4, "4096"), ("one-warp", 300, "4096"), ("thread", 4, "0")):
    os.environ["FSG_DYN_WARP_MAX"] = wmax
    r = D.koi_robot(body, koi_articulation(body))
    rb = D.RobotBatch(r, E)
    sts = [D.JointState.zero(r) for _ in range(E)]
    sts[1].q[0] = np.nan
    rb.set_states(sts)
    fl = rb.step(np.zeros((E, r.n_joints)), np.zeros((E, r.n_dofs)), 1000.0, (0, 0, -9.81), 0.004, 4)
    print(name, "flags", [int(x) for x in fl[:4]])
    rb.close()
