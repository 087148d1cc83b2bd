"""A few robot steps (koi, 8 envs, 4 substeps + hydrostatics): the ncu target
for the device robot kernels (scripts: ncu -k regex:k_dyn ...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2206_01683_b200 import dynamics as D
from paper_2206_01683_b200.scenes import koi_articulation, koi_body
body = koi_body(0.01)
robot = D.koi_robot(body, koi_articulation(body))
E = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rb = D.RobotBatch(robot, E)
for _ in range(4):
    rb.step(np.zeros((E, robot.n_joints)), None, 1000.0, (0, 0, -9.81), 0.004, 4)
print(rb.states()[0].base_pos)
