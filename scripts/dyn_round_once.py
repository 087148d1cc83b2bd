"""A few c5 rounds through fsg_batch_step_dynamic (8 skinned koi envs with
their robots on the device): the target of the round's ncu launch list."""
import os, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0] = [R]
import numpy as np
from paper_2206_01683_b200 import EnvBatch, SessionConfig, dynamics as D
from paper_2206_01683_b200.scenes import make_scene
sc = make_scene("c5"); E = 8
cfg = SessionConfig(dims=sc.dims, dx=sc.dx, dt=sc.dt, rho=sc.rho, nu=sc.nu, frame_mode=sc.frame_mode,
                    precision="fp32", max_markers=sc.m)
b = EnvBatch(cfg, E)
for s in b.envs:
    s.set_skin(*sc.skin())
robot = D.koi_robot(sc.bodies[0], sc.articulations()[0])
rb = D.RobotBatch(robot, E); rb.set_rest(*D.rest_pose(robot))
for k in range(6):
    fr = np.stack([sc.frame(k + 37 * e).packed() for e in range(E)])
    st, fl, _ = b.step_dynamic(rb, np.zeros((E, robot.n_joints)), fr, sc.rho, (0, 0, -9.81), sc.dt, 4)
print("ok", st[0].stable(), fl)
