"""Dev probe: device robot step (fsg_dyn_step_device) time per batched step vs
the fp64 restatement on one host core (koi, 4 substeps, hydrostatics)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2206_01683_b200 import dynamics as D
from paper_2206_01683_b200.scenes import koi_articulation, koi_body
from oracle import bind as B
G = np.array([0, 0, -9.81])
body = koi_body(0.01); robot = D.koi_robot(body, koi_articulation(body))
for E, kern in [(E, k) for E in (8, 64, 512, 4096) for k in ("warp", "thread")]:
    os.environ["FSG_DYN_WARP_MAX"] = "1000000" if kern == "warp" else "0"
    rb = D.RobotBatch(robot, E)
    act = torch.zeros(E, robot.n_joints, dtype=torch.float64, device="cuda")
    tau = torch.zeros(E, robot.n_dofs, dtype=torch.float64, device="cuda")
    for _ in range(5): rb.step_device(act, tau, 1000.0, G, 0.004, 4)
    rb.states()
    t0 = time.perf_counter(); n = 200
    for _ in range(n): rb.step_device(act, tau, 1000.0, G, 0.004, 4)
    rb.states(); dt = (time.perf_counter() - t0) / n
    print(f"{kern} E={E}: {dt*1e6:.1f} us per batched step (wall, incl. launch) = {E/dt:.0f} env-steps/s")
O = B.DynOracle(robot); st = D.JointState.zero(robot); a = np.zeros(robot.n_joints)
t0 = time.perf_counter(); n = 2000
for _ in range(n): O.robot_step(st, a, None, 1000.0, G, 0.004, 4)
dt = (time.perf_counter() - t0) / n
print(f"oracle 1 core: {dt*1e6:.1f} us per env-step = {1/dt:.0f} env-steps/s")
