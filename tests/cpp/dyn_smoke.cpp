// C++ host program over include/fishgym_b200/session.hpp: the reference's
// pendulum KAT (test_robot.cpp:113-139) on the device robot dynamics, and
// Skeleton::validate through the wrapper (test_robot.cpp:346-363).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include <fishgym_b200/session.hpp>

using fishgym_b200::RobotDynamics;

static fsg_robot pendulum(double len, double mass) {
  fsg_robot r;
  std::memset(&r, 0, sizeof r);
  r.n_links = 2;
  for (int i = 0; i < 2; ++i)
    for (int k = 0; k < 9; ++k) r.links[i].joint_rotation[k] = (k % 4 == 0) ? 1.0 : 0.0;
  fsg_link& b = r.links[0];  // base_link(Fixed), test_robot.cpp:17-25
  b.parent = -1, b.joint = FSG_JOINT_FIXED, b.mass = 1.0;
  b.inertia_com[0] = b.inertia_com[4] = b.inertia_com[8] = 1e-3;
  fsg_link& l = r.links[1];  // make_chain(1, len, mass, Fixed, along_x = false)
  l.parent = 0, l.joint = FSG_JOINT_REVOLUTE, l.axis[1] = 1.0, l.mass = mass, l.com[2] = -0.5 * len;
  const double i_rod = mass * len * len / 12.0;
  l.inertia_com[0] = l.inertia_com[4] = i_rod, l.inertia_com[8] = 1e-7;
  l.limit_lo = -3.0, l.limit_hi = 3.0, l.torque_limit = 100.0;
  return r;
}

int main() {
  const double len = 0.5, mass = 0.3, g[3] = {0.0, 0.0, -9.81};
  RobotDynamics rd(pendulum(len, mass), 1);
  std::vector<fsg_joint_state> st(1);
  std::memset(st.data(), 0, sizeof(fsg_joint_state));
  st[0].base_quat[0] = 1.0;
  st[0].q[0] = 0.05;
  rd.set_states(st);
  const double period = 2.0 * M_PI / std::sqrt(3.0 * 9.81 / (2.0 * len)), dt = 1e-4;
  const int steps = static_cast<int>(10.5 * period / dt);
  std::vector<double> crossings;
  double prev = 0.05;
  const std::vector<double> act(1, 0.0);
  for (int k = 0; k < steps; ++k) {  // integrate(..., dt, 1, kGravity) per step
    rd.step(act, {}, 1000.0, nullptr, dt, 1, g);
    const double q = rd.states()[0].q[0];
    if (prev < 0.0 && q >= 0.0) crossings.push_back((k - prev / (q - prev)) * dt);
    prev = q;
  }
  const double measured = (crossings.back() - crossings.front()) / (crossings.size() - 1);
  const double err = std::abs(measured / period - 1.0);
  std::printf("pendulum_period_rel_err %.3e crossings %zu\n", err, crossings.size());
  if (crossings.size() < 10 || !(err < 0.005)) return 1;
  fsg_robot bad = pendulum(len, mass);
  bad.links[1].limit_lo = 4.0;
  try {
    RobotDynamics x(bad, 1);
    return 2;
  } catch (const fishgym_b200::InputError& e) {
    std::printf("validate: %s\n", e.what());
  }
  return 0;
}
