// C++ host smoke test over include/fishgym_b200/session.hpp (the binding a
// FishGym maintainer would use).  Runs the reference KAT "Guo forcing injects
// exactly one unit of momentum per step" (test_lattice.cpp:189-202) and the
// resting-fluid open-boundary KAT (:135-145) through the C++ wrapper.
#include <cmath>
#include <cstdio>
#include <vector>

#include "fishgym_b200/session.hpp"

int main(int argc, char** argv) {
  using namespace fishgym_b200;
  const int prec = argc > 1 ? std::atoi(argv[1]) : FSG_PRECISION_FP64;
  // InputError for an unstable tau (units.hpp:56-68)
  {
    Config bad;
    bad.dims[0] = bad.dims[1] = bad.dims[2] = 16;
    bad.nu = 0.1;
    bad.dx = 0.02;
    try {
      FluidSession s(bad);
      std::printf("FAIL: no InputError\n");
      return 1;
    } catch (const InputError& e) {
      if (std::string(e.what()).find("tau") == std::string::npos) return 1;
    }
  }
  // FrameFollower (frame.hpp:70-125): a step toward a target 1 cm ahead starts
  // with pdd = wn^2 * 0.01 (wn = 5/s) and the yaw pinned in TranslationYaw
  {
    FrameFollower f(FSG_FRAME_TRANSLATION_YAW, 0.2);
    f.reset({0.0, 0.0, 0.0}, 0.5);
    f.step({0.01, 0.0, 0.0}, {1.0, 0.0, 0.0, 0.0}, 0.004);
    const FrameState st = f.state();
    if (std::fabs(st.pdd[0] - 25.0 * 0.01) > 1e-15 || st.omega[0] != 0.0 || st.q[1] != 0.0) {
      std::printf("FAIL: follower\n");
      return 4;
    }
  }
  Config c;
  c.dims[0] = c.dims[1] = c.dims[2] = 8;
  c.dx = c.dt = c.rho = 1.0;
  c.nu = (0.8 - 0.5) / 3.0;
  c.boundary = FSG_BOUNDARY_PERIODIC;
  c.frame_mode = FSG_FRAME_NONE;
  c.precision = prec;
  FluidSession s(c);
  std::vector<double> F(3 * s.n_cells(), 0.0);
  for (size_t k = 0; k < s.n_cells(); ++k) F[3 * k] = 1e-4;
  s.set_force(&F);
  for (int n = 0; n < 50; ++n)
    if (!s.collide_and_stream().stable()) return 2;
  std::vector<double> rho, u;
  s.macroscopic(rho, u);
  double worst = 0.0;
  for (size_t k = 0; k < s.n_cells(); ++k)
    worst = std::fmax(worst, std::fabs(u[3 * k] / (50.5 * 1e-4) - 1.0));
  const double tol = prec == FSG_PRECISION_FP64 ? 1e-10 : 1e-5;
  std::printf("guo_forcing_rel_err %.3e mass %.15f\n", worst, s.total_mass());
  return worst < tol ? 0 : 3;
}
