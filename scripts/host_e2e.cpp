// host_e2e -- end-to-end coupled steps from a C++ host through the C ABI
// (include/fsg.h), the way the FishGym binding in INTEGRATION.md drives it:
// every step uploads this step's frame and per-link poses from host memory,
// runs the coupled fluid step synchronously and reads tau_ext + CouplingStats
// back into host memory (fsg_step_skinned).  No Python on the timed path.
//
// Input: a flat binary written by bench.py (write_host_case):
//   int32  dims[3], frame_mode, n_bodies, n_steps, m
//   f64    dx, dt, rho, nu
//   int64  offsets[n_bodies + 1]
//   fsg_skeleton skeletons[n_bodies]
//   f64    rest_points[3m], rest_normals[3m], areas[m], weights[sum_b m_b * n_links_b]
//   fsg_frame_state frames[n_steps]
//   fsg_body_pose   poses[n_steps][n_bodies]
// Output (stdout, one JSON line): steps, us_per_step (wall, median of 3
// rounds), mlups, the last status.
//
//   g++ -O2 -std=c++17 -I include scripts/host_e2e.cpp -L paper_2206_01683_b200 -lfsg \
//       -Wl,-rpath,paper_2206_01683_b200 -o host_e2e && ./host_e2e case.bin [warmup]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fsg.h"

namespace {
template <class T>
bool rd(FILE* f, T* p, size_t n) {
  return std::fread(p, sizeof(T), n, f) == n;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: host_e2e case.bin [warmup]\n");
    return 2;
  }
  const int warm = argc > 2 ? std::atoi(argv[2]) : 5;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  int hdr[7];
  double ph[4];
  if (!rd(f, hdr, 7) || !rd(f, ph, 4)) return 2;
  const int nb = hdr[4], ns = hdr[5], m = hdr[6];
  std::vector<int64_t> off(nb + 1);
  std::vector<fsg_skeleton> sk(nb);
  if (!rd(f, off.data(), off.size()) || !rd(f, sk.data(), sk.size())) return 2;
  size_t nw = 0;
  for (int b = 0; b < nb; ++b) nw += (size_t)(off[b + 1] - off[b]) * sk[b].n_links;
  std::vector<double> rest(3 * (size_t)m), nrest(3 * (size_t)m), area(m), w(nw);
  if (!rd(f, rest.data(), rest.size()) || !rd(f, nrest.data(), nrest.size()) ||
      !rd(f, area.data(), area.size()) || !rd(f, w.data(), w.size()))
    return 2;
  std::vector<fsg_frame_state> frames(ns);
  std::vector<fsg_body_pose> poses((size_t)ns * nb);
  if (!rd(f, frames.data(), frames.size()) || !rd(f, poses.data(), poses.size())) return 2;
  std::fclose(f);

  fsg_config c{};
  c.dims[0] = hdr[0];
  c.dims[1] = hdr[1];
  c.dims[2] = hdr[2];
  c.dx = ph[0];
  c.dt = ph[1];
  c.rho = ph[2];
  c.nu = ph[3];
  c.boundary = FSG_BOUNDARY_OPEN;
  c.kernel = FSG_KERNEL_PESKIN4;
  c.wall = FSG_WALL_SLIP;
  c.frame_mode = hdr[3];
  c.precision = FSG_PRECISION_FP32;
  c.max_markers = m;
  c.nz_global = hdr[2];
  fsg_session* s = nullptr;
  if (fsg_create(&c, &s)) {
    std::fprintf(stderr, "fsg_create: %s\n", fsg_last_error());
    return 1;
  }
  if (fsg_set_skin(s, nb, off.data(), sk.data(), rest.data(), nrest.data(), w.data(), area.data())) {
    std::fprintf(stderr, "fsg_set_skin: %s\n", fsg_last_error());
    return 1;
  }
  int nt = 0;
  for (int b = 0; b < nb; ++b) nt += sk[b].n_dofs;
  std::vector<double> tau(nt), stats(7 * (size_t)nb);
  fsg_status st{};
  auto step = [&](int k) {
    return fsg_step_skinned(s, &frames[k % ns], &poses[(size_t)(k % ns) * nb], &st, tau.data(),
                            stats.data());
  };
  for (int k = 0; k < warm; ++k)
    if (step(k)) {
      std::fprintf(stderr, "step: %s\n", fsg_last_error());
      return 1;
    }
  std::vector<double> us;
  for (int round = 0; round < 3; ++round) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < ns; ++k)
      if (step(warm + k)) return 1;
    const auto t1 = std::chrono::steady_clock::now();
    us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count() / ns);
  }
  std::sort(us.begin(), us.end());
  const double cells = (double)hdr[0] * hdr[1] * hdr[2];
  if (std::getenv("HOST_E2E_SPLIT")) {  // dev: host time to enqueue vs to wait, per step
    std::vector<double> ta, tl, tw;
    for (int k = 0; k < ns; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      fsg_set_frame(s, &frames[k]);
      fsg_set_pose(s, &poses[(size_t)k * nb]);
      const auto ta0 = std::chrono::steady_clock::now();
      fsg_step_async(s);
      const auto t1 = std::chrono::steady_clock::now();
      fsg_last_status(s, &st);
      const auto t2 = std::chrono::steady_clock::now();
      ta.push_back(std::chrono::duration<double, std::micro>(ta0 - t0).count());
      tl.push_back(std::chrono::duration<double, std::micro>(t1 - ta0).count());
      tw.push_back(std::chrono::duration<double, std::micro>(t2 - t1).count());
    }
    std::sort(ta.begin(), ta.end());
    std::sort(tl.begin(), tl.end());
    std::sort(tw.begin(), tw.end());
    std::fprintf(stderr, "set frame+pose %.2f us, enqueue %.2f us, wait %.2f us (medians)\n", ta[ns / 2],
                 tl[ns / 2], tw[ns / 2]);
  }
  std::printf("{\"steps\": %d, \"us_per_step\": %.2f, \"mlups\": %.1f, \"stable\": %d, \"min_f\": %.6g}\n",
              ns, us[1], cells / us[1], st.finite && st.n_nonpositive_rho == 0 ? 1 : 0, st.min_f);
  fsg_destroy(s);
  return 0;
}
