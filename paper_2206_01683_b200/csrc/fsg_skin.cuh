// fsg_skin.cuh -- skinned bodies on the device: types
// shared by the host session (fsg_session.cu) and the skin kernels
// (fsg_skin.cu, compiled without FMA contraction so the fp64 arithmetic is the
// reference's operation for operation).
#pragma once

#include <cuda_runtime.h>

#include "../../include/fsg.h"

namespace fsg {

constexpr int SKIN_L = FSG_SKIN_MAX_LINKS;
constexpr int SKIN_NB = FSG_SKIN_MAX_BODIES;
constexpr int SKIN_KW = FSG_SKIN_MAX_WEIGHTS;
constexpr int SKIN_NSTAT = 7;  // CouplingStats: force_on_fluid[3], force_on_body[3], power

// One skinned body: its marker range, topology and this step's pose.
struct SkinBody {
  int m0, m1;        // markers [m0, m1)
  int n_links, floating, n_dofs, tau_off;  // tau_off: first entry in the tau/stat output
  int parent[SKIN_L];
  int dof[SKIN_L];
  double axis[SKIN_L][3];
  fsg_body_pose pose;
};

// Kernel parameter block (passed as a __grid_constant__ parameter: the pose
// rides in the launch, no copy node and no pinned-memory read at the head of
// the step).
struct SkinParams {
  int nb;
  int m;
  const double* rest;     // [3m] rest points
  const double* nrest;    // [3m] rest normals
  const int* wb;          // [m][SKIN_KW] bone of each nonzero weight, ascending; -1 = none
  const double* ww;       // [m][SKIN_KW] its weight
  SkinBody body[SKIN_NB];
};

// update_samples: markers -> pts/vel/nrm (device arrays [3m] each)
void skin_update_launch(const SkinParams& P, double* pts, double* vel, double* nrm,
                        cudaStream_t s);
// tau_ext + CouplingStats per body from the marker forces of the step.
// serial = 1: one thread in the reference's order (bit-exact, parity mode);
// serial = 0: fixed-order tree (deterministic, throughput mode).
// out: per body, n_dofs tau entries at tau_off, then 7 stats at
// (sum of n_dofs) + 7*b.
struct MarkerStencil;
void skin_tau_launch(const SkinParams& P, const double* fworld, const MarkerStencil* stencils,
                     const double* vel, double* out, int serial, cudaStream_t s);

}  // namespace fsg
