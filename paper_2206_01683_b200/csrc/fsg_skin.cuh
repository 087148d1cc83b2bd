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
struct SkinBody {  // (a multiple of 8 bytes: copied as doubles)
  int m0, m1;        // markers [m0, m1)
  int n_links, floating, n_dofs, tau_off;  // tau_off: first entry in the tau/stat output
  int parent[SKIN_L];
  int dof[SKIN_L];
  signed char anc[SKIN_L][SKIN_L];  // anc[b][l]: the (l+1)-th link up the chain from bone b
                                    // (anc[b][0] = b), -1 past the base (link 0)
  signed char lvl[SKIN_L][SKIN_L];  // lvl[b][J] = l >= 1 with anc[b][l-1] == J (J > 0), else -1
  signed char dof_link[6 + SKIN_L];  // link whose revolute dof is d (-1: base dof / none)
  signed char max_level;             // deepest joint chain (levels > 7 take a second lane pass)
  double axis[SKIN_L][3];
  fsg_body_pose pose;
};

// Kernel parameter block (passed as a __grid_constant__ parameter: the pose
// rides in the launch, no copy node and no pinned-memory read at the head of
// the step).  The kernels take SkinParamsN<NB> with NB in {1, 2, 4} (the
// smallest that holds the bodies) so a one-fish launch carries ~2 KB.
template <int NB>
struct SkinParamsN {
  int nb;
  int m;
  const double* rest;     // [3m] rest points
  const double* nrest;    // [3m] rest normals
  const int* wb;          // [m][SKIN_KW] bone of each nonzero weight, ascending; -1 = none
  const double* ww;       // [m][SKIN_KW] its weight
  double* part;           // tau scratch: [nb][blocks per body][ACC_N] partial sums
  unsigned* ticket;       // last-block counter (zero between launches)
  SkinBody body[NB];
};
using SkinParams = SkinParamsN<SKIN_NB>;  // host-side master copy
constexpr int SKIN_TAU_MAX = 6 + SKIN_L;  // dofs per body
constexpr int SKIN_ACC_N = SKIN_TAU_MAX + SKIN_NSTAT;
constexpr int SKIN_TAU_THREADS = 32;  // one warp per block: fits beside a full K4 SM

// update_samples: markers -> pts/vel/nrm (device arrays [3m] each)
void skin_update_launch(const SkinParams& P, double* pts, double* vel, double* nrm,
                        cudaStream_t s);
// tau_ext + CouplingStats per body from the marker forces of the step.
// serial = 1: one thread in the reference's order (bit-exact, parity mode);
// serial = 0: fixed-order tree (deterministic, throughput mode).
// out: per body, n_dofs tau entries at tau_off, then 7 stats at
// (sum of n_dofs) + 7*b.
struct MarkerStencil;
// km_done/km_blocks (throughput): the tree kernel is launched as a
// programmatic dependent of K4 (which triggers at its start) and spins until
// all km_blocks marker-kernel blocks have counted themselves done, so it runs
// beside K4's first phase; its last block resets *km_done.
void skin_tau_launch(const SkinParams& P, const double* fworld, const MarkerStencil* stencils,
                     const double* vel, double* out, int serial, unsigned* km_done,
                     unsigned km_blocks, cudaStream_t s);

}  // namespace fsg
