// fsg_skin.cu -- skinned bodies on the device.
//
//   k_skin_update : robot::update_samples (sampling.hpp:307-322) -- linear
//                   blend skinning of each marker's rest point
//                   (skin_point, skinning.hpp:105-112), its exact velocity
//                   (skin_point_velocity, :116-126) and its normal.
//   k_skin_tau    : tau_ext += J^T(-f_world) per valid marker
//                   (accumulate_skinned_force, skinning.hpp:147-156 ->
//                   accumulate_point_force, dynamics.hpp:216-233) and the
//                   CouplingStats sums (session.hpp:139-143).
//
// Compiled with --fmad=false: every product and sum is the reference's, in
// Eigen 3.4's coefficient order for these fixed sizes (oracle/eigen_shim):
// mat*vec and dot ((a0 b0 + a1 b1) + a2 b2), cross3, v / sqrt(|v|^2).  The
// serial tau kernel therefore reproduces the reference bit for bit (parity
// mode); the tree variant sums per-thread partials in a fixed order
// (deterministic, throughput mode).
#include "fsg_device.cuh"
#include "fsg_skin.cuh"

namespace fsg {
namespace {

__device__ __forceinline__ void mv(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = (R[3 * i] * v[0] + R[3 * i + 1] * v[1]) + R[3 * i + 2] * v[2];
}
__device__ __forceinline__ void mtv(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = (R[i] * v[0] + R[3 + i] * v[1]) + R[6 + i] * v[2];
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

__device__ __forceinline__ int body_of(const SkinParams& P, int i) {
  int b = 0;
  while (b + 1 < P.nb && i >= P.body[b].m1) ++b;
  return b;
}

/// BoneTransforms::apply (skinning.hpp:101): R[b] * x + t[b]
__device__ __forceinline__ void bone_apply(const fsg_body_pose& Q, int b, const double* x, double* xb) {
  mv(Q.bone_R[b], x, xb);
#pragma unroll
  for (int c = 0; c < 3; ++c) xb[c] = xb[c] + Q.bone_t[b][c];
}

__global__ void k_skin_update(const __grid_constant__ SkinParams P, double* __restrict__ pts,
                              double* __restrict__ vel, double* __restrict__ nrm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.m) return;
  const fsg_body_pose& Q = P.body[body_of(P, i)].pose;
  const double x[3] = {P.rest[3 * i], P.rest[3 * i + 1], P.rest[3 * i + 2]};
  const double n0[3] = {P.nrest[3 * i], P.nrest[3 * i + 1], P.nrest[3 * i + 2]};
  double out[3] = {0.0, 0.0, 0.0}, vout[3] = {0.0, 0.0, 0.0}, nn[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < SKIN_KW; ++k) {
    const int b = P.wb[SKIN_KW * i + k];
    if (b < 0) break;
    const double w = P.ww[SKIN_KW * i + k];
    double xb[3], d[3], cr[3], rn[3];
    bone_apply(Q, b, x, xb);                      // skin_point: out += w * apply(b, x)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[c] = out[c] + w * xb[c];
      d[c] = xb[c] - Q.p_world[b][c];
    }
    cross3(Q.omega_world[b], d, cr);              // skin_point_velocity
#pragma unroll
    for (int c = 0; c < 3; ++c) vout[c] = vout[c] + w * (Q.v_origin_world[b][c] + cr[c]);
    mv(Q.bone_R[b], n0, rn);                      // normals: nrm += w * (R[b] * n_rest)
#pragma unroll
    for (int c = 0; c < 3; ++c) nn[c] = nn[c] + w * rn[c];
  }
  const double z = dot3(nn, nn);                  // normalized()
  if (z > 0.0) {
    const double sz = sqrt(z);
#pragma unroll
    for (int c = 0; c < 3; ++c) nn[c] = nn[c] / sz;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    pts[3 * i + c] = out[c];
    vel[3 * i + c] = vout[c];
    nrm[3 * i + c] = nn[c];
  }
}

constexpr int TAU_MAX = 6 + SKIN_L;      // dofs per body
constexpr int ACC_N = TAU_MAX + SKIN_NSTAT;

/// One marker's contribution (reference order) into acc[0..n_dofs) and the
/// stats into acc[TAU_MAX..TAU_MAX+7).
__device__ __forceinline__ void marker_contrib(const SkinParams& P, const SkinBody& B, int i,
                                               const double* __restrict__ fworld,
                                               const double* __restrict__ vel, double* acc) {
  const fsg_body_pose& Q = B.pose;
  const double f[3] = {fworld[3 * i], fworld[3 * i + 1], fworld[3 * i + 2]};
  const double fneg[3] = {-f[0], -f[1], -f[2]};
  const double x[3] = {P.rest[3 * i], P.rest[3 * i + 1], P.rest[3 * i + 2]};
  for (int k = 0; k < SKIN_KW; ++k) {
    const int b = P.wb[SKIN_KW * i + k];
    if (b < 0) break;
    const double w = P.ww[SKIN_KW * i + k];
    double p[3], fv[3];
    bone_apply(Q, b, x, p);
#pragma unroll
    for (int c = 0; c < 3; ++c) fv[c] = w * fneg[c];  // w[b] * f_world (f_world = -f)
    if (B.floating) {  // tau.head<3>() += R0^T ((p - p0) x f);  tau.segment<3>(3) += R0^T f
      double d[3], cr[3], h[3], g[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = p[c] - Q.p_world[0][c];
      cross3(d, fv, cr);
      mtv(Q.R_world[0], cr, h);
      mtv(Q.R_world[0], fv, g);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        acc[c] = acc[c] + h[c];
        acc[3 + c] = acc[3 + c] + g[c];
      }
    }
    for (int j = b; j > 0; j = B.parent[j]) {
      const int dof = B.dof[j];
      if (dof < 0) continue;  // not revolute
      double aw[3], d[3], cr[3];
      mv(Q.R_world[j], B.axis[j], aw);
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = p[c] - Q.p_world[j][c];
      cross3(aw, d, cr);
      acc[dof] = acc[dof] + dot3(cr, fv);
    }
  }
  double* st = acc + TAU_MAX;  // CouplingStats
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    st[c] = st[c] + f[c];
    st[3 + c] = st[3 + c] - f[c];
  }
  const double v[3] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
  st[6] = st[6] + dot3(fneg, v);
}

__device__ __forceinline__ int tau_total(const SkinParams& P) {
  int n = 0;
  for (int b = 0; b < P.nb; ++b) n += P.body[b].n_dofs;
  return n;
}

/// Parity: one thread, bodies and markers in the reference's order.
__global__ void k_skin_tau_serial(const __grid_constant__ SkinParams P, const double* __restrict__ fworld,
                                  const MarkerStencil* __restrict__ ms, const double* __restrict__ vel,
                                  double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int nt = tau_total(P);
  for (int b = 0; b < P.nb; ++b) {
    const SkinBody& B = P.body[b];
    double acc[ACC_N];
    for (int k = 0; k < ACC_N; ++k) acc[k] = 0.0;
    for (int i = B.m0; i < B.m1; ++i)
      if (ms[i].valid) marker_contrib(P, B, i, fworld, vel, acc);
    for (int d = 0; d < B.n_dofs; ++d) out[B.tau_off + d] = acc[d];
    for (int k = 0; k < SKIN_NSTAT; ++k) out[nt + SKIN_NSTAT * b + k] = acc[TAU_MAX + k];
  }
}

/// Throughput: one block per body; thread t sums markers t, t + T, ... in
/// ascending order, then a fixed warp butterfly and a fixed in-order sum of
/// the warp partials.  Deterministic run to run.
constexpr int TAU_THREADS = 256;
__global__ void __launch_bounds__(TAU_THREADS)
    k_skin_tau(const __grid_constant__ SkinParams P, const double* __restrict__ fworld,
               const MarkerStencil* __restrict__ ms, const double* __restrict__ vel, double* out) {
  __shared__ double part[TAU_THREADS / 32][ACC_N];
  const int b = blockIdx.x;
  const SkinBody& B = P.body[b];
  double acc[ACC_N];
#pragma unroll
  for (int k = 0; k < ACC_N; ++k) acc[k] = 0.0;
  for (int i = B.m0 + threadIdx.x; i < B.m1; i += TAU_THREADS)
    if (ms[i].valid) marker_contrib(P, B, i, fworld, vel, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < ACC_N; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < ACC_N) {
    const int k = threadIdx.x;
    double v = part[0][k];
    for (int w = 1; w < TAU_THREADS / 32; ++w) v = v + part[w][k];
    const int nt = tau_total(P);
    if (k < B.n_dofs) out[B.tau_off + k] = v;
    if (k >= TAU_MAX) out[nt + SKIN_NSTAT * b + (k - TAU_MAX)] = v;
  }
}

}  // namespace

void skin_update_launch(const SkinParams& P, double* pts, double* vel, double* nrm, cudaStream_t s) {
  if (P.m <= 0) return;
  k_skin_update<<<(P.m + 127) / 128, 128, 0, s>>>(P, pts, vel, nrm);
}

void skin_tau_launch(const SkinParams& P, const double* fworld, const MarkerStencil* ms,
                     const double* vel, double* out, int serial, cudaStream_t s) {
  if (P.nb <= 0) return;
  if (serial)
    k_skin_tau_serial<<<1, 32, 0, s>>>(P, fworld, ms, vel, out);
  else
    k_skin_tau<<<P.nb, TAU_THREADS, 0, s>>>(P, fworld, ms, vel, out);
}

}  // namespace fsg
