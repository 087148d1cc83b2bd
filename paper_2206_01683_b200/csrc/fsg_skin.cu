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

template <int NB>
__device__ __forceinline__ int body_of(const SkinParamsN<NB>& P, int i) {
  int b = 0;
#pragma unroll
  for (int k = 1; k < NB; ++k)
    if (k < P.nb && i >= P.body[k].m0) b = k;
  return b;
}

/// Copy bodies [b0, b1) of the parameter block into shared memory: the
/// kernels index the pose by runtime bone / link numbers, and dependent
/// constant-bank loads at runtime offsets (cold constant cache, one unique
/// address at a time) cost far more than one staged copy per block.
template <int NB>
__device__ __forceinline__ void stage_bodies(const SkinParamsN<NB>& P, SkinBody* dst, int b0, int b1) {
  static_assert(sizeof(SkinBody) % 8 == 0, "SkinBody is copied as doubles");
  constexpr int NW = (int)(sizeof(SkinBody) / 8);
  for (int b = b0; b < b1; ++b) {
    const double* src = reinterpret_cast<const double*>(&P.body[b]);
    double* d = reinterpret_cast<double*>(dst + (b - b0));
    for (int w = threadIdx.x; w < NW; w += blockDim.x) d[w] = src[w];
  }
  __syncthreads();
}

/// BoneTransforms::apply (skinning.hpp:101): R[b] * x + t[b]
__device__ __forceinline__ void bone_apply(const fsg_body_pose& Q, int b, const double* x, double* xb) {
  mv(Q.bone_R[b], x, xb);
#pragma unroll
  for (int c = 0; c < 3; ++c) xb[c] = xb[c] + Q.bone_t[b][c];
}

template <int NB>
__global__ void __launch_bounds__(64)
    k_skin_update(const __grid_constant__ SkinParamsN<NB> P, double* __restrict__ pts,
                  double* __restrict__ vel, double* __restrict__ nrm) {
  // the marker kernel is this kernel's programmatic dependent: let it launch
  // (it waits for this grid's completion before reading the markers)
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ SkinBody sb[NB];
  stage_bodies(P, sb, 0, P.nb);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.m) return;
  const fsg_body_pose& Q = sb[body_of(P, i)].pose;
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

constexpr int TAU_MAX = SKIN_TAU_MAX;
constexpr int ACC_N = SKIN_ACC_N;

/// acc[d] += v for a runtime d, with acc kept in registers (every slot is a
/// compile-time index; the others are left untouched, not added to).
__device__ __forceinline__ void acc_add(double* acc, int d, double v) {
#pragma unroll
  for (int k = 0; k < TAU_MAX; ++k)
    if (k == d) acc[k] = acc[k] + v;
}

/// One marker's contribution (reference order) into acc[0..n_dofs) and the
/// stats into acc[TAU_MAX..TAU_MAX+7).
template <int NB>
__device__ __forceinline__ void marker_contrib(const SkinParamsN<NB>& P, const SkinBody& B, int i,
                                               const double* __restrict__ fworld,
                                               const double* __restrict__ vel, double* acc) {
  const fsg_body_pose& Q = B.pose;
  const double f[3] = {__ldcg(fworld + 3 * i), __ldcg(fworld + 3 * i + 1), __ldcg(fworld + 3 * i + 2)};
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
      acc_add(acc, dof, dot3(cr, fv));
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

template <int NB>
__device__ __forceinline__ int tau_total(const SkinParamsN<NB>& P) {
  int n = 0;
  for (int b = 0; b < P.nb; ++b) n += P.body[b].n_dofs;
  return n;
}

/// Parity: one thread, bodies and markers in the reference's order.
template <int NB>
__global__ void k_skin_tau_serial(const __grid_constant__ SkinParamsN<NB> P,
                                  const double* __restrict__ fworld,
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

/// Throughput: grid (blocks per body, bodies) of one-warp blocks, launched as
/// a programmatic dependent of K4 so it runs beside K4's first phase: spin
/// until the marker kernel has counted all its blocks done, then one marker
/// per thread, a fixed warp butterfly per block, and the last block to finish
/// (ticket) sums the block partials of every body in block order.
/// Deterministic run to run.
constexpr int TAU_THREADS = SKIN_TAU_THREADS;
constexpr int TAU_STAGE = 2016;  // doubles of block partials staged per pass (96 blocks)
template <int NB>
__global__ void __launch_bounds__(TAU_THREADS)
    k_skin_tau(const __grid_constant__ SkinParamsN<NB> P, const double* __restrict__ fworld,
               const MarkerStencil* __restrict__ ms, const double* __restrict__ vel, double* out,
               unsigned* km_done, unsigned km_blocks) {
  __shared__ double part[TAU_THREADS / 32][ACC_N];
  __shared__ double stage[TAU_STAGE];
  __shared__ bool last;
  if (km_done) {
    if (threadIdx.x == 0)
      while (*(volatile unsigned*)km_done < km_blocks) __nanosleep(64);
    __syncthreads();
    __threadfence();
  }
  const int b = blockIdx.y;
  __shared__ SkinBody sb[1];
  stage_bodies(P, sb, b, b + 1);
  const SkinBody& B = sb[0];
  double acc[ACC_N];
#pragma unroll
  for (int k = 0; k < ACC_N; ++k) acc[k] = 0.0;
  const int i = B.m0 + blockIdx.x * TAU_THREADS + threadIdx.x;
  if (i < B.m1 && __ldcg(&ms[i].valid)) marker_contrib(P, B, i, fworld, vel, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < ACC_N; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[warp][k] = v;
  }
  __syncthreads();
  const int bpb = gridDim.x;
  if (threadIdx.x < ACC_N) {
    const int k = threadIdx.x;
    double v = part[0][k];
    for (int w = 1; w < TAU_THREADS / 32; ++w) v = v + part[w][k];
    P.part[((size_t)b * bpb + blockIdx.x) * ACC_N + k] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(P.ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // every body's block partials: staged into shared memory with independent
  // loads (one L2 round trip per chunk), then summed in block order
  const int nt = tau_total(P);
  constexpr int CH = TAU_STAGE / ACC_N;  // blocks per chunk
  for (int bb = 0; bb < P.nb; ++bb) {
    double v = 0.0;  // lane k < ACC_N owns component k
    for (int j0 = 0; j0 < bpb; j0 += CH) {
      const int nj = min(CH, bpb - j0);
      const double* src = P.part + ((size_t)bb * bpb + j0) * ACC_N;
      __syncwarp();
      for (int t = threadIdx.x; t < nj * ACC_N; t += TAU_THREADS) stage[t] = __ldcg(src + t);
      __syncwarp();
      if (threadIdx.x < ACC_N)
        for (int j = 0; j < nj; ++j) v = (j0 + j == 0) ? stage[threadIdx.x] : v + stage[j * ACC_N + threadIdx.x];
    }
    const int k = threadIdx.x;
    if (k < ACC_N) {
      if (k < P.body[bb].n_dofs) out[P.body[bb].tau_off + k] = v;
      if (k >= TAU_MAX) out[nt + SKIN_NSTAT * bb + (k - TAU_MAX)] = v;
    }
  }
  if (threadIdx.x == 0) {
    *P.ticket = 0u;
    if (km_done) *km_done = 0u;
  }
}

template <int NB>
SkinParamsN<NB> narrow(const SkinParams& P) {
  SkinParamsN<NB> q;
  q.nb = P.nb;
  q.m = P.m;
  q.rest = P.rest;
  q.nrest = P.nrest;
  q.wb = P.wb;
  q.ww = P.ww;
  q.part = P.part;
  q.ticket = P.ticket;
  for (int b = 0; b < NB; ++b) q.body[b] = P.body[b];
  return q;
}

template <int NB>
void update_nb(const SkinParams& P, double* pts, double* vel, double* nrm, cudaStream_t s) {
  k_skin_update<NB><<<(P.m + 63) / 64, 64, 0, s>>>(narrow<NB>(P), pts, vel, nrm);
}

template <int NB>
void tau_nb(const SkinParams& P, const double* fworld, const MarkerStencil* ms, const double* vel,
            double* out, int serial, unsigned* km_done, unsigned km_blocks, cudaStream_t s) {
  if (serial) {
    k_skin_tau_serial<NB><<<1, 32, 0, s>>>(narrow<NB>(P), fworld, ms, vel, out);
    return;
  }
  int mmax = 1;
  for (int b = 0; b < P.nb; ++b) mmax = mmax > P.body[b].m1 - P.body[b].m0 ? mmax : P.body[b].m1 - P.body[b].m0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((mmax + TAU_THREADS - 1) / TAU_THREADS), (unsigned)P.nb);
  cfg.blockDim = dim3(TAU_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = km_done ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_skin_tau<NB>, narrow<NB>(P), fworld, ms, vel, out, km_done, km_blocks);
}

}  // namespace

void skin_update_launch(const SkinParams& P, double* pts, double* vel, double* nrm, cudaStream_t s) {
  if (P.m <= 0) return;
  if (P.nb <= 1) update_nb<1>(P, pts, vel, nrm, s);
  else if (P.nb <= 2) update_nb<2>(P, pts, vel, nrm, s);
  else update_nb<4>(P, pts, vel, nrm, s);
}

void skin_tau_launch(const SkinParams& P, const double* fworld, const MarkerStencil* ms,
                     const double* vel, double* out, int serial, unsigned* km_done,
                     unsigned km_blocks, cudaStream_t s) {
  if (P.nb <= 0) return;
  if (P.nb <= 1) tau_nb<1>(P, fworld, ms, vel, out, serial, km_done, km_blocks, s);
  else if (P.nb <= 2) tau_nb<2>(P, fworld, ms, vel, out, serial, km_done, km_blocks, s);
  else tau_nb<4>(P, fworld, ms, vel, out, serial, km_done, km_blocks, s);
}

}  // namespace fsg
