// fsg_drag.cu -- the empirical-drag backend's per-step surface work as a
// batched device kernel: for E envs of one robot each,
// EmpiricalBackend::step (empirical.hpp:74-100) up to the robot integration:
//   update_samples (sampling.hpp:307-322)            -> velocity, normal
//   surface_force (empirical.hpp:25-30)              F = -k (n.v) n A if n.v > 0
//   skip if f.isZero() (Eigen: every |f_c| <= 1e-12)
//   accumulate_skinned_force(..., +f, tau_ext)       (skinning.hpp:147-156)
//   total_force_on_body += f; power_on_body += f.v   (empirical.hpp:88-89)
// Forward kinematics, buoyancy and integrate stay with the host robot code.
//
// Compiled with --fmad=false: fp64, the reference's operation order.  Parity
// mode: one thread per env walks its markers in order (bit-identical to the
// reference loop).  Throughput mode: one thread per marker over every env,
// each marker's terms added to the env's 64-bit fixed-point sums (2^-44;
// integer atomics, deterministic), one small kernel converts them.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "fsg_device.cuh"
#include "fsg_skin.cuh"

namespace fsg {
namespace {

constexpr int DRAG_ACC = 32;  // per env: dofs 0..17, stats 18..24, non-finite flag 25

struct DragDev {
  int E, m;
  const double* rest;   // [3m]
  const double* nrest;  // [3m]
  const int* wb;        // [m][SKIN_KW]
  const double* ww;     // [m][SKIN_KW]
  const double* area;   // [m]
  const int* env;       // [m] env of each marker
  const int* m0;        // [E + 1] marker ranges
  const SkinBody* bodies;  // [E] topology + this step's pose
  double k;
  unsigned long long* acc;  // [E][DRAG_ACC]
};

__device__ __forceinline__ void d_mv(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = (R[3 * i] * v[0] + R[3 * i + 1] * v[1]) + R[3 * i + 2] * v[2];
}
__device__ __forceinline__ void d_mtv(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = (R[i] * v[0] + R[3 + i] * v[1]) + R[6 + i] * v[2];
}
__device__ __forceinline__ void d_cross(const double* a, const double* b, double* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ double d_dot(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}
__device__ __forceinline__ void d_apply(const fsg_body_pose& Q, int b, const double* x, double* xb) {
  d_mv(Q.bone_R[b], x, xb);
#pragma unroll
  for (int c = 0; c < 3; ++c) xb[c] = xb[c] + Q.bone_t[b][c];
}

/// Marker i's drag force (world) and velocity; false when f.isZero().
__device__ __forceinline__ bool drag_force(const DragDev& D, const SkinBody& B, int i, double* f,
                                           double* vel) {
  const fsg_body_pose& Q = B.pose;
  const double x[3] = {D.rest[3 * i], D.rest[3 * i + 1], D.rest[3 * i + 2]};
  const double n0[3] = {D.nrest[3 * i], D.nrest[3 * i + 1], D.nrest[3 * i + 2]};
  double v[3] = {0.0, 0.0, 0.0}, nn[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < SKIN_KW; ++k) {  // skin_point_velocity + normals (sampling.hpp:313-319)
    const int b = D.wb[SKIN_KW * i + k];
    if (b < 0) break;
    const double w = D.ww[SKIN_KW * i + k];
    double xb[3], d[3], cr[3], rn[3];
    d_apply(Q, b, x, xb);
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = xb[c] - Q.p_world[b][c];
    d_cross(Q.omega_world[b], d, cr);
    d_mv(Q.bone_R[b], n0, rn);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      v[c] = v[c] + w * (Q.v_origin_world[b][c] + cr[c]);
      nn[c] = nn[c] + w * rn[c];
    }
  }
  const double z = d_dot(nn, nn);
  if (z > 0.0) {
    const double sz = sqrt(z);
#pragma unroll
    for (int c = 0; c < 3; ++c) nn[c] = nn[c] / sz;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) vel[c] = v[c];
  const double vn = d_dot(nn, v);  // surface_force (empirical.hpp:25-30)
  if (vn <= 0.0) return false;
  const double s = ((-D.k) * vn) * D.area[i];
#pragma unroll
  for (int c = 0; c < 3; ++c) f[c] = s * nn[c];
  // !f.isZero(): Eigen's isZero is |f_k| <= 1e-12 for every k, so a NaN force
  // is NOT zero and is accumulated (the reference propagates it)
  return !(fabs(f[0]) <= 1e-12 && fabs(f[1]) <= 1e-12 && fabs(f[2]) <= 1e-12);
}

/// accumulate_skinned_force(..., f, tau) and the stats into acc (reference order).
__device__ __forceinline__ void drag_contrib(const DragDev& D, const SkinBody& B, int i, const double* f,
                                             const double* vel, double* acc) {
  const fsg_body_pose& Q = B.pose;
  const double x[3] = {D.rest[3 * i], D.rest[3 * i + 1], D.rest[3 * i + 2]};
  for (int k = 0; k < SKIN_KW; ++k) {
    const int b = D.wb[SKIN_KW * i + k];
    if (b < 0) break;
    const double w = D.ww[SKIN_KW * i + k];
    double p[3], fv[3];
    d_apply(Q, b, x, p);
#pragma unroll
    for (int c = 0; c < 3; ++c) fv[c] = w * f[c];
    if (B.floating) {
      double d[3], cr[3], h[3], g[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = p[c] - Q.p_world[0][c];
      d_cross(d, fv, cr);
      d_mtv(Q.R_world[0], cr, h);
      d_mtv(Q.R_world[0], fv, g);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        acc[c] = acc[c] + h[c];
        acc[3 + c] = acc[3 + c] + g[c];
      }
    }
    for (int j = b; j > 0; j = B.parent[j]) {
      const int dof = B.dof[j];
      if (dof < 0) continue;
      double aw[3], d[3], cr[3];
      d_mv(Q.R_world[j], B.axis[j], aw);
#pragma unroll
      for (int c = 0; c < 3; ++c) d[c] = p[c] - Q.p_world[j][c];
      d_cross(aw, d, cr);
#pragma unroll
      for (int q = 0; q < SKIN_TAU_MAX; ++q)
        if (q == dof) acc[q] = acc[q] + d_dot(cr, fv);
    }
  }
  double* st = acc + SKIN_TAU_MAX;  // force on body += f; power += f.v
#pragma unroll
  for (int c = 0; c < 3; ++c) st[3 + c] = st[3 + c] + f[c];
  st[6] = st[6] + d_dot(f, vel);
}

__global__ void __launch_bounds__(128) k_drag(DragDev D) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.m) return;
  const int e = D.env[i];
  const SkinBody& B = D.bodies[e];
  double f[3], vel[3];
  if (!drag_force(D, B, i, f, vel)) return;
  double acc[SKIN_ACC_N];
#pragma unroll
  for (int q = 0; q < SKIN_ACC_N; ++q) acc[q] = 0.0;
  drag_contrib(D, B, i, f, vel, acc);
  unsigned long long* dst = D.acc + (size_t)e * DRAG_ACC;
#pragma unroll
  for (int q = 0; q < SKIN_ACC_N; ++q) {
    if (!(fabs(acc[q]) < SKIN_FIX_RANGE)) atomicOr(dst + SKIN_ACC_N, 1ull);  // non-finite flag
    else if (acc[q] != 0.0) atomicAdd(dst + q, (unsigned long long)__double2ll_rn(acc[q] * SKIN_FIX_SCALE));
  }
}

/// Converts (and re-zeroes) every env's sums: tau at tau_off[e], then 7 stats
/// per env after all the taus.
__global__ void k_drag_finish(DragDev D, const int* tau_off, const int* ndof, int nt, double* out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < D.E * DRAG_ACC; t += gridDim.x * blockDim.x) {
    const int e = t / DRAG_ACC, q = t % DRAG_ACC;
    if (q >= SKIN_ACC_N) continue;
    // a non-finite or out-of-range term anywhere in the env (flag word after
    // its sums) makes every sum NaN, as the reference's would be
    const bool bad = D.acc[(size_t)e * DRAG_ACC + SKIN_ACC_N] != 0ull;
    const double v = bad ? __longlong_as_double(0x7ff8000000000000ll)
                         : (double)(long long)D.acc[t] * SKIN_FIX_INV;
    D.acc[t] = 0ull;
    if (q < ndof[e]) out[tau_off[e] + q] = v;
    if (q >= SKIN_TAU_MAX) out[nt + SKIN_NSTAT * e + (q - SKIN_TAU_MAX)] = v;
  }
}

/// Parity: one thread per env, its markers in order (empirical.hpp:81-90).
__global__ void k_drag_serial(DragDev D, const int* tau_off, const int* ndof, int nt, double* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= D.E) return;
  const SkinBody& B = D.bodies[e];
  double acc[SKIN_ACC_N];
  for (int q = 0; q < SKIN_ACC_N; ++q) acc[q] = 0.0;
  for (int i = D.m0[e]; i < D.m0[e + 1]; ++i) {
    double f[3], vel[3];
    if (drag_force(D, B, i, f, vel)) drag_contrib(D, B, i, f, vel, acc);
  }
  for (int q = 0; q < ndof[e]; ++q) out[tau_off[e] + q] = acc[q];
  for (int q = 0; q < SKIN_NSTAT; ++q) out[nt + SKIN_NSTAT * e + q] = acc[SKIN_TAU_MAX + q];
}

thread_local char g_drag_err[512] = "";
int drag_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_drag_err, sizeof(g_drag_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace
}  // namespace fsg

struct fsg_drag {
  int E = 0, device = 0, precision = 0;
  double k = 40.0;
  cudaStream_t stream = nullptr;
  // host copies of every env's skin (re-uploaded when one changes)
  std::vector<fsg_skeleton> sk;
  std::vector<std::vector<double>> rest, nrest, area;
  std::vector<std::vector<int>> wb;
  std::vector<std::vector<double>> ww;
  std::vector<int> ndof;
  bool dirty = true;
  fsg::SkinBody* h_bodies = nullptr;  // pinned, per env: topology + pose
  std::vector<char> posed;
  // device
  double* d_dbl = nullptr;   // rest | nrest | ww | area
  int* d_int = nullptr;      // wb | env | m0 | tau_off | ndof
  fsg::SkinBody* d_bodies = nullptr;
  unsigned long long* d_acc = nullptr;
  double* h_out = nullptr;   // pinned: tau (all envs) + 7 stats per env
  int m = 0, nt = 0;
  const int* d_tau_off = nullptr;
  const int* d_ndof = nullptr;
  fsg::DragDev D{};
};

namespace {
#define DCU(call)                                                                           \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fsg::drag_err(FSG_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));     \
  } while (0)

int drag_upload(fsg_drag* d) {
  const int E = d->E;
  int m = 0, nt = 0;
  std::vector<int> m0(E + 1), tau_off(E);
  for (int e = 0; e < E; ++e) {
    m0[e] = m;
    tau_off[e] = nt;
    m += (int)d->area[e].size();
    nt += d->ndof[e];
  }
  m0[E] = m;
  const size_t M = (size_t)std::max(m, 1), KW = fsg::SKIN_KW;
  cudaFree(d->d_dbl);
  cudaFree(d->d_int);
  d->d_dbl = nullptr;
  d->d_int = nullptr;
  DCU(cudaMalloc(&d->d_dbl, sizeof(double) * (7 + KW) * M));
  DCU(cudaMalloc(&d->d_int, sizeof(int) * ((KW + 1) * M + 3 * (size_t)E + 1)));
  std::vector<double> dbl((7 + KW) * M, 0.0);
  std::vector<int> in((KW + 1) * M + 3 * (size_t)E + 1, -1);
  for (int e = 0; e < E; ++e)
    for (int i = m0[e]; i < m0[e + 1]; ++i) {
      const int li = i - m0[e];
      for (int c = 0; c < 3; ++c) {
        dbl[3 * i + c] = d->rest[e][3 * li + c];
        dbl[3 * M + 3 * i + c] = d->nrest[e][3 * li + c];
      }
      for (size_t q = 0; q < KW; ++q) {
        dbl[6 * M + KW * i + q] = d->ww[e][KW * li + q];
        in[KW * i + q] = d->wb[e][KW * li + q];
      }
      dbl[(6 + KW) * M + i] = d->area[e][li];
      in[KW * M + i] = e;
    }
  int* tail = in.data() + (KW + 1) * M;
  for (int e = 0; e <= E; ++e) tail[e] = m0[e];
  for (int e = 0; e < E; ++e) {
    tail[E + 1 + e] = tau_off[e];
    tail[2 * E + 1 + e] = d->ndof[e];
  }
  DCU(cudaMemcpy(d->d_dbl, dbl.data(), sizeof(double) * dbl.size(), cudaMemcpyHostToDevice));
  DCU(cudaMemcpy(d->d_int, in.data(), sizeof(int) * in.size(), cudaMemcpyHostToDevice));
  fsg::DragDev& D = d->D;
  D.E = E;
  D.m = m;
  D.rest = d->d_dbl;
  D.nrest = d->d_dbl + 3 * M;
  D.ww = d->d_dbl + 6 * M;
  D.area = d->d_dbl + (6 + KW) * M;
  D.wb = d->d_int;
  D.env = d->d_int + KW * M;
  D.m0 = d->d_int + (KW + 1) * M;
  d->d_tau_off = D.m0 + E + 1;
  d->d_ndof = D.m0 + 2 * E + 1;
  D.bodies = d->d_bodies;
  D.k = d->k;
  D.acc = d->d_acc;
  d->m = m;
  d->nt = nt;
  d->dirty = false;
  return FSG_OK;
}
}  // namespace

extern "C" {

const char* fsg_drag_last_error(void) { return fsg::g_drag_err; }

int fsg_drag_create(int n_envs, double k, int precision, int device, fsg_drag** out) {
  if (!out) return fsg::drag_err(FSG_EINPUT, "null output handle");
  *out = nullptr;
  if (n_envs < 1 || n_envs > 4096) return fsg::drag_err(FSG_EINPUT, "n_envs must be 1..4096");
  if (!(k > 0.0)) return fsg::drag_err(FSG_EINPUT, "empirical drag constant k must be positive");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fsg::drag_err(FSG_ECUDA, "fsg: no CUDA device available (the B200 path has no CPU fallback)");
  DCU(cudaSetDevice(device));
  fsg_drag* d = new fsg_drag();
  d->E = n_envs;
  d->k = k;
  d->precision = precision;
  d->device = device;
  d->sk.resize(n_envs);
  d->rest.resize(n_envs);
  d->nrest.resize(n_envs);
  d->area.resize(n_envs);
  d->wb.resize(n_envs);
  d->ww.resize(n_envs);
  d->ndof.assign(n_envs, 0);
  d->posed.assign(n_envs, 0);
  if (cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&d->h_bodies, sizeof(fsg::SkinBody) * n_envs) != cudaSuccess ||
      cudaMalloc(&d->d_bodies, sizeof(fsg::SkinBody) * n_envs) != cudaSuccess ||
      cudaMalloc(&d->d_acc, sizeof(unsigned long long) * fsg::DRAG_ACC * n_envs) != cudaSuccess ||
      cudaMemset(d->d_acc, 0, sizeof(unsigned long long) * fsg::DRAG_ACC * n_envs) != cudaSuccess ||
      cudaMallocHost(&d->h_out, sizeof(double) * (6 + FSG_SKIN_MAX_LINKS + 7) * n_envs) != cudaSuccess) {
    fsg_drag_destroy(d);
    return fsg::drag_err(FSG_ECUDA, "fsg_drag_create: allocation failed");
  }
  std::memset(d->h_bodies, 0, sizeof(fsg::SkinBody) * n_envs);
  *out = d;
  return FSG_OK;
}

int fsg_drag_destroy(fsg_drag* d) {
  if (!d) return FSG_OK;
  cudaSetDevice(d->device);
  if (d->stream) cudaStreamSynchronize(d->stream);
  if (d->h_bodies) cudaFreeHost(d->h_bodies);
  if (d->h_out) cudaFreeHost(d->h_out);
  cudaFree(d->d_bodies);
  cudaFree(d->d_acc);
  cudaFree(d->d_dbl);
  cudaFree(d->d_int);
  if (d->stream) cudaStreamDestroy(d->stream);
  delete d;
  return FSG_OK;
}

int fsg_drag_set_skin(fsg_drag* d, int env, const fsg_skeleton* k, int m, const double* rest,
                      const double* nrest, const double* weights, const double* areas) {
  if (env < 0 || env >= d->E) return fsg::drag_err(FSG_EINPUT, "env %d out of range", env);
  if (!k || m < 0 || (m > 0 && (!rest || !nrest || !weights || !areas)))
    return fsg::drag_err(FSG_EINPUT, "fsg_drag_set_skin: null array");
  if (k->n_links < 1 || k->n_links > FSG_SKIN_MAX_LINKS || k->n_dofs < 0 ||
      k->n_dofs > 6 + FSG_SKIN_MAX_LINKS || (k->floating_base && k->n_dofs < 6))
    return fsg::drag_err(FSG_EINPUT, "env %d: bad skeleton", env);
  for (int j = 1; j < k->n_links; ++j)
    if (k->parent[j] < 0 || k->parent[j] >= j || k->dof_index[j] >= k->n_dofs)
      return fsg::drag_err(FSG_EINPUT, "env %d: bad skeleton topology", env);
  const int L = k->n_links, KW = fsg::SKIN_KW;
  std::vector<int> wb((size_t)KW * m, -1);
  std::vector<double> ww((size_t)KW * m, 0.0);
  for (int i = 0; i < m; ++i) {
    int nz = 0;
    for (int j = 0; j < L; ++j) {
      const double w = weights[(size_t)i * L + j];
      if (w == 0.0) continue;
      if (nz == KW) return fsg::drag_err(FSG_EINPUT, "marker %d has more than %d nonzero skin weights", i, KW);
      wb[(size_t)KW * i + nz] = j;
      ww[(size_t)KW * i + nz] = w;
      ++nz;
    }
  }
  d->sk[env] = *k;
  d->rest[env].assign(rest, rest + 3 * (size_t)m);
  d->nrest[env].assign(nrest, nrest + 3 * (size_t)m);
  d->area[env].assign(areas, areas + m);
  d->wb[env] = wb;
  d->ww[env] = ww;
  d->ndof[env] = k->n_dofs;
  fsg::SkinBody& B = d->h_bodies[env];
  B.m0 = B.m1 = 0;
  B.n_links = L;
  B.floating = k->floating_base ? 1 : 0;
  B.n_dofs = k->n_dofs;
  B.tau_off = 0;
  B.max_level = 0;  // the drag kernels walk the parent chain
  for (int j = 0; j < FSG_SKIN_MAX_LINKS; ++j) {
    B.parent[j] = j < L ? k->parent[j] : -1;
    B.dof[j] = (j > 0 && j < L) ? k->dof_index[j] : -1;
    for (int c = 0; c < 3; ++c) B.axis[j][c] = j < L ? k->axis[j][c] : 0.0;
  }
  d->dirty = true;
  return FSG_OK;
}

int fsg_drag_set_pose(fsg_drag* d, int env, const fsg_body_pose* pose) {
  if (env < 0 || env >= d->E || !pose) return fsg::drag_err(FSG_EINPUT, "fsg_drag_set_pose: bad env or pose");
  DCU(cudaStreamSynchronize(d->stream));  // the previous step may still read the pinned poses
  d->h_bodies[env].pose = *pose;
  d->posed[env] = 1;
  return FSG_OK;
}

int fsg_drag_set_poses(fsg_drag* d, const fsg_body_pose* poses) {
  if (!poses) return fsg::drag_err(FSG_EINPUT, "fsg_drag_set_poses: null poses");
  DCU(cudaStreamSynchronize(d->stream));
  for (int e = 0; e < d->E; ++e) {
    d->h_bodies[e].pose = poses[e];
    d->posed[e] = 1;
  }
  return FSG_OK;
}

int fsg_drag_step(fsg_drag* d, double* tau_ext, double* stats) {
  DCU(cudaSetDevice(d->device));
  for (int e = 0; e < d->E; ++e)
    if (!d->posed[e]) return fsg::drag_err(FSG_ESTATE, "env %d: fsg_drag_set_pose has not been called", e);
  if (d->dirty) {
    int rc = drag_upload(d);
    if (rc) return rc;
  }
  DCU(cudaMemcpyAsync(d->d_bodies, d->h_bodies, sizeof(fsg::SkinBody) * d->E, cudaMemcpyHostToDevice,
                      d->stream));
  if (d->precision == FSG_PRECISION_FP64) {
    fsg::k_drag_serial<<<(d->E + 31) / 32, 32, 0, d->stream>>>(d->D, d->d_tau_off, d->d_ndof, d->nt, d->h_out);
  } else {
    if (d->m > 0) fsg::k_drag<<<(d->m + 127) / 128, 128, 0, d->stream>>>(d->D);
    fsg::k_drag_finish<<<(d->E * fsg::DRAG_ACC + 255) / 256, 256, 0, d->stream>>>(
        d->D, d->d_tau_off, d->d_ndof, d->nt, d->h_out);
    // every env's non-finite flag word back to zero after the conversion read it
    DCU(cudaMemset2DAsync(d->d_acc + fsg::SKIN_ACC_N, sizeof(unsigned long long) * fsg::DRAG_ACC, 0,
                          sizeof(unsigned long long), d->E, d->stream));
  }
  DCU(cudaGetLastError());
  DCU(cudaStreamSynchronize(d->stream));
  if (tau_ext) std::memcpy(tau_ext, d->h_out, sizeof(double) * d->nt);
  if (stats) std::memcpy(stats, d->h_out + d->nt, sizeof(double) * fsg::SKIN_NSTAT * d->E);
  return FSG_OK;
}

}  // extern "C"
