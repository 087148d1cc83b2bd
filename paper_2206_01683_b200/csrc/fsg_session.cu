// fsg_session.cu -- host orchestration behind the C ABI (include/fsg.h).
//
// One fsg_session owns one device's distribution pair (A/B), the IB band and
// marker buffers, and one CUDA stream; it is the B200 counterpart of
// sim::CoupledSession (session.hpp:29-224) plus the lbm/ib/frame free
// functions the reference's tests drive directly.  All fp64 host arithmetic
// (UnitMap, frame constants, recenter origin update) keeps the reference's
// operation order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fsg.h"
#include "fsg_device.cuh"

using fsg::Band;
using fsg::Grid;
using fsg::Launchers;
using fsg::MarkerStencil;
using fsg::Markers;
using fsg::SessionConsts;
using fsg::StepConsts;
using fsg::StepScratch;

namespace {

thread_local char g_err[1024] = "";

int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return set_err(FSG_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));  \
  } while (0)

#define CU_LAUNCH()                                                                   \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) return set_err(FSG_ECUDA, "kernel launch: %s", cudaGetErrorString(e_)); \
  } while (0)

// Eigen Quaternion::toRotationMatrix (frame.hpp:21), row-major.
void quat_to_R(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0] = 1.0 - (tyy + tzz);
  R[1] = txy - twz;
  R[2] = txz + twy;
  R[3] = txy + twz;
  R[4] = 1.0 - (txx + tzz);
  R[5] = tyz - twx;
  R[6] = txz - twy;
  R[7] = tyz + twx;
  R[8] = 1.0 - (txx + tyy);
}
void mat_t_vec(const double* R, const double* v, double* r) {
  for (int i = 0; i < 3; ++i) r[i] = R[i] * v[0] + R[3 + i] * v[1] + R[6 + i] * v[2];
}
void mat_vec(const double* R, const double* v, double* r) {
  for (int i = 0; i < 3; ++i) r[i] = R[3 * i] * v[0] + R[3 * i + 1] * v[1] + R[3 * i + 2] * v[2];
}

}  // namespace

struct fsg_session {
  fsg_config cfg{};
  const Launchers* L = nullptr;
  Grid g{};
  cudaStream_t stream = nullptr;
  void* A = nullptr;
  void* B = nullptr;
  int pulled = 0;  // A holds post-collision P (1) or post-stream S (0)
  // last session step, for macro()/force readbacks (the buffer it read)
  bool last_valid = false;
  void* prevA = nullptr;
  int prev_pulled = 0;
  bool last_frame_on = false;
  void* Fext = nullptr;  // SoA 3*n in the storage's math type
  SessionConsts hsc{};
  SessionConsts* d_sc = nullptr;
  StepConsts* d_st = nullptr;
  StepConsts* h_st = nullptr;  // pinned
  StepScratch* d_scr = nullptr;
  StepScratch* h_scr = nullptr;  // pinned
  fsg_frame_state frame{};
  // markers
  int cap = 0;
  int m = 0;
  int n_bodies = 0;
  std::vector<int64_t> offsets;
  double* d_mk = nullptr;   // owned [pts 3cap | vel 3cap | nrm 3cap | area cap]
  double* h_mk = nullptr;   // pinned staging
  Markers mk{};
  bool mk_host_vel = false;
  std::vector<double> h_vel;  // for CouplingStats power
  MarkerStencil* d_stencil = nullptr;
  double* d_fworld = nullptr;
  Band band{};
  double* d_tmp = nullptr;  // readback staging, 19*n doubles (lazy)
  size_t tmp_bytes = 0;
  double* d_red = nullptr;  // reduction scratch
  StepScratch* d_junk = nullptr;
  cudaEvent_t ev_st = nullptr;  // h_st consumed
  cudaEvent_t ev_mk = nullptr;  // h_mk consumed
  fsg_status last{};
};

namespace {

int ensure_tmp(fsg_session* s, size_t bytes) {
  if (s->tmp_bytes >= bytes) return FSG_OK;
  if (s->d_tmp) cudaFree(s->d_tmp);
  s->d_tmp = nullptr;
  s->tmp_bytes = 0;
  CU(cudaMalloc(&s->d_tmp, bytes));
  s->tmp_bytes = bytes;
  return FSG_OK;
}

void frame_consts(const fsg_frame_state& f, StepConsts& st) {
  quat_to_R(f.q, st.R);
  for (int k = 0; k < 3; ++k) {
    st.p[k] = f.p[k];
    st.pd[k] = f.pd[k];
  }
  mat_t_vec(st.R, f.pdd, st.a0);
  mat_t_vec(st.R, f.omega, st.wf);
  mat_t_vec(st.R, f.alpha, st.af);
}

void decode_status(const StepScratch& sc, fsg_status* st, bool session) {
  st->finite = sc.nonfinite ? 0 : 1;
  st->min_f = sc.neg_min_key ? fsg::key_to_double(~sc.neg_min_key) : DBL_MAX;
  st->n_nonpositive_rho = session ? sc.nonpos : 0;
  st->out_of_bounds_markers = session ? sc.oob : 0;
  st->stable = (st->finite && st->min_f > -1e-3 && st->n_nonpositive_rho == 0) ? 1 : 0;
}

__global__ void k_plane_sums(const double* f, long long n, double* partial, int nblk) {
  // deterministic: fixed chunking and a fixed in-block tree
  __shared__ double sm[256];
  const int i = blockIdx.y;
  const long long chunk = (n + nblk - 1) / nblk;
  const long long c0 = blockIdx.x * chunk, c1 = min(n, c0 + chunk);
  double s = 0.0;
  for (long long c = c0 + threadIdx.x; c < c1; c += blockDim.x) s += f[i * n + c];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[i * nblk + blockIdx.x] = sm[0];
}

int plane_sums(fsg_session* s, double out[19]) {
  const long long n = s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 19 * (size_t)n);
  if (rc) return rc;
  s->L->get_f(s->g, s->A, s->pulled, s->d_tmp, s->stream);
  CU_LAUNCH();
  const int nblk = 256;
  if (!s->d_red) CU(cudaMalloc(&s->d_red, sizeof(double) * 19 * nblk));
  k_plane_sums<<<dim3(nblk, 19), 256, 0, s->stream>>>(s->d_tmp, n, s->d_red, nblk);
  CU_LAUNCH();
  std::vector<double> part(19 * nblk);
  CU(cudaMemcpyAsync(part.data(), s->d_red, sizeof(double) * part.size(), cudaMemcpyDeviceToHost,
                     s->stream));
  CU(cudaStreamSynchronize(s->stream));
  for (int i = 0; i < 19; ++i) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[i * nblk + b];
    out[i] = acc;
  }
  return FSG_OK;
}

int upload_step_consts(fsg_session* s) {
  CU(cudaEventSynchronize(s->ev_st));  // previous copy out of the pinned buffer done
  frame_consts(s->frame, *s->h_st);
  CU(cudaMemcpyAsync(s->d_st, s->h_st, sizeof(StepConsts), cudaMemcpyHostToDevice, s->stream));
  CU(cudaEventRecord(s->ev_st, s->stream));
  return FSG_OK;
}

}  // namespace

extern "C" {

const char* fsg_last_error(void) { return g_err; }
int fsg_abi_version(void) { return FSG_ABI_VERSION; }

void fsg_config_default(fsg_config* c) {
  std::memset(c, 0, sizeof *c);
  c->dims[0] = c->dims[1] = c->dims[2] = 64;  // session.hpp:13
  c->dx = 0.01;
  c->dt = 0.004;
  c->rho = 1000.0;
  c->nu = 0.00089;
  c->boundary = FSG_BOUNDARY_OPEN;  // session.hpp:37
  c->kernel = FSG_KERNEL_PESKIN4;
  c->wall = FSG_WALL_SLIP;
  c->frame_mode = FSG_FRAME_TRANSLATION_YAW;  // session.hpp:17
  c->precision = FSG_PRECISION_FP32;
  c->device = 0;
  c->max_markers = 0;
  c->z_offset = 0;
  c->nz_global = 0;
}

double fsg_tau(double dx, double dt, double nu) { return 3.0 * (nu * dt / (dx * dx)) + 0.5; }

int fsg_create(const fsg_config* cfg_in, fsg_session** out) {
  if (!cfg_in || !out) return set_err(FSG_EINPUT, "fsg_create: null argument");
  *out = nullptr;
  fsg_config cfg = *cfg_in;
  if (cfg.nz_global <= 0) cfg.nz_global = cfg.dims[2];
  // units.hpp:56-68
  if (!(cfg.dx > 0.0) || !(cfg.dt > 0.0) || !(cfg.rho > 0.0) || !(cfg.nu > 0.0))
    return set_err(FSG_EINPUT, "unit map requires positive dx, dt, rho, nu");
  const double tau = fsg_tau(cfg.dx, cfg.dt, cfg.nu);
  if (!(tau > 0.5) || !(tau <= 1.5))
    return set_err(FSG_EINPUT,
                   "fluid parameters give tau = %g from (nu = %g, dx = %g, dt = %g); stable range "
                   "is (0.5, 1.5]",
                   tau, cfg.nu, cfg.dx, cfg.dt);
  // lattice.hpp:66-67 (slabs: >= 2 owned planes, global z >= 8)
  if (cfg.dims[0] < 8 || cfg.dims[1] < 8 || cfg.nz_global < 8)
    return set_err(FSG_EINPUT, "lattice dims must each be >= 8");
  const bool slab = cfg.nz_global != cfg.dims[2] || cfg.z_offset != 0;
  if (cfg.dims[2] < (slab ? 2 : 8) || cfg.z_offset < 0 || cfg.z_offset + cfg.dims[2] > cfg.nz_global)
    return set_err(FSG_EINPUT, "bad z slab: offset %d depth %d of %d", cfg.z_offset, cfg.dims[2],
                   cfg.nz_global);
  if (cfg.boundary != FSG_BOUNDARY_OPEN && cfg.boundary != FSG_BOUNDARY_PERIODIC)
    return set_err(FSG_EINPUT, "unknown boundary mode %d", cfg.boundary);
  if (cfg.kernel != FSG_KERNEL_PESKIN4 && cfg.kernel != FSG_KERNEL_ROMA3)
    return set_err(FSG_EINPUT, "unknown IB kernel %d (use peskin4 or roma3)", cfg.kernel);
  if (cfg.wall != FSG_WALL_SLIP && cfg.wall != FSG_WALL_NOSLIP)
    return set_err(FSG_EINPUT, "unknown wall condition %d", cfg.wall);
  if (cfg.frame_mode < FSG_FRAME_NONE || cfg.frame_mode > FSG_FRAME_FULL)
    return set_err(FSG_EINPUT, "unknown frame mode %d", cfg.frame_mode);
  if (cfg.precision != FSG_PRECISION_FP32 && cfg.precision != FSG_PRECISION_FP64)
    return set_err(FSG_EINPUT, "unknown precision %d", cfg.precision);
  if (cfg.max_markers <= 0) cfg.max_markers = 65536;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(FSG_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  if (cfg.device < 0 || cfg.device >= ndev)
    return set_err(FSG_EINPUT, "device %d out of range (%d devices)", cfg.device, ndev);
  CU(cudaSetDevice(cfg.device));

  auto* s = new fsg_session();
  s->cfg = cfg;
  s->L = cfg.precision == FSG_PRECISION_FP64 ? &fsg::launchers_fp64() : &fsg::launchers_fp32();
  Grid& g = s->g;
  g.nx = cfg.dims[0];
  g.ny = cfg.dims[1];
  g.nz = cfg.dims[2];
  g.nzg = cfg.nz_global;
  g.z0 = cfg.z_offset;
  g.zpad = slab ? 1 : 0;
  g.periodic = cfg.boundary == FSG_BOUNDARY_PERIODIC ? 1 : 0;
  g.plane = (long long)g.nx * g.ny;
  g.n = g.plane * g.nz;
  g.stride = ((g.plane * (g.nz + 2 * g.zpad) + 31) / 32) * 32;

  // session constants, host fp64 in the reference's order
  SessionConsts& sc = s->hsc;
  sc.omega = 1.0 / tau;                // solver.hpp:109
  sc.guo = 1.0 - 0.5 * sc.omega;       // solver.hpp:110
  sc.dx = cfg.dx;
  sc.dt = cfg.dt;
  sc.rho_phys = cfg.rho;
  sc.v2p = cfg.dx / cfg.dt;            // units.hpp:31
  sc.acc = cfg.dt * cfg.dt / cfg.dx;   // session.hpp:149
  sc.f2l = cfg.dt * cfg.dt / (cfg.rho * cfg.dx * cfg.dx * cfg.dx * cfg.dx);  // session.hpp:128
  const int dg[3] = {cfg.dims[0], cfg.dims[1], cfg.nz_global};
  for (int a = 0; a < 3; ++a) {
    sc.hd[a] = 0.5 * (dg[a] - 1);
    sc.dims_g[a] = dg[a];
  }
  sc.kernel = cfg.kernel;
  sc.wall = cfg.wall;
  sc.frame_on = cfg.frame_mode != FSG_FRAME_NONE;
  s->frame.q[0] = 1.0;

  int rc = FSG_OK;
  auto fail = [&](int code) {
    fsg_destroy(s);
    return code;
  };
#define CUF(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(set_err(FSG_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_))); \
  } while (0)
  CUF(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  const size_t fbytes = (size_t)s->L->elem_bytes * 19 * (size_t)g.stride;
  CUF(cudaMalloc(&s->A, fbytes));
  CUF(cudaMalloc(&s->B, fbytes));
  CUF(cudaMemsetAsync(s->A, 0, fbytes, s->stream));
  CUF(cudaMemsetAsync(s->B, 0, fbytes, s->stream));
  CUF(cudaMalloc(&s->d_sc, sizeof(SessionConsts)));
  CUF(cudaMalloc(&s->d_st, sizeof(StepConsts)));
  CUF(cudaMalloc(&s->d_scr, sizeof(StepScratch)));
  CUF(cudaMallocHost(&s->h_st, sizeof(StepConsts)));
  CUF(cudaMallocHost(&s->h_scr, sizeof(StepScratch)));
  CUF(cudaMemcpyAsync(s->d_sc, &s->hsc, sizeof(SessionConsts), cudaMemcpyHostToDevice, s->stream));
  CUF(cudaMemsetAsync(s->d_scr, 0, sizeof(StepScratch), s->stream));
  s->cap = cfg.max_markers;
  CUF(cudaMalloc(&s->d_mk, sizeof(double) * 10 * (size_t)s->cap));
  CUF(cudaMallocHost(&s->h_mk, sizeof(double) * 10 * (size_t)s->cap));
  CUF(cudaMalloc(&s->d_stencil, sizeof(MarkerStencil) * (size_t)s->cap));
  CUF(cudaMalloc(&s->d_fworld, sizeof(double) * 3 * (size_t)s->cap));
  s->band.cap = std::min<long long>(g.n, 16ll << 20);
  CUF(cudaMalloc(&s->band.u, sizeof(double) * 3 * (size_t)s->band.cap));
  CUF(cudaMalloc(&s->band.F, sizeof(double) * 3 * (size_t)s->band.cap));
  CUF(cudaMalloc(&s->d_junk, sizeof(StepScratch)));
  CUF(cudaEventCreateWithFlags(&s->ev_st, cudaEventDisableTiming));
  CUF(cudaEventCreateWithFlags(&s->ev_mk, cudaEventDisableTiming));
  CUF(cudaEventRecord(s->ev_st, s->stream));
  CUF(cudaEventRecord(s->ev_mk, s->stream));
#undef CUF
  s->L->fill_rest(g, s->A, s->stream);
  if (cudaGetLastError() != cudaSuccess) return fail(set_err(FSG_ECUDA, "fill_rest launch failed"));
  if (cudaStreamSynchronize(s->stream) != cudaSuccess)
    return fail(set_err(FSG_ECUDA, "session init failed"));
  s->pulled = 0;
  (void)rc;
  *out = s;
  return FSG_OK;
}

int fsg_destroy(fsg_session* s) {
  if (!s) return FSG_OK;
  cudaSetDevice(s->cfg.device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  cudaFree(s->A);
  cudaFree(s->B);
  cudaFree(s->Fext);
  cudaFree(s->d_sc);
  cudaFree(s->d_st);
  cudaFree(s->d_scr);
  if (s->h_st) cudaFreeHost(s->h_st);
  if (s->h_scr) cudaFreeHost(s->h_scr);
  cudaFree(s->d_mk);
  if (s->h_mk) cudaFreeHost(s->h_mk);
  cudaFree(s->d_stencil);
  cudaFree(s->d_fworld);
  cudaFree(s->band.u);
  cudaFree(s->band.F);
  cudaFree(s->d_tmp);
  cudaFree(s->d_red);
  cudaFree(s->d_junk);
  if (s->ev_st) cudaEventDestroy(s->ev_st);
  if (s->ev_mk) cudaEventDestroy(s->ev_mk);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return FSG_OK;
}

void* fsg_stream(fsg_session* s) { return s ? (void*)s->stream : nullptr; }

// --------------------------------------------------------------- state --
int fsg_reset_rest(fsg_session* s) {
  CU(cudaSetDevice(s->cfg.device));
  s->L->fill_rest(s->g, s->A, s->stream);
  CU_LAUNCH();
  s->pulled = 0;
  s->last_valid = false;
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_initialize(fsg_session* s, const double* rho, const double* u) {
  if (!rho || !u) return set_err(FSG_EINPUT, "fsg_initialize: null field");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 4 * n);
  if (rc) return rc;
  CU(cudaMemcpyAsync(s->d_tmp, rho, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
  CU(cudaMemcpyAsync(s->d_tmp + n, u, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, s->stream));
  s->L->init_eq(s->g, s->d_tmp, s->d_tmp + n, s->A, s->stream);
  CU_LAUNCH();
  s->pulled = 0;
  s->last_valid = false;
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_set_f(fsg_session* s, const double* f) {
  if (!f) return set_err(FSG_EINPUT, "fsg_set_f: null");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 19 * n);
  if (rc) return rc;
  CU(cudaMemcpyAsync(s->d_tmp, f, sizeof(double) * 19 * n, cudaMemcpyHostToDevice, s->stream));
  s->L->set_f(s->g, s->d_tmp, s->A, s->stream);
  CU_LAUNCH();
  s->pulled = 0;
  s->last_valid = false;
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_get_f(fsg_session* s, double* f) {
  if (!f) return set_err(FSG_EINPUT, "fsg_get_f: null");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 19 * n);
  if (rc) return rc;
  s->L->get_f(s->g, s->A, s->pulled, s->d_tmp, s->stream);
  CU_LAUNCH();
  CU(cudaMemcpyAsync(f, s->d_tmp, sizeof(double) * 19 * n, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_set_force(fsg_session* s, const double* F) {
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  if (!F) {
    cudaFree(s->Fext);
    s->Fext = nullptr;
    return FSG_OK;
  }
  const size_t eb = (size_t)s->L->elem_bytes;
  if (!s->Fext) CU(cudaMalloc(&s->Fext, eb * 3 * n));
  // AoS double -> SoA in the storage's arithmetic type
  if (eb == 8) {
    std::vector<double> soa(3 * n);
    for (size_t c = 0; c < n; ++c)
      for (int k = 0; k < 3; ++k) soa[k * n + c] = F[3 * c + k];
    CU(cudaMemcpy(s->Fext, soa.data(), eb * 3 * n, cudaMemcpyHostToDevice));
  } else {
    std::vector<float> soa(3 * n);
    for (size_t c = 0; c < n; ++c)
      for (int k = 0; k < 3; ++k) soa[k * n + c] = (float)F[3 * c + k];
    CU(cudaMemcpy(s->Fext, soa.data(), eb * 3 * n, cudaMemcpyHostToDevice));
  }
  return FSG_OK;
}

int fsg_collide_and_stream(fsg_session* s, fsg_status* st) {
  CU(cudaSetDevice(s->cfg.device));
  CU(cudaMemsetAsync(s->d_scr, 0, sizeof(StepScratch), s->stream));
  s->L->collide(s->g, s->A, s->pulled, s->B, s->Fext, nullptr, nullptr, s->d_sc, s->d_st, s->d_scr,
                0, 0, s->stream);
  CU_LAUNCH();
  CU(cudaMemcpyAsync(s->h_scr, s->d_scr, sizeof(StepScratch), cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  std::swap(s->A, s->B);
  s->pulled = 1;
  s->last_valid = false;
  decode_status(*s->h_scr, &s->last, false);
  if (st) *st = s->last;
  return FSG_OK;
}

int fsg_macroscopic(fsg_session* s, double* rho, double* u, int* nonpos) {
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 4 * n);
  if (rc) return rc;
  CU(cudaMemsetAsync(s->d_scr, 0, sizeof(StepScratch), s->stream));
  s->L->macroscopic(s->g, s->A, s->pulled, s->Fext, s->d_tmp, s->d_tmp + n, s->d_scr, s->stream);
  CU_LAUNCH();
  if (rho) CU(cudaMemcpyAsync(rho, s->d_tmp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
  if (u) CU(cudaMemcpyAsync(u, s->d_tmp + n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaMemcpyAsync(s->h_scr, s->d_scr, sizeof(StepScratch), cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  if (nonpos) *nonpos = s->h_scr->nonpos;
  s->last_valid = false;  // scratch reused
  return FSG_OK;
}

int fsg_total_mass(fsg_session* s, double* mass) {
  CU(cudaSetDevice(s->cfg.device));
  double p[19];
  int rc = plane_sums(s, p);
  if (rc) return rc;
  double acc = 0.0;
  for (int i = 0; i < 19; ++i) acc += p[i];
  *mass = acc;
  return FSG_OK;
}

int fsg_total_momentum(fsg_session* s, double* out) {
  CU(cudaSetDevice(s->cfg.device));
  double p[19];
  int rc = plane_sums(s, p);
  if (rc) return rc;
  double m[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < 19; ++i) {  // solver.hpp:189-200
    m[0] = m[0] + p[i] * (double)fsg::ex_of(i);
    m[1] = m[1] + p[i] * (double)fsg::ey_of(i);
    m[2] = m[2] + p[i] * (double)fsg::ez_of(i);
  }
  std::memcpy(out, m, sizeof m);
  return FSG_OK;
}

// --------------------------------------------------------------- frame --
int fsg_set_frame(fsg_session* s, const fsg_frame_state* fs) {
  if (!fs) return set_err(FSG_EINPUT, "fsg_set_frame: null");
  s->frame = *fs;
  return FSG_OK;
}
int fsg_get_frame(fsg_session* s, fsg_frame_state* fs) {
  if (!fs) return set_err(FSG_EINPUT, "fsg_get_frame: null");
  *fs = s->frame;
  return FSG_OK;
}

int fsg_recenter(fsg_session* s, const int shift[3]) {
  if (s->g.zpad) return set_err(FSG_EINPUT, "recenter is not defined for z-slab sessions");
  CU(cudaSetDevice(s->cfg.device));
  s->L->recenter(s->g, s->A, s->pulled, s->B, shift[0], shift[1], shift[2], s->stream);
  CU_LAUNCH();
  CU(cudaStreamSynchronize(s->stream));
  std::swap(s->A, s->B);
  s->pulled = 0;
  s->last_valid = false;
  // frame.hpp:152-153: p += R * (shift * dx)
  double R[9];
  quat_to_R(s->frame.q, R);
  const double off[3] = {shift[0] * s->cfg.dx, shift[1] * s->cfg.dx, shift[2] * s->cfg.dx};
  double r[3];
  mat_vec(R, off, r);
  for (int k = 0; k < 3; ++k) s->frame.p[k] = s->frame.p[k] + r[k];
  return FSG_OK;
}

// -------------------------------------------------------------- markers --
static int set_markers_common(fsg_session* s, int n_bodies, const int64_t* off) {
  if (n_bodies < 0) return set_err(FSG_EINPUT, "negative body count");
  if (n_bodies > 0 && !off) return set_err(FSG_EINPUT, "null body offsets");
  const int64_t m = n_bodies > 0 ? off[n_bodies] : 0;
  if (n_bodies > 0 && off[0] != 0) return set_err(FSG_EINPUT, "body_offsets[0] must be 0");
  for (int b = 0; b < n_bodies; ++b)
    if (off[b + 1] < off[b]) return set_err(FSG_EINPUT, "body offsets must be non-decreasing");
  if (m > s->cap) return set_err(FSG_EINPUT, "%lld markers exceed capacity %d", (long long)m, s->cap);
  s->n_bodies = n_bodies;
  s->offsets.assign(off, off + (n_bodies + 1));
  if (n_bodies == 0) s->offsets.assign(1, 0);
  s->m = (int)m;
  return FSG_OK;
}

int fsg_set_markers(fsg_session* s, int n_bodies, const int64_t* off, const double* pts,
                    const double* vel, const double* nrm, const double* area) {
  int rc = set_markers_common(s, n_bodies, off);
  if (rc) return rc;
  const size_t m = (size_t)s->m;
  CU(cudaSetDevice(s->cfg.device));
  if (m) {
    if (!pts || !vel || !nrm || !area) return set_err(FSG_EINPUT, "fsg_set_markers: null array");
    // one pinned staging buffer [pts | vel | nrm | area] -> one H2D copy
    CU(cudaEventSynchronize(s->ev_mk));
    double* h = s->h_mk;
    std::memcpy(h, pts, sizeof(double) * 3 * m);
    std::memcpy(h + 3 * m, vel, sizeof(double) * 3 * m);
    std::memcpy(h + 6 * m, nrm, sizeof(double) * 3 * m);
    std::memcpy(h + 9 * m, area, sizeof(double) * m);
    CU(cudaMemcpyAsync(s->d_mk, h, sizeof(double) * 10 * m, cudaMemcpyHostToDevice, s->stream));
    CU(cudaEventRecord(s->ev_mk, s->stream));
    s->h_vel.assign(vel, vel + 3 * m);
  }
  s->mk = Markers{s->d_mk, s->d_mk + 3 * m, s->d_mk + 6 * m, s->d_mk + 9 * m, (int)m};
  s->mk_host_vel = true;
  return FSG_OK;
}

int fsg_set_markers_device(fsg_session* s, int n_bodies, const int64_t* off, const double* pts,
                           const double* vel, const double* nrm, const double* area) {
  int rc = set_markers_common(s, n_bodies, off);
  if (rc) return rc;
  s->mk = Markers{pts, vel, nrm, area, s->m};
  s->mk_host_vel = false;
  return FSG_OK;
}

// ----------------------------------------------------------------- step --
int fsg_step_async(fsg_session* s) {
  CU(cudaSetDevice(s->cfg.device));
  const Grid& g = s->g;
  int rc = upload_step_consts(s);
  if (rc) return rc;
  CU(cudaMemsetAsync(s->d_scr, 0, sizeof(StepScratch), s->stream));
  const bool frame_on = s->cfg.frame_mode != FSG_FRAME_NONE;
  if (s->m > 0) {
    s->L->markers_prepare(g, s->mk, s->d_sc, s->d_st, s->d_stencil, s->d_scr, s->stream);
    s->L->band_moments(g, s->A, s->pulled, s->band, s->d_scr, s->d_scr, s->stream);
    s->L->markers_force(g, s->mk, s->d_sc, s->d_st, s->d_stencil, s->band, s->d_scr, s->d_fworld,
                        s->stream);
    s->L->spread(g, s->m, s->d_stencil, s->band, s->d_scr, s->stream);
  }
  s->L->collide(g, s->A, s->pulled, s->B, nullptr, &s->band, s->d_scr, s->d_sc, s->d_st, s->d_scr,
                1, frame_on ? 1 : 0, s->stream);
  CU_LAUNCH();
  CU(cudaMemcpyAsync(s->h_scr, s->d_scr, sizeof(StepScratch), cudaMemcpyDeviceToHost, s->stream));
  s->prevA = s->A;
  s->prev_pulled = s->pulled;
  s->last_frame_on = frame_on;
  std::swap(s->A, s->B);
  s->pulled = 1;
  s->last_valid = true;
  return FSG_OK;
}

int fsg_last_status(fsg_session* s, fsg_status* st) {
  CU(cudaStreamSynchronize(s->stream));
  if (s->h_scr->band_overflow)
    return set_err(FSG_ESTATE, "IB band bounding box exceeds capacity (%lld cells)",
                   (long long)s->band.cap);
  decode_status(*s->h_scr, &s->last, true);
  if (st) *st = s->last;
  return FSG_OK;
}

int fsg_step(fsg_session* s, fsg_status* st) {
  int rc = fsg_step_async(s);
  if (rc) return rc;
  return fsg_last_status(s, st);
}

int fsg_get_marker_forces(fsg_session* s, double* fw, int* valid, double* stats) {
  CU(cudaSetDevice(s->cfg.device));
  const size_t m = (size_t)s->m;
  std::vector<double> f(3 * m);
  std::vector<MarkerStencil> st(m);
  if (m) {
    CU(cudaMemcpyAsync(f.data(), s->d_fworld, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaMemcpyAsync(st.data(), s->d_stencil, sizeof(MarkerStencil) * m, cudaMemcpyDeviceToHost,
                       s->stream));
  }
  CU(cudaStreamSynchronize(s->stream));
  if (fw) std::memcpy(fw, f.data(), sizeof(double) * 3 * m);
  if (valid)
    for (size_t i = 0; i < m; ++i) valid[i] = st[i].valid;
  if (stats) {
    std::vector<double> vel;
    const double* v = nullptr;
    if (s->mk_host_vel) {
      v = s->h_vel.data();
    } else if (m) {
      vel.resize(3 * m);
      CU(cudaMemcpy(vel.data(), s->mk.vel, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost));
      v = vel.data();
    }
    // CouplingStats, serial in marker order (session.hpp:141-143)
    for (int b = 0; b < s->n_bodies; ++b) {
      double tf[3] = {0, 0, 0}, tb[3] = {0, 0, 0}, power = 0.0;
      for (int64_t i = s->offsets[b]; i < s->offsets[b + 1]; ++i) {
        if (!st[i].valid) continue;
        const double* w = &f[3 * i];
        for (int k = 0; k < 3; ++k) {
          tf[k] = tf[k] + w[k];
          tb[k] = tb[k] - w[k];
        }
        power += (-w[0]) * v[3 * i] + (-w[1]) * v[3 * i + 1] + (-w[2]) * v[3 * i + 2];
      }
      for (int k = 0; k < 3; ++k) {
        stats[7 * b + k] = tf[k];
        stats[7 * b + 3 + k] = tb[k];
      }
      stats[7 * b + 6] = power;
    }
  }
  return FSG_OK;
}

int fsg_get_stencils(fsg_session* s, int* lo_hi) {
  CU(cudaSetDevice(s->cfg.device));
  const size_t m = (size_t)s->m;
  std::vector<MarkerStencil> st(m);
  if (m)
    CU(cudaMemcpyAsync(st.data(), s->d_stencil, sizeof(MarkerStencil) * m, cudaMemcpyDeviceToHost,
                       s->stream));
  CU(cudaStreamSynchronize(s->stream));
  for (size_t i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) {
      lo_hi[6 * i + a] = st[i].valid ? st[i].lo[a] : 0;
      lo_hi[6 * i + 3 + a] = st[i].valid ? st[i].hi[a] : -1;
    }
  return FSG_OK;
}

int fsg_get_macro(fsg_session* s, double* rho, double* u) {
  if (!s->last_valid) return set_err(FSG_ESTATE, "no coupled step since the last state change");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 4 * n);
  if (rc) return rc;
  s->L->macroscopic(s->g, s->prevA, s->prev_pulled, nullptr, s->d_tmp, s->d_tmp + n, s->d_junk,
                    s->stream);
  CU_LAUNCH();
  if (rho) CU(cudaMemcpyAsync(rho, s->d_tmp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
  if (u) CU(cudaMemcpyAsync(u, s->d_tmp + n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_get_force(fsg_session* s, double* F) {
  if (!s->last_valid) return set_err(FSG_ESTATE, "no coupled step since the last state change");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 3 * n);
  if (rc) return rc;
  s->L->session_force(s->g, s->prevA, s->prev_pulled, &s->band, s->d_scr, s->d_sc, s->d_st,
                      s->last_frame_on ? 1 : 0, s->d_tmp, s->stream);
  CU_LAUNCH();
  CU(cudaMemcpyAsync(F, s->d_tmp, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

// --------------------------------------------------------------- halos --
size_t fsg_halo_bytes(fsg_session* s) { return (size_t)5 * s->g.plane * s->L->elem_bytes; }

int fsg_halo_pack(fsg_session* s, void* lo, void* hi) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  CU(cudaSetDevice(s->cfg.device));
  s->L->halo_pack(s->g, s->A, lo, hi, s->stream);
  CU_LAUNCH();
  return FSG_OK;
}

int fsg_halo_unpack(fsg_session* s, const void* lo, const void* hi) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  CU(cudaSetDevice(s->cfg.device));
  s->L->halo_unpack(s->g, s->A, lo, hi, s->stream);
  CU_LAUNCH();
  return FSG_OK;
}

}  // extern "C"
