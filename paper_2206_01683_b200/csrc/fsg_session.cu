// fsg_session.cu -- host orchestration behind the C ABI (include/fsg.h).
//
// One fsg_session owns one device's distribution pair (A/B), the IB band and
// marker buffers, and one CUDA stream; it is the B200 counterpart of
// sim::CoupledSession (session.hpp:29-224) plus the lbm/ib/frame free
// functions the reference's tests drive directly.  All fp64 host arithmetic
// (UnitMap, frame constants, recenter origin update) keeps the reference's
// operation order.
//
// Parity mode (fp64): the coupled step is replayed as a CUDA graph:
//   [H2D marker state] -> [H2D frame constants] -> [reset step scratch]
//   -> K_m markers -> K_s spread -> K4 collide/stream -> [D2H status]
// Host staging (pinned), step scratch and the status readback slot are
// double-buffered by the parity of the A/B pair, so step n+1 can be
// enqueued while step n still runs; each graph bakes in its parity's
// buffers.
// Throughput mode (fp32): two direct launches per coupled step, frame
// constants by value -- the marker kernel (fixed-point spread) and the
// banded K4 as its programmatic dependent (fsg_k4.cuh) -- or one K4 when
// there are no markers.  The host never waits before enqueueing; the status
// is copied out of the device scratch only when asked for.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

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
#include "fsg_skin.cuh"
#include "fsg_dyn_internal.h"

using fsg::Band;
using fsg::Grid;
using fsg::Launchers;
using fsg::MarkerBox;
using fsg::MarkerStencil;
using fsg::Markers;
using fsg::SessionConsts;
using fsg::StepConsts;
using fsg::StepScratch;

namespace {

thread_local char g_err[1024] = "";
// fsg_batch_create: sessions created while this is set adopt the batch's stream
thread_local cudaStream_t g_shared_stream = nullptr;

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

struct GraphEntry {
  int par, pulled, m, copy_mk, frame_on;
  const void* mkp;
  cudaGraphExec_t exec;
};

}  // namespace

struct fsg_session {
  fsg_config cfg{};
  const Launchers* L = nullptr;
  Grid g{};
  cudaStream_t stream = nullptr;
  bool own_stream = true;  // false: a batch's shared stream
  void* buf[2] = {nullptr, nullptr};
  int par = 0;     // A = buf[par], B = buf[par ^ 1]
  int pulled = 0;  // A holds post-collision P (1) or post-stream S (0)
  // last coupled step, for macro()/force readbacks (the buffer it read)
  bool last_valid = false;
  int last_par = 0;
  int prev_pulled = 0;
  bool last_frame_on = false;
  bool stepped = false;
  void* Fext = nullptr;  // SoA 3*n in the storage's math type
  SessionConsts hsc{};
  SessionConsts* d_sc = nullptr;
  StepConsts* d_st = nullptr;
  // per-parity resources
  StepConsts* h_st[2] = {nullptr, nullptr};     // pinned
  StepScratch* d_scr[2] = {nullptr, nullptr};
  StepScratch* h_scr[2] = {nullptr, nullptr};   // pinned
  double* h_mk[2] = {nullptr, nullptr};         // pinned marker slots (copied to d_mk slots)
  double* h_fw[2] = {nullptr, nullptr};         // pinned marker forces (written in place)
  int* h_valid[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};       // last graph of that parity done
  cudaEvent_t ev_mk[2] = {nullptr, nullptr};    // last step that read marker slot k done
  int mk_slot = -1;                             // slot the current marker pointers read
  fsg_frame_state frame{};
  // markers
  int cap = 0;
  int m = 0;
  int n_bodies = 0;
  std::vector<int64_t> offsets;
  double* d_mk = nullptr;  // 2 device slots of [pts 3cap | vel 3cap | nrm 3cap | area cap]
  cudaStream_t cstream = nullptr;                // marker upload (copy) stream
  cudaEvent_t ev_cp[2] = {nullptr, nullptr};     // upload out of pinned slot k done
  Markers mk{};
  bool mk_host = false;
  bool mk_dirty = false;
  int last_mk_slot = 0;       // pinned marker slot the last step read (CouplingStats power)
  MarkerStencil* d_stencil = nullptr;
  MarkerBox* d_boxes = nullptr;
  double* d_fworld = nullptr;
  Band band{};
  double* d_tmp = nullptr;  // readback staging (lazy)
  size_t tmp_bytes = 0;
  double* d_red = nullptr;  // reduction scratch
  std::vector<GraphEntry> graphs;
  fsg_status last{};
  // throughput (fp32) IB: fixed-point tile band
  fsg::FixBand fix{};
  unsigned stamp = 0;          // coupled step stamp (fix.tflag)
  float* d_fcap = nullptr;     // fsg_set_force_capture: the force K4 consumed (AoS fp32)
  // z-slab peer transport (fsg_peer_*): delivery counters written by the
  // neighbours ([0] from the lower, [1] from the upper), the neighbours'
  // buffers, and this session's step count since connecting
  unsigned* d_peer_flags = nullptr;
  struct PeerLink {
    bool on = false, ipc = false, owner = false;
    void* buf[2] = {nullptr, nullptr};
    unsigned* flags = nullptr;
    int nz = 0;
  } nbr[2];
  int nbr_pid_[2] = {0, 0};
  bool peer_on = false;
  unsigned peer_step = 0;
  bool fcap_on = false, last_fcap = false;
  // z-slab halo exchange: session-owned device planes and the event after
  // which this step's boundary planes are packed
  void* d_hsend[2] = {nullptr, nullptr};  // lo, hi
  void* d_hrecv[2] = {nullptr, nullptr};
  cudaEvent_t ev_hpack = nullptr, ev_hrecv = nullptr;
  bool scr_dirty[2] = {false, false};  // d_scr[k] not known to be zero
  bool status_pub[2] = {false, false};  // h_scr[k] written by the step's k_step_end (no copy needed)
  StepConsts last_st{};     // frame constants of the last step (diagnostics)
  StepScratch* d_diag = nullptr;
  // measurement: an event pair around every step
  static constexpr int PROF_CAP = 4096;
  // skinned bodies (fsg_set_skin / fsg_set_pose)
  bool skin = false;
  bool pose_set = false;
  fsg::SkinParams skp{};              // topology + the next step's pose (launch parameter)
  int n_tau = 0;                      // sum of n_dofs over the skinned bodies
  double* d_skin = nullptr;           // rest [3m] | nrest [3m] | ww [KW m] | pts | vel | nrm [3m] | area [m]
  int* d_skin_wb = nullptr;           // [KW m]
  double* d_skin_part = nullptr;      // tau block partials (split path)
  unsigned long long* d_skin_fix = nullptr;  // fused path: fixed-point sums [2][32]
  unsigned* d_skin_ticket = nullptr;
  double* h_wrench[2] = {nullptr, nullptr};  // pinned: tau + stats written by the step of parity p
  // asynchronous macro snapshot (fsg_snapshot_begin / _wait, fsg_write_vtk)
  double* d_snap = nullptr;           // rho [n] | u [3n] of the snapshotted step
  double* h_snap = nullptr;           // pinned copy
  cudaEvent_t ev_snap_k = nullptr;    // snapshot kernel done (session stream)
  cudaEvent_t ev_snap = nullptr;      // copy to h_snap done (copy stream)
  bool snap_pending = false;
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;
  int prof_n = 0;

  void* A() const { return buf[par]; }
  void* B() const { return buf[par ^ 1]; }
};

namespace {

// Wait for the session stream with a short spin before blocking: the
// synchronous step API waits ~10-100 us, where a blocking sync's wake-up
// latency is a visible share of the end-to-end step.
cudaError_t stream_wait(cudaStream_t st) {
  for (int i = 0; i < 20000; ++i) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e != cudaErrorNotReady) return e;
  }
  return cudaStreamSynchronize(st);
}

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
  for (int k = 0; k < 3; ++k) {
    st.a0_f[k] = (float)st.a0[k];
    st.wf_f[k] = (float)st.wf[k];
    st.af_f[k] = (float)st.af[k];
  }
  st._padf = 0.0f;
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
  s->L->get_f(s->g, s->A(), s->pulled, s->d_tmp, s->stream);
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

// Step prologue: pull the frame constants from mapped pinned host memory and
// reset the step scratch (one tiny kernel instead of a copy + a memset node).
__global__ void k_step_begin(const StepConsts* __restrict__ h_st, StepConsts* d_st,
                             StepScratch* d_scr) {
  constexpr int NW = (int)(sizeof(StepConsts) / 4), NS = (int)(sizeof(StepScratch) / 4);
  for (int k = threadIdx.x; k < NW; k += blockDim.x)
    reinterpret_cast<int*>(d_st)[k] = reinterpret_cast<const volatile int*>(h_st)[k];
  for (int k = threadIdx.x; k < NS; k += blockDim.x) reinterpret_cast<int*>(d_scr)[k] = 0;
}
// Step epilogue: publish the step status into mapped pinned host memory.
// Also the throughput path's synchronous steps (fsg_step): launched as a
// programmatic dependent of the banded K4 (which triggers at its start), it
// is resident before K4 ends and copies the status as soon as K4's writes are
// visible -- instead of a device-to-host copy queued behind K4 (C++-host
// synchronous step: c3 148.9 -> 146.7 us, c2 58.8 -> 52 us; publishing from
// K4's last block instead cost the device-timed step 1 us).
// griddepcontrol.wait is a no-op in a normal launch.
__global__ void k_step_end(const StepScratch* __restrict__ d_scr, StepScratch* h_scr) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int NS = (int)(sizeof(StepScratch) / 4);
  for (int k = threadIdx.x; k < NS; k += blockDim.x)
    reinterpret_cast<volatile int*>(h_scr)[k] = reinterpret_cast<const int*>(d_scr)[k];
  __threadfence_system();
}

// Enqueue the body of one coupled step for parity p on the session stream
// (used both for graph capture and, with FSG_NO_GRAPH set, direct launch).
void enqueue_step(fsg_session* s, int p, bool copy_mk, bool frame_on) {
  const Grid& g = s->g;
  const size_t m = (size_t)s->m;
  (void)copy_mk;  // host markers: uploaded by fsg_set_markers (copy stream), waited on by the caller
  k_step_begin<<<1, 64, 0, s->stream>>>(s->h_st[p], s->d_st, s->d_scr[p]);
  if (m && s->skin)
    fsg::skin_update_launch(s->skp, (double*)s->mk.pts, (double*)s->mk.vel, (double*)s->mk.nrm,
                            s->stream);
  if (m) {
    s->L->markers(g, s->buf[p], s->pulled, s->mk, s->d_sc, s->d_st, s->d_stencil, s->d_boxes,
                  s->d_fworld, s->h_fw[p], s->h_valid[p], s->d_scr[p], s->stream);
    if (s->skin)  // parity: the reference's serial order (session.hpp:129-143)
      fsg::skin_tau_launch(s->skp, s->d_fworld, s->d_stencil, s->mk.vel, s->h_wrench[p], 1,
                           nullptr, 0, s->stream);
    s->L->spread(g, s->m, s->d_stencil, s->d_boxes, s->band, s->d_scr[p], s->stream);
  }
  s->L->collide(g, s->buf[p], s->pulled, s->buf[p ^ 1], nullptr, &s->band, s->d_scr[p], s->d_sc,
                s->d_st, s->d_scr[p], 1, frame_on ? 1 : 0, s->stream);
  k_step_end<<<1, 32, 0, s->stream>>>(s->d_scr[p], s->h_scr[p]);
}

bool use_graphs() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("FSG_NO_GRAPH");
    v = (e && e[0] && e[0] != '0') ? 0 : 1;
  }
  return v == 1;
}

void clear_graphs(fsg_session* s) {
  for (auto& e : s->graphs) cudaGraphExecDestroy(e.exec);
  s->graphs.clear();
}

int launch_step(fsg_session* s, int p, bool copy_mk, bool frame_on) {
  if (!use_graphs() || s->skin) {  // skinned: the pose is a launch parameter (not graphable)
    enqueue_step(s, p, copy_mk, frame_on);
    CU_LAUNCH();
    return FSG_OK;
  }
  const void* mkp = s->mk.pts;
  for (auto& e : s->graphs)
    if (e.par == p && e.pulled == s->pulled && e.m == s->m && e.copy_mk == (int)copy_mk &&
        e.frame_on == (int)frame_on && e.mkp == mkp) {
      CU(cudaGraphLaunch(e.exec, s->stream));
      return FSG_OK;
    }
  if (s->graphs.size() >= 16) clear_graphs(s);
  cudaGraph_t graph = nullptr;
  CU(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
  enqueue_step(s, p, copy_mk, frame_on);
  const cudaError_t cap_err = cudaGetLastError();
  cudaError_t e = cudaStreamEndCapture(s->stream, &graph);
  if (cap_err != cudaSuccess || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    return set_err(FSG_ECUDA, "step graph capture failed: %s",
                   cudaGetErrorString(cap_err != cudaSuccess ? cap_err : e));
  }
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_err(FSG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  s->graphs.push_back(GraphEntry{p, s->pulled, s->m, (int)copy_mk, (int)frame_on, mkp, exec});
  CU(cudaGraphLaunch(exec, s->stream));
  return FSG_OK;
}

}  // namespace

// fp32 collision constants (throughput mode) chosen so that the lattice
// conservation identities hold EXACTLY in real arithmetic on the rounded
// constants: with ow1 = omega'/18, ow2 = ow1/2, ow0 = 6 ow1 and
// om1 = 1 - 18 ow1 all exactly representable,
//   mass      om1 + ow0 + 6 ow1 + 12 ow2 = 1
//   momentum  om1 + 3 (2 ow1 + 8 ow2)   = 1
// (the same for guo * w_i).  Independently rounded constants break both by
// ~1e-7 per step -- a systematic drift of rho - 1 and u that reached 7e-5 /
// 2e-4 rel-L2 after 1000 steps of the c2 koi scene; the exact identities leave
// only data-dependent rounding.  omega' differs from omega by a few ulp of
// fp32 (a viscosity change < 1e-6 relative).
static float consistent_w18(double c, bool with_om1) {
  const float a0 = (float)(c / 18.0);
  float best = a0;
  double err = 1e300;
  float up = a0, dn = a0;
  for (int k = 0; k < 64; ++k) {
    for (float a : {up, dn}) {
      const double ad = (double)a;
      const bool ok6 = (double)(float)(6.0 * ad) == 6.0 * ad && (double)(a * 0.5f) == 0.5 * ad;
      const bool ok18 = !with_om1 || (double)(float)(1.0 - 18.0 * ad) == 1.0 - 18.0 * ad;
      const double e = fabs(ad - c / 18.0);
      if (ok6 && ok18 && e < err) {
        err = e;
        best = a;
      }
    }
    up = nextafterf(up, 1e30f);
    dn = nextafterf(dn, -1e30f);
  }
  return best;
}

static void conserving_consts_f32(double omega, double guo, float& om1, float ow[3], float gw[3]) {
  const float o1 = consistent_w18(omega, true);
  ow[1] = o1;
  ow[2] = o1 * 0.5f;
  ow[0] = (float)(6.0 * (double)o1);
  om1 = (float)(1.0 - 18.0 * (double)o1);
  const float g1 = consistent_w18(guo, false);
  gw[1] = g1;
  gw[2] = g1 * 0.5f;
  gw[0] = (float)(6.0 * (double)g1);
}

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
  // kernels address the state with a 32-bit unsigned element index
  if (19ll * cfg.dims[0] * cfg.dims[1] * (cfg.dims[2] + 2) >= (1ll << 32))
    return set_err(FSG_EINPUT, "slab too large: 19 x cells (with halo planes) must be < 2^32");
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
  {
    // dev A/B: elements of padding between direction planes (DRAM channel /
    // L2 slice spread of the 19 per-warp streams on power-of-two planes)
    const char* e = getenv("FSG_PLANE_PAD");
    g.stride = g.plane + (e ? atoll(e) : 0);
  }
  g.zs = 19 * g.stride;
  fsg::grid_offsets(g);

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
    sc.hd_f[a] = (float)sc.hd[a];
  }
  sc.dx_f = (float)sc.dx;
  sc.v2p_f = (float)sc.v2p;
  sc.acc_f = (float)sc.acc;
  sc.kernel = cfg.kernel;
  sc.wall = cfg.wall;
  sc.frame_on = cfg.frame_mode != FSG_FRAME_NONE;
  conserving_consts_f32(sc.omega, sc.guo, sc.om1_f, sc.ow_f, sc.gw_f);
  s->frame.q[0] = 1.0;

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
  if (g_shared_stream) {
    s->stream = g_shared_stream;
    s->own_stream = false;
  } else {
    CUF(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  }
  const size_t fbytes = (size_t)s->L->elem_bytes * (size_t)g.zs * (size_t)(g.nz + 2 * g.zpad);
  for (int k = 0; k < 2; ++k) {
    CUF(cudaMalloc(&s->buf[k], fbytes));
    CUF(cudaMemsetAsync(s->buf[k], 0, fbytes, s->stream));
    CUF(cudaMalloc(&s->d_scr[k], sizeof(StepScratch)));
    CUF(cudaMemsetAsync(s->d_scr[k], 0, sizeof(StepScratch), s->stream));
    CUF(cudaMallocHost(&s->h_st[k], sizeof(StepConsts)));
    CUF(cudaMallocHost(&s->h_scr[k], sizeof(StepScratch)));
    std::memset(s->h_scr[k], 0, sizeof(StepScratch));
    CUF(cudaEventCreateWithFlags(&s->ev[k], cudaEventDisableTiming));
    CUF(cudaEventRecord(s->ev[k], s->stream));
  }
  CUF(cudaMalloc(&s->d_sc, sizeof(SessionConsts)));
  CUF(cudaMalloc(&s->d_st, sizeof(StepConsts)));
  CUF(cudaMemcpyAsync(s->d_sc, &s->hsc, sizeof(SessionConsts), cudaMemcpyHostToDevice, s->stream));
  s->cap = cfg.max_markers;
  CUF(cudaMalloc(&s->d_mk, sizeof(double) * 2 * 10 * (size_t)s->cap));
  CUF(cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    CUF(cudaEventCreateWithFlags(&s->ev_cp[k], cudaEventDisableTiming));
    CUF(cudaEventRecord(s->ev_cp[k], s->cstream));
  }
  for (int k = 0; k < 2; ++k) {
    CUF(cudaMallocHost(&s->h_mk[k], sizeof(double) * 10 * (size_t)s->cap));
    CUF(cudaMallocHost(&s->h_fw[k], sizeof(double) * 3 * (size_t)s->cap));
    CUF(cudaMallocHost(&s->h_valid[k], sizeof(int) * (size_t)s->cap));
    CUF(cudaEventCreateWithFlags(&s->ev_mk[k], cudaEventDisableTiming));
    CUF(cudaEventRecord(s->ev_mk[k], s->stream));
  }
  CUF(cudaMalloc(&s->d_stencil, sizeof(MarkerStencil) * (size_t)s->cap));
  CUF(cudaMalloc(&s->d_boxes, sizeof(MarkerBox) * (size_t)s->cap));
  CUF(cudaMalloc(&s->d_fworld, sizeof(double) * 3 * (size_t)s->cap));
  s->band.cap = std::min<long long>(g.n, 16ll << 20);
  CUF(cudaMalloc(&s->band.F, sizeof(double) * 3 * (size_t)s->band.cap));
  CUF(cudaMalloc(&s->d_diag, sizeof(StepScratch)));
  if (s->L->markers_fix) {
    fsg::FixBand& fb = s->fix;
    fb.tnx = (g.nx + 3) / 4;
    fb.tny = (g.ny + 3) / 4;
    fb.tnz = (g.nz + 3) / 4;
    const size_t ntile = (size_t)fb.tnx * fb.tny * fb.tnz;
    CUF(cudaMalloc(&fb.F, sizeof(unsigned long long) * 3 * (size_t)g.n));
    CUF(cudaMemsetAsync(fb.F, 0, sizeof(unsigned long long) * 3 * (size_t)g.n, s->stream));
    CUF(cudaMalloc(&fb.tflag, sizeof(unsigned) * ntile));
    CUF(cudaMemsetAsync(fb.tflag, 0, sizeof(unsigned) * ntile, s->stream));
    // "every tile of the step stamped" flag (release by the marker grid,
    // acquire by the banded K4 before its first stamp load); FSG_STAMP_FLAG=0:
    // the block fence before the marker blocks' trigger only
    const char* sf = getenv("FSG_STAMP_FLAG");
    if (!(sf && sf[0] == '0')) {
      CUF(cudaMalloc(&fb.ready, sizeof(unsigned)));
      CUF(cudaMemsetAsync(fb.ready, 0, sizeof(unsigned), s->stream));
    }
    // stamped-tile list: the band phase takes the listed tiles dynamically
    // instead of scanning every tile's flag, so blocks leaving phase A early
    // take the band while the late ones finish.  On by default when the state
    // exceeds L2 (the phase-A tail is then several us wide: c3 141.4 ->
    // 137.6 us with 3 marker blocks per SM); off for L2-resident grids (c2
    // 43.1 -> 44.8 us).  FSG_TILE_LIST=0/1 overrides.
    const char* tl = getenv("FSG_TILE_LIST");
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, cfg.device);
    const bool big = (double)g.n * 152.0 > (double)l2;
    if (tl ? tl[0] == '1' : big) {
      const size_t tcap = std::min<size_t>(ntile, 8 * (size_t)std::max(1, cfg.max_markers));
      CUF(cudaMalloc(&fb.tlist, sizeof(int) * tcap));
    }

  }
  if (g.zpad) {
    const size_t hb = (size_t)5 * g.plane * s->L->elem_bytes;
    for (int k = 0; k < 2; ++k) {
      CUF(cudaMalloc(&s->d_hsend[k], hb));
      CUF(cudaMalloc(&s->d_hrecv[k], hb));
    }
    CUF(cudaEventCreateWithFlags(&s->ev_hpack, cudaEventDisableTiming));
    CUF(cudaEventCreateWithFlags(&s->ev_hrecv, cudaEventDisableTiming));
    CUF(cudaEventRecord(s->ev_hpack, s->stream));
  }
  s->L->fill_rest(g, s->A(), s->stream);
  if (cudaGetLastError() != cudaSuccess) return fail(set_err(FSG_ECUDA, "fill_rest launch failed"));
  if (cudaStreamSynchronize(s->stream) != cudaSuccess)
    return fail(set_err(FSG_ECUDA, "session init failed"));
#undef CUF
  s->pulled = 0;
  *out = s;
  return FSG_OK;
}

int fsg_destroy(fsg_session* s) {
  if (!s) return FSG_OK;
  cudaSetDevice(s->cfg.device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  clear_graphs(s);
  for (auto& e : s->prof_ev) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    cudaFree(s->buf[k]);
    cudaFree(s->d_scr[k]);
    if (s->h_st[k]) cudaFreeHost(s->h_st[k]);
    if (s->h_scr[k]) cudaFreeHost(s->h_scr[k]);
    if (s->h_mk[k]) cudaFreeHost(s->h_mk[k]);
    if (s->h_fw[k]) cudaFreeHost(s->h_fw[k]);
    if (s->h_valid[k]) cudaFreeHost(s->h_valid[k]);
    if (s->ev[k]) cudaEventDestroy(s->ev[k]);
    if (s->ev_mk[k]) cudaEventDestroy(s->ev_mk[k]);
  }
  cudaFree(s->Fext);
  cudaFree(s->d_sc);
  cudaFree(s->d_st);
  cudaFree(s->d_mk);
  for (int k = 0; k < 2; ++k)
    if (s->ev_cp[k]) cudaEventDestroy(s->ev_cp[k]);
  if (s->cstream) {
    cudaStreamSynchronize(s->cstream);
    cudaStreamDestroy(s->cstream);
  }
  cudaFree(s->d_stencil);
  cudaFree(s->d_boxes);
  cudaFree(s->d_fworld);
  cudaFree(s->band.F);
  cudaFree(s->fix.F);
  cudaFree(s->fix.tflag);
  cudaFree(s->fix.tlist);
  cudaFree(s->fix.ready);
  cudaFree(s->d_fcap);
  fsg_peer_disconnect(s);
  cudaFree(s->d_peer_flags);
  for (int k = 0; k < 2; ++k) {
    cudaFree(s->d_hsend[k]);
    cudaFree(s->d_hrecv[k]);
  }
  if (s->ev_hpack) cudaEventDestroy(s->ev_hpack);
  if (s->ev_hrecv) cudaEventDestroy(s->ev_hrecv);
  cudaFree(s->d_diag);
  if (s->snap_pending && s->ev_snap) cudaEventSynchronize(s->ev_snap);
  cudaFree(s->d_snap);
  if (s->h_snap) cudaFreeHost(s->h_snap);
  if (s->ev_snap) cudaEventDestroy(s->ev_snap);
  if (s->ev_snap_k) cudaEventDestroy(s->ev_snap_k);
  cudaFree(s->d_skin);
  cudaFree(s->d_skin_wb);
  cudaFree(s->d_skin_part);
  cudaFree(s->d_skin_fix);
  cudaFree(s->d_skin_ticket);
  for (int k = 0; k < 2; ++k)
    if (s->h_wrench[k]) cudaFreeHost(s->h_wrench[k]);
  cudaFree(s->d_tmp);
  cudaFree(s->d_red);
  if (s->stream && s->own_stream) cudaStreamDestroy(s->stream);
  delete s;
  return FSG_OK;
}

void* fsg_stream(fsg_session* s) { return s ? (void*)s->stream : nullptr; }

// --------------------------------------------------------------- state --
static void state_changed(fsg_session* s) {
  s->last_valid = false;
  s->stepped = false;
}

int fsg_reset_rest(fsg_session* s) {
  CU(cudaSetDevice(s->cfg.device));
  s->L->fill_rest(s->g, s->A(), s->stream);
  CU_LAUNCH();
  s->pulled = 0;
  state_changed(s);
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
  s->L->init_eq(s->g, s->d_tmp, s->d_tmp + n, s->A(), s->stream);
  CU_LAUNCH();
  s->pulled = 0;
  state_changed(s);
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
  s->L->set_f(s->g, s->d_tmp, s->A(), s->stream);
  CU_LAUNCH();
  s->pulled = 0;
  state_changed(s);
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_get_f(fsg_session* s, double* f) {
  if (!f) return set_err(FSG_EINPUT, "fsg_get_f: null");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 19 * n);
  if (rc) return rc;
  s->L->get_f(s->g, s->A(), s->pulled, s->d_tmp, s->stream);
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
  const int p = s->par;
  CU(cudaEventSynchronize(s->ev[p]));
  CU(cudaMemsetAsync(s->d_scr[p], 0, sizeof(StepScratch), s->stream));
  s->L->collide(s->g, s->A(), s->pulled, s->B(), s->Fext, nullptr, nullptr, s->d_sc, s->d_st,
                s->d_scr[p], 0, 0, s->stream);
  CU_LAUNCH();
  CU(cudaMemcpyAsync(s->h_scr[p], s->d_scr[p], sizeof(StepScratch), cudaMemcpyDeviceToHost,
                     s->stream));
  CU(cudaEventRecord(s->ev[p], s->stream));
  CU(cudaStreamSynchronize(s->stream));
  s->par ^= 1;
  s->pulled = 1;
  state_changed(s);
  decode_status(*s->h_scr[p], &s->last, false);
  s->scr_dirty[p] = true;
  if (st) *st = s->last;
  return FSG_OK;
}

int fsg_macroscopic(fsg_session* s, double* rho, double* u, int* nonpos) {
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 4 * n);
  if (rc) return rc;
  const int p = s->par;
  CU(cudaStreamSynchronize(s->stream));
  CU(cudaMemsetAsync(s->d_scr[p], 0, sizeof(StepScratch), s->stream));
  s->L->macroscopic(s->g, s->A(), s->pulled, s->Fext, s->d_tmp, s->d_tmp + n, s->d_scr[p], s->stream);
  CU_LAUNCH();
  if (rho) CU(cudaMemcpyAsync(rho, s->d_tmp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
  if (u) CU(cudaMemcpyAsync(u, s->d_tmp + n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s->stream));
  StepScratch sc;
  CU(cudaMemcpyAsync(&sc, s->d_scr[p], sizeof(StepScratch), cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  if (nonpos) *nonpos = sc.nonpos;
  s->scr_dirty[p] = true;
  s->last_valid = false;  // the step scratch of parity p was reused
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

// frame::recenter (frame.hpp:132-154) enqueued on the session stream: the
// shifted, clamped gather of the post-stream state, and the frame origin.
static int recenter_async(fsg_session* s, const int shift[3]) {
  s->L->recenter(s->g, s->A(), s->pulled, s->B(), shift[0], shift[1], shift[2], s->stream);
  CU_LAUNCH();
  s->par ^= 1;
  s->pulled = 0;
  state_changed(s);
  // frame.hpp:152-153: p += R * (shift * dx)
  double R[9];
  quat_to_R(s->frame.q, R);
  const double off[3] = {shift[0] * s->cfg.dx, shift[1] * s->cfg.dx, shift[2] * s->cfg.dx};
  double r[3];
  mat_vec(R, off, r);
  for (int k = 0; k < 3; ++k) s->frame.p[k] = s->frame.p[k] + r[k];
  return FSG_OK;
}

int fsg_recenter(fsg_session* s, const int shift[3]) {
  if (s->g.zpad) return set_err(FSG_EINPUT, "recenter is not defined for z-slab sessions");
  CU(cudaSetDevice(s->cfg.device));
  const int rc = recenter_async(s, shift);
  if (rc) return rc;
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

// -------------------------------------------------------------- markers --
static int set_markers_common(fsg_session* s, int n_bodies, const int64_t* off) {
  if (n_bodies < 0) return set_err(FSG_EINPUT, "negative body count");
  if (n_bodies > 0 && s->g.zpad)
    return set_err(FSG_EINPUT, "IB markers on a z-slab session are not supported (the sharded "
                               "config is pure LBM, SURVEY.md 8(e))");
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
  // two slot pairs (pinned host + device), alternated so the host fills one
  // while a queued step may still read the other.  The pinned slot is copied
  // to its device slot on the copy stream right away -- while the host goes
  // on to enqueue the step -- and the marker kernel reads device memory (a
  // zero-copy read from pinned memory would put PCIe round trips at the head
  // of the marker kernel, which gates the collide kernel's start).
  const int p = s->mk_slot < 0 ? 0 : (s->mk_slot ^ 1);
  double* d = s->d_mk + (size_t)p * 10 * (size_t)s->cap;
  if (m) {
    if (!pts || !vel || !nrm || !area) return set_err(FSG_EINPUT, "fsg_set_markers: null array");
    CU(cudaEventSynchronize(s->ev_cp[p]));  // the previous copy out of this pinned slot is done
    double* h = s->h_mk[p];
    std::memcpy(h, pts, sizeof(double) * 3 * m);
    std::memcpy(h + 3 * m, vel, sizeof(double) * 3 * m);
    std::memcpy(h + 6 * m, nrm, sizeof(double) * 3 * m);
    std::memcpy(h + 9 * m, area, sizeof(double) * m);
    CU(cudaStreamWaitEvent(s->cstream, s->ev_mk[p], 0));  // the last step that read device slot p
    CU(cudaMemcpyAsync(d, h, sizeof(double) * 10 * m, cudaMemcpyHostToDevice, s->cstream));
    CU(cudaEventRecord(s->ev_cp[p], s->cstream));
  }
  s->mk = Markers{d, d + 3 * m, d + 6 * m, d + 9 * m, (int)m};
  s->skin = false;
  s->mk_slot = p;
  s->mk_host = true;
  s->mk_dirty = m > 0;
  return FSG_OK;
}

int fsg_set_markers_device(fsg_session* s, int n_bodies, const int64_t* off, const double* pts,
                           const double* vel, const double* nrm, const double* area) {
  int rc = set_markers_common(s, n_bodies, off);
  if (rc) return rc;
  s->mk = Markers{pts, vel, nrm, area, s->m};
  s->skin = false;
  s->mk_host = false;
  s->mk_slot = -1;
  s->mk_dirty = false;
  return FSG_OK;
}

// -------------------------------------------------------- skinned bodies --
int fsg_set_skin(fsg_session* s, int n_bodies, const int64_t* off, const fsg_skeleton* sk,
                 const double* rest, const double* nrest, const double* weights,
                 const double* areas) {
  if (n_bodies < 1 || n_bodies > FSG_SKIN_MAX_BODIES)
    return set_err(FSG_EINPUT, "fsg_set_skin: 1..%d bodies", FSG_SKIN_MAX_BODIES);
  if (!sk || !rest || !nrest || !weights || !areas) return set_err(FSG_EINPUT, "fsg_set_skin: null array");
  int rc = set_markers_common(s, n_bodies, off);
  if (rc) return rc;
  const int m = s->m;
  fsg::SkinParams& P = s->skp;
  P = fsg::SkinParams{};
  P.nb = n_bodies;
  P.m = m;
  std::vector<int> wb((size_t)fsg::SKIN_KW * m, -1);
  std::vector<double> ww((size_t)fsg::SKIN_KW * m, 0.0);
  size_t wpos = 0;  // weights: per body, n_links columns per marker
  int nt = 0;
  for (int b = 0; b < n_bodies; ++b) {
    const fsg_skeleton& k = sk[b];
    if (k.n_links < 1 || k.n_links > FSG_SKIN_MAX_LINKS)
      return set_err(FSG_EINPUT, "body %d: n_links must be 1..%d", b, FSG_SKIN_MAX_LINKS);
    if (k.n_dofs < 0 || k.n_dofs > 6 + FSG_SKIN_MAX_LINKS)
      return set_err(FSG_EINPUT, "body %d: bad n_dofs %d", b, k.n_dofs);
    if (k.floating_base && k.n_dofs < 6) return set_err(FSG_EINPUT, "body %d: floating base needs 6 dofs", b);
    for (int j = 1; j < k.n_links; ++j) {
      if (k.parent[j] < 0 || k.parent[j] >= j)
        return set_err(FSG_EINPUT, "body %d: link %d parent must precede it", b, j);
      if (k.dof_index[j] >= k.n_dofs) return set_err(FSG_EINPUT, "body %d: dof index out of range", b);
    }
    fsg::SkinBody& B = P.body[b];
    B.m0 = (int)off[b];
    B.m1 = (int)off[b + 1];
    B.n_links = k.n_links;
    B.floating = k.floating_base ? 1 : 0;
    B.n_dofs = k.n_dofs;
    B.tau_off = nt;
    nt += k.n_dofs;
    for (int j = 0; j < FSG_SKIN_MAX_LINKS; ++j) {
      int a = j < k.n_links ? j : -1;  // chain tables for the fused marker kernel
      for (int l = 0; l < FSG_SKIN_MAX_LINKS; ++l) B.lvl[j][l] = -1;
      for (int l = 0; l < FSG_SKIN_MAX_LINKS; ++l) {
        B.anc[j][l] = (signed char)(a > 0 ? a : -1);
        if (a > 0) B.lvl[j][a] = (signed char)(l + 1);
        a = a > 0 ? k.parent[a] : -1;
      }
      B.parent[j] = j < k.n_links ? k.parent[j] : -1;
      B.dof[j] = (j > 0 && j < k.n_links) ? k.dof_index[j] : -1;
      for (int c = 0; c < 3; ++c) B.axis[j][c] = j < k.n_links ? k.axis[j][c] : 0.0;
    }
    B.max_level = 0;
    for (int j = 0; j < FSG_SKIN_MAX_LINKS; ++j)
      for (int l = 0; l < FSG_SKIN_MAX_LINKS; ++l)
        if (B.lvl[j][l] > B.max_level) B.max_level = B.lvl[j][l];
    for (int d = 0; d < 6 + FSG_SKIN_MAX_LINKS; ++d) B.dof_link[d] = -1;
    for (int j = 1; j < k.n_links; ++j)
      if (k.dof_index[j] >= 0) B.dof_link[k.dof_index[j]] = (signed char)j;
    for (int i = B.m0; i < B.m1; ++i) {
      int nz = 0;
      for (int j = 0; j < k.n_links; ++j) {
        const double w = weights[wpos + (size_t)(i - B.m0) * k.n_links + j];
        if (w == 0.0) continue;  // skin_point skips zero weights (skinning.hpp:108)
        if (nz == fsg::SKIN_KW)
          return set_err(FSG_EINPUT, "marker %d has more than %d nonzero skin weights", i, fsg::SKIN_KW);
        wb[(size_t)fsg::SKIN_KW * i + nz] = j;
        ww[(size_t)fsg::SKIN_KW * i + nz] = w;
        ++nz;
      }
    }
    wpos += (size_t)(B.m1 - B.m0) * k.n_links;
  }
  s->n_tau = nt;
  CU(cudaSetDevice(s->cfg.device));
  CU(cudaStreamSynchronize(s->stream));  // a queued step may still read the old arrays
  cudaFree(s->d_skin);
  cudaFree(s->d_skin_wb);
  s->d_skin = nullptr;
  s->d_skin_wb = nullptr;
  const size_t M = (size_t)std::max(m, 1);
  CU(cudaMalloc(&s->d_skin, sizeof(double) * (3 + 3 + fsg::SKIN_KW + 9 + 1) * M));
  CU(cudaMalloc(&s->d_skin_wb, sizeof(int) * fsg::SKIN_KW * M));
  double* d = s->d_skin;
  CU(cudaMemcpy(d, rest, sizeof(double) * 3 * m, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d + 3 * M, nrest, sizeof(double) * 3 * m, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d + 6 * M, ww.data(), sizeof(double) * ww.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d + (6 + fsg::SKIN_KW + 9) * M, areas, sizeof(double) * m, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(s->d_skin_wb, wb.data(), sizeof(int) * wb.size(), cudaMemcpyHostToDevice));
  {
    int mmax = 1;
    for (int b = 0; b < n_bodies; ++b) mmax = std::max(mmax, (int)(off[b + 1] - off[b]));
    const size_t bpb = (size_t)(mmax + fsg::SKIN_TAU_THREADS - 1) / fsg::SKIN_TAU_THREADS;
    // block partials of the split tau kernel [bodies][blocks][ACC_N]
    cudaFree(s->d_skin_part);
    s->d_skin_part = nullptr;
    CU(cudaMalloc(&s->d_skin_part, sizeof(double) * fsg::SKIN_ACC_N * bpb * n_bodies));
    if (!s->d_skin_ticket) {  // [0] tau ticket, [1] marker blocks done (split path)
      CU(cudaMalloc(&s->d_skin_ticket, 2 * sizeof(unsigned)));
      CU(cudaMemset(s->d_skin_ticket, 0, 2 * sizeof(unsigned)));
    }
  }
  if (!s->d_skin_fix) {
    CU(cudaMalloc(&s->d_skin_fix, sizeof(unsigned long long) * 64 * fsg::SKIN_FIX_REP));
    CU(cudaMemset(s->d_skin_fix, 0, sizeof(unsigned long long) * 64 * fsg::SKIN_FIX_REP));
  }
  P.part = s->d_skin_part;
  P.ticket = s->d_skin_ticket;
  P.rest = d;
  P.nrest = d + 3 * M;
  P.ww = d + 6 * M;
  P.wb = s->d_skin_wb;
  double* mk = d + (6 + fsg::SKIN_KW) * M;
  s->mk = Markers{mk, mk + 3 * M, mk + 6 * M, mk + 9 * M, m};
  for (int k = 0; k < 2; ++k)
    if (!s->h_wrench[k]) {
      CU(cudaMallocHost(&s->h_wrench[k], sizeof(double) * (6 + FSG_SKIN_MAX_LINKS + fsg::SKIN_NSTAT) *
                                             FSG_SKIN_MAX_BODIES));
      std::memset(s->h_wrench[k], 0, sizeof(double) * (6 + FSG_SKIN_MAX_LINKS + fsg::SKIN_NSTAT) *
                                         FSG_SKIN_MAX_BODIES);
    }
  s->mk_host = false;
  s->mk_slot = -1;
  s->mk_dirty = false;
  s->skin = true;
  s->pose_set = false;
  return FSG_OK;
}

int fsg_set_pose(fsg_session* s, const fsg_body_pose* poses) {
  if (!s->skin) return set_err(FSG_ESTATE, "fsg_set_pose: no skinned bodies (fsg_set_skin)");
  if (!poses) return set_err(FSG_EINPUT, "fsg_set_pose: null poses");
  for (int b = 0; b < s->skp.nb; ++b) s->skp.body[b].pose = poses[b];
  s->pose_set = true;
  return FSG_OK;
}

int fsg_get_body_wrench(fsg_session* s, double* tau, double* stats) {
  CU(cudaSetDevice(s->cfg.device));
  if (!s->skin) return set_err(FSG_ESTATE, "fsg_get_body_wrench: no skinned bodies");
  CU(stream_wait(s->stream));
  if (!s->stepped) return set_err(FSG_ESTATE, "no coupled step yet");
  const double* w = s->h_wrench[s->last_par];
  if (tau) std::memcpy(tau, w, sizeof(double) * s->n_tau);
  if (stats) std::memcpy(stats, w + s->n_tau, sizeof(double) * fsg::SKIN_NSTAT * s->skp.nb);
  return FSG_OK;
}

int fsg_step_skinned(fsg_session* s, const fsg_frame_state* fs, const fsg_body_pose* poses,
                     fsg_status* st, double* tau, double* stats) {
  int rc = FSG_OK;
  if (fs && (rc = fsg_set_frame(s, fs))) return rc;
  if ((rc = fsg_set_pose(s, poses))) return rc;
  if ((rc = fsg_step(s, st))) return rc;
  return fsg_get_body_wrench(s, tau, stats);
}

int fsg_get_markers(fsg_session* s, double* pts, double* vel, double* nrm) {
  CU(cudaSetDevice(s->cfg.device));
  CU(stream_wait(s->stream));
  const size_t m = (size_t)s->m;
  if (!m) return FSG_OK;
  if (pts) CU(cudaMemcpy(pts, s->mk.pts, sizeof(double) * 3 * m, cudaMemcpyDefault));
  if (vel) CU(cudaMemcpy(vel, s->mk.vel, sizeof(double) * 3 * m, cudaMemcpyDefault));
  if (nrm) CU(cudaMemcpy(nrm, s->mk.nrm, sizeof(double) * 3 * m, cudaMemcpyDefault));
  return FSG_OK;
}

static int peer_wait(fsg_session* s, unsigned* flag, unsigned v);
static int peer_signal(fsg_session* s, unsigned* flag, unsigned v);

// ----------------------------------------------------------------- step --
// publish: the throughput step's status goes to pinned h_scr by k_step_end
// (a synchronous step then needs no device-to-host copy)
static int step_impl(fsg_session* s, bool publish);

int fsg_step_async(fsg_session* s) { return step_impl(s, false); }

static int step_impl(fsg_session* s, bool publish) {
  CU(cudaSetDevice(s->cfg.device));
  if (s->skin && s->m && !s->pose_set)
    return set_err(FSG_ESTATE, "skinned bodies: fsg_set_pose has not been called");
  const int p = s->par;
  // the fp64 graph reads its frame constants from pinned slot p: wait until
  // the step that last used it is done.  The throughput path passes them by
  // value and the device only WRITES its pinned slots (status, marker
  // forces), which the host reads after a stream sync -- no wait, so the
  // host can run several steps ahead.
  if (!s->L->markers_fix) CU(cudaEventSynchronize(s->ev[p]));
  frame_consts(s->frame, *s->h_st[p]);
  const bool frame_on = s->cfg.frame_mode != FSG_FRAME_NONE;
  const bool copy_mk = s->mk_host && s->mk_dirty;
  if (copy_mk) CU(cudaStreamWaitEvent(s->stream, s->ev_cp[s->mk_slot], 0));  // markers uploaded
  if (s->L->markers_fix) {
    // throughput path: frame constants by value; the status stays in the
    // device scratch until the host asks for it (fsg_last_status)
    const StepConsts st = *s->h_st[p];
    s->last_st = st;
    if (s->scr_dirty[p]) CU(cudaMemsetAsync(s->d_scr[p], 0, sizeof(StepScratch), s->stream));
    const bool prof = s->prof && s->prof_n < fsg_session::PROF_CAP;
    cudaEvent_t* pe = prof ? &s->prof_ev[2 * (size_t)s->prof_n] : nullptr;
    if (prof) CU(cudaEventRecord(pe[0], s->stream));
    if (s->m) {
      // coupled step: markers, then the banded K4 as their programmatic
      // dependent (no event between the two, or the overlap is lost).  The
      // fixed-point force field is consumed (re-zeroed) by that K4, so a step
      // without markers is the plain fluid K4 below.
      fsg::FixBand fb = s->fix;
      fb.stamp = ++s->stamp;
      fb.fcap = s->fcap_on ? s->d_fcap : nullptr;
      // skinned bodies: up to two are skinned and reduced inside the marker
      // kernel; more take the separate skin kernels around it
      const bool fused = s->skin && s->skp.nb <= 2;
      const bool split = s->skin && !fused;
      fsg::SkinOut so{};
      if (fused) {
        so.acc = s->d_skin_fix;
        so.out = s->h_wrench[p];
        so.nb = s->skp.nb;
        so.nt = s->n_tau;
        for (int b = 0; b < s->skp.nb; ++b) {
          so.ndof[b] = s->skp.body[b].n_dofs;
          so.off[b] = s->skp.body[b].tau_off;
        }
      }
      if (split)
        fsg::skin_update_launch(s->skp, (double*)s->mk.pts, (double*)s->mk.vel,
                                (double*)s->mk.nrm, s->stream);
      const int km_blocks =
          s->L->markers_fix(s->g, s->buf[p], s->pulled, s->mk, s->d_sc, st, s->d_stencil, s->d_fworld,
                            s->h_fw[p], s->h_valid[p], fb, s->d_scr[p],
                            split ? s->d_skin_ticket + 1 : nullptr, split ? 1 : 0,
                            fused ? &s->skp : nullptr, fused ? s->d_skin_fix : nullptr, s->stream);
      s->L->collide_band(s->g, s->buf[p], s->pulled, s->buf[p ^ 1], fb, s->d_sc, st,
                         frame_on ? 1 : 0, s->d_scr[p], s->d_scr[p ^ 1], 1, so, s->stream);
      if (split)  // beside K4's first phase; fixed tree order; tau + stats into pinned memory
        fsg::skin_tau_launch(s->skp, s->d_fworld, s->d_stencil, s->mk.vel, s->h_wrench[p], 0,
                             s->d_skin_ticket + 1, (unsigned)km_blocks, s->stream);
    } else if (s->g.zpad && s->peer_on) {
      // z-slab, peer transport: the interior planes (no halo needed), then a
      // stream-ordered wait until both neighbours delivered their previous
      // step's crossing planes into this session's halo (and finished reading
      // the halo this step overwrites in theirs), then the two boundary planes
      // with their crossing populations stored straight into the neighbours'
      // halo planes, then the delivery counter written into each neighbour
      const unsigned n = ++s->peer_step;
      s->L->collide_fix(s->g, s->buf[p], s->pulled, s->buf[p ^ 1], s->d_sc, st, frame_on ? 1 : 0,
                        s->d_scr[p], s->d_scr[p ^ 1], 2, fsg::PeerOut{nullptr, nullptr}, s->stream);
      for (int k = 0; k < 2; ++k)
        if (s->nbr[k].on) {
          int rc = peer_wait(s, s->d_peer_flags + k, n);
          if (rc) return rc;
        }
      fsg::PeerOut po{nullptr, nullptr};
      if (s->nbr[0].on)  // lower neighbour: its top halo plane (local z = its nz)
        po.lo = (float*)s->nbr[0].buf[p ^ 1] + s->g.zs * (long long)(s->nbr[0].nz + s->g.zpad);
      if (s->nbr[1].on)  // upper neighbour: its bottom halo plane (local z = -1)
        po.hi = (float*)s->nbr[1].buf[p ^ 1];
      s->L->collide_fix(s->g, s->buf[p], s->pulled, s->buf[p ^ 1], s->d_sc, st, frame_on ? 1 : 0,
                        s->d_scr[p], s->d_scr[p ^ 1], 1, po, s->stream);
      CU_LAUNCH();
      if (s->nbr[0].on) {
        int rc = peer_signal(s, s->nbr[0].flags + 1, n + 1);
        if (rc) return rc;
      }
      if (s->nbr[1].on) {
        int rc = peer_signal(s, s->nbr[1].flags + 0, n + 1);
        if (rc) return rc;
      }
    } else if (s->g.zpad) {
      // z-slab: the two boundary planes first, packed for the neighbours
      // (fsg_halo_begin lets a comm stream start on them), then the interior
      s->L->collide_fix(s->g, s->buf[p], s->pulled, s->buf[p ^ 1], s->d_sc, st, frame_on ? 1 : 0,
                        s->d_scr[p], s->d_scr[p ^ 1], 1, fsg::PeerOut{nullptr, nullptr}, s->stream);
      s->L->halo_pack(s->g, s->buf[p ^ 1], s->d_hsend[0], s->d_hsend[1], s->stream);
      CU(cudaEventRecord(s->ev_hpack, s->stream));
      s->L->collide_fix(s->g, s->buf[p], s->pulled, s->buf[p ^ 1], s->d_sc, st, frame_on ? 1 : 0,
                        s->d_scr[p], s->d_scr[p ^ 1], 2, fsg::PeerOut{nullptr, nullptr}, s->stream);
    } else {
      s->L->collide_fix(s->g, s->buf[p], s->pulled, s->buf[p ^ 1], s->d_sc, st, frame_on ? 1 : 0,
                        s->d_scr[p], s->d_scr[p ^ 1], 0, fsg::PeerOut{nullptr, nullptr}, s->stream);
    }
    CU_LAUNCH();
    s->status_pub[p] = false;
    if (publish) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(32);
      cfg.stream = s->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CU(cudaLaunchKernelEx(&cfg, k_step_end, (const StepScratch*)s->d_scr[p], s->h_scr[p]));
      s->status_pub[p] = true;
    }
    if (prof) {
      CU(cudaEventRecord(pe[1], s->stream));
      ++s->prof_n;
    }
    s->scr_dirty[p] = true;       // holds this step's status
    s->scr_dirty[p ^ 1] = false;  // reset by K4 for the next step
  } else {
    int rc = launch_step(s, p, copy_mk, frame_on);
    if (rc) return rc;
    if (s->g.zpad) {  // parity mode: the whole step, then the planes for the neighbours
      s->L->halo_pack(s->g, s->buf[p ^ 1], s->d_hsend[0], s->d_hsend[1], s->stream);
      CU(cudaEventRecord(s->ev_hpack, s->stream));
    }
  }
  CU(cudaEventRecord(s->ev[p], s->stream));
  if (s->mk_host && s->mk_slot >= 0) CU(cudaEventRecord(s->ev_mk[s->mk_slot], s->stream));
  s->last_par = p;
  if (s->mk_host && s->mk_slot >= 0) s->last_mk_slot = s->mk_slot;
  s->prev_pulled = s->pulled;
  s->last_frame_on = frame_on;
  s->last_fcap = s->fcap_on && s->m > 0 && s->L->markers_fix != nullptr;
  s->par ^= 1;
  s->pulled = 1;
  s->last_valid = true;
  s->stepped = true;
  s->mk_dirty = false;
  return FSG_OK;
}

int fsg_last_status(fsg_session* s, fsg_status* st) {
  if (s->stepped && s->L->markers_fix && !s->status_pub[s->last_par]) {
    // throughput path: the last step's status is still in its device
    // scratch (the next K4 would reset it, but none is enqueued)
    CU(cudaMemcpyAsync(s->h_scr[s->last_par], s->d_scr[s->last_par], sizeof(StepScratch),
                       cudaMemcpyDeviceToHost, s->stream));
  }
  CU(stream_wait(s->stream));
  if (!s->stepped) {
    if (st) *st = s->last;
    return FSG_OK;
  }
  const StepScratch& sc = *s->h_scr[s->last_par];
  if (sc.band_overflow)
    return set_err(FSG_ESTATE, "IB band bounding box exceeds capacity (%lld cells)",
                   (long long)s->band.cap);
  decode_status(sc, &s->last, true);
  if (st) *st = s->last;
  return FSG_OK;
}

int fsg_step(fsg_session* s, fsg_status* st) {
  int rc = step_impl(s, true);
  if (rc) return rc;
  return fsg_last_status(s, st);
}

int fsg_get_marker_forces(fsg_session* s, double* fw, int* valid, double* stats) {
  CU(cudaSetDevice(s->cfg.device));
  const size_t m = (size_t)s->m;
  // the marker kernel wrote the forces straight into mapped pinned memory
  CU(stream_wait(s->stream));
  if (!s->stepped) return set_err(FSG_ESTATE, "no coupled step yet");
  const double* f = s->h_fw[s->last_par];
  const int* vv = s->h_valid[s->last_par];
  if (fw) std::memcpy(fw, f, sizeof(double) * 3 * m);
  if (valid) std::memcpy(valid, vv, sizeof(int) * m);
  if (stats) {
    std::vector<double> vel;
    const double* v = nullptr;
    if (s->mk_host) {
      v = s->h_mk[s->last_mk_slot] + 3 * m;  // the velocities the last step read
    } else if (m) {
      vel.resize(3 * m);
      CU(cudaMemcpy(vel.data(), s->mk.vel, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost));
      v = vel.data();
    }
    // CouplingStats, serial in marker order (session.hpp:141-143)
    for (int b = 0; b < s->n_bodies; ++b) {
      double tf[3] = {0, 0, 0}, tb[3] = {0, 0, 0}, power = 0.0;
      for (int64_t i = s->offsets[b]; i < s->offsets[b + 1]; ++i) {
        if (!vv[i]) continue;
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
  std::vector<MarkerBox> bx(m);
  if (m) {
    CU(cudaMemcpyAsync(st.data(), s->d_stencil, sizeof(MarkerStencil) * m, cudaMemcpyDeviceToHost,
                       s->stream));
    CU(cudaMemcpyAsync(bx.data(), s->d_boxes, sizeof(MarkerBox) * m, cudaMemcpyDeviceToHost, s->stream));
  }
  CU(cudaStreamSynchronize(s->stream));
  for (size_t i = 0; i < m; ++i)
    for (int a = 0; a < 3; ++a) {
      lo_hi[6 * i + a] = st[i].valid ? st[i].lo[a] : 0;
      lo_hi[6 * i + 3 + a] = st[i].valid ? st[i].hi[a] : -1;
    }
  return FSG_OK;
}

// ------------------------------------------------------- output snapshots --
int fsg_snapshot_begin(fsg_session* s) {
  if (!s->last_valid) return set_err(FSG_ESTATE, "no coupled step since the last state change");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  if (!s->d_snap) {
    CU(cudaMalloc(&s->d_snap, sizeof(double) * 4 * n));
    CU(cudaMallocHost(&s->h_snap, sizeof(double) * 4 * n));
    CU(cudaEventCreateWithFlags(&s->ev_snap, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&s->ev_snap_k, cudaEventDisableTiming));
  }
  if (s->snap_pending) CU(cudaEventSynchronize(s->ev_snap));  // one snapshot in flight
  // bare moments of the state the last step read (macro(), session.hpp:95-96),
  // in stream order, into the snapshot's own buffer; the copy to pinned host
  // memory runs on the copy stream while later steps proceed
  s->L->macroscopic(s->g, s->buf[s->last_par], s->prev_pulled, nullptr, s->d_snap, s->d_snap + n,
                    s->d_diag, s->stream);
  CU_LAUNCH();
  CU(cudaEventRecord(s->ev_snap_k, s->stream));
  CU(cudaStreamWaitEvent(s->cstream, s->ev_snap_k, 0));
  CU(cudaMemcpyAsync(s->h_snap, s->d_snap, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, s->cstream));
  CU(cudaEventRecord(s->ev_snap, s->cstream));
  s->snap_pending = true;
  return FSG_OK;
}

int fsg_snapshot_wait(fsg_session* s, double* rho, double* u) {
  if (!s->snap_pending && !s->h_snap) return set_err(FSG_ESTATE, "no snapshot taken (fsg_snapshot_begin)");
  CU(cudaSetDevice(s->cfg.device));
  if (s->snap_pending) CU(cudaEventSynchronize(s->ev_snap));
  s->snap_pending = false;
  const size_t n = (size_t)s->g.n;
  if (rho) std::memcpy(rho, s->h_snap, sizeof(double) * n);
  if (u) std::memcpy(u, s->h_snap + n, sizeof(double) * 3 * n);
  return FSG_OK;
}

int fsg_write_vtk(fsg_session* s, const char* path, const double origin[3]) {
  if (!path || !origin) return set_err(FSG_EINPUT, "fsg_write_vtk: null path or origin");
  const size_t n = (size_t)s->g.n;
  if (s->g.zpad) return set_err(FSG_EINPUT, "fsg_write_vtk: z-slab sessions dump per slab (not supported)");
  std::vector<double> rho(n), u(3 * n);
  int rc = fsg_snapshot_wait(s, rho.data(), u.data());
  if (rc) return rc;
  rc = fsg_write_vtk_fields(path, s->cfg.dims, rho.data(), u.data(), s->cfg.dx, s->cfg.dt, s->cfg.rho,
                            origin);
  if (rc) return set_err(rc, "%s", fsg_io_last_error());
  return FSG_OK;
}

int fsg_get_macro(fsg_session* s, double* rho, double* u) {
  if (!s->last_valid) return set_err(FSG_ESTATE, "no coupled step since the last state change");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 4 * n);
  if (rc) return rc;
  CU(cudaStreamSynchronize(s->stream));
  StepScratch* junk = s->d_diag;  // nonpos count not needed here
  s->L->macroscopic(s->g, s->buf[s->last_par], s->prev_pulled, nullptr, s->d_tmp, s->d_tmp + n,
                    junk, s->stream);
  CU_LAUNCH();
  if (rho) CU(cudaMemcpyAsync(rho, s->d_tmp, sizeof(double) * n, cudaMemcpyDeviceToHost, s->stream));
  if (u) CU(cudaMemcpyAsync(u, s->d_tmp + n, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

int fsg_set_force_capture(fsg_session* s, int on) {
  if (!s) return set_err(FSG_EINPUT, "null session");
  CU(cudaSetDevice(s->cfg.device));
  if (on && !s->d_fcap) CU(cudaMalloc(&s->d_fcap, sizeof(float) * 3 * (size_t)s->g.n));
  s->fcap_on = on != 0;
  return FSG_OK;
}

int fsg_get_force(fsg_session* s, double* F) {
  if (!s->last_valid) return set_err(FSG_ESTATE, "no coupled step since the last state change");
  CU(cudaSetDevice(s->cfg.device));
  const size_t n = (size_t)s->g.n;
  int rc = ensure_tmp(s, sizeof(double) * 3 * n);
  if (rc) return rc;
  StepScratch* bscr = s->d_scr[s->last_par];
  if (s->last_fcap) {
    // the field the throughput K4 itself consumed (fixed-point IB band
    // decoded + virtual force), captured as it collided each cell
    std::vector<float> f(3 * n);
    CU(cudaMemcpyAsync(f.data(), s->d_fcap, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost,
                       s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (size_t i = 0; i < 3 * n; ++i) F[i] = (double)f[i];
    return FSG_OK;
  }
  if (s->L->markers_fix) {
    // Throughput path: K4 consumed (and re-zeroed) the fixed-point band, so
    // this diagnostic rebuilds the IB field from the stored stencil records
    // with the ordered spread kernel (agrees with the fixed-point sum to
    // ~1e-12 relative) and restores the step's frame constants.
    const size_t m = (size_t)s->m;
    std::vector<MarkerStencil> st(m);
    std::vector<MarkerBox> bx(m);
    if (m)
      CU(cudaMemcpy(st.data(), s->d_stencil, sizeof(MarkerStencil) * m, cudaMemcpyDeviceToHost));
    StepScratch sc{};
    int lo[3] = {1 << 29, 1 << 29, 1 << 29}, hi[3] = {-1, -1, -1};
    for (size_t i = 0; i < m; ++i) {
      bx[i] = MarkerBox{};
      bx[i].valid = (short)st[i].valid;
      for (int a = 0; a < 3; ++a) {
        const int off = a == 2 ? s->g.z0 : 0;
        bx[i].lo[a] = (short)(st[i].lo[a] - off);
        bx[i].hi[a] = (short)(st[i].hi[a] - off);
        if (st[i].valid) {
          lo[a] = std::min(lo[a], st[i].lo[a] - off);
          hi[a] = std::max(hi[a], st[i].hi[a] - off);
        }
      }
    }
    for (int a = 0; a < 3; ++a) {
      sc.bbox_lo_enc[a] = hi[a] >= 0 ? fsg::LO_BIAS - lo[a] : 0;
      sc.bbox_hi_enc[a] = hi[a] >= 0 ? hi[a] + 1 : 0;
    }
    if (m) CU(cudaMemcpy(s->d_boxes, bx.data(), sizeof(MarkerBox) * m, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(s->d_diag, &sc, sizeof sc, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(s->d_st, &s->last_st, sizeof(StepConsts), cudaMemcpyHostToDevice));
    s->L->spread(s->g, s->m, s->d_stencil, s->d_boxes, s->band, s->d_diag, s->stream);
    bscr = s->d_diag;
  }
  s->L->session_force(s->g, s->buf[s->last_par], s->prev_pulled, &s->band, bscr,
                      s->d_sc, s->d_st, s->last_frame_on ? 1 : 0, s->d_tmp, s->stream);
  CU_LAUNCH();
  CU(cudaMemcpyAsync(F, s->d_tmp, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, s->stream));
  CU(cudaStreamSynchronize(s->stream));
  return FSG_OK;
}

// --------------------------------------------------------- measurement --
int fsg_profile_enable(fsg_session* s, int enable) {
  CU(cudaSetDevice(s->cfg.device));
  if (enable && s->prof_ev.empty()) {
    s->prof_ev.resize(2 * (size_t)fsg_session::PROF_CAP);
    for (auto& e : s->prof_ev) CU(cudaEventCreate(&e));
  }
  s->prof = enable != 0;
  s->prof_n = 0;
  return FSG_OK;
}

int fsg_profile_read(fsg_session* s, double* step_ms, int* steps) {
  CU(cudaStreamSynchronize(s->stream));
  double a = 0.0;
  for (int k = 0; k < s->prof_n; ++k) {
    float t = 0.f;
    const cudaEvent_t* e = &s->prof_ev[2 * (size_t)k];
    CU(cudaEventElapsedTime(&t, e[0], e[1]));
    a += t;
  }
  if (step_ms) *step_ms = a;
  if (steps) *steps = s->prof_n;
  s->prof_n = 0;
  return FSG_OK;
}

// --------------------------------------------------------------- halos --
size_t fsg_halo_bytes(fsg_session* s) { return (size_t)5 * s->g.plane * s->L->elem_bytes; }

int fsg_halo_pack(fsg_session* s, void* lo, void* hi) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  CU(cudaSetDevice(s->cfg.device));
  s->L->halo_pack(s->g, s->A(), lo, hi, s->stream);
  CU_LAUNCH();
  return FSG_OK;
}

int fsg_halo_unpack(fsg_session* s, const void* lo, const void* hi) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  CU(cudaSetDevice(s->cfg.device));
  s->L->halo_unpack(s->g, s->A(), lo, hi, s->stream);
  CU_LAUNCH();
  return FSG_OK;
}

int fsg_halo_buffers(fsg_session* s, void** send_lo, void** send_hi, void** recv_lo,
                     void** recv_hi) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  if (send_lo) *send_lo = s->d_hsend[0];
  if (send_hi) *send_hi = s->d_hsend[1];
  if (recv_lo) *recv_lo = s->d_hrecv[0];
  if (recv_hi) *recv_hi = s->d_hrecv[1];
  return FSG_OK;
}

int fsg_halo_begin(fsg_session* s, void* comm_stream) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  CU(cudaSetDevice(s->cfg.device));
  CU(cudaStreamWaitEvent((cudaStream_t)comm_stream, s->ev_hpack, 0));
  return FSG_OK;
}

int fsg_halo_end(fsg_session* s, void* comm_stream, int have_lo, int have_hi) {
  if (!s->g.zpad) return set_err(FSG_EINPUT, "not a z-slab session");
  CU(cudaSetDevice(s->cfg.device));
  CU(cudaEventRecord(s->ev_hrecv, (cudaStream_t)comm_stream));
  CU(cudaStreamWaitEvent(s->stream, s->ev_hrecv, 0));
  if (have_lo || have_hi) {
    s->L->halo_unpack(s->g, s->A(), have_lo ? s->d_hrecv[0] : nullptr,
                      have_hi ? s->d_hrecv[1] : nullptr, s->stream);
    CU_LAUNCH();
  }
  return FSG_OK;
}


// ------------------------------------------------------ peer transport --
// z-slab halo exchange inside the library: the boundary
// planes' collision kernel stores the 5 crossing populations of each face
// straight into the neighbour's halo plane (NVLink peer memory, CUDA IPC
// across processes), ordered by stream memory operations on 32-bit delivery
// counters -- no pack/unpack kernels, no host exchange, no NCCL on the data
// path.  Protocol (every rank runs the same step sequence, so the A/B parity
// of all slabs agrees): before the boundary planes of step n (n = 1, 2, ...
// since connecting) a session waits until each neighbour's counter slot is
// >= n, i.e. that neighbour finished its boundary planes of step n-1 (their
// crossing populations are in this session's halo, and it has finished
// reading the halo this step overwrites in its buffer); after them it writes
// n + 1 into the neighbours' slots (the write is fenced after the kernel's
// stores).  fsg_peer_connect delivers the current state's boundary planes
// once (counter 1).
namespace {
struct PeerExport {
  unsigned magic, version;
  int pid, device;
  int nx, ny, nz, z0, nzg, zpad, elem, par, periodic, pad_;
  unsigned long long raw_buf[2], raw_flags;
  cudaIpcMemHandle_t h_buf[2], h_flags;
};
constexpr unsigned kPeerMagic = 0x46534750u;  // "FSGP"
static_assert(sizeof(PeerExport) <= FSG_PEER_HANDLE_BYTES, "peer handle too small");

using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_write32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_wait32 g_wait32 = nullptr;
PFN_write32 g_write32 = nullptr;
unsigned g_wait_flags = CU_STREAM_WAIT_VALUE_GEQ;

int load_stream_memops(int device) {
  if (g_wait32 && g_write32) return FSG_OK;
  cudaDriverEntryPointQueryResult q1, q2;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&g_wait32, cudaEnableDefault, &q1) !=
          cudaSuccess ||
      cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&g_write32, cudaEnableDefault, &q2) !=
          cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !g_wait32 ||
      !g_write32) {
    g_wait32 = nullptr;
    g_write32 = nullptr;
    return set_err(FSG_ECUDA, "peer transport: stream memory operations unavailable");
  }
  int flush = 0;
  if (cudaDeviceGetAttribute(&flush, (cudaDeviceAttr)CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES,
                             device) == cudaSuccess &&
      flush)
    g_wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
  return FSG_OK;
}
}  // namespace

static int peer_wait(fsg_session* s, unsigned* flag, unsigned v) {
  if (g_wait32((CUstream)s->stream, (CUdeviceptr)flag, v, g_wait_flags) != CUDA_SUCCESS)
    return set_err(FSG_ECUDA, "cuStreamWaitValue32 failed");
  return FSG_OK;
}

static int peer_signal(fsg_session* s, unsigned* flag, unsigned v) {
  if (g_write32((CUstream)s->stream, (CUdeviceptr)flag, v, CU_STREAM_WRITE_VALUE_DEFAULT) !=
      CUDA_SUCCESS)
    return set_err(FSG_ECUDA, "cuStreamWriteValue32 failed");
  return FSG_OK;
}

int fsg_peer_export(fsg_session* s, fsg_peer_handle* out) {
  if (!s || !out) return set_err(FSG_EINPUT, "null argument");
  if (!s->g.zpad) return set_err(FSG_EINPUT, "fsg_peer_export: not a z-slab session");
  if (!s->L->markers_fix) return set_err(FSG_EINPUT, "fsg_peer_export: the peer transport runs fp32 (throughput) sessions");
  if (s->peer_on) return set_err(FSG_ESTATE, "fsg_peer_export: session already connected");
  CU(cudaSetDevice(s->cfg.device));
  int rc = load_stream_memops(s->cfg.device);
  if (rc) return rc;
  if (!s->d_peer_flags) CU(cudaMalloc(&s->d_peer_flags, 2 * sizeof(unsigned)));
  CU(cudaStreamSynchronize(s->stream));
  CU(cudaMemset(s->d_peer_flags, 0, 2 * sizeof(unsigned)));
  CU(cudaDeviceSynchronize());
  PeerExport e{};
  e.magic = kPeerMagic;
  e.version = 1;
  e.pid = (int)getpid();
  e.device = s->cfg.device;
  e.nx = s->g.nx;
  e.ny = s->g.ny;
  e.nz = s->g.nz;
  e.z0 = s->g.z0;
  e.nzg = s->g.nzg;
  e.zpad = s->g.zpad;
  e.elem = s->L->elem_bytes;
  e.par = s->par;
  e.periodic = s->g.periodic;
  for (int k = 0; k < 2; ++k) {
    e.raw_buf[k] = (unsigned long long)(uintptr_t)s->buf[k];
    CU(cudaIpcGetMemHandle(&e.h_buf[k], s->buf[k]));
  }
  e.raw_flags = (unsigned long long)(uintptr_t)s->d_peer_flags;
  CU(cudaIpcGetMemHandle(&e.h_flags, s->d_peer_flags));
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->bytes, &e, sizeof e);
  return FSG_OK;
}

static int peer_open(fsg_session* s, const fsg_peer_handle* h, int side) {
  PeerExport e;
  std::memcpy(&e, h->bytes, sizeof e);
  if (e.magic != kPeerMagic || e.version != 1)
    return set_err(FSG_EINPUT, "fsg_peer_connect: not a peer handle");
  if (e.nx != s->g.nx || e.ny != s->g.ny || e.nzg != s->g.nzg || e.zpad != s->g.zpad ||
      e.elem != s->L->elem_bytes || e.periodic != s->g.periodic)
    return set_err(FSG_EINPUT, "fsg_peer_connect: neighbour slab of another grid");
  if (e.par != s->par)
    return set_err(FSG_ESTATE, "fsg_peer_connect: neighbour at another step parity");
  // geometry: the lower neighbour ends where this slab starts, the upper
  // starts where it ends (global z, periodic wrap)
  const int nzg = s->g.nzg;
  const bool adj = side == 0 ? (e.z0 + e.nz) % nzg == s->g.z0 % nzg
                             : e.z0 % nzg == (s->g.z0 + s->g.nz) % nzg;
  if (!adj) return set_err(FSG_EINPUT, "fsg_peer_connect: %s handle is not the adjacent slab",
                           side == 0 ? "lower" : "upper");
  auto& L = s->nbr[side];
  L.nz = e.nz;
  if (e.pid == (int)getpid()) {  // same process: the pointers themselves
    if (e.device != s->cfg.device) {
      const cudaError_t pe = cudaDeviceEnablePeerAccess(e.device, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
        return set_err(FSG_ECUDA, "cudaDeviceEnablePeerAccess failed: %s", cudaGetErrorString(pe));
      cudaGetLastError();
    }
    L.buf[0] = (void*)(uintptr_t)e.raw_buf[0];
    L.buf[1] = (void*)(uintptr_t)e.raw_buf[1];
    L.flags = (unsigned*)(uintptr_t)e.raw_flags;
    L.ipc = false;
  } else {
    // the same neighbour may be both lower and upper (periodic, 2 slabs):
    // open its handles once (a process may open a handle only once)
    const auto& O = s->nbr[side ^ 1];
    if (O.on && O.ipc && s->nbr_pid_[side ^ 1] == e.pid) {
      for (int k = 0; k < 2; ++k) L.buf[k] = O.buf[k];
      L.flags = O.flags;
      L.owner = false;
    } else {
      for (int k = 0; k < 2; ++k)
        CU(cudaIpcOpenMemHandle(&L.buf[k], e.h_buf[k], cudaIpcMemLazyEnablePeerAccess));
      void* f = nullptr;
      CU(cudaIpcOpenMemHandle(&f, e.h_flags, cudaIpcMemLazyEnablePeerAccess));
      L.flags = (unsigned*)f;
      L.owner = true;
    }
    L.ipc = true;
  }
  s->nbr_pid_[side] = e.pid;
  L.on = true;
  return FSG_OK;
}

int fsg_peer_connect(fsg_session* s, const fsg_peer_handle* lower, const fsg_peer_handle* upper) {
  if (!s) return set_err(FSG_EINPUT, "null session");
  if (!s->g.zpad) return set_err(FSG_EINPUT, "fsg_peer_connect: not a z-slab session");
  if (!s->d_peer_flags) return set_err(FSG_ESTATE, "fsg_peer_connect: call fsg_peer_export first");
  if (s->peer_on) return set_err(FSG_ESTATE, "fsg_peer_connect: already connected");
  if (!lower && !upper) return set_err(FSG_EINPUT, "fsg_peer_connect: no neighbour");
  CU(cudaSetDevice(s->cfg.device));
  int rc = FSG_OK;
  if (lower && (rc = peer_open(s, lower, 0))) return rc;
  if (upper && (rc = peer_open(s, upper, 1))) {
    fsg_peer_disconnect(s);
    return rc;
  }
  // a pulled state needs the neighbours' boundary planes in its halo: deliver
  // this session's crossing planes of the current state once (counter 1)
  const size_t eb = (size_t)s->L->elem_bytes, pb = eb * (size_t)s->g.plane;
  const char* A = (const char*)s->buf[s->par];
  static const int dn[5] = {6, 12, 13, 16, 17}, up[5] = {5, 11, 14, 15, 18};
  if (s->pulled) {
    for (int k = 0; k < 5; ++k) {
      if (s->nbr[0].on) {  // plane 0 -> lower's top halo plane
        char* d = (char*)s->nbr[0].buf[s->par] +
                  eb * (size_t)(s->g.zs * (s->nbr[0].nz + s->g.zpad) + dn[k] * s->g.stride);
        CU(cudaMemcpyAsync(d, A + eb * (size_t)(s->g.zs * s->g.zpad + dn[k] * s->g.stride), pb,
                           cudaMemcpyDefault, s->stream));
      }
      if (s->nbr[1].on) {  // plane nz-1 -> upper's bottom halo plane
        char* d = (char*)s->nbr[1].buf[s->par] + eb * (size_t)(up[k] * s->g.stride);
        CU(cudaMemcpyAsync(
            d, A + eb * (size_t)(s->g.zs * (s->g.nz - 1 + s->g.zpad) + up[k] * s->g.stride), pb,
            cudaMemcpyDefault, s->stream));
      }
    }
  }
  if (s->nbr[0].on && (rc = peer_signal(s, s->nbr[0].flags + 1, 1))) return rc;
  if (s->nbr[1].on && (rc = peer_signal(s, s->nbr[1].flags + 0, 1))) return rc;
  s->peer_step = 0;
  s->peer_on = true;
  return FSG_OK;
}

int fsg_peer_disconnect(fsg_session* s) {
  if (!s) return FSG_OK;
  if (!s->nbr[0].on && !s->nbr[1].on) return FSG_OK;
  cudaSetDevice(s->cfg.device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (int side = 0; side < 2; ++side) {
    auto& L = s->nbr[side];
    if (L.on && L.ipc && L.owner) {
      cudaIpcCloseMemHandle(L.buf[0]);
      cudaIpcCloseMemHandle(L.buf[1]);
      cudaIpcCloseMemHandle(L.flags);
    }
    L = fsg_session::PeerLink{};
  }
  s->peer_on = false;
  return FSG_OK;
}

// ---------------------------------------------------------------- batch --
// E env sessions of one configuration sharing one stream, stepped together
// by ONE marker launch and ONE banded K4 launch (fsg_batch.cuh; SURVEY.md
// §8(e): the batched-RL config, 8 envs per GPU).  Env e is an ordinary
// fsg_session (fsg_batch_session): frames, markers and every readback use
// the per-session calls.
struct fsg_batch {
  int E = 0;
  cudaStream_t stream = nullptr;
  std::vector<fsg_session*> envs;
  fsg::EnvPack* h_packs[2] = {nullptr, nullptr};  // pinned, by batch step parity
  fsg::EnvPack* d_packs[2] = {nullptr, nullptr};
  unsigned* d_work = nullptr;                      // [2] phase-A counters by parity
  StepScratch* h_stat = nullptr;                   // pinned: every env's status (one-call step)
  fsg::SkinBody* h_skb[2] = {nullptr, nullptr};    // pinned: skinned envs' topology + pose
  fsg::SkinBody* d_skb[2] = {nullptr, nullptr};
  bool skb_up[2] = {false, false};                 // d_skb[q] topology current (device-pose steps)
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int par = 0;
  dim3 block;
  fsg_dyn* dyn = nullptr;                          // set during fsg_batch_step_dynamic
  // the robot loop on the device (fsg_batch_step_dynamic): tau_ext + stats of
  // every env stay in device memory for the robot step; one copy comes back
  static constexpr int WSTRIDE = 6 + FSG_SKIN_MAX_LINKS + fsg::SKIN_NSTAT;
  double* d_wrench = nullptr;                      // [E][WSTRIDE]
  double* h_wbatch = nullptr;                      // pinned copy
  const double** d_tauptr = nullptr;               // [E] -> d_wrench rows
  fsg_joint_state* h_states = nullptr;             // pinned: post-step robot states
  int* h_flags = nullptr;
  // frame following + recentring inside the loop (session.hpp:177-195)
  int follow = 0;
  double follow_thresh = 2.0;
  std::vector<fsg_follower*> fol;
  double* d_com = nullptr;                         // [3E] com_world of the post-step states
  double* h_com = nullptr;
  std::vector<int> shifts;                         // [3E] last call's recentre shifts
};

int fsg_batch_destroy(fsg_batch* b) {
  if (!b) return FSG_OK;
  if (b->stream) cudaStreamSynchronize(b->stream);
  for (auto* s : b->envs) fsg_destroy(s);
  for (int k = 0; k < 2; ++k) {
    if (b->h_packs[k]) cudaFreeHost(b->h_packs[k]);
    cudaFree(b->d_packs[k]);
    if (b->h_skb[k]) cudaFreeHost(b->h_skb[k]);
    cudaFree(b->d_skb[k]);
    if (b->ev[k]) cudaEventDestroy(b->ev[k]);
  }
  cudaFree(b->d_tauptr);
  cudaFree(b->d_wrench);
  cudaFree(b->d_com);
  if (b->h_wbatch) cudaFreeHost(b->h_wbatch);
  if (b->h_states) cudaFreeHost(b->h_states);
  if (b->h_flags) cudaFreeHost(b->h_flags);
  if (b->h_com) cudaFreeHost(b->h_com);
  for (auto* f : b->fol) fsg_follower_destroy(f);
  cudaFree(b->d_work);
  if (b->h_stat) cudaFreeHost(b->h_stat);
  if (b->stream) cudaStreamDestroy(b->stream);
  delete b;
  return FSG_OK;
}

int fsg_batch_create(const fsg_config* cfg, int n_envs, fsg_batch** out) {
  if (!cfg || !out) return set_err(FSG_EINPUT, "fsg_batch_create: null argument");
  *out = nullptr;
  if (n_envs < 1 || n_envs > fsg::BATCH_MAX)
    return set_err(FSG_EINPUT, "a batch holds 1..%d envs (got %d)", fsg::BATCH_MAX, n_envs);
  if (cfg->precision != FSG_PRECISION_FP32)
    return set_err(FSG_EINPUT, "batches run the throughput (fp32) step");
  if (cfg->z_offset != 0 || (cfg->nz_global > 0 && cfg->nz_global != cfg->dims[2]))
    return set_err(FSG_EINPUT, "batch envs are whole grids, not z-slabs");
  CU(cudaSetDevice(cfg->device));
  fsg_batch* b = new fsg_batch();
  b->E = n_envs;
  auto fail = [&](int code) {
    g_shared_stream = nullptr;
    fsg_batch_destroy(b);
    return code;
  };
#define CUB(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(set_err(FSG_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_))); \
  } while (0)
  CUB(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  g_shared_stream = b->stream;
  for (int e = 0; e < n_envs; ++e) {
    fsg_session* s = nullptr;
    const int rc = fsg_create(cfg, &s);
    if (rc) return fail(rc);
    b->envs.push_back(s);
  }
  g_shared_stream = nullptr;
  for (int k = 0; k < 2; ++k) {
    CUB(cudaMallocHost(&b->h_packs[k], sizeof(fsg::EnvPack) * n_envs));
    CUB(cudaMalloc(&b->d_packs[k], sizeof(fsg::EnvPack) * n_envs));
    CUB(cudaMallocHost(&b->h_skb[k], sizeof(fsg::SkinBody) * n_envs));
    CUB(cudaMalloc(&b->d_skb[k], sizeof(fsg::SkinBody) * n_envs));
    CUB(cudaEventCreateWithFlags(&b->ev[k], cudaEventDisableTiming));
    CUB(cudaEventRecord(b->ev[k], b->stream));
  }
  CUB(cudaMalloc(&b->d_work, sizeof(unsigned) * 2));
  CUB(cudaMemsetAsync(b->d_work, 0, sizeof(unsigned) * 2, b->stream));
  b->block = fsg::cell_block_dims(b->envs[0]->g);
#undef CUB
  *out = b;
  return FSG_OK;
}

fsg_session* fsg_batch_session(fsg_batch* b, int e) {
  return (b && e >= 0 && e < b->E) ? b->envs[e] : nullptr;
}

int fsg_batch_step_async(fsg_batch* b) {
  CU(cudaSetDevice(b->envs[0]->cfg.device));
  const int q = b->par;
  CU(cudaEventSynchronize(b->ev[q]));  // pinned packs of parity q are free again
  fsg::EnvPack* packs = b->h_packs[q];
  const fsg::Grid& g0 = b->envs[0]->g;
  const fsg::FixBand& fb0 = b->envs[0]->fix;
  fsg::BatchHead h{b->E, 0, 0, 0, fb0.tnx, fb0.tny, fb0.tnz, 1,
                   b->envs[0]->cfg.frame_mode != FSG_FRAME_NONE ? 1 : 0, 0, 0};
  int npulled = 0, nskin = 0;
  bool skb_dirty = !b->dyn;  // robot loop: the pose is made on the device, the topology rarely changes
  const int tx_n = (g0.nx + (int)b->block.x - 1) / (int)b->block.x;
  const int ty_n = (g0.ny + (int)b->block.y - 1) / (int)b->block.y;
  // phase-A items: the deepest of 4 / 2 / 1 planes (one tile layer, so one
  // stamp load per item) that still leaves >= 3 items per resident block
  // (c5, 8 envs of 96x48x48: 4 planes, round 165 -> 157 us; the per-item
  // fetch, barrier pair and status reduction were a third of phase A)
  const long long per_env4 = (long long)tx_n * ty_n * ((g0.nz + 3) / 4);
  const long long per_env2 = (long long)tx_n * ty_n * ((g0.nz + 1) / 2);
  static const int zc_env = [] {  // dev A/B: phase-A item depth of the batch
    const char* e = getenv("FSG_BATCH_ZC");
    return e ? atoi(e) : 0;
  }();
  const int zc = zc_env > 0 ? zc_env
                            : (per_env4 * b->E >= 3ll * 148 * 6 ? 4
                                                                 : (per_env2 * b->E >= 3ll * 148 * 6 ? 2 : 1));
  h.zc = zc;
  for (int e = 0; e < b->E; ++e) {
    fsg_session* s = b->envs[e];
    const int p = s->par;
    frame_consts(s->frame, *s->h_st[p]);
    const StepConsts st = *s->h_st[p];
    s->last_st = st;
    if (s->mk_host && s->mk_dirty) CU(cudaStreamWaitEvent(b->stream, s->ev_cp[s->mk_slot], 0));
    if (s->scr_dirty[p]) CU(cudaMemsetAsync(s->d_scr[p], 0, sizeof(StepScratch), b->stream));
    fsg::EnvPack& P = packs[e];
    P.st = st;
    P.A = (const float*)s->buf[p];
    P.B = (float*)s->buf[p ^ 1];
    P.F = s->fix.F;
    P.tflag = s->fix.tflag;
    P.stamp = ++s->stamp;  // fresh: with no markers no tile carries it
    P.mk = s->mk;
    P.rec = s->d_stencil;
    P.fworld = s->d_fworld;
    P.fworld_h = s->h_fw[p];
    P.valid_h = s->h_valid[p];
    P.out = s->d_scr[p];
    P.next = s->d_scr[p ^ 1];
    P.pulled = s->pulled;
    P.frame_on = s->cfg.frame_mode != FSG_FRAME_NONE;
    P.skb = nullptr;
    if (s->skin && s->m) {  // skinned env: its topology + pose go up with the packs
      if (s->skp.nb != 1)
        return set_err(FSG_EINPUT, "batched envs: one skinned body per env (env %d has %d)", e, s->skp.nb);
      if (!s->pose_set) return set_err(FSG_ESTATE, "env %d: fsg_set_pose has not been called", e);
      if (b->dyn && !skb_dirty &&
          std::memcmp(&b->h_skb[q][e], &s->skp.body[0], offsetof(fsg::SkinBody, pose)) != 0)
        skb_dirty = true;
      b->h_skb[q][e] = s->skp.body[0];
      P.skb = b->d_skb[q] + e;
      P.sk_rest = s->skp.rest;
      P.sk_nrest = s->skp.nrest;
      P.sk_wb = s->skp.wb;
      P.sk_ww = s->skp.ww;
      P.sk_acc = s->d_skin_fix;
      // robot loop on the device: tau_ext stays in HBM for the robot step
      P.sk_out = (b->dyn && b->d_wrench) ? b->d_wrench + (size_t)e * fsg_batch::WSTRIDE : s->h_wrench[p];
      P.sk_ndof = s->skp.body[0].n_dofs;
      ++nskin;
    }
    P.mk_begin = h.m_total;
    P.item_begin = h.item_total;
    P.tile_begin = h.tile_total;
    h.m_total += s->m;  // (device or host markers; host ones were uploaded on the copy stream)
    npulled += s->pulled ? 1 : 0;
    h.item_total += tx_n * ty_n * ((s->g.nz + zc - 1) / zc);
    h.tile_total += s->fix.tnx * s->fix.tny * s->fix.tnz;
  }
  h.pmode = npulled == b->E ? 1 : (npulled == 0 ? 0 : 2);
  h.skin = nskin > 0 ? 1 : 0;
  CU(cudaMemcpyAsync(b->d_packs[q], packs, sizeof(fsg::EnvPack) * b->E, cudaMemcpyHostToDevice,
                     b->stream));
  if (nskin && (skb_dirty || !b->skb_up[q])) {
    CU(cudaMemcpyAsync(b->d_skb[q], b->h_skb[q], sizeof(fsg::SkinBody) * b->E, cudaMemcpyHostToDevice,
                       b->stream));
    b->skb_up[q] = b->dyn != nullptr;  // valid topology for the next device-pose step of parity q
  }
  if (b->dyn) {  // this step's poses from the robot states, written over the uploaded ones
    const int rc = fsg::dyn_launch_pose(b->dyn,
                                        reinterpret_cast<char*>(b->d_skb[q]) + offsetof(fsg::SkinBody, pose),
                                        sizeof(fsg::SkinBody), b->stream);
    if (rc) return set_err(rc, "%s", fsg_dyn_last_error());
  }
  CU(cudaMemsetAsync(b->d_work + q, 0, sizeof(unsigned), b->stream));
  b->envs[0]->L->step_batch(g0, b->envs[0]->d_sc, b->d_packs[q], h, b->block, b->d_work + q,
                            b->stream);
  CU_LAUNCH();
  CU(cudaEventRecord(b->ev[q], b->stream));
  for (fsg_session* s : b->envs) {
    const int p = s->par;
    if (s->mk_host && s->mk_slot >= 0) {
      CU(cudaEventRecord(s->ev_mk[s->mk_slot], b->stream));
      s->last_mk_slot = s->mk_slot;
    }
    s->scr_dirty[p] = true;
    s->scr_dirty[p ^ 1] = false;
    s->status_pub[p] = false;  // batched steps: fsg_last_status copies
    s->last_par = p;
    s->prev_pulled = s->pulled;
    s->last_frame_on = s->cfg.frame_mode != FSG_FRAME_NONE;
    s->par ^= 1;
    s->pulled = 1;
    s->last_valid = true;
    s->stepped = true;
    s->mk_dirty = false;
  }
  b->par ^= 1;
  return FSG_OK;
}

namespace {
// every env's step status into pinned host memory in one launch (the batched
// K4 left each in its env's device scratch, packs[e].out)
// Launched as a programmatic dependent of the batched K4 (which triggers at
// its start) where it directly follows it: resident before K4 ends, it copies
// as soon as K4's writes are visible.  griddepcontrol.wait is a no-op in a
// normal launch.
__global__ void k_batch_status(const fsg::EnvPack* __restrict__ packs, int E, StepScratch* dst) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int NS = (int)(sizeof(StepScratch) / 4);
  for (int k = threadIdx.x; k < E * NS; k += blockDim.x)
    reinterpret_cast<volatile int*>(dst)[k] = reinterpret_cast<const int*>(packs[k / NS].out)[k % NS];
}
// The robots-on-device step's whole readback into pinned host memory in one
// launch: every env's status, tau_ext + stats, robot state and flag, and the
// robots' COM (null: no follower) -- instead of a status kernel and four
// device-to-host copies queued behind the robot step (each ~5-9 us of
// latency on a synchronous call).
__global__ void k_batch_readback(const fsg::EnvPack* __restrict__ packs, int E, StepScratch* hst,
                                 const double* __restrict__ wr, double* hwr, int nwr,
                                 const int* __restrict__ st, int* hst_state, int nst,
                                 const int* __restrict__ fl, int* hfl,
                                 const double* __restrict__ com, double* hcom) {
  constexpr int NS = (int)(sizeof(StepScratch) / 4);
  const int t = threadIdx.x;
  for (int k = t; k < E * NS; k += blockDim.x)
    reinterpret_cast<volatile int*>(hst)[k] = reinterpret_cast<const int*>(packs[k / NS].out)[k % NS];
  for (int k = t; k < nwr; k += blockDim.x) reinterpret_cast<volatile double*>(hwr)[k] = wr[k];
  for (int k = t; k < nst; k += blockDim.x) reinterpret_cast<volatile int*>(hst_state)[k] = st[k];
  for (int k = t; k < E; k += blockDim.x) reinterpret_cast<volatile int*>(hfl)[k] = fl[k];
  if (com)
    for (int k = t; k < 3 * E; k += blockDim.x) reinterpret_cast<volatile double*>(hcom)[k] = com[k];
}
}  // namespace

int fsg_batch_step_skinned(fsg_batch* b, const fsg_frame_state* frames, const fsg_body_pose* poses,
                           fsg_status* statuses, double* tau, double* stats) {
  CU(cudaSetDevice(b->envs[0]->cfg.device));
  for (int e = 0; e < b->E; ++e) {
    fsg_session* s = b->envs[e];
    if (!s->skin || s->skp.nb != 1)
      return set_err(FSG_ESTATE, "fsg_batch_step_skinned: env %d has no single skinned body", e);
    if (frames) s->frame = frames[e];
    s->skp.body[0].pose = poses[e];
    s->pose_set = true;
  }
  const int q = b->par;  // the packs this step uploads
  int rc = fsg_batch_step_async(b);
  if (rc) return rc;
  if (!b->h_stat) CU(cudaMallocHost(&b->h_stat, sizeof(StepScratch) * b->E));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(256);
    cfg.stream = b->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU(cudaLaunchKernelEx(&cfg, k_batch_status, (const fsg::EnvPack*)b->d_packs[q], b->E, b->h_stat));
  }
  CU_LAUNCH();
  CU(stream_wait(b->stream));
  int off = 0;
  for (int e = 0; e < b->E; ++e) {
    fsg_session* s = b->envs[e];
    if (b->h_stat[e].band_overflow) return set_err(FSG_ESTATE, "env %d: IB band overflow", e);
    decode_status(b->h_stat[e], &s->last, true);
    if (statuses) statuses[e] = s->last;
    const double* w = s->h_wrench[s->last_par];
    const int nd = s->skp.body[0].n_dofs;
    if (tau) std::memcpy(tau + off, w, sizeof(double) * nd);
    if (stats) std::memcpy(stats + fsg::SKIN_NSTAT * e, w + nd, sizeof(double) * fsg::SKIN_NSTAT);
    off += nd;
  }
  return FSG_OK;
}

// the device-resident robot loop's buffers (allocated at the first call)
static int batch_dyn_buffers(fsg_batch* b) {
  if (b->d_wrench) return FSG_OK;
  CU(cudaMalloc(&b->d_wrench, sizeof(double) * fsg_batch::WSTRIDE * b->E));
  CU(cudaMemsetAsync(b->d_wrench, 0, sizeof(double) * fsg_batch::WSTRIDE * b->E, b->stream));
  CU(cudaMallocHost(&b->h_wbatch, sizeof(double) * fsg_batch::WSTRIDE * b->E));
  CU(cudaMalloc(&b->d_tauptr, sizeof(double*) * b->E));
  std::vector<const double*> tp(b->E);
  for (int e = 0; e < b->E; ++e) tp[e] = b->d_wrench + (size_t)e * fsg_batch::WSTRIDE;
  CU(cudaMemcpyAsync(b->d_tauptr, tp.data(), sizeof(double*) * b->E, cudaMemcpyHostToDevice,
                     b->stream));
  CU(cudaMallocHost(&b->h_states, sizeof(fsg_joint_state) * b->E));
  CU(cudaMallocHost(&b->h_flags, sizeof(int) * b->E));
  CU(cudaMalloc(&b->d_com, sizeof(double) * 3 * b->E));
  CU(cudaMallocHost(&b->h_com, sizeof(double) * 3 * b->E));
  CU(stream_wait(b->stream));
  b->shifts.assign(3 * (size_t)b->E, 0);
  return FSG_OK;
}

int fsg_batch_set_follow(fsg_batch* b, double time_constant, double recenter_threshold_cells) {
  if (!b) return set_err(FSG_EINPUT, "fsg_batch_set_follow: NULL handle");
  for (auto* f : b->fol) fsg_follower_destroy(f);
  b->fol.clear();
  b->follow = 0;
  if (!(time_constant > 0.0)) return FSG_OK;
  const int mode = b->envs[0]->cfg.frame_mode;
  if (mode == FSG_FRAME_NONE)
    return set_err(FSG_EINPUT, "fsg_batch_set_follow: frame_mode NONE is the static domain (nothing to follow)");
  if (!(recenter_threshold_cells >= 0.0))
    return set_err(FSG_EINPUT, "fsg_batch_set_follow: negative recenter threshold");
  for (int e = 0; e < b->E; ++e) {
    fsg_follower* f = nullptr;
    if (fsg_follower_create(mode, time_constant, &f)) return set_err(FSG_EINPUT, "bad follow mode");
    b->fol.push_back(f);
    fsg_follower_state(f, &b->envs[e]->frame);
  }
  b->follow = 1;
  b->follow_thresh = recenter_threshold_cells;
  return FSG_OK;
}

int fsg_batch_center_frames(fsg_batch* b, fsg_dyn* d) {
  if (!b || !d) return set_err(FSG_EINPUT, "fsg_batch_center_frames: NULL handle");
  if (!b->follow) return set_err(FSG_ESTATE, "fsg_batch_center_frames: following is off");
  if (fsg::dyn_n_envs(d) != b->E)
    return set_err(FSG_EINPUT, "fsg_batch_center_frames: %d robots for %d envs", fsg::dyn_n_envs(d), b->E);
  std::vector<fsg_joint_state> st(b->E);
  if (fsg_dyn_get_state(d, st.data())) return set_err(FSG_ECUDA, "%s", fsg_dyn_last_error());
  for (int e = 0; e < b->E; ++e) {
    fsg_follower_center(b->fol[e], st[e].base_pos, st[e].base_quat);
    fsg_follower_state(b->fol[e], &b->envs[e]->frame);
  }
  return FSG_OK;
}

int fsg_batch_last_shifts(const fsg_batch* b, int* shifts) {
  if (!b || !shifts) return set_err(FSG_EINPUT, "fsg_batch_last_shifts: NULL argument");
  for (int k = 0; k < 3 * b->E; ++k) shifts[k] = b->shifts.empty() ? 0 : b->shifts[k];
  return FSG_OK;
}

int fsg_batch_step_dynamic(fsg_batch* b, fsg_dyn* d, const fsg_frame_state* frames,
                           const double* actuation, double rho_fluid, const double* g_hydro,
                           double dt, int substeps, fsg_status* statuses, int* flags,
                           fsg_joint_state* states) {
  if (!b || !d) return set_err(FSG_EINPUT, "fsg_batch_step_dynamic: NULL handle");
  if (fsg::dyn_n_envs(d) != b->E)
    return set_err(FSG_EINPUT, "fsg_batch_step_dynamic: %d robots for %d envs", fsg::dyn_n_envs(d), b->E);
  if (fsg::dyn_device(d) != b->envs[0]->cfg.device)
    return set_err(FSG_EINPUT, "fsg_batch_step_dynamic: robots and envs on different devices");
  if (!fsg::dyn_rest_set(d))
    return set_err(FSG_ESTATE, "fsg_batch_step_dynamic: fsg_dyn_set_rest has not been called");
  const fsg_config& c0 = b->envs[0]->cfg;
  if (dt != c0.dt || rho_fluid != c0.rho)
    return set_err(FSG_EINPUT, "fsg_batch_step_dynamic: dt %g / rho %g differ from the envs' %g / %g "
                               "(the robots integrate with the session's units, session.hpp:171-174)",
                   dt, rho_fluid, c0.dt, c0.rho);
  if (b->follow && frames)
    return set_err(FSG_EINPUT, "fsg_batch_step_dynamic: frames come from the followers (pass NULL)");
  // every check before any env is touched
  for (int e = 0; e < b->E; ++e) {
    fsg_session* s = b->envs[e];
    if (!s->skin || s->skp.nb != 1)
      return set_err(FSG_ESTATE, "fsg_batch_step_dynamic: env %d has no single skinned body", e);
    if (s->skp.body[0].n_dofs != fsg_dyn_n_dofs(d) || s->skp.body[0].n_links != fsg::dyn_n_links(d))
      return set_err(FSG_EINPUT, "fsg_batch_step_dynamic: env %d's skeleton is not the robot's", e);
  }
  CU(cudaSetDevice(c0.device));
  int rc = batch_dyn_buffers(b);
  if (rc) return rc;
  std::vector<char> had_pose(b->E);
  for (int e = 0; e < b->E; ++e) {
    fsg_session* s = b->envs[e];
    if (b->follow) fsg_follower_state(b->fol[e], &s->frame);
    else if (frames) s->frame = frames[e];
    had_pose[e] = s->pose_set;
    s->pose_set = true;  // this step's pose is produced on the device
  }
  auto restore_pose = [&] {  // the host pose was not updated: plain steps need fsg_set_pose again
    for (int e = 0; e < b->E; ++e) b->envs[e]->pose_set = false;
  };
  double* d_act = nullptr;
  rc = fsg::dyn_upload_actuation(d, actuation, b->stream, &d_act);
  if (rc) return restore_pose(), set_err(rc, "%s", fsg_dyn_last_error());
  const int q = b->par;
  b->dyn = d;
  rc = fsg_batch_step_async(b);
  b->dyn = nullptr;
  restore_pose();
  if (rc) return rc;
  // session.hpp:169-175: buoyancy on the pre-step kinematics + integrate
  // (gravity enters through the hydrostatics only); tau_ext from HBM
  rc = fsg::dyn_launch_step(d, d_act, nullptr, b->d_tauptr, rho_fluid, g_hydro, dt, substeps, nullptr,
                            fsg::dyn_flags(d), b->stream);
  if (rc) return set_err(rc, "%s", fsg_dyn_last_error());
  if (!b->h_stat) CU(cudaMallocHost(&b->h_stat, sizeof(StepScratch) * b->E));
  if (b->follow) {
    rc = fsg::dyn_launch_com(d, b->d_com, b->stream);
    if (rc) return set_err(rc, "%s", fsg_dyn_last_error());
  }
  static_assert(sizeof(fsg_joint_state) % sizeof(int) == 0, "copied as ints");
  k_batch_readback<<<1, 256, 0, b->stream>>>(
      b->d_packs[q], b->E, b->h_stat, b->d_wrench, b->h_wbatch, fsg_batch::WSTRIDE * b->E,
      reinterpret_cast<const int*>(fsg::dyn_states_dev(d)), reinterpret_cast<int*>(b->h_states),
      (int)(sizeof(fsg_joint_state) / sizeof(int)) * b->E, fsg::dyn_flags(d), b->h_flags,
      b->follow ? b->d_com : nullptr, b->h_com);
  CU_LAUNCH();
  CU(stream_wait(b->stream));
  for (int e = 0; e < b->E; ++e) {
    fsg_session* s = b->envs[e];
    if (b->h_stat[e].band_overflow) return set_err(FSG_ESTATE, "env %d: IB band overflow", e);
    decode_status(b->h_stat[e], &s->last, true);
    if (statuses) statuses[e] = s->last;
    // tau_ext + stats of the step for fsg_get_body_wrench
    std::memcpy(s->h_wrench[s->last_par], b->h_wbatch + (size_t)e * fsg_batch::WSTRIDE,
                sizeof(double) * fsg_batch::WSTRIDE);
  }
  if (states) std::memcpy(states, b->h_states, sizeof(fsg_joint_state) * b->E);
  if (flags) std::memcpy(flags, b->h_flags, sizeof(int) * b->E);
  if (b->follow) {
    // session.hpp:177-195: follower toward the new base pose, then the
    // integer-cell recentre when the robot's COM (frame coordinates) is more
    // than threshold cells from the centre on any axis
    for (int e = 0; e < b->E; ++e) {
      fsg_session* s = b->envs[e];
      const fsg_joint_state& st = b->h_states[e];
      fsg_follower_step(b->fol[e], st.base_pos, st.base_quat, dt);
      fsg_follower_state(b->fol[e], &s->frame);
      double R[9], d3[3], cf[3];
      quat_to_R(s->frame.q, R);
      for (int a = 0; a < 3; ++a) d3[a] = b->h_com[3 * e + a] - s->frame.p[a];
      mat_t_vec(R, d3, cf);  // world_to_frame_point (frame.hpp:24-26)
      int shift[3] = {0, 0, 0};
      bool need = false;
      for (int a = 0; a < 3; ++a) {
        const double cells = cf[a] / c0.dx;
        if (std::abs(cells) > b->follow_thresh) {
          shift[a] = (int)std::round(cells);
          need = true;
        }
      }
      for (int a = 0; a < 3; ++a) b->shifts[3 * e + a] = shift[a];
      if (need) {
        rc = recenter_async(s, shift);
        if (rc) return rc;
        s->stepped = true;  // the step's outputs (tau_ext, marker forces) stay readable
        fsg_follower_set_state(b->fol[e], &s->frame);  // the origin advanced by R shift dx
      }
    }
  }
  return FSG_OK;
}

int fsg_batch_step(fsg_batch* b, fsg_status* statuses) {
  int rc = fsg_batch_step_async(b);
  if (rc) return rc;
  for (int e = 0; e < b->E; ++e) {
    rc = fsg_last_status(b->envs[e], statuses ? &statuses[e] : nullptr);
    if (rc) return rc;
  }
  return FSG_OK;
}

}  // extern "C"
