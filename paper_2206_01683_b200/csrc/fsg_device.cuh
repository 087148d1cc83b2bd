// fsg_device.cuh -- shared device-side definitions for the FishGym IB-LBM
// hot path on B200 (sm_100a).  Included by the two precision translation
// units (fsg_kernels_fp32.cu, fsg_kernels_fp64.cu) and by the host session.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fsg.h"

// minimum resident 128-thread blocks per SM asked of ptxas for the
// throughput K4 and marker kernels (register caps: 65536 / (128 * MINB))
#ifndef FSG_K4_MINB
#define FSG_K4_MINB 6
#endif
// the banded (coupled) K4: 8 blocks (64 registers) -- measured c3 135.5 vs
// 141.7 us per coupled step at 6; the pure-fluid K4 stays at 6 (512^3: 3.74
// vs 4.28 ms at 8)
#ifndef FSG_K4B_MINB
#define FSG_K4B_MINB 8  // 64 registers (L2-resident grids)
#endif
#ifndef FSG_K4B_MINB_PAIR
#define FSG_K4B_MINB_PAIR 6  // 80 registers: room for the paired phase-A loads
#endif
#ifndef FSG_KM_PER_SM_DEFAULT
#define FSG_KM_PER_SM_DEFAULT 3.0  // persistent marker grid: c3 141.4 -> 139.8 us vs one wave
#endif
// batched marker kernel: register budget (min resident blocks) and grid cap
// per SM (it is persistent over every env's markers).  Both batched kernels
// at 64 registers: the 4 marker blocks per SM leave room for 4 K4 blocks, so
// phase A runs beside the markers instead of behind them (c5 round 148.1 ->
// 143.6 us; 80/80 registers with 5 marker blocks: 148.1; 64/64 with 3, 5, 6
// marker blocks: 154.8, 148.4, 150.9; K4 at 80: 145.0)
#ifndef FSG_K4BB_MINB  // batched banded K4: resident 128-thread blocks per SM
#define FSG_K4BB_MINB 8
#endif
#ifndef FSG_KMB_MINB
#define FSG_KMB_MINB 8
#endif
#ifndef FSG_KMB_PER_SM
#define FSG_KMB_PER_SM 4
#endif
#ifndef FSG_KM_MINB
#define FSG_KM_MINB 6
#endif


namespace fsg {

// ----------------------------------------------------- dev instrumentation --
// Built only with -DFSG_TIMING (make dbg -> libfsg_dbg.so): per-step phase
// timestamps (%globaltimer) in a ring indexed by the step stamp, read back by
// fsg_debug_timeline (scripts/probe_timeline.py).  Even slots take the min,
// odd slots the max.  Compiled out of the product library.
#ifdef FSG_TIMING
constexpr int TL_SLOTS = 8;
__device__ unsigned long long g_tl[64 * TL_SLOTS];  // only the fp32 TU is built with FSG_TIMING
// per banded-K4 block of the latest step: start, phase-A end, items, SM id
__device__ unsigned long long g_blk[8192 * 4];
__device__ __forceinline__ unsigned smid_() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// per marker warp (first marker of the warp): phase timestamps, 16 slots
__device__ unsigned long long g_mkt[4096 * 16];
#define FSG_MKT(first, slot)                                                               \
  do {                                                                                     \
    if ((first) && (threadIdx.x & 31) == 0) {                                              \
      const unsigned w_ = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);             \
      if (w_ < 4096) fsg::g_mkt[w_ * 16 + (slot)] = fsg::tl_now();                         \
    }                                                                                      \
  } while (0)
#define FSG_TL(stamp, slot) \
  ((slot) & 1 ? atomicMax(&fsg::g_tl[((stamp) & 63) * fsg::TL_SLOTS + (slot)], fsg::tl_now()) \
              : atomicMin(&fsg::g_tl[((stamp) & 63) * fsg::TL_SLOTS + (slot)], fsg::tl_now()))
#else
#define FSG_TL(stamp, slot) ((void)0)
#define FSG_MKT(first, slot) ((void)0)
#endif

// ----------------------------------------------------------------- D3Q19 --
// lattice.hpp:17-38 : 0 rest, 1-6 axes (+x,-x,+y,-y,+z,-z), 7-18 diagonals.
__host__ __device__ __forceinline__ constexpr int ex_of(int i) {
  constexpr int t[19] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
  return t[i];
}
__host__ __device__ __forceinline__ constexpr int ey_of(int i) {
  constexpr int t[19] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
  return t[i];
}
__host__ __device__ __forceinline__ constexpr int ez_of(int i) {
  constexpr int t[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
  return t[i];
}
__host__ __device__ __forceinline__ constexpr double w_of(int i) {
  return i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0);
}
constexpr int Q = 19;

// --------------------------------------------------------------- layout --
// Plane-interleaved SoA: for every z plane (the slab's owned planes plus
// `zpad` halo planes below and above, z-slab decomposition) the 19 direction
// planes are stored back to back.  Element (i, x, y, z_local) lives at
//   i*stride + x + nx*y + zs*(z_local + zpad),   stride = nx*ny, zs = 19*stride.
// Each direction plane is still one contiguous, coalesced run (the reference's
// direction-major order within a plane, lattice.hpp:89-90), and every pull
// source is still a constant offset from the cell's own slot; but one step
// touches 2 regions of memory near the current z (read A, write B) instead
// of 38 streams a whole direction array apart (measured +11-17 % on a
// K4-shaped stream at 1.3-20 GB, scripts/probe_layout.cu).
struct Grid {
  int nx, ny, nz;    // local (owned) dims
  int nzg, z0;       // global z extent, global z of local plane 0
  int zpad;          // halo planes per side (0 single GPU, 1 slab)
  int periodic;
  int _pad;
  long long n;       // owned cells nx*ny*nz
  long long plane;   // nx*ny
  long long stride;  // elements between direction planes of one z (= plane)
  long long zs;      // elements between z planes (= 19*plane)
  // per-direction element offsets relative to the cell's own slot (host-made,
  // land in the constant bank): own[i] = i*stride, pull[i] = i*stride - off_i
  // with off_i = ex + nx*(ey + ny*ez) (interior pull source)
  long long own[19];
  long long pull[19];
};

inline void grid_offsets(Grid& g) {
  for (int i = 0; i < 19; ++i) {
    g.own[i] = (long long)i * g.stride;
    g.pull[i] = g.own[i] - ((long long)ex_of(i) + (long long)g.nx * ey_of(i) + g.zs * ez_of(i));
  }
}

__host__ __device__ __forceinline__ long long mem_index(const Grid& g, int x, int y, int z) {
  return (long long)x + (long long)g.nx * (long long)y + g.zs * (long long)(z + g.zpad);
}

// ------------------------------------------------------ device constants --
// Per-session constants (host-computed in fp64 exactly as the reference).
struct SessionConsts {
  double omega;      // 1/tau                            solver.hpp:109
  double guo;        // 1 - omega/2                      solver.hpp:110
  double dx, dt, rho_phys;
  double v2p;        // dx/dt          vel_to_physical  units.hpp:31
  double acc;        // dt*dt/dx       session.hpp:149
  double f2l;        // dt^2/(rho dx^4) session.hpp:128
  double hd[3];      // 0.5*(d-1)      session.hpp:79-85 (global dims)
  int dims_g[3];     // global dims (marker_in_bounds)
  int kernel;        // 0 Peskin4, 1 Roma3
  int wall;          // 0 slip, 1 no-slip
  int frame_on;      // frame_mode != None
  // fp32 collision constants (throughput mode), rounded once on the host
  float om1_f;       // 1 - omega
  float ow_f[3];     // omega * w  for w in {1/3, 1/18, 1/36}
  float gw_f[3];     // guo * w
  float dx_f, v2p_f, acc_f, hd_f[3];
};

// Per-step frame constants (frame.hpp:21-53), host-computed in fp64.
struct StepConsts {
  double R[9];       // row-major rotation()
  double p[3], pd[3];
  double a0[3];      // R^T pdd
  double wf[3];      // R^T omega
  double af[3];      // R^T alpha
  float a0_f[3], wf_f[3], af_f[3];  // fp32 copies for the throughput kernels
  float _padf;
};

// Per-step scratch, reset to all-zero bytes before every step.  Encodings are
// chosen so that zero bytes == "empty": min via max of ~key, bbox lo via max
// of (LO_BIAS - lo), bbox hi via max of (hi + 1).
struct StepScratch {
  unsigned long long neg_min_key;  // ~ordered_key(min post), 0 == +inf
  int nonfinite;                   // 1 if any cell had non-finite rho+u2
  int nonpos;                      // count of rho <= 0 cells
  int oob;                         // out-of-bounds markers
  int band_overflow;               // bbox exceeded band capacity
  int bbox_lo_enc[3];
  int bbox_hi_enc[3];
  unsigned work;                     // banded K4: phase-A dynamic work counter
  int _pad;
  // tile list: tiles stamped this step (the length of FixBand::tlist),
  // band-phase work counter, marker-kernel block ticket (stamps published)
  unsigned tcount, bwork, ticket;
  int _pad2;
};
constexpr int LO_BIAS = 0x40000000;

// Throughput-mode IB force field: 64-bit fixed point (2^-40 lattice force
// units), accumulated with integer atomics -- associative, hence bit-
// deterministic whatever the order -- over 4x4x4 tiles flagged per step.
constexpr double FIX_SCALE = 1099511627776.0;        // 2^40
constexpr double FIX_INV = 1.0 / 1099511627776.0;   // 2^-40
// Skinned bodies, fused path: the marker kernel adds every block's tau_ext /
// CouplingStats sums to 64-bit fixed-point accumulators (integer atomics:
// order-independent, deterministic); the banded K4, after it has waited for
// the marker grid, converts them into the output (pinned host memory) and
// re-zeroes them.  acc = nullptr: no skinned bodies.
constexpr double SKIN_FIX_SCALE = 17592186044416.0;      // 2^44
constexpr double SKIN_FIX_INV = 1.0 / 17592186044416.0;  // 2^-44
constexpr double SKIN_FIX_RANGE = 524288.0;               // 2^19: |sum| * 2^44 < 2^63
constexpr int SKIN_FIX_REP = 16;  // copies of the fused path's [2][32] accumulators
struct SkinOut {
  unsigned long long* acc;  // [nb][32]: dof c (< 14) and stat 14 + k
  double* out;              // tau (concatenated) then 7 stats per body
  int nb, nt;               // bodies, total dofs
  int ndof[2], off[2];      // per body: n_dofs, first tau entry
};

struct FixBand {
  unsigned long long* F;     // 3 per owned cell (x + nx*(y + ny*z))
  unsigned* tflag;           // per 4^3 tile: stamp of the last step a stencil touched it
  int tnx, tny, tnz;         // tile grid
  unsigned stamp;            // step stamp (coupled step index + 1; 0 = never)
  float* fcap;               // diagnostic (fsg_set_force_capture): the body force K4
                             // consumed this step, IB + virtual, AoS fp32; null = off
  // tile list (null: the band phase scans every tile's flag)
  int* tlist;                // tiles stamped this step, in stamping order (StepScratch::tcount)
  unsigned* ready;           // set to `stamp` (release) once every tile of the step is stamped
};

#ifdef __CUDACC__
// release / acquire at GPU scope (PTX memory model): the marker chain's
// "every tile stamped" flag (fsg_ib_fix.cuh) and its consumer (fsg_k4.cuh)
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#endif

__host__ __device__ __forceinline__ unsigned long long ordered_key(double v) {
#ifdef __CUDA_ARCH__
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
#else
  unsigned long long b;
  __builtin_memcpy(&b, &v, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double key_to_double(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double v;
  __builtin_memcpy(&v, &b, 8);
  return v;
#endif
}

// Per-marker stencil record written by the marker kernel.
struct __align__(16) MarkerStencil {
  double ph[3][5];   // phi(k - x_a) for k = lo_a .. hi_a (kernel.hpp:22-33)
  double fl[3];      // lattice force to spread (session.hpp:128, :136-138)
  int lo[3], hi[3];  // inclusive global ranges (kernel.hpp:36-40)
  int valid;
  int _pad;
};

// Compact stencil box (local coordinates) for the spread kernel's cull.
struct __align__(16) MarkerBox {
  short lo[3];
  short valid;
  short hi[3];
  short _pad;
};

// Marker input arrays (SI world frame, session.hpp:113-126).
struct Markers {
  const double* pts;
  const double* vel;
  const double* nrm;
  const double* area;
  int m;
};

// Compact IB band (bounding box of all valid stencils, local coordinates).
struct Band {
  double* F;         // spread IB force, 3 per band cell
  long long cap;     // capacity in cells
};

// Cell-kernel block shape: up to 128 threads along x, the rest along y.
inline dim3 cell_block_dims(const Grid& g) {
  // always 128 threads (the kernels' launch bounds and residency assume it):
  // whole 128-cell rows when they tile nx, else 32 x 4 (e.g. nx = 96: a
  // 96 x 1 block left a quarter of every SM's warp slots empty)
  int bx;
  if (g.nx >= 128 && g.nx % 128 == 0) bx = 128;
  else if (g.nx == 64) bx = 64;
  else bx = 32;
  return dim3(bx, 128 / bx, 1);
}

// Open-boundary pull of a face cell (solver.hpp:59-97 as a pull): an unknown
// population (standard source c - e_i outside the domain) comes from
// clamp(c, 1, n-2) - e_i, i.e. the standard source shifted by the cell's
// clamp displacement D = clamp(c) - c (memory units) -- one offset for every
// unknown direction of the cell, so face cells stay on the constant-offset
// fast path (bit-identical to the general gather).
struct FaceFlags {
  bool x0, x1, y0, y1, z0, z1;
  int D;
};
__device__ __forceinline__ FaceFlags face_flags(const Grid& g, int x, int y, int zg) {
  FaceFlags f;
  f.x0 = x == 0;
  f.x1 = x == g.nx - 1;
  f.y0 = y == 0;
  f.y1 = y == g.ny - 1;
  f.z0 = zg == 0;
  f.z1 = zg == g.nzg - 1;
  f.D = ((int)f.x0 - (int)f.x1) + g.nx * ((int)f.y0 - (int)f.y1) + (int)g.zs * ((int)f.z0 - (int)f.z1);
  return f;
}
__device__ __forceinline__ bool face_unknown(int ex, int ey, int ez, const FaceFlags& f) {
  return (ex > 0 && f.x0) || (ex < 0 && f.x1) || (ey > 0 && f.y0) || (ey < 0 && f.y1) ||
         (ez > 0 && f.z0) || (ez < 0 && f.z1);
}

// Throughput kernels address the 19 pull sources / destinations through
// per-direction base pointers passed as kernel parameters.
struct DirPtrs {
  const float* a[Q];  // A + pull[i]  (interior pull source of direction i)
  float* b[Q];        // B + own[i]   (destination plane of direction i)
};

// Batched throughput step (fsg_batch.cuh): the envs share one configuration,
// so the grid geometry (with its pull/own offsets) and the session constants
// are common kernel parameters; each env contributes one small pack per step.
struct SkinBody;  // fsg_skin.cuh
struct EnvPack {
  StepConsts st;           // this env's frame constants
  const float* A;          // state read this step
  float* B;                // state written this step
  unsigned long long* F;   // fixed-point IB force
  unsigned* tflag;         // tile stamps
  Markers mk;
  MarkerStencil* rec;
  double* fworld;
  double* fworld_h;
  int* valid_h;
  StepScratch* out;
  StepScratch* next;
  unsigned stamp;
  int pulled, frame_on;
  // skinned body (fsg_set_skin, one per env), nullptr: plain markers
  const SkinBody* skb;           // topology + this step's pose (device copy)
  const double* sk_rest;
  const double* sk_nrest;
  const int* sk_wb;
  const double* sk_ww;
  unsigned long long* sk_acc;    // fixed-point tau/stat sums [32]
  double* sk_out;                // tau then 7 stats (pinned)
  int sk_ndof;
  int mk_begin;            // first global marker index of this env
  int item_begin;          // first global phase-A item
  int tile_begin;          // first global band tile
};

constexpr int BATCH_MAX = 64;

struct BatchHead {
  int E;
  int m_total, item_total, tile_total;
  int tnx, tny, tnz;       // tile grid (every env)
  int zc;                  // phase-A planes per item
  int frame_on;            // the batch's frame mode is not None
  int pmode;               // 1 every env pulled, 0 none, 2 mixed
  int skin;                // some env has a skinned body
};

// ---------------------------------------------------------- kernel table --
template <int NB>
struct SkinParamsN;

// z-slab peer transport (fsg_peer_connect): where the two boundary planes'
// crossing populations go besides the session's own buffer -- the lower
// neighbour's top halo plane (ez = -1 populations of local plane 0) and the
// upper neighbour's bottom halo plane (ez = +1 populations of plane nz-1),
// each the base of direction 0 of that plane in the neighbour's write buffer
// (peer memory over NVLink, or the same device).  Null = no neighbour.
struct PeerOut {
  float* lo;
  float* hi;
};

// Launchers exported by each precision translation unit.
struct Launchers {
  void (*fill_rest)(const Grid&, void* A, cudaStream_t);
  void (*set_f)(const Grid&, const double* f, void* A, cudaStream_t);
  void (*init_eq)(const Grid&, const double* rho, const double* u, void* A, cudaStream_t);
  // S readback (post-stream state) into double f[19*n]
  void (*get_f)(const Grid&, const void* A, int pulled, double* f, cudaStream_t);
  // moments of S with optional external force (SoA 3 x n, math type); rho[n], u[3n]
  void (*macroscopic)(const Grid&, const void* A, int pulled, const void* Fext, double* rho,
                      double* u, StepScratch*, cudaStream_t);
  // collide + stream (+ open BC via clamped pull) A -> B
  void (*collide)(const Grid&, const void* A, int pulled, void* B, const void* Fext,
                  const Band*, const StepScratch*, const SessionConsts*, const StepConsts*,
                  StepScratch*, int session_force, int frame_on, cudaStream_t);
  // full F readback of a session step: IB band + virtual force, AoS double
  void (*session_force)(const Grid&, const void* A, int pulled, const Band*, const StepScratch*,
                        const SessionConsts*, const StepConsts*, int frame_on, double* F,
                        cudaStream_t);
  void (*recenter)(const Grid&, const void* A, int pulled, void* B, int sx, int sy, int sz,
                   cudaStream_t);
  // IB: per-marker fused kernel, then the ordered spread into the band
  void (*markers)(const Grid&, const void* A, int pulled, Markers, const SessionConsts*,
                  const StepConsts*, MarkerStencil*, MarkerBox*, double* fworld,
                  double* fworld_host, int* valid_host, StepScratch*, cudaStream_t);
  void (*spread)(const Grid&, int m, const MarkerStencil*, const MarkerBox*, Band,
                 const StepScratch*, cudaStream_t);
  // throughput path (fp32 only; nullptr in the fp64 table): markers scatter
  // fixed-point forces; K4 consumes them.  Both K4 variants reset the next
  // step's scratch from block 0; the host copies the status out on demand.
  // km_done (nullable): every block adds 1 when its markers are complete (a
  // concurrent consumer spins on it); pdl: launched as a programmatic
  // dependent of the kernel before it (which must trigger early).  Returns
  // the grid size.
  // skin (nullable, <= 2 bodies): skinned bodies fused into the marker kernel
  // (fsg_skin_fused.cuh), tau + stats added to the fixed-point skin_acc.
  int (*markers_fix)(const Grid&, const void* A, int pulled, Markers, const SessionConsts*,
                     const StepConsts& st, MarkerStencil*, double* fworld, double* fworld_host,
                     int* valid_host, FixBand, StepScratch*, unsigned* km_done, int pdl,
                     const SkinParamsN<FSG_SKIN_MAX_BODIES>* skin, unsigned long long* skin_acc,
                     cudaStream_t);
  // pure-fluid step (no IB band); planes: 0 all, 1 the two z-boundary planes,
  // 2 the interior planes (z-slab step: boundary first, halo send, interior)
  // po (planes == 1, peer-connected slabs): the boundary planes' crossing
  // populations are also stored into the neighbours' halo planes
  void (*collide_fix)(const Grid&, const void* A, int pulled, void* B, const SessionConsts*,
                      const StepConsts& st, int frame_on, StepScratch* scr, StepScratch* scr_next,
                      int planes, PeerOut po, cudaStream_t);
  // banded coupled step: one K4 launch, a programmatic dependent (pdl != 0)
  // of the marker kernel launched just before it on the same stream
  void (*collide_band)(const Grid&, const void* A, int pulled, void* B, FixBand,
                       const SessionConsts*, const StepConsts& st, int frame_on,
                       StepScratch* scr, StepScratch* scr_next, int pdl, const SkinOut& so,
                       cudaStream_t);
  // batched coupled step over E env sessions (fp32): markers + banded K4 of
  // every env in one launch each; d_packs: E EnvPacks in device memory
  void (*step_batch)(const Grid&, const SessionConsts*, const EnvPack* d_packs, BatchHead h,
                     dim3 block, unsigned* work, cudaStream_t);
  // halo planes (z-slab): pack owned boundary planes / unpack into halo planes
  void (*halo_pack)(const Grid&, const void* B, void* send_lo, void* send_hi, cudaStream_t);
  void (*halo_unpack)(const Grid&, void* B, const void* recv_lo, const void* recv_hi,
                      cudaStream_t);
  int elem_bytes;
};

const Launchers& launchers_fp32();
const Launchers& launchers_fp64();

}  // namespace fsg
