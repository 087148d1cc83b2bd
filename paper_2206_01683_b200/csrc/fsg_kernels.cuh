// fsg_kernels.cuh -- the IB-LBM hot-path kernels, written once and compiled
// twice (included by fsg_kernels_fp32.cu and fsg_kernels_fp64.cu with
// FSG_PREC set to 32 or 64).
//
//   FSG_PREC == 64 : parity mode.  f stored as fp64; every expression keeps
//                    the reference's operation order and the TU is built
//                    with --fmad=false, so results are bit-identical to the
//                    reference (oracle/_ref) on the same inputs.
//   FSG_PREC == 32 : throughput mode.  f stored as fp32 deviations
//                    g_i = f_i - w_i (152 B per cell update); the collision is
//                    evaluated in deviation form, so rounding is relative to
//                    O(|u|) quantities rather than O(1) ones.
//
// Streaming is PULL (gather) with the reference's push + open-boundary
// semantics re-expressed as clamped gathers (solver.hpp:59-97, :157-169):
//   source(c, i) = c - e_i                        if c - e_i is inside the box
//                = wrap(c - e_i)                  periodic
//                = clamp(c, 1, n-2) - e_i         open (neighbour copy)
// The stored array therefore holds POST-COLLISION populations P_n; the
// reference's post-stream state S_{n+1} is gather(P_n).  After set/init/
// recenter the array holds S directly ("pulled" == 0) and the next step is
// collide-only.
#pragma once

#include <float.h>
#include <type_traits>
#include <math.h>

#include "fsg_device.cuh"
#include "fsg_skin.cuh"

#ifndef FSG_PREC
#error "define FSG_PREC to 32 or 64"
#endif

namespace fsg {
#if FSG_PREC == 64
namespace p64 {
using Store = double;
using Real = double;
#else
namespace p32 {
using Store = float;
using Real = float;
#endif

// -------------------------------------------------------------- helpers --
template <int i>
__device__ __forceinline__ double to_abs(Store s) {
#if FSG_PREC == 64
  return s;
#else
  return (double)s + w_of(i);
#endif
}
template <int i>
__device__ __forceinline__ Store from_abs(double f) {
#if FSG_PREC == 64
  return f;
#else
  return (float)(f - w_of(i));
#endif
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/// Memory index of the population that streams into (x,y,z) along i
/// (pull form of solver.hpp:157-169 + apply_open_boundary :65-97).
template <int i>
__device__ __forceinline__ long long pull_src(const Grid& g, int x, int y, int z, bool interior) {
  constexpr int ex = ex_of(i), ey = ey_of(i), ez = ez_of(i);
  if (interior) return mem_index(g, x - ex, y - ey, z - ez);
  const int sx = x - ex, sy = y - ey, sz = z - ez;
  const int szg = g.z0 + sz;
  const bool known = (unsigned)sx < (unsigned)g.nx && (unsigned)sy < (unsigned)g.ny &&
                     (unsigned)szg < (unsigned)g.nzg;
  if (known) return mem_index(g, sx, sy, sz);
  if (g.periodic) {
    const int wx = (sx + g.nx) % g.nx, wy = (sy + g.ny) % g.ny;
    const int wz = g.zpad == 0 ? (sz + g.nz) % g.nz : sz;  // slab: halo holds the wrap
    return mem_index(g, wx, wy, wz);
  }
  const int cx = clampi(x, 1, g.nx - 2), cy = clampi(y, 1, g.ny - 2);
  const int cz = clampi(g.z0 + z, 1, g.nzg - 2) - g.z0;
  return mem_index(g, cx - ex, cy - ey, cz - ez);
}

__device__ __forceinline__ bool is_interior(const Grid& g, int x, int y, int z) {
  const int zg = g.z0 + z;
  return x > 0 && x < g.nx - 1 && y > 0 && y < g.ny - 1 && zg > 0 && zg < g.nzg - 1;
}

/// Gather the 19 post-stream populations S(x,y,z) in storage form.
/// Interior cells (the overwhelming majority) take one branch with constant
/// 32-bit neighbour offsets; boundary cells take the general clamped path.
template <bool PULLED>
__device__ __forceinline__ void gather(const Grid& g, const Store* __restrict__ A, int x, int y,
                                       int z, Store s[Q]) {
  const unsigned m = (unsigned)mem_index(g, x, y, z);  // 19 * cells < 2^32 for every supported grid
  const Store* __restrict__ base = A + m;
  if (!PULLED) {
#pragma unroll
    for (int i = 0; i < Q; ++i) s[i] = base[g.own[i]];
  } else if (is_interior(g, x, y, z)) {
#pragma unroll
    for (int i = 0; i < Q; ++i) s[i] = base[g.pull[i]];
  } else {
    s[0] = A[pull_src<0>(g, x, y, z, false)];
#define FSG_G(I) s[I] = A[(long long)(I)*g.stride + pull_src<I>(g, x, y, z, false)];
    FSG_G(1) FSG_G(2) FSG_G(3) FSG_G(4) FSG_G(5) FSG_G(6) FSG_G(7) FSG_G(8) FSG_G(9)
    FSG_G(10) FSG_G(11) FSG_G(12) FSG_G(13) FSG_G(14) FSG_G(15) FSG_G(16) FSG_G(17) FSG_G(18)
#undef FSG_G
  }
}

template <int a, int b, int c, class T>
__device__ __forceinline__ T edot(T x, T y, T z) {
  // e.v for a D3Q19 direction without multiplying by zero components
  if constexpr (a == 0 && b == 0 && c == 0) return T(0);
  else if constexpr (b == 0 && c == 0) return a > 0 ? x : -x;
  else if constexpr (a == 0 && c == 0) return b > 0 ? y : -y;
  else if constexpr (a == 0 && b == 0) return c > 0 ? z : -z;
  else if constexpr (c == 0) return (a > 0 ? x : -x) + (b > 0 ? y : -y);
  else if constexpr (b == 0) return (a > 0 ? x : -x) + (c > 0 ? z : -z);
  else return (b > 0 ? y : -y) + (c > 0 ? z : -z);
}

// ---------------------------------------------------- cell moments -------
#if FSG_PREC == 64
/// rho, (mx,my,mz) in the reference's accumulation order (solver.hpp:129-136).
__device__ __forceinline__ void moments(const Store s[Q], double& rho, double& mx, double& my,
                                        double& mz) {
  rho = 0.0;
  mx = 0.0;
  my = 0.0;
  mz = 0.0;
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    rho += s[i];
    mx += s[i] * (double)ex_of(i);
    my += s[i] * (double)ey_of(i);
    mz += s[i] * (double)ez_of(i);
  }
}
#else
/// deviation moments: drho = sum g, m = sum e g (sum w e = 0 exactly)
__device__ __forceinline__ void moments_dev(const Store g[Q], float& drho, float& mx, float& my,
                                            float& mz) {
  drho = ((g[0] + (g[1] + g[2])) + ((g[3] + g[4]) + (g[5] + g[6]))) +
         (((g[7] + g[8]) + (g[9] + g[10])) + ((g[11] + g[12]) + (g[13] + g[14]))) +
         ((g[15] + g[16]) + (g[17] + g[18]));
  mx = ((g[1] - g[2]) + (g[7] - g[8])) + ((g[9] - g[10]) + ((g[11] - g[12]) + (g[13] - g[14])));
  my = ((g[3] - g[4]) + (g[7] - g[8])) + ((g[10] - g[9]) + ((g[15] - g[16]) + (g[17] - g[18])));
  mz = ((g[5] - g[6]) + (g[11] - g[12])) + ((g[14] - g[13]) + ((g[15] - g[16]) + (g[18] - g[17])));
}
#endif

// ------------------------------------------------------- virtual force ---
/// frame.hpp:47-53 with the session's lattice scaling (session.hpp:148-163):
/// returns rho*acc*a for the cell at lattice (i,j,k) with bare velocity u.
template <class T>
__device__ __forceinline__ void vf_term(const SessionConsts& sc, const StepConsts& st, int i,
                                        int j, int k, T rho, T ubx, T uby, T ubz, T& fx, T& fy,
                                        T& fz) {
  const T dx = (T)sc.dx, v2p = (T)sc.v2p;
  // cell_frame_position (session.hpp:77-81)
  const T x0 = ((T)i - (T)sc.hd[0]) * dx;
  const T x1 = ((T)j - (T)sc.hd[1]) * dx;
  const T x2 = ((T)k - (T)sc.hd[2]) * dx;
  const T u0 = ubx * v2p, u1 = uby * v2p, u2 = ubz * v2p;
  const T w0 = (T)st.wf[0], w1 = (T)st.wf[1], w2 = (T)st.wf[2];
  const T a0 = (T)st.af[0], a1 = (T)st.af[1], a2 = (T)st.af[2];
  // alpha' x x
  const T ax0 = a1 * x2 - a2 * x1, ax1 = a2 * x0 - a0 * x2, ax2 = a0 * x1 - a1 * x0;
  // omega' x x, omega' x (omega' x x)
  const T wx0 = w1 * x2 - w2 * x1, wx1 = w2 * x0 - w0 * x2, wx2 = w0 * x1 - w1 * x0;
  const T ww0 = w1 * wx2 - w2 * wx1, ww1 = w2 * wx0 - w0 * wx2, ww2 = w0 * wx1 - w1 * wx0;
  // omega' x u
  const T wu0 = w1 * u2 - w2 * u1, wu1 = w2 * u0 - w0 * u2, wu2 = w0 * u1 - w1 * u0;
  const T A0 = -(T)st.a0[0] - ax0 - ww0 - (T)2 * wu0;
  const T A1 = -(T)st.a0[1] - ax1 - ww1 - (T)2 * wu1;
  const T A2 = -(T)st.a0[2] - ax2 - ww2 - (T)2 * wu2;
  const T ra = rho * (T)sc.acc;
  fx = ra * A0;
  fy = ra * A1;
  fz = ra * A2;
}

/// vf_term with the host-rounded fp32 constants (throughput mode).
__device__ __forceinline__ void vf_term32(const SessionConsts& sc, const StepConsts& st, int i,
                                          int j, int k, float rho, float ubx, float uby, float ubz,
                                          float& fx, float& fy, float& fz) {
  const float dx = sc.dx_f, v2p = sc.v2p_f;
  const float x0 = ((float)i - sc.hd_f[0]) * dx;
  const float x1 = ((float)j - sc.hd_f[1]) * dx;
  const float x2 = ((float)k - sc.hd_f[2]) * dx;
  const float u0 = ubx * v2p, u1 = uby * v2p, u2 = ubz * v2p;
  const float w0 = st.wf_f[0], w1 = st.wf_f[1], w2 = st.wf_f[2];
  const float a0 = st.af_f[0], a1 = st.af_f[1], a2 = st.af_f[2];
  const float ax0 = a1 * x2 - a2 * x1, ax1 = a2 * x0 - a0 * x2, ax2 = a0 * x1 - a1 * x0;
  const float wx0 = w1 * x2 - w2 * x1, wx1 = w2 * x0 - w0 * x2, wx2 = w0 * x1 - w1 * x0;
  const float ww0 = w1 * wx2 - w2 * wx1, ww1 = w2 * wx0 - w0 * wx2, ww2 = w0 * wx1 - w1 * wx0;
  const float wu0 = w1 * u2 - w2 * u1, wu1 = w2 * u0 - w0 * u2, wu2 = w0 * u1 - w1 * u0;
  const float ra = rho * sc.acc_f;
  fx = ra * (-st.a0_f[0] - ax0 - ww0 - 2.0f * wu0);
  fy = ra * (-st.a0_f[1] - ax1 - ww1 - 2.0f * wu1);
  fz = ra * (-st.a0_f[2] - ax2 - ww2 - 2.0f * wu2);
}

__device__ __forceinline__ void decode_bbox(const StepScratch* sc, int lo[3], int hi[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = LO_BIAS - sc->bbox_lo_enc[a];
    hi[a] = sc->bbox_hi_enc[a] - 1;
  }
}

// ------------------------------------------------------ block reduction --
__device__ __forceinline__ void report_min(StepScratch* out, double v) {
  // warp min, then one lane per warp does check-then-atomic (few atomics/step)
#if FSG_PREC == 32
  float vf = (float)v;  // fp32 mode: post values are fp32 already
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vf = fminf(vf, __shfl_xor_sync(0xffffffffu, vf, o));
  v = vf == FLT_MAX ? DBL_MAX : (double)vf;
#else
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
#endif
  if ((threadIdx.x & 31) == 0 && !isnan(v)) {
    const unsigned long long nk = ~ordered_key(v);
    const unsigned long long cur = *(volatile unsigned long long*)&out->neg_min_key;
    if (nk > cur) {
      atomicMax(&out->neg_min_key, nk);
      __threadfence();
    }
  }
}

#if FSG_PREC == 32
// Arithmetic type of the throughput collision: the populations are STORED as
// fp32 deviations g_i = f_i - w_i (152 B per cell update) in every variant;
// FSG_C32_MATH selects the arithmetic between the load and the store:
//   0  fp32 (the default) with conservation-exact constants (the host picks
//      fp32 omega*w_i, 1 - omega so that the mass and momentum identities
//      hold exactly, fsg_session.cu conserving_consts_f32) and the odd part
//      of the equilibrium built from j = m + F/2 directly.  Independently
//      rounded constants made rho - 1 and u drift ~1e-7 per step (7e-5 / 2e-4
//      rel-L2 after 1000 c2 steps); with exact identities c1/c2/c3 stay at
//      1e-7 .. 3e-6 (tests/test_long_parity_gpu.py)
//   1  fp64 (the session's fp64 constants, vf_term<double>): ~2e-7 but
//      spills at 80 registers, 512^3 K4 10-20 % slower
//   2  fp64 moments (rho - 1, m summed in fp64), the rest fp32
#ifndef FSG_C32_MATH
#define FSG_C32_MATH 0
#endif
#if FSG_C32_MATH == 1
using CMath = double;
#else
using CMath = float;
#endif
constexpr bool kMoments64 = FSG_C32_MATH == 2;

__device__ __forceinline__ float fma_m(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fma_m(double a, double b, double c) { return fma(a, b, c); }

/// BGK + Guo collision of one cell in deviation form (solver.hpp:129-154
/// restated for g_i = f_i - w_i), with the session force assembled as the
/// reference does (IB band force, then + virtual force, session.hpp:148-163),
/// in arithmetic type M on fp32 storage.  Overwrites s with the
/// post-collision deviations (rounded to fp32); returns min(post f).
template <class M, int FMODE, bool VF>
__device__ __forceinline__ float collide_cell_m(float (&s)[Q], int x, int y, int z, const Grid& g,
                                                float Fx_in, float Fy_in, float Fz_in, bool in_band,
                                                long long lc, const Band& band,
                                                const SessionConsts& sc, const StepConsts& st,
                                                StepScratch* out, float* fcap = nullptr,
                                                long long cidx = 0) {
  constexpr bool D = sizeof(M) == 8;
  // moment arithmetic: fp64 when M is, or when only the moments are
  using MM = typename std::conditional<D || kMoments64, double, float>::type;
  M v[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) v[i] = (M)s[i];
  M drho, mx, my, mz, rho;
  {
    MM w[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) w[i] = (MM)s[i];
    // moments from opposite-pair sums/differences (pairs (1,2),(3,4),...,(17,18))
    const MM d1 = w[1] - w[2], d3 = w[3] - w[4], d5 = w[5] - w[6], d7 = w[7] - w[8],
             d9 = w[9] - w[10], d11 = w[11] - w[12], d13 = w[13] - w[14], d15 = w[15] - w[16],
             d17 = w[17] - w[18];
    const MM dr = ((w[0] + ((w[1] + w[2]) + (w[3] + w[4]))) + ((w[5] + w[6]) + (w[7] + w[8]))) +
                  (((w[9] + w[10]) + (w[11] + w[12])) + ((w[13] + w[14]) + ((w[15] + w[16]) + (w[17] + w[18]))));
    drho = (M)dr;
    mx = (M)((d1 + d7) + (d9 + (d11 + d13)));
    my = (M)((d3 + d7) + ((d15 + d17) - d9));
    mz = (M)((d5 + d11) + ((d15 - d13) - d17));
    rho = (M)((MM)1 + dr);
  }
  M Fx = (M)Fx_in, Fy = (M)Fy_in, Fz = (M)Fz_in;
  if constexpr (FMODE == 2 || FMODE == 3) {  // 3: IB force already in Fx..Fz (fixed-point band)
    if constexpr (FMODE == 2) {
      Fx = in_band ? (M)band.F[3 * lc] : (M)0;
      Fy = in_band ? (M)band.F[3 * lc + 1] : (M)0;
      Fz = in_band ? (M)band.F[3 * lc + 2] : (M)0;
    }
    if constexpr (VF) {
      M bx = 0, by = 0, bz = 0;
      if (rho > (M)0) {
        const M ir = (M)1 / rho;
        bx = mx * ir;
        by = my * ir;
        bz = mz * ir;
      }
#ifndef FSG_VF64
#define FSG_VF64 (FSG_C32_MATH == 1)
#endif
      if constexpr (FSG_VF64) {
        double vx, vy, vz;
        vf_term<double>(sc, st, x, y, g.z0 + z, (double)rho, (double)bx, (double)by, (double)bz,
                        vx, vy, vz);
        Fx = (M)((double)Fx + vx);
        Fy = (M)((double)Fy + vy);
        Fz = (M)((double)Fz + vz);
      } else {
        float vx, vy, vz;
        vf_term32(sc, st, x, y, g.z0 + z, (float)rho, (float)bx, (float)by, (float)bz, vx, vy, vz);
        Fx += (M)vx;
        Fy += (M)vy;
        Fz += (M)vz;
      }
    }
    if (!(rho > (M)0)) {
      atomicAdd(&out->nonpos, 1);
      __threadfence();
    }
  }
  if (fcap) {  // diagnostic: the force this collision consumes
    fcap[3 * cidx] = (float)Fx;
    fcap[3 * cidx + 1] = (float)Fy;
    fcap[3 * cidx + 2] = (float)Fz;
  }
  const M inv_rho = (M)1 / rho;
  // equilibrium momentum j = rho u = m + F/2 (solver.hpp:134-137); the odd
  // (momentum-carrying) part of the equilibrium is built from j itself, not
  // from rho * (j / rho), so momentum relaxes exactly toward j
  const M jx = mx + (M)0.5 * Fx, jy = my + (M)0.5 * Fy, jz = mz + (M)0.5 * Fz;
  const M ux = jx * inv_rho;
  const M uy = jy * inv_rho;
  const M uz = jz * inv_rho;
  const M u2 = ux * ux + uy * uy + uz * uz;
  if (!isfinite(rho + u2)) {
    out->nonfinite = 1;
    __threadfence();
  }
  const M uF3 = (M)3 * (ux * Fx + uy * Fy + uz * Fz);
  const M h15u2 = (M)1.5 * u2;
  // Pair form of  g'_i = (1-w) g_i + w w_i (drho + rho X_i) + guo w_i S_i  with
  // X = 3 eu + 4.5 eu^2 - 1.5 u^2 and S = 3(e-u).F + 9 eu e.F: for e_j = -e_i the
  // even parts (4.5 t^2 - 1.5u^2, 9 t q - 3 u.F) are shared and the odd parts
  // (3t, 3q) flip sign, t = e.u, q = e.F; rho 3t is taken as 3 e.j.
  M om1, ow0, ow1, ow2, gw0, gw1, gw2;
  if constexpr (D) {
    om1 = 1.0 - sc.omega;
    ow0 = sc.omega * (1.0 / 3.0);
    ow1 = sc.omega * (1.0 / 18.0);
    ow2 = sc.omega * (1.0 / 36.0);
    gw0 = sc.guo * (1.0 / 3.0);
    gw1 = sc.guo * (1.0 / 18.0);
    gw2 = sc.guo * (1.0 / 36.0);
  } else {
    om1 = sc.om1_f;
    ow0 = sc.ow_f[0], ow1 = sc.ow_f[1], ow2 = sc.ow_f[2];
    gw0 = sc.gw_f[0], gw1 = sc.gw_f[1], gw2 = sc.gw_f[2];
  }
  const M owr1 = ow1 * rho, owr2 = ow2 * rho;
  const M owd1 = fma_m(ow1, drho, -gw1 * uF3);
  const M owd2 = fma_m(ow2, drho, -gw2 * uF3);
  const M g9_1 = (M)9 * gw1, g9_2 = (M)9 * gw2;
  const M g3_1 = (M)3 * gw1, g3_2 = (M)3 * gw2;
  const float p0 = (float)fma_m(om1, v[0], fma_m(ow0, fma_m(rho, -h15u2, drho), -gw0 * uF3));
  s[0] = p0;
  float min1 = FLT_MAX, min2 = FLT_MAX;
#define FSG_PAIR(I, OWR, OW, OWD, G9, G3, MN)                                            \
  {                                                                                       \
    constexpr int a = ex_of(I), b = ey_of(I), c = ez_of(I);                               \
    const M t = edot<a, b, c, M>(ux, uy, uz);                                             \
    const M q = edot<a, b, c, M>(Fx, Fy, Fz);                                             \
    const M S = fma_m(G9, t * q, fma_m(OWR, fma_m((M)4.5 * t, t, -h15u2), OWD));          \
    const M A = fma_m(OW, (M)3 * edot<a, b, c, M>(jx, jy, jz), G3 * q);                  \
    const float gi = (float)fma_m(om1, v[I], S + A);                                      \
    const float gj = (float)fma_m(om1, v[(I) + 1], S - A);                                \
    s[I] = gi;                                                                            \
    s[(I) + 1] = gj;                                                                      \
    MN = fminf(MN, fminf(gi, gj));                                                        \
  }
  FSG_PAIR(1, owr1, ow1, owd1, g9_1, g3_1, min1)
  FSG_PAIR(3, owr1, ow1, owd1, g9_1, g3_1, min1)
  FSG_PAIR(5, owr1, ow1, owd1, g9_1, g3_1, min1)
  FSG_PAIR(7, owr2, ow2, owd2, g9_2, g3_2, min2)
  FSG_PAIR(9, owr2, ow2, owd2, g9_2, g3_2, min2)
  FSG_PAIR(11, owr2, ow2, owd2, g9_2, g3_2, min2)
  FSG_PAIR(13, owr2, ow2, owd2, g9_2, g3_2, min2)
  FSG_PAIR(15, owr2, ow2, owd2, g9_2, g3_2, min2)
  FSG_PAIR(17, owr2, ow2, owd2, g9_2, g3_2, min2)
#undef FSG_PAIR
  // min over post-collision f = g' + w_i, per weight class (monotone in g')
  return fminf(p0 + (float)(1.0 / 3.0), fminf(min1 + (float)(1.0 / 18.0), min2 + (float)(1.0 / 36.0)));
}

template <int FMODE, bool VF>
__device__ __forceinline__ float collide_cell32(float (&s)[Q], int x, int y, int z, const Grid& g,
                                                float Fx, float Fy, float Fz, bool in_band,
                                                long long lc, const Band& band,
                                                const SessionConsts& sc, const StepConsts& st,
                                                StepScratch* out, float* fcap = nullptr,
                                                long long cidx = 0) {
  return collide_cell_m<CMath, FMODE, VF>(s, x, y, z, g, Fx, Fy, Fz, in_band, lc, band, sc, st, out,
                                          fcap, cidx);
}
#endif

// =============================================================== K4 ======
// Fused: [moments of S] + [virtual force] + [IB band force] + BGK/Guo
// collide (solver.hpp:103-178) + pull stream + open/periodic BC.
// FMODE: 0 no force, 1 external full-grid force (SoA, Real), 2 session force
// (IB band from K_d, plus virtual force when frame_on).
template <bool PULLED, int FMODE, bool VF>
__global__ void __launch_bounds__(128) k_collide(Grid g, const Store* __restrict__ A,
                                                 Store* __restrict__ B,
                                                 const Real* __restrict__ Fext, Band band,
                                                 const StepScratch* __restrict__ bscr,
                                                 const SessionConsts* __restrict__ scp,
                                                 const StepConsts* __restrict__ stp,
                                                 StepScratch* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  const bool live = x < g.nx && y < g.ny;
  double vmin = DBL_MAX;
  if (live) {
    Store s[Q];
    gather<PULLED>(g, A, x, y, z, s);
    const unsigned m = (unsigned)mem_index(g, x, y, z);
    const SessionConsts& sc = *scp;
    // -------- force F for this cell
    Real Fx = 0, Fy = 0, Fz = 0;
    if constexpr (FMODE == 1) {
      const long long c = (long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z);
      Fx = Fext[c];
      Fy = Fext[g.n + c];
      Fz = Fext[2 * g.n + c];
    }
    bool in_band = false;
    long long lc = 0;
    if constexpr (FMODE == 2) {
      int lo[3], hi[3];
      decode_bbox(bscr, lo, hi);
      in_band = x >= lo[0] && x <= hi[0] && y >= lo[1] && y <= hi[1] && z >= lo[2] && z <= hi[2];
      if (in_band)
        lc = (long long)(x - lo[0]) +
             (long long)(hi[0] - lo[0] + 1) * ((long long)(y - lo[1]) + (long long)(hi[1] - lo[1] + 1) * (z - lo[2]));
    }
#if FSG_PREC == 64
    double rho, mx, my, mz;
    moments(s, rho, mx, my, mz);
    if constexpr (FMODE == 2) {
      // BodyForceField cleared to zero, IB spread accumulated (K_d), then the
      // virtual force added on top (session.hpp:95, :129-144, :148-163)
      Fx = in_band ? band.F[3 * lc] : 0.0;
      Fy = in_band ? band.F[3 * lc + 1] : 0.0;
      Fz = in_band ? band.F[3 * lc + 2] : 0.0;
      if constexpr (VF) {
        double bx = 0.0, by = 0.0, bz = 0.0;
        if (rho > 0.0) {  // macroscopic_into with F = 0 (solver.hpp:42-48)
          bx = (mx + 0.5 * 0.0) / rho;
          by = (my + 0.5 * 0.0) / rho;
          bz = (mz + 0.5 * 0.0) / rho;
        }
        double vx, vy, vz;
        vf_term<double>(sc, *stp, x, y, g.z0 + z, rho, bx, by, bz, vx, vy, vz);
        Fx = Fx + vx;
        Fy = Fy + vy;
        Fz = Fz + vz;
      }
      if (!(rho > 0.0)) atomicAdd(&out->nonpos, 1);
    }
    const double omega = sc.omega, guo = sc.guo;
    const double inv_rho = 1.0 / rho;
    const double ux = (mx + 0.5 * Fx) * inv_rho;
    const double uy = (my + 0.5 * Fy) * inv_rho;
    const double uz = (mz + 0.5 * Fz) * inv_rho;
    const double u2 = ux * ux + uy * uy + uz * uz;
    if (!isfinite(rho + u2)) out->nonfinite = 1;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const double exd = ex_of(i), eyd = ey_of(i), ezd = ez_of(i);
      const double eu = exd * ux + eyd * uy + ezd * uz;
      const double feq = w_of(i) * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * u2);
      const double sx = 3.0 * (exd - ux) + 9.0 * eu * exd;
      const double sy = 3.0 * (eyd - uy) + 9.0 * eu * eyd;
      const double sz = 3.0 * (ezd - uz) + 9.0 * eu * ezd;
      const double src = guo * w_of(i) * (sx * Fx + sy * Fy + sz * Fz);
      const double post = s[i] - omega * (s[i] - feq) + src;
      vmin = post < vmin ? post : vmin;
      B[g.own[i] + m] = post;
    }
#else
    const float fmin_dev = collide_cell32<FMODE, VF>(s, x, y, z, g, Fx, Fy, Fz, in_band, lc, band,
                                                     sc, *stp, out);
    Store* __restrict__ ob = B + m;
#pragma unroll
    for (int i = 0; i < Q; ++i) ob[g.own[i]] = s[i];
    vmin = (double)fmin_dev;
#endif
  }
  report_min(out, vmin);
}

#if FSG_PREC == 32
#include "fsg_k4.cuh"
#include "fsg_k4_tma.cuh"
#endif

// ====================================================== small kernels =====
__global__ void k_fill_rest(Grid g, Store* A) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= g.n) return;
  const int x = (int)(t % g.nx);
  const int y = (int)((t / g.nx) % g.ny);
  const int z = (int)(t / g.plane);
  const long long m = mem_index(g, x, y, z);
  // LatticeGrid::reset_to_rest (lattice.hpp:98-104): f_i = w_i (deviation 0)
#pragma unroll
  for (int i = 0; i < Q; ++i) {
#if FSG_PREC == 64
    A[i * g.stride + m] = w_of(i);
#else
    A[i * g.stride + m] = 0.0f;
#endif
  }
}

__global__ void k_set_f(Grid g, const double* __restrict__ f, Store* A) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int z = (int)(c / g.plane);
  const long long m = mem_index(g, x, y, z);
#define FSG_S(I) A[(long long)(I)*g.stride + m] = from_abs<I>(f[(long long)(I)*g.n + c]);
  FSG_S(0) FSG_S(1) FSG_S(2) FSG_S(3) FSG_S(4) FSG_S(5) FSG_S(6) FSG_S(7) FSG_S(8) FSG_S(9)
  FSG_S(10) FSG_S(11) FSG_S(12) FSG_S(13) FSG_S(14) FSG_S(15) FSG_S(16) FSG_S(17) FSG_S(18)
#undef FSG_S
}

/// LatticeGrid::initialize (lattice.hpp:107-116) with equilibrium_dir (:41-45).
__global__ void k_init_eq(Grid g, const double* __restrict__ rho, const double* __restrict__ u,
                          Store* A) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int z = (int)(c / g.plane);
  const long long m = mem_index(g, x, y, z);
  const double r = rho[c], ux = u[3 * c], uy = u[3 * c + 1], uz = u[3 * c + 2];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const double eu = ex_of(i) * ux + ey_of(i) * uy + ez_of(i) * uz;
    const double u2 = ux * ux + uy * uy + uz * uz;
    const double feq = w_of(i) * r * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * u2);
#if FSG_PREC == 64
    A[i * g.stride + m] = feq;
#else
    // deviation computed without cancellation: w*(r-1 + r*(3eu + 4.5eu^2 - 1.5u2))
    A[i * g.stride + m] = (float)(w_of(i) * ((r - 1.0) + r * (3.0 * eu + 4.5 * eu * eu - 1.5 * u2)));
    (void)feq;
#endif
  }
}

template <bool PULLED>
__global__ void k_get_f(Grid g, const Store* __restrict__ A, double* __restrict__ f) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int z = (int)(c / g.plane);
  Store s[Q];
  gather<PULLED>(g, A, x, y, z, s);
#define FSG_O(I) f[(long long)(I)*g.n + c] = to_abs<I>(s[I]);
  FSG_O(0) FSG_O(1) FSG_O(2) FSG_O(3) FSG_O(4) FSG_O(5) FSG_O(6) FSG_O(7) FSG_O(8) FSG_O(9)
  FSG_O(10) FSG_O(11) FSG_O(12) FSG_O(13) FSG_O(14) FSG_O(15) FSG_O(16) FSG_O(17) FSG_O(18)
#undef FSG_O
}

/// Moments of S (solver.hpp:25-51) into rho[n], u[3n] (fp64 out).
template <bool PULLED, bool BARE>
__device__ __forceinline__ void cell_moments(const Grid& g, const Store* __restrict__ A, int x,
                                             int y, int z, double Fx, double Fy, double Fz,
                                             double& rho_o, double& ux, double& uy, double& uz,
                                             bool& bad) {
  Store s[Q];
  gather<PULLED>(g, A, x, y, z, s);
#if FSG_PREC == 64
  double rho, mx, my, mz;
  moments(s, rho, mx, my, mz);
  rho_o = rho;
  bad = !(rho > 0.0);
  if (bad) {
    ux = uy = uz = 0.0;
    return;
  }
  ux = (mx + 0.5 * Fx) / rho;
  uy = (my + 0.5 * Fy) / rho;
  uz = (mz + 0.5 * Fz) / rho;
#else
  float drho, mx, my, mz;
  moments_dev(s, drho, mx, my, mz);
  const float rho = 1.0f + drho;
  rho_o = 1.0 + (double)drho;
  bad = !(rho > 0.0f);
  if (bad) {
    ux = uy = uz = 0.0;
    return;
  }
  ux = (mx + 0.5f * (float)Fx) / rho;
  uy = (my + 0.5f * (float)Fy) / rho;
  uz = (mz + 0.5f * (float)Fz) / rho;
#endif
  (void)BARE;
}

/// Bare velocity of gathered populations: macroscopic_into with F = 0
/// (solver.hpp:42-48, session.hpp:95-96); u = 0 where rho <= 0.
__device__ __forceinline__ void bare_velocity(const Store s[Q], double& ux, double& uy, double& uz) {
#if FSG_PREC == 64
  double rho, mx, my, mz;
  moments(s, rho, mx, my, mz);
  if (!(rho > 0.0)) {
    ux = uy = uz = 0.0;
    return;
  }
  ux = (mx + 0.5 * 0.0) / rho;
  uy = (my + 0.5 * 0.0) / rho;
  uz = (mz + 0.5 * 0.0) / rho;
#else
  float drho, mx, my, mz;
  moments_dev(s, drho, mx, my, mz);
  const float rho = 1.0f + drho;
  if (!(rho > 0.0f)) {
    ux = uy = uz = 0.0;
    return;
  }
  ux = (mx + 0.0f) / rho;
  uy = (my + 0.0f) / rho;
  uz = (mz + 0.0f) / rho;
#endif
}

template <bool PULLED>
__global__ void k_macroscopic(Grid g, const Store* __restrict__ A, const Real* __restrict__ Fext,
                              double* __restrict__ rho, double* __restrict__ u, StepScratch* out) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int z = (int)(c / g.plane);
  const double Fx = Fext ? (double)Fext[c] : 0.0, Fy = Fext ? (double)Fext[g.n + c] : 0.0,
               Fz = Fext ? (double)Fext[2 * g.n + c] : 0.0;
  double r, ux, uy, uz;
  bool bad;
  cell_moments<PULLED, false>(g, A, x, y, z, Fx, Fy, Fz, r, ux, uy, uz, bad);
  rho[c] = r;
  u[3 * c] = ux;
  u[3 * c + 1] = uy;
  u[3 * c + 2] = uz;
  if (bad) atomicAdd(&out->nonpos, 1);
}

/// Session BodyForceField readback: band IB force + virtual force (AoS).
template <bool PULLED>
__global__ void k_session_force(Grid g, const Store* __restrict__ A, Band band,
                                const StepScratch* __restrict__ bscr,
                                const SessionConsts* __restrict__ scp,
                                const StepConsts* __restrict__ stp, int frame_on,
                                double* __restrict__ F) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int z = (int)(c / g.plane);
  int lo[3], hi[3];
  decode_bbox(bscr, lo, hi);
  double Fx = 0.0, Fy = 0.0, Fz = 0.0;
  if (x >= lo[0] && x <= hi[0] && y >= lo[1] && y <= hi[1] && z >= lo[2] && z <= hi[2]) {
    const long long lc = (long long)(x - lo[0]) +
                         (long long)(hi[0] - lo[0] + 1) *
                             ((long long)(y - lo[1]) + (long long)(hi[1] - lo[1] + 1) * (z - lo[2]));
    Fx = band.F[3 * lc];
    Fy = band.F[3 * lc + 1];
    Fz = band.F[3 * lc + 2];
  }
  if (frame_on) {
    double r, ux, uy, uz;
    bool bad;
    cell_moments<PULLED, true>(g, A, x, y, z, 0.0, 0.0, 0.0, r, ux, uy, uz, bad);
    double vx, vy, vz;
#if FSG_PREC == 64
    vf_term<double>(*scp, *stp, x, y, g.z0 + z, r, ux, uy, uz, vx, vy, vz);
#else
    float fx, fy, fz;
    vf_term<float>(*scp, *stp, x, y, g.z0 + z, (float)r, (float)ux, (float)uy, (float)uz, fx, fy,
                   fz);
    vx = fx;
    vy = fy;
    vz = fz;
#endif
    Fx = Fx + vx;
    Fy = Fy + vy;
    Fz = Fz + vz;
  }
  F[3 * c] = Fx;
  F[3 * c + 1] = Fy;
  F[3 * c + 2] = Fz;
}

/// frame::recenter (frame.hpp:132-154): B(x) = S(clamp(x + shift)).
template <bool PULLED>
__global__ void k_recenter(Grid g, const Store* __restrict__ A, Store* __restrict__ B, int sx,
                           int sy, int sz) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= g.n) return;
  const int x = (int)(c % g.nx);
  const int y = (int)((c / g.nx) % g.ny);
  const int z = (int)(c / g.plane);
  const int qx = clampi(x + sx, 0, g.nx - 1), qy = clampi(y + sy, 0, g.ny - 1),
            qz = clampi(z + sz, 0, g.nz - 1);
  Store s[Q];
  gather<PULLED>(g, A, qx, qy, qz, s);
  const long long m = mem_index(g, x, y, z);
#pragma unroll
  for (int i = 0; i < Q; ++i) B[i * g.stride + m] = s[i];
}

// ====================================================== IB kernels =======
#include "fsg_ib.cuh"
#if FSG_PREC == 32
#include "fsg_ib_fix.cuh"
#include "fsg_batch.cuh"
#endif

// ======================================================= halo (slabs) ====
// Populations crossing a z face (lattice.hpp:25-26): ez=+1 {5,11,14,15,18},
// ez=-1 {6,12,13,16,17}.
__device__ __forceinline__ int up_dir(int k) { return k == 0 ? 5 : k == 1 ? 11 : k == 2 ? 14 : k == 3 ? 15 : 18; }
__device__ __forceinline__ int dn_dir(int k) { return k == 0 ? 6 : k == 1 ? 12 : k == 2 ? 13 : k == 3 ? 16 : 17; }

__global__ void k_halo_pack(Grid g, const Store* __restrict__ B, Store* send_lo, Store* send_hi) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 5 * g.plane) return;
  const int k = (int)(t / g.plane);
  const long long xy = t % g.plane;
  // top owned plane, ez=+1 populations -> upper neighbour
  send_hi[t] = B[up_dir(k) * g.stride + g.zs * (g.nz - 1 + g.zpad) + xy];
  // bottom owned plane, ez=-1 populations -> lower neighbour
  send_lo[t] = B[dn_dir(k) * g.stride + g.zs * (0 + g.zpad) + xy];
}
__global__ void k_halo_unpack(Grid g, Store* B, const Store* __restrict__ recv_lo,
                              const Store* __restrict__ recv_hi) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 5 * g.plane) return;
  const int k = (int)(t / g.plane);
  const long long xy = t % g.plane;
  // lower neighbour's top plane (ez=+1) -> halo plane z = -1
  if (recv_lo) B[up_dir(k) * g.stride + xy] = recv_lo[t];
  // upper neighbour's bottom plane (ez=-1) -> halo plane z = nz
  if (recv_hi) B[dn_dir(k) * g.stride + g.zs * (g.nz + g.zpad) + xy] = recv_hi[t];
}

// ======================================================== launchers =====
inline dim3 cell_block(const Grid& g) { return cell_block_dims(g); }
inline dim3 cell_grid(const Grid& g, dim3 b) {
  return dim3((g.nx + b.x - 1) / b.x, (g.ny + b.y - 1) / b.y, g.nz);
}
inline unsigned lin_blocks(long long n, int t) { return (unsigned)((n + t - 1) / t); }

static void L_fill_rest(const Grid& g, void* A, cudaStream_t s) {
  k_fill_rest<<<lin_blocks(g.n, 256), 256, 0, s>>>(g, (Store*)A);
}
static void L_set_f(const Grid& g, const double* f, void* A, cudaStream_t s) {
  k_set_f<<<lin_blocks(g.n, 256), 256, 0, s>>>(g, f, (Store*)A);
}
static void L_init_eq(const Grid& g, const double* rho, const double* u, void* A, cudaStream_t s) {
  k_init_eq<<<lin_blocks(g.n, 256), 256, 0, s>>>(g, rho, u, (Store*)A);
}
static void L_get_f(const Grid& g, const void* A, int pulled, double* f, cudaStream_t s) {
  if (pulled)
    k_get_f<true><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, f);
  else
    k_get_f<false><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, f);
}
static void L_macroscopic(const Grid& g, const void* A, int pulled, const void* Fext, double* rho,
                          double* u, StepScratch* out, cudaStream_t s) {
  if (pulled)
    k_macroscopic<true><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, (const Real*)Fext, rho, u, out);
  else
    k_macroscopic<false><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, (const Real*)Fext, rho, u, out);
}
template <bool P, int FM, bool VF>
static void launch_collide_t(const Grid& g, const void* A, void* B, const void* Fext,
                             const Band* band, const StepScratch* bscr, const SessionConsts* sc,
                             const StepConsts* st, StepScratch* out, cudaStream_t s) {
  Band bd = band ? *band : Band{nullptr, 0};
  const dim3 b = cell_block(g);
#if FSG_PREC == 32
  if (P) {
    DirPtrs dp;
    for (int i = 0; i < Q; ++i) {
      dp.a[i] = (const float*)A + g.pull[i];
      dp.b[i] = (float*)B + g.own[i];
    }
    k_collide_fast<FM, VF><<<cell_grid(g, b), b, 0, s>>>(g, dp, (const float*)A, (const float*)Fext,
                                                         bd, bscr, sc, st, out);
    return;
  }
#endif
  k_collide<P, FM, VF><<<cell_grid(g, b), b, 0, s>>>(g, (const Store*)A, (Store*)B, (const Real*)Fext,
                                                     bd, bscr, sc, st, out);
}
static void L_collide(const Grid& g, const void* A, int pulled, void* B, const void* Fext,
                      const Band* band, const StepScratch* bscr, const SessionConsts* sc,
                      const StepConsts* st, StepScratch* out, int session_force, int frame_on,
                      cudaStream_t s) {
  const int fm = session_force ? 2 : (Fext ? 1 : 0);
#define FSG_LC(P, FM, VF) launch_collide_t<P, FM, VF>(g, A, B, Fext, band, bscr, sc, st, out, s)
  if (pulled) {
    if (fm == 0) FSG_LC(true, 0, false);
    else if (fm == 1) FSG_LC(true, 1, false);
    else if (frame_on) FSG_LC(true, 2, true);
    else FSG_LC(true, 2, false);
  } else {
    if (fm == 0) FSG_LC(false, 0, false);
    else if (fm == 1) FSG_LC(false, 1, false);
    else if (frame_on) FSG_LC(false, 2, true);
    else FSG_LC(false, 2, false);
  }
#undef FSG_LC
}
static void L_session_force(const Grid& g, const void* A, int pulled, const Band* band,
                            const StepScratch* bscr, const SessionConsts* sc, const StepConsts* st,
                            int frame_on, double* F, cudaStream_t s) {
  if (pulled)
    k_session_force<true><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, *band, bscr, sc, st, frame_on, F);
  else
    k_session_force<false><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, *band, bscr, sc, st, frame_on, F);
}
static void L_recenter(const Grid& g, const void* A, int pulled, void* B, int sx, int sy, int sz,
                       cudaStream_t s) {
  if (pulled)
    k_recenter<true><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, (Store*)B, sx, sy, sz);
  else
    k_recenter<false><<<lin_blocks(g.n, 128), 128, 0, s>>>(g, (const Store*)A, (Store*)B, sx, sy, sz);
}
static void L_markers(const Grid& g, const void* A, int pulled, Markers mk,
                      const SessionConsts* sc, const StepConsts* st, MarkerStencil* ms,
                      MarkerBox* boxes, double* fworld, double* fworld_h, int* valid_h,
                      StepScratch* out, cudaStream_t s) {
  if (mk.m == 0) return;
  const unsigned nb = (unsigned)((mk.m + MK_PER_BLOCK - 1) / MK_PER_BLOCK);
  if (pulled)
    k_markers<true><<<nb, 128, 0, s>>>(g, (const Store*)A, mk, sc, st, ms, boxes, fworld, fworld_h,
                                       valid_h, out);
  else
    k_markers<false><<<nb, 128, 0, s>>>(g, (const Store*)A, mk, sc, st, ms, boxes, fworld, fworld_h,
                                        valid_h, out);
}
static void L_spread(const Grid& g, int m, const MarkerStencil* ms, const MarkerBox* boxes,
                     Band band, const StepScratch* bscr, cudaStream_t s) {
  if (m == 0) return;
  k_spread<<<296, SP_THREADS, 0, s>>>(g, m, ms, boxes, band, bscr);
}
static void L_halo_pack(const Grid& g, const void* B, void* lo, void* hi, cudaStream_t s) {
  k_halo_pack<<<lin_blocks(5 * g.plane, 256), 256, 0, s>>>(g, (const Store*)B, (Store*)lo, (Store*)hi);
}
static void L_halo_unpack(const Grid& g, void* B, const void* lo, const void* hi, cudaStream_t s) {
  k_halo_unpack<<<lin_blocks(5 * g.plane, 256), 256, 0, s>>>(g, (Store*)B, (const Store*)lo, (const Store*)hi);
}

#if FSG_PREC == 32
template <int NB>
static SkinParamsN<NB> skin_narrow(const SkinParams& P) {
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

static int L_markers_fix(const Grid& g, const void* A, int pulled, Markers mk,
                         const SessionConsts* sc, const StepConsts& st, MarkerStencil* rec,
                         double* fworld, double* fworld_h, int* valid_h, FixBand fb,
                         StepScratch* out, unsigned* km_done, int pdl, const SkinParams* skin,
                         unsigned long long* skin_acc, cudaStream_t s) {
  if (mk.m == 0) return 0;
  // marker blocks per SM (FSG_KM_PER_SM overrides; 0 = one marker per warp,
  // a single wave of up to m/4 blocks).  Default: a persistent grid of
  // FSG_KM_PER_SM_DEFAULT blocks per SM when the state exceeds L2 (K4's phase
  // A is long enough to hide the longer marker chain and keeps more of every
  // SM: c3 141.4 -> 139.8 us), one wave otherwise (the marker chain is the
  // step's critical path: c1 40.5 vs 48.0 us at 3 per SM)
  static int nsm = 0, l2 = 0, env_cap = -2;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const char* e = getenv("FSG_KM_PER_SM");
    env_cap = e ? (atof(e) > 0 ? std::max(1, (int)(atof(e) * nsm)) : 0) : -1;
  }
  const bool big = (double)g.n * 152.0 > (double)l2;
  const int cap = env_cap >= 0 ? env_cap
                               : (big ? std::max(1, (int)(FSG_KM_PER_SM_DEFAULT * nsm)) : 0);
  unsigned nb = (unsigned)((mk.m + FX_PER_BLOCK - 1) / FX_PER_BLOCK);
  if (cap > 0) nb = std::min(nb, (unsigned)cap);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (skin) {  // skinned bodies fused into the marker kernel (fsg_skin_fused.cuh)
#define FSG_KS(P, NB)                                                                        \
  cudaLaunchKernelEx(&cfg, k_markers_skin<P, NB>, g, (const float*)A, mk, sc, st, rec, fworld, \
                     fworld_h, valid_h, fb, out, skin_narrow<NB>(*skin), skin_acc)
    if (skin->nb <= 1) {
      if (pulled) FSG_KS(true, 1);
      else FSG_KS(false, 1);
    } else {
      if (pulled) FSG_KS(true, 2);
      else FSG_KS(false, 2);
    }
#undef FSG_KS
    return (int)nb;
  }
  if (pulled)
    cudaLaunchKernelEx(&cfg, k_markers_fix<true>, g, (const float*)A, mk, sc, st, rec, fworld,
                       fworld_h, valid_h, fb, out, km_done);
  else
    cudaLaunchKernelEx(&cfg, k_markers_fix<false>, g, (const float*)A, mk, sc, st, rec, fworld,
                       fworld_h, valid_h, fb, out, km_done);
  return (int)nb;
}
static void L_collide_fix(const Grid& g, const void* A, int pulled, void* B,
                          const SessionConsts* sc, const StepConsts& st, int frame_on,
                          StepScratch* scr, StepScratch* scr_next, int planes, PeerOut po,
                          cudaStream_t s) {
  DirPtrs dp;
  for (int i = 0; i < Q; ++i) {
    dp.a[i] = (const float*)A + (pulled ? g.pull[i] : g.own[i]);
    dp.b[i] = (float*)B + g.own[i];
  }
  // bulk-async staged variant (fsg_k4_tma.cuh), opt-in with FSG_K4_TMA=1:
  // whole-grid steps of a pulled state on grids whose planes keep 16-byte row
  // alignment.  Bit-identical to the default, but measured slower on large
  // grids (256x128x128: 134 vs 112 us; 512^3: 4.45 vs 4.16 ms) and mixed on
  // small ones (96x48x48: 10.8 vs 11.8 us; 64^3: 12.3 vs 11.3 us).
  static const bool use_tma = [] {
    const char* e = getenv("FSG_K4_TMA");
    return e && e[0] == '1';
  }();
  if (use_tma && pulled && planes == 0 && g.nx % 4 == 0) {
    static int nsm_t = 0, res_t = 0;
    if (!nsm_t) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm_t, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res_t, k_collide_tma<true>, TMA_TW, 0);
      res_t = std::max(res_t, 1);
    }
    const long long ntile = ((g.plane + TMA_TW - 1) / TMA_TW) * g.nz;
    const unsigned grid = (unsigned)std::min<long long>(ntile, (long long)nsm_t * res_t);
    if (frame_on)
      k_collide_tma<true><<<grid, TMA_TW, 0, s>>>(g, dp, (const float*)A, sc, st, scr, scr_next);
    else
      k_collide_tma<false><<<grid, TMA_TW, 0, s>>>(g, dp, (const float*)A, sc, st, scr, scr_next);
    return;
  }
  // planes: 0 all, 1 the two boundary planes (z-slab), 2 the interior planes
  ZRange zr{0, g.nz, 1};
  if (planes == 1) zr = ZRange{0, g.nz, std::max(1, g.nz - 1)};
  if (planes == 2) zr = ZRange{1, g.nz - 1, 1};
  const int nq = (zr.hi - zr.lo + zr.step - 1) / zr.step;
  if (nq <= 0) return;
  const dim3 b = cell_block(g), g3 = cell_grid(g, b);
  const long long ntile = (long long)g3.x * g3.y * nq;
  static int resident = 0;  // blocks of k_collide_fix resident per SM (same for all variants)
  static int nsm = 0;
  if (!resident) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_collide_fix<true, true>, 128, 0);
    const char* e = getenv("FSG_K4_PER_SM");  // dev A/B: resident fluid-K4 blocks per SM
    if (e && atoi(e) > 0) resident = std::min(resident, atoi(e));
    if (resident < 1) resident = 1;
  }
  const long long grid = std::min<long long>(ntile, (long long)nsm * resident);
  const dim3 gr((unsigned)grid);
  // z chunk: >= ~8 work items per resident block for balance, and at most 2
  // planes (1 for wide planes) so the blocks in flight stay within a few
  // planes of every direction array (measured: 512^3 32.1 vs 28.7 GLUPS at
  // zc 1 vs 128; 256x128x128 best at 2)
  const long long ncol = (long long)g3.x * g3.y;
  const long long nzc_want = (8 * grid + ncol - 1) / ncol;
  int zc = (int)std::max<long long>(1, nq / std::max<long long>(1, nzc_want));
  zc = std::min(zc, g.plane >= (1 << 17) ? 1 : 2);
  static const int zc_env = [] {  // dev A/B: fluid-K4 item depth
    const char* e = getenv("FSG_K4F_ZC");
    return e ? atoi(e) : 0;
  }();
  if (zc_env > 0) zc = zc_env;
#define FSG_LF(P, V) \
  k_collide_fix<P, V><<<gr, b, 0, s>>>(g, dp, (const float*)A, sc, st, scr, scr_next, zc, zr, po)
  if (pulled) {
    if (frame_on) FSG_LF(true, true);
    else FSG_LF(true, false);
  } else {
    if (frame_on) FSG_LF(false, true);
    else FSG_LF(false, false);
  }
#undef FSG_LF
}

// Batched step: markers of every env, then the batched banded K4 as their
// programmatic dependent.  work: this step's phase-A counter (zeroed).
static void L_step_batch(const Grid& g, const SessionConsts* sc, const EnvPack* d_packs,
                         BatchHead h, dim3 block, unsigned* work, cudaStream_t s) {
  static int nsm = 0, res = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, k_collide_band_batch<2, true>, 128, 0);
    res = std::max(res, 1);
  }
  if (h.m_total > 0) {
    const int need = (h.m_total + FX_PER_BLOCK - 1) / FX_PER_BLOCK;
    const int grid = std::min(need, nsm * FSG_KMB_PER_SM);
    if (h.skin)
      k_markers_batch<true><<<grid, 128, 0, s>>>(g, sc, d_packs, h);
    else
      k_markers_batch<false><<<grid, 128, 0, s>>>(g, sc, d_packs, h);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min<long long>(h.item_total, (long long)nsm * res));
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = h.m_total > 0 ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define FSG_BB(PM, V) cudaLaunchKernelEx(&cfg, k_collide_band_batch<PM, V>, g, sc, d_packs, h, work)
  if (h.frame_on) {
    if (h.pmode == 1) FSG_BB(1, true);
    else if (h.pmode == 0) FSG_BB(0, true);
    else FSG_BB(2, true);
  } else {
    if (h.pmode == 1) FSG_BB(1, false);
    else if (h.pmode == 0) FSG_BB(0, false);
    else FSG_BB(2, false);
  }
#undef FSG_BB
}

// Banded K4 as a programmatic dependent of the marker kernel just launched on
// the same stream (see k_collide_band).
static void L_collide_band(const Grid& g, const void* A, int pulled, void* B, FixBand fb,
                           const SessionConsts* sc, const StepConsts& st, int frame_on,
                           StepScratch* scr, StepScratch* scr_next, int pdl, const SkinOut& so,
                           cudaStream_t s) {
  DirPtrs dp;
  for (int i = 0; i < Q; ++i) {
    dp.a[i] = (const float*)A + (pulled ? g.pull[i] : g.own[i]);
    dp.b[i] = (float*)B + g.own[i];
  }
  static int nsm = 0, res1 = 0, res2 = 0, l2 = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res1, k_collide_band<true, true, false>, 128, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res2, k_collide_band<true, true, true>, 128, 0);
    const char* e = getenv("FSG_K4B_PER_SM");  // dev A/B: resident banded-K4 blocks per SM
    if (e && atoi(e) > 0) res1 = std::min(res1, atoi(e)), res2 = std::min(res2, atoi(e));
    res1 = std::max(res1, 1);
    res2 = std::max(res2, 1);
  }
  static const int pair_env = [] {  // dev A/B: FSG_K4_PAIR=0/1 forces the variant
    const char* e = getenv("FSG_K4_PAIR");
    return e ? atoi(e) : -1;
  }();
  const bool pair = pair_env >= 0 ? pair_env > 0 : (double)g.n * 152.0 > (double)l2;
  const int res = pair ? res2 : res1;
  const dim3 b = cell_block(g);
  // phase-A item: one block row x zc planes inside one tile layer (zc | 4);
  // 2 planes when that still leaves >= 8 items per block, else 1
  const long long ncol = (long long)((g.nx + b.x - 1) / b.x) * ((g.ny + b.y - 1) / b.y);
  const long long full = (long long)nsm * res;
  static int zc_env = -1;
  if (zc_env < 0) {
    const char* e = getenv("FSG_K4_ZC");  // dev A/B: phase-A item depth
    zc_env = e ? atoi(e) : 0;
  }
  const int zc = zc_env > 0 ? zc_env
                            : ((g.plane < (1 << 17) && ncol * ((g.nz + 1) / 2) >= 8 * full) ? 2 : 1);
  // 2-plane items end at plane zs1 (a multiple of 4); the last planes are
  // single-plane items, about 3 per block (FSG_K4_TAIL: that count, 0 = none).
  // The paired-load variant takes none: its single-plane items are unpaired
  // and the dynamic band phase already evens out the tail (c3 132.8 -> 130.0 us)
  static int tail_env = -2;
  if (tail_env == -2) {
    const char* e = getenv("FSG_K4_TAIL");
    tail_env = e ? atoi(e) : -1;
  }
  const int tail_n = tail_env >= 0 ? tail_env : (pair ? 0 : 3);
  int zs1 = g.nz;
  if (zc > 1) {
    const long long want = (tail_n * full + ncol - 1) / ncol;  // single planes
    zs1 = (int)std::max<long long>(0, ((g.nz - want) / 4) * 4);
  } else {
    zs1 = 0;
  }
  const long long nitem = ncol * (zs1 / zc) + ncol * (g.nz - zs1);
  const unsigned grid = (unsigned)std::min<long long>(nitem, full);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define FSG_PB(P, V, PR)                                                                     \
  cudaLaunchKernelEx(&cfg, k_collide_band<P, V, PR>, g, dp, (const float*)A, fb, sc, st, scr, \
                     scr_next, zc, zs1, so)
  if (pair) {
    if (pulled) {
      if (frame_on) FSG_PB(true, true, true);
      else FSG_PB(true, false, true);
    } else {
      if (frame_on) FSG_PB(false, true, true);
      else FSG_PB(false, false, true);
    }
  } else {
    if (pulled) {
      if (frame_on) FSG_PB(true, true, false);
      else FSG_PB(true, false, false);
    } else {
      if (frame_on) FSG_PB(false, true, false);
      else FSG_PB(false, false, false);
    }
  }
#undef FSG_PB
}
#endif

static const Launchers kLaunchers = {
    L_fill_rest,    L_set_f,          L_init_eq,      L_get_f,         L_macroscopic,
    L_collide,      L_session_force,  L_recenter,     L_markers,       L_spread,
#if FSG_PREC == 32
    L_markers_fix,  L_collide_fix,    L_collide_band, L_step_batch,
#else
    nullptr,        nullptr,          nullptr,        nullptr,
#endif
    L_halo_pack,    L_halo_unpack,    (int)sizeof(Store)};

}  // namespace p32 / p64
}  // namespace fsg
