// fsg_ib_fix.cuh -- throughput-mode immersed boundary (fp32 session), included
// inside namespace fsg::p32 after fsg_ib.cuh.
//
// One warp per marker does the whole reference chain of
// session.hpp:113-138 (position, bounds, stencil, bare moments of the
// stencil cells, interpolate_velocity, body velocity, direct forcing) and then
// SPREADS its own force: every stencil contribution w * f (coupling.hpp:52-71)
// is converted to 64-bit fixed point (2^-40) and added with an integer atomic.
// Integer addition is associative, so the accumulated field is bit-identical
// run to run whatever order the atomics land in -- deterministic without a
// separate ordered-spread kernel.  Touched 4^3 tiles are stamped first thing;
// the collide/stream pass reads (and re-zeroes) the force only in stamped
// tiles.  The interpolation sum uses a fixed warp butterfly (deterministic);
// the fp64 parity path keeps the reference's serial order instead
// (fsg_ib.cuh).
//
// The per-marker work is split into device functions (stencil, stamp, finish)
// so the kernel's block-level stamp / fence / trigger sequence stays visible.

#ifndef FSG_FX_LANES
#define FSG_FX_LANES 32
#endif
constexpr int FX_LANES = FSG_FX_LANES;     // lanes per marker (a warp or half a warp)
constexpr int FX_PER_BLOCK = 128 / FX_LANES;  // markers per 128-thread block

/// shuffle mask of this thread's marker group
__device__ __forceinline__ unsigned fx_mask() {
  return FX_LANES == 32 ? 0xFFFFFFFFu : (0xFFFFu << (threadIdx.x & 16));
}
#ifndef FSG_FX_CPL
#define FSG_FX_CPL 1
#endif
constexpr int FX_CPL = FSG_FX_CPL;  // stencil cells per lane per round trip (register pressure)

__device__ __forceinline__ unsigned long long to_fix(double v) {
  return (unsigned long long)__double2ll_rn(v * FIX_SCALE);
}

/// Marker t in the lattice: frame position, bounds check, stencil ranges.
struct MkStencil {
  double xf[3];         // frame position (m)
  double xl[3];         // lattice position
  int lo[3], hi[3], cnt[3];
  bool ok;              // marker_in_bounds (coupling.hpp:18-24)
};

/// From the world position x (SI).
__device__ __forceinline__ void mk_stencil_x(const double* x, const SessionConsts& sc,
                                             const StepConsts& st, MkStencil& S) {
  double xw[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) xw[k] = x[k] - st.p[k];
  mat_t_vec(st.R, xw, S.xf);
#pragma unroll
  for (int k = 0; k < 3; ++k) S.xl[k] = S.xf[k] / sc.dx + sc.hd[k];
  const double half = 0.5 * (sc.kernel == 0 ? 4 : 3);
  S.ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (S.xl[a] < half || S.xl[a] > sc.dims_g[a] - 1 - half) S.ok = false;
    S.lo[a] = (int)ceil(S.xl[a] - half);  // kernel.hpp:36-40
    S.hi[a] = (int)floor(S.xl[a] + half);
    S.cnt[a] = S.hi[a] - S.lo[a] + 1;
  }
}

__device__ __forceinline__ void mk_stencil(const Markers& mk, int t, const SessionConsts& sc,
                                           const StepConsts& st, MkStencil& S) {
  const double x[3] = {mk.pts[3 * t], mk.pts[3 * t + 1], mk.pts[3 * t + 2]};
  mk_stencil_x(x, sc, st, S);
}

/// Stamp the (<= 2x2x2: the stencil spans <= 5 cells) tiles the stencil touches.
__device__ __forceinline__ void mk_stamp(const Grid& g, const FixBand& fb, const MkStencil& S,
                                         int lane) {
  if (S.ok && lane < 8) {
    const int tx = ((lane & 1) ? S.hi[0] : S.lo[0]) >> 2;
    const int ty = ((lane & 2) ? S.hi[1] : S.lo[1]) >> 2;
    const int tz = ((lane & 4) ? S.hi[2] - g.z0 : S.lo[2] - g.z0) >> 2;
    fb.tflag[tx + fb.tnx * (ty + fb.tny * tz)] = fb.stamp;
  }
}

/// Stamp with the step's tile list (fb.tlist): the first stamp of a tile
/// this step appends it, so the banded K4's band phase takes the stamped
/// tiles dynamically from a list instead of scanning every tile's flag.
__device__ __forceinline__ void mk_stamp_list(const Grid& g, const FixBand& fb, const MkStencil& S,
                                              int lane, StepScratch* out) {
  if (S.ok && lane < 8) {
    const int tx = ((lane & 1) ? S.hi[0] : S.lo[0]) >> 2;
    const int ty = ((lane & 2) ? S.hi[1] : S.lo[1]) >> 2;
    const int tz = ((lane & 4) ? S.hi[2] - g.z0 : S.lo[2] - g.z0) >> 2;
    const int T = tx + fb.tnx * (ty + fb.tny * tz);
    if (atomicExch(fb.tflag + T, fb.stamp) != fb.stamp)
      fb.tlist[atomicAdd(&out->tcount, 1u)] = T;  // < 8 m <= list capacity
  }
}

/// End of the stamp phase of a marker block, then its dependents' trigger.
/// Every lane's stamps (and list entries) are ordered before the block
/// barrier; thread 0's fence + ticket carries them (causality order, PTX
/// memory model) to the grid's last block, whose release store of
/// `ready = stamp` the banded K4 acquires before its phase A reads a stamp.
/// Without a tile list (fb.ready null): barrier + fence only.
__device__ __forceinline__ void mk_publish_stamps(const FixBand& fb, StepScratch* out) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (fb.ready && atomicAdd(&out->ticket, 1u) == gridDim.x - 1) {
      __threadfence();
      st_release_gpu(fb.ready, fb.stamp);
    }
  }
  __syncthreads();
#ifndef FSG_KM_LATE_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;");
#endif
}

/// The rest of marker t's chain on one warp: phi, gathers + bare moments,
/// interpolation, forcing, the diagnostic record and the fixed-point spread.
/// phs: this warp's 15-double scratch in shared memory.
template <bool PULLED>
__device__ __forceinline__ void mk_finish(const Grid& g, const float* __restrict__ A, const Markers& mk,
                                          int t, int lane, const SessionConsts& sc, const StepConsts& st,
                                          const MkStencil& S, double (*phs)[5],
                                          MarkerStencil* __restrict__ rec_out, double* __restrict__ fworld,
                                          double* fworld_h, int* valid_h, const FixBand& fb,
                                          StepScratch* out, const double* vel_in = nullptr,
                                          const double* nrm_in = nullptr, double* fw_out = nullptr) {
  const unsigned full = fx_mask();
  const bool mkt_first = t == (int)(blockIdx.x * FX_PER_BLOCK + threadIdx.x / FX_LANES);
  (void)mkt_first;
  FSG_MKT(mkt_first, 5);
  if (!S.ok) {
    if (lane == 0) {
      rec_out[t].valid = 0;
      fworld[3 * t] = fworld[3 * t + 1] = fworld[3 * t + 2] = 0.0;
      if (fworld_h) {
        fworld_h[3 * t] = fworld_h[3 * t + 1] = fworld_h[3 * t + 2] = 0.0;
        valid_h[t] = 0;
      }
      atomicAdd(&out->oob, 1);
    }
    return;
  }
  if (lane < 15) {
    const int a = lane / 5, q = lane % 5;
    const int la = a == 0 ? S.lo[0] : (a == 1 ? S.lo[1] : S.lo[2]);
    const double xa = a == 0 ? S.xl[0] : (a == 1 ? S.xl[1] : S.xl[2]);
    const int ca = a == 0 ? S.cnt[0] : (a == 1 ? S.cnt[1] : S.cnt[2]);
    phs[a][q] = q < ca ? ib_phi(sc.kernel, (la + q) - xa) : 0.0;
  }
  __syncwarp(full);
  FSG_MKT(mkt_first, 6);
  const int ncell = S.cnt[0] * S.cnt[1] * S.cnt[2];
  const float r0 = 1.0f / (float)S.cnt[0], r01 = 1.0f / (float)(S.cnt[0] * S.cnt[1]);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  {
  // this lane's cells c = lane + 32 r: FX_CPL gathered per round trip
  for (int c0 = 0; c0 < ncell; c0 += FX_CPL * FX_LANES) {
    float sv[FX_CPL][Q];
    int cio[FX_CPL], cjo[FX_CPL], cko[FX_CPL];
#pragma unroll
    for (int r = 0; r < FX_CPL; ++r) {
      const int c = c0 + lane + FX_LANES * r;
      const int ko = (int)(((float)c + 0.5f) * r01);
      const int rem = c - ko * S.cnt[0] * S.cnt[1];
      const int jo = (int)(((float)rem + 0.5f) * r0);
      cio[r] = rem - jo * S.cnt[0];
      cjo[r] = jo;
      cko[r] = ko;
#ifndef FSG_KM_NO_GATHER  // dev attribution only (wrong results)
      if (c < ncell) gather_cell<PULLED>(g, A, S.lo[0] + cio[r], S.lo[1] + jo, S.lo[2] + ko - g.z0, sv[r]);
#else
      for (int i = 0; i < Q; ++i) sv[r][i] = 0.f;
#endif
    }
#pragma unroll
    for (int r = 0; r < FX_CPL; ++r) {
      const int c = c0 + lane + FX_LANES * r;
      if (c < ncell) {
        float drho, mx, my, mz;
        moments_dev(sv[r], drho, mx, my, mz);
        const float rho = 1.0f + drho;
        const float ir = rho > 0.0f ? 1.0f / rho : 0.0f;  // bare u; 0 where rho <= 0
        const double w = (phs[2][cko[r]] * phs[1][cjo[r]]) * phs[0][cio[r]];
        a0 += w * (double)(mx * ir);
        a1 += w * (double)(my * ir);
        a2 += w * (double)(mz * ir);
      }
    }
  }
  }
  FSG_MKT(mkt_first, 7);
#pragma unroll
  for (int o = FX_LANES / 2; o > 0; o >>= 1) {  // fixed butterfly: every lane gets the total
    a0 += __shfl_xor_sync(full, a0, o);
    a1 += __shfl_xor_sync(full, a1, o);
    a2 += __shfl_xor_sync(full, a2, o);
  }
  FSG_MKT(mkt_first, 8);
  // body velocity, direct forcing, world force (identical on every lane);
  // the rest of the marker state is loaded only now (register pressure)
  const double uf[3] = {a0 * sc.v2p, a1 * sc.v2p, a2 * sc.v2p};
  double vel[3], nrm[3], vw[3], vf[3], nf[3], fl[3], fw[3], ff[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    vel[k] = vel_in ? vel_in[k] : mk.vel[3 * t + k];
    nrm[k] = nrm_in ? nrm_in[k] : mk.nrm[3 * t + k];
  }
  const double area = mk.area[t];
#pragma unroll
  for (int k = 0; k < 3; ++k) vw[k] = vel[k] - st.pd[k];
  mat_t_vec(st.R, vw, vf);
  const double* xf = S.xf;
  double du[3] = {vf[0] - (st.wf[1] * xf[2] - st.wf[2] * xf[1]) - uf[0],
                  vf[1] - (st.wf[2] * xf[0] - st.wf[0] * xf[2]) - uf[1],
                  vf[2] - (st.wf[0] * xf[1] - st.wf[1] * xf[0]) - uf[2]};
  mat_t_vec(st.R, nrm, nf);
  if (sc.wall == 0) {
    const double s = du[0] * nf[0] + du[1] * nf[1] + du[2] * nf[2];
    du[0] = s * nf[0];
    du[1] = s * nf[1];
    du[2] = s * nf[2];
  }
  const double kf = sc.rho_phys * area * sc.dx / sc.dt;
  fl[0] = kf * du[0];
  fl[1] = kf * du[1];
  fl[2] = kf * du[2];
  mat_vec(st.R, fl, fw);
  mat_t_vec(st.R, fw, ff);
  const double fx = ff[0] * sc.f2l, fy = ff[1] * sc.f2l, fz = ff[2] * sc.f2l;
  if (fw_out) {
    fw_out[0] = fw[0];
    fw_out[1] = fw[1];
    fw_out[2] = fw[2];
  }
  if (lane == 0) {
    fworld[3 * t] = fw[0];
    fworld[3 * t + 1] = fw[1];
    fworld[3 * t + 2] = fw[2];
    if (fworld_h) {
      fworld_h[3 * t] = fw[0];
      fworld_h[3 * t + 1] = fw[1];
      fworld_h[3 * t + 2] = fw[2];
      valid_h[t] = 1;
    }
    MarkerStencil r;  // kept for diagnostics (fsg_get_force / fsg_get_stencils)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
#pragma unroll
      for (int q = 0; q < 5; ++q) r.ph[a][q] = phs[a][q];
      r.lo[a] = S.lo[a];
      r.hi[a] = S.hi[a];
    }
    r.fl[0] = fx;
    r.fl[1] = fy;
    r.fl[2] = fz;
    r.valid = 1;
    r._pad = 0;
    rec_out[t] = r;
  }
  FSG_MKT(mkt_first, 9);
  // spread: this lane's own cells, fixed-point integer atomics
  for (int c = lane; c < ncell; c += FX_LANES) {
    const int ko = (int)(((float)c + 0.5f) * r01);
    const int rem = c - ko * S.cnt[0] * S.cnt[1];
    const int jo = (int)(((float)rem + 0.5f) * r0);
    const int io = rem - jo * S.cnt[0];
    const double w = (phs[2][ko] * phs[1][jo]) * phs[0][io];
    const long long cell = (long long)(S.lo[0] + io) +
                           (long long)g.nx * ((long long)(S.lo[1] + jo) + (long long)g.ny * (S.lo[2] + ko - g.z0));
    unsigned long long* F = fb.F + 3 * cell;
#ifndef FSG_KM_NO_SPREAD  // dev attribution only (wrong results)
    atomicAdd(F, to_fix(w * fx));
    atomicAdd(F + 1, to_fix(w * fy));
    atomicAdd(F + 2, to_fix(w * fz));
#else
    if (w * fx == 12345.0) atomicAdd(F, 1ull);
#endif
  }
}

/// Standalone marker kernel: a programmatic primary of the banded K4.
/// Persistent over the markers (grid capped by the host, L_markers_fix): each
/// warp first stamps the tiles of ALL its markers, the block fences and only
/// then triggers its dependents, before the slow part.  Fewer marker blocks
/// leave more of every SM to the concurrent phase A of K4 (the marker chain is
/// off the critical path while phase A runs).
template <bool PULLED>
__global__ void __launch_bounds__(128, FSG_KM_MINB)
    k_markers_fix(Grid g, const float* __restrict__ A, Markers mk, const SessionConsts* __restrict__ scp,
                  const StepConsts st, MarkerStencil* __restrict__ rec_out, double* __restrict__ fworld,
                  double* fworld_h, int* valid_h, FixBand fb, StepScratch* out, unsigned* km_done) {
  __shared__ double phs[FX_PER_BLOCK][3][5];
  const int lane = threadIdx.x & (FX_LANES - 1);
  const int slot = threadIdx.x / FX_LANES;
  const int stride = gridDim.x * FX_PER_BLOCK;
  const SessionConsts& sc = *scp;
  // skinned bodies: launched as a programmatic dependent of the skinning
  // kernel (its launch latency overlaps it); wait for the marker state.  A
  // no-op for an ordinary launch.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) FSG_TL(fb.stamp, 0);  // timeline (dev build): marker kernel start
  for (int t = blockIdx.x * FX_PER_BLOCK + slot; t < mk.m; t += stride) {
    MkStencil S;
    mk_stencil(mk, t, sc, st, S);
    if (fb.tlist) mk_stamp_list(g, fb, S, lane, out);
    else mk_stamp(g, fb, S, lane);
  }
  // every warp's stamps are published before this block lets the banded K4
  // (programmatic dependent) launch: K4's first phase skips stamped tiles and
  // waits for this grid's completion before updating them
  mk_publish_stamps(fb, out);
  for (int t = blockIdx.x * FX_PER_BLOCK + slot; t < mk.m; t += stride) {
    MkStencil S;
    mk_stencil(mk, t, sc, st, S);  // cheap; recomputed rather than kept in registers
    mk_finish<PULLED>(g, A, mk, t, lane, sc, st, S, phs[slot], rec_out, fworld, fworld_h, valid_h, fb,
                      out);
    __syncwarp(fx_mask());  // phs[slot] is reused by the group's next marker
  }
  if (lane == 0) FSG_TL(fb.stamp, 1);  // last marker warp done
  if (km_done) {  // this block's forces and validity flags are complete
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(km_done, 1u);
    }
  }
}

#include "fsg_skin_fused.cuh"

/// The marker kernel for skinned bodies (fsg_set_skin, up to two): each warp
/// skins its marker from the pose (launch parameter) before stamping, skins
/// velocity and normal before the forcing, and adds the marker's tau_ext
/// terms and stats to the warp's running sums; the block tail reduces them
/// (fsg_skin_fused.cuh).  Same stamp / fence / trigger protocol as
/// k_markers_fix.
template <bool PULLED, int NB>
__global__ void __launch_bounds__(128, FSG_KM_MINB)
    k_markers_skin(Grid g, const float* __restrict__ A, Markers mk, const SessionConsts* __restrict__ scp,
                   const StepConsts st, MarkerStencil* __restrict__ rec_out, double* __restrict__ fworld,
                   double* fworld_h, int* valid_h, FixBand fb, StepScratch* out,
                   const __grid_constant__ SkinParamsN<NB> P, unsigned long long* fixacc) {
  __shared__ double phs[FX_PER_BLOCK][3][5];
  // the bodies' topology and this step's pose, staged once per block after
  // the trigger: the heavy phase indexes them by lane-dependent bone / joint,
  // which in the kernel parameter space (constant bank) serializes per
  // distinct address.  The stamp phase reads its (<= 4 distinct) bone
  // transforms straight from the parameters, so the staging (~3-4 us per
  // block) is off the path to K4's launch.
  __shared__ __align__(16) SkinBody sbody[NB];
  FSG_MKT(true, 0);
  __syncthreads();
  FSG_MKT(true, 1);
  const int lane = threadIdx.x & (FX_LANES - 1);
  const int slot = threadIdx.x / FX_LANES;
  const int stride = gridDim.x * FX_PER_BLOCK;
  const SessionConsts& sc = *scp;
  // the stencil of the group's last stamped marker, reused after the trigger
  // (one marker per group in the default single-wave grid)
  __shared__ MkStencil s_st[FX_PER_BLOCK];
  __shared__ int s_t[FX_PER_BLOCK];
  if (lane == 0) s_t[slot] = -1;
  if (threadIdx.x == 0) FSG_TL(fb.stamp, 0);
  for (int t = blockIdx.x * FX_PER_BLOCK + slot; t < mk.m; t += stride) {
    const SkinSlot sl = skin_slot(P, t, lane);
    double xw[3];
    skin_point_warp(P, P.body[skin_body_of(P, t)].pose, t, sl, xw);
    if (lane == 0) {
      double* pts = const_cast<double*>(mk.pts);
      pts[3 * t] = xw[0];
      pts[3 * t + 1] = xw[1];
      pts[3 * t + 2] = xw[2];
    }
    MkStencil S;
    mk_stencil_x(xw, sc, st, S);
    if (fb.tlist) mk_stamp_list(g, fb, S, lane, out);
    else mk_stamp(g, fb, S, lane);
    if (lane == 0) {
      s_st[slot] = S;
      s_t[slot] = t;
    }
  }
  FSG_MKT(true, 2);
  mk_publish_stamps(fb, out);
  FSG_MKT(true, 3);
  skin_stage_bodies(P, sbody);
  double acc[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) acc[b] = 0.0;
  // the heavy loop runs the group's markers last-stamped first, so the first
  // one reuses the stencil cached by the stamp phase
  const int t_first = blockIdx.x * FX_PER_BLOCK + slot;
  const int t_last = t_first < mk.m ? t_first + stride * ((mk.m - 1 - t_first) / stride) : -1;
  for (int t = t_last; t >= t_first; t -= stride) {
    const int bi = skin_body_of(P, t);
    const SkinBody& B = sbody[bi];
    const SkinSlot sl = skin_slot(P, t, lane);
    double vel[3], nrm[3], fw[3], xb[3] = {0.0, 0.0, 0.0};
    skin_vel_nrm_warp(P, B.pose, t, sl, vel, nrm, xb);
    FSG_MKT(t == t_last, 4);
    MkStencil S;
    if (s_t[slot] == t) {
      S = s_st[slot];  // lane 0's copy from the stamp phase (the block barrier since orders it)
    } else {
      // the position this warp skinned before the stamps (the block barrier
      // since orders lane 0's store before these loads)
      double xw[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) xw[c] = __ldcg(mk.pts + 3 * t + c);
      mk_stencil_x(xw, sc, st, S);
    }
    if (lane == 0) {
      double* v = const_cast<double*>(mk.vel);
      double* n = const_cast<double*>(mk.nrm);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        v[3 * t + c] = vel[c];
        n[3 * t + c] = nrm[c];
      }
    }
    mk_finish<PULLED>(g, A, mk, t, lane, sc, st, S, phs[slot], rec_out, fworld, fworld_h, valid_h, fb,
                      out, vel, nrm, fw);
    __syncwarp(fx_mask());
    FSG_MKT(t == t_last, 10);
#ifndef FSG_SKIN_NO_TAU
    if (S.ok) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (b == bi) skin_tau_pre(B, lane, sl, xb, fw, vel, acc[b]);
    }
#endif
    FSG_MKT(t == t_last, 11);
  }
  FSG_MKT(true, 12);
  if (lane == 0) FSG_TL(fb.stamp, 1);
#ifndef FSG_SKIN_NO_TAIL
  skin_block_red(acc, fixacc);
#endif
  FSG_MKT(true, 13);
}

