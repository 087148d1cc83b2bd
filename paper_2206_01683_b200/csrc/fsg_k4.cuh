// fsg_k4.cuh -- throughput K4 (fp32 deviations), included inside namespace
// fsg::p32.  One cell per thread; the 19 pull sources and 19 destinations are
// addressed through per-direction base pointers passed as kernel parameters
// (constant bank), so each access costs one LDC + one IMAD.WIDE instead of a
// runtime 64-bit index product.  Interior cells use the constant neighbour
// offsets folded into those pointers; boundary cells take the generic
// clamped/periodic gather (solver.hpp:59-97 re-expressed as a pull).

// DirPtrs (fsg_device.cuh): per-direction base pointers A + pull[i] / B + own[i]

// load / store flavour of the fast-path populations (dev A/B: FSG_K4_CS=1
// streaming .cs hints, evict-first in L2)
#if FSG_K4_CS
#define K4_LD(p) __ldcs(p)
#define K4_ST(p, v) __stcs((p), (v))
#else
#define K4_LD(p) __ldg(p)
#define K4_ST(p, v) (*(p) = (v))
#endif

template <int FMODE, bool VF>
__global__ void __launch_bounds__(128)
    k_collide_fast(Grid g, DirPtrs dp, const float* __restrict__ A, const float* __restrict__ Fext,
                   Band band, const StepScratch* __restrict__ bscr,
                   const SessionConsts* __restrict__ scp, const StepConsts* __restrict__ stp,
                   StepScratch* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int z = blockIdx.z;
  float vmin = FLT_MAX;
  if (x < g.nx && y < g.ny) {
    const unsigned m = (unsigned)mem_index(g, x, y, z);
    float s[Q];
    if (is_interior(g, x, y, z)) {
#pragma unroll
      for (int i = 0; i < Q; ++i) s[i] = __ldg(dp.a[i] + m);
    } else {
      gather<true>(g, A, x, y, z, s);
    }
    float Fx = 0.f, Fy = 0.f, Fz = 0.f;
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
             (long long)(hi[0] - lo[0] + 1) *
                 ((long long)(y - lo[1]) + (long long)(hi[1] - lo[1] + 1) * (z - lo[2]));
    }
    vmin = collide_cell32<FMODE, VF>(s, x, y, z, g, Fx, Fy, Fz, in_band, lc, band, *scp, *stp, out);
#pragma unroll
    for (int i = 0; i < Q; ++i) dp.b[i][m] = s[i];
  }
  report_min(out, vmin == FLT_MAX ? DBL_MAX : (double)vmin);
}

/// One cell: pull gather (x faces on the fast path; FACE: open y/z face rows
/// too), collide, store.  The banded K4 keeps FACE off: at 64 registers the
/// extra path spills and the coupled step measured slower (c3 143 vs 141 us),
/// while the fluid K4 gains (c1 15.9 -> 13.8 us, c2 22.5 -> 20.5 us).
template <bool PULLED, bool VF, bool FACE = false>
__device__ __forceinline__ float cell_update(const Grid& g, const DirPtrs& dp,
                                             const float* __restrict__ A, int x, int y, int z,
                                             float Fx, float Fy, float Fz,
                                             const SessionConsts& sc, const StepConsts& st,
                                             StepScratch* out, float* fcap = nullptr,
                                             PeerOut po = PeerOut{nullptr, nullptr}) {
  const unsigned m = (unsigned)mem_index(g, x, y, z);
  const int zg = g.z0 + z;
  float s[Q];
  if (!PULLED) {
#pragma unroll
    for (int i = 0; i < Q; ++i) s[i] = __ldg(dp.a[i] + m);
  } else if (y > 0 && y < g.ny - 1 && zg > 0 && zg < g.nzg - 1) {
    // x faces stay on the fast path: the pull source of an unknown population
    // moves by +-1 (open: clamped copy, solver.hpp:59-97) or +-nx (periodic)
    const int cxp = x == 0 ? (g.periodic ? g.nx : 1) : 0;
    const int cxm = x == g.nx - 1 ? (g.periodic ? -g.nx : -1) : 0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const int cx = ex_of(i) > 0 ? cxp : (ex_of(i) < 0 ? cxm : 0);
      s[i] = K4_LD(dp.a[i] + (m + cx));
    }
  } else if (FACE && !g.periodic) {
    // open y/z face rows (warp-uniform): unknown populations shifted by the
    // cell's clamp displacement, still constant offsets (FaceFlags)
    const FaceFlags f = face_flags(g, x, y, zg);
#pragma unroll
    for (int i = 0; i < Q; ++i)
      s[i] = __ldg(dp.a[i] + (m + (face_unknown(ex_of(i), ey_of(i), ez_of(i), f) ? f.D : 0)));
  } else {
    gather<true>(g, A, x, y, z, s);  // y/z face rows (warp-uniform)
  }
  Band none{nullptr, 0};
  const float v = collide_cell32<3, VF>(s, x, y, z, g, Fx, Fy, Fz, false, 0, none, sc, st, out, fcap,
                                        (long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z));
#pragma unroll
  for (int i = 0; i < Q; ++i) K4_ST(dp.b[i] + m, s[i]);
  // peer-connected slab: the crossing populations of the boundary planes go
  // straight into the neighbours' halo planes (lattice.hpp:25-26: ez = -1
  // {6,12,13,16,17}, ez = +1 {5,11,14,15,18})
  if (po.lo && z == 0) {
    float* d = po.lo + (x + (long long)g.nx * y);
    d[6 * g.stride] = s[6];
    d[12 * g.stride] = s[12];
    d[13 * g.stride] = s[13];
    d[16 * g.stride] = s[16];
    d[17 * g.stride] = s[17];
  }
  if (po.hi && z == g.nz - 1) {
    float* d = po.hi + (x + (long long)g.nx * y);
    d[5 * g.stride] = s[5];
    d[11 * g.stride] = s[11];
    d[14 * g.stride] = s[14];
    d[15 * g.stride] = s[15];
    d[18 * g.stride] = s[18];
  }
  return v;
}

/// Two cells of one column, planes z and z + 1, both with y and z interior
/// (pulled state, no IB force): all 38 pull loads are issued before either
/// cell collides, so a warp keeps twice the bytes in flight (c3 coupled step
/// 138.2 -> 134.9 us at 80 registers / 6 blocks per SM; at 64 registers the
/// pair spills and is slower).
/// Same per-cell arithmetic as cell_update (bit-identical).
template <bool VF>
__device__ __forceinline__ float cell_update_pair(const Grid& g, const DirPtrs& dp, int x, int y, int z,
                                                  const SessionConsts& sc, const StepConsts& st,
                                                  StepScratch* out, float* fcap) {
  const unsigned m0 = (unsigned)mem_index(g, x, y, z);
  const unsigned m1 = m0 + (unsigned)g.zs;
  const int cxp = x == 0 ? (g.periodic ? g.nx : 1) : 0;
  const int cxm = x == g.nx - 1 ? (g.periodic ? -g.nx : -1) : 0;
  float s0[Q], s1[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int cx = ex_of(i) > 0 ? cxp : (ex_of(i) < 0 ? cxm : 0);
    s0[i] = __ldg(dp.a[i] + (m0 + cx));
    s1[i] = __ldg(dp.a[i] + (m1 + cx));
  }
  Band none{nullptr, 0};
  const long long c0 = (long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z);
  const float v0 = collide_cell32<3, VF>(s0, x, y, z, g, 0.f, 0.f, 0.f, false, 0, none, sc, st, out, fcap, c0);
#pragma unroll
  for (int i = 0; i < Q; ++i) dp.b[i][m0] = s0[i];
  const float v1 = collide_cell32<3, VF>(s1, x, y, z + 1, g, 0.f, 0.f, 0.f, false, 0, none, sc, st, out, fcap,
                                        c0 + g.plane);
#pragma unroll
  for (int i = 0; i < Q; ++i) dp.b[i][m1] = s1[i];
  return fminf(v0, v1);
}

/// NP cells of one column (planes z .. z + NP - 1, all y/z-interior), every
/// pull load issued before any cell collides (generalises cell_update_pair).
template <bool VF, int NP>
__device__ __forceinline__ float cell_update_multi(const Grid& g, const DirPtrs& dp, int x, int y, int z,
                                                   const SessionConsts& sc, const StepConsts& st,
                                                   StepScratch* out, float* fcap) {
  const unsigned m0 = (unsigned)mem_index(g, x, y, z);
  const int cxp = x == 0 ? (g.periodic ? g.nx : 1) : 0;
  const int cxm = x == g.nx - 1 ? (g.periodic ? -g.nx : -1) : 0;
  float s[NP][Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int cx = ex_of(i) > 0 ? cxp : (ex_of(i) < 0 ? cxm : 0);
#pragma unroll
    for (int k = 0; k < NP; ++k) s[k][i] = __ldg(dp.a[i] + (m0 + (unsigned)(k * g.zs) + cx));
  }
  Band none{nullptr, 0};
  const long long c0 = (long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z);
  float v = FLT_MAX;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    v = fminf(v, collide_cell32<3, VF>(s[k], x, y, z + k, g, 0.f, 0.f, 0.f, false, 0, none, sc, st, out,
                                       fcap, c0 + k * g.plane));
#pragma unroll
    for (int i = 0; i < Q; ++i) dp.b[i][m0 + (unsigned)(k * g.zs)] = s[k][i];
  }
  return v;
}

/// Block 0 zeroes the next step's scratch (status + work counters).  Nothing
/// is published from the kernel: the host copies the status out of the
/// device scratch when it asks for it, after a stream sync, so the kernel
/// needs no last-block detection and no system-scope fence on its tail.
__device__ __forceinline__ void reset_next(StepScratch* next, int tid) {
  constexpr int NS = (int)(sizeof(StepScratch) / 4);
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid < NS)
    reinterpret_cast<int*>(next)[tid] = 0;
}

// Pure-fluid K4 of the throughput session (no IB band): virtual force inline,
// collide/stream.  Persistent: work item = (xy column, chunk of zc planes)
// over the planes z = zr.lo + q * zr.step < zr.hi (all planes; or, in a z-slab
// step, the two boundary planes first and the interior behind the halo send).
struct ZRange {
  int lo, hi, step;
};

template <bool PULLED, bool VF>
__global__ void __launch_bounds__(128, FSG_K4_MINB)
    k_collide_fix(Grid g, DirPtrs dp, const float* __restrict__ A,
                  const SessionConsts* __restrict__ scp, const StepConsts st,
                  StepScratch* __restrict__ out, StepScratch* __restrict__ next, int zc, ZRange zr,
                  PeerOut po) {
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  reset_next(next, tid);
  const int tx_n = (g.nx + blockDim.x - 1) / blockDim.x;
  const int ty_n = (g.ny + blockDim.y - 1) / blockDim.y;
  const int nq = (zr.hi - zr.lo + zr.step - 1) / zr.step;
  const int ncol = tx_n * ty_n, nzc = (nq + zc - 1) / zc;
  const int nitem = ncol * nzc;
  const SessionConsts& sc = *scp;
  float vmin = FLT_MAX;
  for (int it = blockIdx.x; it < nitem; it += gridDim.x) {
    const int col = it % ncol, zk = it / ncol;
    const int x = (col % tx_n) * blockDim.x + threadIdx.x;
    const int y = (col / tx_n) * blockDim.y + threadIdx.y;
    const int q0 = zk * zc, q1 = min(nq, q0 + zc);
    if (x >= g.nx || y >= g.ny) continue;
#ifdef FSG_K4F_PAIR  // dev A/B: 512^3 3.77 -> 3.70 ms at 2-plane items, but c3 104 -> 111 us, and
                     // a runtime switch alone (path compiled in) slowed every grid 2-10 %
    if (PULLED && q1 - q0 == 2 && zr.step == 1 && !po.lo && !po.hi && y > 0 && y < g.ny - 1) {
      const int z = zr.lo + q0;
      if (g.z0 + z > 0 && g.z0 + z + 1 < g.nzg - 1) {
        vmin = fminf(vmin, cell_update_pair<VF>(g, dp, x, y, z, sc, st, out, nullptr));
        continue;
      }
    }
#endif
    for (int q = q0; q < q1; ++q)
      vmin = fminf(vmin, cell_update<PULLED, VF, true>(g, dp, A, x, y, zr.lo + q * zr.step, 0.f, 0.f,
                                                       0.f, sc, st, out, nullptr, po));
  }
  report_min(out, vmin == FLT_MAX ? DBL_MAX : (double)vmin);
}

// ---------------------------------------------------------------------------
// Banded coupled K4 (one launch per step).  Launched on the session stream as
// a programmatic dependent of the marker kernel, whose blocks stamp the 4^3
// tiles their stencils touch, fence, and only then trigger their dependents
// -- before their slow part (gathers, forcing, spread).  So K4 starts while
// the markers still run, with every stamp of this step visible, and
//   phase A  updates every cell outside the stamped tiles (no IB force), with
//            dynamic work fetch (prefetched one item ahead) so blocks that
//            land late on SMs freed by the marker kernel take less;
//   phase B  waits for the marker grid (griddepcontrol.wait: completion +
//            memory visibility) and updates the stamped tiles with the fresh
//            fixed-point IB force, found by an interleaved scan of the stamps.
// Each cell is written exactly once per step.

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// PAIR (grids larger than L2): 80 registers / 6 blocks per SM and paired
// phase-A loads; else 64 registers / 8 blocks, one cell at a time (the pair
// variant measured slower on the L2-resident c2: 45.7 vs 42.9 us)
template <bool PULLED, bool VF, bool PAIR>
__global__ void __launch_bounds__(128, PAIR ? FSG_K4B_MINB_PAIR : FSG_K4B_MINB)
    k_collide_band(Grid g, DirPtrs dp, const float* __restrict__ A, FixBand fb,
                   const SessionConsts* __restrict__ scp, const StepConsts st,
                   StepScratch* __restrict__ out, StepScratch* __restrict__ next, int zc,
                   int zs1, SkinOut so) {
  __shared__ int item;
  __shared__ int tl[128];
  __shared__ int ntl;
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  // a programmatic dependent (the skinned bodies' tau reduction) may start now:
  // it waits on the marker kernel, not on this one
  asm volatile("griddepcontrol.launch_dependents;");
  reset_next(next, tid);
  const SessionConsts& sc = *scp;
  const int tx_n = (g.nx + blockDim.x - 1) / blockDim.x;
  const int ty_n = (g.ny + blockDim.y - 1) / blockDim.y;
  // items: zc-plane items over planes [0, zs1), then single-plane items over
  // [zs1, nz) -- the queue ends with short items, so the blocks' phase-A
  // finishing times spread by half an item less (an item's cells are one per
  // thread per plane; under full HBM load a 2-plane item takes ~7 us at c3)
  const int ncol = tx_n * ty_n;
  const int nbig = ncol * (zs1 / zc);
  const int nitem = nbig + ncol * (g.nz - zs1);
  int nxt = 0;
  if (tid == 0) {
    // phase A may read the stamps once every tile of this step is stamped:
    // acquire of the marker grid's release (normally set before K4 starts)
    if (fb.ready)
      while (ld_acquire_gpu(fb.ready) != fb.stamp) __nanosleep(64);
    nxt = (int)atomicAdd(&out->work, 1u);
    FSG_TL(fb.stamp, 2);  // timeline (dev build): K4 start
#ifdef FSG_TIMING
    if (blockIdx.x < 8192) {
      g_blk[4 * blockIdx.x] = tl_now();
      g_blk[4 * blockIdx.x + 3] = smid_();
    }
#endif
  }
#ifdef FSG_TIMING
  unsigned n_items = 0;
#endif
  // ---- phase A: cells outside the stamped tiles (no IB force), per-block fetch
  float vmin = FLT_MAX;
  for (;;) {
    if (tid == 0) item = nxt;
    __syncthreads();
    const int it = item;
    __syncthreads();
    if (it >= nitem) break;
#ifdef FSG_TIMING
    ++n_items;
#endif
    if (tid == 0) nxt = (int)atomicAdd(&out->work, 1u);  // consumed next iteration
    const bool big = it < nbig;
    const int r = big ? it : it - nbig;
    const int col = r % ncol;
    const int x = (col % tx_n) * blockDim.x + threadIdx.x;
    const int y = (col / tx_n) * blockDim.y + threadIdx.y;
    const int z0 = big ? (r / ncol) * zc : zs1 + r / ncol;
    const int z1 = big ? z0 + zc : z0 + 1;
    if (x >= g.nx || y >= g.ny) continue;
    // the item's planes (1 or 2, zs1 a multiple of 4) share a tile layer:
    // one stamp load per item (stamped: the band phase's)
    if (__ldcg(fb.tflag + (x >> 2) + fb.tnx * ((y >> 2) + fb.tny * (z0 >> 2))) == fb.stamp) continue;
#ifndef FSG_K4_NO_PAIR
#ifndef FSG_K4_NP
#define FSG_K4_NP 2
#endif
    if (PAIR && PULLED && z1 - z0 == FSG_K4_NP && y > 0 && y < g.ny - 1 && g.z0 + z0 > 0 &&
        g.z0 + z1 < g.nzg) {
      if (FSG_K4_NP == 2)
        vmin = fminf(vmin, cell_update_pair<VF>(g, dp, x, y, z0, sc, st, out, fb.fcap));
      else
        vmin = fminf(vmin, cell_update_multi<VF, FSG_K4_NP>(g, dp, x, y, z0, sc, st, out, fb.fcap));
      continue;
    }
#endif
    for (int z = z0; z < z1; ++z)
      vmin = fminf(vmin, cell_update<PULLED, VF>(g, dp, A, x, y, z, 0.f, 0.f, 0.f, sc, st, out,
                                                 fb.fcap));
  }
  // ---- phase B: the stamped tiles, after the marker grid completed.  Block b
  // scans tiles b, b + G, b + 2G ... (G = gridDim.x), one per thread per
  // chunk, so a body's clustered tiles spread over all blocks; each 64
  // threads take one stamped tile per pass.
  if (tid == 0) FSG_TL(fb.stamp, 3);  // phase A done (this block)
#ifdef FSG_TIMING
  if (tid == 0 && blockIdx.x < 8192) {
    g_blk[4 * blockIdx.x + 1] = tl_now();
    g_blk[4 * blockIdx.x + 2] = n_items;
  }
#endif
  pdl_wait();
  if (tid == 0) FSG_TL(fb.stamp, 4);  // band phase start
  // skinned bodies: the marker grid's tau_ext / stats sums are complete
  if (so.acc && blockIdx.x == gridDim.x - 1 && tid < so.nb * 32) {
    const int b = tid >> 5, c = tid & 31;
    long long v = 0;  // the SKIN_FIX_REP copies, summed as integers (wraps alike)
#pragma unroll 4
    for (int r = 0; r < SKIN_FIX_REP; ++r) v += (long long)__ldcg(so.acc + 64 * r + tid);
    const bool bad = __shfl_sync(0xffffffffu, v, 31) != 0;  // slot 31: non-finite flag
#pragma unroll 4
    for (int r = 0; r < SKIN_FIX_REP; ++r) so.acc[64 * r + tid] = 0ull;
    const double d = bad ? __longlong_as_double(0x7ff8000000000000ll) : (double)v * SKIN_FIX_INV;
    if (c < so.ndof[b]) so.out[so.off[b] + c] = d;
    if (c >= SKIN_TAU_MAX && c < SKIN_TAU_MAX + SKIN_NSTAT)
      so.out[so.nt + SKIN_NSTAT * b + (c - SKIN_TAU_MAX)] = d;
  }
  const int ntile = fb.tnx * fb.tny * fb.tnz;
  const int nthr = blockDim.x * blockDim.y;  // 96 or 128 (cell_block)
  const int tpp = nthr >> 6;                 // tiles per pass (64 threads each)
  const int half = tid >> 6, lt = tid & 63;
  if (fb.tlist) {
    // tile list: the step's stamped tiles are listed; blocks take them
    // dynamically, so blocks out of phase A early take more of the band
    const unsigned nt = __ldcg(&out->tcount);
    for (;;) {
      if (tid == 0) item = (int)atomicAdd(&out->bwork, (unsigned)tpp);
      __syncthreads();
      const unsigned k = (unsigned)item + (unsigned)half;
      const bool more = (unsigned)item < nt;
      __syncthreads();
      if (!more) break;
      if (half >= tpp || k >= nt) continue;
      const int T = __ldcg(fb.tlist + k);
      const int tx = T % fb.tnx, ty = (T / fb.tnx) % fb.tny, tz = T / (fb.tnx * fb.tny);
      const int x = 4 * tx + (lt & 3), y = 4 * ty + ((lt >> 2) & 3), z = 4 * tz + (lt >> 4);
      if (x >= g.nx || y >= g.ny || z >= g.nz) continue;
      unsigned long long* F = fb.F + 3 * ((long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z));
      const long long f0 = (long long)F[0], f1 = (long long)F[1], f2 = (long long)F[2];
      F[0] = 0ull;
      F[1] = 0ull;
      F[2] = 0ull;
      const float Fx = (float)((double)f0 * FIX_INV);
      const float Fy = (float)((double)f1 * FIX_INV);
      const float Fz = (float)((double)f2 * FIX_INV);
      vmin = fminf(vmin, cell_update<PULLED, VF>(g, dp, A, x, y, z, Fx, Fy, Fz, sc, st, out, fb.fcap));
    }
  } else {
  for (int base = 0; (long long)base * gridDim.x < ntile; base += nthr) {
    if (tid == 0) ntl = 0;
    __syncthreads();
    const long long T0 = (long long)blockIdx.x + (long long)gridDim.x * (base + tid);
    if (T0 < ntile && fb.tflag[T0] == fb.stamp) tl[atomicAdd(&ntl, 1)] = (int)T0;
    __syncthreads();
    const int n = half < tpp ? ntl : 0;
    for (int k = half; k < n; k += tpp) {
      const int T = tl[k];
      const int tx = T % fb.tnx, ty = (T / fb.tnx) % fb.tny, tz = T / (fb.tnx * fb.tny);
      const int x = 4 * tx + (lt & 3), y = 4 * ty + ((lt >> 2) & 3), z = 4 * tz + (lt >> 4);
      if (x >= g.nx || y >= g.ny || z >= g.nz) continue;
      // consume and re-zero the fixed-point force
      unsigned long long* F = fb.F + 3 * ((long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z));
      const long long f0 = (long long)F[0], f1 = (long long)F[1], f2 = (long long)F[2];
      F[0] = 0ull;
      F[1] = 0ull;
      F[2] = 0ull;
      const float Fx = (float)((double)f0 * FIX_INV);
      const float Fy = (float)((double)f1 * FIX_INV);
      const float Fz = (float)((double)f2 * FIX_INV);
      vmin = fminf(vmin, cell_update<PULLED, VF>(g, dp, A, x, y, z, Fx, Fy, Fz, sc, st, out, fb.fcap));
    }
    __syncthreads();
  }
  }
  report_min(out, vmin == FLT_MAX ? DBL_MAX : (double)vmin);
  if (tid == 0) FSG_TL(fb.stamp, 5);  // K4 end
}
