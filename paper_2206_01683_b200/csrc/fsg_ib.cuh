// fsg_ib.cuh -- immersed-boundary kernels (included inside the precision
// namespace of fsg_kernels.cuh; uses its Store/gather/cell_moments helpers).
//
// K_m  (k_markers, one warp per marker) fuses, for one marker:
//   world -> frame -> lattice position       frame.hpp:24-26, session.hpp:82-85
//   marker_in_bounds                         coupling.hpp:18-24
//   stencil ranges + per-axis phi            kernel.hpp:22-40
//   bare moments of the stencil cells        solver.hpp:25-51 with F = 0 (session.hpp:95-96)
//   interpolate_velocity                     coupling.hpp:27-48
//   body_velocity_to_frame, direct_forcing   frame.hpp:39-42, coupling.hpp:80-85
//   world force + lattice force to spread    session.hpp:124-138
// The stencil cells are gathered by the 32 lanes in parallel; the products
// w * u_cell land in shared memory and one lane sums them in the reference's
// k, j, i order, so the result is the reference's serial sum bit-for-bit.
//
// K_s  (k_spread) re-expresses the serial spreading loop (session.hpp:129-144,
// coupling.hpp:52-71) as an ordered gather: each band tile culls the markers
// whose stencil box overlaps it (ascending marker index, ballot compaction),
// stages their stencil records in shared memory, and every cell accumulates
// its contributions in ascending marker order.  No float atomics; results
// are independent of the launch shape and bit-identical to the serial loop.

/// IBKernel::phi (kernel.hpp:22-33), fp64.
__device__ __forceinline__ double ib_phi(int kernel, double r) {
  const double a = fabs(r);
  if (kernel == 0) {
    if (a >= 2.0) return 0.0;
    if (a <= 1.0) return 0.125 * (3.0 - 2.0 * a + sqrt(1.0 + 4.0 * a - 4.0 * a * a));
    return 0.125 * (5.0 - 2.0 * a - sqrt(-7.0 + 12.0 * a - 4.0 * a * a));
  }
  if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * r * r)) / 3.0;
  if (a <= 1.5) return (5.0 - 3.0 * a - sqrt(-3.0 * (1.0 - a) * (1.0 - a) + 1.0)) / 6.0;
  return 0.0;
}

/// r = R^T v in Eigen's coefficient order (R row-major).
__device__ __forceinline__ void mat_t_vec(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = R[i] * v[0] + R[3 + i] * v[1] + R[6 + i] * v[2];
}
__device__ __forceinline__ void mat_vec(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = R[3 * i] * v[0] + R[3 * i + 1] * v[1] + R[3 * i + 2] * v[2];
}

constexpr int MK_LANES = 16;      // lanes per marker (half a warp)
constexpr int MK_PER_BLOCK = 8;   // markers per 128-thread block
constexpr int MK_MAXC = 125;      // 5^3 (Peskin4 with x +- 2 integral)

/// Boundary-cell gather (rare for stencil cells).  Inline: an out-of-line
/// call forces the caller's gathered values through local memory.
template <bool PULLED>
__device__ __forceinline__ void gather_slow(const Grid& g, const Store* __restrict__ A, int x, int y,
                                         int z, Store* s) {
  Store t[Q];
  gather<PULLED>(g, A, x, y, z, t);
#pragma unroll
  for (int i = 0; i < Q; ++i) s[i] = t[i];
}

template <bool PULLED>
__device__ __forceinline__ void gather_cell(const Grid& g, const Store* __restrict__ A, int x, int y,
                                            int z, Store (&s)[Q]) {
  // 32-bit direction offsets (|pull| < 38 planes < 2^31 under the host's
  // 19 x cells < 2^32 bound): one IMAD.WIDE per load
  const Store* __restrict__ base = A + (unsigned)mem_index(g, x, y, z);
  if (!PULLED) {
#pragma unroll
    for (int i = 0; i < Q; ++i) s[i] = base[(int)g.own[i]];
  } else if (is_interior(g, x, y, z)) {
#pragma unroll
    for (int i = 0; i < Q; ++i) s[i] = base[(int)g.pull[i]];
  } else {
    gather_slow<PULLED>(g, A, x, y, z, s);
  }
}

template <bool PULLED>
__global__ void __launch_bounds__(128)
    k_markers(Grid g, const Store* __restrict__ A, Markers mk, const SessionConsts* __restrict__ scp,
              const StepConsts* __restrict__ stp, MarkerStencil* __restrict__ st,
              MarkerBox* __restrict__ boxes, double* __restrict__ fworld, double* fworld_h,
              int* valid_h, StepScratch* out) {
#if FSG_PREC == 64
  __shared__ double prod[MK_PER_BLOCK][MK_MAXC][3];
#endif
  __shared__ double phs[MK_PER_BLOCK][3][5];
  const int hl = threadIdx.x & (MK_LANES - 1);
  const int slot = threadIdx.x / MK_LANES;
  const unsigned hmask = 0xFFFFu << (threadIdx.x & 16);
  const int t = blockIdx.x * MK_PER_BLOCK + slot;
  if (t >= mk.m) return;  // uniform over the half-warp
  const SessionConsts& sc = *scp;
  const StepConsts& fs = *stp;
  // lane 0 prefetches the rest of the marker state (may be mapped host memory)
  double vel[3] = {0, 0, 0}, nrm[3] = {0, 0, 0}, area = 0.0;
  if (hl == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      vel[k] = mk.vel[3 * t + k];
      nrm[k] = mk.nrm[3 * t + k];
    }
    area = mk.area[t];
  }
  // position chain, identical on every lane (frame.hpp:24-26, session.hpp:82-85)
  double xw[3], xf[3], xl[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) xw[k] = mk.pts[3 * t + k] - fs.p[k];
  mat_t_vec(fs.R, xw, xf);
#pragma unroll
  for (int k = 0; k < 3; ++k) xl[k] = xf[k] / sc.dx + sc.hd[k];
  const double margin = 0.5 * (sc.kernel == 0 ? 4 : 3);
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (xl[a] < margin || xl[a] > sc.dims_g[a] - 1 - margin) ok = false;
  if (!ok) {
    if (hl == 0) {
      st[t].valid = 0;
      MarkerBox b;
      b.lo[0] = b.lo[1] = b.lo[2] = 1;
      b.hi[0] = b.hi[1] = b.hi[2] = 0;
      b.valid = 0;
      b._pad = 0;
      boxes[t] = b;
      fworld[3 * t] = fworld[3 * t + 1] = fworld[3 * t + 2] = 0.0;
      if (fworld_h) {
        fworld_h[3 * t] = fworld_h[3 * t + 1] = fworld_h[3 * t + 2] = 0.0;
        valid_h[t] = 0;
      }
      atomicAdd(&out->oob, 1);
    }
    return;
  }
  const double half = 0.5 * (sc.kernel == 0 ? 4 : 3);
  int lo[3], hi[3], cnt[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = (int)ceil(xl[a] - half);  // kernel.hpp:36-40
    hi[a] = (int)floor(xl[a] + half);
    cnt[a] = hi[a] - lo[a] + 1;
  }
  if (hl < 15) {
    const int a = hl / 5, q = hl % 5;
    phs[slot][a][q] = q < cnt[a] ? ib_phi(sc.kernel, (lo[a] + q) - xl[a]) : 0.0;
  }
  __syncwarp(hmask);
  // valid markers keep the whole stencil inside the box (coupling.hpp:35-39 clip is a no-op)
  const int ncell = cnt[0] * cnt[1] * cnt[2];
  const float r0 = 1.0f / (float)cnt[0], r01 = 1.0f / (float)(cnt[0] * cnt[1]);
#if FSG_PREC == 32
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;  // this lane's partial sums
#endif
  for (int c0 = 0; c0 < ncell; c0 += 4 * MK_LANES) {  // <= 2 rounds, one global round trip each
    Store sv[4][Q];
    int cio[4], cjo[4], cko[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = c0 + hl + MK_LANES * r;
      const int ko = (int)(((float)c + 0.5f) * r01);
      const int rem = c - ko * cnt[0] * cnt[1];
      const int jo = (int)(((float)rem + 0.5f) * r0);
      cio[r] = rem - jo * cnt[0];
      cjo[r] = jo;
      cko[r] = ko;
      if (c < ncell) gather_cell<PULLED>(g, A, lo[0] + cio[r], lo[1] + jo, lo[2] + ko - g.z0, sv[r]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int c = c0 + hl + MK_LANES * r;
      if (c < ncell) {
        double ux, uy, uz;
        bare_velocity(sv[r], ux, uy, uz);
        // coupling.hpp:40-43: wz = phi(k-z); wyz = wz*phi(j-y); w = wyz*phi(i-x)
        const double w = (phs[slot][2][cko[r]] * phs[slot][1][cjo[r]]) * phs[slot][0][cio[r]];
#if FSG_PREC == 64
        prod[slot][c][0] = w * ux;
        prod[slot][c][1] = w * uy;
        prod[slot][c][2] = w * uz;
#else
        a0 += w * ux;
        a1 += w * uy;
        a2 += w * uz;
#endif
      }
    }
  }
#if FSG_PREC == 64
  __syncwarp(hmask);
  if (hl != 0) return;
  double u0 = 0.0, u1 = 0.0, u2 = 0.0;
  for (int c = 0; c < ncell; ++c) {  // u += w * u_cell in the reference's k, j, i order
    u0 = u0 + prod[slot][c][0];
    u1 = u1 + prod[slot][c][1];
    u2 = u2 + prod[slot][c][2];
  }
#else
  // throughput mode: fixed-shape tree over the half-warp (deterministic)
#pragma unroll
  for (int o = MK_LANES / 2; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(hmask, a0, o, MK_LANES);
    a1 += __shfl_xor_sync(hmask, a1, o, MK_LANES);
    a2 += __shfl_xor_sync(hmask, a2, o, MK_LANES);
  }
  if (hl != 0) return;
  const double u0 = a0, u1 = a1, u2 = a2;
#endif
  const double uf[3] = {u0 * sc.v2p, u1 * sc.v2p, u2 * sc.v2p};  // vel_to_physical
  double vw[3], vf[3], ub[3], nf[3], fl[3], fw[3], ff[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) vw[k] = vel[k] - fs.pd[k];
  mat_t_vec(fs.R, vw, vf);
  const double wx0 = fs.wf[1] * xf[2] - fs.wf[2] * xf[1];
  const double wx1 = fs.wf[2] * xf[0] - fs.wf[0] * xf[2];
  const double wx2 = fs.wf[0] * xf[1] - fs.wf[1] * xf[0];
  ub[0] = vf[0] - wx0;
  ub[1] = vf[1] - wx1;
  ub[2] = vf[2] - wx2;
  mat_t_vec(fs.R, nrm, nf);
  double du[3] = {ub[0] - uf[0], ub[1] - uf[1], ub[2] - uf[2]};
  if (sc.wall == 0) {  // slip: (du . n) n
    const double s = du[0] * nf[0] + du[1] * nf[1] + du[2] * nf[2];
    du[0] = s * nf[0];
    du[1] = s * nf[1];
    du[2] = s * nf[2];
  }
  const double kf = sc.rho_phys * area * sc.dx / sc.dt;  // rho A h / dt
  fl[0] = kf * du[0];
  fl[1] = kf * du[1];
  fl[2] = kf * du[2];
  mat_vec(fs.R, fl, fw);
  fworld[3 * t] = fw[0];
  fworld[3 * t + 1] = fw[1];
  fworld[3 * t + 2] = fw[2];
  if (fworld_h) {
    fworld_h[3 * t] = fw[0];
    fworld_h[3 * t + 1] = fw[1];
    fworld_h[3 * t + 2] = fw[2];
    valid_h[t] = 1;
  }
  mat_t_vec(fs.R, fw, ff);
  MarkerStencil rec;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int q = 0; q < 5; ++q) rec.ph[a][q] = phs[slot][a][q];
    rec.fl[a] = ff[a] * sc.f2l;
    rec.lo[a] = lo[a];
    rec.hi[a] = hi[a];
  }
  rec.valid = 1;
  rec._pad = 0;
  st[t] = rec;
  MarkerBox b;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int off = a == 2 ? g.z0 : 0;  // local coordinates
    b.lo[a] = (short)(lo[a] - off);
    b.hi[a] = (short)(hi[a] - off);
  }
  b.valid = 1;
  b._pad = 0;
  boxes[t] = b;
  atomicMax(&out->bbox_lo_enc[0], LO_BIAS - lo[0]);
  atomicMax(&out->bbox_lo_enc[1], LO_BIAS - lo[1]);
  atomicMax(&out->bbox_lo_enc[2], LO_BIAS - max(lo[2] - g.z0, 0));
  atomicMax(&out->bbox_hi_enc[0], hi[0] + 1);
  atomicMax(&out->bbox_hi_enc[1], hi[1] + 1);
  atomicMax(&out->bbox_hi_enc[2], min(hi[2] - g.z0, g.nz - 1) + 1);
}

constexpr int SP_TX = 8, SP_TY = 4, SP_TZ = 4, SP_THREADS = 128;
constexpr int SP_BATCH = 8;                      // marker chunks culled per global round trip
constexpr int SP_LIST = SP_BATCH * SP_THREADS;  // candidates per batch (upper bound)
constexpr int SP_STAGE = 96;                     // candidate records staged per round

__global__ void __launch_bounds__(SP_THREADS)
    k_spread(Grid g, int m, const MarkerStencil* __restrict__ st, const MarkerBox* __restrict__ boxes,
             Band band, const StepScratch* __restrict__ bscr) {
  __shared__ int list[SP_LIST];
  __shared__ int wcount[SP_BATCH][SP_THREADS / 32];
  __shared__ MarkerStencil cand[SP_STAGE];
  int lo[3], hi[3];
  decode_bbox(bscr, lo, hi);
  if (hi[0] < lo[0] || hi[1] < lo[1] || hi[2] < lo[2]) return;
  const int bnx = hi[0] - lo[0] + 1, bny = hi[1] - lo[1] + 1, bnz = hi[2] - lo[2] + 1;
  if ((long long)bnx * bny * bnz > band.cap) return;
  const int tnx = (bnx + SP_TX - 1) / SP_TX, tny = (bny + SP_TY - 1) / SP_TY,
            tnz = (bnz + SP_TZ - 1) / SP_TZ;
  const int ntiles = tnx * tny * tnz;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx0 = lo[0] + (tile % tnx) * SP_TX;
    const int ty0 = lo[1] + ((tile / tnx) % tny) * SP_TY;
    const int tz0 = lo[2] + (tile / (tnx * tny)) * SP_TZ;  // local z
    const int tx1 = min(tx0 + SP_TX - 1, hi[0]), ty1 = min(ty0 + SP_TY - 1, hi[1]),
              tz1 = min(tz0 + SP_TZ - 1, hi[2]);
    const int cx = tx0 + (threadIdx.x % SP_TX);
    const int cy = ty0 + ((threadIdx.x / SP_TX) % SP_TY);
    const int cz = tz0 + threadIdx.x / (SP_TX * SP_TY);
    const int czg = cz + g.z0;
    double F0 = 0.0, F1 = 0.0, F2 = 0.0;
    for (int base = 0; base < m; base += SP_LIST) {
      // ---- cull one batch (SP_BATCH chunks, one global round trip)
      MarkerBox bx[SP_BATCH];
#pragma unroll
      for (int k = 0; k < SP_BATCH; ++k) {
        const int mi = base + k * SP_THREADS + threadIdx.x;
        if (mi < m) bx[k] = boxes[mi];
        else bx[k].valid = 0;
      }
      unsigned bal[SP_BATCH];
#pragma unroll
      for (int k = 0; k < SP_BATCH; ++k) {
        const bool hit = bx[k].valid && bx[k].lo[0] <= tx1 && bx[k].hi[0] >= tx0 &&
                         bx[k].lo[1] <= ty1 && bx[k].hi[1] >= ty0 && bx[k].lo[2] <= tz1 &&
                         bx[k].hi[2] >= tz0;
        bal[k] = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) wcount[k][wid] = __popc(bal[k]);
      }
      __syncthreads();
      int total = 0, before = 0;
#pragma unroll
      for (int k = 0; k < SP_BATCH; ++k) {
        int kb = 0;
#pragma unroll
        for (int w = 0; w < SP_THREADS / 32; ++w) {
          if (w == wid) before = total + kb;
          kb += wcount[k][w];
        }
        if ((bal[k] >> lane) & 1u)
          list[before + __popc(bal[k] & ((1u << lane) - 1u))] = base + k * SP_THREADS + threadIdx.x;
        total += kb;
      }
      __syncthreads();
      // ---- drain in ascending marker order, SP_STAGE records per round
      for (int q0 = 0; q0 < total; q0 += SP_STAGE) {
        const int nq = min(SP_STAGE, total - q0);
        // stage the records with 16-byte loads, all issued before any store
        constexpr int V = (int)(sizeof(MarkerStencil) / 16);
        constexpr int PER = (SP_STAGE * V + SP_THREADS - 1) / SP_THREADS;
        int4 tmp[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int e = threadIdx.x + k * SP_THREADS;
          if (e < nq * V) tmp[k] = reinterpret_cast<const int4*>(st + list[q0 + e / V])[e % V];
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const int e = threadIdx.x + k * SP_THREADS;
          if (e < nq * V) reinterpret_cast<int4*>(cand)[e] = tmp[k];
        }
        __syncthreads();
        for (int q = 0; q < nq; ++q) {
          const MarkerStencil& r = cand[q];
          if (cx >= r.lo[0] && cx <= r.hi[0] && cy >= r.lo[1] && cy <= r.hi[1] && czg >= r.lo[2] &&
              czg <= r.hi[2]) {
            const double w = (r.ph[2][czg - r.lo[2]] * r.ph[1][cy - r.lo[1]]) * r.ph[0][cx - r.lo[0]];
            F0 = F0 + w * r.fl[0];
            F1 = F1 + w * r.fl[1];
            F2 = F2 + w * r.fl[2];
          }
        }
        __syncthreads();
      }
    }
    if (cx <= tx1 && cy <= ty1 && cz <= tz1) {
      const long long lc = (long long)(cx - lo[0]) +
                           (long long)bnx * ((long long)(cy - lo[1]) + (long long)bny * (cz - lo[2]));
      band.F[3 * lc] = F0;
      band.F[3 * lc + 1] = F1;
      band.F[3 * lc + 2] = F2;
    }
  }
}
