// fsg_k4v4.cuh -- throughput K4 (fp32 deviations), included inside namespace
// fsg::p32.  One cell per thread; the 19 pull sources and 19 destinations are
// addressed through per-direction base pointers passed as kernel parameters
// (constant bank), so each access costs one LDC + one IMAD.WIDE instead of a
// runtime 64-bit index product.  Interior cells use the constant neighbour
// offsets folded into those pointers; boundary cells take the generic
// clamped/periodic gather (solver.hpp:59-97 re-expressed as a pull).

struct DirPtrs {
  const float* a[Q];  // A + pull[i]  (interior pull source of direction i)
  float* b[Q];        // B + own[i]   (destination plane of direction i)
};

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
    const int m = (int)mem_index(g, x, y, z);
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

// Coupled-step K4 of the throughput session: IB force from the fixed-point
// tile band (read and re-zeroed), virtual force inline, then collide/stream.
// Block (0,0,0) resets the next step's scratch; the last block to finish
// publishes the step status into mapped pinned host memory.
template <bool PULLED, bool VF>
__global__ void __launch_bounds__(128)
    k_collide_fix(Grid g, DirPtrs dp, const float* __restrict__ A, FixBand fb, int has_ib,
                  const SessionConsts* __restrict__ scp, const StepConsts st,
                  StepScratch* __restrict__ out, StepScratch* __restrict__ next,
                  StepScratch* publish, unsigned* tickets, unsigned* tickets_next, int zc) {
  constexpr int NS = (int)(sizeof(StepScratch) / 4);
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    if (tid < NS) reinterpret_cast<int*>(next)[tid] = 0;
    for (int k = tid; k <= TICKET_GROUPS; k += blockDim.x * blockDim.y) tickets_next[k] = 0u;
  }
  // persistent: work item = (xy tile column, chunk of zc planes); a block
  // walks its items, stepping z by one plane (no per-cell index division)
  const int tx_n = (g.nx + blockDim.x - 1) / blockDim.x;
  const int ty_n = (g.ny + blockDim.y - 1) / blockDim.y;
  const int ncol = tx_n * ty_n, nzc = (g.nz + zc - 1) / zc;
  const int nitem = ncol * nzc;
  float vmin = FLT_MAX;
  for (int it = blockIdx.x; it < nitem; it += gridDim.x) {
  const int col = it % ncol, zk = it / ncol;
  const int x = (col % tx_n) * blockDim.x + threadIdx.x;
  const int y = (col / tx_n) * blockDim.y + threadIdx.y;
  const int z0 = zk * zc, z1 = min(g.nz, z0 + zc);
  if (x < g.nx && y < g.ny) {
  const bool yin = y > 0 && y < g.ny - 1;
  // x faces stay on the fast path: the pull source of an unknown population
  // moves by +-1 (open: clamped copy, solver.hpp:59-97) or +-nx (periodic)
  const int cxp = x == 0 ? (g.periodic ? g.nx : 1) : 0;             // ex = +1
  const int cxm = x == g.nx - 1 ? (g.periodic ? -g.nx : -1) : 0;    // ex = -1
  int m = (int)mem_index(g, x, y, z0);
  for (int z = z0; z < z1; ++z, m += (int)g.plane) {
    float s[Q];
    const int zg = g.z0 + z;
    if (!PULLED) {
#pragma unroll
      for (int i = 0; i < Q; ++i) s[i] = __ldg(dp.a[i] + m);  // dp.a = A + own[i]
    } else if (yin && zg > 0 && zg < g.nzg - 1) {
#pragma unroll
      for (int i = 0; i < Q; ++i) {  // dp.a = A + pull[i]
        const int cx = ex_of(i) > 0 ? cxp : (ex_of(i) < 0 ? cxm : 0);
        s[i] = __ldg(dp.a[i] + (m + cx));
      }
    } else {
      gather<true>(g, A, x, y, z, s);  // y/z face rows (warp-uniform)
    }
    float Fx = 0.f, Fy = 0.f, Fz = 0.f;
    if (has_ib) {
      const int tile = (x >> 2) + fb.tnx * ((y >> 2) + fb.tny * (z >> 2));
      if (fb.flag_cur[tile]) {
        unsigned long long* F = fb.F + 3 * ((long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z));
        const long long f0 = (long long)F[0], f1 = (long long)F[1], f2 = (long long)F[2];
        F[0] = 0ull;
        F[1] = 0ull;
        F[2] = 0ull;
        Fx = (float)((double)f0 * FIX_INV);
        Fy = (float)((double)f1 * FIX_INV);
        Fz = (float)((double)f2 * FIX_INV);
      }
      if (((x | y | z) & 3) == 0) fb.flag_prev[tile] = 0;  // the previous step's flags
    }
    Band none{nullptr, 0};
    vmin = fminf(vmin, collide_cell32<3, VF>(s, x, y, z, g, Fx, Fy, Fz, false, 0, none, *scp, st, out));
#pragma unroll
    for (int i = 0; i < Q; ++i) dp.b[i][m] = s[i];
  }  // z
  }  // live column
  }  // work items
  report_min(out, vmin == FLT_MAX ? DBL_MAX : (double)vmin);
  if (publish) {
    __shared__ int last;
    // status writers (report_min's lane 0, rare nonfinite/nonpos stores)
    // fence themselves; the ticket below orders the block after them
    __syncthreads();
    if (tid == 0) {
      // hierarchical ticket: one same-address atomic per block would
      // serialise ~n/128 atomics on one L2 slice
      const unsigned nblk = gridDim.x * gridDim.y * gridDim.z;
      const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
      const unsigned G = max(64u, (nblk + TICKET_GROUPS - 1) / TICKET_GROUPS);
      const unsigned grp = bid / G, ngrp = (nblk + G - 1) / G;
      const unsigned gsize = min(G, nblk - grp * G);
      __threadfence();
      last = 0;
      if (atomicAdd(&tickets[grp], 1u) == gsize - 1) {
        __threadfence();
        last = atomicAdd(&tickets[TICKET_GROUPS], 1u) == ngrp - 1;
      }
    }
    __syncthreads();
    if (last && tid < NS) {
      __threadfence();
      reinterpret_cast<volatile int*>(publish)[tid] = reinterpret_cast<volatile int*>(out)[tid];
      __threadfence_system();
    }
  }
}
