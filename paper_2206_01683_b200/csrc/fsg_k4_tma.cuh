// fsg_k4_tma.cuh -- pure-fluid K4 with bulk-async (TMA 1D) staging of the
// pull sources, included inside namespace fsg::p32 after fsg_k4.cuh.
//
// A tile is TW = 128 consecutive cells of one z-plane in the flattened
// (x + nx*y) order.  The pull source of direction i for cell c is element
// c - (ex_i + nx*ey_i + plane*ez_i) of plane i; for the whole tile that is a
// contiguous window.  One elected thread copies, per direction, the
// 16-byte-aligned superset [c0 - 4, c0 + TW + 4) of the window shifted by
// the row/plane part only (-nx*ey - plane*ez, a multiple of 4 elements) into
// shared memory with cp.async.bulk, completing on the tile's mbarrier; the
// -ex_i and the open-face clamp are applied when reading shared memory.  A
// ring of NST stages keeps NST - 1 tiles in flight per block while it
// computes the current one, so the memory-level parallelism comes from the
// bulk-copy engine, not from registers.  Reads from shared memory are
// consecutive words (conflict-free); results are stored straight to global.
//
// Planes on a global z face are not staged (the whole tile takes the generic
// clamped gather); cells on a y face, and periodic x-face cells whose wrapped
// source lies outside the window, take the global path individually.

constexpr int TMA_NST = 3;    // ring stages
constexpr int TMA_TW = 128;   // cells per tile (= threads per block)
constexpr int TMA_PAD = 4;    // staged margin on each side (16 B)
constexpr int TMA_ROW = TMA_TW + 2 * TMA_PAD;

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

template <bool VF>
__global__ void __launch_bounds__(TMA_TW, FSG_K4_MINB)
    k_collide_tma(Grid g, DirPtrs dp, const float* __restrict__ A,
                  const SessionConsts* __restrict__ scp, const StepConsts st,
                  StepScratch* __restrict__ out, StepScratch* __restrict__ next) {
  __shared__ __align__(16) float sm[TMA_NST][Q][TMA_ROW];
  __shared__ __align__(8) unsigned long long bar[TMA_NST];
  const int tid = threadIdx.x;
  const int plane = (int)g.plane;
  const int tpp = (plane + TMA_TW - 1) / TMA_TW;  // tiles per plane
  const int ntile = tpp * g.nz;
  reset_next(next, tid);
  const SessionConsts& sc = *scp;
  if (tid == 0) {
    for (int s = 0; s < TMA_NST; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // producer (one elected thread): stage tile t into ring slot s
  auto issue = [&](int t, int s) {
    const int z = t / tpp, c0 = (t - z * tpp) * TMA_TW;
    const int zg = g.z0 + z;
    if (zg <= 0 || zg >= g.nzg - 1) {  // z-face plane: nothing staged
      mbar_arrive(&bar[s]);
      return;
    }
    constexpr unsigned bytes = TMA_ROW * sizeof(float);
    mbar_expect_tx(&bar[s], bytes * Q);
    const long long m0 = (long long)c0 + g.zs * (z + g.zpad) - TMA_PAD;
#pragma unroll
    for (int i = 0; i < Q; ++i)  // dp.a[i] + ex_i: the row/plane shift only (16 B aligned)
      bulk_g2s(&sm[s][i][0], dp.a[i] + ex_of(i) + m0, bytes, &bar[s]);
  };
  int t = blockIdx.x;
  if (tid == 0)
    for (int k = 0; k < TMA_NST; ++k)
      if (t + k * (int)gridDim.x < ntile) issue(t + k * gridDim.x, k);
  float vmin = FLT_MAX;
  unsigned phase = 0;
  for (int k = 0; t < ntile; t += gridDim.x, ++k) {
    const int s = k % TMA_NST;
    const int z = t / tpp, c = (t - z * tpp) * TMA_TW + tid;
    const int zg = g.z0 + z;
    mbar_wait(&bar[s], phase);
    if (c < plane) {
      const int y = c / g.nx, x = c - y * g.nx;
      const bool face = zg <= 0 || zg >= g.nzg - 1 || y == 0 || y == g.ny - 1;
      const int cxp = x == 0 ? (g.periodic ? g.nx : 1) : 0;
      const int cxm = x == g.nx - 1 ? (g.periodic ? -g.nx : -1) : 0;
      if (face || (g.periodic && (cxp || cxm))) {
        vmin = fminf(vmin, cell_update<true, VF>(g, dp, A, x, y, z, 0.f, 0.f, 0.f, sc, st, out));
      } else {
        float v[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const int cx = ex_of(i) > 0 ? cxp : (ex_of(i) < 0 ? cxm : 0);
          v[i] = sm[s][i][TMA_PAD + tid - ex_of(i) + cx];
        }
        Band none{nullptr, 0};
        vmin = fminf(vmin, collide_cell32<3, VF>(v, x, y, z, g, 0.f, 0.f, 0.f, false, 0, none, sc, st,
                                                 out));
        const unsigned m = (unsigned)mem_index(g, x, y, z);
#pragma unroll
        for (int i = 0; i < Q; ++i) dp.b[i][m] = v[i];
      }
    }
    __syncthreads();  // everyone is done with slot s
    if (s == TMA_NST - 1) phase ^= 1u;
    if (tid == 0) {
      const int tn = t + TMA_NST * (int)gridDim.x;
      if (tn < ntile) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
        issue(tn, s);
      }
    }
  }
  report_min(out, vmin == FLT_MAX ? DBL_MAX : (double)vmin);
}
