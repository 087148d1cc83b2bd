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
