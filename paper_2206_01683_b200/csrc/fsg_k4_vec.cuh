// fsg_k4_vec.cuh -- pure-fluid K4 with 128-bit loads and stores (fp32
// session), included inside namespace fsg::p32 after fsg_k4v4.cuh.
//
// Each lane owns 4 consecutive x-cells of a row, a warp 128 (nx % 128 == 0).
// Per direction i the lane loads the 16-byte-aligned float4 of the UNSHIFTED
// source row (y - ey_i, z - ez_i) at its 4 cells; the x shift -ex_i is then a
// one-element rotation across lanes: the missing element comes from the
// neighbouring lane by shuffle, and lanes 0 / 31 load it directly (or apply
// the open-face clamp / periodic wrap at the row ends, as the scalar fast
// path: solver.hpp:59-97 re-expressed as a pull).  Results are stored as
// float4.  Rows on a global y or z face take the scalar clamped path (warp-
// uniform: a warp covers one row segment).  Arithmetic per cell is exactly
// cell_update's (bit-identical, tests/test_k4_variants_gpu.py).

#ifndef FSG_K4V_MINB
#define FSG_K4V_MINB 3
#endif

template <bool VF>
__global__ void __launch_bounds__(128, FSG_K4V_MINB)
    k_collide_vec4(Grid g, DirPtrs dp, const float* __restrict__ A,
                   const SessionConsts* __restrict__ scp, const StepConsts st,
                   StepScratch* __restrict__ out, StepScratch* __restrict__ next, ZRange zr) {
  constexpr unsigned full = 0xFFFFFFFFu;
  const int tid = threadIdx.x, lane = tid & 31;
  reset_next(next, tid);
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (tid >> 5), W = gridDim.x * wpb;
  const int nseg = g.nx >> 7;  // 128-cell segments per row
  const int nq = (zr.hi - zr.lo + zr.step - 1) / zr.step;
  const int nitem = nseg * g.ny * nq;
  const SessionConsts& sc = *scp;
  Band none{nullptr, 0};
  float vmin = FLT_MAX;
  for (int it = gw; it < nitem; it += W) {  // warp-uniform item: one row segment
    const int sx = it % nseg, rest = it / nseg;
    const int y = rest % g.ny, z = zr.lo + (rest / g.ny) * zr.step;
    const int x0 = (sx << 7) + (lane << 2);
    const int zg = g.z0 + z;
    if (y == 0 || y == g.ny - 1 || zg == 0 || zg == g.nzg - 1) {
#pragma unroll 1
      for (int k = 0; k < 4; ++k)
        vmin = fminf(vmin, cell_update<true, VF>(g, dp, A, x0 + k, y, z, 0.f, 0.f, 0.f, sc, st, out));
      continue;
    }
    const int m = (int)mem_index(g, x0, y, z);
    float v[Q][4];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const float* rb = dp.a[i] + ex_of(i);  // unshifted source row: 16-byte aligned at m
      const float4 q = __ldg(reinterpret_cast<const float4*>(rb + m));
      if (ex_of(i) == 0) {
        v[i][0] = q.x; v[i][1] = q.y; v[i][2] = q.z; v[i][3] = q.w;
      } else if (ex_of(i) > 0) {  // source x - 1
        float l = __shfl_up_sync(full, q.w, 1);
        if (lane == 0) l = x0 > 0 ? __ldg(rb + m - 1) : (g.periodic ? __ldg(rb + m + g.nx - 1) : q.x);
        v[i][0] = l; v[i][1] = q.x; v[i][2] = q.y; v[i][3] = q.z;
      } else {  // source x + 1
        float r = __shfl_down_sync(full, q.x, 1);
        if (lane == 31)
          r = x0 + 4 < g.nx ? __ldg(rb + m + 4) : (g.periodic ? __ldg(rb + m + 4 - g.nx) : q.w);
        v[i][0] = q.y; v[i][1] = q.z; v[i][2] = q.w; v[i][3] = r;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float s[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) s[i] = v[i][k];
      vmin = fminf(vmin, collide_cell32<3, VF>(s, x0 + k, y, z, g, 0.f, 0.f, 0.f, false, 0, none, sc,
                                               st, out));
#pragma unroll
      for (int i = 0; i < Q; ++i) v[i][k] = s[i];
    }
#pragma unroll
    for (int i = 0; i < Q; ++i)
      *reinterpret_cast<float4*>(dp.b[i] + m) = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
  }
  report_min(out, vmin == FLT_MAX ? DBL_MAX : (double)vmin);
}
