// fsg_batch.cuh -- batched throughput coupled step: E independent env
// sessions of one configuration stepped by ONE marker launch and ONE banded
// K4 launch (BASELINE config 5: 64 envs, 8 per GPU).
// Included inside namespace fsg::p32 after fsg_ib_fix.cuh.
//
// The envs share one configuration, so the grid (dims and the pull/own
// offsets, in the constant bank) and the session constants are common
// kernel parameters; each env contributes an EnvPack (state pointers, frame
// constants, tile stamp, markers, outputs) uploaded by the host per step and
// staged in shared memory when a block moves to that env.  Work is flattened
// across envs -- markers, phase-A items and band tiles by prefix offsets --
// so the small per-env grids fill the GPU together and the launch overhead is
// paid once per batch.  Arithmetic per cell and per marker is exactly the
// single-session kernels' (bit-identical results, tests/test_batch_gpu.py).

/// env of global index v given the prefix field of each pack (linear scan in
/// shared memory; E <= 64)
__device__ __forceinline__ int env_of(const int* pref, int E, int v) {
  int e = 0;
  while (e + 1 < E && pref[e + 1] <= v) ++e;
  return e;
}

/// env_of for a non-decreasing sequence of v: advances the previous answer e
/// (a thread's markers, a block's fetched items), amortised O(1) per call.
__device__ __forceinline__ int env_adv(const int* pref, int E, int v, int e) {
  while (e + 1 < E && pref[e + 1] <= v) ++e;
  return e;
}

/// cell_update addressed from the env's state base pointers: the 19 source
/// and destination offsets are the common grid's (constant bank).
template <bool PULLED, bool VF>
__device__ __forceinline__ float cell_update_ab(const Grid& g, const float* __restrict__ A,
                                                float* __restrict__ B, int x, int y, int z,
                                                float Fx, float Fy, float Fz,
                                                const SessionConsts& sc, const StepConsts& st,
                                                StepScratch* out) {
  const unsigned m = (unsigned)mem_index(g, x, y, z);
  const int zg = g.z0 + z;
  // cell base pointers + 32-bit direction offsets: one IMAD.WIDE per access
  // (m + offset in unsigned arithmetic cost ~8 instructions per access)
  const float* __restrict__ Am = A + m;
  float* __restrict__ Bm = B + m;
  float s[Q];
  if (!PULLED) {
#pragma unroll
    for (int i = 0; i < Q; ++i) s[i] = __ldg(Am + (int)g.own[i]);
  } else if (y > 0 && y < g.ny - 1 && zg > 0 && zg < g.nzg - 1) {
    const int cxp = x == 0 ? (g.periodic ? g.nx : 1) : 0;
    const int cxm = x == g.nx - 1 ? (g.periodic ? -g.nx : -1) : 0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const int cx = ex_of(i) > 0 ? cxp : (ex_of(i) < 0 ? cxm : 0);
      s[i] = __ldg(Am + ((int)g.pull[i] + cx));
    }
  } else if (!g.periodic) {  // open y/z face rows: constant offsets (FaceFlags)
    const FaceFlags f = face_flags(g, x, y, zg);
#pragma unroll
    for (int i = 0; i < Q; ++i)
      s[i] = __ldg(Am + ((int)g.pull[i] + (face_unknown(ex_of(i), ey_of(i), ez_of(i), f) ? f.D : 0)));
  } else {
    gather<true>(g, A, x, y, z, s);
  }
  Band none{nullptr, 0};
  const float v = collide_cell32<3, VF>(s, x, y, z, g, Fx, Fy, Fz, false, 0, none, sc, st, out);
#pragma unroll
  for (int i = 0; i < Q; ++i) Bm[(int)g.own[i]] = s[i];
  return v;
}

/// PMODE: 1 every env pulled, 0 none (first step after set/init/recenter),
/// 2 mixed (runtime flag per env).  The frame mode is the batch's (VF).
template <int PMODE, bool VF>
__device__ __forceinline__ float cell_update_env(const Grid& g, const SessionConsts& sc,
                                                 const EnvPack& P, int x, int y, int z, float Fx,
                                                 float Fy, float Fz) {
  if (PMODE == 1 || (PMODE == 2 && P.pulled))
    return cell_update_ab<true, VF>(g, P.A, P.B, x, y, z, Fx, Fy, Fz, sc, P.st, P.out);
  return cell_update_ab<false, VF>(g, P.A, P.B, x, y, z, Fx, Fy, Fz, sc, P.st, P.out);
}

/// Per-env status minimum: warp min, then a fire-and-forget atomic by lane 0
/// (a block's consecutive items usually belong to different envs).  All 32
/// lanes must call it.
__device__ __forceinline__ void report_min_red(StepScratch* out, float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v < FLT_MAX) atomicMax(&out->neg_min_key, ~ordered_key((double)v));
}

/// Persistent over the markers of every env (the grid is capped at a few
/// blocks per SM: a batch's markers would otherwise take several waves, and
/// the dependent K4 launches only once every marker block has triggered).
/// Each group first stamps the tiles of ALL its markers, the block fences
/// and triggers K4, then the groups do the heavy per-marker work (the cheap
/// stencil is recomputed rather than kept).  Skinned envs: the group's
/// markers are skinned SKC at a time into a shared-memory cache (one lane per
/// marker and bone slot) before their stamps; the heavy loop takes position,
/// velocity, normal and the tau slot data from it (c5 round 145.1 -> 141.8
/// us against one marker per warp pass).
template <bool SKIN>  // SKIN: some env has a skinned body (P.skb)
__global__ void __launch_bounds__(128, FSG_KMB_MINB)
    k_markers_batch(Grid g, const SessionConsts* __restrict__ scp, const EnvPack* __restrict__ packs,
                    BatchHead h) {
  __shared__ double phs[FX_PER_BLOCK][3][5];
  __shared__ int mkb[BATCH_MAX];
  for (int e = threadIdx.x; e < h.E; e += blockDim.x) mkb[e] = packs[e].mk_begin;
  __syncthreads();
  const int lane = threadIdx.x & (FX_LANES - 1);
  const int slot = threadIdx.x / FX_LANES;
  const int stride = gridDim.x * FX_PER_BLOCK;
  const SessionConsts& sc = *scp;
  // the stencils of a group's first 4 markers, reused by the heavy loop
  __shared__ MkStencil s_st[FX_PER_BLOCK][4];
  // skinned envs: the group's markers skinned SKC at a time (fsg_skin_fused.cuh)
  __shared__ SkinCache s_sk[SKIN ? FX_PER_BLOCK : 1];
  const int tg0 = blockIdx.x * FX_PER_BLOCK + slot;
  auto fill = [&](int k) {  // warp-uniform: the cache for markers k .. k + SKC - 1
    skin_cache_fill(s_sk[slot], tg0 + k * stride, stride, h.m_total,
                    [&](int tg, SkinView& V, const fsg_body_pose*& Q, int& t, double** outp) {
                      const EnvPack& P = packs[env_of(mkb, h.E, tg)];
                      if (!P.skb) return false;
                      V = SkinView{P.sk_rest, P.sk_nrest, P.sk_wb, P.sk_ww};
                      Q = &P.skb->pose;
                      t = tg - P.mk_begin;
                      outp[0] = const_cast<double*>(P.mk.pts);
                      outp[1] = const_cast<double*>(P.mk.vel);
                      outp[2] = const_cast<double*>(P.mk.nrm);
                      return true;
                    });
  };
  int ev = 0;  // the group's markers run in increasing order: env by advancing
  for (int tg = tg0, k = 0; tg < h.m_total; tg += stride, ++k) {
    if (SKIN && k % SKC == 0) fill(k);
    ev = env_adv(mkb, h.E, tg, ev);
    const EnvPack& P = packs[ev];
    const FixBand fb{P.F, P.tflag, h.tnx, h.tny, h.tnz, P.stamp};
    const int t = tg - P.mk_begin;
    MkStencil S;
    if (SKIN && P.skb) {
      const double* xc = s_sk[slot].x[k % SKC];
      const double xw[3] = {xc[0], xc[1], xc[2]};
      mk_stencil_x(xw, sc, P.st, S);
    } else {
      mk_stencil(P.mk, t, sc, P.st, S);
    }
    mk_stamp(g, fb, S, lane);
    if (k < 4 && lane == 0) s_st[slot][k] = S;
  }
  __syncthreads();  // all stamps of the block before the K4 trigger (k_markers_fix)
  if (threadIdx.x == 0) __threadfence();
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  // a group with more than SKC markers refills the cache chunk by chunk again
  const bool refill = tg0 + SKC * stride < h.m_total;
  ev = 0;
  for (int tg = tg0, k = 0; tg < h.m_total; tg += stride, ++k) {
    if (SKIN && refill && k % SKC == 0) fill(k);
    ev = env_adv(mkb, h.E, tg, ev);
    const EnvPack& P = packs[ev];
    const FixBand fb{P.F, P.tflag, h.tnx, h.tny, h.tnz, P.stamp};
    const int t = tg - P.mk_begin;
    MkStencil S;
    if (k < 4) {
      S = s_st[slot][k];  // from the stamp phase (the block barrier since orders it)
    } else if (SKIN && P.skb) {
      const double* xc = s_sk[slot].x[k % SKC];
      const double xw[3] = {xc[0], xc[1], xc[2]};
      mk_stencil_x(xw, sc, P.st, S);
    } else {
      mk_stencil(P.mk, t, sc, P.st, S);
    }
    if (SKIN && P.skb) {
      const SkinCache& C = s_sk[slot];
      const int kc = k % SKC;
      const double vel[3] = {C.v[kc][0], C.v[kc][1], C.v[kc][2]};
      const double nrm[3] = {C.n[kc][0], C.n[kc][1], C.n[kc][2]};
      double fw[3];
      if (P.pulled)
        mk_finish<true>(g, P.A, P.mk, t, lane, sc, P.st, S, phs[slot], P.rec, P.fworld, P.fworld_h,
                        P.valid_h, fb, P.out, vel, nrm, fw);
      else
        mk_finish<false>(g, P.A, P.mk, t, lane, sc, P.st, S, phs[slot], P.rec, P.fworld, P.fworld_h,
                         P.valid_h, fb, P.out, vel, nrm, fw);
      __syncwarp(fx_mask());
      if (S.ok) {
        double acc = 0.0;
        const int q = lane >> 3;  // the bone slot this lane's tau terms belong to
        const double p[3] = {C.xb[kc][q][0], C.xb[kc][q][1], C.xb[kc][q][2]};
        skin_tau_core<true>(*P.skb, lane, C.b[kc][q], C.w[kc][q], p, fw, vel, acc);
        skin_red_marker(acc, lane, P.sk_acc, t);
      }
      __syncwarp();  // the cache may be refilled for the next chunk
      continue;
    }
    if (P.pulled)
      mk_finish<true>(g, P.A, P.mk, t, lane, sc, P.st, S, phs[slot], P.rec, P.fworld, P.fworld_h,
                      P.valid_h, fb, P.out);
    else
      mk_finish<false>(g, P.A, P.mk, t, lane, sc, P.st, S, phs[slot], P.rec, P.fworld, P.fworld_h,
                       P.valid_h, fb, P.out);
    __syncwarp(fx_mask());  // phs[slot] is reused by the group's next marker
  }
}

/// Banded K4 over every env (see k_collide_band); a programmatic dependent
/// of k_markers_batch.  The status minimum is reported per env.
template <int PMODE, bool VF>
__global__ void __launch_bounds__(128, FSG_K4BB_MINB)
    k_collide_band_batch(Grid g, const SessionConsts* __restrict__ scp,
                         const EnvPack* __restrict__ packs, BatchHead h, unsigned* work) {
  __shared__ int item;
  __shared__ int tl[128];
  __shared__ int ntl;
  __shared__ int ib[BATCH_MAX], tb[BATCH_MAX];
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  const int nthr = blockDim.x * blockDim.y;
  const SessionConsts& sc = *scp;
  // a programmatic dependent (the one-call step's status copy) may start now
  asm volatile("griddepcontrol.launch_dependents;");
  for (int e = tid; e < h.E; e += nthr) {
    ib[e] = packs[e].item_begin;
    tb[e] = packs[e].tile_begin;
  }
  if (blockIdx.x == 0) {  // zero every env's next-step scratch
    constexpr int NS = (int)(sizeof(StepScratch) / 4);
    for (int k = tid; k < h.E * NS; k += nthr) reinterpret_cast<int*>(packs[k / NS].next)[k % NS] = 0;
  }
  __syncthreads();
  const int tx_n = (g.nx + blockDim.x - 1) / blockDim.x;
  const int ty_n = (g.ny + blockDim.y - 1) / blockDim.y;
  const int ncol = tx_n * ty_n;
  // ---- phase A: every env's cells outside its stamped tiles.  A fetch takes
  // CH consecutive items (CH = 4 kept blocks within one env longer but left
  // too few work units for small batches: E = 8 unchanged, E = 1 slower)
  constexpr int CH = 1;
  int nxt = 0;
  if (tid == 0) nxt = (int)atomicAdd(work, 1u) * CH;
  int itg = h.item_total, iend = 0, ev = 0;
  for (;;) {
    if (itg >= iend) {  // block-uniform: next chunk
      if (tid == 0) item = nxt;
      __syncthreads();
      itg = item;
      iend = min(itg + CH, h.item_total);
      if (itg >= h.item_total) break;
      if (tid == 0) nxt = (int)atomicAdd(work, 1u) * CH;
    }
    // the env's few per-item fields come straight from the (L1-resident)
    // pack array: restaging a pack in shared memory on nearly every item (a
    // block's successive items usually belong to different envs) costs an
    // L2 round trip and two barriers
    ev = env_adv(ib, h.E, itg, ev);  // a block's items are fetched in increasing order
    const EnvPack& P = packs[ev];
    const int it = itg - P.item_begin;
    const int col = it % ncol, zk = it / ncol;
    const int x = (col % tx_n) * blockDim.x + threadIdx.x;
    const int y = (col / tx_n) * blockDim.y + threadIdx.y;
    const int z0 = zk * h.zc, z1 = min(g.nz, z0 + h.zc);
    float vmin = FLT_MAX;
    // stamped tiles are the band phase's (one stamp load per tile-aligned item)
    if (x < g.nx && y < g.ny &&
        __ldcg(P.tflag + (x >> 2) + h.tnx * ((y >> 2) + h.tny * (z0 >> 2))) != P.stamp)
      for (int z = z0; z < z1; ++z)
        vmin = fminf(vmin, cell_update_env<PMODE, VF>(g, sc, P, x, y, z, 0.f, 0.f, 0.f));
    report_min_red(P.out, vmin);
    ++itg;
    if (itg >= iend) __syncthreads();  // `item` is rewritten for the next chunk
  }
  // ---- phase B: every env's stamped tiles, after the marker grid completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == gridDim.x - 1)  // skinned envs: tau_ext / stats sums are complete
    for (int k = tid; k < h.E * 32; k += nthr) {
      const EnvPack& Q0 = packs[k >> 5];
      const int c = k & 31;
      if (!Q0.skb) continue;
      long long v = 0, bad = 0;  // the replicas summed as integers; slot 31 the flag
      for (int r = 0; r < SKIN_FIX_REP; ++r) {
        v += (long long)__ldcg(Q0.sk_acc + 64 * r + c);
        bad |= (long long)__ldcg(Q0.sk_acc + 64 * r + 31);
      }
      __syncwarp();  // (env, c) pairs are warp-aligned: every read before the re-zeroing
      for (int r = 0; r < SKIN_FIX_REP; ++r) Q0.sk_acc[64 * r + c] = 0ull;
      const double d = bad ? __longlong_as_double(0x7ff8000000000000ll) : (double)v * SKIN_FIX_INV;
      if (c < Q0.sk_ndof) Q0.sk_out[c] = d;
      if (c >= SKIN_TAU_MAX && c < SKIN_TAU_MAX + SKIN_NSTAT) Q0.sk_out[Q0.sk_ndof + (c - SKIN_TAU_MAX)] = d;
    }
  const int tpp = nthr >> 6;
  const int half = tid >> 6, lt = tid & 63;
  for (int base = 0; (long long)base * gridDim.x < h.tile_total; base += nthr) {
    if (tid == 0) ntl = 0;
    __syncthreads();
    const long long T0 = (long long)blockIdx.x + (long long)gridDim.x * (base + tid);
    if (T0 < h.tile_total) {
      const EnvPack& Q0 = packs[env_of(tb, h.E, (int)T0)];
      if (Q0.tflag[T0 - Q0.tile_begin] == Q0.stamp) tl[atomicAdd(&ntl, 1)] = (int)T0;
    }
    __syncthreads();
    const int n = half < tpp ? ntl : 0;
    for (int k = half; k < n; k += tpp) {
      const int Tg = tl[k];
      const EnvPack& R = packs[env_of(tb, h.E, Tg)];
      const int T = Tg - R.tile_begin;
      const int tx = T % h.tnx, ty = (T / h.tnx) % h.tny, tz = T / (h.tnx * h.tny);
      const int x = 4 * tx + (lt & 3), y = 4 * ty + ((lt >> 2) & 3), z = 4 * tz + (lt >> 4);
      float v = FLT_MAX;
      if (x < g.nx && y < g.ny && z < g.nz) {
        unsigned long long* F = R.F + 3 * ((long long)x + (long long)g.nx * ((long long)y + (long long)g.ny * z));
        const long long f0 = (long long)F[0], f1 = (long long)F[1], f2 = (long long)F[2];
        F[0] = 0ull;
        F[1] = 0ull;
        F[2] = 0ull;
        v = cell_update_env<PMODE, VF>(g, sc, R, x, y, z, (float)((double)f0 * FIX_INV),
                                       (float)((double)f1 * FIX_INV), (float)((double)f2 * FIX_INV));
      }
      report_min_red(R.out, v);
    }
    __syncthreads();
  }
}
