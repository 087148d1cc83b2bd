// fsg_skin_fused.cuh -- skinned bodies fused into the throughput marker
// kernel, included inside namespace fsg::p32 by
// fsg_ib_fix.cuh.  For up to two skinned bodies the coupled fp32 step stays
// two launches: the marker kernel skins its own markers from the pose it
// receives as a __grid_constant__ parameter and reduces tau_ext and the
// CouplingStats in its tail (off the critical path: the banded K4's first
// phase runs meanwhile).
//
// * LBS (update_samples, sampling.hpp:307-322; skin_point /
//   skin_point_velocity, skinning.hpp:105-126): lane l < SKIN_KW evaluates
//   bone slot l, the warp adds the slots in ascending bone order.  Explicit
//   round-to-nearest intrinsics keep this TU's FMA contraction out, so the
//   marker state is bit-identical to the fp64 parity path's.
// * tau_ext (accumulate_skinned_force -> accumulate_point_force,
//   skinning.hpp:147-156, dynamics.hpp:216-233): lane k*8 + l evaluates, for
//   bone slot k, the floating-base wrench (l = 0) or the l-th joint up the
//   chain, and on chains deeper than 7 joints (the eel) also the (l+8)-th;
//   the warp gathers a marker's terms in slot order, lane c keeps dof c's
//   running sum over the warp's markers; the block sums its warps in order
//   and adds the total to 64-bit fixed-point accumulators (2^-44) with integer
//   atomics, which the banded K4 converts once the marker grid is complete:
//   deterministic run to run (throughput mode; parity mode keeps the
//   reference's serial order).

__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ void rn_mv(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    r[i] = rn_add(rn_add(rn_mul(R[3 * i], v[0]), rn_mul(R[3 * i + 1], v[1])), rn_mul(R[3 * i + 2], v[2]));
}
__device__ __forceinline__ void rn_mtv(const double* R, const double* v, double* r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    r[i] = rn_add(rn_add(rn_mul(R[i], v[0]), rn_mul(R[3 + i], v[1])), rn_mul(R[6 + i], v[2]));
}
__device__ __forceinline__ void rn_cross(const double* a, const double* b, double* r) {
  r[0] = rn_sub(rn_mul(a[1], b[2]), rn_mul(a[2], b[1]));
  r[1] = rn_sub(rn_mul(a[2], b[0]), rn_mul(a[0], b[2]));
  r[2] = rn_sub(rn_mul(a[0], b[1]), rn_mul(a[1], b[0]));
}
__device__ __forceinline__ double rn_dot(const double* a, const double* b) {
  return rn_add(rn_add(rn_mul(a[0], b[0]), rn_mul(a[1], b[1])), rn_mul(a[2], b[2]));
}
/// BoneTransforms::apply (skinning.hpp:101)
__device__ __forceinline__ void rn_apply(const fsg_body_pose& Q, int b, const double* x, double* xb) {
  rn_mv(Q.bone_R[b], x, xb);
#pragma unroll
  for (int c = 0; c < 3; ++c) xb[c] = rn_add(xb[c], Q.bone_t[b][c]);
}

/// The per-marker skin arrays (SkinParamsN, or one env's in a batch).
struct SkinView {
  const double* rest;   // [3m]
  const double* nrest;  // [3m]
  const int* wb;        // [m][SKIN_KW]
  const double* ww;     // [m][SKIN_KW]
};

/// Stage the bodies (topology + pose) of the launch parameters in shared
/// memory, compacted to the links in use: the topology part whole, each pose
/// array only its first n_links rows (the koi uses 6 of the 12 slots).  Ends
/// with a block barrier.
template <int NB>
__device__ __forceinline__ void skin_stage_bodies(const SkinParamsN<NB>& P, SkinBody* dst) {
  static_assert(sizeof(SkinBody) % 8 == 0 && offsetof(SkinBody, pose) % 8 == 0, "copied as doubles");
  constexpr int TOPO = (int)(offsetof(SkinBody, pose) / 8);
  constexpr int POSE0 = TOPO;
  constexpr int L = SKIN_L;
  // pose arrays (doubles per link): bone_R 9, bone_t 3, R_world 9, p_world 3, v_origin 3, omega 3
  for (int b = 0; b < NB; ++b) {
    if (b >= P.nb) break;
    const double* src = reinterpret_cast<const double*>(&P.body[b]);
    double* d = reinterpret_cast<double*>(&dst[b]);
    const int nl = P.body[b].n_links;
    const int n = TOPO + 30 * nl;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      int off;
      if (k < TOPO) {
        off = k;
      } else {
        int r = k - TOPO, base = POSE0;
        const int w[6] = {9, 3, 9, 3, 3, 3};
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          if (r < w[a] * nl) break;
          r -= w[a] * nl;
          base += w[a] * L;
        }
        off = base + r;
      }
      d[off] = src[off];
    }
  }
  __syncthreads();
}

/// This lane's bone slot of marker t (lanes >= SKIN_KW: none).
struct SkinSlot {
  int b;     // bone (-1: none)
  double w;  // its weight
};

template <int NB>
__device__ __forceinline__ int skin_body_of(const SkinParamsN<NB>& P, int t) {
  int b = 0;
#pragma unroll
  for (int k = 1; k < NB; ++k)
    if (k < P.nb && t >= P.body[k].m0) b = k;
  return b;
}

template <class SP>
__device__ __forceinline__ SkinSlot skin_slot(const SP& P, int t, int lane) {
  SkinSlot s{-1, 0.0};
  if (lane < SKIN_KW) {
    s.b = __ldg(P.wb + SKIN_KW * t + lane);
    if (s.b >= 0) s.w = __ldg(P.ww + SKIN_KW * t + lane);
  }
  return s;
}

/// Warp sum of the per-slot vectors in ascending slot order, starting from 0
/// (out += w[b] * term_b for the nonzero weights, skinning.hpp:108-110); the
/// slot lanes' vectors go through a per-warp shared-memory buffer.
__device__ __forceinline__ void slot_sum(const SkinSlot& s, const double* term, double* out) {
  __shared__ double sb[FX_PER_BLOCK][SKIN_KW][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < SKIN_KW) {
#pragma unroll
    for (int c = 0; c < 3; ++c) sb[warp][lane][c] = term[c];
    sb[warp][lane][3] = s.b >= 0 ? 1.0 : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = 0.0;
#pragma unroll
  for (int l = 0; l < SKIN_KW; ++l) {
    if (sb[warp][l][3] == 0.0) break;  // slots are packed: the first empty one ends the list
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = rn_add(out[c], sb[warp][l][c]);
  }
  __syncwarp();  // the buffer is rewritten by the next sum
}

/// skin_point: world position of marker t (all lanes).
template <class SP>
__device__ __forceinline__ void skin_point_warp(const SP& P, const fsg_body_pose& Q, int t,
                                                const SkinSlot& s, double* xw) {
  const double x[3] = {__ldg(P.rest + 3 * t), __ldg(P.rest + 3 * t + 1), __ldg(P.rest + 3 * t + 2)};
  double term[3] = {0.0, 0.0, 0.0};
  if (s.b >= 0) {
    double xb[3];
    rn_apply(Q, s.b, x, xb);
#pragma unroll
    for (int c = 0; c < 3; ++c) term[c] = rn_mul(s.w, xb[c]);
  }
  slot_sum(s, term, xw);
}

/// skin_point_velocity and the blended normal, normalized() (all lanes).
/// xb_out (nullable): this slot lane's bone-transformed point (the p of the
/// tau terms, skin_tau_pre).
template <class SP>
__device__ __forceinline__ void skin_vel_nrm_warp(const SP& P, const fsg_body_pose& Q, int t,
                                                  const SkinSlot& s, double* vel, double* nrm,
                                                  double* xb_out = nullptr) {
  double tv[3] = {0.0, 0.0, 0.0}, tn[3] = {0.0, 0.0, 0.0};
  if (s.b >= 0) {
    const double x[3] = {__ldg(P.rest + 3 * t), __ldg(P.rest + 3 * t + 1), __ldg(P.rest + 3 * t + 2)};
    const double n0[3] = {__ldg(P.nrest + 3 * t), __ldg(P.nrest + 3 * t + 1), __ldg(P.nrest + 3 * t + 2)};
    double xb[3], d[3], cr[3], rn[3];
    rn_apply(Q, s.b, x, xb);
    if (xb_out) {
#pragma unroll
      for (int c = 0; c < 3; ++c) xb_out[c] = xb[c];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = rn_sub(xb[c], Q.p_world[s.b][c]);
    rn_cross(Q.omega_world[s.b], d, cr);
    rn_mv(Q.bone_R[s.b], n0, rn);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      tv[c] = rn_mul(s.w, rn_add(Q.v_origin_world[s.b][c], cr[c]));
      tn[c] = rn_mul(s.w, rn[c]);
    }
  }
  slot_sum(s, tv, vel);
  slot_sum(s, tn, nrm);
  const double z = rn_dot(nrm, nrm);
  if (z > 0.0) {
    const double sz = __dsqrt_rn(z);
#pragma unroll
    for (int c = 0; c < 3; ++c) nrm[c] = __ddiv_rn(nrm[c], sz);
  }
}

/// Skinning of up to SKC of a warp's markers at once: lane 4j + s evaluates
/// bone slot s of the warp's j-th marker (SKIN_KW == 4 slots), the four lanes
/// of a group add their slot terms in ascending slot order by shuffles.  Per
/// slot the arithmetic, and per marker the order of the sums, are
/// skin_point_warp's and skin_vel_nrm_warp's (bit-identical), at an eighth of
/// their warp instructions (those evaluate one marker per warp, 4 lanes busy).
constexpr int SKC = 8;
struct SkinCache {
  double x[SKC][3], v[SKC][3], n[SKC][3];  // position, velocity, unit normal
  double xb[SKC][SKIN_KW][3];              // slot s's bone-transformed point (tau terms)
  double w[SKC][SKIN_KW];
  int b[SKC][SKIN_KW];
};

/// Sum over the 4 lanes of this lane's group in slot order from 0, stopping at
/// the first empty slot (slot_sum's rule); every lane of the group gets it.
__device__ __forceinline__ void grp_slot_sum(bool has, const double* term, double* out) {
  static_assert(SKIN_KW == 4, "4 lanes per marker");
  const int g0 = (threadIdx.x & 31) & ~3;
  bool live = true;
#pragma unroll
  for (int c = 0; c < 3; ++c) out[c] = 0.0;
#pragma unroll
  for (int l = 0; l < SKIN_KW; ++l) {
    const int h = __shfl_sync(0xffffffffu, has ? 1 : 0, g0 + l);
    double t[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) t[c] = __shfl_sync(0xffffffffu, term[c], g0 + l);
    live = live && h;
    if (live) {
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = rn_add(out[c], t[c]);
    }
  }
}

/// Fill C (all 32 lanes): marker j (< SKC) of the warp is global index
/// tg0 + j * stride if below m_total; `locate(tg, V, Q, t)` gives its skin
/// view, pose and local index (false: not a skinned marker).  Writes the
/// markers' pts / vel / nrm (lanes s = 0, 1, 2 of the group).  Ends with
/// __syncwarp.
template <class Locate>
__device__ __forceinline__ void skin_cache_fill(SkinCache& C, int tg0, int stride, int m_total,
                                                Locate locate) {
  static_assert(FX_LANES == 32, "a warp per marker group");
  const int lane = threadIdx.x & 31, j = lane >> 2, s = lane & 3;
  const int tg = tg0 + j * stride;
  int b = -1;
  double w = 0.0, tx[3] = {0.0, 0.0, 0.0}, tv[3] = {0.0, 0.0, 0.0}, tn[3] = {0.0, 0.0, 0.0};
  double xb[3] = {0.0, 0.0, 0.0};
  double* outp[3] = {nullptr, nullptr, nullptr};
  int t = 0;
  SkinView V;
  const fsg_body_pose* Q = nullptr;
  if (tg < m_total && locate(tg, V, Q, t, outp)) {
    b = __ldg(V.wb + SKIN_KW * t + s);
    if (b >= 0) {
      w = __ldg(V.ww + SKIN_KW * t + s);
      const double x[3] = {__ldg(V.rest + 3 * t), __ldg(V.rest + 3 * t + 1), __ldg(V.rest + 3 * t + 2)};
      const double n0[3] = {__ldg(V.nrest + 3 * t), __ldg(V.nrest + 3 * t + 1), __ldg(V.nrest + 3 * t + 2)};
      double d[3], cr[3], rn[3];
      rn_apply(*Q, b, x, xb);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        tx[c] = rn_mul(w, xb[c]);
        d[c] = rn_sub(xb[c], Q->p_world[b][c]);
      }
      rn_cross(Q->omega_world[b], d, cr);
      rn_mv(Q->bone_R[b], n0, rn);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        tv[c] = rn_mul(w, rn_add(Q->v_origin_world[b][c], cr[c]));
        tn[c] = rn_mul(w, rn[c]);
      }
    }
  }
  double X[3], Vv[3], N[3];
  grp_slot_sum(b >= 0, tx, X);
  grp_slot_sum(b >= 0, tv, Vv);
  grp_slot_sum(b >= 0, tn, N);
  const double z = rn_dot(N, N);
  if (z > 0.0) {
    const double sz = __dsqrt_rn(z);
#pragma unroll
    for (int c = 0; c < 3; ++c) N[c] = __ddiv_rn(N[c], sz);
  }
  if (s == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C.x[j][c] = X[c];
      C.v[j][c] = Vv[c];
      C.n[j][c] = N[c];
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) C.xb[j][s][c] = xb[c];
  C.b[j][s] = b;
  C.w[j][s] = w;
  if (s < 3 && outp[s]) {
    const double* src = s == 0 ? X : (s == 1 ? Vv : N);
#pragma unroll
    for (int c = 0; c < 3; ++c) outp[s][3 * t + c] = src[c];
  }
  __syncwarp();
}

template <class SP>
__device__ __forceinline__ void skin_tau_warp(const SP& P, const SkinBody& B, int t, int lane,
                                              const double* fw, const double* vel, double& acc);

/// skin_tau_warp with the slot data the velocity phase already has: lane k
/// (< SKIN_KW) holds slot k's bone, weight and bone-transformed point; the
/// lanes of slot k take them by shuffle instead of reloading the marker and
/// re-applying the bone transform (same values: bit-identical).
__device__ __forceinline__ void skin_tau_pre(const SkinBody& B, int lane, const SkinSlot& sl,
                                             const double* xb, const double* fw, const double* vel,
                                             double& acc);

/// Add marker t's J^T(-f) terms and CouplingStats to the warp's running sums:
/// lane c (< SKIN_TAU_MAX) holds dof c, lane SKIN_TAU_MAX + k stat k.
template <bool PRE>
__device__ __forceinline__ void skin_tau_core(const SkinBody& B, int lane, int b, double w,
                                              const double* p_in, const double* fw, const double* vel,
                                              double& acc);

template <class SP>
__device__ __forceinline__ void skin_tau_warp(const SP& P, const SkinBody& B, int t, int lane,
                                              const double* fw, const double* vel, double& acc) {
  const int k = lane >> 3;
  int b = -1;
  double w = 0.0;
  if (k < SKIN_KW) {
    b = __ldg(P.wb + SKIN_KW * t + k);
    if (b >= 0) w = __ldg(P.ww + SKIN_KW * t + k);
  }
  double p[3] = {0.0, 0.0, 0.0};
  if (b >= 0) {
    const double x[3] = {__ldg(P.rest + 3 * t), __ldg(P.rest + 3 * t + 1), __ldg(P.rest + 3 * t + 2)};
    rn_apply(B.pose, b, x, p);
  }
  skin_tau_core<false>(B, lane, b, w, p, fw, vel, acc);
}

__device__ __forceinline__ void skin_tau_pre(const SkinBody& B, int lane, const SkinSlot& sl,
                                             const double* xb, const double* fw, const double* vel,
                                             double& acc) {
  const int k = lane >> 3;  // SKIN_KW == 4: every lane's slot is a real lane
  static_assert(SKIN_KW == 4, "slot k lives on lane k");
  const int b = __shfl_sync(0xffffffffu, sl.b, k);
  const double w = __shfl_sync(0xffffffffu, sl.w, k);
  const double p[3] = {__shfl_sync(0xffffffffu, xb[0], k), __shfl_sync(0xffffffffu, xb[1], k),
                       __shfl_sync(0xffffffffu, xb[2], k)};
  skin_tau_core<true>(B, lane, b, w, p, fw, vel, acc);
}

template <bool PRE>
__device__ __forceinline__ void skin_tau_core(const SkinBody& B, int lane, int b, double w,
                                              const double* p_in, const double* fw, const double* vel,
                                              double& acc) {
  const fsg_body_pose& Q = B.pose;
  const int k = lane >> 3, l = lane & 7;  // bone slot, level (0: base wrench, l: l-th joint up)
  double term[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double term2 = 0.0;  // level l + 8 (chains deeper than 7 joints)
  const bool deep = B.max_level > 7;  // uniform over the warp
  int comp = -1;  // l > 0: the dof this lane's term goes to
  if (b >= 0) {
    const double p[3] = {p_in[0], p_in[1], p_in[2]};
    double fv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) fv[c] = rn_mul(w, -fw[c]);
    if (l == 0) {
      if (B.floating) {
        double d[3], cr[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) d[c] = rn_sub(p[c], Q.p_world[0][c]);
        rn_cross(d, fv, cr);
        rn_mtv(Q.R_world[0], cr, term);
        rn_mtv(Q.R_world[0], fv, term + 3);
      }
    } else {
      const int j = B.anc[b][l - 1];
      if (j > 0 && B.dof[j] >= 0) {
        double aw[3], d[3], cr[3];
        rn_mv(Q.R_world[j], B.axis[j], aw);
#pragma unroll
        for (int c = 0; c < 3; ++c) d[c] = rn_sub(p[c], Q.p_world[j][c]);
        rn_cross(aw, d, cr);
        term[0] = rn_dot(cr, fv);
        comp = B.dof[j];
      }
    }
    if (deep && l + 8 <= SKIN_L) {
      const int j2 = B.anc[b][l + 7];
      if (j2 > 0 && B.dof[j2] >= 0) {
        double aw[3], d[3], cr[3];
        rn_mv(Q.R_world[j2], B.axis[j2], aw);
#pragma unroll
        for (int c = 0; c < 3; ++c) d[c] = rn_sub(p[c], Q.p_world[j2][c]);
        rn_cross(aw, d, cr);
        term2 = rn_dot(cr, fv);
      }
    }
  }
  // marker total of every dof, lane c keeps dof c.  Base dofs (c < 6): the
  // four level-0 lanes' wrenches through shared memory, in slot order.
  // Joint dofs: lane c pulls, for each bone slot k, the term of the lane that
  // evaluated its joint (k * 8 + lvl[b_k][J]), in slot order.
  __shared__ double wr[FX_PER_BLOCK][SKIN_KW][6];
  const int warp = threadIdx.x >> 5;
  if (l == 0) {
#pragma unroll
    for (int c = 0; c < 6; ++c) wr[warp][k][c] = term[c];
  }
  __syncwarp();
  const int J = (lane >= 6 && lane < SKIN_TAU_MAX) ? B.dof_link[lane] : -1;
  double v = 0.0;
#pragma unroll
  for (int kk = 0; kk < SKIN_KW; ++kk) {
    const int bk = __shfl_sync(0xffffffffu, b, kk * 8);
    const int lv = (J > 0 && bk >= 0) ? B.lvl[bk][J] : -1;
    const int src = kk * 8 + (lv > 0 ? (lv & 7) : 0);
    double jt = __shfl_sync(0xffffffffu, term[0], src);
    if (deep) {
      const double jt2 = __shfl_sync(0xffffffffu, term2, src);
      if (lv >= 8) jt = jt2;
    }
    if (lane < 6) v += wr[warp][kk][lane];
    else if (lv > 0) v += jt;
  }
  __syncwarp();  // wr is rewritten by the warp's next marker
  if (lane < SKIN_TAU_MAX && lane < B.n_dofs) acc += v;
  // CouplingStats (session.hpp:141-143)
  const int sidx = lane - SKIN_TAU_MAX;
  if (sidx >= 0 && sidx < 3) acc += fw[sidx];
  else if (sidx >= 3 && sidx < 6) acc -= fw[sidx - 3];
  else if (sidx == 6) acc += (-fw[0]) * vel[0] + (-fw[1]) * vel[1] + (-fw[2]) * vel[2];
}

/// Block tail: sum the warps' running sums in warp order and add the block's
/// total to the fixed-point accumulators (integer atomics: the accumulated
/// value does not depend on the order the blocks land in).  The blocks spread
/// over SKIN_FIX_REP copies of the accumulators (summed, as integers, by the
/// banded K4's conversion) so ~700 blocks do not queue on the same 50 words.
/// A non-finite or out-of-range (|v| >= 2^19) block sum sets the body's flag
/// word (slot 31), which the conversion turns into NaN (the reference
/// propagates a blown-up fluid's NaN into tau_ext).
template <int NB>
__device__ __forceinline__ void skin_block_red(const double (&acc)[NB], unsigned long long* fixacc) {
  __shared__ double wsum[FX_PER_BLOCK][NB * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int b = 0; b < NB; ++b) wsum[warp][b * 32 + lane] = acc[b];
  __syncthreads();
  if (threadIdx.x < NB * 32 && (threadIdx.x & 31) < SKIN_TAU_MAX + SKIN_NSTAT) {
    double v = wsum[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < FX_PER_BLOCK; ++w) v = v + wsum[w][threadIdx.x];
    unsigned long long* a = fixacc + 64 * (blockIdx.x % SKIN_FIX_REP);
    if (!(fabs(v) < SKIN_FIX_RANGE)) atomicOr(a + (threadIdx.x | 31), 1ull);
    else if (v != 0.0) atomicAdd(a + threadIdx.x, (unsigned long long)__double2ll_rn(v * SKIN_FIX_SCALE));
  }
}

/// Batched envs: one marker's terms straight into its env's fixed-point sums
/// (copy `rep` of the SKIN_FIX_REP replicas; non-finite / out-of-range terms
/// set the flag word, slot 31, as skin_block_red).
__device__ __forceinline__ void skin_red_marker(double v, int lane, unsigned long long* fixacc, int rep) {
  unsigned long long* a = fixacc + 64 * (rep % SKIN_FIX_REP);
  if (lane < SKIN_TAU_MAX + SKIN_NSTAT) {
    if (!(fabs(v) < SKIN_FIX_RANGE)) atomicOr(a + 31, 1ull);
    else if (v != 0.0) atomicAdd(a + lane, (unsigned long long)__double2ll_rn(v * SKIN_FIX_SCALE));
  }
}
