// k_fit.cu — the fused fit-step kernel for the MSE loss (SURVEY §8(a) S2+S3+S4 in one pass per
// work item).
//
// Per work item (<= 32 sorted queries of one brick, one warp, persistent warps in Morton order):
//   1. the queries' shift bounds mh_j >= m_j (computed by k_gather_queries_mh) and the warp's box
//      test over the brick's candidate list -> the item's candidate key ids in the warp's scratch
//      (every skipped pair has a_ij - m_j > cutoff_T, reading R-1);
//   2. forward, lanes = candidate keys, queries broadcast as packed pairs: Z_j = sum_i e^-a_ij,
//      M_j = sum_i e^-a_ij f_i(q_j) (Alg. 1), O_j = M_j / Z_j, the MSE loss and
//      r_j = 2(O_j - o_j)/J (Eq. loss);
//   3. backward over the same candidate ids, lanes = keys (Alg. 2), two
//      red.global.add.v4 per (key, item) into the padded gradient.
// The MSE upstream of a query depends on that query alone, so nothing crosses items.
//
// Item-local expansion. With o the centre of the item's box, q' = q - o and k' = k - o,
//   a_ij log2(e) = bl_i |q'_j - k'_i|^2 = bl_i qq_j - A_i . q'_j - C_i,
//   qq_j = |q'_j|^2, A_i = 2 bl_i k'_i, C_i = -bl_i |k'_i|^2,
// so the exponent of a pair is 4 FMAs (instead of 3 subtractions, 3 for |d|^2 and the scale), and
//   f_i(q_j) = c_i + g_i . (q_j - k_i) = c'_i + g_i . q'_j,  c'_i = c_i - g_i . k'_i.
// Both are exact rewrites; rounding stays at the level of the direct form because |q'|, |k'| are
// small (a cell and the cutoff radius). The forward is unshifted: Z_j = sum 2^(-a_ij log2 e)
// needs m_j < ~100 log2 units, else the item goes to the split kernels (exact shift). The
// backward sums are taken in q' and mapped to d = q' - k' per key at the end:
//   sum t d = sum t q' - k' sum t,   sum u |d|^2 = sum u qq - 2 k' . sum u q' + |k'|^2 sum u,
// with t_ij = r_j p_ij = (r_j / Z_j) 2^(-a_ij log2 e) and u_ij = t_ij (f_i(q_j) - O_j).
// Items without a brick list, or whose Z underflowed, are left to the split kernels.
#include <algorithm>

#include "k_pair.cuh"

namespace ef {

#ifndef FT_B1_UNROLL
#define FT_B1_UNROLL 8  // one-key backward query-pair loop (measured 2/4/8: 8 best by ~0.4%)
#endif
#ifndef FT_B2_UNROLL
#define FT_B2_UNROLL 1  // two-key backward query-pair loop
#endif
#define FT_PRAGMA(x) _Pragma(#x)
#define FT_UNROLL(n) FT_PRAGMA(unroll n)
#ifndef FT_MIN_WARPS
#define FT_MIN_WARPS 16  // warps per SM (measured 16..28; the 16-pair forward needs 128 registers)
#endif
#ifndef FT_BWD2
#define FT_BWD2 1  // backward: two candidate keys per lane
#endif
constexpr int FT_WARPS = 4;
constexpr int FT_BLOCKS = 148 * (FT_MIN_WARPS / FT_WARPS);
static_assert(FT_BLOCKS * FT_WARPS <= SCRATCH_WARPS, "one scratch slot per warp");
// 2^-97: smaller Z_j (m_j > 97 log2 units) -> the exact-shift split path. The unshifted weights
// 2^-a_ij then stay normal floats (>= 2^-126, ex2.approx.ftz flushes below) for every pair within
// the certified cutoff a_ij - m_j <= T = 20 nats = 28.85 log2 units (reading R-1)
constexpr float FT_ZMIN = 6.3109e-30f;

struct FitSmem {
  float4 qa[QW / 2], qb[QW / 2];              // {x'0,x'1,y'0,y'1}, {z'0,z'1,qq0,qq1}
  float4 pc[QW / 2];                          // backward: {rho0,rho1,-O0,-O1}
};

// per-key constants of the expansion
struct KeyX {
  float nbl, C, Ax, Ay, Az, c, gx, gy, gz, kx, ky, kz, kk;
};

__device__ __forceinline__ KeyX key_x(const float4 a, const float4 b, const float3 o) {
  KeyX k;
  k.kx = a.x - o.x;
  k.ky = a.y - o.y;
  k.kz = a.z - o.z;
  k.kk = fmaf(k.kx, k.kx, fmaf(k.ky, k.ky, k.kz * k.kz));
  k.nbl = -a.w;
  k.C = -a.w * k.kk;
  const float bl2 = 2.0f * a.w;
  k.Ax = bl2 * k.kx;
  k.Ay = bl2 * k.ky;
  k.Az = bl2 * k.kz;
  k.c = fmaf(-b.w, k.kz, fmaf(-b.z, k.ky, fmaf(-b.y, k.kx, b.x)));
  k.gx = b.y;
  k.gy = b.z;
  k.gz = b.w;
  return k;
}

// The key's 5 / 8 channel gradients of one item: float reds (bwd_mse_red), or in deterministic mode
// 64-bit fixed-point integer atomics (order-independent sums, reading R-D) in k_backward's layout.
__device__ __forceinline__ void bwd_mse_out(const FitArgs& F, const MseSums& s, const float4 a, const float4 b,
                                            const int id) {
  const int n_nodes = F.f.kv.n_nodes;
  if (!F.gfix) {
    bwd_mse_red(s, a, b, id, n_nodes, F.gpad);
    return;
  }
  const float um = *F.umax;
  const float scale = um > 0.0f ? (float)(1ull << FIX_BITS) / um : 0.0f;
  auto fix_add = [&](unsigned long long* p, float v) {
    const float qv = v * scale;
    if (fabsf(qv) < 4.0e18f) atomicAdd(p, (unsigned long long)(long long)rintf(qv));
    else atomicOr(F.fix_overflow, 1u);
  };
  const float beta = a.w * EF_LN2;
  const float dsv = -beta * s.ss;
  if (id < n_nodes) {
    unsigned long long* gp = F.gfix + (size_t)id * 16;
    fix_add(gp + 0, dsv); fix_add(gp + 1, s.sc); fix_add(gp + 2, s.sgx); fix_add(gp + 3, s.sgy);
    fix_add(gp + 4, s.sgz);
  } else {
    unsigned long long* gp = F.gfix + (size_t)(id - n_nodes) * 16 + 8;
    fix_add(gp + 0, fmaf(-b.y, s.sc, 2.0f * beta * s.sdx));
    fix_add(gp + 1, fmaf(-b.z, s.sc, 2.0f * beta * s.sdy));
    fix_add(gp + 2, fmaf(-b.w, s.sc, 2.0f * beta * s.sdz));
    fix_add(gp + 3, dsv);
    fix_add(gp + 4, s.sc); fix_add(gp + 5, s.sgx); fix_add(gp + 6, s.sgy); fix_add(gp + 7, s.sgz);
  }
}

// Dense kernels: the origin's w is the item's exponent shift max_j mh_j (log2 units), so the
// weights are 2^(shift - a_ij): Z_j >= 1 and no pair is flushed to zero however large m_j is.
__device__ __forceinline__ KeyX key_x(const float4 a, const float4 b, const float4 o) {
  KeyX k = key_x(a, b, make_float3(o.x, o.y, o.z));
  k.C += o.w;
  return k;
}

// exponent (log2 units, <= 0) and polynomial value of one key at a packed query pair
#define FX_EF(K, QA, QB, e, f)                                                   \
  float2 e = __ffma2_rn(make_float2(K.nbl, K.nbl), make_float2(QB.z, QB.w), make_float2(K.C, K.C)); \
  e = __ffma2_rn(make_float2(K.Ax, K.Ax), make_float2(QA.x, QA.y), e);          \
  e = __ffma2_rn(make_float2(K.Ay, K.Ay), make_float2(QA.z, QA.w), e);          \
  e = __ffma2_rn(make_float2(K.Az, K.Az), make_float2(QB.x, QB.y), e);          \
  float2 f = __ffma2_rn(make_float2(K.gx, K.gx), make_float2(QA.x, QA.y), make_float2(K.c, K.c)); \
  f = __ffma2_rn(make_float2(K.gy, K.gy), make_float2(QA.z, QA.w), f);          \
  f = __ffma2_rn(make_float2(K.gz, K.gz), make_float2(QB.x, QB.y), f);

// Forward sums, lanes = keys: one round = 32 candidate keys (records one round ahead, ids two),
// every lane walks the item's query pairs; Z, M per query pair in registers; one transpose-
// reduction per item returns Z_j, M_j to lane j. NPM = query pairs held (8: <= 16 queries).
template <int NPM, class OT>
__device__ __forceinline__ void fwd_accum_x(const KeysView& kv, const uint32_t* L, const uint32_t wn,
                                            const int nact, const OT o, const float4* sQA,
                                            const float4* sQB, float2 (&Z)[NPM], float2 (&M)[NPM]) {
  const int lane = threadIdx.x & 31;
  const int npairs = (nact + 1) >> 1;
  auto round = [&](const KeyX& K) {
#define FX_PAIR(pp)                                  \
  {                                                  \
    const float4 QA = sQA[pp], QB = sQB[pp];         \
    FX_EF(K, QA, QB, e, f)                           \
    const float2 w = make_float2(ex2f(e.x), ex2f(e.y)); \
    Z[pp] = __fadd2_rn(Z[pp], w);                    \
    M[pp] = __ffma2_rn(w, f, M[pp]);                 \
  }
    // groups of 4 pairs without a branch inside; a last group of 1-2 pairs runs as 2, of 3 as 4
    // (padding slots are idle queries with qq = 1e30: weight exactly 0)
#pragma unroll
    for (int pg = 0; pg < NPM; pg += 4) {
      const int rem = npairs - pg;
      if (rem >= 3) {
        FX_PAIR(pg) FX_PAIR(pg + 1) FX_PAIR(pg + 2) FX_PAIR(pg + 3)
      } else if (rem > 0) {
        FX_PAIR(pg) FX_PAIR(pg + 1)
      }
    }
#undef FX_PAIR
  };
  // idle lanes of the last round get a far-away zero key: weight exactly 0
  const float4 far_a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t id1 = ((uint32_t)lane < wn) ? L[lane] : 0u;
  uint32_t id2 = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
  float4 a1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1]) : far_a;
  float4 b1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
  for (uint32_t base = 0; base < wn; base += 32) {
    const uint32_t k = base + lane;
    const float4 ka = a1, kb = b1;
    id1 = id2;
    id2 = (k + 64 < wn) ? L[k + 64] : 0u;
    a1 = far_a;
    b1 = z4;
    if (k + 32 < wn) {
      a1 = __ldg(&kv.grid_raw[2 * id1]);
      b1 = __ldg(&kv.grid_raw[2 * id1 + 1]);
    }
    round(key_x(ka, kb, o));
  }
}

// transpose-reduce {Zx, Zy, Mx, My} of every pair; lane j then fetches its query's totals
template <int NPM>
__device__ __forceinline__ void fwd_reduce_x(const float2 (&Z)[NPM], const float2 (&M)[NPM], float& Zj, float& Mj) {
  const int lane = threadIdx.x & 31;
  if (NPM == 8) {
    float v[32];
#pragma unroll
    for (int pp = 0; pp < 8; ++pp) {
      v[4 * pp] = Z[pp].x; v[4 * pp + 1] = Z[pp].y; v[4 * pp + 2] = M[pp].x; v[4 * pp + 3] = M[pp].y;
    }
    warp_reduce_scatter<32>(v, lane);  // lane l holds value l
    const int j = lane & 15;
    Zj = __shfl_sync(~0u, v[0], 4 * (j >> 1) + (j & 1));
    Mj = __shfl_sync(~0u, v[0], 4 * (j >> 1) + 2 + (j & 1));
  } else {
    float v[64];
#pragma unroll
    for (int pp = 0; pp < NPM; ++pp) {
      v[4 * pp] = Z[pp].x; v[4 * pp + 1] = Z[pp].y; v[4 * pp + 2] = M[pp].x; v[4 * pp + 3] = M[pp].y;
    }
    warp_reduce_scatter<64>(v, lane);  // lane l holds values 2l, 2l+1
    const int src = lane & ~1;
    const float z0 = __shfl_sync(~0u, v[0], src), z1 = __shfl_sync(~0u, v[1], src);
    const float m0 = __shfl_sync(~0u, v[0], src + 1), m1 = __shfl_sync(~0u, v[1], src + 1);
    Zj = (lane & 1) ? z1 : z0;
    Mj = (lane & 1) ? m1 : m0;
  }
}

template <int NPM, class OT>
__device__ __forceinline__ void fwd_sums_x(const KeysView& kv, const uint32_t* L, const uint32_t wn,
                                           const int nact, const OT o, const float4* sQA,
                                           const float4* sQB, float& Zj, float& Mj) {
  float2 Z[NPM], M[NPM];
#pragma unroll
  for (int pp = 0; pp < NPM; ++pp) {
    Z[pp] = make_float2(0.f, 0.f);
    M[pp] = make_float2(0.f, 0.f);
  }
  fwd_accum_x<NPM, OT>(kv, L, wn, nact, o, sQA, sQB, Z, M);
  fwd_reduce_x<NPM>(Z, M, Zj, Mj);
}

// Backward sums of one key (lane) over the item's query pairs in q' coordinates, mapped to the
// d = q - k sums of MseSums (k_pair.cuh) at the end.
__device__ __forceinline__ MseSums bwd_sums_x(const KeyX& K, const int npairs, const float4* pA, const float4* pB,
                                              const float4* pC) {
  float2 Sc = make_float2(0.f, 0.f), Stx = Sc, Sty = Sc, Stz = Sc, Su = Sc, Sux = Sc, Suy = Sc, Suz = Sc, Suq = Sc;
  auto pair = [&](const int jp) {
    const float4 QA = pA[jp], QB = pB[jp], QC = pC[jp];
    FX_EF(K, QA, QB, e, f)
    const float2 p = make_float2(ex2f(e.x), ex2f(e.y));
    const float2 del = __fadd2_rn(f, make_float2(QC.z, QC.w));
    const float2 t = __fmul2_rn(make_float2(QC.x, QC.y), p);
    const float2 u = __fmul2_rn(t, del);
    Sc = __fadd2_rn(Sc, t);
    Stx = __ffma2_rn(t, make_float2(QA.x, QA.y), Stx);
    Sty = __ffma2_rn(t, make_float2(QA.z, QA.w), Sty);
    Stz = __ffma2_rn(t, make_float2(QB.x, QB.y), Stz);
    Su = __fadd2_rn(Su, u);
    Sux = __ffma2_rn(u, make_float2(QA.x, QA.y), Sux);
    Suy = __ffma2_rn(u, make_float2(QA.z, QA.w), Suy);
    Suz = __ffma2_rn(u, make_float2(QB.x, QB.y), Suz);
    Suq = __ffma2_rn(u, make_float2(QB.z, QB.w), Suq);
  };
  // an even number of pairs (a padding slot is an idle query: qq = 1e30, rho = 0 -> exactly 0)
  const int np2 = (npairs + 1) & ~1;
  FT_UNROLL(FT_B1_UNROLL)
  for (int jp = 0; jp < np2; jp += 2) {
    pair(jp);
    pair(jp + 1);
  }
  const float sc = Sc.x + Sc.y, su = Su.x + Su.y;
  const float sux = Sux.x + Sux.y, suy = Suy.x + Suy.y, suz = Suz.x + Suz.y;
  MseSums s;
  s.sc = sc;
  s.sgx = fmaf(-K.kx, sc, Stx.x + Stx.y);
  s.sgy = fmaf(-K.ky, sc, Sty.x + Sty.y);
  s.sgz = fmaf(-K.kz, sc, Stz.x + Stz.y);
  s.ss = fmaf(K.kk, su, fmaf(-2.0f * K.kx, sux, fmaf(-2.0f * K.ky, suy, fmaf(-2.0f * K.kz, suz, Suq.x + Suq.y))));
  s.sdx = fmaf(-K.kx, su, sux);
  s.sdy = fmaf(-K.ky, su, suy);
  s.sdz = fmaf(-K.kz, su, suz);
  return s;
}

// Two keys per lane (rounds of 64 keys): every query pair loaded from shared memory serves both,
// halving the backward's shared-memory wavefronts per pair and doubling the independent chains.
__device__ __forceinline__ void bwd_sums_x2(const KeyX& KA, const KeyX& KB, const int npairs, const float4* pA,
                                            const float4* pB, const float4* pC, MseSums& sa, MseSums& sb) {
  float2 Sc[2], Stx[2], Sty[2], Stz[2], Su[2], Sux[2], Suy[2], Suz[2], Suq[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    Sc[u] = Stx[u] = Sty[u] = Stz[u] = Su[u] = Sux[u] = Suy[u] = Suz[u] = Suq[u] = make_float2(0.f, 0.f);
  }
  auto pair = [&](const int u, const KeyX& K, const float4 QA, const float4 QB, const float4 QC) {
    FX_EF(K, QA, QB, e, f)
    const float2 p = make_float2(ex2f(e.x), ex2f(e.y));
    const float2 del = __fadd2_rn(f, make_float2(QC.z, QC.w));
    const float2 t = __fmul2_rn(make_float2(QC.x, QC.y), p);
    const float2 uu = __fmul2_rn(t, del);
    Sc[u] = __fadd2_rn(Sc[u], t);
    Stx[u] = __ffma2_rn(t, make_float2(QA.x, QA.y), Stx[u]);
    Sty[u] = __ffma2_rn(t, make_float2(QA.z, QA.w), Sty[u]);
    Stz[u] = __ffma2_rn(t, make_float2(QB.x, QB.y), Stz[u]);
    Su[u] = __fadd2_rn(Su[u], uu);
    Sux[u] = __ffma2_rn(uu, make_float2(QA.x, QA.y), Sux[u]);
    Suy[u] = __ffma2_rn(uu, make_float2(QA.z, QA.w), Suy[u]);
    Suz[u] = __ffma2_rn(uu, make_float2(QB.x, QB.y), Suz[u]);
    Suq[u] = __ffma2_rn(uu, make_float2(QB.z, QB.w), Suq[u]);
  };
  const int np2 = (npairs + 1) & ~1;
  FT_UNROLL(FT_B2_UNROLL)
  for (int jp = 0; jp < np2; jp += 2) {
    const float4 QA0 = pA[jp], QB0 = pB[jp], QC0 = pC[jp];
    const float4 QA1 = pA[jp + 1], QB1 = pB[jp + 1], QC1 = pC[jp + 1];
    pair(0, KA, QA0, QB0, QC0);
    pair(1, KB, QA0, QB0, QC0);
    pair(0, KA, QA1, QB1, QC1);
    pair(1, KB, QA1, QB1, QC1);
  }
  auto fin = [&](const int u, const KeyX& K, MseSums& s) {
    const float sc = Sc[u].x + Sc[u].y, su = Su[u].x + Su[u].y;
    const float sux = Sux[u].x + Sux[u].y, suy = Suy[u].x + Suy[u].y, suz = Suz[u].x + Suz[u].y;
    s.sc = sc;
    s.sgx = fmaf(-K.kx, sc, Stx[u].x + Stx[u].y);
    s.sgy = fmaf(-K.ky, sc, Sty[u].x + Sty[u].y);
    s.sgz = fmaf(-K.kz, sc, Stz[u].x + Stz[u].y);
    s.ss = fmaf(K.kk, su, fmaf(-2.0f * K.kx, sux, fmaf(-2.0f * K.ky, suy, fmaf(-2.0f * K.kz, suz, Suq[u].x + Suq[u].y))));
    s.sdx = fmaf(-K.kx, su, sux);
    s.sdy = fmaf(-K.ky, su, suy);
    s.sdz = fmaf(-K.kz, su, suz);
  };
  fin(0, KA, sa);
  fin(1, KB, sb);
}

// The backward over candidate ids L[0 .. wn) (rounds of 64: two keys per lane), the item's query
// table in S (qa, qb: positions; pc: rho, -O).
__device__ __forceinline__ void bwd_pass_x(const FitArgs& F, const uint32_t* L, const uint32_t wn,
                                           const int npairs, const float3 o, FitSmem& S) {
  const KeysView& kv = F.f.kv;
  const int lane = threadIdx.x & 31;
#if FT_BWD2
  // rounds of 64 candidates: lane keys base + lane and base + 32 + lane (records one round ahead;
  // a missing second key is a far zero key whose sums are discarded)
  const float4 far_a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t iA = ((uint32_t)lane < wn) ? L[lane] : 0u, iB = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
  float4 aA = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * iA]) : far_a;
  float4 bA = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * iA + 1]) : z4;
  float4 aB = ((uint32_t)lane + 32 < wn) ? __ldg(&kv.grid_raw[2 * iB]) : far_a;
  float4 bB = ((uint32_t)lane + 32 < wn) ? __ldg(&kv.grid_raw[2 * iB + 1]) : z4;
  for (uint32_t base = 0; base < wn; base += 64) {
    const uint32_t k = base + lane;
    const uint32_t idA = iA, idB = iB;
    const float4 a0 = aA, b0 = bA, a1 = aB, b1 = bB;
    iA = (k + 64 < wn) ? L[k + 64] : 0u;
    iB = (k + 96 < wn) ? L[k + 96] : 0u;
    aA = far_a; bA = z4; aB = far_a; bB = z4;
    if (k + 64 < wn) {
      ld_rec(&kv.grid_raw[2 * iA], aA, bA);
    }
    if (k + 96 < wn) {
      ld_rec(&kv.grid_raw[2 * iB], aB, bB);
    }
    if (base + 32 < wn) {  // warp-uniform: two keys per lane
      MseSums s0, s1;
      bwd_sums_x2(key_x(a0, b0, o), key_x(a1, b1, o), npairs, S.qa, S.qb, S.pc, s0, s1);
      if (k < wn) bwd_mse_out(F, s0, a0, b0, (int)idA);
      if (k + 32 < wn) bwd_mse_out(F, s1, a1, b1, (int)idB);
    } else if (k < wn) {
      const MseSums ms = bwd_sums_x(key_x(a0, b0, o), npairs, S.qa, S.qb, S.pc);
      bwd_mse_out(F, ms, a0, b0, (int)idA);
    }
  }
#else
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t id1 = ((uint32_t)lane < wn) ? L[lane] : 0u;
  uint32_t id2 = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
  float4 a1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1]) : z4;
  float4 b1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
  for (uint32_t base = 0; base < wn; base += 32) {
    const uint32_t k = base + lane;
    const uint32_t id = id1;
    const float4 a = a1, b = b1;
    id1 = id2;
    id2 = (k + 64 < wn) ? L[k + 64] : 0u;
    if (k + 32 < wn) {
      ld_rec(&kv.grid_raw[2 * id1], a1, b1);
    }
    if (k < wn) {
      const MseSums ms = bwd_sums_x(key_x(a, b, o), npairs, S.qa, S.qb, S.pc);
      bwd_mse_out(F, ms, a, b, (int)id);
    }
  }
#endif
}

// Items of overflowed bricks (C4b at 128^3: ~35k keys per brick).
__device__ __forceinline__ void fit_item_enum(const FitArgs& F, const uint32_t item, FitSmem& S, uint32_t* Lw) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  const bool dense = F.iota != nullptr;  // cutoff_T = inf: every key is a candidate, no lists
  if (it.z < 0) {  // out-of-domain queries: the split kernels
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  const uint32_t nb = dense ? 0u : __ldg(&kv.bl_n[it.z]);
  // an overflowed brick (no list): candidates by direct enumeration of the lattice cells around
  // the item, in chunks of ENUM_CAP ids (each chunk re-enumerates: cheap next to its pair work)
  const bool enum_mode = !dense && nb == BL_OVERFLOW;
  // 1. box, candidate ids
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY;
  if (act) {
    q = A.qs[js];
    mh = A.qmh[js];  // shift bound from k_gather_queries_mh
  }
  Box box = warp_box(act, q.x, q.y, q.z, mh);
  box.thr += A.T_l;
  const float3 o = make_float3(0.5f * (box.lx + box.hx), 0.5f * (box.ly + box.hy), 0.5f * (box.lz + box.hz));
  __syncwarp();  // the previous item's readers of L and S are done
  uint32_t total = 0;  // candidates of the item (all chunks)
  const uint32_t* L = Lw;  // the candidate ids the passes read
  // builds chunk c of the candidate ids into Lw (or points L at them); returns its length
  auto build = [&](const uint32_t c) -> uint32_t {
    if (dense) {  // every enabled key in id order (coalesced record loads)
      L = F.iota;
      total = F.iota_n;
      return total;
    }
    uint32_t cnt = 0;
    if (!enum_mode) {
      stream_list<4>(kv, kv.bl_pool + __ldg(&kv.bl_off[it.z]), nb, box, [&](bool pass, uint32_t id) {
        const uint32_t bal = __ballot_sync(~0u, pass);
        if (pass) Lw[cnt + __popc(bal & lanemask_lt())] = id;
        cnt += __popc(bal);
      });
      total = cnt;
      return cnt;
    }
    const uint32_t lo = c * (uint32_t)ENUM_CAP;
    enumerate(kv, box, [&](bool pass, uint32_t kp, float4) {
      const uint32_t bal = __ballot_sync(~0u, pass);
      const uint32_t idx = cnt + __popc(bal & lanemask_lt());
      if (pass && idx >= lo && idx < lo + (uint32_t)ENUM_CAP) Lw[idx - lo] = (uint32_t)__ldg(&kv.kid[kp]);
      cnt += __popc(bal);
    });
    total = cnt;
    return cnt > lo ? min(cnt - lo, (uint32_t)ENUM_CAP) : 0u;
  };
  // 2. forward
  const float qx = q.x - o.x, qy = q.y - o.y, qz = q.z - o.z;
  const float qq = act ? fmaf(qx, qx, fmaf(qy, qy, qz * qz)) : 1e30f;  // idle slot: weight 0 (finite: u qq = 0)
  {
    const float xo = __shfl_xor_sync(~0u, qx, 1), yo = __shfl_xor_sync(~0u, qy, 1);
    const float zo = __shfl_xor_sync(~0u, qz, 1), qo = __shfl_xor_sync(~0u, qq, 1);
    if ((lane & 1) == 0) {
      S.qa[lane >> 1] = make_float4(qx, xo, qy, yo);
      S.qb[lane >> 1] = make_float4(qz, zo, qq, qo);
    }
  }
  uint32_t wn = build(0);
  __syncwarp();
  float Z, M;
  if (!enum_mode) {
    if (IQ <= 16 || nact <= 16) fwd_sums_x<8>(kv, L, wn, nact, o, S.qa, S.qb, Z, M);
    else fwd_sums_x<(IQ > 16 ? 16 : 8)>(kv, L, wn, nact, o, S.qa, S.qb, Z, M);
  } else {
    float2 Za[16], Ma[16];
#pragma unroll
    for (int pp = 0; pp < 16; ++pp) Za[pp] = Ma[pp] = make_float2(0.f, 0.f);
    for (uint32_t c = 0;; ++c) {
      if (c > 0) {
        __syncwarp();  // readers of the previous chunk are done
        wn = build(c);
        __syncwarp();
      }
      fwd_accum_x<16>(kv, L, wn, nact, o, S.qa, S.qb, Za, Ma);
      if ((c + 1) * (uint32_t)ENUM_CAP >= total) break;
    }
    fwd_reduce_x<16>(Za, Ma, Z, M);
  }
  const bool bad = act && !(Z >= FT_ZMIN && isfinite(Z) && isfinite(M));
  if (__any_sync(~0u, bad)) {  // Z underflow (far queries): the split kernels shift exactly
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  float O = 0.f, rho = 0.f, lossj = 0.f;
  if (act) {
    const float iz = 1.0f / Z;
    O = M * iz;
    const float diff = O - q.w;
    const float r = 2.0f * diff * A.inv_J;
    rho = r * iz;  // t_ij = r_j p_ij = (r_j / Z_j) 2^(-a_ij log2 e)
    lossj = diff * diff * A.inv_J;
    if (A.O) A.O[A.perm[js]] = O;
  }
  for (int s = 16; s > 0; s >>= 1) lossj += __shfl_xor_sync(~0u, lossj, s);
  if (lane == 0) {
    A.loss_part[item] = lossj;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)total * (unsigned long long)nact);
  }
  // 3. backward over the same candidates
  {
    const float nO = -O;
    const float ro = __shfl_xor_sync(~0u, rho, 1), nOo = __shfl_xor_sync(~0u, nO, 1);
    if ((lane & 1) == 0) S.pc[lane >> 1] = make_float4(rho, ro, nO, nOo);
  }
  __syncwarp();
  const uint32_t nchunks = enum_mode ? (total + ENUM_CAP - 1) / ENUM_CAP : 1u;
  for (uint32_t c = 0; c < nchunks; ++c) {
    if (nchunks > 1) {  // the scratch holds the last forward chunk: rebuild chunk c
      __syncwarp();
      wn = build(c);
      __syncwarp();
    }
    bwd_pass_x(F, L, wn, (nact + 1) >> 1, o, S);
  }
}

// Item types the list builder hands on
constexpr uint32_t IT_NORMAL = 0, IT_ENUM = 1, IT_SKIP = 2;

// Part 1 of a work item: the box and its candidate ids (into Lw, or the all-keys list in dense
// mode). Returns IT_NORMAL with L, wn, o set; IT_ENUM for an overflowed brick (fit_item_enum
// builds its own chunks); IT_SKIP for out-of-domain items (queued for the split kernels).
__device__ __forceinline__ uint32_t fit_item_build(const FitArgs& F, const uint32_t item, const int4 it, uint32_t* Lw,
                                                   const uint32_t*& L, uint32_t& wn, float3& o) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int nact = it.y;
  const bool dense = F.iota != nullptr;  // cutoff_T = inf: every key is a candidate, no lists
  if (F.pre) {  // k_fit_lists built this item's candidate ids (unless it had no list / no room)
    const uint32_t pn = __ldcg(&A.wl_n[item]);
    if (pn != BL_OVERFLOW) {
      L = A.wl_pool + __ldcg(&A.wl_off[item]);
      wn = pn;
      const float4 oo = __ldcg(&F.item_o[item]);
      o = make_float3(oo.x, oo.y, oo.z);
      return IT_NORMAL;
    }
  }
  uint32_t nb = BL_OVERFLOW;
  if (it.z >= 0) nb = dense ? 0u : __ldg(&kv.bl_n[it.z]);
  if (nb == BL_OVERFLOW) {
    if (it.z >= 0) return IT_ENUM;  // an overflowed brick: candidates by direct enumeration
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;  // out of domain: split kernels
    return IT_SKIP;
  }
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY;
  if (act) {
    q = A.qs[js];
    mh = A.qmh[js];  // shift bound from k_gather_queries_mh
  }
  Box box = warp_box(act, q.x, q.y, q.z, mh);
  box.thr += A.T_l;
  o = make_float3(0.5f * (box.lx + box.hx), 0.5f * (box.ly + box.hy), 0.5f * (box.lz + box.hz));
  __syncwarp();  // the previous item's readers of L are done
  wn = 0;
  L = Lw;
  if (dense) {  // every enabled key in id order (coalesced record loads)
    L = F.iota;
    wn = F.iota_n;
  } else {
    uint32_t cnt = 0;
    stream_list<4>(kv, kv.bl_pool + __ldg(&kv.bl_off[it.z]), nb, box, [&](bool pass, uint32_t id) {
      const uint32_t bal = __ballot_sync(~0u, pass);
      if (pass) Lw[cnt + __popc(bal & lanemask_lt())] = id;
      cnt += __popc(bal);
    });
    wn = cnt;
  }
  return IT_NORMAL;
}

// Part 2 of a work item: forward, loss, backward over the candidate ids L[0 .. wn).
__device__ __forceinline__ void fit_item_compute(const FitArgs& F, const uint32_t item, const int4 it, FitSmem& S,
                                                 const uint32_t* L, const uint32_t wn, const float3 o) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int nact = it.y;
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  if (act) q = A.qs[js];
  __syncwarp();  // the previous item's readers of S are done
  // 2. forward
  const float qx = q.x - o.x, qy = q.y - o.y, qz = q.z - o.z;
  const float qq = act ? fmaf(qx, qx, fmaf(qy, qy, qz * qz)) : 1e30f;  // idle slot: weight 0 (finite: u qq = 0)
  {
    const float xo = __shfl_xor_sync(~0u, qx, 1), yo = __shfl_xor_sync(~0u, qy, 1);
    const float zo = __shfl_xor_sync(~0u, qz, 1), qo = __shfl_xor_sync(~0u, qq, 1);
    if ((lane & 1) == 0) {
      S.qa[lane >> 1] = make_float4(qx, xo, qy, yo);
      S.qb[lane >> 1] = make_float4(qz, zo, qq, qo);
    }
  }
  __syncwarp();
  float Z, M;
  if (IQ <= 16 || nact <= 16) fwd_sums_x<8>(kv, L, wn, nact, o, S.qa, S.qb, Z, M);
  else fwd_sums_x<(IQ > 16 ? 16 : 8)>(kv, L, wn, nact, o, S.qa, S.qb, Z, M);
  const bool bad = act && !(Z >= FT_ZMIN && isfinite(Z) && isfinite(M));
  if (__any_sync(~0u, bad)) {  // Z underflow (far queries): the split kernels shift exactly
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  float O = 0.f, rho = 0.f, lossj = 0.f;
  if (act) {
    const float iz = 1.0f / Z;
    O = M * iz;
    const float diff = O - q.w;
    const float r = 2.0f * diff * A.inv_J;
    rho = r * iz;  // t_ij = r_j p_ij = (r_j / Z_j) 2^(-a_ij log2 e)
    lossj = diff * diff * A.inv_J;
    if (A.O) A.O[A.perm[js]] = O;
  }
  for (int s = 16; s > 0; s >>= 1) lossj += __shfl_xor_sync(~0u, lossj, s);
  if (lane == 0) {
    A.loss_part[item] = lossj;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)wn * (unsigned long long)nact);
  }
  // 3. backward over the same candidates
  {
    const float nO = -O;
    const float ro = __shfl_xor_sync(~0u, rho, 1), nOo = __shfl_xor_sync(~0u, nO, 1);
    if ((lane & 1) == 0) S.pc[lane >> 1] = make_float4(rho, ro, nO, nOo);
  }
  __syncwarp();
  const int npairs = (nact + 1) >> 1;
#if FT_BWD2
  // rounds of 64 candidates: lane keys base + lane and base + 32 + lane (records one round ahead;
  // a missing second key is a far zero key whose sums are discarded)
  // ids two rounds ahead, records one round ahead: a record gather never waits on an id load
  // issued in the same round
  const float4 far_a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t iA = ((uint32_t)lane < wn) ? L[lane] : 0u, iB = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
  uint32_t iA2 = ((uint32_t)lane + 64 < wn) ? L[lane + 64] : 0u, iB2 = ((uint32_t)lane + 96 < wn) ? L[lane + 96] : 0u;
  float4 aA = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * iA]) : far_a;
  float4 bA = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * iA + 1]) : z4;
  float4 aB = ((uint32_t)lane + 32 < wn) ? __ldg(&kv.grid_raw[2 * iB]) : far_a;
  float4 bB = ((uint32_t)lane + 32 < wn) ? __ldg(&kv.grid_raw[2 * iB + 1]) : z4;
  for (uint32_t base = 0; base < wn; base += 64) {
    const uint32_t k = base + lane;
    const uint32_t idA = iA, idB = iB;
    const float4 a0 = aA, b0 = bA, a1 = aB, b1 = bB;
    iA = iA2;
    iB = iB2;
    iA2 = (k + 128 < wn) ? L[k + 128] : 0u;
    iB2 = (k + 160 < wn) ? L[k + 160] : 0u;
    aA = far_a; bA = z4; aB = far_a; bB = z4;
    if (k + 64 < wn) {
      ld_rec(&kv.grid_raw[2 * iA], aA, bA);
    }
    if (k + 96 < wn) {
      ld_rec(&kv.grid_raw[2 * iB], aB, bB);
    }
    if (base + 32 < wn) {  // warp-uniform: two keys per lane
      MseSums s0, s1;
      bwd_sums_x2(key_x(a0, b0, o), key_x(a1, b1, o), npairs, S.qa, S.qb, S.pc, s0, s1);
      if (k < wn) bwd_mse_out(F, s0, a0, b0, (int)idA);
      if (k + 32 < wn) bwd_mse_out(F, s1, a1, b1, (int)idB);
    } else if (k < wn) {
      const MseSums ms = bwd_sums_x(key_x(a0, b0, o), npairs, S.qa, S.qb, S.pc);
      bwd_mse_out(F, ms, a0, b0, (int)idA);
    }
  }
#else
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t id1 = ((uint32_t)lane < wn) ? L[lane] : 0u;
  uint32_t id2 = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
  float4 a1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1]) : z4;
  float4 b1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
  for (uint32_t base = 0; base < wn; base += 32) {
    const uint32_t k = base + lane;
    const uint32_t id = id1;
    const float4 a = a1, b = b1;
    id1 = id2;
    id2 = (k + 64 < wn) ? L[k + 64] : 0u;
    if (k + 32 < wn) {
      ld_rec(&kv.grid_raw[2 * id1], a1, b1);
    }
    if (k < wn) {
      const MseSums ms = bwd_sums_x(key_x(a, b, o), npairs, S.qa, S.qb, S.pc);
      bwd_mse_out(F, ms, a, b, (int)id);
    }
  }
#endif
}

// the item record is loaded once here and handed to both parts
__device__ __forceinline__ void fit_item(const FitArgs& F, const uint32_t item, FitSmem& S, uint32_t* Lw) {
  const uint32_t* L;
  uint32_t wn;
  float3 o;
  const int4 it = F.f.items[item];
  const uint32_t t = fit_item_build(F, item, it, Lw, L, wn, o);
  if (t == IT_ENUM) fit_item_enum(F, item, S, Lw);
  else if (t == IT_NORMAL) fit_item_compute(F, item, it, S, L, wn, o);
}

#ifndef FT_HSPLIT
#define FT_HSPLIT 4  // the heavy class is fetched from this many interleaved Morton streams
#endif
// fetch g: while g < the heavy-class count, the item at stream g % S, position g / S (the heavy
// items in flight come from S regions of the surface: fewer concurrent reds on the same keys)
__device__ __forceinline__ int64_t fetch_item_hsplit(const FitArgs& F) {
  const uint32_t n = *F.f.n_items, nh = *F.n_heavy, len = (nh + FT_HSPLIT - 1) / FT_HSPLIT;
  for (;;) {
    uint32_t g = 0;
    if ((threadIdx.x & 31) == 0) g = atomicAdd(&F.f.ds->fit_next, 1u);
    g = __shfl_sync(~0u, g, 0);
    if (g >= len * FT_HSPLIT) {
      const uint32_t it = nh + (g - len * FT_HSPLIT);
      return it < n ? (int64_t)it : -1;
    }
    const uint32_t it = (g % FT_HSPLIT) * len + g / FT_HSPLIT;
    if (it < nh) return (int64_t)it;
  }
}

__global__ void __launch_bounds__(32 * FT_WARPS, FT_MIN_WARPS / FT_WARPS) k_fit(const FitArgs F) {
  __shared__ FitSmem smem[FT_WARPS];
  const int w = threadIdx.x >> 5;
  uint32_t* L = F.scratch + (size_t)(blockIdx.x * FT_WARPS + w) * SCRATCH_STRIDE;
  for (;;) {
#if FT_HSPLIT > 1
    const int64_t item = F.n_heavy ? fetch_item_hsplit(F) : fetch_item(&F.f.ds->fit_next, F.f.n_items, nullptr, nullptr);
#else
    const int64_t item = fetch_item(&F.f.ds->fit_next, F.f.n_items, nullptr, nullptr);
#endif
    if (item < 0) break;
    fit_item(F, (uint32_t)item, smem[w], L);
  }
}

// The list phase of k_fit as its own launch: per item, the box of its queries (threshold
// max_j mh_j + T) tested against every key of its brick's list, the passing ids written to the
// item's slice of wl_pool (reserved: the brick list length), and the box centre. Latency-bound
// (id -> key record -> test): few registers, 16 warps per CTA, the whole SM's warp slots.
constexpr int FL_WARPS = 16;
#ifndef FL_UNROLL
#define FL_UNROLL 2  // list batches of 32 in flight per warp (48 warps/SM hide the rest)
#endif
__global__ void __launch_bounds__(32 * FL_WARPS, 3) k_fit_lists(const FitArgs F) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const uint32_t item = blockIdx.x * FL_WARPS + (threadIdx.x >> 5);
  if (item >= *A.n_items) return;
  const int4 it = A.items[item];
  const bool act = lane < it.y;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY;
  if (act) {
    q = A.qs[js];
    mh = A.qmh[js];
  }
  uint32_t nb = BL_OVERFLOW, base = 0;
  if (it.z >= 0) nb = __ldg(&kv.bl_n[it.z]);
  if (lane == 0 && nb != BL_OVERFLOW) base = atomicAdd(&A.ds->wl_top, nb);
  base = __shfl_sync(~0u, base, 0);
  Box box = warp_box(act, q.x, q.y, q.z, mh);
  box.thr += A.T_l;
  if (nb == BL_OVERFLOW || base + nb > A.wl_cap) {  // k_fit handles the item (enumerate / split kernels)
    if (lane == 0) A.wl_n[item] = BL_OVERFLOW;
    return;
  }
  uint32_t cnt = 0;
  uint32_t* out = A.wl_pool + base;
  stream_list<FL_UNROLL>(kv, kv.bl_pool + __ldg(&kv.bl_off[it.z]), nb, box, [&](bool pass, uint32_t id) {
    const uint32_t bal = __ballot_sync(~0u, pass);
    if (pass) out[cnt + __popc(bal & lanemask_lt())] = id;
    cnt += __popc(bal);
  });
  if (lane == 0) {
    A.wl_off[item] = base;
    A.wl_n[item] = cnt;
    F.item_o[item] = make_float4(0.5f * (box.lx + box.hx), 0.5f * (box.ly + box.hy), 0.5f * (box.lz + box.hz), 0.f);
  }
}

// ------------------------------------------------------------------ dense mode (cutoff_T = inf)
// every (query, key) pair, the paper's own Table 4 setting.
// With few queries (Table 4: J = 16384, ~550 work items) one warp per item leaves most of the 2368
// warp slots idle, so the pass is split three ways:
//   k_dense_fwd      (item, key slice) units: the slice's partial Z_j, M_j of the item's queries
//                    (lanes = keys, the item-local expansion of k_fit's forward);
//   k_dense_combine  per item: Z_j, M_j summed over the slices in slice order, O_j, the MSE loss,
//                    rho_j = r_j / Z_j and the item's packed query table for the backward;
//   k_dense_bwd      (block of 64 keys, group of items) units, key-stationary as Alg. 2
//                    (PAPER.md:L540-568): two keys per lane accumulate over every query of the
//                    group in registers (direct form, d = q - k), two red.v4 per key and group.
constexpr int DN_WARPS = 4;
// item box diagonal^2 above which the dense forward uses the direct form: the expansion about the
// box centre rounds the exponent by ~eps bl D^2 (2e-5 log2 units at D = 0.6, beta = e^7)
#ifndef DN_LOCAL2_V
#define DN_LOCAL2_V 0.36f
#endif
constexpr float DN_LOCAL2 = DN_LOCAL2_V;

__global__ void __launch_bounds__(32 * DN_WARPS) k_dense_fwd(const FitArgs F, float2* __restrict__ zm, int S,
                                                             uint32_t ks) {
  __shared__ FitSmem smem[DN_WARPS];
  FitSmem& Sm = smem[threadIdx.x >> 5];
  const FwdArgs& A = F.f;
  const uint32_t u = blockIdx.x * DN_WARPS + (threadIdx.x >> 5);
  const uint32_t item = u / (uint32_t)S, sl = u % (uint32_t)S;
  if (item >= *A.n_items) return;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  const float4 q = act ? A.qs[js] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float mh = act ? A.qmh[js] : -INFINITY;
  const Box box = warp_box(act, q.x, q.y, q.z, mh);
  const float4 o = make_float4(0.5f * (box.lx + box.hx), 0.5f * (box.ly + box.hy), 0.5f * (box.lz + box.hz), box.thr);
  const uint32_t k0 = sl * ks;
  const uint32_t wn = k0 < F.iota_n ? min(ks, F.iota_n - k0) : 0u;
  float Z, M;
  const float ex = box.hx - box.lx, ey = box.hy - box.ly, ez = box.hz - box.lz;
  if (fmaf(ex, ex, fmaf(ey, ey, ez * ez)) > DN_LOCAL2) {
    // a spread item (small J: a Morton run of the whole domain): the expansion about its centre
    // would round the exponent by ~eps bl |q - o|^2, so the direct form d = q - k (k_pair.cuh)
    {
      const float xo = __shfl_xor_sync(~0u, q.x, 1), yo = __shfl_xor_sync(~0u, q.y, 1);
      const float zo = __shfl_xor_sync(~0u, q.z, 1);
      const float sh = act ? o.w : -INFINITY, so = __shfl_xor_sync(~0u, sh, 1);
      if ((lane & 1) == 0) {
        Sm.qa[lane >> 1] = make_float4(q.x, xo, q.y, yo);
        Sm.qb[lane >> 1] = make_float4(q.z, zo, sh, so);
      }
    }
    __syncwarp();
    if (nact <= 16) fwd_keys_sums<8>(A.kv, F.iota + k0, wn, nact, Sm.qa, Sm.qb, Z, M);
    else fwd_keys_sums<16>(A.kv, F.iota + k0, wn, nact, Sm.qa, Sm.qb, Z, M);
    zm[(size_t)u * 32 + lane] = make_float2(Z, M);
    return;
  }
  const float qx = q.x - o.x, qy = q.y - o.y, qz = q.z - o.z;
  const float qq = act ? fmaf(qx, qx, fmaf(qy, qy, qz * qz)) : 1e30f;
  {
    const float xo = __shfl_xor_sync(~0u, qx, 1), yo = __shfl_xor_sync(~0u, qy, 1);
    const float zo = __shfl_xor_sync(~0u, qz, 1), qo = __shfl_xor_sync(~0u, qq, 1);
    if ((lane & 1) == 0) {
      Sm.qa[lane >> 1] = make_float4(qx, xo, qy, yo);
      Sm.qb[lane >> 1] = make_float4(qz, zo, qq, qo);
    }
  }
  __syncwarp();
  if (nact <= 16) fwd_sums_x<8>(A.kv, F.iota + k0, wn, nact, o, Sm.qa, Sm.qb, Z, M);
  else fwd_sums_x<16>(A.kv, F.iota + k0, wn, nact, o, Sm.qa, Sm.qb, Z, M);
  zm[(size_t)u * 32 + lane] = make_float2(Z, M);
}

__global__ void k_dense_combine(const FitArgs F, const float2* __restrict__ zm, int S, float4* __restrict__ dq) {
  const FwdArgs& A = F.f;
  const uint32_t item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= *A.n_items) return;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float Z = 0.f, M = 0.f;
  for (int s = 0; s < S; ++s) {  // slice order: the sums do not depend on the schedule
    const float2 v = zm[((size_t)item * S + s) * 32 + lane];
    Z += v.x;
    M += v.y;
  }
  const float4 q = act ? A.qs[js] : make_float4(1e6f, 1e6f, 1e6f, 0.f);
  const bool bad = act && !(Z >= FT_ZMIN && isfinite(Z) && isfinite(M));
  // Z underflow or out-of-domain queries (their item box is not local): the split kernels shift
  // exactly in the direct form
  const bool slow = __any_sync(~0u, bad) || it.z < 0;
  // the item's exponent shift (k_dense_fwd: max_j mh_j), for the backward's weights
  const float mh = act ? A.qmh[js] : -INFINITY;
  float shift = mh;
  for (int s2 = 16; s2 > 0; s2 >>= 1) shift = fmaxf(shift, __shfl_xor_sync(~0u, shift, s2));
  float O = 0.f, rho = 0.f, lossj = 0.f;
  if (act && !slow) {
    const float iz = 1.0f / Z;
    O = M * iz;
    const float diff = O - q.w;
    rho = 2.0f * diff * A.inv_J * iz;
    lossj = diff * diff * A.inv_J;
    if (A.O) A.O[A.perm[js]] = O;
  }
  for (int s = 16; s > 0; s >>= 1) lossj += __shfl_xor_sync(~0u, lossj, s);
  if (lane == 0) {
    if (slow) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    else A.loss_part[item] = lossj;
    if (!slow)  // the split kernels count the slow items' pairs
      atomicAdd(&A.ds->cand_pairs, (unsigned long long)F.iota_n * (unsigned long long)nact);
  }
  // packed query pairs for the backward: {x0,x1,y0,y1}, {z0,z1,rho0,rho1}, {-O0,-O1,s,s}; an idle
  // (or slow-path) slot is far away with rho = 0: it contributes exactly 0
  const float x = (act && !slow) ? q.x : 1e6f, y = (act && !slow) ? q.y : 1e6f, z = (act && !slow) ? q.z : 1e6f;
  const float xo = __shfl_xor_sync(~0u, x, 1), yo = __shfl_xor_sync(~0u, y, 1), zo = __shfl_xor_sync(~0u, z, 1);
  const float ro = __shfl_xor_sync(~0u, rho, 1), Oo = __shfl_xor_sync(~0u, O, 1);
  if ((lane & 1) == 0) {
    float4* d = dq + (size_t)item * 48;
    d[lane >> 1] = make_float4(x, xo, y, yo);
    d[16 + (lane >> 1)] = make_float4(z, zo, rho, ro);
    d[32 + (lane >> 1)] = make_float4(-O, -Oo, shift, shift);
  }
}

// OFF: the block's keys are offset-bank keys (the Delta sums are needed; grid keys are fixed)
template <bool OFF>
__device__ __forceinline__ void dense_bwd_unit(const FitArgs& F, const float4* __restrict__ dq, float4* Q,
                                               uint32_t kb, uint32_t i0, uint32_t i1) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const float4 far_a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t kA = kb * 64u + lane, kB = kA + 32u;
  const uint32_t idA = kA < F.iota_n ? F.iota[kA] : 0u, idB = kB < F.iota_n ? F.iota[kB] : 0u;
  float4 aA = far_a, bA = z4, aB = far_a, bB = z4;
  if (kA < F.iota_n) ld_rec(&kv.grid_raw[2 * idA], aA, bA);
  if (kB < F.iota_n) ld_rec(&kv.grid_raw[2 * idB], aB, bB);
  float2 Sc[2], Sgx[2], Sgy[2], Sgz[2], Ss[2], Sdx[2], Sdy[2], Sdz[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) Sc[k] = Sgx[k] = Sgy[k] = Sgz[k] = Ss[k] = Sdx[k] = Sdy[k] = Sdz[k] = make_float2(0.f, 0.f);
  auto pair = [&](const int k, const float4 a, const float4 b, const float4 QA, const float4 QB, const float4 QC) {
    const float2 dx = __fadd2_rn(make_float2(QA.x, QA.y), make_float2(-a.x, -a.x));
    const float2 dy = __fadd2_rn(make_float2(QA.z, QA.w), make_float2(-a.y, -a.y));
    const float2 dz = __fadd2_rn(make_float2(QB.x, QB.y), make_float2(-a.z, -a.z));
    float2 dd = __fmul2_rn(dz, dz);
    dd = __ffma2_rn(dy, dy, dd);
    dd = __ffma2_rn(dx, dx, dd);
    const float2 e = __ffma2_rn(make_float2(-a.w, -a.w), dd, make_float2(QC.z, QC.w));  // shift - a
    const float2 t = __fmul2_rn(make_float2(QB.z, QB.w), make_float2(ex2f(e.x), ex2f(e.y)));
    float2 f = __ffma2_rn(make_float2(b.y, b.y), dx, make_float2(b.x, b.x));
    f = __ffma2_rn(make_float2(b.z, b.z), dy, f);
    f = __ffma2_rn(make_float2(b.w, b.w), dz, f);
    const float2 uu = __fmul2_rn(t, __fadd2_rn(f, make_float2(QC.x, QC.y)));
    Sc[k] = __fadd2_rn(Sc[k], t);
    Sgx[k] = __ffma2_rn(t, dx, Sgx[k]);
    Sgy[k] = __ffma2_rn(t, dy, Sgy[k]);
    Sgz[k] = __ffma2_rn(t, dz, Sgz[k]);
    Ss[k] = __ffma2_rn(uu, dd, Ss[k]);
    if (OFF) {
      Sdx[k] = __ffma2_rn(uu, dx, Sdx[k]);
      Sdy[k] = __ffma2_rn(uu, dy, Sdy[k]);
      Sdz[k] = __ffma2_rn(uu, dz, Sdz[k]);
    }
  };
  for (uint32_t item = i0; item < i1; ++item) {
    const int npairs = (__ldg(&A.items[item].y) + 1) >> 1;
    __syncwarp();
    const float4* src = dq + (size_t)item * 48;
    Q[lane] = __ldcg(&src[lane]);
    if (lane < 16) Q[32 + lane] = __ldcg(&src[32 + lane]);
    __syncwarp();
    for (int p = 0; p < npairs; ++p) {
      const float4 QA = Q[p], QB = Q[16 + p], QC = Q[32 + p];
      pair(0, aA, bA, QA, QB, QC);
      pair(1, aB, bB, QA, QB, QC);
    }
  }
  auto fin = [&](const int k, MseSums& m) {
    m.sc = Sc[k].x + Sc[k].y;
    m.sgx = Sgx[k].x + Sgx[k].y; m.sgy = Sgy[k].x + Sgy[k].y; m.sgz = Sgz[k].x + Sgz[k].y;
    m.ss = Ss[k].x + Ss[k].y;
    m.sdx = Sdx[k].x + Sdx[k].y; m.sdy = Sdy[k].x + Sdy[k].y; m.sdz = Sdz[k].x + Sdz[k].y;
  };
  MseSums m0, m1;
  fin(0, m0);
  fin(1, m1);
  if (i0 < i1) {
    if (kA < F.iota_n) bwd_mse_red(m0, aA, bA, (int)idA, kv.n_nodes, F.gpad);
    if (kB < F.iota_n) bwd_mse_red(m1, aB, bB, (int)idB, kv.n_nodes, F.gpad);
  }
}

#ifndef DN_BWD_MINB
#define DN_BWD_MINB 1  // resident CTAs per SM the dense backward is compiled for
#endif
__global__ void __launch_bounds__(32 * DN_WARPS, DN_BWD_MINB) k_dense_bwd(const FitArgs F, const float4* __restrict__ dq, int G) {
  __shared__ float4 stage[DN_WARPS][48];
  const uint32_t u = blockIdx.x * DN_WARPS + (threadIdx.x >> 5);
  const uint32_t kb = u / (uint32_t)G, g = u % (uint32_t)G;
  if (kb * 64u >= F.iota_n) return;
  const uint32_t n_items = *F.f.n_items;
  const uint32_t ipg = (n_items + G - 1) / G;
  const uint32_t i0 = g * ipg, i1 = min(n_items, i0 + ipg);
  // a block holds grid keys only or offset keys only unless it straddles the bank boundary
  const uint32_t last = min(kb * 64u + 63u, F.iota_n - 1u);
  if (F.iota[last] < (uint32_t)F.f.kv.n_nodes) dense_bwd_unit<false>(F, dq, stage[threadIdx.x >> 5], kb, i0, i1);
  else dense_bwd_unit<true>(F, dq, stage[threadIdx.x >> 5], kb, i0, i1);
}

// work split of the three dense kernels for n_items items (a launch bound) and iota_n keys
void dense_split_dims(int64_t n_items, uint32_t iota_n, int& S, uint32_t& ks, int& G) {
  const int64_t target = 148 * 16 * 4;  // units: ~4 per warp slot
  S = (int)std::max<int64_t>(1, std::min<int64_t>((target + n_items - 1) / std::max<int64_t>(n_items, 1),
                                                    (iota_n + 255) / 256));
  ks = ((iota_n + S - 1) / S + 31) & ~31u;
  const int64_t kblocks = (iota_n + 63) / 64;
  G = (int)std::max<int64_t>(1, std::min<int64_t>((target + kblocks - 1) / kblocks, n_items));
}

int64_t dense_zm_elems(int64_t n_items, uint32_t iota_n) {
  int S, G;
  uint32_t ks;
  dense_split_dims(n_items, iota_n, S, ks, G);
  return n_items * S * 32;
}

int launch_dense_fit(const FitArgs& a, int64_t n_items, float2* zm, float4* dq, cudaStream_t s, int* fwd_launches) {
  if (n_items <= 0) return 0;
  int S, G;
  uint32_t ks;
  dense_split_dims(n_items, a.iota_n, S, ks, G);
  const int64_t ufwd = n_items * S;
  k_dense_fwd<<<(unsigned)((ufwd + DN_WARPS - 1) / DN_WARPS), 32 * DN_WARPS, 0, s>>>(a, zm, S, ks);
  k_dense_combine<<<(unsigned)((n_items + 3) / 4), 128, 0, s>>>(a, zm, S, dq);
  const int64_t ubwd = ((a.iota_n + 63) / 64) * (int64_t)G;
  k_dense_bwd<<<(unsigned)((ubwd + DN_WARPS - 1) / DN_WARPS), 32 * DN_WARPS, 0, s>>>(a, dq, G);
  if (fwd_launches) *fwd_launches = 2;
  return 3;
}

int launch_fit_lists(const FitArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  k_fit_lists<<<(unsigned)((n_items + FL_WARPS - 1) / FL_WARPS), 32 * FL_WARPS, 0, s>>>(a);
  return 1;
}

// ------------------------------------------------------------------ tensor-core pair loops (k_fit_tc)
// The same work items, lists and outputs as k_fit, with the per-pair contractions on the tensor
// cores (warp-level mma.sync m16n8k8, TF32 inputs, FP32 accumulation):
//   exponent   e_ij = phi_j . E_i,  phi_j = [qq_j, x'_j, y'_j, z'_j, 1],  E_i = [-bl_i, A_i, C_i]
//   polynomial f_ij = phi_j . P_i,  P_i = [0, g_i, c'_i]      (the item-local expansion of k_fit)
//   backward   sum_j t_ij X_j = sum_j p_ij (rho_j X_j),  sum_j u_ij X_j = sum_j (p_ij del_ij)(rho_j X_j)
//              with p_ij = 2^e_ij, del_ij = f_ij - O_j, X_j in {1, q'_j} (t) and {1, q'_j, qq_j} (u)
// (Alg. 1 PAPER.md:L505-518 and Alg. 2 L540-568 as contractions over a 5-term feature axis and the
// item's query axis). Every contraction runs as three TF32 products (3xTF32: hi*hi + hi*lo + lo*hi
// with hi = the top 11 significand bits, lo = x - hi), which keeps ~2^-21 relative accuracy per
// product, so the exponent of a kept pair (|terms| <= ~50 log2 units) carries ~2e-5 log2 units of
// error, well inside the 1e-5 value / 1e-4 gradient tolerances (DESIGN.md R-T, R-TC).
// The CUDA cores keep what is not a contraction: 2^e (MUFU.EX2), the forward's Z and M sums, f - O,
// p del and the hi/lo splits. One warp per item as in k_fit; the forward's M dimension is the
// item's queries (two 16-query tiles), the backward's the round's 32 candidate keys (two tiles).
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t a0, const uint32_t a1, const uint32_t a2,
                                         const uint32_t a3, const uint32_t b0, const uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float tf_hi(const float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ uint32_t fu(const float x) { return __float_as_uint(x); }

// K axis (16) of every exponent / polynomial contraction: positions 0-4 the hi parts of both sides,
// 5-9 query hi x key lo, 10-14 query lo x key hi, 15 zero. A thread (g = lane/4, t = lane%4) of an
// m16n8k8 fragment holds K positions {t, t+4} (k-step 0) and {8+t, 12+t} (k-step 1) of its rows /
// columns, stored as one float4 per (row, t).
__device__ __forceinline__ void tc_query_rec(float4* rec, const float* v) {  // query side (v: 5 features)
  float h[5], l[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    h[i] = tf_hi(v[i]);
    l[i] = v[i] - h[i];
  }
  rec[0] = make_float4(h[0], h[4], h[3], l[2]);
  rec[1] = make_float4(h[1], h[0], h[4], l[3]);
  rec[2] = make_float4(h[2], h[1], l[0], l[4]);
  rec[3] = make_float4(h[3], h[2], l[1], 0.f);
}
__device__ __forceinline__ void tc_key_rec(float4* rec, const float* v) {  // key side
  float h[5], l[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    h[i] = tf_hi(v[i]);
    l[i] = v[i] - h[i];
  }
  rec[0] = make_float4(h[0], h[4], l[3], h[2]);
  rec[1] = make_float4(h[1], l[0], l[4], h[3]);
  rec[2] = make_float4(h[2], l[1], h[0], h[4]);
  rec[3] = make_float4(h[3], l[2], h[1], 0.f);
}

struct TcSmem {
  float4 qrec[QW][4];  // per query and t: phi_j on the query side of the K axis
  union {
    float4 krec[32 * 9];  // per round key and (type, t): E_i (type 0) / P_i (type 1), index 9 key + 4 type + t
    float sx[32][12];     // backward: the round's per-key sums (after the A fragments are loaded)
  };
  float4 yrec[4][2][32];  // backward B fragments per 8-query tile: [tile][t-sums / u-sums][lane]
  float nO[QW];           // -O_j
};

// the round's key lane -> its E / P records (far keys: E = -huge, P = 0: weight exactly 0)
__device__ __forceinline__ void tc_key_prep(TcSmem& S, const KeyX& K, const int lane) {
  const float E[5] = {K.nbl, K.Ax, K.Ay, K.Az, K.C};
  const float P[5] = {0.f, K.gx, K.gy, K.gz, K.c};
  tc_key_rec(&S.krec[9 * lane], E);
  tc_key_rec(&S.krec[9 * lane + 4], P);
}

__device__ __forceinline__ void fit_item_tc(const FitArgs& F, const uint32_t item, TcSmem& S, const uint32_t* L,
                                            const uint32_t wn, const float3 o) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int4 it = A.items[item];
  const int nact = it.y;
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  if (act) q = A.qs[js];
  __syncwarp();  // the previous item's readers of S are done
  const float qx = q.x - o.x, qy = q.y - o.y, qz = q.z - o.z;
  const float qq = act ? fmaf(qx, qx, fmaf(qy, qy, qz * qz)) : 1e30f;  // idle slot: weight exactly 0
  {
    const float phi[5] = {qq, qx, qy, qz, 1.0f};
    tc_query_rec(S.qrec[lane], phi);
  }
  const float4 far_a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  // ---- forward: M = queries (tiles of 16), N = 4 keys x {e, f} per group, 8 groups per round
  __syncwarp();
  const bool two_q = nact > 16;
  const float4 qa0 = S.qrec[g][t], qa1 = S.qrec[g + 8][t], qa2 = S.qrec[16 + g][t], qa3 = S.qrec[24 + g][t];
  float2 Z0 = make_float2(0.f, 0.f), M0 = Z0, Z1 = Z0, M1 = Z0;
  {
    uint32_t id1 = ((uint32_t)lane < wn) ? L[lane] : 0u;
    uint32_t id2 = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
    float4 a1 = far_a, b1 = z4;
    if ((uint32_t)lane < wn) ld_rec(&kv.grid_raw[2 * id1], a1, b1);
    for (uint32_t base = 0; base < wn; base += 32) {
      const uint32_t k = base + lane;
      const float4 ka = a1, kb = b1;
      id1 = id2;
      id2 = (k + 64 < wn) ? L[k + 64] : 0u;
      a1 = far_a;
      b1 = z4;
      if (k + 32 < wn) ld_rec(&kv.grid_raw[2 * id1], a1, b1);
      tc_key_prep(S, key_x(ka, kb, o), lane);
      __syncwarp();
      const uint32_t left = wn - base;
#pragma unroll
      for (int G = 0; G < 8; ++G) {
        if ((uint32_t)(4 * G) < left) {
          const float4 B = S.krec[36 * G + lane + (lane >> 3)];
          float d[4] = {0.f, 0.f, 0.f, 0.f};
          mma_tf32(d, fu(qa0.x), fu(qa1.x), fu(qa0.y), fu(qa1.y), fu(B.x), fu(B.y));
          mma_tf32(d, fu(qa0.z), fu(qa1.z), fu(qa0.w), fu(qa1.w), fu(B.z), fu(B.w));
          const float2 w = make_float2(ex2f(d[0]), ex2f(d[2]));
          Z0 = __fadd2_rn(Z0, w);
          M0 = __ffma2_rn(w, make_float2(d[1], d[3]), M0);
          if (two_q) {
            float d1[4] = {0.f, 0.f, 0.f, 0.f};
            mma_tf32(d1, fu(qa2.x), fu(qa3.x), fu(qa2.y), fu(qa3.y), fu(B.x), fu(B.y));
            mma_tf32(d1, fu(qa2.z), fu(qa3.z), fu(qa2.w), fu(qa3.w), fu(B.z), fu(B.w));
            const float2 w1 = make_float2(ex2f(d1[0]), ex2f(d1[2]));
            Z1 = __fadd2_rn(Z1, w1);
            M1 = __ffma2_rn(w1, make_float2(d1[1], d1[3]), M1);
          }
        }
      }
      __syncwarp();  // krec readers done before the next round's records
    }
  }
  // sum over the quad (t holds keys t mod 4 of every group), then lane j takes query j's totals:
  // query 16 mt + 8 h + g sits in lane 4g, component h of tile mt
#pragma unroll
  for (int o2 = 1; o2 <= 2; o2 <<= 1) {
    Z0.x += __shfl_xor_sync(~0u, Z0.x, o2); Z0.y += __shfl_xor_sync(~0u, Z0.y, o2);
    M0.x += __shfl_xor_sync(~0u, M0.x, o2); M0.y += __shfl_xor_sync(~0u, M0.y, o2);
    Z1.x += __shfl_xor_sync(~0u, Z1.x, o2); Z1.y += __shfl_xor_sync(~0u, Z1.y, o2);
    M1.x += __shfl_xor_sync(~0u, M1.x, o2); M1.y += __shfl_xor_sync(~0u, M1.y, o2);
  }
  float Z, M;
  {
    const int src = 4 * (lane & 7), sel = lane >> 3;
    const float za = __shfl_sync(~0u, Z0.x, src), zb = __shfl_sync(~0u, Z0.y, src);
    const float zc = __shfl_sync(~0u, Z1.x, src), zd = __shfl_sync(~0u, Z1.y, src);
    const float ma = __shfl_sync(~0u, M0.x, src), mb = __shfl_sync(~0u, M0.y, src);
    const float mc = __shfl_sync(~0u, M1.x, src), md = __shfl_sync(~0u, M1.y, src);
    Z = sel == 0 ? za : sel == 1 ? zb : sel == 2 ? zc : zd;
    M = sel == 0 ? ma : sel == 1 ? mb : sel == 2 ? mc : md;
  }
  const bool bad = act && !(Z >= FT_ZMIN && isfinite(Z) && isfinite(M));
  if (__any_sync(~0u, bad)) {  // Z underflow (far queries): the split kernels shift exactly
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  float O = 0.f, rho = 0.f, lossj = 0.f;
  if (act) {
    const float iz = 1.0f / Z;
    O = M * iz;
    const float diff = O - q.w;
    const float r = 2.0f * diff * A.inv_J;
    rho = r * iz;  // t_ij = r_j p_ij = (r_j / Z_j) 2^(-a_ij log2 e)
    lossj = diff * diff * A.inv_J;
    if (A.O) A.O[A.perm[js]] = O;
  }
  for (int s2 = 16; s2 > 0; s2 >>= 1) lossj += __shfl_xor_sync(~0u, lossj, s2);
  if (lane == 0) {
    A.loss_part[item] = lossj;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)wn * (unsigned long long)nact);
  }
  // ---- backward: B fragments of the query side. Tile nt holds queries 8 nt .. 8 nt + 7, its K
  // (query) order pairs query 8 nt + 2t with A column t and 8 nt + 2t + 1 with column t + 4, so the
  // exponent MMA's accumulator is the accumulation MMA's A fragment as it stands.
  {
    S.nO[lane] = -O;
    const int nt = lane >> 3, tt = (lane >> 1) & 3, h = lane & 1;
    const float Y[5] = {rho, rho * qx, rho * qy, rho * qz, rho * (act ? qq : 0.f)};
    float* yt = reinterpret_cast<float*>(&S.yrec[nt][0][0]);
    float* yu = reinterpret_cast<float*>(&S.yrec[nt][1][0]);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float v = c < 5 ? Y[c] : 0.f;
      const float hi = tf_hi(v), lo = v - hi;
      if (c < 4) {
        yt[(4 * c + tt) * 4 + h] = hi;
        yt[(4 * c + tt) * 4 + 2 + h] = lo;
      } else {
        yt[(4 * c + tt) * 4 + h] = 0.f;
        yt[(4 * c + tt) * 4 + 2 + h] = 0.f;
      }
      yu[(4 * c + tt) * 4 + h] = hi;
      yu[(4 * c + tt) * 4 + 2 + h] = lo;
    }
  }
  __syncwarp();
  const int ntiles = (nact + 7) >> 3;
  uint32_t iA = ((uint32_t)lane < wn) ? L[lane] : 0u;
  uint32_t iA2 = ((uint32_t)lane + 32 < wn) ? L[lane + 32] : 0u;
  float4 aA = far_a, bA = z4;
  if ((uint32_t)lane < wn) ld_rec(&kv.grid_raw[2 * iA], aA, bA);
  for (uint32_t base = 0; base < wn; base += 32) {
    const uint32_t k = base + lane;
    const uint32_t id = iA;
    const float4 a0 = aA, b0 = bA;
    iA = iA2;
    iA2 = (k + 64 < wn) ? L[k + 64] : 0u;
    aA = far_a;
    bA = z4;
    if (k + 32 < wn) ld_rec(&kv.grid_raw[2 * iA], aA, bA);
    const KeyX K = key_x(a0, b0, o);
    tc_key_prep(S, K, lane);
    __syncwarp();
    const bool two_k = base + 16 < wn;
    // A fragments of the round's two 16-key tiles (E and P records)
    uint32_t ae[2][8], ap[2][8];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const float4 u = S.krec[9 * (16 * mt + g) + t], v = S.krec[9 * (16 * mt + g + 8) + t];
      const float4 up = S.krec[9 * (16 * mt + g) + 4 + t], vp = S.krec[9 * (16 * mt + g + 8) + 4 + t];
      ae[mt][0] = fu(u.x); ae[mt][1] = fu(v.x); ae[mt][2] = fu(u.y); ae[mt][3] = fu(v.y);
      ae[mt][4] = fu(u.z); ae[mt][5] = fu(v.z); ae[mt][6] = fu(u.w); ae[mt][7] = fu(v.w);
      ap[mt][0] = fu(up.x); ap[mt][1] = fu(vp.x); ap[mt][2] = fu(up.y); ap[mt][3] = fu(vp.y);
      ap[mt][4] = fu(up.z); ap[mt][5] = fu(vp.z); ap[mt][6] = fu(up.w); ap[mt][7] = fu(vp.w);
    }
    float dt[2][4], du[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int c = 0; c < 4; ++c) dt[mt][c] = du[mt][c] = 0.f;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      if (nt < ntiles) {
        const float4 Bq = S.qrec[8 * nt + g][t];
        const float4 Yt = S.yrec[nt][0][lane], Yu = S.yrec[nt][1][lane];
        const float2 nO = *reinterpret_cast<const float2*>(&S.nO[8 * nt + 2 * t]);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (mt == 0 || two_k) {
            float de[4] = {0.f, 0.f, 0.f, 0.f}, df[4] = {0.f, 0.f, 0.f, 0.f};
            mma_tf32(de, ae[mt][0], ae[mt][1], ae[mt][2], ae[mt][3], fu(Bq.x), fu(Bq.y));
            mma_tf32(de, ae[mt][4], ae[mt][5], ae[mt][6], ae[mt][7], fu(Bq.z), fu(Bq.w));
            mma_tf32(df, ap[mt][0], ap[mt][1], ap[mt][2], ap[mt][3], fu(Bq.x), fu(Bq.y));
            mma_tf32(df, ap[mt][4], ap[mt][5], ap[mt][6], ap[mt][7], fu(Bq.z), fu(Bq.w));
            // de/df: (key g, q 2t), (key g, q 2t+1), (key g+8, q 2t), (key g+8, q 2t+1)
            const float2 p01 = make_float2(ex2f(de[0]), ex2f(de[1])), p23 = make_float2(ex2f(de[2]), ex2f(de[3]));
            const float2 u01 = __fmul2_rn(p01, __fadd2_rn(make_float2(df[0], df[1]), nO));
            const float2 u23 = __fmul2_rn(p23, __fadd2_rn(make_float2(df[2], df[3]), nO));
            const float ph0 = tf_hi(p01.x), ph1 = tf_hi(p01.y), ph2 = tf_hi(p23.x), ph3 = tf_hi(p23.y);
            const float2 pl01 = __fadd2_rn(p01, make_float2(-ph0, -ph1)), pl23 = __fadd2_rn(p23, make_float2(-ph2, -ph3));
            const float uh0 = tf_hi(u01.x), uh1 = tf_hi(u01.y), uh2 = tf_hi(u23.x), uh3 = tf_hi(u23.y);
            const float2 ul01 = __fadd2_rn(u01, make_float2(-uh0, -uh1)), ul23 = __fadd2_rn(u23, make_float2(-uh2, -uh3));
            // A fragment: a0 = (key g, col t) = q 2t, a1 = (key g+8, q 2t), a2 = (key g, q 2t+1), a3 = (key g+8, q 2t+1)
            mma_tf32(dt[mt], fu(ph0), fu(ph2), fu(ph1), fu(ph3), fu(Yt.x), fu(Yt.y));
            mma_tf32(dt[mt], fu(pl01.x), fu(pl23.x), fu(pl01.y), fu(pl23.y), fu(Yt.x), fu(Yt.y));
            mma_tf32(dt[mt], fu(ph0), fu(ph2), fu(ph1), fu(ph3), fu(Yt.z), fu(Yt.w));
            mma_tf32(du[mt], fu(uh0), fu(uh2), fu(uh1), fu(uh3), fu(Yu.x), fu(Yu.y));
            mma_tf32(du[mt], fu(ul01.x), fu(ul23.x), fu(ul01.y), fu(ul23.y), fu(Yu.x), fu(Yu.y));
            mma_tf32(du[mt], fu(uh0), fu(uh2), fu(uh1), fu(uh3), fu(Yu.z), fu(Yu.w));
          }
        }
      }
    }
    __syncwarp();  // every lane's krec reads are done: sx aliases krec
    // dt/du: (key 16mt+g, feature 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1); t-sums in features 0-3,
    // u-sums in 0-4
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      if (t < 2) {
        *reinterpret_cast<float2*>(&S.sx[16 * mt + g][2 * t]) = make_float2(dt[mt][0], dt[mt][1]);
        *reinterpret_cast<float2*>(&S.sx[16 * mt + g + 8][2 * t]) = make_float2(dt[mt][2], dt[mt][3]);
      }
      if (t < 3) {
        *reinterpret_cast<float2*>(&S.sx[16 * mt + g][4 + 2 * t]) = make_float2(du[mt][0], du[mt][1]);
        *reinterpret_cast<float2*>(&S.sx[16 * mt + g + 8][4 + 2 * t]) = make_float2(du[mt][2], du[mt][3]);
      }
    }
    __syncwarp();
    if (k < wn) {
      const float4 s0 = *reinterpret_cast<const float4*>(&S.sx[lane][0]);
      const float4 s1 = *reinterpret_cast<const float4*>(&S.sx[lane][4]);
      const float suq = S.sx[lane][8];
      // q' sums -> d = q' - k' sums (as k_fit's bwd_sums_x)
      const float sc = s0.x, su = s1.x;
      MseSums ms;
      ms.sc = sc;
      ms.sgx = fmaf(-K.kx, sc, s0.y);
      ms.sgy = fmaf(-K.ky, sc, s0.z);
      ms.sgz = fmaf(-K.kz, sc, s0.w);
      ms.ss = fmaf(K.kk, su, fmaf(-2.0f * K.kx, s1.y, fmaf(-2.0f * K.ky, s1.z, fmaf(-2.0f * K.kz, s1.w, suq))));
      ms.sdx = fmaf(-K.kx, su, s1.y);
      ms.sdy = fmaf(-K.ky, su, s1.z);
      ms.sdz = fmaf(-K.kz, su, s1.w);
      bwd_mse_out(F, ms, a0, b0, (int)id);
    }
    __syncwarp();  // sx readers done before the next round's krec
  }
}

__device__ __forceinline__ void fit_item_tc_any(const FitArgs& F, const uint32_t item, TcSmem& S, FitSmem& S2,
                                                uint32_t* Lw) {
  const uint32_t* L;
  uint32_t wn;
  float3 o;
  const uint32_t ty = fit_item_build(F, item, F.f.items[item], Lw, L, wn, o);
  if (ty == IT_ENUM) fit_item_enum(F, item, S2, Lw);
  else if (ty == IT_NORMAL) fit_item_tc(F, item, S, L, wn, o);
}

#ifndef TC_MIN_BLOCKS
#define TC_MIN_BLOCKS 4
#endif
static_assert(148 * TC_MIN_BLOCKS * FT_WARPS <= SCRATCH_WARPS, "one scratch slot per warp");
__global__ void __launch_bounds__(32 * FT_WARPS, TC_MIN_BLOCKS) k_fit_tc(const FitArgs F) {
  __shared__ TcSmem smem[FT_WARPS];
  __shared__ FitSmem smem2[FT_WARPS];  // the overflowed-brick path (fit_item_enum)
  const int w = threadIdx.x >> 5;
  uint32_t* L = F.scratch + (size_t)(blockIdx.x * FT_WARPS + w) * SCRATCH_STRIDE;
  for (;;) {
    const int64_t item = fetch_item(&F.f.ds->fit_next, F.f.n_items, nullptr, nullptr);
    if (item < 0) break;
    fit_item_tc_any(F, (uint32_t)item, smem[w], smem2[w], L);
  }
}

int launch_fit_tc(const FitArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)std::min<int64_t>((n_items + FT_WARPS - 1) / FT_WARPS, 148 * TC_MIN_BLOCKS);
  k_fit_tc<<<blocks, 32 * FT_WARPS, 0, s>>>(a);
  return 1;
}

int launch_fit(const FitArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
#ifdef FT_CARVEOUT
  static const bool carve = [] {  // shared-memory carveout (percent of the max) for A/B runs
    return cudaFuncSetAttribute(k_fit, cudaFuncAttributePreferredSharedMemoryCarveout, FT_CARVEOUT) == cudaSuccess;
  }();
  (void)carve;
#endif
  const unsigned blocks = (unsigned)std::min<int64_t>((n_items + FT_WARPS - 1) / FT_WARPS, FT_BLOCKS);
  k_fit<<<blocks, 32 * FT_WARPS, 0, s>>>(a);
  return 1;
}

}  // namespace ef
