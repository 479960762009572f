// k_pair.cuh — the per-pair inner loops shared by the split kernels (k_forward_keys, k_backward)
// and the fused fit kernel (k_fit): lanes = candidate keys, the item's queries broadcast from
// shared memory as packed pairs (f32x2: two queries per instruction).
#pragma once
#include "k_common.cuh"

namespace ef {

// Reduce-scatter of N per-lane values over the warp: afterwards lane l holds in v[0 .. N/32) the
// warp totals of values [l N/32, (l+1) N/32) (N = 32 or 64). 31 (N=32) / 62 (N=64) shuffles.
template <int N>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[N], const int lane) {
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int o = 16 >> st;
    const int c = N >> (st + 1);  // values kept after this step (compile-time once unrolled)
    if (c >= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < c; ++i) {
        const float send = up ? v[i] : v[i + c];
        const float keep = up ? v[i + c] : v[i];
        v[i] = keep + __shfl_xor_sync(~0u, send, o);
      }
    } else {
      v[0] += __shfl_xor_sync(~0u, v[0], o);
    }
  }
}

// S2b (value-only forward, part 2): lanes = the item's candidate keys (its wl list, ids two
// rounds ahead, records one round ahead), the item's queries broadcast from shared memory as
// packed pairs (f32x2: two queries per instruction), per-query partial sums Z_j, M_j in
// registers, one transpose-reduction per item (Alg. 1).
// NPM = max query pairs (8: <= 16 queries, 16: <= 32). Returns Z_j, M_j to lane j.
#define FK_PAIR(pp) \
  { \
    const float4 QA = sQA[pp], QB = sQB[pp]; /* {x0,x1,y0,y1}, {z0,z1,mh0,mh1} */ \
    const float2 dx = __fadd2_rn(make_float2(QA.x, QA.y), nx); \
    const float2 dy = __fadd2_rn(make_float2(QA.z, QA.w), ny); \
    const float2 dz = __fadd2_rn(make_float2(QB.x, QB.y), nz); \
    float2 dd = __fmul2_rn(dz, dz); \
    dd = __ffma2_rn(dy, dy, dd); \
    dd = __ffma2_rn(dx, dx, dd); \
    const float2 e = __ffma2_rn(nbl, dd, make_float2(QB.z, QB.w)); \
    const float2 wv = make_float2(ex2f(e.x), ex2f(e.y)); \
    float2 f = __ffma2_rn(gx, dx, c); \
    f = __ffma2_rn(gy, dy, f); \
    f = __ffma2_rn(gz, dz, f); \
    Z[pp] = __fadd2_rn(Z[pp], wv); \
    M[pp] = __ffma2_rn(wv, f, M[pp]); \
  }
template <int NPM>
__device__ __forceinline__ void fwd_keys_sums(const KeysView& kv, const uint32_t* L, const uint32_t wn,
                                              const int nact, const float4* sQA, const float4* sQB,
                                              float& Zj, float& Mj) {
  const int lane = threadIdx.x & 31;
  const int npairs = (nact + 1) >> 1;
  float2 Z[NPM], M[NPM];
#pragma unroll
  for (int pp = 0; pp < NPM; ++pp) {
    Z[pp] = make_float2(0.f, 0.f);
    M[pp] = make_float2(0.f, 0.f);
  }
  // one round: lane = one key, loop over the item's query pairs
  auto round = [&](const float4 ka, const float4 kb) {
    const float2 nx = make_float2(-ka.x, -ka.x), ny = make_float2(-ka.y, -ka.y), nz = make_float2(-ka.z, -ka.z);
    const float2 nbl = make_float2(-ka.w, -ka.w);
    const float2 c = make_float2(kb.x, kb.x), gx = make_float2(kb.y, kb.y), gy = make_float2(kb.z, kb.z),
                 gz = make_float2(kb.w, kb.w);
    // groups of 4 pairs without a branch inside, so the scheduler can interleave their chains;
    // a last group of 1-2 pairs runs as 2, of 3 as 4: the padding slots hold idle queries (shift
    // -inf: weight exactly 0), wasted FP32 work instead of a latency-bound serial tail
#pragma unroll
    for (int pg = 0; pg < NPM; pg += 4) {
      const int rem = npairs - pg;
      if (rem >= 3) {
        FK_PAIR(pg) FK_PAIR(pg + 1) FK_PAIR(pg + 2) FK_PAIR(pg + 3)
      } else if (rem > 0) {
        FK_PAIR(pg) FK_PAIR(pg + 1)
      }
    }
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
    round(ka, kb);
  }
  // transpose-reduce {Zx, Zy, Mx, My} of every pair; lane j then fetches its query's totals
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


// S4 (MSE, Alg. 2), one key per lane over the item's query pairs:
// dO/dc = p, dO/dg = p d, dO/ds = -p a (f - O), dO/dk = p(-g + 2 beta d (f - O)), weighted by the
// upstream r_j. Queries as packed pairs {x0,x1,y0,y1}, {z0,z1,w0,w1}, {r0,r1,-O0,-O1} (w = -lambda
// log2e; an idle slot has w = -inf and r = 0: it contributes exactly 0).
#ifndef BWD_UNROLL
#define BWD_UNROLL 2
#endif
constexpr int kBwdUnroll = BWD_UNROLL;

struct MseSums {
  float sc, sgx, sgy, sgz, ss, sdx, sdy, sdz;
};

__device__ __forceinline__ MseSums bwd_mse_sums(const float4 a, const float4 b, const int npairs, const float4* pA,
                                                const float4* pB, const float4* pC) {
  const float2 nx = make_float2(-a.x, -a.x), ny = make_float2(-a.y, -a.y), nz = make_float2(-a.z, -a.z);
  const float2 nbl = make_float2(-a.w, -a.w);
  const float2 c2 = make_float2(b.x, b.x), gx2 = make_float2(b.y, b.y), gy2 = make_float2(b.z, b.z),
               gz2 = make_float2(b.w, b.w);
  float2 Sc = make_float2(0.f, 0.f), Sgx = Sc, Sgy = Sc, Sgz = Sc, Ss = Sc, Sdx = Sc, Sdy = Sc, Sdz = Sc;
  // an even number of pairs (the padding slot is an idle query: w = -inf, r = 0 -> exactly 0), two
  // independent chains per iteration and no serial remainder
  const int np2 = (npairs + 1) & ~1;
  auto pair = [&](const int jp) {
    const float4 QA = pA[jp], QB = pB[jp], QC = pC[jp];
    const float2 dx = __fadd2_rn(make_float2(QA.x, QA.y), nx);
    const float2 dy = __fadd2_rn(make_float2(QA.z, QA.w), ny);
    const float2 dz = __fadd2_rn(make_float2(QB.x, QB.y), nz);
    float2 dd = __fmul2_rn(dz, dz);
    dd = __ffma2_rn(dy, dy, dd);
    dd = __ffma2_rn(dx, dx, dd);
    const float2 e = __ffma2_rn(nbl, dd, make_float2(QB.z, QB.w));
    const float2 p = make_float2(ex2f(e.x), ex2f(e.y));
    float2 f = __ffma2_rn(gx2, dx, c2);
    f = __ffma2_rn(gy2, dy, f);
    f = __ffma2_rn(gz2, dz, f);
    const float2 del = __fadd2_rn(f, make_float2(QC.z, QC.w));
    const float2 t = __fmul2_rn(make_float2(QC.x, QC.y), p);
    const float2 u = __fmul2_rn(t, del);
    Sc = __fadd2_rn(Sc, t);
    Sgx = __ffma2_rn(t, dx, Sgx);
    Sgy = __ffma2_rn(t, dy, Sgy);
    Sgz = __ffma2_rn(t, dz, Sgz);
    Ss = __ffma2_rn(u, dd, Ss);
    Sdx = __ffma2_rn(u, dx, Sdx);
    Sdy = __ffma2_rn(u, dy, Sdy);
    Sdz = __ffma2_rn(u, dz, Sdz);
  };
#pragma unroll(kBwdUnroll)
  for (int jp = 0; jp < np2; jp += 2) {
    pair(jp);
    pair(jp + 1);
  }
  MseSums s;
  s.sc = Sc.x + Sc.y; s.sgx = Sgx.x + Sgx.y; s.sgy = Sgy.x + Sgy.y; s.sgz = Sgz.x + Sgz.y;
  s.ss = Ss.x + Ss.y; s.sdx = Sdx.x + Sdx.y; s.sdy = Sdy.x + Sdy.y; s.sdz = Sdz.x + Sdz.y;
  return s;
}

// The key's 5 (grid bank) or 8 (offset bank) channel gradients into the padded accumulator:
// node n -> 16 floats {s0,c0,g0x,g0y | g0z,-,-,- | dx,dy,dz,s1 | c1,g1x,g1y,g1z}.
__device__ __forceinline__ void bwd_mse_red(const MseSums& s, const float4 a, const float4 b, const int id,
                                            const int n_nodes, float* gpad) {
  const float beta = a.w * EF_LN2;
  const float dsv = -beta * s.ss;
  if (id < n_nodes) {
    float* gp = gpad + (size_t)id * 16;
    red_v4(gp, dsv, s.sc, s.sgx, s.sgy);
    atomicAdd(gp + 4, s.sgz);
  } else {
    const float dkx = fmaf(-b.y, s.sc, 2.0f * beta * s.sdx);
    const float dky = fmaf(-b.z, s.sc, 2.0f * beta * s.sdy);
    const float dkz = fmaf(-b.w, s.sc, 2.0f * beta * s.sdz);
    float* gp = gpad + (size_t)(id - n_nodes) * 16 + 8;
    red_v4(gp, dkx, dky, dkz, dsv);
    red_v4(gp + 4, s.sc, s.sgx, s.sgy, s.sgz);
  }
}

}  // namespace ef
