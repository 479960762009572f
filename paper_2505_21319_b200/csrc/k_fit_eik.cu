// k_fit_eik.cu — the fused fit-step kernel for the MSE + Eikonal loss (BASELINE config C3;
// SURVEY §8(a) S2+S3+S4 with the analytic spatial gradient).
//
// The Eikonal upstream h_j = 2 lambda_E (|G_j| - 1) G_j / (|G_j| J) (reading R-12) depends on query
// j alone, like the MSE upstream, so a work item's forward (O_j and G_j, Eq. func-normal
// PAPER.md:L425-436), losses and backward (Alg. 2 plus the second-order terms)
// run in one kernel per item:
//   1. shift bound, box, brick-list stream + test -> candidate ids in the warp's scratch;
//   2. forward, lanes = queries (each lane owns one query and its 11 running sums), the round's
//      32 candidate keys staged in shared memory as packed pairs and walked two keys per f32x2
//      instruction;
//   3. O_j, G_j, u_j, losses, r_j, h_j, h.u_j, h.G_j -> the item's query table in shared memory;
//   4. backward, lanes = candidate keys (two per lane), the item's queries broadcast as packed
//      pairs: the grid-bank candidates first (8 accumulators per key, no Delta terms), then the
//      offset-bank ones (14 accumulators); up to three red.global.add.v4 per (key, item).
// Items without a brick list or whose shift bound overflowed go to the split kernels.
#include <algorithm>

#include "k_pair.cuh"

namespace ef {

#ifndef FE_MIN_WARPS
#define FE_MIN_WARPS 16  // warps per SM
#endif
#ifndef FE_FWD_UNROLL
#define FE_FWD_UNROLL 16  // forward key-pair loop (measured 1/2/4/8/16: 16 best, C3 k_fit_eik 5.16 -> 5.06 ms)
#endif
#ifndef FE_BWD1_UNROLL
#define FE_BWD1_UNROLL 2  // one-key backward query-pair loop (the last < 64 keys of a bank; 2/4/8 within noise)
#endif
#ifndef FE_BWD_UNROLL
#define FE_BWD_UNROLL 1  // two-key backward query-pair loop (2 spills: slower)
#endif
#define FE_PRAGMA(x) _Pragma(#x)
#define FE_UNROLL(n) FE_PRAGMA(unroll n)
constexpr int FE_WARPS = 4;
constexpr int FE_BLOCKS = 148 * (FE_MIN_WARPS / FE_WARPS);
static_assert(FE_BLOCKS * FE_WARPS <= SCRATCH_WARPS, "one scratch slot per warp");

struct EikSmem {
  // forward: the round's keys as pairs {x0,x1,y0,y1}, {z0,z1,bl0,bl1}, {c0,c1,gx0,gx1}, {gy0,gy1,gz0,gz1}
  float kA[QW / 2][4], kB[QW / 2][4], kC[QW / 2][4], kD[QW / 2][4];
  // backward: the item's queries as pairs {x,y}, {z,w}, {r+hu, O}, {hx,hy}, {hz, T}
  float4 pA[QW / 2], pB[QW / 2], pC[QW / 2], pD[QW / 2], pE[QW / 2];
};

// forward sums of one query (lane) over the staged keys
struct EikFwd {
  float2 Z, M, sgx, sgy, sgz, sux, suy, suz, sfx, sfy, sfz;
};

__device__ __forceinline__ void eik_fwd_round(const EikSmem& S, const int npk, const float2 qx, const float2 qy,
                                              const float2 qz, const float2 sh, const float2 f0, EikFwd& a) {
  FE_UNROLL(FE_FWD_UNROLL)
  for (int p = 0; p < npk; ++p) {
    const float4 A = *reinterpret_cast<const float4*>(S.kA[p]);
    const float4 B = *reinterpret_cast<const float4*>(S.kB[p]);
    const float4 C = *reinterpret_cast<const float4*>(S.kC[p]);
    const float4 D = *reinterpret_cast<const float4*>(S.kD[p]);
    const float2 dx = __fadd2_rn(qx, make_float2(-A.x, -A.y));
    const float2 dy = __fadd2_rn(qy, make_float2(-A.z, -A.w));
    const float2 dz = __fadd2_rn(qz, make_float2(-B.x, -B.y));
    float2 dd = __fmul2_rn(dz, dz);
    dd = __ffma2_rn(dy, dy, dd);
    dd = __ffma2_rn(dx, dx, dd);
    const float2 bl = make_float2(B.z, B.w);
    const float2 e = __ffma2_rn(make_float2(-B.z, -B.w), dd, sh);
    const float2 w = make_float2(ex2f(e.x), ex2f(e.y));
    // f - f0: the shift key's value (accuracy of O and G); S_g = sum w g needs no
    // shift (a positive-weight mean of the g's)
    float2 f = __ffma2_rn(make_float2(C.z, C.w), dx, __fadd2_rn(make_float2(C.x, C.y), f0));
    f = __ffma2_rn(make_float2(D.x, D.y), dy, f);
    f = __ffma2_rn(make_float2(D.z, D.w), dz, f);
    a.Z = __fadd2_rn(a.Z, w);
    a.M = __ffma2_rn(w, f, a.M);
    a.sgx = __ffma2_rn(w, make_float2(C.z, C.w), a.sgx);
    a.sgy = __ffma2_rn(w, make_float2(D.x, D.y), a.sgy);
    a.sgz = __ffma2_rn(w, make_float2(D.z, D.w), a.sgz);
    const float2 wbl = __fmul2_rn(w, bl);
    a.sux = __ffma2_rn(wbl, dx, a.sux);
    a.suy = __ffma2_rn(wbl, dy, a.suy);
    a.suz = __ffma2_rn(wbl, dz, a.suz);
    const float2 wbf = __fmul2_rn(wbl, f);
    a.sfx = __ffma2_rn(wbf, dx, a.sfx);
    a.sfy = __ffma2_rn(wbf, dy, a.sfy);
    a.sfz = __ffma2_rn(wbf, dz, a.sfz);
  }
}

// backward sums of one key over the item's query pairs (MSE + Eikonal second-order terms)
struct EikBwd {
  float2 sc, sgx, sgy, sgz, phx, phy, phz, ss, sdx, sdy, sdz, pdx, pdy, pdz;
};

// OFF: an offset-bank key (also accumulates the Delta sums sd, pd; grid-bank keys have no Delta)
template <bool OFF>
__device__ __forceinline__ void eik_bwd_pair(const float4 a, const float4 b, const float beta2,
                                             const float4 QA, const float4 QB, const float4 QC,
                                             const float4 QD, const float4 QE, EikBwd& s) {
  const float2 dx = __fadd2_rn(make_float2(QA.x, QA.y), make_float2(-a.x, -a.x));
  const float2 dy = __fadd2_rn(make_float2(QA.z, QA.w), make_float2(-a.y, -a.y));
  const float2 dz = __fadd2_rn(make_float2(QB.x, QB.y), make_float2(-a.z, -a.z));
  float2 dd = __fmul2_rn(dz, dz);
  dd = __ffma2_rn(dy, dy, dd);
  dd = __ffma2_rn(dx, dx, dd);
  const float2 p = [&] {
    const float2 e = __ffma2_rn(make_float2(-a.w, -a.w), dd, make_float2(QB.z, QB.w));
    return make_float2(ex2f(e.x), ex2f(e.y));
  }();
  float2 f = __ffma2_rn(make_float2(b.y, b.y), dx, make_float2(b.x, b.x));
  f = __ffma2_rn(make_float2(b.z, b.z), dy, f);
  f = __ffma2_rn(make_float2(b.w, b.w), dz, f);
  const float2 hx = make_float2(QD.x, QD.y), hy = make_float2(QD.z, QD.w), hz = make_float2(QE.x, QE.y);
  const float2 del = __fadd2_rn(f, make_float2(-QC.z, -QC.w));                       // f - O
  float2 hd = __fmul2_rn(hz, dz);
  hd = __ffma2_rn(hy, dy, hd);
  hd = __ffma2_rn(hx, dx, hd);
  const float2 hu = __fmul2_rn(make_float2(beta2, beta2), hd);                        // 2 beta h.d
  float2 hgT = __ffma2_rn(hz, make_float2(b.w, b.w), make_float2(-QE.z, -QE.w));
  hgT = __ffma2_rn(hy, make_float2(b.z, b.z), hgT);
  hgT = __ffma2_rn(hx, make_float2(b.y, b.y), hgT);                                   // h.g - h.G
  const float2 rh = make_float2(QC.x, QC.y);                                          // r + h.u
  const float2 alpha = __fadd2_rn(rh, make_float2(-hu.x, -hu.y));
  // gam = (r + h.u) del + h.g - h.u del - h.G
  const float2 gam = __ffma2_rn(alpha, del, hgT);
  const float2 pa = __fmul2_rn(p, alpha);
  s.sc = __fadd2_rn(s.sc, pa);
  s.sgx = __ffma2_rn(pa, dx, s.sgx);
  s.sgy = __ffma2_rn(pa, dy, s.sgy);
  s.sgz = __ffma2_rn(pa, dz, s.sgz);
  s.phx = __ffma2_rn(p, hx, s.phx);
  s.phy = __ffma2_rn(p, hy, s.phy);
  s.phz = __ffma2_rn(p, hz, s.phz);
  // ss: p (beta dd gam + hu del), beta = beta2 / 2
  const float2 bdd = __fmul2_rn(make_float2(0.5f * beta2, 0.5f * beta2), dd);
  s.ss = __ffma2_rn(p, __ffma2_rn(bdd, gam, __fmul2_rn(hu, del)), s.ss);
  if (OFF) {
    const float2 pg = __fmul2_rn(p, gam);
    s.sdx = __ffma2_rn(pg, dx, s.sdx);
    s.sdy = __ffma2_rn(pg, dy, s.sdy);
    s.sdz = __ffma2_rn(pg, dz, s.sdz);
    const float2 pdel = __fmul2_rn(p, del);
    s.pdx = __ffma2_rn(pdel, hx, s.pdx);
    s.pdy = __ffma2_rn(pdel, hy, s.pdy);
    s.pdz = __ffma2_rn(pdel, hz, s.pdz);
  }
}

__device__ __forceinline__ float hsum(const float2 v) { return v.x + v.y; }

// one key's gradients into the padded accumulator (k_backward's EIK channel map)
template <bool OFF>
__device__ __forceinline__ void eik_red(const EikBwd& s, const float4 a, const float4 b, const int id,
                                        const int n_nodes, float* gpad) {
  const float beta = a.w * EF_LN2;
  const float sc = hsum(s.sc);
  const float dsv = -hsum(s.ss);
  const float dgx = hsum(s.sgx) + hsum(s.phx), dgy = hsum(s.sgy) + hsum(s.phy), dgz = hsum(s.sgz) + hsum(s.phz);
  if (!OFF) {
    float* gp = gpad + (size_t)id * 16;
    red_v4(gp, dsv, sc, dgx, dgy);
    atomicAdd(gp + 4, dgz);
  } else {
    const float dkx = fmaf(-b.y, sc, 2.0f * beta * (hsum(s.sdx) + hsum(s.pdx)));
    const float dky = fmaf(-b.z, sc, 2.0f * beta * (hsum(s.sdy) + hsum(s.pdy)));
    const float dkz = fmaf(-b.w, sc, 2.0f * beta * (hsum(s.sdz) + hsum(s.pdz)));
    float* gp = gpad + (size_t)(id - n_nodes) * 16 + 8;
    red_v4(gp, dkx, dky, dkz, dsv);
    red_v4(gp + 4, sc, dgx, dgy, dgz);
  }
}

// backward over one bank's candidates Ls[0, n), lanes = keys (two per lane)
template <bool OFF>
__device__ __forceinline__ void eik_bwd_segment(const FitArgs& F, const KeysView& kv, const uint32_t* Ls,
                                                const uint32_t n, const EikSmem& S, const int np2) {
  const int lane = threadIdx.x & 31;
  for (uint32_t base = 0; base < n; base += 64) {
    const uint32_t k0 = base + lane, k1 = base + 32 + lane;
    const bool h0 = k0 < n, h1 = k1 < n;
    uint32_t id0 = 0, id1 = 0;
    float4 a0 = make_float4(1e18f, 1e18f, 1e18f, 1.0f), b0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b1 = b0;
    if (h0) {
      id0 = Ls[k0];
      ld_rec(&kv.grid_raw[2 * id0], a0, b0);
    }
    if (h1) {
      id1 = Ls[k1];
      ld_rec(&kv.grid_raw[2 * id1], a1, b1);
    }
    const float beta20 = 2.0f * a0.w * EF_LN2, beta21 = 2.0f * a1.w * EF_LN2;
    EikBwd s0, s1;
    s0.sc = s0.sgx = s0.sgy = s0.sgz = s0.phx = s0.phy = s0.phz = s0.ss = s0.sdx = s0.sdy = s0.sdz = s0.pdx =
        s0.pdy = s0.pdz = make_float2(0.f, 0.f);
    s1 = s0;
    if (base + 32 < n) {  // warp-uniform: two keys per lane
      FE_UNROLL(FE_BWD_UNROLL)
      for (int jp = 0; jp < np2; ++jp) {
        const float4 QA = S.pA[jp], QB = S.pB[jp], QC = S.pC[jp], QD = S.pD[jp], QE = S.pE[jp];
        eik_bwd_pair<OFF>(a0, b0, beta20, QA, QB, QC, QD, QE, s0);
        eik_bwd_pair<OFF>(a1, b1, beta21, QA, QB, QC, QD, QE, s1);
      }
    } else {
      FE_UNROLL(FE_BWD1_UNROLL)
      for (int jp = 0; jp < np2; ++jp) {
        const float4 QA = S.pA[jp], QB = S.pB[jp], QC = S.pC[jp], QD = S.pD[jp], QE = S.pE[jp];
        eik_bwd_pair<OFF>(a0, b0, beta20, QA, QB, QC, QD, QE, s0);
      }
    }
    if (h0) eik_red<OFF>(s0, a0, b0, (int)id0, kv.n_nodes, F.gpad);
    if (h1) eik_red<OFF>(s1, a1, b1, (int)id1, kv.n_nodes, F.gpad);
  }
}

__device__ __forceinline__ void eik_item(const FitArgs& F, const uint32_t item, EikSmem& S, uint32_t* L) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  uint32_t nb = BL_OVERFLOW;
  if (it.z >= 0) nb = __ldg(&kv.bl_n[it.z]);
  if (nb == BL_OVERFLOW) {
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  // 1. shift bound (and the shift key's f0), box, candidates
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY, f0 = 0.f;
  if (act) {  // the shift bound and its key's f0 from k_gather_queries_mh
    q = A.qs[js];
    mh = A.qmh[js];
    f0 = A.qf0[js];
  }
  Box box = warp_box(act, q.x, q.y, q.z, mh);
  box.thr += A.T_l;
  __syncwarp();  // the previous item's readers of L and S are done
  // candidates split by bank: grid keys at L[0, wg), offset keys at LO[0, wo)
  uint32_t* const LO = L + SCRATCH_HALF;
  uint32_t wg = 0, wo = 0;
  stream_list<4>(kv, kv.bl_pool + __ldg(&kv.bl_off[it.z]), nb, box, [&](bool pass, uint32_t id) {
    const bool grid = id < (uint32_t)kv.n_nodes;
    const uint32_t bg = __ballot_sync(~0u, pass && grid), bo = __ballot_sync(~0u, pass && !grid);
    if (pass) {
      if (grid) L[wg + __popc(bg & lanemask_lt())] = id;
      else LO[wo + __popc(bo & lanemask_lt())] = id;
    }
    wg += __popc(bg);
    wo += __popc(bo);
  });
  const uint32_t wn = wg + wo;
  __syncwarp();
  // 2. forward, lanes = queries
  EikFwd fa;
  fa.Z = fa.M = fa.sgx = fa.sgy = fa.sgz = fa.sux = fa.suy = fa.suz = fa.sfx = fa.sfy = fa.sfz = make_float2(0.f, 0.f);
  {
    const float sh = act ? mh : -INFINITY;
    const float2 qx = make_float2(q.x, q.x), qy = make_float2(q.y, q.y), qz = make_float2(q.z, q.z);
    const float2 sh2 = make_float2(sh, sh), nf0 = make_float2(-f0, -f0);
    const int hi = lane & 1, slot = lane >> 1;
    for (uint32_t base = 0; base < wn; base += 32) {
      const uint32_t k = base + lane;
      float4 a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), b = make_float4(0.f, 0.f, 0.f, 0.f);  // far: weight 0
      if (k < wn) {
        const uint32_t id = k < wg ? L[k] : LO[k - wg];
        ld_rec(&kv.grid_raw[2 * id], a, b);
      }
      __syncwarp();  // the previous round's readers are done
      S.kA[slot][hi] = a.x; S.kA[slot][2 + hi] = a.y;
      S.kB[slot][hi] = a.z; S.kB[slot][2 + hi] = a.w;
      S.kC[slot][hi] = b.x; S.kC[slot][2 + hi] = b.y;
      S.kD[slot][hi] = b.z; S.kD[slot][2 + hi] = b.w;
      __syncwarp();
      const int npk = ((int)min(wn - base, 32u) + 1) >> 1;
      eik_fwd_round(S, npk, qx, qy, qz, sh2, nf0, fa);
    }
  }
  const float Z = hsum(fa.Z), M = hsum(fa.M);
  const bool bad = act && !(isfinite(Z) && isfinite(M) && Z > 0.0f);
  if (__any_sync(~0u, bad)) {
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  // 3. O, G, u, losses and upstreams (Eq. func-normal; Eq. loss; reading R-12)
  float lossj = 0.f;
  float4 PA = make_float4(0.f, 0.f, 0.f, 0.f);
  float rh = 0.f, Oj = 0.f, hx = 0.f, hy = 0.f, hz = 0.f, Tj = 0.f, nlam = -INFINITY;
  if (act) {
    const float iz = 1.0f / Z;
    Oj = f0 + M * iz;
    nlam = mh - log2f(Z);
    const float c2 = 2.0f * EF_LN2 * iz;
    const float Of = M * iz;  // O - f0 before rounding O (PoU: Oj - f0 would round to 0)
    const float Gx = fmaf(hsum(fa.sgx), iz, c2 * fmaf(Of, hsum(fa.sux), -hsum(fa.sfx)));
    const float Gy = fmaf(hsum(fa.sgy), iz, c2 * fmaf(Of, hsum(fa.suy), -hsum(fa.sfy)));
    const float Gz = fmaf(hsum(fa.sgz), iz, c2 * fmaf(Of, hsum(fa.suz), -hsum(fa.sfz)));
    const float ux = c2 * hsum(fa.sux), uy = c2 * hsum(fa.suy), uz = c2 * hsum(fa.suz);
    const float diff = Oj - q.w;
    const float r = 2.0f * diff * A.inv_J;
    lossj = diff * diff * A.inv_J;
    const float nrm = sqrtf(fmaf(Gx, Gx, fmaf(Gy, Gy, Gz * Gz)));
    lossj = fmaf(A.eik_lambda * (nrm - 1.0f) * (nrm - 1.0f), A.inv_J, lossj);
    const float sc = nrm > 0.0f ? 2.0f * A.eik_lambda * (nrm - 1.0f) / nrm * A.inv_J : 0.0f;
    hx = sc * Gx; hy = sc * Gy; hz = sc * Gz;
    rh = r + (hx * ux + hy * uy + hz * uz);
    Tj = hx * Gx + hy * Gy + hz * Gz;
    const int ju = A.perm[js];
    if (A.O) A.O[ju] = Oj;
    if (A.G) {
      A.G[3 * (size_t)ju] = Gx;
      A.G[3 * (size_t)ju + 1] = Gy;
      A.G[3 * (size_t)ju + 2] = Gz;
    }
  }
  for (int o = 16; o > 0; o >>= 1) lossj += __shfl_xor_sync(~0u, lossj, o);
  if (lane == 0) {
    A.loss_part[item] = lossj;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)wn * (unsigned long long)nact);
  }
  // the item's query table as packed pairs (an idle slot: w = -inf, all upstreams 0)
  {
    auto pk = [&](float v, float4& dst, bool second) {
      const float o = __shfl_xor_sync(~0u, v, 1);
      if ((lane & 1) == 0) {
        if (!second) { dst.x = v; dst.y = o; } else { dst.z = v; dst.w = o; }
      }
    };
    const int sl = lane >> 1;
    pk(q.x, S.pA[sl], false); pk(q.y, S.pA[sl], true);
    pk(q.z, S.pB[sl], false); pk(nlam, S.pB[sl], true);
    pk(rh, S.pC[sl], false); pk(Oj, S.pC[sl], true);
    pk(hx, S.pD[sl], false); pk(hy, S.pD[sl], true);
    pk(hz, S.pE[sl], false); pk(Tj, S.pE[sl], true);
  }
  __syncwarp();
  // 4. backward, lanes = keys (two per lane), one bank at a time
  const int np2 = (((nact + 1) >> 1) + 1) & ~1;  // even (padding slots are idle queries)
  eik_bwd_segment<false>(F, kv, L, wg, S, np2);
  eik_bwd_segment<true>(F, kv, LO, wo, S, np2);
}

__global__ void __launch_bounds__(32 * FE_WARPS, FE_MIN_WARPS / FE_WARPS) k_fit_eik(const FitArgs F) {
  __shared__ EikSmem smem[FE_WARPS];
  const int w = threadIdx.x >> 5;
  uint32_t* L = F.scratch + (size_t)(blockIdx.x * FE_WARPS + w) * SCRATCH_STRIDE;
  for (;;) {
    const int64_t item = fetch_item(&F.f.ds->fit_next, F.f.n_items, nullptr, nullptr);
    if (item < 0) break;
    eik_item(F, (uint32_t)item, smem[w], L);
  }
}

// ------------------------------------------------------------------ dense mode (cutoff_T = inf)
// The MSE + Eikonal loss with every (query, key) pair, split like the MSE
// dense path (k_fit.cu) so that small batches fill the GPU:
//   k_dense_eik_fwd      (item, key slice) units, lanes = queries: the slice's 11 partial sums of
//                        eik_fwd_round (Z, M, S_g, S_u, S_uf; each query's own shift mh_j and f0);
//   k_dense_eik_combine  per item: the sums over the slices in slice order, then O, G, u, both
//                        losses and upstreams (the epilogue of eik_item) -> the item's packed table;
//   k_dense_eik_bwd      (64-key block, item group) units, key-stationary: two keys per lane
//                        accumulate the second-order sums over every query of the group.
constexpr int DE_WARPS = 4;
constexpr int DE_NSUM = 11;

__global__ void __launch_bounds__(32 * DE_WARPS) k_dense_eik_fwd(const FitArgs F, float* __restrict__ part, int S,
                                                                uint32_t ks) {
  __shared__ EikSmem smem[DE_WARPS];
  EikSmem& Sm = smem[threadIdx.x >> 5];
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const uint32_t u = blockIdx.x * DE_WARPS + (threadIdx.x >> 5);
  const uint32_t item = u / (uint32_t)S, sl = u % (uint32_t)S;
  if (item >= *A.n_items) return;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const bool act = lane < it.y;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY, f0 = 0.f;
  if (act) {
    q = A.qs[js];
    mh = A.qmh[js];
    f0 = A.qf0[js];
  }
  const uint32_t k0 = sl * ks;
  const uint32_t wn = k0 < F.iota_n ? min(ks, F.iota_n - k0) : 0u;
  EikFwd fa;
  fa.Z = fa.M = fa.sgx = fa.sgy = fa.sgz = fa.sux = fa.suy = fa.suz = fa.sfx = fa.sfy = fa.sfz = make_float2(0.f, 0.f);
  const float sh = act ? mh : -INFINITY;
  const float2 qx = make_float2(q.x, q.x), qy = make_float2(q.y, q.y), qz = make_float2(q.z, q.z);
  const float2 sh2 = make_float2(sh, sh), nf0 = make_float2(-f0, -f0);
  const int hi = lane & 1, slot = lane >> 1;
  for (uint32_t base = 0; base < wn; base += 32) {
    const uint32_t k = base + lane;
    float4 a = make_float4(1e18f, 1e18f, 1e18f, 1.0f), b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < wn) ld_rec(&kv.grid_raw[2 * F.iota[k0 + k]], a, b);
    __syncwarp();
    Sm.kA[slot][hi] = a.x; Sm.kA[slot][2 + hi] = a.y;
    Sm.kB[slot][hi] = a.z; Sm.kB[slot][2 + hi] = a.w;
    Sm.kC[slot][hi] = b.x; Sm.kC[slot][2 + hi] = b.y;
    Sm.kD[slot][hi] = b.z; Sm.kD[slot][2 + hi] = b.w;
    __syncwarp();
    const int npk = ((int)min(wn - base, 32u) + 1) >> 1;
    eik_fwd_round(Sm, npk, qx, qy, qz, sh2, nf0, fa);
  }
  float* d = part + (size_t)u * DE_NSUM * 32 + lane;
  d[0] = hsum(fa.Z); d[32] = hsum(fa.M);
  d[64] = hsum(fa.sgx); d[96] = hsum(fa.sgy); d[128] = hsum(fa.sgz);
  d[160] = hsum(fa.sux); d[192] = hsum(fa.suy); d[224] = hsum(fa.suz);
  d[256] = hsum(fa.sfx); d[288] = hsum(fa.sfy); d[320] = hsum(fa.sfz);
}

__global__ void k_dense_eik_combine(const FitArgs F, const float* __restrict__ part, int S, float4* __restrict__ dq) {
  const FwdArgs& A = F.f;
  const uint32_t item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= *A.n_items) return;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const bool act = lane < it.y;
  const int64_t js = (int64_t)it.x + lane;
  float v[DE_NSUM];
#pragma unroll
  for (int c = 0; c < DE_NSUM; ++c) v[c] = 0.f;
  for (int s = 0; s < S; ++s) {  // slice order: the sums do not depend on the schedule
    const float* p = part + ((size_t)item * S + s) * DE_NSUM * 32 + lane;
#pragma unroll
    for (int c = 0; c < DE_NSUM; ++c) v[c] += p[32 * c];
  }
  const float Z = v[0], M = v[1];
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = 0.f, f0 = 0.f;
  if (act) {
    q = A.qs[js];
    mh = A.qmh[js];
    f0 = A.qf0[js];
  }
  const bool bad = act && !(isfinite(Z) && isfinite(M) && Z > 0.0f);
  const bool slow = __any_sync(~0u, bad) || it.z < 0;  // the split kernels (exact shift, direct form)
  float lossj = 0.f, rh = 0.f, Oj = 0.f, hx = 0.f, hy = 0.f, hz = 0.f, Tj = 0.f, nlam = -INFINITY;
  if (act && !slow) {  // the epilogue of eik_item (Eq. func-normal; Eq. loss; reading R-12)
    const float iz = 1.0f / Z;
    Oj = f0 + M * iz;
    nlam = mh - log2f(Z);
    const float c2 = 2.0f * EF_LN2 * iz;
    const float Of = M * iz;
    const float Gx = fmaf(v[2], iz, c2 * fmaf(Of, v[5], -v[8]));
    const float Gy = fmaf(v[3], iz, c2 * fmaf(Of, v[6], -v[9]));
    const float Gz = fmaf(v[4], iz, c2 * fmaf(Of, v[7], -v[10]));
    const float ux = c2 * v[5], uy = c2 * v[6], uz = c2 * v[7];
    const float diff = Oj - q.w;
    const float r = 2.0f * diff * A.inv_J;
    lossj = diff * diff * A.inv_J;
    const float nrm = sqrtf(fmaf(Gx, Gx, fmaf(Gy, Gy, Gz * Gz)));
    lossj = fmaf(A.eik_lambda * (nrm - 1.0f) * (nrm - 1.0f), A.inv_J, lossj);
    const float sc = nrm > 0.0f ? 2.0f * A.eik_lambda * (nrm - 1.0f) / nrm * A.inv_J : 0.0f;
    hx = sc * Gx; hy = sc * Gy; hz = sc * Gz;
    rh = r + (hx * ux + hy * uy + hz * uz);
    Tj = hx * Gx + hy * Gy + hz * Gz;
    const int ju = A.perm[js];
    if (A.O) A.O[ju] = Oj;
    if (A.G) {
      A.G[3 * (size_t)ju] = Gx;
      A.G[3 * (size_t)ju + 1] = Gy;
      A.G[3 * (size_t)ju + 2] = Gz;
    }
  }
  for (int o = 16; o > 0; o >>= 1) lossj += __shfl_xor_sync(~0u, lossj, o);
  if (lane == 0) {
    if (slow) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    else A.loss_part[item] = lossj;
    if (!slow)  // the split kernels count the slow items' pairs
      atomicAdd(&A.ds->cand_pairs, (unsigned long long)F.iota_n * (unsigned long long)it.y);
  }
  // the item's table as packed pairs {x,y}, {z,w}, {r + h.u, O}, {hx, hy}, {hz, T}; an idle (or
  // slow-path) slot has w = -inf and zero upstreams: it contributes exactly 0
  float4* d = dq + (size_t)item * 80;
  const float vals[10] = {q.x, q.y, q.z, nlam, rh, Oj, hx, hy, hz, Tj};
#pragma unroll
  for (int c = 0; c < 5; ++c) {
    const float a0 = vals[2 * c], a1 = vals[2 * c + 1];
    const float o0 = __shfl_xor_sync(~0u, a0, 1), o1 = __shfl_xor_sync(~0u, a1, 1);
    if ((lane & 1) == 0) d[16 * c + (lane >> 1)] = make_float4(a0, o0, a1, o1);
  }
}

template <bool OFF>
__device__ __forceinline__ void dense_eik_unit(const FitArgs& F, const float4* __restrict__ dq, EikSmem& S,
                                               uint32_t kb, uint32_t i0, uint32_t i1) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const uint32_t kA = kb * 64u + lane, kB = kA + 32u;
  const bool hA = kA < F.iota_n, hB = kB < F.iota_n;
  const uint32_t idA = hA ? F.iota[kA] : 0u, idB = hB ? F.iota[kB] : 0u;
  float4 aA = make_float4(1e18f, 1e18f, 1e18f, 1.0f), bA = make_float4(0.f, 0.f, 0.f, 0.f), aB = aA, bB = bA;
  if (hA) ld_rec(&kv.grid_raw[2 * idA], aA, bA);
  if (hB) ld_rec(&kv.grid_raw[2 * idB], aB, bB);
  const float beta2A = 2.0f * aA.w * EF_LN2, beta2B = 2.0f * aB.w * EF_LN2;
  EikBwd s0, s1;
  s0.sc = s0.sgx = s0.sgy = s0.sgz = s0.phx = s0.phy = s0.phz = s0.ss = s0.sdx = s0.sdy = s0.sdz = s0.pdx =
      s0.pdy = s0.pdz = make_float2(0.f, 0.f);
  s1 = s0;
  float4* const tab = reinterpret_cast<float4*>(S.pA);  // pA..pE are contiguous: 5 x 16 float4
  for (uint32_t item = i0; item < i1; ++item) {
    const int np2 = (((__ldg(&A.items[item].y) + 1) >> 1) + 1) & ~1;
    __syncwarp();
    const float4* src = dq + (size_t)item * 80;
    tab[lane] = __ldcg(&src[lane]);
    tab[32 + lane] = __ldcg(&src[32 + lane]);
    if (lane < 16) tab[64 + lane] = __ldcg(&src[64 + lane]);
    __syncwarp();
    for (int jp = 0; jp < np2; ++jp) {
      const float4 QA = S.pA[jp], QB = S.pB[jp], QC = S.pC[jp], QD = S.pD[jp], QE = S.pE[jp];
      eik_bwd_pair<OFF>(aA, bA, beta2A, QA, QB, QC, QD, QE, s0);
      eik_bwd_pair<OFF>(aB, bB, beta2B, QA, QB, QC, QD, QE, s1);
    }
  }
  if (i0 < i1) {
    if (hA) eik_red<OFF>(s0, aA, bA, (int)idA, kv.n_nodes, F.gpad);
    if (hB) eik_red<OFF>(s1, aB, bB, (int)idB, kv.n_nodes, F.gpad);
  }
}

__global__ void __launch_bounds__(32 * DE_WARPS) k_dense_eik_bwd(const FitArgs F, const float4* __restrict__ dq, int G) {
  __shared__ EikSmem smem[DE_WARPS];
  const uint32_t u = blockIdx.x * DE_WARPS + (threadIdx.x >> 5);
  const uint32_t kb = u / (uint32_t)G, g = u % (uint32_t)G;
  if (kb * 64u >= F.iota_n) return;
  const uint32_t n_items = *F.f.n_items;
  const uint32_t ipg = (n_items + G - 1) / G;
  const uint32_t i0 = g * ipg, i1 = min(n_items, i0 + ipg);
  const uint32_t last = min(kb * 64u + 63u, F.iota_n - 1u);
  if (F.iota[last] < (uint32_t)F.f.kv.n_nodes) dense_eik_unit<false>(F, dq, smem[threadIdx.x >> 5], kb, i0, i1);
  else dense_eik_unit<true>(F, dq, smem[threadIdx.x >> 5], kb, i0, i1);
}

int64_t dense_eik_part_elems(int64_t n_items, uint32_t iota_n) {
  int S, G;
  uint32_t ks;
  dense_split_dims(n_items, iota_n, S, ks, G);
  return n_items * S * DE_NSUM * 32;
}

int launch_dense_fit_eik(const FitArgs& a, int64_t n_items, float* part, float4* dq, cudaStream_t s) {
  if (n_items <= 0) return 0;
  int S, G;
  uint32_t ks;
  dense_split_dims(n_items, a.iota_n, S, ks, G);
  const int64_t ufwd = n_items * S;
  k_dense_eik_fwd<<<(unsigned)((ufwd + DE_WARPS - 1) / DE_WARPS), 32 * DE_WARPS, 0, s>>>(a, part, S, ks);
  k_dense_eik_combine<<<(unsigned)((n_items + 3) / 4), 128, 0, s>>>(a, part, S, dq);
  const int64_t ubwd = ((a.iota_n + 63) / 64) * (int64_t)G;
  k_dense_eik_bwd<<<(unsigned)((ubwd + DE_WARPS - 1) / DE_WARPS), 32 * DE_WARPS, 0, s>>>(a, dq, G);
  return 3;
}

int launch_fit_eik(const FitArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)std::min<int64_t>((n_items + FE_WARPS - 1) / FE_WARPS, FE_BLOCKS);
  k_fit_eik<<<blocks, 32 * FE_WARPS, 0, s>>>(a);
  return 1;
}

}  // namespace ef
