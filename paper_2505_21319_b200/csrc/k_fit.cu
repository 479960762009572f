// k_fit.cu — the fused fit-step kernel for the MSE loss (SURVEY §8(a) S2+S3+S4 in one pass per
// work item).
//
// Per work item (<= 32 sorted queries of one brick, one warp, persistent warps in Morton order):
//   1. shift bounds mh_j >= m_j (the "maximum-reduce" of PAPER.md:L501) and the warp's box test
//      over the brick's candidate list -> the item's candidate key ids in the warp's scratch;
//   2. forward, lanes = candidate keys, queries broadcast as packed pairs: Z_j, M_j (Alg. 1,
//      PAPER.md:L505-518), O_j = M_j / Z_j, lambda_j, the MSE loss and r_j = 2(O_j - o_j)/J
//      (Eq. loss);
//   3. backward over the same candidate ids, lanes = keys (Alg. 2), two
//      red.global.add.v4 per (key, item) into the padded gradient.
// The MSE upstream of a query depends on that query alone, so nothing crosses items: the split
// path's k_item_lists / k_forward_keys / k_backward launches, their candidate-id hand-off through
// HBM and two of the three passes over the queries collapse into one kernel whose latency-bound
// list phase overlaps other warps' FP32 phases. Items without a brick list, or whose shift bound
// overflowed, are left to the split kernels (ds->slow_items).
#include <algorithm>

#include "k_pair.cuh"

namespace ef {

#ifndef FT_MIN_WARPS
#define FT_MIN_WARPS 16  // warps per SM (measured 16/20/24/28 with FT_NPM 8 and 16: 16 + 16 best)
#endif
#ifndef FT_NPM
#define FT_NPM 16  // forward: query pairs per accumulator set (8: two passes for > 16 queries)
#endif
constexpr int FT_WARPS = 4;
constexpr int FT_BLOCKS = 148 * (FT_MIN_WARPS / FT_WARPS);

struct FitSmem {
  float4 qa[QW / 2], qb[QW / 2];            // forward: {x0,x1,y0,y1}, {z0,z1,mh0,mh1}
  float4 pa[QW / 2], pb[QW / 2], pc[QW / 2];  // backward: {x,y}, {z,w}, {r,-O} pairs
};

__device__ __forceinline__ void fit_item(const FitArgs& F, const uint32_t item, FitSmem& S, uint32_t* L) {
  const FwdArgs& A = F.f;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  uint32_t nb = BL_OVERFLOW;
  if (it.z >= 0) nb = __ldg(&kv.bl_n[it.z]);
  if (nb == BL_OVERFLOW) {  // no brick list (out of domain / overflowed brick): split kernels
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  // 1. shift bounds, box, candidate ids
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY, f0 = 0.f;
  float3 g0 = make_float3(0.f, 0.f, 0.f);
  if (act) {
    q = A.qs[js];
    shift_bound(kv, q, mh, f0, g0);
  }
  Box box = warp_box(act, q.x, q.y, q.z, mh);
  box.thr += A.T_l;
  __syncwarp();  // the previous item's readers of L and S are done
  uint32_t wn = 0;
  stream_list<4>(kv, kv.bl_pool + __ldg(&kv.bl_off[it.z]), nb, box, [&](bool pass, uint32_t id) {
    const uint32_t bal = __ballot_sync(~0u, pass);
    if (pass) L[wn + __popc(bal & lanemask_lt())] = id;
    wn += __popc(bal);
  });
  // 2. forward
  {
    const float mhs = act ? mh : -INFINITY;  // an idle slot has shift -inf (weight 0)
    const float xo = __shfl_xor_sync(~0u, q.x, 1), yo = __shfl_xor_sync(~0u, q.y, 1);
    const float zo = __shfl_xor_sync(~0u, q.z, 1), mo = __shfl_xor_sync(~0u, mhs, 1);
    if ((lane & 1) == 0) {
      S.qa[lane >> 1] = make_float4(q.x, xo, q.y, yo);
      S.qb[lane >> 1] = make_float4(q.z, zo, mhs, mo);
    }
  }
  __syncwarp();
  float Z, M;
  if (FT_NPM == 16) {
    if (nact <= 16) fwd_keys_sums<8>(kv, L, wn, nact, S.qa, S.qb, Z, M);
    else fwd_keys_sums<16>(kv, L, wn, nact, S.qa, S.qb, Z, M);
  } else {
    float Z0, M0, Z1 = 0.f, M1 = 0.f;
    fwd_keys_sums<8>(kv, L, wn, min(nact, 16), S.qa, S.qb, Z0, M0);
    if (nact > 16) fwd_keys_sums<8>(kv, L, wn, nact - 16, S.qa + 8, S.qb + 8, Z1, M1);
    Z = lane < 16 ? Z0 : Z1;
    M = lane < 16 ? M0 : M1;
  }
  const bool bad = act && !(isfinite(Z) && isfinite(M) && Z > 0.0f);
  if (__any_sync(~0u, bad)) {  // shift bound overflowed: the split kernels redo it exactly
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  float O = 0.f, nlam = -INFINITY, r = 0.f, lossj = 0.f;
  if (act) {
    O = M * (1.0f / Z);
    nlam = mh - log2f(Z);  // -lambda_j * log2(e):  p_ij = 2^(nlam - bl_i dd_ij)
    const float diff = O - q.w;
    r = 2.0f * diff * A.inv_J;
    lossj = diff * diff * A.inv_J;
    if (A.O) A.O[A.perm[js]] = O;
  }
  for (int o = 16; o > 0; o >>= 1) lossj += __shfl_xor_sync(~0u, lossj, o);
  if (lane == 0) {
    A.loss_part[item] = lossj;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)wn * (unsigned long long)nact);
  }
  // 3. backward over the same candidates
  {
    const float nO = -O;
    const float xo = __shfl_xor_sync(~0u, q.x, 1), yo = __shfl_xor_sync(~0u, q.y, 1);
    const float zo = __shfl_xor_sync(~0u, q.z, 1), wo = __shfl_xor_sync(~0u, nlam, 1);
    const float ro = __shfl_xor_sync(~0u, r, 1), nOo = __shfl_xor_sync(~0u, nO, 1);
    if ((lane & 1) == 0) {
      S.pa[lane >> 1] = make_float4(q.x, xo, q.y, yo);
      S.pb[lane >> 1] = make_float4(q.z, zo, nlam, wo);
      S.pc[lane >> 1] = make_float4(r, ro, nO, nOo);
    }
  }
  __syncwarp();
  const int npairs = (nact + 1) >> 1;
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
      a1 = __ldg(&kv.grid_raw[2 * id1]);
      b1 = __ldg(&kv.grid_raw[2 * id1 + 1]);
    }
    if (k < wn) {
      const MseSums ms = bwd_mse_sums(a, b, npairs, S.pa, S.pb, S.pc);
      bwd_mse_red(ms, a, b, (int)id, kv.n_nodes, F.gpad);
    }
  }
}

__global__ void __launch_bounds__(32 * FT_WARPS, FT_MIN_WARPS / FT_WARPS) k_fit(const FitArgs F) {
  __shared__ FitSmem smem[FT_WARPS];
  const int w = threadIdx.x >> 5;
  uint32_t* L = F.scratch + (size_t)(blockIdx.x * FT_WARPS + w) * BL_CAP;
  for (;;) {
    const int64_t item = fetch_item(&F.f.ds->fit_next, F.f.n_items, nullptr, nullptr);
    if (item < 0) break;
    fit_item(F, (uint32_t)item, smem[w], L);
  }
}

size_t fit_scratch_entries() { return (size_t)FT_BLOCKS * FT_WARPS * BL_CAP; }

int launch_fit(const FitArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)std::min<int64_t>((n_items + FT_WARPS - 1) / FT_WARPS, FT_BLOCKS);
  k_fit<<<blocks, 32 * FT_WARPS, 0, s>>>(a);
  return 1;
}

}  // namespace ef
