// k_forward.cu — S2/S3 forward (+ loss epilogue).
//
// A work item is up to QW queries of one brick (sorted by brick and octant). A warp streams the
// brick's candidate list (k_lists.cu), keeps key k iff bl_k * dist^2(k, item AABB) <= thr with
// thr = max_j mh_j + T_l, where mh_j >= m_j is the exponent of the best key among the query's 8
// lattice corners and its own cell (the shift of the paper's "maximum-reduce").
// Every skipped pair has a - m_j > cutoff_T (reading R-1). The kept ids are handed to
// the backward (wl lists).
//   k_forward_keys (value-only forward, the fit step's): lanes = compacted candidate keys, the
//     item's queries broadcast from shared memory two per packed f32x2 instruction, per-query
//     partial sums in registers, one transpose-reduction per item (Alg. 1).
//   k_forward (G forward, exact-min slow path, kept-pair census): lanes = queries, staged keys
//     broadcast (Alg. 1 and the G sums of Eq. func-normal).
#include <algorithm>

#include "k_pair.cuh"

namespace ef {

// ------------------------------------------------------------------------------ forward
struct FwdAcc {
  float Z, M, sgx, sgy, sgz, sux, suy, suz, sfx, sfy, sfz;
};

template <bool WANT_G>
__device__ __forceinline__ void fwd_pair(const float4 q, const float4 a, const float4 b, float shift, float f0,
                                         const float3 g0, FwdAcc& s) {
  const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
  const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float wgt = ex2f(fmaf(-a.w, dd, shift));
  s.Z += wgt;
  if (WANT_G) {
    const float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x - f0)));
    s.sgx = fmaf(wgt, b.y - g0.x, s.sgx);  // relative to the shift key's g (accuracy)
    s.sgy = fmaf(wgt, b.z - g0.y, s.sgy);
    s.sgz = fmaf(wgt, b.w - g0.z, s.sgz);
    const float wbl = wgt * a.w;
    s.sux = fmaf(wbl, dx, s.sux);
    s.suy = fmaf(wbl, dy, s.suy);
    s.suz = fmaf(wbl, dz, s.suz);
    const float wbf = wbl * f;
    s.sfx = fmaf(wbf, dx, s.sfx);
    s.sfy = fmaf(wbf, dy, s.sfy);
    s.sfz = fmaf(wbf, dz, s.sfz);
    s.M = fmaf(wgt, f, s.M);
  } else {
    const float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x)));
    s.M = fmaf(wgt, f, s.M);
  }
}

// Each lane owns up to two queries of the warp item (j = lane and lane + 32): every broadcast
// key serves both, halving the shared-memory loads and the list stream per pair.
template <bool WANT_G>
__device__ __forceinline__ void forward_item(const FwdArgs& A, const uint32_t item) {
  __shared__ float4 ws_a[NWARP][WSLICE];
  __shared__ float4 ws_b[NWARP][WSLICE];
  __shared__ int ws_id[NWARP][WSLICE];
  const KeysView& kv = A.kv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int4 it = A.items[item];
  const int nact = it.y;       // queries of this warp's item, <= QW (warps are independent)
  const bool two = nact > 32;  // warp-uniform: the second query slot is in use
  bool act[2];
  int64_t js[2];
  float4 q[2];
  float mh[2], f0[2];
  float3 g0[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    act[u] = lane + 32 * u < nact;
    js[u] = (int64_t)it.x + lane + 32 * u;
    q[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    mh[u] = INFINITY;
    f0[u] = 0.f;
    g0[u] = make_float3(0.f, 0.f, 0.f);
    if (act[u]) {
      q[u] = A.qs[js[u]];
      shift_bound(kv, q[u], mh[u], f0[u], g0[u]);
    }
  }
  Box box = warp_box(act[0], q[0].x, q[0].y, q[0].z, mh[0]);
  if (two) {
    const Box b1 = warp_box(act[1], q[1].x, q[1].y, q[1].z, mh[1]);
    box.lx = fminf(box.lx, b1.lx); box.ly = fminf(box.ly, b1.ly); box.lz = fminf(box.lz, b1.lz);
    box.hx = fmaxf(box.hx, b1.hx); box.hy = fmaxf(box.hy, b1.hy); box.hz = fmaxf(box.hz, b1.hz);
    box.thr = fmaxf(box.thr, b1.thr);
  }
  box.thr += A.T_l;

  // mode 0: accumulate with `shift`; 1: exact min of the exponent; 2: count kept pairs
  const FwdAcc zero = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  FwdAcc s[2] = {zero, zero};
  float shift[2] = {mh[0], mh[1]};
  float mexact[2] = {INFINITY, INFINITY};
  unsigned long long cand = 0, kept = 0, kept_off = 0;
  bool emit = false;
  uint32_t wl_cnt = 0, wl_base = 0;
  float4* sa = ws_a[w];
  float4* sb = ws_b[w];
  int* sid = ws_id[w];
  auto run = [&](const int mode) {
    uint32_t cnt = 0;
    auto consume = [&]() {
      __syncwarp();
      if (mode == 0) cand += cnt;
      if (mode == 0) {
        // register double-buffering of the broadcast key loads hides the LDS latency
        float4 a0 = sa[0], b0 = sb[0];
        if (two) {
#pragma unroll 2
          for (uint32_t i = 1; i < cnt; ++i) {
            const float4 a1 = sa[i], b1 = sb[i];
            fwd_pair<WANT_G>(q[0], a0, b0, shift[0], f0[0], g0[0], s[0]);
            fwd_pair<WANT_G>(q[1], a0, b0, shift[1], f0[1], g0[1], s[1]);
            a0 = a1;
            b0 = b1;
          }
          fwd_pair<WANT_G>(q[0], a0, b0, shift[0], f0[0], g0[0], s[0]);
          fwd_pair<WANT_G>(q[1], a0, b0, shift[1], f0[1], g0[1], s[1]);
        } else {
#pragma unroll 4
          for (uint32_t i = 1; i < cnt; ++i) {
            const float4 a1 = sa[i], b1 = sb[i];
            fwd_pair<WANT_G>(q[0], a0, b0, shift[0], f0[0], g0[0], s[0]);
            a0 = a1;
            b0 = b1;
          }
          fwd_pair<WANT_G>(q[0], a0, b0, shift[0], f0[0], g0[0], s[0]);
        }
      } else {
        for (uint32_t i = 0; i < cnt; ++i) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float e = exponent(q[u], sa[i]);
            if (mode == 1) {
              mexact[u] = fminf(mexact[u], e);
            } else if (act[u]) {
              const bool kp = e - mexact[u] <= A.T_l;
              kept += kp ? 1ull : 0ull;
              kept_off += (kp && sid[i] >= kv.n_nodes) ? 1ull : 0ull;
            }
          }
        }
      }
      __syncwarp();
      cnt = 0;
    };
    candidates(kv, it.z, box, [&](bool pass, uint32_t kp, float4 a, float4 b) {
      const uint32_t bal = __ballot_sync(~0u, pass);
      if (pass) {
        const uint32_t rank = __popc(bal & lanemask_lt());
        const uint32_t slot = cnt + rank;
        sa[slot] = a;
        if (mode == 0) sb[slot] = b;
        if (mode == 2) sid[slot] = (int)kp;
        if (emit) A.wl_pool[wl_base + wl_cnt + rank] = kp;  // hand the candidate set to the backward
      }
      cnt += __popc(bal);
      wl_cnt += __popc(bal);
      if (cnt >= WSLICE - 32) consume();
    });
    if (cnt) consume();
  };

  // reserve room for this item's candidate ids (at most its brick list) in the hand-off pool
  uint32_t nb = BL_OVERFLOW;
  if (it.z >= 0) nb = __ldg(&kv.bl_n[it.z]);
  if (lane == 0 && nb != BL_OVERFLOW) wl_base = atomicAdd(&A.ds->wl_top, nb);
  wl_base = __shfl_sync(~0u, wl_base, 0);
  emit = (nb != BL_OVERFLOW) && (wl_base + nb <= A.wl_cap);
  run(0);
  if (lane == 0) {
    A.wl_off[item] = wl_base;
    A.wl_n[item] = emit ? wl_cnt : BL_OVERFLOW;
  }
  emit = false;
  bool bad = false;
#pragma unroll
  for (int u = 0; u < 2; ++u) bad |= act[u] && !(isfinite(s[u].Z) && isfinite(s[u].M) && s[u].Z > 0.0f);
  if (__any_sync(~0u, bad)) {
    // exact-shift slow path: the warp's candidate set contains every argmin key
    run(1);
    shift[0] = mexact[0];
    shift[1] = mexact[1];
    s[0] = zero;
    s[1] = zero;
    cand = 0;
    run(0);
    if (lane == 0) atomicAdd(&A.ds->overflow_items, 1u);
  }
  if (A.count_kept) {
    mexact[0] = mexact[1] = INFINITY;
    run(1);
    run(2);
    for (int o = 16; o > 0; o >>= 1) {
      kept += __shfl_xor_sync(~0u, kept, o);
      kept_off += __shfl_xor_sync(~0u, kept_off, o);
    }
    if (lane == 0) {
      atomicAdd(&A.ds->kept_pairs, kept);
      atomicAdd(&A.ds->kept_pairs_offset, kept_off);
    }
  }
  if (lane == 0) atomicAdd(&A.ds->cand_pairs, cand * (unsigned long long)nact);

  // epilogue: O, lambda, G, loss and its upstream
  float lossj = 0.0f;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!act[u]) continue;
    const FwdAcc& t = s[u];
    const float iz = 1.0f / t.Z;
    const float O = (WANT_G ? f0[u] : 0.0f) + t.M * iz;
    const float nlam = shift[u] - log2f(t.Z);  // -lambda_j * log2(e):  p_ij = 2^(nlam - bl_i dd_ij)
    const int ju = A.perm[js[u]];
    float r = 0.0f;
    float Gx = 0.f, Gy = 0.f, Gz = 0.f;
    if (WANT_G) {
      const float c2 = 2.0f * EF_LN2 * iz;
      const float Of = t.M * iz;  // O - f0 before rounding O: (O - f0) loses M/Z below ulp(O)
      Gx = g0[u].x + (t.sgx * iz + c2 * fmaf(Of, t.sux, -t.sfx));
      Gy = g0[u].y + (t.sgy * iz + c2 * fmaf(Of, t.suy, -t.sfy));
      Gz = g0[u].z + (t.sgz * iz + c2 * fmaf(Of, t.suz, -t.sfz));
      A.gs[js[u]] = make_float4(Gx, Gy, Gz, 0.f);
      A.us[js[u]] = make_float4(c2 * t.sux, c2 * t.suy, c2 * t.suz, 0.f);
      if (A.G) {
        A.G[3 * (size_t)ju] = Gx;
        A.G[3 * (size_t)ju + 1] = Gy;
        A.G[3 * (size_t)ju + 2] = Gz;
      }
    }
    if (A.loss_kind >= EFUNC_LOSS_MSE) {
      const float diff = O - q[u].w;
      r = 2.0f * diff * A.inv_J;
      lossj = fmaf(diff * diff, A.inv_J, lossj);
    }
    if (WANT_G && A.loss_kind == EFUNC_LOSS_MSE_EIKONAL) {
      const float nrm = sqrtf(fmaf(Gx, Gx, fmaf(Gy, Gy, Gz * Gz)));
      lossj = fmaf(A.eik_lambda * (nrm - 1.0f) * (nrm - 1.0f), A.inv_J, lossj);
      const float sc = nrm > 0.0f ? 2.0f * A.eik_lambda * (nrm - 1.0f) / nrm * A.inv_J : 0.0f;
      A.hs[js[u]] = make_float4(sc * Gx, sc * Gy, sc * Gz, 0.f);
    }
    A.rec[js[u]] = make_float4(nlam, r, O, 0.f);
    if (A.O) A.O[ju] = O;
  }
  if (A.loss_kind >= EFUNC_LOSS_MSE) {
    for (int o = 16; o > 0; o >>= 1) lossj += __shfl_xor_sync(~0u, lossj, o);
    if (lane == 0) A.loss_part[item] = lossj;
  }
}

// from_list: the items flagged by k_forward_keys (ds->slow_n of them in A.slow_items), grid-strided
template <bool WANT_G>
__global__ void __launch_bounds__(NTHREADS) k_forward(const FwdArgs A, const int from_list) {
  if (!from_list) {
    const uint32_t item = blockIdx.x * NWARP + (threadIdx.x >> 5);
    if (item < *A.n_items) forward_item<WANT_G>(A, item);
    return;
  }
  const uint32_t n = *(volatile uint32_t*)&A.ds->slow_n;
  for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) forward_item<WANT_G>(A, A.slow_items[i]);
}

// ------------------------------------------------------------------ forward, lanes = keys
// S2a (value-only forward, part 1): per item, the shift bounds mh_j and the compacted candidate
// ids (the item's warp-box test over its brick list) written to the item's slice of wl_pool.
// Latency-bound gathers: few registers and 4 independent warps per CTA for occupancy.
constexpr int IL_WARPS = 4;
__global__ void __launch_bounds__(32 * IL_WARPS) k_item_lists(const FwdArgs A) {
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const uint32_t item = blockIdx.x * IL_WARPS + (threadIdx.x >> 5);
  if (item >= *A.n_items) return;
  const int4 it = A.items[item];
  const int nact = it.y;
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = INFINITY, f0 = 0.f;
  float3 g0 = make_float3(0.f, 0.f, 0.f);
  if (act) {
    q = A.qs[js];
    shift_bound(kv, q, mh, f0, g0);
    A.qmh[js] = mh;
  }
  Box box = warp_box(act, q.x, q.y, q.z, mh);
  box.thr += A.T_l;
  // reserve room for this item's candidate ids (at most its brick list)
  uint32_t nb = BL_OVERFLOW, wl_base = 0;
  if (it.z >= 0) nb = __ldg(&kv.bl_n[it.z]);
  if (lane == 0 && nb != BL_OVERFLOW) wl_base = atomicAdd(&A.ds->wl_top, nb);
  wl_base = __shfl_sync(~0u, wl_base, 0);
  if (nb == BL_OVERFLOW || wl_base + nb > A.wl_cap) {
    if (lane == 0) {  // no list: k_forward (slow list) and the backward's fallback stream handle it
      A.wl_off[item] = 0;
      A.wl_n[item] = BL_OVERFLOW;
    }
    return;
  }
  uint32_t cnt = 0;
  uint32_t* out = A.wl_pool + wl_base;
  stream_list<4>(kv, kv.bl_pool + __ldg(&kv.bl_off[it.z]), nb, box, [&](bool pass, uint32_t kp) {
    const uint32_t bal = __ballot_sync(~0u, pass);
    if (pass) out[cnt + __popc(bal & lanemask_lt())] = kp;
    cnt += __popc(bal);
  });
  if (lane == 0) {
    A.wl_off[item] = wl_base;
    A.wl_n[item] = cnt;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)cnt * (unsigned long long)nact);
  }
}

#ifndef FK_MIN_BLOCKS
#define FK_MIN_BLOCKS 16  // warps per SM: <= 128 registers (measured: 1/16/20/24; half-item warps were slower)
#endif
constexpr int FK_WARPS = 4;  // persistent: warps per CTA, each fetching items heaviest-first
__device__ __forceinline__ void forward_keys_item(const FwdArgs& A, const uint32_t item, float4* sQA, float4* sQB) {
  static_assert(QW == 32, "k_forward_keys: <= 32 queries per item");
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  const uint32_t wn = A.wl_n[item];
  if (wn == BL_OVERFLOW) {  // no candidate list: the lanes = queries kernel streams this item
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  const bool act = lane < nact;
  const int64_t js = (int64_t)it.x + lane;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  float mh = -INFINITY;  // an idle slot has shift -inf (weight 0)
  if (act) {
    q = A.qs[js];
    mh = A.qmh[js];
  }
  __syncwarp();  // the previous item's readers of sQA/sQB are done
  {
    const float xo = __shfl_xor_sync(~0u, q.x, 1), yo = __shfl_xor_sync(~0u, q.y, 1);
    const float zo = __shfl_xor_sync(~0u, q.z, 1), mo = __shfl_xor_sync(~0u, mh, 1);
    if ((lane & 1) == 0) {
      sQA[lane >> 1] = make_float4(q.x, xo, q.y, yo);
      sQB[lane >> 1] = make_float4(q.z, zo, mh, mo);
    }
  }
  __syncwarp();
  const uint32_t* L = A.wl_pool + A.wl_off[item];
  float Z, M;
  if (nact <= 16) fwd_keys_sums<8>(A.kv, L, wn, nact, sQA, sQB, Z, M);
  else fwd_keys_sums<16>(A.kv, L, wn, nact, sQA, sQB, Z, M);
  const bool bad = act && !(isfinite(Z) && isfinite(M) && Z > 0.0f);
  if (__any_sync(~0u, bad)) {
    // the shift bound overflowed: k_forward redoes the item with the exact-min shift
    if (lane == 0) A.slow_items[atomicAdd(&A.ds->slow_n, 1u)] = item;
    return;
  }
  // epilogue: O, lambda, loss and its upstream (value-only forward)
  float lossj = 0.0f;
  if (act) {
    const float O = M * (1.0f / Z);
    const float nlam = mh - log2f(Z);  // -lambda_j * log2(e):  p_ij = 2^(nlam - bl_i dd_ij)
    const int ju = A.perm[js];
    float r = 0.0f;
    if (A.loss_kind >= EFUNC_LOSS_MSE) {
      const float diff = O - q.w;
      r = 2.0f * diff * A.inv_J;
      lossj = diff * diff * A.inv_J;
    }
    A.rec[js] = make_float4(nlam, r, O, 0.f);
    if (A.O) A.O[ju] = O;
  }
  if (A.loss_kind >= EFUNC_LOSS_MSE) {
    for (int o = 16; o > 0; o >>= 1) lossj += __shfl_xor_sync(~0u, lossj, o);
    if (lane == 0) A.loss_part[item] = lossj;
  }
}

__global__ void __launch_bounds__(32 * FK_WARPS, FK_MIN_BLOCKS / FK_WARPS) k_forward_keys(const FwdArgs A) {
  __shared__ float4 sQA[FK_WARPS][QW / 2], sQB[FK_WARPS][QW / 2];
  const int w = threadIdx.x >> 5;
  for (;;) {
    const int64_t item = fetch_item(&A.ds->fwd_next, A.n_items, nullptr, nullptr);
    if (item < 0) break;
    forward_keys_item(A, (uint32_t)item, sQA[w], sQB[w]);
  }
}

// S1 gather for the fused path: sorted {x,y,z,o}, the permutation, and each query's shift bound
// mh_j >= m_j, one query per thread at full occupancy instead of inside the FP32-bound k_fit. The
// bound is shift_bound's (same keys, same visit order, same strict minimum), with the candidates'
// records loaded together (8 corners, then the own cell's keys 4 at a time) and the argmin key's
// polynomial record read once at the end.
__global__ void k_gather_queries_mh(const KeysView kv, const uint32_t* __restrict__ order, const float* __restrict__ q,
                                    const float* __restrict__ o, int64_t J, float4* __restrict__ qs,
                                    int* __restrict__ perm, float* __restrict__ qmh, float* __restrict__ qf0) {
  const int R = kv.R, NC = kv.NC;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < J; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = order[p];
    const float4 v = make_float4(q[3 * (size_t)j], q[3 * (size_t)j + 1], q[3 * (size_t)j + 2], o ? o[j] : 0.0f);
    qs[p] = v;
    perm[p] = (int)j;
    const int cx = cellc(v.x, kv.inv_h, NC), cy = cellc(v.y, kv.inv_h, NC), cz = cellc(v.z, kv.inv_h, NC);
    const int cid = (cz * NC + cy) * NC + cx;
    const uint32_t s0 = __ldg(&kv.cell_start[cid]);
    const uint32_t s1 = min(__ldg(&kv.cell_start[cid + 1]), s0 + 32u);
    float4 ka[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      ka[c] = __ldg(&kv.grid_raw[2 * ((cx + (c & 1)) + R * ((cy + ((c >> 1) & 1)) + R * (cz + (c >> 2))))]);
    float mh = INFINITY;
    const float4* best = kv.grid_raw;
    float4 bk = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float e = exponent(v, ka[c]);
      if (e < mh) {
        mh = e;
        best = &kv.grid_raw[2 * ((cx + (c & 1)) + R * ((cy + ((c >> 1) & 1)) + R * (cz + (c >> 2))))];
        bk = ka[c];
      }
    }
    for (uint32_t k0 = s0; k0 < s1; k0 += 4) {
      float4 kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) kk[u] = (k0 + u < s1) ? __ldg(&kv.ks[2 * (k0 + u)]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < s1) {
          const float e = exponent(v, kk[u]);
          if (e < mh) {
            mh = e;
            best = &kv.ks[2 * (k0 + u)];
            bk = kk[u];
          }
        }
      }
    }
    qmh[p] = mh;
    if (qf0) {
      const float4 b = __ldg(best + 1);
      const float dx = v.x - bk.x, dy = v.y - bk.y, dz = v.z - bk.z;
      qf0[p] = (mh < INFINITY) ? fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x))) : 0.0f;
    }
  }
}

int launch_gather_queries_mh(const KeysView& kv, const uint32_t* order, const float* q, const float* o, int64_t J,
                             float4* qs, int* perm, float* qmh, float* qf0, cudaStream_t s) {
  if (J == 0) return 0;
  const int64_t blocks = std::min<int64_t>((J + 255) / 256, 148 * 16);
  k_gather_queries_mh<<<(unsigned)blocks, 256, 0, s>>>(kv, order, q, o, J, qs, perm, qmh, qf0);
  return 1;
}

int launch_forward_slow(const FwdArgs& a, int want_g, cudaStream_t s) {
  // the items in a.slow_items (usually none)
  if (want_g) k_forward<true><<<148 * 4, NTHREADS, 0, s>>>(a, 1);
  else k_forward<false><<<148 * 4, NTHREADS, 0, s>>>(a, 1);
  return 1;
}

int launch_item_lists(const FwdArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  k_item_lists<<<(unsigned)((n_items + IL_WARPS - 1) / IL_WARPS), 32 * IL_WARPS, 0, s>>>(a);
  return 1;
}

int launch_forward(const FwdArgs& a, int want_g, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)((n_items + NWARP - 1) / NWARP);
  if (want_g || a.count_kept) {
    if (want_g) k_forward<true><<<blocks, NTHREADS, 0, s>>>(a, 0);
    else k_forward<false><<<blocks, NTHREADS, 0, s>>>(a, 0);
    return 1;
  }
  k_item_lists<<<(unsigned)((n_items + IL_WARPS - 1) / IL_WARPS), 32 * IL_WARPS, 0, s>>>(a);
  const unsigned pblocks =
      (unsigned)std::min<int64_t>((n_items + FK_WARPS - 1) / FK_WARPS, 148 * (FK_MIN_BLOCKS / FK_WARPS));
  k_forward_keys<<<pblocks, 32 * FK_WARPS, 0, s>>>(a);
  k_forward<false><<<148 * 4, NTHREADS, 0, s>>>(a, 1);  // slow-path items (usually none)
  return 3;
}

}  // namespace ef
