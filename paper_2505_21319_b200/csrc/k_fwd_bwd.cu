// k_fwd_bwd.cu — S2/S3 forward (+ loss epilogue) and S4 backward.
//
// One CTA = one work item = up to QITEM Morton-consecutive queries inside one coarse cell,
// split into 4 query groups of 32 (one per warp). Both kernels first stage, chunk by chunk,
// the item's candidate keys in shared memory: keys of the lattice cells overlapping the
// item's AABB grown by rho = sqrt(thr / bl_min), kept iff bl_k * dist^2(k, AABB) <= thr.
// Every skipped pair therefore has a - m_j > cutoff_T (reading R-1):
//   forward : thr = max_j mh_j + T_l, mh_j >= m_j the exponent of the best key among the 8
//             lattice corners and the keys of the query's own cell (the shift of the paper's
//             "maximum-reduce"). Each warp then filters the staged keys
//             against its own 32-query sub-box and loops over its list with lanes = queries
//             (Alg. 1). An exact-min slow path runs if sums overflow.
//   backward: thr_g = max_{j in g} (-lambda_j log2e) + T_l per query group g (exact: the
//             forward saved lambda_j). Each staged key gets a 4-bit mask of the groups within
//             reach; keys are bucketed by mask so warps see uniform masks; lanes = keys loop
//             over the queries of their groups with register accumulators (Alg. 2,
//             PAPER.md:L540-568) and issue one red.global.add per channel per (item, key).
#include "efunc_internal.cuh"

namespace ef {

constexpr int NWARP = NTHREADS / 32;
constexpr int TRAV_UNR_MAX = 4;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ int cellc(float p, float inv_h, int NC) {
  float c = floorf((p + 1.0f) * inv_h);
  c = fminf(fmaxf(c, 0.0f), (float)(NC - 1));
  return (int)c;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

struct Box {
  float lx, ly, lz, hx, hy, hz, thr;
};

__device__ __forceinline__ bool within(const float4 a, const Box& b) {
  const float dx = fmaxf(fmaxf(b.lx - a.x, a.x - b.hx), 0.0f);
  const float dy = fmaxf(fmaxf(b.ly - a.y, a.y - b.hy), 0.0f);
  const float dz = fmaxf(fmaxf(b.lz - a.z, a.z - b.hz), 0.0f);
  return a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= b.thr;
}

// warp-level AABB + max(v) of the lanes with act; inactive lanes contribute nothing
__device__ __forceinline__ Box warp_box(bool act, float x, float y, float z, float v) {
  float r[7] = {act ? x : INFINITY, act ? y : INFINITY, act ? z : INFINITY, act ? -x : INFINITY,
                act ? -y : INFINITY, act ? -z : INFINITY, act ? -v : INFINITY};
#pragma unroll
  for (int i = 0; i < 7; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r[i] = fminf(r[i], __shfl_xor_sync(~0u, r[i], o));
  }
  Box b;
  b.lx = r[0]; b.ly = r[1]; b.lz = r[2];
  b.hx = -r[3]; b.hy = -r[4]; b.hz = -r[5];
  b.thr = -r[6];
  return b;
}

struct SmemList {
  float4 a[LCAP];
  float4 b[LCAP];
  int id[LCAP];
  uint16_t widx[NWARP][LCAP];  // forward: per-warp index lists; backward: widx[0] = mask order
  uint8_t mask[LCAP];
  uint32_t row_start[NTHREADS];
  uint32_t row_off[NTHREADS];
  uint32_t wcnt[TRAV_UNR_MAX * NWARP];
  uint32_t wscan[NWARP];
  uint32_t hist[16];
  uint32_t boff[17];
  Box gbox[NWARP];
  Box ibox;
};

// exclusive scan over the 128 threads of the CTA; returns offset, writes total
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t v, uint32_t* s_w, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(~0u, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  uint32_t off = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < NWARP; ++k) {
    const uint32_t c = s_w[k];
    off += (k < w) ? c : 0u;
    tot += c;
  }
  total = tot;
  return incl - v + off;
}

// Stage the candidate keys of an item in chunks of <= LCAP; proc(cnt) consumes sm.a/b/id[0,cnt).
// Every thread of the CTA must call this (it contains __syncthreads); proc is called by all.
// Keys are visited in (row, position) order and compacted in that order, so the staged list is
// deterministic. If gout != nullptr the sorted-key positions of the list are also written to
// gout[0, gcap) (the forward hands its list to the backward). Returns the list length.
constexpr int TRAV_UNR = 2;  // candidates per thread per round (loads in flight)

template <bool NEED_ID, class Proc>
__device__ __forceinline__ uint32_t traverse(const KeysView& kv, const Box box, SmemList& sm, Proc&& proc,
                                             uint32_t* gout = nullptr, uint32_t gcap = 0) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const float rho = sqrtf(box.thr / *kv.bl_min);
  const int NC = kv.NC;
  const int cx0 = cellc(box.lx - rho, kv.inv_h, NC), cx1 = cellc(box.hx + rho, kv.inv_h, NC);
  const int cy0 = cellc(box.ly - rho, kv.inv_h, NC), cy1 = cellc(box.hy + rho, kv.inv_h, NC);
  const int cz0 = cellc(box.lz - rho, kv.inv_h, NC), cz1 = cellc(box.hz + rho, kv.inv_h, NC);
  const int ny = cy1 - cy0 + 1;
  const int nrows = ny * (cz1 - cz0 + 1);
  uint32_t cnt = 0, staged = 0;
  for (int rb = 0; rb < nrows; rb += NTHREADS) {
    const int r = rb + tid;
    uint32_t s = 0, len = 0;
    if (r < nrows) {
      const int cy = cy0 + r % ny, cz = cz0 + r / ny;
      const int base = (cz * NC + cy) * NC;
      s = __ldg(&kv.cell_start[base + cx0]);
      len = __ldg(&kv.cell_start[base + cx1 + 1]) - s;
    }
    uint32_t total;
    const uint32_t off = cta_excl_scan(len, sm.wscan, total);
    sm.row_start[tid] = s;
    sm.row_off[tid] = off;
    __syncthreads();
    int row = 0;  // per-thread row cursor; f only grows, so the walk is amortised O(1)
    for (uint32_t f0 = 0; f0 < total; f0 += TRAV_UNR * NTHREADS) {
      bool pass[TRAV_UNR];
      float4 ka[TRAV_UNR];
      uint32_t kp[TRAV_UNR], bal[TRAV_UNR];
#pragma unroll
      for (int u = 0; u < TRAV_UNR; ++u) {
        const uint32_t f = f0 + u * NTHREADS + tid;
        pass[u] = false;
        kp[u] = 0;
        if (f < total) {
          while (row + 1 < NTHREADS && sm.row_off[row + 1] <= f) ++row;
          kp[u] = sm.row_start[row] + (f - sm.row_off[row]);
          ka[u] = __ldg(&kv.ks[2 * kp[u]]);
        }
      }
#pragma unroll
      for (int u = 0; u < TRAV_UNR; ++u) {
        const uint32_t f = f0 + u * NTHREADS + tid;
        if (f < total) pass[u] = within(ka[u], box);
        bal[u] = __ballot_sync(~0u, pass[u]);
        if (lane == 0) sm.wcnt[u * NWARP + w] = __popc(bal[u]);
      }
      __syncthreads();
      uint32_t base = cnt;
#pragma unroll
      for (int u = 0; u < TRAV_UNR; ++u) {
        uint32_t woff = 0, btot = 0;
#pragma unroll
        for (int k = 0; k < NWARP; ++k) {
          const uint32_t c = sm.wcnt[u * NWARP + k];
          woff += (k < w) ? c : 0u;
          btot += c;
        }
        if (pass[u]) {
          const uint32_t slot = base + woff + __popc(bal[u] & lanemask_lt());
          sm.a[slot] = ka[u];
          sm.b[slot] = __ldg(&kv.ks[2 * kp[u] + 1]);
          if (NEED_ID) sm.id[slot] = __ldg(&kv.kid[kp[u]]);
          if (gout && staged + (slot - cnt) < gcap) gout[staged + (slot - cnt)] = kp[u];
        }
        base += btot;
      }
      staged += base - cnt;
      cnt = base;
      __syncthreads();
      if (cnt > (uint32_t)(LCAP - TRAV_UNR * NTHREADS)) {
        proc(cnt);
        cnt = 0;
        __syncthreads();
      }
    }
  }
  if (cnt > 0) {
    proc(cnt);
    __syncthreads();
  }
  return staged;
}

// Stage a list saved by the forward (sorted-key positions) in chunks of <= LCAP.
template <class Proc>
__device__ __forceinline__ void stage_list(const KeysView& kv, const uint32_t* __restrict__ list, uint32_t n,
                                           SmemList& sm, Proc&& proc) {
  const int tid = threadIdx.x;
  for (uint32_t c0 = 0; c0 < n; c0 += LCAP) {
    const uint32_t cnt = min((uint32_t)LCAP, n - c0);
    for (uint32_t k = tid; k < cnt; k += NTHREADS) {
      const uint32_t kp = __ldg(&list[c0 + k]);
      sm.a[k] = __ldg(&kv.ks[2 * kp]);
      sm.b[k] = __ldg(&kv.ks[2 * kp + 1]);
      sm.id[k] = __ldg(&kv.kid[kp]);
    }
    __syncthreads();
    proc(cnt);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ forward
template <bool WANT_G>
__global__ void __launch_bounds__(NTHREADS) k_forward(const FwdArgs A) {
  __shared__ SmemList sm;
  __shared__ float s_red[NWARP];
  const KeysView& kv = A.kv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t item = blockIdx.x;
  if (item >= *A.n_items) return;
  const int2 it = A.items[item];
  const int64_t j0 = it.x;
  const int nq = it.y;
  const bool act = tid < nq;
  const int nact_w = max(0, min(32, nq - 32 * w));  // active queries of this warp
  const float4 q = act ? A.qs[j0 + tid] : make_float4(0.f, 0.f, 0.f, 0.f);

  // shift bound mh_j >= m_j (log2 units): best of the 8 lattice-corner grid keys and of (up to
  // 32) keys staged in the query's own cell; f0 = f of that key at q (accuracy shift, App. D)
  float mh = INFINITY, f0 = 0.0f;
  if (act) {
    const int R = kv.R, NC = kv.NC;
    const int cx = cellc(q.x, kv.inv_h, NC), cy = cellc(q.y, kv.inv_h, NC), cz = cellc(q.z, kv.inv_h, NC);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int n = (cx + (c & 1)) + R * ((cy + ((c >> 1) & 1)) + R * (cz + (c >> 2)));
      const float4 ka = __ldg(&kv.grid_raw[2 * n]);
      const float dx = q.x - ka.x, dy = q.y - ka.y, dz = q.z - ka.z;
      const float e = ka.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      if (e < mh) {
        mh = e;
        if (WANT_G) {
          const float4 kb = __ldg(&kv.grid_raw[2 * n + 1]);
          f0 = fmaf(kb.w, dz, fmaf(kb.z, dy, fmaf(kb.y, dx, kb.x)));
        }
      }
    }
    const int cid = (cz * NC + cy) * NC + cx;
    const uint32_t s = __ldg(&kv.cell_start[cid]);
    const uint32_t e_ = min(__ldg(&kv.cell_start[cid + 1]), s + 32u);
    for (uint32_t k = s; k < e_; ++k) {
      const float4 ka = __ldg(&kv.ks[2 * k]);
      const float dx = q.x - ka.x, dy = q.y - ka.y, dz = q.z - ka.z;
      const float e = ka.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      if (e < mh) {
        mh = e;
        if (WANT_G) {
          const float4 kb = __ldg(&kv.ks[2 * k + 1]);
          f0 = fmaf(kb.w, dz, fmaf(kb.z, dy, fmaf(kb.y, dx, kb.x)));
        }
      }
    }
  }
  // warp sub-box and item box (union of the warp boxes)
  Box wb = warp_box(act, q.x, q.y, q.z, mh);
  wb.thr += A.T_l;
  if (lane == 0) sm.gbox[w] = wb;
  __syncthreads();
  if (tid == 0) {
    Box ib = sm.gbox[0];
    for (int k = 1; k < NWARP; ++k) {
      const Box g = sm.gbox[k];
      ib.lx = fminf(ib.lx, g.lx); ib.ly = fminf(ib.ly, g.ly); ib.lz = fminf(ib.lz, g.lz);
      ib.hx = fmaxf(ib.hx, g.hx); ib.hy = fmaxf(ib.hy, g.hy); ib.hz = fmaxf(ib.hz, g.hz);
      ib.thr = fmaxf(ib.thr, g.thr);
    }
    sm.ibox = ib;
  }
  __syncthreads();
  const Box ibox = sm.ibox;

  float Z = 0.f, M = 0.f;
  float sgx = 0.f, sgy = 0.f, sgz = 0.f, sux = 0.f, suy = 0.f, suz = 0.f, sfx = 0.f, sfy = 0.f, sfz = 0.f;
  float shift = mh;
  unsigned long long cand = 0;
  auto accum = [&](uint32_t cnt) {
    if (nact_w == 0) return;  // warp-uniform
    // per-warp filter against the warp's own sub-box
    uint32_t nw = 0;
    for (uint32_t base = 0; base < cnt; base += 32) {
      const uint32_t k = base + lane;
      const bool pass = (k < cnt) && within(sm.a[k], wb);
      const uint32_t bal = __ballot_sync(~0u, pass);
      if (pass) sm.widx[w][nw + __popc(bal & lanemask_lt())] = (uint16_t)k;
      nw += __popc(bal);
    }
    __syncwarp();
    cand += (unsigned long long)nw;
    if (!act) return;
#pragma unroll 4
    for (uint32_t i = 0; i < nw; ++i) {
      const uint32_t k = sm.widx[w][i];
      const float4 a = sm.a[k];
      const float4 b = sm.b[k];
      const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
      const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float wgt = ex2f(fmaf(-a.w, dd, shift));
      Z += wgt;
      if (WANT_G) {
        const float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x - f0)));
        sgx = fmaf(wgt, b.y, sgx);
        sgy = fmaf(wgt, b.z, sgy);
        sgz = fmaf(wgt, b.w, sgz);
        const float wbl = wgt * a.w;
        sux = fmaf(wbl, dx, sux);
        suy = fmaf(wbl, dy, suy);
        suz = fmaf(wbl, dz, suz);
        const float wbf = wbl * f;
        sfx = fmaf(wbf, dx, sfx);
        sfy = fmaf(wbf, dy, sfy);
        sfz = fmaf(wbf, dz, sfz);
        M = fmaf(wgt, f, M);
      } else {
        const float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x)));
        M = fmaf(wgt, f, M);
      }
    }
  };
  {
    const uint32_t n = traverse<false>(kv, ibox, sm, accum, A.lists + (size_t)item * A.list_cap, A.list_cap);
    if (tid == 0) A.list_n[item] = n;
  }

  const bool bad = act && !(isfinite(Z) && isfinite(M) && Z > 0.0f);
  if (__syncthreads_or(bad)) {
    // exact-shift slow path: shift = min over the staged set (it contains every argmin key)
    float mexact = INFINITY;
    auto minpass = [&](uint32_t cnt) {
      if (!act) return;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4 a = sm.a[k];
        const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
        mexact = fminf(mexact, a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
      }
    };
    traverse<false>(kv, ibox, sm, minpass);
    shift = mexact;
    Z = M = 0.f;
    sgx = sgy = sgz = sux = suy = suz = sfx = sfy = sfz = 0.f;
    cand = 0;
    traverse<false>(kv, ibox, sm, accum);
    if (tid == 0) atomicAdd(&A.ds->overflow_items, 1u);
  }

  if (A.count_kept) {
    // diagnostic: exact per-query min over the staged set, then count pairs with e - m <= T_l
    float mexact = INFINITY;
    auto minpass = [&](uint32_t cnt) {
      if (!act) return;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4 a = sm.a[k];
        const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
        mexact = fminf(mexact, a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
      }
    };
    traverse<false>(kv, ibox, sm, minpass);
    unsigned long long kept = 0, kept_off = 0;
    auto countpass = [&](uint32_t cnt) {
      if (!act) return;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4 a = sm.a[k];
        const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
        const bool kp = a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)) - mexact <= A.T_l;
        kept += kp ? 1ull : 0ull;
        kept_off += (kp && sm.id[k] >= kv.n_nodes) ? 1ull : 0ull;
      }
    };
    traverse<true>(kv, ibox, sm, countpass);
    for (int o = 16; o > 0; o >>= 1) {
      kept += __shfl_xor_sync(~0u, kept, o);
      kept_off += __shfl_xor_sync(~0u, kept_off, o);
    }
    if (lane == 0) {
      atomicAdd(&A.ds->kept_pairs, kept);
      atomicAdd(&A.ds->kept_pairs_offset, kept_off);
    }
  }
  if (lane == 0 && nact_w > 0) atomicAdd(&A.ds->cand_pairs, cand * (unsigned long long)nact_w);

  // epilogue: O, lambda, G, loss and its upstream
  float lossj = 0.0f;
  if (act) {
    const float iz = 1.0f / Z;
    const float O = (WANT_G ? f0 : 0.0f) + M * iz;
    const float nlam = shift - log2f(Z);  // -lambda_j * log2(e):  p_ij = 2^(nlam - bl_i dd_ij)
    const int64_t js = j0 + tid;
    const int ju = A.perm[js];
    float r = 0.0f;
    float Gx = 0.f, Gy = 0.f, Gz = 0.f;
    if (WANT_G) {
      const float c2 = 2.0f * EF_LN2 * iz;
      const float Of = O - f0;
      Gx = sgx * iz + c2 * fmaf(Of, sux, -sfx);
      Gy = sgy * iz + c2 * fmaf(Of, suy, -sfy);
      Gz = sgz * iz + c2 * fmaf(Of, suz, -sfz);
      A.gs[js] = make_float4(Gx, Gy, Gz, 0.f);
      A.us[js] = make_float4(c2 * sux, c2 * suy, c2 * suz, 0.f);
      if (A.G) {
        A.G[3 * (size_t)ju] = Gx;
        A.G[3 * (size_t)ju + 1] = Gy;
        A.G[3 * (size_t)ju + 2] = Gz;
      }
    }
    if (A.loss_kind >= EFUNC_LOSS_MSE) {
      const float diff = O - q.w;
      r = 2.0f * diff * A.inv_J;
      lossj = diff * diff * A.inv_J;
    }
    if (WANT_G && A.loss_kind == EFUNC_LOSS_MSE_EIKONAL) {
      const float n = sqrtf(fmaf(Gx, Gx, fmaf(Gy, Gy, Gz * Gz)));
      lossj = fmaf(A.eik_lambda * (n - 1.0f) * (n - 1.0f), A.inv_J, lossj);
      const float s = n > 0.0f ? 2.0f * A.eik_lambda * (n - 1.0f) / n * A.inv_J : 0.0f;
      A.hs[js] = make_float4(s * Gx, s * Gy, s * Gz, 0.f);
    }
    A.rec[js] = make_float4(nlam, r, O, 0.f);
    if (A.O) A.O[ju] = O;
  }
  if (A.loss_kind >= EFUNC_LOSS_MSE) {
    for (int o = 16; o > 0; o >>= 1) lossj += __shfl_xor_sync(~0u, lossj, o);
    if (lane == 0) s_red[w] = lossj;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
      for (int k = 0; k < NWARP; ++k) t += s_red[k];
      A.loss_part[item] = t;
    }
  }
}

int launch_forward(const FwdArgs& a, int want_g, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  if (want_g) k_forward<true><<<(unsigned)n_items, NTHREADS, 0, s>>>(a);
  else k_forward<false><<<(unsigned)n_items, NTHREADS, 0, s>>>(a);
  return 1;
}

// ------------------------------------------------------------------------------ backward
template <bool EIK>
__global__ void __launch_bounds__(NTHREADS) k_backward(const BwdArgs A) {
  __shared__ SmemList sm;
  __shared__ float4 sq[QITEM];  // x, y, z, -lambda_l
  __shared__ float4 sv[QITEM];  // r, O, h.ubar, h.G
  __shared__ float4 sh[EIK ? QITEM : 1];
  const KeysView& kv = A.kv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t item = blockIdx.x;
  if (item >= *A.n_items) return;
  const int2 it = A.items[item];
  const int64_t j0 = it.x;
  const int nq = it.y;
  const int ng = (nq + 31) / 32;
  const bool act = tid < nq;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  if (act) {
    const int64_t js = j0 + tid;
    q = A.qs[js];
    const float4 rc = A.rec[js];
    const int ju = A.perm[js];
    const float r = A.dL_dO ? A.dL_dO[ju] : rc.y;
    float hub = 0.f, T = 0.f;
    if (EIK) {
      float4 hv;
      if (A.dL_dG) hv = make_float4(A.dL_dG[3 * (size_t)ju], A.dL_dG[3 * (size_t)ju + 1], A.dL_dG[3 * (size_t)ju + 2], 0.f);
      else hv = A.hs[js];
      const float4 G = A.gs[js], ub = A.us[js];
      hub = hv.x * ub.x + hv.y * ub.y + hv.z * ub.z;
      T = hv.x * G.x + hv.y * G.y + hv.z * G.z;
      sh[tid] = hv;
    }
    q.w = rc.x;
    sq[tid] = q;
    sv[tid] = make_float4(r, rc.z, hub, T);
  }
  // query-group boxes with the exact threshold max_j(-lambda_l) + T_l (pairs with p < 2^-T_l skip)
  Box gb = warp_box(act, q.x, q.y, q.z, q.w);
  gb.thr += A.T_l;
  if (lane == 0) sm.gbox[w] = gb;
  __syncthreads();
  if (tid == 0) {
    Box ib = sm.gbox[0];
    for (int k = 1; k < ng; ++k) {
      const Box g = sm.gbox[k];
      ib.lx = fminf(ib.lx, g.lx); ib.ly = fminf(ib.ly, g.ly); ib.lz = fminf(ib.lz, g.lz);
      ib.hx = fmaxf(ib.hx, g.hx); ib.hy = fmaxf(ib.hy, g.hy); ib.hz = fmaxf(ib.hz, g.hz);
      ib.thr = fmaxf(ib.thr, g.thr);
    }
    sm.ibox = ib;
  }
  __syncthreads();
  const Box ibox = sm.ibox;

  auto proc = [&](uint32_t cnt) {
    // 1. mask of query groups within reach, histogram over masks
    if (tid < 16) sm.hist[tid] = 0;
    __syncthreads();
    for (uint32_t k = tid; k < cnt; k += NTHREADS) {
      const float4 a = sm.a[k];
      uint32_t m = 0;
      for (int g = 0; g < ng; ++g) m |= within(a, sm.gbox[g]) ? (1u << g) : 0u;
      sm.mask[k] = (uint8_t)m;
      if (m) atomicAdd(&sm.hist[m], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t o = 0;
      for (int m = 0; m < 16; ++m) {
        sm.boff[m] = o;
        o += sm.hist[m];
      }
      sm.boff[16] = o;
    }
    __syncthreads();
    const uint32_t nz = sm.boff[16];
    for (uint32_t k = tid; k < cnt; k += NTHREADS) {
      const uint32_t m = sm.mask[k];
      if (m) sm.widx[0][atomicAdd(&sm.boff[m], 1u)] = (uint16_t)k;
    }
    __syncthreads();
    // 2. lanes = keys (mask-bucketed), loop over the queries of the groups in the mask
    for (uint32_t i = tid; i < nz; i += NTHREADS) {
      const uint32_t k = sm.widx[0][i];
      const uint32_t m = sm.mask[k];
      const float4 a = sm.a[k];
      const float4 b = sm.b[k];
      const int id = sm.id[k];
      const float beta = a.w * EF_LN2;
      float sc = 0.f, sgx = 0.f, sgy = 0.f, sgz = 0.f, ss = 0.f, sdx = 0.f, sdy = 0.f, sdz = 0.f;
      float phx = 0.f, phy = 0.f, phz = 0.f, pdx = 0.f, pdy = 0.f, pdz = 0.f;  // EIK only
      for (int g = 0; g < ng; ++g) {
        if (!((m >> g) & 1u)) continue;
        const int jend = min(nq, 32 * g + 32);
#pragma unroll 4
        for (int j = 32 * g; j < jend; ++j) {
          const float4 P = sq[j];
          const float4 V = sv[j];
          const float dx = P.x - a.x, dy = P.y - a.y, dz = P.z - a.z;
          const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
          const float p = ex2f(fmaf(-a.w, dd, P.w));
          const float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x)));
          const float del = f - V.y;
          if (!EIK) {
            // Alg. 2: dO/dc = p, dO/dg = p d, dO/ds = -p a (f - O), dO/dk = p(-g + 2 beta d (f - O))
            const float t = V.x * p;
            const float u = t * del;
            sc += t;
            sgx = fmaf(t, dx, sgx);
            sgy = fmaf(t, dy, sgy);
            sgz = fmaf(t, dz, sgz);
            ss = fmaf(u, dd, ss);
            sdx = fmaf(u, dx, sdx);
            sdy = fmaf(u, dy, sdy);
            sdz = fmaf(u, dz, sdz);
          } else {
            // MSE + second-order (dL/dG) terms, DESIGN.md "Eikonal backward"
            const float4 H = sh[j];
            const float hd = fmaf(H.x, dx, fmaf(H.y, dy, H.z * dz));
            const float hu = 2.0f * beta * hd;
            const float hg = fmaf(H.x, b.y, fmaf(H.y, b.z, H.z * b.w));
            const float tt = fmaf(-hu, del, hg);
            const float alpha = V.x + V.z - hu;
            const float gam = fmaf(V.x + V.z, del, tt - V.w);
            const float pa = p * alpha;
            sc += pa;
            sgx = fmaf(pa, dx, sgx);
            sgy = fmaf(pa, dy, sgy);
            sgz = fmaf(pa, dz, sgz);
            phx = fmaf(p, H.x, phx);
            phy = fmaf(p, H.y, phy);
            phz = fmaf(p, H.z, phz);
            ss = fmaf(p, fmaf(beta * dd, gam, hu * del), ss);
            const float pg = p * gam;
            sdx = fmaf(pg, dx, sdx);
            sdy = fmaf(pg, dy, sdy);
            sdz = fmaf(pg, dz, sdz);
            const float pdel = p * del;
            pdx = fmaf(pdel, H.x, pdx);
            pdy = fmaf(pdel, H.y, pdy);
            pdz = fmaf(pdel, H.z, pdz);
          }
        }
      }
      float dsv, dgx, dgy, dgz, dkx, dky, dkz;
      if (!EIK) {
        dsv = -beta * ss;
        dgx = sgx; dgy = sgy; dgz = sgz;
        dkx = fmaf(-b.y, sc, 2.0f * beta * sdx);
        dky = fmaf(-b.z, sc, 2.0f * beta * sdy);
        dkz = fmaf(-b.w, sc, 2.0f * beta * sdz);
      } else {
        dsv = -ss;
        dgx = sgx + phx; dgy = sgy + phy; dgz = sgz + phz;
        dkx = fmaf(-b.y, sc, 2.0f * beta * (sdx + pdx));
        dky = fmaf(-b.z, sc, 2.0f * beta * (sdy + pdy));
        dkz = fmaf(-b.w, sc, 2.0f * beta * (sdz + pdz));
      }
      if (id < kv.n_nodes) {
        float* gp = A.grad + (size_t)id * EF_NCH;
        atomicAdd(gp + 0, dsv);
        atomicAdd(gp + 1, sc);
        atomicAdd(gp + 2, dgx);
        atomicAdd(gp + 3, dgy);
        atomicAdd(gp + 4, dgz);
      } else {
        float* gp = A.grad + (size_t)(id - kv.n_nodes) * EF_NCH;
        atomicAdd(gp + 5, dkx);
        atomicAdd(gp + 6, dky);
        atomicAdd(gp + 7, dkz);
        atomicAdd(gp + 8, dsv);
        atomicAdd(gp + 9, sc);
        atomicAdd(gp + 10, dgx);
        atomicAdd(gp + 11, dgy);
        atomicAdd(gp + 12, dgz);
      }
    }
  };
  const uint32_t ln = A.list_n[item];
  if (ln <= A.list_cap) stage_list(kv, A.lists + (size_t)item * A.list_cap, ln, sm, proc);
  else traverse<true>(kv, ibox, sm, proc);
}

int launch_backward(const BwdArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  if (a.eik) k_backward<true><<<(unsigned)n_items, NTHREADS, 0, s>>>(a);
  else k_backward<false><<<(unsigned)n_items, NTHREADS, 0, s>>>(a);
  return 1;
}

}  // namespace ef
