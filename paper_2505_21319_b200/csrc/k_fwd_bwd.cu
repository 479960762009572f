// k_fwd_bwd.cu — S2/S3 forward (+ loss epilogue) and S4 backward.
//
// One CTA = one work item = QITEM consecutive Morton-sorted queries. Both kernels walk the
// same candidate key set of the item: keys in the lattice cells overlapping the item's AABB
// grown by rho = sqrt(thr / bl_min), kept iff bl_k * dist^2(k, AABB) <= thr, where
// thr = max_j mh_j + T_l (log2 units) and mh_j >= m_j is the exponent of the nearest of the
// 8 lattice-corner grid keys of query j. A skipped pair therefore has a - m_j > cutoff_T
// (reading R-1). Candidates are staged in shared memory (LCAP per chunk) and
// broadcast to the lanes:
//   forward : lanes = queries, loop over staged keys (Alg. 1; the
//             shift of the paper's "maximum-reduce", L501, is the corner bound mh_j; an
//             exact-min slow path runs if an item's sums overflow)
//   backward: lanes = staged keys, loop over the item's queries in shared memory; per key
//             register accumulators (Alg. 2, PAPER.md:L540-568 restricted to the item), one
//             red.global.add per gradient channel per (item, key).
#include "efunc_internal.cuh"

namespace ef {

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

struct SmemList {
  float4 a[LCAP];
  float4 b[LCAP];
  int id[LCAP];
  uint32_t row_start[NTHREADS];
  uint32_t row_off[NTHREADS];
  uint32_t wcnt[NTHREADS / 32];
  uint32_t wscan[NTHREADS / 32];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

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
  for (int k = 0; k < NTHREADS / 32; ++k) {
    const uint32_t c = s_w[k];
    off += (k < w) ? c : 0u;
    tot += c;
  }
  total = tot;
  return incl - v + off;
}

// Walk the candidate keys of an item in chunks of <= LCAP; proc(cnt) consumes sm.a/b/id[0,cnt).
// Every thread of the CTA must call this (it contains __syncthreads). Returns candidates seen.
template <bool NEED_ID, class Proc>
__device__ __forceinline__ uint32_t traverse(const KeysView& kv, const ItemBox& box, SmemList& sm, Proc&& proc) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const float thr = box.lo.w;
  const float rho = sqrtf(thr / *kv.bl_min);
  const int NC = kv.NC;
  const int cx0 = cellc(box.lo.x - rho, kv.inv_h, NC), cx1 = cellc(box.hi.x + rho, kv.inv_h, NC);
  const int cy0 = cellc(box.lo.y - rho, kv.inv_h, NC), cy1 = cellc(box.hi.y + rho, kv.inv_h, NC);
  const int cz0 = cellc(box.lo.z - rho, kv.inv_h, NC), cz1 = cellc(box.hi.z + rho, kv.inv_h, NC);
  const int ny = cy1 - cy0 + 1;
  const int nrows = ny * (cz1 - cz0 + 1);
  uint32_t cnt = 0, seen = 0;
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
    for (uint32_t f0 = 0; f0 < total; f0 += NTHREADS) {
      const uint32_t f = f0 + tid;
      bool pass = false;
      float4 ka = make_float4(0.f, 0.f, 0.f, 0.f);
      uint32_t kp = 0;
      if (f < total) {
        int lo = 0, hi = NTHREADS;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (sm.row_off[mid] <= f) lo = mid; else hi = mid;
        }
        kp = sm.row_start[lo] + (f - sm.row_off[lo]);
        ka = __ldg(&kv.ks[2 * kp]);
        const float dx = fmaxf(fmaxf(box.lo.x - ka.x, ka.x - box.hi.x), 0.0f);
        const float dy = fmaxf(fmaxf(box.lo.y - ka.y, ka.y - box.hi.y), 0.0f);
        const float dz = fmaxf(fmaxf(box.lo.z - ka.z, ka.z - box.hi.z), 0.0f);
        pass = ka.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= thr;
      }
      const uint32_t bal = __ballot_sync(~0u, pass);
      if (lane == 0) sm.wcnt[w] = __popc(bal);
      __syncthreads();
      uint32_t woff = 0, btot = 0;
#pragma unroll
      for (int k = 0; k < NTHREADS / 32; ++k) {
        const uint32_t c = sm.wcnt[k];
        woff += (k < w) ? c : 0u;
        btot += c;
      }
      if (pass) {
        const uint32_t slot = cnt + woff + __popc(bal & lanemask_lt());
        sm.a[slot] = ka;
        sm.b[slot] = __ldg(&kv.ks[2 * kp + 1]);
        if (NEED_ID) sm.id[slot] = __ldg(&kv.kid[kp]);
      }
      cnt += btot;
      __syncthreads();
      if (cnt > (uint32_t)(LCAP - NTHREADS)) {
        proc(cnt);
        seen += cnt;
        cnt = 0;
        __syncthreads();
      }
    }
  }
  if (cnt > 0) {
    proc(cnt);
    seen += cnt;
    __syncthreads();
  }
  return seen;
}

// ------------------------------------------------------------------------------ forward
template <bool WANT_G>
__global__ void __launch_bounds__(NTHREADS) k_forward(const FwdArgs A) {
  __shared__ SmemList sm;
  __shared__ float s_red[7][NTHREADS / 32];
  const KeysView& kv = A.kv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t j0 = (int64_t)blockIdx.x * QITEM;
  const int nq = (int)((A.J - j0) < (int64_t)QITEM ? (A.J - j0) : (int64_t)QITEM);
  const bool act = tid < nq;
  const float4 q = act ? A.qs[j0 + tid] : make_float4(0.f, 0.f, 0.f, 0.f);

  // shift bound mh_j: exponent (log2 units) of the best of the 8 lattice-corner grid keys
  float mh = INFINITY, f0 = 0.0f;
  if (act) {
    const int R = kv.R;
    const int cx = cellc(q.x, kv.inv_h, kv.NC), cy = cellc(q.y, kv.inv_h, kv.NC), cz = cellc(q.z, kv.inv_h, kv.NC);
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
  }
  // item box: AABB of the active queries + max shift bound
  float r7[7] = {act ? q.x : INFINITY, act ? q.y : INFINITY, act ? q.z : INFINITY,
                 act ? -q.x : INFINITY, act ? -q.y : INFINITY, act ? -q.z : INFINITY,
                 act ? -mh : INFINITY};
#pragma unroll
  for (int i = 0; i < 7; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r7[i] = fminf(r7[i], __shfl_xor_sync(~0u, r7[i], o));
    if (lane == 0) s_red[i][w] = r7[i];
  }
  __syncthreads();
  ItemBox box;
  {
    float v[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      v[i] = s_red[i][0];
#pragma unroll
      for (int k = 1; k < NTHREADS / 32; ++k) v[i] = fminf(v[i], s_red[i][k]);
    }
    box.lo = make_float4(v[0], v[1], v[2], -v[6] + A.T_l);
    box.hi = make_float4(-v[3], -v[4], -v[5], 0.0f);
  }
  if (tid == 0) A.boxes[blockIdx.x] = box;

  float Z = 0.f, M = 0.f;
  float sgx = 0.f, sgy = 0.f, sgz = 0.f, sux = 0.f, suy = 0.f, suz = 0.f, sfx = 0.f, sfy = 0.f, sfz = 0.f;
  float shift = mh;
  auto accum = [&](uint32_t cnt) {
    if (!act) return;
#pragma unroll 4
    for (uint32_t k = 0; k < cnt; ++k) {
      const float4 a = sm.a[k];
      const float4 b = sm.b[k];
      const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
      const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float wgt = ex2f(fmaf(-a.w, dd, shift));
      float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x)));
      Z += wgt;
      if (WANT_G) {
        f -= f0;
        sgx = fmaf(wgt, b.y, sgx);
        sgy = fmaf(wgt, b.z, sgy);
        sgz = fmaf(wgt, b.w, sgz);
        const float wb = wgt * a.w;
        sux = fmaf(wb, dx, sux);
        suy = fmaf(wb, dy, suy);
        suz = fmaf(wb, dz, suz);
        const float wbf = wb * f;
        sfx = fmaf(wbf, dx, sfx);
        sfy = fmaf(wbf, dy, sfy);
        sfz = fmaf(wbf, dz, sfz);
      }
      M = fmaf(wgt, f, M);
    }
  };
  uint32_t cand = traverse<false>(kv, box, sm, accum);

  const bool bad = act && !(isfinite(Z) && isfinite(M) && Z > 0.0f);
  if (__syncthreads_or(bad)) {
    // exact-shift slow path: shift = min over the candidate set (contains the argmin key)
    float mexact = INFINITY;
    auto minpass = [&](uint32_t cnt) {
      if (!act) return;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4 a = sm.a[k];
        const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
        mexact = fminf(mexact, a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
      }
    };
    traverse<false>(kv, box, sm, minpass);
    shift = mexact;
    Z = M = 0.f;
    sgx = sgy = sgz = sux = suy = suz = sfx = sfy = sfz = 0.f;
    traverse<false>(kv, box, sm, accum);
    if (tid == 0) atomicAdd(&A.ds->overflow_items, 1u);
  }

  if (A.count_kept) {
    // diagnostic: exact per-query min over candidates, then count pairs with e - m <= T_l
    float mexact = INFINITY;
    auto minpass = [&](uint32_t cnt) {
      if (!act) return;
      for (uint32_t k = 0; k < cnt; ++k) {
        const float4 a = sm.a[k];
        const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
        mexact = fminf(mexact, a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
      }
    };
    traverse<false>(kv, box, sm, minpass);
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
    traverse<true>(kv, box, sm, countpass);
    for (int o = 16; o > 0; o >>= 1) {
      kept += __shfl_xor_sync(~0u, kept, o);
      kept_off += __shfl_xor_sync(~0u, kept_off, o);
    }
    if (lane == 0) {
      atomicAdd(&A.ds->kept_pairs, kept);
      atomicAdd(&A.ds->kept_pairs_offset, kept_off);
    }
  }
  if (tid == 0) atomicAdd(&A.ds->cand_pairs, (unsigned long long)cand * (unsigned long long)nq);

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
    __syncthreads();
    if (lane == 0) s_red[0][w] = lossj;
    __syncthreads();
    if (tid == 0) {
      float t = 0.f;
      for (int k = 0; k < NTHREADS / 32; ++k) t += s_red[0][k];
      A.loss_part[blockIdx.x] = t;
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
  const int tid = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * QITEM;
  const int nq = (int)((A.J - j0) < (int64_t)QITEM ? (A.J - j0) : (int64_t)QITEM);
  if (tid < nq) {
    const int64_t js = j0 + tid;
    const float4 q = A.qs[js];
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
    sq[tid] = make_float4(q.x, q.y, q.z, rc.x);
    sv[tid] = make_float4(r, rc.z, hub, T);
  }
  const ItemBox box = A.boxes[blockIdx.x];
  __syncthreads();

  auto proc = [&](uint32_t cnt) {
    for (uint32_t k = tid; k < cnt; k += NTHREADS) {
      const float4 a = sm.a[k];
      const float4 b = sm.b[k];
      const int id = sm.id[k];
      const float beta = a.w * EF_LN2;
      float sc = 0.f, sgx = 0.f, sgy = 0.f, sgz = 0.f, ss = 0.f, sdx = 0.f, sdy = 0.f, sdz = 0.f;
      float phx = 0.f, phy = 0.f, phz = 0.f, pdx = 0.f, pdy = 0.f, pdz = 0.f;  // EIK only
#pragma unroll 4
      for (int j = 0; j < nq; ++j) {
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
        float* g = A.grad + (size_t)id * EF_NCH;
        atomicAdd(g + 0, dsv);
        atomicAdd(g + 1, sc);
        atomicAdd(g + 2, dgx);
        atomicAdd(g + 3, dgy);
        atomicAdd(g + 4, dgz);
      } else {
        float* g = A.grad + (size_t)(id - kv.n_nodes) * EF_NCH;
        atomicAdd(g + 5, dkx);
        atomicAdd(g + 6, dky);
        atomicAdd(g + 7, dkz);
        atomicAdd(g + 8, dsv);
        atomicAdd(g + 9, sc);
        atomicAdd(g + 10, dgx);
        atomicAdd(g + 11, dgy);
        atomicAdd(g + 12, dgz);
      }
    }
  };
  traverse<true>(kv, box, sm, proc);
}

int launch_backward(const BwdArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  if (a.eik) k_backward<true><<<(unsigned)n_items, NTHREADS, 0, s>>>(a);
  else k_backward<false><<<(unsigned)n_items, NTHREADS, 0, s>>>(a);
  return 1;
}

}  // namespace ef
