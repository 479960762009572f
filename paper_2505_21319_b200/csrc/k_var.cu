// k_var.cu — NEXT-4: the Table 3 model families beyond the
// default O^{+Delta} with degree-1 polynomials.
//
//   * Layout conversion between the user's per-variant parameter layout (include/efunc.h,
//     efunc_channels) and the internal one: the 13-channel record the fused kernels read
//     (grid bank s0 c0 g0 | Delta | offset bank s1 c1 g1; a bank the variant does not have is
//     disabled in S0, see k_prep_keys) plus, for degree 2, the two symmetric squares
//     H = (Hxx, Hyy, Hzz, Hxy, Hxz, Hyz) of Eq. poly-func per node.
//   * Degree 2 (f = c + g.d + 1/2 d^T H d, d = q - k): forward (O, and G of Eq. func-normal,
//     PAPER.md:L425-436, with df/dq = g + H d) and MSE backward (Alg. 2, with
//     dO/dH_ab = p d_a d_b (1/2 on the diagonal), dO/dk = p [-(g + H d) + 2 beta d (f - O)]).
//     One warp per work item over the item's certified candidate list (k_item_lists, reading R-1);
//     the forward takes the exact per-query minimum exponent (two passes over the candidates),
//     lanes = queries; the backward lanes = candidate keys, queries broadcast from shared memory.
#include "efunc_internal.cuh"
#include "k_common.cuh"

namespace ef {

// ------------------------------------------------------------------ layout conversion
__global__ void k_var_unpack(const float* __restrict__ tv, int n, VarLayout L, float* __restrict__ t13,
                             float* __restrict__ tH) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float* s = tv + (size_t)i * L.nch;
    float* d = t13 + (size_t)i * EF_NCH;
    float* h = tH ? tH + (size_t)i * 12 : nullptr;
#pragma unroll
    for (int c = 0; c < EF_NCH; ++c) d[c] = 0.0f;
    if (h) {
#pragma unroll
      for (int c = 0; c < 12; ++c) h[c] = 0.0f;
    }
    auto bank = [&](int s0, int o13, int oH) {
      d[o13] = s[s0];
      d[o13 + 1] = s[s0 + 1];
      if (L.deg >= 1) {
        d[o13 + 2] = s[s0 + 2];
        d[o13 + 3] = s[s0 + 3];
        d[o13 + 4] = s[s0 + 4];
      }
      if (L.deg >= 2 && h) {
#pragma unroll
        for (int c = 0; c < 6; ++c) h[oH + c] = s[s0 + 5 + c];
      }
    };
    if (L.grid >= 0) bank(L.grid, 0, 0);
    if (L.off >= 0) {
      bank(L.off, 8, 6);
      d[5] = s[L.delta];
      d[6] = s[L.delta + 1];
      d[7] = s[L.delta + 2];
    }
  }
}

// grad_v += the internal gradients (13-channel record + the H channels)
__global__ void k_var_pack_grad(const float* __restrict__ g13, const float* __restrict__ gH, int n, VarLayout L,
                                float* __restrict__ gv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float* d = gv + (size_t)i * L.nch;
    const float* s = g13 + (size_t)i * EF_NCH;
    const float* h = gH ? gH + (size_t)i * 12 : nullptr;
    auto bank = [&](int s0, int o13, int oH) {
      d[s0] += s[o13];
      d[s0 + 1] += s[o13 + 1];
      if (L.deg >= 1) {
        d[s0 + 2] += s[o13 + 2];
        d[s0 + 3] += s[o13 + 3];
        d[s0 + 4] += s[o13 + 4];
      }
      if (L.deg >= 2 && h) {
#pragma unroll
        for (int c = 0; c < 6; ++c) d[s0 + 5 + c] += h[oH + c];
      }
    };
    if (L.grid >= 0) bank(L.grid, 0, 0);
    if (L.off >= 0) {
      bank(L.off, 8, 6);
      d[L.delta] += s[5];
      d[L.delta + 1] += s[6];
      d[L.delta + 2] += s[7];
    }
  }
}

// the internal Delta channels (after the mean-shift initialisation) into the user layout
__global__ void k_var_delta_out(const float* __restrict__ t13, int n, VarLayout L, float* __restrict__ tv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) tv[(size_t)i * L.nch + L.delta + c] = t13[(size_t)i * EF_NCH + 5 + c];
  }
}

// key id -> its square: {Hxx, Hyy, Hzz, Hxy}, {Hxz, Hyz, 0, 0}
__global__ void k_var_keyH(const float* __restrict__ tH, int n, float4* __restrict__ keyH) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += gridDim.x * blockDim.x) {
    const int node = i < n ? i : i - n;
    const float* h = tH + (size_t)node * 12 + (i < n ? 0 : 6);
    keyH[2 * i] = make_float4(h[0], h[1], h[2], h[3]);
    keyH[2 * i + 1] = make_float4(h[4], h[5], 0.0f, 0.0f);
  }
}

static unsigned grid_for(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

int launch_var_unpack(const float* tv, int n, const VarLayout& L, float* t13, float* tH, cudaStream_t s) {
  k_var_unpack<<<grid_for(n), 256, 0, s>>>(tv, n, L, t13, tH);
  return 1;
}
int launch_var_pack_grad(const float* g13, const float* gH, int n, const VarLayout& L, float* gv, cudaStream_t s) {
  k_var_pack_grad<<<grid_for(n), 256, 0, s>>>(g13, gH, n, L, gv);
  return 1;
}
int launch_var_delta_out(const float* t13, int n, const VarLayout& L, float* tv, cudaStream_t s) {
  k_var_delta_out<<<grid_for(n), 256, 0, s>>>(t13, n, L, tv);
  return 1;
}
int launch_var_keyH(const float* tH, int n, float4* keyH, cudaStream_t s) {
  k_var_keyH<<<grid_for(2 * (int64_t)n), 256, 0, s>>>(tH, n, keyH);
  return 1;
}

// ------------------------------------------------------------------ degree 2
// df/dq = g + H d and f - f0 = (c - f0) + 1/2 (g.d + (g + H d).d): the constant is taken off the
// coefficient before the sum, so the rounding scales with |f - f0| rather than |f| (the u-term of
// G and the backward's f - O multiply it by 2 beta |d| ~ 300)
__device__ __forceinline__ float quad_f(const float4 b, const float4 h1, const float4 h2, float dx, float dy, float dz,
                                        float f0, float& fx, float& fy, float& fz) {
  fx = fmaf(h2.x, dz, fmaf(h1.w, dy, fmaf(h1.x, dx, b.y)));
  fy = fmaf(h2.y, dz, fmaf(h1.y, dy, fmaf(h1.w, dx, b.z)));
  fz = fmaf(h1.z, dz, fmaf(h2.y, dy, fmaf(h2.x, dx, b.w)));
  const float gd = fmaf(b.w, dz, fmaf(b.z, dy, b.y * dx));
  const float fd = fmaf(fz, dz, fmaf(fy, dy, fx * dx));
  return fmaf(0.5f, gd + fd, b.x - f0);
}

constexpr int VQ_WARPS = 4;

struct VarStage {
  float4 a[32], b[32], h1[32], h2[32];
};

// the item's candidate ids: its certified list (k_item_lists) or, without one (overflowed brick,
// out-of-domain item, dense mode), every enabled key
__device__ __forceinline__ void var_item_list(const FwdArgs& A, const uint32_t item, const uint32_t* iota,
                                              uint32_t iota_n, const uint32_t*& L, uint32_t& wn) {
  const uint32_t n = (A.wl_n != nullptr && !isinf(A.T_l)) ? A.wl_n[item] : BL_OVERFLOW;
  if (n == BL_OVERFLOW) {
    L = iota;
    wn = iota_n;
  } else {
    L = A.wl_pool + A.wl_off[item];
    wn = n;
  }
}

__device__ __forceinline__ void var_stage(const KeysView& kv, const float4* keyH, const uint32_t* L, uint32_t base,
                                          uint32_t wn, VarStage& S) {
  const uint32_t lane = threadIdx.x & 31;
  __syncwarp();
  if (base + lane < wn) {
    const uint32_t id = L[base + lane];
    S.a[lane] = __ldg(&kv.grid_raw[2 * id]);
    S.b[lane] = __ldg(&kv.grid_raw[2 * id + 1]);
    S.h1[lane] = __ldg(&keyH[2 * id]);
    S.h2[lane] = __ldg(&keyH[2 * id + 1]);
  }
  __syncwarp();
}

template <bool WANT_G>
__global__ void __launch_bounds__(32 * VQ_WARPS) k_var_forward(const FwdArgs A, const float4* __restrict__ keyH,
                                                               const uint32_t* __restrict__ iota, uint32_t iota_n) {
  __shared__ VarStage stage[VQ_WARPS];
  VarStage& S = stage[threadIdx.x >> 5];
  const uint32_t item = blockIdx.x * VQ_WARPS + (threadIdx.x >> 5);
  if (item >= *A.n_items) return;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const bool act = lane < it.y;
  const int64_t js = (int64_t)it.x + lane;
  const float4 q = act ? A.qs[js] : make_float4(0.f, 0.f, 0.f, 0.f);
  const uint32_t* L;
  uint32_t wn;
  var_item_list(A, item, iota, iota_n, L, wn);
  // pass 1: m_j = min_i a_ij (log2 units) and its key (the accuracy shift f0)
  float m = INFINITY;
  uint32_t arg = 0;
  for (uint32_t base = 0; base < wn; base += 32) {
    var_stage(kv, keyH, L, base, wn, S);
    const uint32_t cnt = min(32u, wn - base);
    for (uint32_t k = 0; k < cnt; ++k) {
      const float4 a = S.a[k];
      const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
      const float al = a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      if (al < m) {
        m = al;
        arg = base + k;
      }
    }
  }
  // f0 and df0/dq of the argmin key: the sums below are taken relative to them (accuracy)
  float f0 = 0.0f, fx0 = 0.0f, fy0 = 0.0f, fz0 = 0.0f;
  if (act && wn > 0) {
    const uint32_t id = L[arg];
    const float4 a = __ldg(&kv.grid_raw[2 * id]), b = __ldg(&kv.grid_raw[2 * id + 1]);
    const float4 h1 = __ldg(&keyH[2 * id]), h2 = __ldg(&keyH[2 * id + 1]);
    f0 = quad_f(b, h1, h2, q.x - a.x, q.y - a.y, q.z - a.z, 0.0f, fx0, fy0, fz0);
  }
  // pass 2: Z = sum w, M = sum w (f - f0), G sums (Eq. func-normal)
  float Z = 0.f, M = 0.f, sfx = 0.f, sfy = 0.f, sfz = 0.f, sux = 0.f, suy = 0.f, suz = 0.f, svx = 0.f, svy = 0.f,
        svz = 0.f;
  unsigned long long kept = 0;
  for (uint32_t base = 0; base < wn; base += 32) {
    var_stage(kv, keyH, L, base, wn, S);
    const uint32_t cnt = min(32u, wn - base);
    for (uint32_t k = 0; k < cnt; ++k) {
      const float4 a = S.a[k];
      const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
      const float al = a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      if (al - m > A.T_l) continue;  // certified cutoff (reading R-1)
      ++kept;
      const float w = ex2f(m - al);
      float fx, fy, fz;
      const float f = quad_f(S.b[k], S.h1[k], S.h2[k], dx, dy, dz, f0, fx, fy, fz);  // f - f0
      Z += w;
      M = fmaf(w, f, M);
      if (WANT_G) {
        sfx = fmaf(w, fx - fx0, sfx);
        sfy = fmaf(w, fy - fy0, sfy);
        sfz = fmaf(w, fz - fz0, sfz);
        const float wb = w * a.w;
        sux = fmaf(wb, dx, sux);
        suy = fmaf(wb, dy, suy);
        suz = fmaf(wb, dz, suz);
        const float wbf = wb * f;
        svx = fmaf(wbf, dx, svx);
        svy = fmaf(wbf, dy, svy);
        svz = fmaf(wbf, dz, svz);
      }
    }
  }
  float lossj = 0.f;
  if (act) {
    const float iz = 1.0f / Z;
    const float Mz = M * iz;  // O - f0
    const float O = f0 + Mz;
    float r = 0.f;
    if (A.loss_kind != EFUNC_LOSS_NONE) {
      const float diff = O - q.w;
      r = 2.0f * diff * A.inv_J;
      lossj = diff * diff * A.inv_J;
    }
    const int p = A.perm[js];
    if (A.O) A.O[p] = O;
    // -lambda_j (log2 units) = m_j - log2 Z_j: the backward's p_ij = 2^(-lambda_j - a_ij)
    A.rec[js] = make_float4(m - __log2f(Z), r, O, 0.f);
    if (WANT_G && A.G) {
      // G = f_d0 + sum p (g + H d - f_d0) + 2 beta sum p d (O - f), beta = bl ln 2,
      // (O - f) = (O - f0) - (f - f0)
      const float c2 = 2.0f * EF_LN2 * iz;
      A.G[3 * (int64_t)p] = fx0 + fmaf(c2, fmaf(Mz, sux, -svx), sfx * iz);
      A.G[3 * (int64_t)p + 1] = fy0 + fmaf(c2, fmaf(Mz, suy, -svy), sfy * iz);
      A.G[3 * (int64_t)p + 2] = fz0 + fmaf(c2, fmaf(Mz, suz, -svz), sfz * iz);
    }
    if (!isfinite(q.x) || !isfinite(q.y) || !isfinite(q.z)) A.ds->nonfinite = 1u;
  }
  for (int s = 16; s > 0; s >>= 1) lossj += __shfl_xor_sync(~0u, lossj, s);
  for (int s = 16; s > 0; s >>= 1) kept += __shfl_xor_sync(~0u, kept, s);
  if (lane == 0) {
    A.loss_part[item] = lossj;
    atomicAdd(&A.ds->cand_pairs, (unsigned long long)wn * (unsigned long long)it.y);
    if (A.count_kept) atomicAdd(&A.ds->kept_pairs, kept);
  }
}

struct VarQ {
  float x[32], y[32], z[32], nl[32], r[32], O[32];
};

__global__ void __launch_bounds__(32 * VQ_WARPS) k_var_backward(const FwdArgs A, const float4* __restrict__ keyH,
                                                                const uint32_t* __restrict__ iota, uint32_t iota_n,
                                                                const float* __restrict__ dL_dO,
                                                                float* __restrict__ g13, float* __restrict__ gH) {
  __shared__ VarQ sq[VQ_WARPS];
  VarQ& Q = sq[threadIdx.x >> 5];
  const uint32_t item = blockIdx.x * VQ_WARPS + (threadIdx.x >> 5);
  if (item >= *A.n_items) return;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  if (lane < nact) {
    const int64_t js = (int64_t)it.x + lane;
    const float4 q = A.qs[js];
    const float4 rc = A.rec[js];
    Q.x[lane] = q.x;
    Q.y[lane] = q.y;
    Q.z[lane] = q.z;
    Q.nl[lane] = rc.x;
    Q.r[lane] = dL_dO ? dL_dO[A.perm[js]] : rc.y;
    Q.O[lane] = rc.z;
  }
  __syncwarp();
  const uint32_t* L;
  uint32_t wn;
  var_item_list(A, item, iota, iota_n, L, wn);
  const int n = kv.n_nodes;
  for (uint32_t base = 0; base < wn; base += 32) {
    if (base + lane >= wn) break;
    const uint32_t id = L[base + lane];
    const float4 a = __ldg(&kv.grid_raw[2 * id]), b = __ldg(&kv.grid_raw[2 * id + 1]);
    const float4 h1 = __ldg(&keyH[2 * id]), h2 = __ldg(&keyH[2 * id + 1]);
    float sc = 0.f, sgx = 0.f, sgy = 0.f, sgz = 0.f, hxx = 0.f, hyy = 0.f, hzz = 0.f, hxy = 0.f, hxz = 0.f,
          hyz = 0.f, ss = 0.f, sdx = 0.f, sdy = 0.f, sdz = 0.f;
    for (int j = 0; j < nact; ++j) {
      const float dx = Q.x[j] - a.x, dy = Q.y[j] - a.y, dz = Q.z[j] - a.z;
      const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float e = fmaf(-a.w, dd, Q.nl[j]);  // log2 p_ij
      if (e < -A.T_l) continue;                  // p < 2^-T (reading R-1)
      const float t = Q.r[j] * ex2f(e);
      float fx, fy, fz;
      const float u = t * quad_f(b, h1, h2, dx, dy, dz, Q.O[j], fx, fy, fz);  // t (f - O_j)
      sc += t;
      sgx = fmaf(t, dx, sgx);
      sgy = fmaf(t, dy, sgy);
      sgz = fmaf(t, dz, sgz);
      const float tx = t * dx, ty = t * dy;
      hxx = fmaf(tx, dx, hxx);
      hyy = fmaf(ty, dy, hyy);
      hzz = fmaf(t * dz, dz, hzz);
      hxy = fmaf(tx, dy, hxy);
      hxz = fmaf(tx, dz, hxz);
      hyz = fmaf(ty, dz, hyz);
      ss = fmaf(u, dd, ss);
      sdx = fmaf(u, dx, sdx);
      sdy = fmaf(u, dy, sdy);
      sdz = fmaf(u, dz, sdz);
    }
    const float beta = a.w * EF_LN2;
    const float ds = -beta * ss;
    float* gr;
    float* gq;
    if ((int)id < n) {
      gr = g13 + (size_t)id * EF_NCH;
      gq = gH + (size_t)id * 12;
      atomicAdd(gr + 0, ds);
      atomicAdd(gr + 1, sc);
      atomicAdd(gr + 2, sgx);
      atomicAdd(gr + 3, sgy);
      atomicAdd(gr + 4, sgz);
    } else {
      gr = g13 + (size_t)(id - n) * EF_NCH;
      gq = gH + (size_t)(id - n) * 12 + 6;
      // dO/dk = p [-(g + H d) + 2 beta d (f - O)]: sum_j t (g + H d) = g sc + H sg
      const float tb = 2.0f * beta;
      atomicAdd(gr + 5, fmaf(tb, sdx, -fmaf(b.y, sc, fmaf(h1.x, sgx, fmaf(h1.w, sgy, h2.x * sgz)))));
      atomicAdd(gr + 6, fmaf(tb, sdy, -fmaf(b.z, sc, fmaf(h1.w, sgx, fmaf(h1.y, sgy, h2.y * sgz)))));
      atomicAdd(gr + 7, fmaf(tb, sdz, -fmaf(b.w, sc, fmaf(h2.x, sgx, fmaf(h2.y, sgy, h1.z * sgz)))));
      atomicAdd(gr + 8, ds);
      atomicAdd(gr + 9, sc);
      atomicAdd(gr + 10, sgx);
      atomicAdd(gr + 11, sgy);
      atomicAdd(gr + 12, sgz);
    }
    atomicAdd(gq + 0, 0.5f * hxx);
    atomicAdd(gq + 1, 0.5f * hyy);
    atomicAdd(gq + 2, 0.5f * hzz);
    atomicAdd(gq + 3, hxy);
    atomicAdd(gq + 4, hxz);
    atomicAdd(gq + 5, hyz);
  }
}

int launch_var_forward(const FwdArgs& a, const float4* keyH, const uint32_t* iota, uint32_t iota_n, int want_g,
                       int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)((n_items + VQ_WARPS - 1) / VQ_WARPS);
  if (want_g) k_var_forward<true><<<blocks, 32 * VQ_WARPS, 0, s>>>(a, keyH, iota, iota_n);
  else k_var_forward<false><<<blocks, 32 * VQ_WARPS, 0, s>>>(a, keyH, iota, iota_n);
  return 1;
}

int launch_var_backward(const FwdArgs& a, const float4* keyH, const uint32_t* iota, uint32_t iota_n,
                        const float* dL_dO, float* g13, float* gH, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)((n_items + VQ_WARPS - 1) / VQ_WARPS);
  k_var_backward<<<blocks, 32 * VQ_WARPS, 0, s>>>(a, keyH, iota, iota_n, dL_dO, g13, gH);
  return 1;
}

}  // namespace ef
