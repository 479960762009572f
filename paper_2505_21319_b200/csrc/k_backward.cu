// k_backward.cu — S4 backward: lanes = the item's candidate keys, the item's queries
// broadcast from shared memory, register accumulators (Alg. 2); per (key,
// item) two red.global.add.v4.f32 into a 16-float-per-node padded gradient folded to the ABI
// layout by k_fold, or 64-bit fixed-point atomics in deterministic mode.
#include <algorithm>

#include "k_pair.cuh"

namespace ef {

// ------------------------------------------------------------------------------ backward
// DET: deterministic mode, 64-bit fixed-point accumulation (see BwdArgs::gfix)
#ifndef BK_MIN_BLOCKS
#define BK_MIN_BLOCKS 28  // warps per SM: <= 72 registers (measured best of 1/28/32)
#endif
constexpr int BW_WARPS = 4;  // persistent: warps per CTA, each fetching items heaviest-first

// per-warp shared memory of the backward
template <bool EIK>
struct BwdSmem {
  float4 sq[QW];  // x, y, z, -lambda_l
  float4 sv[QW];  // r, O, h.ubar, h.G
  float4 sh[EIK ? QW : 1];
  // MSE: the item's queries as packed pairs for f32x2 arithmetic: {x0,x1,y0,y1}, {z0,z1,w0,w1},
  // {r0,r1,-O0,-O1} (an idle slot has w = -inf and r = 0: it contributes exactly 0)
  float4 pA[EIK ? 1 : QW / 2], pB[EIK ? 1 : QW / 2], pC[EIK ? 1 : QW / 2];
  float4 ka[WSLICE];  // fallback staging ring
  float4 kb[WSLICE];
  int kid[WSLICE];
};

template <bool EIK, bool DET>
__device__ __forceinline__ void backward_item(const BwdArgs& A, const uint32_t item, BwdSmem<EIK>& S,
                                              const float fix_scale) {
  auto fix_add = [&](unsigned long long* p, float v) {
    const float qv = v * fix_scale;
    if (fabsf(qv) < 4.0e18f) {
      atomicAdd(p, (unsigned long long)(long long)rintf(qv));
    } else {
      atomicOr(A.fix_overflow, 1u);
    }
  };
  float4* const pA = S.pA;
  float4* const pB = S.pB;
  float4* const pC = S.pC;
  const KeysView& kv = A.kv;
  const int lane = threadIdx.x & 31;
  const int4 it = A.items[item];
  const int nact = it.y;
  Box box;
#pragma unroll
  for (int u = 0; u < QW / 32; ++u) {
    const int j = lane + 32 * u;
    const bool act = j < nact;
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
      const int64_t js = (int64_t)it.x + j;
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
        S.sh[j] = hv;
      }
      q.w = rc.x;
      S.sq[j] = q;
      S.sv[j] = make_float4(r, rc.z, hub, T);
    }
    if (!EIK) {
      const float x = q.x, y = q.y, z = q.z, wv = act ? q.w : -INFINITY;
      const float r = act ? S.sv[j].x : 0.f, nO = act ? -S.sv[j].y : 0.f;
      const float xo = __shfl_xor_sync(~0u, x, 1), yo = __shfl_xor_sync(~0u, y, 1), zo = __shfl_xor_sync(~0u, z, 1);
      const float wo = __shfl_xor_sync(~0u, wv, 1), ro = __shfl_xor_sync(~0u, r, 1), nOo = __shfl_xor_sync(~0u, nO, 1);
      if ((lane & 1) == 0) {
        pA[j >> 1] = make_float4(x, xo, y, yo);
        pB[j >> 1] = make_float4(z, zo, wv, wo);
        pC[j >> 1] = make_float4(r, ro, nO, nOo);
      }
    }
    // item box with the exact threshold max_j(-lambda_l) + T_l (fallback path only)
    const Box b = warp_box(act, q.x, q.y, q.z, q.w);
    if (u == 0) {
      box = b;
    } else {
      box.lx = fminf(box.lx, b.lx); box.ly = fminf(box.ly, b.ly); box.lz = fminf(box.lz, b.lz);
      box.hx = fmaxf(box.hx, b.hx); box.hy = fmaxf(box.hy, b.hy); box.hz = fmaxf(box.hz, b.hz);
      box.thr = fmaxf(box.thr, b.thr);
    }
  }
  box.thr += A.T_l;
  __syncwarp();
  const float4* Q = S.sq;
  const float4* V = S.sv;
  const float4* H = S.sh;
  float4* sa = S.ka;
  float4* sb = S.kb;
  int* sid = S.kid;
  float* gpad = A.gpad;
  const int n_nodes = kv.n_nodes;

  // lanes = keys: lane i takes staged key head + i, loops over the group's queries
  // one key per lane over the item's queries; register accumulators, reds at the end
  auto process = [&](const bool has, const float4 a, const float4 b, const int id) {
    if (!has) return;
    const float beta = a.w * EF_LN2;
    float sc = 0.f, sgx = 0.f, sgy = 0.f, sgz = 0.f, ss = 0.f, sdx = 0.f, sdy = 0.f, sdz = 0.f;
    float phx = 0.f, phy = 0.f, phz = 0.f, pdx = 0.f, pdy = 0.f, pdz = 0.f;  // EIK only
    auto pair = [&](const float4 P, const float4 U, const float4 h) {
      const float dx = P.x - a.x, dy = P.y - a.y, dz = P.z - a.z;
      const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float p = ex2f(fmaf(-a.w, dd, P.w));
      const float f = fmaf(b.w, dz, fmaf(b.z, dy, fmaf(b.y, dx, b.x)));
      const float del = f - U.y;
      if (!EIK) {
        // Alg. 2: dO/dc = p, dO/dg = p d, dO/ds = -p a (f - O), dO/dk = p(-g + 2 beta d (f - O))
        const float t = U.x * p;
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
        const float hd = fmaf(h.x, dx, fmaf(h.y, dy, h.z * dz));
        const float hu = 2.0f * beta * hd;
        const float hg = fmaf(h.x, b.y, fmaf(h.y, b.z, h.z * b.w));
        const float tt = fmaf(-hu, del, hg);
        const float alpha = U.x + U.z - hu;
        const float gam = fmaf(U.x + U.z, del, tt - U.w);
        const float pa = p * alpha;
        sc += pa;
        sgx = fmaf(pa, dx, sgx);
        sgy = fmaf(pa, dy, sgy);
        sgz = fmaf(pa, dz, sgz);
        phx = fmaf(p, h.x, phx);
        phy = fmaf(p, h.y, phy);
        phz = fmaf(p, h.z, phz);
        ss = fmaf(p, fmaf(beta * dd, gam, hu * del), ss);
        const float pg = p * gam;
        sdx = fmaf(pg, dx, sdx);
        sdy = fmaf(pg, dy, sdy);
        sdz = fmaf(pg, dz, sdz);
        const float pdel = p * del;
        pdx = fmaf(pdel, h.x, pdx);
        pdy = fmaf(pdel, h.y, pdy);
        pdz = fmaf(pdel, h.z, pdz);
      }
    };
    if (!EIK) {
      // two queries per f32x2 instruction (k_pair.cuh)
      const MseSums ms = bwd_mse_sums(a, b, (nact + 1) >> 1, pA, pB, pC);
      sc = ms.sc; sgx = ms.sgx; sgy = ms.sgy; sgz = ms.sgz;
      ss = ms.ss; sdx = ms.sdx; sdy = ms.sdy; sdz = ms.sdz;
    } else {
      // register double-buffering of the broadcast query loads hides the LDS latency
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 P0 = Q[0], U0 = V[0], H0 = EIK ? H[0] : z4;
#pragma unroll 4
      for (int j = 1; j < nact; ++j) {
        const float4 P1 = Q[j], U1 = V[j], H1 = EIK ? H[j] : z4;
        pair(P0, U0, H0);
        P0 = P1;
        U0 = U1;
        H0 = H1;
      }
      pair(P0, U0, H0);
    }
    float dsv, dgx, dgy, dgz;
    if (!EIK) {
      dsv = -beta * ss;
      dgx = sgx; dgy = sgy; dgz = sgz;
    } else {
      dsv = -ss;
      dgx = sgx + phx; dgy = sgy + phy; dgz = sgz + phz;
    }
    // padded gradient: node n -> 16 floats {s0,c0,g0x,g0y | g0z,-,-,- | dx,dy,dz,s1 | c1,g1x,g1y,g1z}
    if (id < n_nodes) {
      if (!DET) {
        float* gp = gpad + (size_t)id * 16;
        red_v4(gp, dsv, sc, dgx, dgy);
        atomicAdd(gp + 4, dgz);
      } else {
        unsigned long long* gp = A.gfix + (size_t)id * 16;
        fix_add(gp + 0, dsv); fix_add(gp + 1, sc); fix_add(gp + 2, dgx); fix_add(gp + 3, dgy);
        fix_add(gp + 4, dgz);
      }
    } else {
      float dkx, dky, dkz;
      if (!EIK) {
        dkx = fmaf(-b.y, sc, 2.0f * beta * sdx);
        dky = fmaf(-b.z, sc, 2.0f * beta * sdy);
        dkz = fmaf(-b.w, sc, 2.0f * beta * sdz);
      } else {
        dkx = fmaf(-b.y, sc, 2.0f * beta * (sdx + pdx));
        dky = fmaf(-b.z, sc, 2.0f * beta * (sdy + pdy));
        dkz = fmaf(-b.w, sc, 2.0f * beta * (sdz + pdz));
      }
      if (!DET) {
        float* gp = gpad + (size_t)(id - n_nodes) * 16 + 8;
        red_v4(gp, dkx, dky, dkz, dsv);
        red_v4(gp + 4, sc, dgx, dgy, dgz);
      } else {
        unsigned long long* gp = A.gfix + (size_t)(id - n_nodes) * 16 + 8;
        fix_add(gp + 0, dkx); fix_add(gp + 1, dky); fix_add(gp + 2, dkz); fix_add(gp + 3, dsv);
        fix_add(gp + 4, sc); fix_add(gp + 5, dgx); fix_add(gp + 6, dgy); fix_add(gp + 7, dgz);
      }
    }
  };

  const uint32_t wn = A.wl_n[item];
  if (wn != BL_OVERFLOW) {
    // the forward's candidate ids of this item: one key per lane, records gathered straight into
    // registers; ids prefetched two batches ahead and records one batch ahead, so neither
    // gather waits on a load issued just before it; no test, no staging
    const uint32_t* L = A.wl_pool + A.wl_off[item];
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t id1 = ((uint32_t)lane < wn) ? __ldg(&L[lane]) : 0u;
    uint32_t id2 = ((uint32_t)lane + 32 < wn) ? __ldg(&L[lane + 32]) : 0u;
    float4 a1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1]) : z4;
    float4 b1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
    for (uint32_t base = 0; base < wn; base += 32) {
      const uint32_t k = base + lane;
      const bool has = k < wn;
      const uint32_t id = id1;
      const float4 a = a1, b = b1;
      id1 = id2;
      id2 = (k + 64 < wn) ? __ldg(&L[k + 64]) : 0u;
      if (k + 32 < wn) {
        a1 = __ldg(&kv.grid_raw[2 * id1]);
        b1 = __ldg(&kv.grid_raw[2 * id1 + 1]);
      }
      process(has, a, b, (int)id);
    }
    return;
  }
  // fallback: stream the brick list (or enumerate) with this item's own test, stage in a ring
  auto consume = [&](uint32_t head, uint32_t count) {
    __syncwarp();
    const bool has = (uint32_t)lane < count;
    const uint32_t slot = (head + lane) % WSLICE;
    const float4 a = has ? sa[slot] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b = has ? sb[slot] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int id = has ? sid[slot] : 0;
    __syncwarp();
    process(has, a, b, id);
  };
  uint32_t head = 0, cnt = 0;  // ring buffer of staged keys
  candidates(kv, it.z, box, [&](bool pass, uint32_t kp, float4 a, float4 b) {
    const uint32_t bal = __ballot_sync(~0u, pass);
    if (pass) {
      const uint32_t slot = (head + cnt + __popc(bal & lanemask_lt())) % WSLICE;
      sa[slot] = a;
      sb[slot] = b;
      sid[slot] = (int)kp;
    }
    cnt += __popc(bal);
    if (cnt >= 32) {
      consume(head, 32);
      head = (head + 32) % WSLICE;
      cnt -= 32;
    }
  });
  if (cnt) consume(head, cnt);
}

template <bool EIK, bool DET>
__global__ void __launch_bounds__(32 * BW_WARPS, BK_MIN_BLOCKS / BW_WARPS) k_backward(const BwdArgs A) {
  __shared__ BwdSmem<EIK> smem[BW_WARPS];
  float fix_scale = 0.0f;
  if (DET) {
    const float um = *A.umax;
    fix_scale = um > 0.0f ? (float)(1ull << FIX_BITS) / um : 0.0f;
  }
  BwdSmem<EIK>& S = smem[threadIdx.x >> 5];
  for (;;) {
    const int64_t item = fetch_item(A.next, A.n_items, A.list, A.list_n);
    if (item < 0) break;
    __syncwarp();  // the previous item's readers of S are done
    backward_item<EIK, DET>(A, (uint32_t)item, S, fix_scale);
  }
}

static unsigned bwd_blocks(int64_t n_items) {
  return (unsigned)std::min<int64_t>((n_items + BW_WARPS - 1) / BW_WARPS, 148 * (BK_MIN_BLOCKS / BW_WARPS));
}

int launch_backward(const BwdArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  // list mode (the fused path's leftover items, usually none): one CTA per SM
  const unsigned blocks = a.list ? 148u : bwd_blocks(n_items);
  if (a.eik) k_backward<true, false><<<blocks, 32 * BW_WARPS, 0, s>>>(a);
  else k_backward<false, false><<<blocks, 32 * BW_WARPS, 0, s>>>(a);
  return 1;
}

// max_j (|dL/dO_j| + |dL/dG_j|_1): the fixed-point unit of the deterministic backward (a max is
// independent of the order the atomics land in)
__global__ void k_upstream_max(const BwdArgs A, float* umax) {
  float m = 0.0f;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < A.J; j += (int64_t)gridDim.x * blockDim.x) {
    float v = fabsf(A.dL_dO ? A.dL_dO[j] : A.rec[j].y);
    if (A.eik) {
      if (A.dL_dG) v += fabsf(A.dL_dG[3 * j]) + fabsf(A.dL_dG[3 * j + 1]) + fabsf(A.dL_dG[3 * j + 2]);
      else v += fabsf(A.hs[j].x) + fabsf(A.hs[j].y) + fabsf(A.hs[j].z);
    }
    m = fmaxf(m, v);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(~0u, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(reinterpret_cast<unsigned int*>(umax), __float_as_uint(m));
}

int launch_backward_det(const BwdArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  long ub = (a.J + 255) / 256;
  if (ub > 148 * 8) ub = 148 * 8;
  k_upstream_max<<<(unsigned)(ub < 1 ? 1 : ub), 256, 0, s>>>(a, const_cast<float*>(a.umax));
  const unsigned blocks = bwd_blocks(n_items);
  if (a.eik) k_backward<true, true><<<blocks, 32 * BW_WARPS, 0, s>>>(a);
  else k_backward<false, true><<<blocks, 32 * BW_WARPS, 0, s>>>(a);
  return 2;
}

// Deterministic fused path: the fixed-point unit must be known before the fused kernel computes
// the upstreams, so it comes from an a-priori bound of max_j |r_j| = 2 |O_j - o_j| / J: O_j is a
// convex combination of key polynomials f_i(q_j) = c_i + g_i.(q_j - k_i) with |q_a - k_a| <= 2 +
// |Delta_a| for in-domain queries, so |r_j| <= 2/J (max_i (|c_i| + |g_i|_1 (2 + |Delta_i|_inf))
// + max_j |o_j|) <= 4/J max(...). A max is independent of the order the atomics land in.
__global__ void k_det_bound(const float* __restrict__ theta, int n_nodes, const float4* __restrict__ qs, int64_t J,
                            float inv_J, float* umax) {
  float m = 0.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n_nodes + J;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n_nodes) {
      const float* t = theta + (size_t)i * EF_NCH;
      const float dm = fmaxf(fabsf(t[5]), fmaxf(fabsf(t[6]), fabsf(t[7])));
      const float f0 = fabsf(t[1]) + (fabsf(t[2]) + fabsf(t[3]) + fabsf(t[4])) * 2.0f;
      const float f1 = fabsf(t[9]) + (fabsf(t[10]) + fabsf(t[11]) + fabsf(t[12])) * (2.0f + dm);
      m = fmaxf(m, fmaxf(f0, f1));
    } else {
      m = fmaxf(m, fabsf(qs[i - n_nodes].w));
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(~0u, m, o));
  m *= 4.0f * inv_J;
  if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(reinterpret_cast<unsigned int*>(umax), __float_as_uint(m));
}

int launch_det_bound(const float* theta, int n_nodes, const float4* qs, int64_t J, float inv_J, float* umax,
                     cudaStream_t s) {
  const int64_t n = (int64_t)n_nodes + J;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
  k_det_bound<<<blocks, 256, 0, s>>>(theta, n_nodes, qs, J, inv_J, umax);
  return 1;
}

// the deterministic backward of the items in a.list (the fused path's leftovers) with the unit in
// *a.umax as set before the fused kernel
int launch_backward_list_det(const BwdArgs& a, cudaStream_t s) {
  k_backward<false, true><<<148u, 32 * BW_WARPS, 0, s>>>(a);
  return 1;
}

// grad[n][13] += fixed-point sums * umax * 2^-FIX_BITS; zero the accumulator
__global__ void k_fold_fix(unsigned long long* __restrict__ gfix, const float* __restrict__ umax,
                           float* __restrict__ grad, int n_nodes) {
  const double unit = (double)*umax / (double)(1ull << FIX_BITS);
  const int map[13] = {0, 1, 2, 3, 4, 8, 9, 10, 11, 12, 13, 14, 15};
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += gridDim.x * blockDim.x) {
    unsigned long long* p = gfix + (size_t)n * 16;
    float* g = grad + (size_t)n * EF_NCH;
#pragma unroll
    for (int c = 0; c < 13; ++c) g[c] += (float)((double)(long long)p[map[c]] * unit);
#pragma unroll
    for (int c = 0; c < 16; ++c) p[c] = 0ull;
  }
}

int launch_fold_fix(unsigned long long* gfix, const float* umax, float* grad, int n_nodes, cudaStream_t s) {
  int blocks = (n_nodes + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_fold_fix<<<blocks, 256, 0, s>>>(gfix, umax, grad, n_nodes);
  return 1;
}

// grad[n][13] += padded gradient (channel map above); zero the padded buffer for the next call
__global__ void k_fold(float* __restrict__ gpad, float* __restrict__ grad, int n_nodes) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += gridDim.x * blockDim.x) {
    float4* p = reinterpret_cast<float4*>(gpad + (size_t)n * 16);
    const float4 v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3];
    float* g = grad + (size_t)n * EF_NCH;
    g[0] += v0.x; g[1] += v0.y; g[2] += v0.z; g[3] += v0.w; g[4] += v1.x;
    g[5] += v2.x; g[6] += v2.y; g[7] += v2.z; g[8] += v2.w;
    g[9] += v3.x; g[10] += v3.y; g[11] += v3.z; g[12] += v3.w;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    p[0] = z; p[1] = z; p[2] = z; p[3] = z;
  }
}

// The fold fused with the data-parallel reduction: thread i takes gradient floats 4i .. 4i+3 of the
// [R^3][13] layout (their gpad slots, zeroed after reading) and adds the float4 into every rank's
// copy of the symmetric gradient buffer: one NVLS multimem.red through the multicast address, or
// one red.global.add.v4 per peer mapping (NVLink P2P). gpad slot of channel c: the grid bank's 5
// channels at 0..4, the offset bank's 8 at 8..15 (k_fold's map).
__device__ __forceinline__ int gpad_slot(const int c) { return c < 5 ? c : c + 3; }

__global__ void k_fold_peers(float* __restrict__ gpad, int n_nodes, float* const* __restrict__ peers, int n_peers,
                             float* __restrict__ mc) {
  const int64_t n4 = (int64_t)n_nodes * EF_NCH / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t f = 4 * i + k;
      const int64_t n = f / EF_NCH;
      float* p = gpad + n * 16 + gpad_slot((int)(f - n * EF_NCH));
      v[k] = *p;
      *p = 0.0f;
    }
    if (mc) {
      asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(v[0]),
                   "f"(v[1]), "f"(v[2]), "f"(v[3])
                   : "memory");
    } else {
      for (int r = 0; r < n_peers; ++r) red_v4(peers[r] + 4 * i, v[0], v[1], v[2], v[3]);
    }
  }
}

int launch_fold_peers(float* gpad, int n_nodes, float* const* peers, int n_peers, float* mc, cudaStream_t s) {
  const int64_t n4 = (int64_t)n_nodes * EF_NCH / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_fold_peers<<<blocks, 256, 0, s>>>(gpad, n_nodes, peers, n_peers, mc);
  return 1;
}

int launch_fold(float* gpad, float* grad, int n_nodes, cudaStream_t s) {
  int blocks = (n_nodes + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_fold<<<blocks, 256, 0, s>>>(gpad, grad, n_nodes);
  return 1;
}

}  // namespace ef
