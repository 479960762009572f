// k_fwd_bwd.cu — S2/S3 forward (+ loss epilogue) and S4 backward.
//
// A work item is up to QITEM Morton-consecutive queries inside one coarse cell; each of the
// CTA's 4 warps owns one group of 32 of them and runs independently (no block barrier on the
// hot path). A warp enumerates the lattice cells overlapping its group's AABB grown by
// rho = sqrt(thr / bl_min), keeps key k iff bl_k * dist^2(k, AABB) <= thr (warp-level
// flattened row scan, deterministic order), stages the kept keys in its own shared-memory
// slice and consumes them 32 at a time:
//   forward : thr = max_j mh_j + T_l, mh_j >= m_j the exponent of the best key among the
//             query's 8 lattice corners and its own cell (the shift of the paper's
//             "maximum-reduce"). Every skipped pair has a - m_j > cutoff_T
//             (reading R-1). Lanes = queries, staged keys broadcast (Alg. 1,
//             PAPER.md:L505-518, and the G sums of Eq. func-normal). An exact-min
//             slow path runs if a query's sums overflow.
//   backward: thr = max_j(-lambda_j log2e) + T_l (the forward saved lambda_j; a skipped pair
//             has p_ij < e^-T). Lanes = staged keys, the group's queries broadcast from shared
//             memory, register accumulators (Alg. 2); per (key, group) two
//             red.global.add.v4.f32 into a 16-float-per-node padded gradient, folded into the
//             ABI layout by k_fold.
#include "efunc_internal.cuh"

namespace ef {

constexpr int WSLICE = 64;  // staged keys per warp

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

__device__ __forceinline__ void red_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
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

// distance from a lattice cell's extent along one axis to [lo, hi]; boundary cells extend to
// infinity (out-of-domain keys are clamped into them); the cell is widened by a rounding margin
__device__ __forceinline__ float cell_gap(int c, int NC, float h, float lo, float hi) {
  const float m = 1e-3f * h;
  const float clo = (c == 0) ? -INFINITY : fmaf((float)c, h, -1.0f) - m;
  const float chi = (c == NC - 1) ? INFINITY : fmaf((float)(c + 1), h, -1.0f) + m;
  return fmaxf(fmaxf(lo - chi, clo - hi), 0.0f);
}

// Warp-level candidate enumeration. Visits, in (row, position) order, the keys of the lattice-
// cell rows (x-runs) that can hold a key within rho = sqrt(thr / bl_min) of the box: rows whose
// y-z gap exceeds rho are skipped and each row's x-range is cut to the ball's chord. Calls
// stage(pass, kp, a) on every lane for each batch of 32 (warp-uniform call; a valid iff pass).
template <class Stage>
__device__ __forceinline__ void enumerate(const KeysView& kv, const Box& box, Stage&& stage) {
  const int lane = threadIdx.x & 31;
  const float rho2 = box.thr / *kv.bl_min;
  const float rho = sqrtf(rho2);
  const int NC = kv.NC;
  const int cy0 = cellc(box.ly - rho, kv.inv_h, NC), cy1 = cellc(box.hy + rho, kv.inv_h, NC);
  const int cz0 = cellc(box.lz - rho, kv.inv_h, NC), cz1 = cellc(box.hz + rho, kv.inv_h, NC);
  const int ny = cy1 - cy0 + 1;
  const int nrows = ny * (cz1 - cz0 + 1);
  for (int rb = 0; rb < nrows; rb += 32) {
    const int r = rb + lane;
    uint32_t s = 0, len = 0;
    if (r < nrows) {
      const int cy = cy0 + r % ny, cz = cz0 + r / ny;
      const float gy = cell_gap(cy, NC, kv.h, box.ly, box.hy);
      const float gz = cell_gap(cz, NC, kv.h, box.lz, box.hz);
      const float g2 = fmaf(gy, gy, gz * gz);
      if (!(g2 > rho2)) {
        const float rx = sqrtf(fmaxf(rho2 - g2, 0.0f));
        const int cx0 = cellc(box.lx - rx, kv.inv_h, NC), cx1 = cellc(box.hx + rx, kv.inv_h, NC);
        const int base = (cz * NC + cy) * NC;
        s = __ldg(&kv.cell_start[base + cx0]);
        len = __ldg(&kv.cell_start[base + cx1 + 1]) - s;
      }
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(~0u, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(~0u, incl, 31);
    const uint32_t off = incl - len;
    for (uint32_t f0 = 0; f0 < total; f0 += 32) {
      const uint32_t f = f0 + lane;
      // source row: the largest lane l with off_l <= f (empty rows resolve to the next one)
      int lo = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const uint32_t o = __shfl_sync(~0u, off, lo + st);
        if (o <= f) lo += st;
      }
      const uint32_t srow = __shfl_sync(~0u, s, lo);
      const uint32_t soff = __shfl_sync(~0u, off, lo);
      const bool valid = f < total;
      const uint32_t kp = srow + (f - soff);
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      bool pass = false;
      if (valid) {
        a = __ldg(&kv.ks[2 * kp]);
        pass = within(a, box);
      }
      stage(pass, kp, a);
    }
  }
}

// Same visit order as enumerate(), but the flattened position -> row map of each 32-row batch
// is materialised in a per-warp byte array (owner), so every lane resolves its row with one
// shared-memory load instead of a 5-step shuffle search, and two loads per lane are in flight.
// Batches longer than cap fall back to the shuffle search.
constexpr int OWN_CAP = 4096;

template <class Stage>
__device__ __forceinline__ void enumerate_owned(const KeysView& kv, const Box& box, uint8_t* owner,
                                                uint32_t* rs, uint32_t* ro, Stage&& stage) {
  const int lane = threadIdx.x & 31;
  const float rho2 = box.thr / *kv.bl_min;
  const float rho = sqrtf(rho2);
  const int NC = kv.NC;
  const int cy0 = cellc(box.ly - rho, kv.inv_h, NC), cy1 = cellc(box.hy + rho, kv.inv_h, NC);
  const int cz0 = cellc(box.lz - rho, kv.inv_h, NC), cz1 = cellc(box.hz + rho, kv.inv_h, NC);
  const int ny = cy1 - cy0 + 1;
  const int nrows = ny * (cz1 - cz0 + 1);
  for (int rb = 0; rb < nrows; rb += 32) {
    const int r = rb + lane;
    uint32_t s = 0, len = 0;
    if (r < nrows) {
      const int cy = cy0 + r % ny, cz = cz0 + r / ny;
      const float gy = cell_gap(cy, NC, kv.h, box.ly, box.hy);
      const float gz = cell_gap(cz, NC, kv.h, box.lz, box.hz);
      const float g2 = fmaf(gy, gy, gz * gz);
      if (!(g2 > rho2)) {
        const float rx = sqrtf(fmaxf(rho2 - g2, 0.0f));
        const int cx0 = cellc(box.lx - rx, kv.inv_h, NC), cx1 = cellc(box.hx + rx, kv.inv_h, NC);
        const int base = (cz * NC + cy) * NC;
        s = __ldg(&kv.cell_start[base + cx0]);
        len = __ldg(&kv.cell_start[base + cx1 + 1]) - s;
      }
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(~0u, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(~0u, incl, 31);
    const uint32_t off = incl - len;
    if (total > (uint32_t)OWN_CAP) {
      for (uint32_t f0 = 0; f0 < total; f0 += 32) {
        const uint32_t f = f0 + lane;
        int lo = 0;
#pragma unroll
        for (int st = 16; st > 0; st >>= 1) {
          const uint32_t o = __shfl_sync(~0u, off, lo + st);
          if (o <= f) lo += st;
        }
        const uint32_t kp = __shfl_sync(~0u, s, lo) + (f - __shfl_sync(~0u, off, lo));
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        bool pass = false;
        if (f < total) {
          a = __ldg(&kv.ks[2 * kp]);
          pass = within(a, box);
        }
        stage(pass, kp, a);
      }
      continue;
    }
    rs[lane] = s;
    ro[lane] = off;
    for (int rr = 0; rr < 32; ++rr) {
      const uint32_t l = __shfl_sync(~0u, len, rr), o = __shfl_sync(~0u, off, rr);
      for (uint32_t t = lane; t < l; t += 32) owner[o + t] = (uint8_t)rr;
    }
    __syncwarp();
    for (uint32_t f0 = 0; f0 < total; f0 += 64) {
      uint32_t kp[2];
      float4 a[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t f = f0 + 32 * u + lane;
        kp[u] = 0;
        a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (f < total) {
          const int rw = owner[f];
          kp[u] = rs[rw] + (f - ro[rw]);
          a[u] = __ldg(&kv.ks[2 * kp[u]]);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t f = f0 + 32 * u + lane;
        if (f0 + 32 * u < total) stage(f < total && within(a[u], box), kp[u], a[u]);
      }
    }
    __syncwarp();
  }
}

// Candidate keys of a warp item: stream its brick's precomputed list (k_brick_lists, key ids)
// through the warp's own test, or enumerate directly for out-of-domain items and overflowed
// bricks. stage(pass, key id, a) as for enumerate().
// The list stream is software-pipelined: ids two batches ahead, both key records one batch
// ahead, so the L2 latency of the gathers overlaps the previous batch's compute.
template <class Stage>
__device__ __forceinline__ void candidates(const KeysView& kv, int brick, const Box& box, Stage&& stage) {
  uint32_t n = BL_OVERFLOW;
  if (brick >= 0) n = __ldg(&kv.bl_n[brick]);
  if (n == BL_OVERFLOW) {
    enumerate(kv, box, [&](bool pass, uint32_t kp, float4 a) {
      const float4 b = pass ? __ldg(&kv.ks[2 * kp + 1]) : make_float4(0.f, 0.f, 0.f, 0.f);
      stage(pass, pass ? (uint32_t)__ldg(&kv.kid[kp]) : 0u, a, b);
    });
    return;
  }
  const uint32_t* L = kv.bl_pool + __ldg(&kv.bl_off[brick]);
  const uint32_t lane = threadIdx.x & 31;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t id1 = (lane < n) ? __ldg(&L[lane]) : 0u;            // batch i
  uint32_t id2 = (lane + 32 < n) ? __ldg(&L[lane + 32]) : 0u;  // batch i+1
  float4 a1 = (lane < n) ? __ldg(&kv.grid_raw[2 * id1]) : z4;
  float4 b1 = (lane < n) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t k = base + lane;
    const uint32_t id = id1;
    const float4 a = a1, b = b1;
    // prefetch
    id1 = id2;
    id2 = (k + 64 < n) ? __ldg(&L[k + 64]) : 0u;
    if (k + 32 < n) {
      a1 = __ldg(&kv.grid_raw[2 * id1]);
      b1 = __ldg(&kv.grid_raw[2 * id1 + 1]);
    }
    const bool pass = (k < n) && within(a, box);
    stage(pass, id, a, b);
  }
}

__device__ __forceinline__ uint32_t compact3(uint32_t v) {  // inverse of the Morton spread
  v &= 0x09249249u;
  v = (v | (v >> 2)) & 0x030C30C3u;
  v = (v | (v >> 4)) & 0x0300F00Fu;
  v = (v | (v >> 8)) & 0x030000FFu;
  v = (v | (v >> 16)) & 0x000003FFu;
  return v;
}

// Per brick (one warp each): every key that can reach some query inside the brick. A query in
// cell c has mh <= bl_max(c's corners) * 3h^2/4 (its nearest corner is within sqrt(3) h / 2),
// so thr_brick = bl_max(brick nodes) * 3h^2/4 + T_l bounds every warp threshold of the step.
constexpr int KB_WARPS = 2;
__global__ void __launch_bounds__(32 * KB_WARPS) k_brick_lists(const KeysView kv, const BrickGeom bg, float T_l,
                                                          uint32_t* __restrict__ pool, uint32_t pool_cap,
                                                          uint32_t* __restrict__ off, uint32_t* __restrict__ nout,
                                                          DevScalars* ds) {
  __shared__ uint32_t st[KB_WARPS][BL_CAP];
  __shared__ uint8_t own[KB_WARPS][OWN_CAP];
  __shared__ uint32_t rs[KB_WARPS][32], ro[KB_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (!ds->lists_invalid) return;  // the lists of an earlier step are still valid (Verlet skin)
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ds->list_builds, 1u);
  for (uint32_t code = blockIdx.x * KB_WARPS + w; code < bg.n_codes; code += gridDim.x * KB_WARPS) {
  const int bx = (int)compact3(code), by = (int)compact3(code >> 1), bz = (int)compact3(code >> 2);
  if (bx >= bg.nb || by >= bg.nb || bz >= bg.nb) {
    if (lane == 0) {
      off[code] = 0;
      nout[code] = 0;
    }
    continue;
  }
  const int NC = kv.NC, R = kv.R, B = bg.B;
  const int c0x = bx * B, c1x = min(NC, c0x + B) - 1;
  const int c0y = by * B, c1y = min(NC, c0y + B) - 1;
  const int c0z = bz * B, c1z = min(NC, c0z + B) - 1;
  const int nx = c1x - c0x + 2, ny = c1y - c0y + 2, nz = c1z - c0z + 2;
  float blmax = 0.0f;
  for (int t = lane; t < nx * ny * nz; t += 32) {
    const int ix = c0x + t % nx, iy = c0y + (t / nx) % ny, iz = c0z + t / (nx * ny);
    blmax = fmaxf(blmax, __ldg(&kv.grid_raw[2 * (ix + R * (iy + R * iz))]).w);
  }
  for (int o = 16; o > 0; o >>= 1) blmax = fmaxf(blmax, __shfl_xor_sync(~0u, blmax, o));
  // Verlet skin: valid while every key stays within skin of its build position and its bl within a
  // factor (1+mu): grow the box by skin and the threshold by (1+mu) for both the key's and the
  // corner keys' bl drift.
  const float h = kv.h, m = 1e-3f * h + SKIN_H * h;
  const float mu1 = 1.0f + SKIN_MU;
  Box box;
  box.lx = fmaf((float)c0x, h, -1.0f) - m; box.hx = fmaf((float)(c1x + 1), h, -1.0f) + m;
  box.ly = fmaf((float)c0y, h, -1.0f) - m; box.hy = fmaf((float)(c1y + 1), h, -1.0f) + m;
  box.lz = fmaf((float)c0z, h, -1.0f) - m; box.hz = fmaf((float)(c1z + 1), h, -1.0f) + m;
  box.thr = mu1 * (mu1 * blmax * 0.75f * h * h * 1.001f + T_l) + 1e-3f;
  uint32_t cnt = 0;
  enumerate_owned(kv, box, own[w], rs[w], ro[w], [&](bool pass, uint32_t kp, float4 a) {
    const uint32_t bal = __ballot_sync(~0u, pass);
    if (pass) {
      const uint32_t slot = cnt + __popc(bal & lanemask_lt());
      if (slot < (uint32_t)BL_CAP) st[w][slot] = (uint32_t)__ldg(&kv.kid[kp]);  // key id
    }
    cnt += __popc(bal);
  });
  uint32_t base = 0;
  if (lane == 0 && cnt <= (uint32_t)BL_CAP) base = atomicAdd(&ds->pool_top, cnt);
  base = __shfl_sync(~0u, base, 0);
  if (cnt > (uint32_t)BL_CAP || base + cnt > pool_cap) {
    if (lane == 0) {
      off[code] = 0;
      nout[code] = BL_OVERFLOW;
      atomicAdd(&ds->ovf_count, 1u);
    }
    continue;
  }
  __syncwarp();
  for (uint32_t i = lane; i < cnt; i += 32) pool[base + i] = st[w][i];
  if (lane == 0) {
    off[code] = base;
    nout[code] = cnt;
  }
  __syncwarp();
  }
}

int launch_brick_lists(const KeysView& kv, const BrickGeom& bg, float T_l, uint32_t* pool, uint32_t pool_cap,
                       uint32_t* off, uint32_t* n, DevScalars* ds, cudaStream_t s) {
  uint32_t blocks = (bg.n_codes + KB_WARPS - 1) / KB_WARPS;
  if (blocks > 148u * 16u) blocks = 148u * 16u;
  k_brick_lists<<<blocks, 32 * KB_WARPS, 0, s>>>(kv, bg, T_l, pool, pool_cap, off, n, ds);
  return 1;
}

// Shift bound mh_j >= m_j (log2 units): best of the 8 lattice-corner grid keys and of (up to 32)
// keys in the query's own cell; f0 = f of that key at q (accuracy shift of SURVEY App. D).
__device__ __forceinline__ void shift_bound(const KeysView& kv, const float4 q, float& mh, float& f0, float3& g0) {
  const int R = kv.R, NC = kv.NC;
  const int cx = cellc(q.x, kv.inv_h, NC), cy = cellc(q.y, kv.inv_h, NC), cz = cellc(q.z, kv.inv_h, NC);
  mh = INFINITY;
  f0 = 0.0f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int n = (cx + (c & 1)) + R * ((cy + ((c >> 1) & 1)) + R * (cz + (c >> 2)));
    const float4 ka = __ldg(&kv.grid_raw[2 * n]);
    const float dx = q.x - ka.x, dy = q.y - ka.y, dz = q.z - ka.z;
    const float e = ka.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    if (e < mh) {
      mh = e;
      const float4 kb = __ldg(&kv.grid_raw[2 * n + 1]);
      f0 = fmaf(kb.w, dz, fmaf(kb.z, dy, fmaf(kb.y, dx, kb.x)));
      g0 = make_float3(kb.y, kb.z, kb.w);
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
      const float4 kb = __ldg(&kv.ks[2 * k + 1]);
      f0 = fmaf(kb.w, dz, fmaf(kb.z, dy, fmaf(kb.y, dx, kb.x)));
      g0 = make_float3(kb.y, kb.z, kb.w);
    }
  }
}

__device__ __forceinline__ float exponent(const float4 q, const float4 a) {
  const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
  return a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

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
__global__ void __launch_bounds__(NTHREADS) k_forward(const FwdArgs A) {
  __shared__ float4 ws_a[NWARP][WSLICE];
  __shared__ float4 ws_b[NWARP][WSLICE];
  __shared__ int ws_id[NWARP][WSLICE];
  const KeysView& kv = A.kv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t item = blockIdx.x * NWARP + w;
  if (item >= *A.n_items) return;
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
      const float Of = O - f0[u];
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

int launch_forward(const FwdArgs& a, int want_g, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)((n_items + NWARP - 1) / NWARP);
  if (want_g) k_forward<true><<<blocks, NTHREADS, 0, s>>>(a);
  else k_forward<false><<<blocks, NTHREADS, 0, s>>>(a);
  return 1;
}

// ------------------------------------------------------------------------------ backward
// DET: deterministic mode, 64-bit fixed-point accumulation (see BwdArgs::gfix)
template <bool EIK, bool DET>
__global__ void __launch_bounds__(NTHREADS) k_backward(const BwdArgs A) {
  float fix_scale = 0.0f;
  if (DET) {
    const float um = *A.umax;
    fix_scale = um > 0.0f ? (float)(1ull << FIX_BITS) / um : 0.0f;
  }
  auto fix_add = [&](unsigned long long* p, float v) {
    const float qv = v * fix_scale;
    if (fabsf(qv) < 4.0e18f) {
      atomicAdd(p, (unsigned long long)(long long)rintf(qv));
    } else {
      atomicOr(A.fix_overflow, 1u);
    }
  };
  __shared__ float4 sq[NWARP][QW];  // x, y, z, -lambda_l
  __shared__ float4 sv[NWARP][QW];  // r, O, h.ubar, h.G
  __shared__ float4 sh[EIK ? NWARP : 1][EIK ? QW : 1];
  __shared__ float4 ka_s[NWARP][WSLICE];
  __shared__ float4 kb_s[NWARP][WSLICE];
  __shared__ int kid_s[NWARP][WSLICE];
  const KeysView& kv = A.kv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t item = blockIdx.x * NWARP + w;
  if (item >= *A.n_items) return;
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
        sh[w][j] = hv;
      }
      q.w = rc.x;
      sq[w][j] = q;
      sv[w][j] = make_float4(r, rc.z, hub, T);
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
  const float4* Q = sq[w];
  const float4* V = sv[w];
  const float4* H = sh[EIK ? w : 0];
  float4* sa = ka_s[w];
  float4* sb = kb_s[w];
  int* sid = kid_s[w];
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
    // registers (prefetched one batch ahead); no test, no staging
    const uint32_t* L = A.wl_pool + A.wl_off[item];
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t id1 = ((uint32_t)lane < wn) ? __ldg(&L[lane]) : 0u;
    float4 a1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1]) : z4;
    float4 b1 = ((uint32_t)lane < wn) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
    for (uint32_t base = 0; base < wn; base += 32) {
      const uint32_t k = base + lane;
      const bool has = k < wn;
      const uint32_t id = id1;
      const float4 a = a1, b = b1;
      if (k + 32 < wn) {
        id1 = __ldg(&L[k + 32]);
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

int launch_backward(const BwdArgs& a, int64_t n_items, cudaStream_t s) {
  if (n_items <= 0) return 0;
  const unsigned blocks = (unsigned)((n_items + NWARP - 1) / NWARP);
  if (a.eik) k_backward<true, false><<<blocks, NTHREADS, 0, s>>>(a);
  else k_backward<false, false><<<blocks, NTHREADS, 0, s>>>(a);
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
  const unsigned blocks = (unsigned)((n_items + NWARP - 1) / NWARP);
  if (a.eik) k_backward<true, true><<<blocks, NTHREADS, 0, s>>>(a);
  else k_backward<false, true><<<blocks, NTHREADS, 0, s>>>(a);
  return 2;
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

int launch_fold(float* gpad, float* grad, int n_nodes, cudaStream_t s) {
  int blocks = (n_nodes + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_fold<<<blocks, 256, 0, s>>>(gpad, grad, n_nodes);
  return 1;
}

}  // namespace ef
