// k_common.cuh — device helpers shared by the forward, backward and list kernels: base-2
// exponentials, the warp-level AABB/threshold test, candidate enumeration over the sorted key
// grid, the brick-list stream, and the per-query shift bound.
#pragma once
#include "efunc_internal.cuh"

namespace ef {

constexpr int WSLICE = 64;  // staged keys per warp

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One key record (2 float4, 32-byte aligned) in one 256-bit read-only load (sm_100: LDG.256).
__device__ __forceinline__ void ld_rec(const float4* rec, float4& a, float4& b) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(rec));
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
template <bool LOAD_B = true, class Stage>
__device__ __forceinline__ void candidates(const KeysView& kv, int brick, const Box& box, Stage&& stage) {
  uint32_t n = BL_OVERFLOW;
  if (brick >= 0) n = __ldg(&kv.bl_n[brick]);
  if (n == BL_OVERFLOW) {
    enumerate(kv, box, [&](bool pass, uint32_t kp, float4 a) {
      const float4 b = (LOAD_B && pass) ? __ldg(&kv.ks[2 * kp + 1]) : make_float4(0.f, 0.f, 0.f, 0.f);
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
  float4 b1 = (LOAD_B && lane < n) ? __ldg(&kv.grid_raw[2 * id1 + 1]) : z4;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t k = base + lane;
    const uint32_t id = id1;
    const float4 a = a1, b = b1;
    // prefetch
    id1 = id2;
    id2 = (k + 64 < n) ? __ldg(&L[k + 64]) : 0u;
    if (k + 32 < n) {
      a1 = __ldg(&kv.grid_raw[2 * id1]);
      if (LOAD_B) b1 = __ldg(&kv.grid_raw[2 * id1 + 1]);
    }
    const bool pass = (k < n) && within(a, box);
    stage(pass, id, a, b);
  }
}

// Test-only stream of a brick list (n != BL_OVERFLOW) in chunks of U batches of 32: the U record
// gathers of a chunk are in flight together and the next chunk's ids load during this chunk's
// tests, so a chunk costs about one L2 round trip instead of one per batch. stage(pass, id) is
// called once per batch (warp-uniform).
template <int U, class Stage>
__device__ __forceinline__ void stream_list(const KeysView& kv, const uint32_t* L, const uint32_t n, const Box& box,
                                            Stage&& stage) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t idn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) idn[u] = (32u * u + lane < n) ? __ldg(&L[32u * u + lane]) : 0u;
  for (uint32_t base = 0; base < n; base += 32u * U) {
    uint32_t id[U];
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      id[u] = idn[u];
      a[u] = (base + 32u * u + lane < n) ? __ldg(&kv.grid_raw[2 * id[u]]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t k = base + 32u * (U + u) + lane;
      idn[u] = (k < n) ? __ldg(&L[k]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + 32u * u < n) stage((base + 32u * u + lane < n) && within(a[u], box), id[u]);
    }
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

// Persistent-kernel work fetch (warp-uniform): the next item in index order (Morton order keeps
// the co-resident warps of an SM on neighbouring items, which share key records in L1/L2), or
// -1 when all are taken. With a list, the g-th item is list[g] of *list_n.
__device__ __forceinline__ int64_t fetch_item(uint32_t* next, const uint32_t* n_items, const uint32_t* list,
                                              const uint32_t* list_n) {
  uint32_t g = 0;
  if ((threadIdx.x & 31) == 0) g = atomicAdd(next, 1u);
  g = __shfl_sync(~0u, g, 0);
  if (list) return g < __ldcg(list_n) ? (int64_t)__ldcg(&list[g]) : -1;
  return g < *n_items ? (int64_t)g : -1;
}

__device__ __forceinline__ float exponent(const float4 q, const float4 a) {
  const float dx = q.x - a.x, dy = q.y - a.y, dz = q.z - a.z;
  return a.w * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}

}  // namespace ef
