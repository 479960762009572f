// k_bin.cu — S0 key prep and S1 binning kernels.
//
// S0 (PAPER.md:L456 parameter space, L908 beta = e^s): theta [R^3][13] -> 2R^3 key records
//    {x,y,z, beta*log2e | c, gx, gy, gz}; cell id per key; per-cell histogram; min beta
//    (k_prep_keys, or k_adamw_keys fused with the S6 AdamW update of the same pass).
// S1: queries -> (brick, sub-cell) Morton bins, histogram -> exclusive scan -> scatter (rank from
//    the histogram atomic; the stable radix sort in deterministic mode), then work items of <= 32
//    queries per brick, laid out in cost classes (heavy bricks first, Morton order within a class).
// Also the one-launch fills (k_fill_segs) that replace runs of memset nodes in the step graph.
#include "efunc_internal.cuh"

namespace ef {

__device__ __forceinline__ int cell_clamp(float p, float inv_h, int NC) {
  float c = floorf((p + 1.0f) * inv_h);
  c = fminf(fmaxf(c, 0.0f), (float)(NC - 1));
  return (int)c;
}

// ------------------------------------------------------------------------------ S0
// Also checks the brick lists' Verlet skin: a key that moved more than skin from its position at
// the last list build, or whose bl left [ref/(1+mu), ref*(1+mu)], invalidates the lists.
struct PrepOut {
  float local_min = INFINITY;
  bool moved = false, resort = false;
};

// node n's two key records from its 13 channels t (S0; see k_prep_keys)
__device__ __forceinline__ void prep_key_node(const int n, const float* t, const int R, const int banks,
                                              float4* __restrict__ key_raw, uint32_t* __restrict__ key_cell,
                                              uint32_t* __restrict__ key_rank, uint32_t* __restrict__ cell_count,
                                              const float4* __restrict__ key_ref, const float skin2, const float mu,
                                              PrepOut& po) {
  const int N = R * R * R;
  const int NC = R - 1;
  const float inv_h = (float)((R - 1) / 2.0);
  const int x = n % R, y = (n / R) % R, z = n / (R * R);
  // lattice k(i) = float32(-1 + 2 i/(R-1))  (reading R-2), evaluated in double
  const float kx = (float)(-1.0 + 2.0 * x / (double)(R - 1));
  const float ky = (float)(-1.0 + 2.0 * y / (double)(R - 1));
  const float kz = (float)(-1.0 + 2.0 * z / (double)(R - 1));
  const float bl0 = expf(t[0]) * EF_LOG2E;
  const float bl1 = expf(t[8]) * EF_LOG2E;
  const bool on0 = banks & 1, on1 = banks & 2;
  // a bank the variant does not have (NEXT-4: O only / O^Delta only): its keys sit far away
  // (weight exactly 0) in the sentinel cell n_cells that no enumeration visits
  constexpr float FAR = 1e15f;
  const float px = on1 ? kx + t[5] : FAR, py = on1 ? ky + t[6] : FAR, pz = on1 ? kz + t[7] : FAR;
  const float gx = on0 ? kx : FAR, gy = on0 ? ky : FAR, gz = on0 ? kz : FAR;
  key_raw[2 * n] = make_float4(gx, gy, gz, bl0);
  key_raw[2 * n + 1] = make_float4(t[1], t[2], t[3], t[4]);
  key_raw[2 * (N + n)] = make_float4(px, py, pz, bl1);
  key_raw[2 * (N + n) + 1] = make_float4(t[9], t[10], t[11], t[12]);
  const uint32_t nc3 = (uint32_t)(NC * NC * NC);
  const uint32_t c0 = on0 ? (uint32_t)((cell_clamp(kz, inv_h, NC) * NC + cell_clamp(ky, inv_h, NC)) * NC +
                                       cell_clamp(kx, inv_h, NC))
                          : nc3;
  const uint32_t c1 = on1 ? (uint32_t)((cell_clamp(pz, inv_h, NC) * NC + cell_clamp(py, inv_h, NC)) * NC +
                                       cell_clamp(px, inv_h, NC))
                          : nc3;
  po.resort |= key_cell[N + n] != c1;  // grid-bank cells never change
  key_cell[n] = c0;
  key_cell[N + n] = c1;
  const uint32_t rk0 = atomicAdd(&cell_count[c0], 1u), rk1 = atomicAdd(&cell_count[c1], 1u);
  if (key_rank) {  // positions inside the cells for the ranked scatter (non-deterministic mode)
    key_rank[n] = rk0;
    key_rank[N + n] = rk1;
  }
  po.local_min = fminf(po.local_min, fminf(on0 ? bl0 : INFINITY, on1 ? bl1 : INFINITY));
  const float4 r0 = key_ref[n], r1 = key_ref[N + n];
  const float ex = px - r1.x, ey = py - r1.y, ez = pz - r1.z;
  if (on1) {
    po.moved |= fmaf(ex, ex, fmaf(ey, ey, ez * ez)) > skin2;
    po.moved |= !(bl1 <= r1.w * (1.0f + mu) && bl1 * (1.0f + mu) >= r1.w);
  }
  if (on0) po.moved |= !(bl0 <= r0.w * (1.0f + mu) && bl0 * (1.0f + mu) >= r0.w);
}

__device__ __forceinline__ void prep_key_flush(const PrepOut& po, DevScalars* ds) {
  float local_min = po.local_min;
  // bl > 0: the IEEE bit pattern orders like the value
  for (int o = 16; o > 0; o >>= 1) local_min = fminf(local_min, __shfl_xor_sync(~0u, local_min, o));
  if ((threadIdx.x & 31) == 0 && local_min < INFINITY)
    atomicMin(reinterpret_cast<unsigned int*>(&ds->bl_min), __float_as_uint(local_min));
  if (__any_sync(~0u, po.moved) && (threadIdx.x & 31) == 0) atomicOr(&ds->lists_invalid, 1u);
  if (__any_sync(~0u, po.resort) && (threadIdx.x & 31) == 0) atomicOr(&ds->keys_resort, 1u);
}

__global__ void k_prep_keys(const float* __restrict__ theta, int R, int banks, float4* __restrict__ key_raw,
                            uint32_t* __restrict__ key_cell, uint32_t* __restrict__ key_rank,
                            uint32_t* __restrict__ cell_count,
                            const float4* __restrict__ key_ref, float skin2, float mu, DevScalars* ds) {
  const int N = R * R * R;
  PrepOut po;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    float t[EF_NCH];
#pragma unroll
    for (int c = 0; c < EF_NCH; ++c) t[c] = theta[(size_t)n * EF_NCH + c];
    prep_key_node(n, t, R, banks, key_raw, key_cell, key_rank, cell_count, key_ref, skin2, mu, po);
  }
  prep_key_flush(po, ds);
}

// S6 + S0 fused (13-channel layout): a block takes a tile of AK_NODES nodes; its threads run AdamW
// over the tile's AK_NODES x 13 elements in element order (coalesced; adamw_elem: the op order of
// k_adamw) and stage the updated theta in shared memory, then one thread per node writes the
// node's key records (prep_key_node). The step counter advances as in k_adamw (the last block).
constexpr int AK_NODES = 64, AK_THREADS = 128;
__global__ void __launch_bounds__(AK_THREADS) k_adamw_keys(float* __restrict__ theta, const float* __restrict__ grad,
                                                           float* __restrict__ m, float* __restrict__ v,
                                                           const AdamWConst hc, int R, int banks,
                                                           float4* __restrict__ key_raw, uint32_t* __restrict__ key_cell,
                                                           uint32_t* __restrict__ key_rank, uint32_t* __restrict__ cell_count,
                                                           const float4* __restrict__ key_ref, float skin2, float mu,
                                                           DevScalars* ds) {
  __shared__ AdamWScal c;
  __shared__ unsigned long long t_next;
  __shared__ float tile[AK_NODES * EF_NCH];
  if (threadIdx.x == 0) {
    t_next = ds->adam_t + 1;
    c = adamw_scal(hc, t_next);
  }
  __syncthreads();
  const AdamWScal cs = c;
  const int N = R * R * R;
  PrepOut po;
  for (int n0 = blockIdx.x * AK_NODES; n0 < N; n0 += gridDim.x * AK_NODES) {
    const int nn = min(AK_NODES, N - n0);
    const size_t e0 = (size_t)n0 * EF_NCH;
    for (int i = threadIdx.x; i < nn * EF_NCH; i += AK_THREADS) {
      const int ch = i % EF_NCH;
      float p = theta[e0 + i];
      if (!((hc.frozen_mask >> ch) & 1u)) {  // degree 0: g channels stay exactly 0
        float mi = m[e0 + i], vi = v[e0 + i];
        p = adamw_elem(p, grad[e0 + i], mi, vi, (hc.decay_mask >> ch) & 1u, cs);
        theta[e0 + i] = p;
        m[e0 + i] = mi;
        v[e0 + i] = vi;
      }
      tile[i] = p;
    }
    __syncthreads();
    if (threadIdx.x < nn)
      prep_key_node(n0 + threadIdx.x, &tile[threadIdx.x * EF_NCH], R, banks, key_raw, key_cell, key_rank, cell_count,
                    key_ref, skin2, mu, po);
    __syncthreads();
  }
  prep_key_flush(po, ds);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ds->adam_done, 1u) == gridDim.x - 1) {
      ds->adam_t = t_next;
      ds->adam_done = 0;
    }
  }
}

int launch_adamw_keys(float* theta, const float* grad, float* m, float* v, const AdamWConst& hc, int R, int banks,
                      float4* key_raw, uint32_t* key_cell, uint32_t* key_rank, uint32_t* cell_count,
                      const float4* key_ref, float skin2, float mu, DevScalars* ds, cudaStream_t s) {
  const int N = R * R * R;
  int blocks = (N + AK_NODES - 1) / AK_NODES;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_adamw_keys<<<blocks, AK_THREADS, 0, s>>>(theta, grad, m, v, hc, R, banks, key_raw, key_cell, key_rank, cell_count,
                                     key_ref, skin2, mu, ds);
  return 1;
}

int launch_prep_keys(const float* theta, int R, int banks, float4* key_raw, uint32_t* key_cell, uint32_t* key_rank,
                     uint32_t* cell_count,
                     const float4* key_ref, float skin2, float mu, DevScalars* ds, cudaStream_t s) {
  const int N = R * R * R;
  int blocks = (N + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prep_keys<<<blocks, 256, 0, s>>>(theta, R, banks, key_raw, key_cell, key_rank, cell_count, key_ref, skin2, mu,
                                     ds);
  return 1;
}

// After a list rebuild: remember every key's position and bl (the skin reference).
// Also closes the build's counters (pool cursor, overflow count) for the next build.
__global__ void k_list_snapshot(const float4* __restrict__ key_raw, float4* __restrict__ key_ref, int n_keys,
                                DevScalars* ds) {
  if (!ds->lists_invalid) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ds->pool_used = ds->pool_top;
    ds->pool_top = 0;
    ds->ovf_last = ds->ovf_count;
    ds->ovf_count = 0;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_keys; i += gridDim.x * blockDim.x)
    key_ref[i] = key_raw[2 * i];
}

int launch_list_snapshot(const float4* key_raw, float4* key_ref, int n_keys, DevScalars* ds,
                         cudaStream_t s) {
  int blocks = (n_keys + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_list_snapshot<<<blocks, 256, 0, s>>>(key_raw, key_ref, n_keys, ds);
  return 1;
}

// ------------------------------------------------------------------------------ scan
constexpr int SCAN_T = 1024;
constexpr int SCAN_PER = 4;
constexpr int SCAN_TILE = SCAN_T * SCAN_PER;

__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t v, uint32_t* s_w, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(~0u, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t x = s_w[lane];
    uint32_t xi = x;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(~0u, xi, o);
      if (lane >= o) xi += t;
    }
    s_w[lane] = xi - x;
    if (lane == 31) s_w[32] = xi;
  }
  __syncthreads();
  *total = s_w[32];
  return incl - v + s_w[w];
}

// gate (nullable): the kernels of a scan / counting sort do nothing when *gate == 0
#define GATED if (gate && *gate == 0u) return

__global__ void k_scan_tiles(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t n,
                             uint32_t* __restrict__ tile_sums, const uint32_t* gate) {
  GATED;
  __shared__ uint32_t s_w[33];
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER;
  uint32_t v[SCAN_PER];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0u;
    sum += v[i];
  }
  uint32_t total;
  uint32_t off = block_excl_scan_1024(sum, s_w, &total);
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i) {
    if (base + i < n) out[base + i] = off;
    off += v[i];
  }
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_tile_sums(uint32_t* __restrict__ tile_sums, uint32_t nt, const uint32_t* gate) {
  GATED;
  __shared__ uint32_t s_w[33];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nt; b0 += SCAN_TILE) {
    const uint32_t base = b0 + threadIdx.x * SCAN_PER;
    uint32_t v[SCAN_PER];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_PER; ++i) {
      v[i] = (base + i < nt) ? tile_sums[base + i] : 0u;
      sum += v[i];
    }
    uint32_t total;
    uint32_t off = block_excl_scan_1024(sum, s_w, &total) + carry;
#pragma unroll
    for (int i = 0; i < SCAN_PER; ++i) {
      if (base + i < nt) tile_sums[base + i] = off;
      off += v[i];
    }
    carry += total;
    __syncthreads();
  }
}

__global__ void k_scan_add(uint32_t* __restrict__ out, uint32_t n, const uint32_t* __restrict__ tile_sums,
                           const uint32_t* gate) {
  GATED;
  const uint32_t add = tile_sums[blockIdx.x];
  const uint32_t base = blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER;
#pragma unroll
  for (int i = 0; i < SCAN_PER; ++i)
    if (base + i < n) out[base + i] += add;
}

int launch_scan_u32(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* block_tmp, cudaStream_t s,
                    const uint32_t* gate) {
  const uint32_t nt = (n + SCAN_TILE - 1) / SCAN_TILE;
  k_scan_tiles<<<nt, SCAN_T, 0, s>>>(in, out, n, block_tmp, gate);
  if (nt > 1) {
    k_scan_tile_sums<<<1, SCAN_T, 0, s>>>(block_tmp, nt, gate);
    k_scan_add<<<nt, SCAN_T, 0, s>>>(out, n, block_tmp, gate);
    return 3;
  }
  return 1;
}

// ------------------------------------------------------------------------------ counting sort
__global__ void k_scatter(const uint32_t* __restrict__ bin, uint32_t n, const uint32_t* __restrict__ bin_start,
                          uint32_t* __restrict__ fill, uint32_t* __restrict__ tmp_idx, const uint32_t* gate) {
  GATED;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t b = bin[i];
    tmp_idx[bin_start[b] + atomicAdd(&fill[b], 1u)] = i;
  }
}

// ---- stable sort by bin: LSD radix sort, 8-bit digits (deterministic, O(n) per pass)
// Pass p orders the elements by digit p of their bin, stably: a tile's elements keep their input
// order inside each digit (ranks from __match_any_sync within a warp and per-warp digit counts in
// shared memory, chunk by chunk in index order). After ceil(bits/8) passes the elements are sorted
// by bin and, inside a bin, by their original index: the order does not depend on scheduling.
constexpr int RX_T = 256, RX_CHUNKS = 16, RX_TILE = RX_T * RX_CHUNKS, RX_W = RX_T / 32;

__global__ void __launch_bounds__(RX_T) k_radix_hist(const uint32_t* __restrict__ key, uint32_t n, int shift,
                                                      uint32_t* __restrict__ hist, uint32_t ntiles,
                                                      const uint32_t* gate) {
  GATED;
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * RX_TILE;
  for (int c = 0; c < RX_CHUNKS; ++c) {
    const uint32_t e = base + c * RX_T + threadIdx.x;
    if (e < n) atomicAdd(&h[(key[e] >> shift) & 255u], 1u);  // counts: order-independent
  }
  __syncthreads();
  hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];  // digit-major: one scan gives offsets
}

__global__ void __launch_bounds__(RX_T) k_radix_scatter(const uint32_t* __restrict__ key, const uint32_t* __restrict__ val,
                                                         uint32_t n, int shift, const uint32_t* __restrict__ off,
                                                         uint32_t ntiles, uint32_t* __restrict__ key_out,
                                                         uint32_t* __restrict__ val_out, const uint32_t* gate) {
  GATED;
  __shared__ uint32_t run[256];
  __shared__ uint32_t wc[RX_W][256];
  const int w = threadIdx.x >> 5;
  run[threadIdx.x] = off[threadIdx.x * ntiles + blockIdx.x];
#pragma unroll
  for (int k = 0; k < RX_W; ++k) wc[k][threadIdx.x] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * RX_TILE;
  for (int c = 0; c < RX_CHUNKS; ++c) {
    const uint32_t e = base + c * RX_T + threadIdx.x;
    const bool valid = e < n;
    const uint32_t k = valid ? key[e] : 0u;
    const uint32_t v = valid ? (val ? val[e] : e) : 0u;
    const uint32_t d = valid ? ((k >> shift) & 255u) : 256u;
    const uint32_t peers = __match_any_sync(~0u, d);
    const uint32_t rank = __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
    if (valid && rank == 0) wc[w][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pre = run[d] + rank;
      for (int k2 = 0; k2 < w; ++k2) pre += wc[k2][d];
      if (key_out) key_out[pre] = k;
      val_out[pre] = v;
    }
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int k2 = 0; k2 < RX_W; ++k2) {
      add += wc[k2][threadIdx.x];
      wc[k2][threadIdx.x] = 0;
    }
    run[threadIdx.x] += add;
    __syncthreads();
  }
}

static int grid_for(uint32_t n, int threads) {
  long b = ((long)n + threads - 1) / threads;
  if (b > 148L * 32) b = 148L * 32;
  if (b < 1) b = 1;
  return (int)b;
}

size_t radix_hist_elems(uint32_t n) { return (size_t)256 * ((n + RX_TILE - 1) / RX_TILE); }

// Stable sort of the indices 0..n-1 by bin[i] < 2^bits into out_idx. rk: 2n u32 key scratch,
// tmp_idx: n u32 value scratch, hist: radix_hist_elems(n) u32, scan_tmp: the scan's tile sums.
int launch_stable_sort(const uint32_t* bin, uint32_t n, int bits, uint32_t* rk, uint32_t* hist, uint32_t* scan_tmp,
                       uint32_t* tmp_idx, uint32_t* out_idx, cudaStream_t s, const uint32_t* gate) {
  if (n == 0) return 0;
  const uint32_t ntiles = (n + RX_TILE - 1) / RX_TILE;
  const int passes = bits <= 8 ? 1 : (bits + 7) / 8;
  int launches = 0;
  const uint32_t* kin = bin;
  const uint32_t* vin = nullptr;  // identity on the first pass
  for (int p = 0; p < passes; ++p) {
    const bool last = p == passes - 1;
    // ping-pong so that the last pass lands in out_idx
    uint32_t* vout = last ? out_idx : (((passes - 1 - p) & 1) ? tmp_idx : out_idx);
    uint32_t* kout = last ? nullptr : rk + (size_t)(p & 1) * n;
    k_radix_hist<<<ntiles, RX_T, 0, s>>>(kin, n, 8 * p, hist, ntiles, gate);
    launches += 1 + launch_scan_u32(hist, hist, 256u * ntiles, scan_tmp, s, gate);
    k_radix_scatter<<<ntiles, RX_T, 0, s>>>(kin, vin, n, 8 * p, hist, ntiles, kout, vout, gate);
    ++launches;
    kin = kout;
    vin = vout;
  }
  return launches;
}

// The counting sort without the stable rank (bin order only; within a bin, atomics' order).
int launch_scatter_only(const uint32_t* bin, uint32_t n, const uint32_t* bin_start, uint32_t* fill,
                        uint32_t* out_idx, cudaStream_t s, const uint32_t* gate) {
  if (n == 0) return 0;
  k_scatter<<<grid_for(n, 256), 256, 0, s>>>(bin, n, bin_start, fill, out_idx, gate);
  return 1;
}

__global__ void k_gather_keys(const uint32_t* __restrict__ order, const float4* __restrict__ key_raw,
                              float4* __restrict__ key_sorted, int* __restrict__ kid, uint32_t n) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint32_t i = order[p];
    key_sorted[2 * p] = key_raw[2 * i];
    key_sorted[2 * p + 1] = key_raw[2 * i + 1];
    kid[p] = (int)i;
  }
}

int launch_gather_keys(const uint32_t* order, const float4* key_raw, float4* key_sorted, int* kid,
                        uint32_t n, cudaStream_t s) {
  k_gather_keys<<<grid_for(n, 256), 256, 0, s>>>(order, key_raw, key_sorted, kid, n);
  return 1;
}

// ------------------------------------------------------------------------------ query bins
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every 3rd bit
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

// Bin = Morton code of the query's brick (B^3 lattice cells); queries outside [-1,1]^3 (or
// non-finite) go to the last bin, whose items enumerate keys directly instead of a brick list.
__global__ void k_query_bins(const float* __restrict__ q, const float* __restrict__ o, int64_t J, BrickGeom bg,
                             int NC, float inv_h, uint32_t* __restrict__ bins, uint32_t* __restrict__ count,
                             uint32_t* __restrict__ rank, DevScalars* ds) {
  const uint32_t outside = bg.n_codes * bg.qsub;
  const float sub_scale = (float)bg.sdiv * inv_h;  // sub-cells (half or quarter cells)
  const int ns = bg.sdiv * bg.B;
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
    const float x = q[3 * j], y = q[3 * j + 1], z = q[3 * j + 2];
    bool fin = isfinite(x) && isfinite(y) && isfinite(z);
    if (o) fin = fin && isfinite(o[j]);
    bad |= !fin;
    uint32_t b = outside;
    if (fin && fabsf(x) <= 1.0f && fabsf(y) <= 1.0f && fabsf(z) <= 1.0f) {
      const int bx = cell_clamp(x, inv_h, NC) / bg.B;
      const int by = cell_clamp(y, inv_h, NC) / bg.B;
      const int bz = cell_clamp(z, inv_h, NC) / bg.B;
      // sub-cell of the query inside its brick (Morton order): a brick's sub-bins stay contiguous
      const int sx = min(max((int)floorf((x + 1.0f) * sub_scale) - ns * bx, 0), ns - 1);
      const int sy = min(max((int)floorf((y + 1.0f) * sub_scale) - ns * by, 0), ns - 1);
      const int sz = min(max((int)floorf((z + 1.0f) * sub_scale) - ns * bz, 0), ns - 1);
      b = (spread3(bx) | (spread3(by) << 1) | (spread3(bz) << 2)) * bg.qsub +
          (spread3(sx) | (spread3(sy) << 1) | (spread3(sz) << 2));
    }
    bins[j] = b;
    const uint32_t r = atomicAdd(&count[b], 1u);
    if (rank) rank[j] = r;  // position inside the bin (any order is valid outside deterministic mode)
  }
  if (__any_sync(~0u, bad) && (threadIdx.x & 31) == 0) atomicOr(&ds->nonfinite, 1u);
}

int launch_query_bins(const float* q, const float* o, int64_t J, const BrickGeom& bg, int NC, float inv_h,
                      uint32_t* bins, uint32_t* count, uint32_t* rank, DevScalars* ds, cudaStream_t s) {
  if (J == 0) return 0;
  k_query_bins<<<grid_for((uint32_t)J, 256), 256, 0, s>>>(q, o, J, bg, NC, inv_h, bins, count, rank, ds);
  return 1;
}

__global__ void k_scatter_ranked(const uint32_t* __restrict__ bin, const uint32_t* __restrict__ rank, uint32_t n,
                                 const uint32_t* __restrict__ bin_start, uint32_t* __restrict__ out_idx,
                                 const uint32_t* gate) {
  GATED;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out_idx[bin_start[bin[i]] + rank[i]] = i;
}

int launch_scatter_ranked(const uint32_t* bin, const uint32_t* rank, uint32_t n, const uint32_t* bin_start,
                          uint32_t* out_idx, cudaStream_t s, const uint32_t* gate) {
  if (n == 0) return 0;
  k_scatter_ranked<<<grid_for(n, 256), 256, 0, s>>>(bin, rank, n, bin_start, out_idx, gate);
  return 1;
}

__global__ void k_gather_queries(const uint32_t* __restrict__ order, const float* __restrict__ q,
                                 const float* __restrict__ o, int64_t J, float4* __restrict__ qs,
                                 int* __restrict__ perm) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < J; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = order[p];
    qs[p] = make_float4(q[3 * (size_t)j], q[3 * (size_t)j + 1], q[3 * (size_t)j + 2], o ? o[j] : 0.0f);
    perm[p] = (int)j;
  }
}

int launch_gather_queries(const uint32_t* order, const float* q, const float* o, int64_t J, float4* qs,
                           int* perm, cudaStream_t s) {
  if (J == 0) return 0;
  k_gather_queries<<<grid_for((uint32_t)J, 256), 256, 0, s>>>(order, q, o, J, qs, perm);
  return 1;
}

// ------------------------------------------------------------------------------ misc
__global__ void k_fill_zero(float* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.0f;
}

int launch_fill_zero_f32(float* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  k_fill_zero<<<grid_for((uint32_t)n, 256), 256, 0, s>>>(p, n);
  return 1;
}

// Several u32 fills in one launch (replaces a run of cudaMemsetAsync calls: a memset node costs a
// few microseconds of graph-node gap each, a kernel node ~0.3 us)
__global__ void k_fill_segs(const FillSegs f) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
#pragma unroll
  for (int i = 0; i < FillSegs::MAX; ++i) {
    if (i >= f.k) break;
    const FillSeg g = f.s[i];
    for (uint32_t j = t; j < g.n; j += stride) g.p[j] = g.v;
  }
}

int launch_fill_segs(const FillSegs& f, cudaStream_t s) {
  uint32_t mx = 0;
  for (int i = 0; i < f.k; ++i) mx = mx > f.s[i].n ? mx : f.s[i].n;
  if (mx == 0) return 0;
  uint32_t blocks = (mx + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  k_fill_segs<<<blocks, 256, 0, s>>>(f);
  return 1;
}

// ------------------------------------------------------------------------------ work items
// A work item is a balanced run of <= QW queries of one brick (its qsub half-cell bins are
// contiguous in the sorted stream): ceil(n/QW) items per brick. The brick field is the brick's
// Morton code, or -1 for the out-of-domain bin (index nb = number of bricks).
__device__ __forceinline__ void brick_range(const uint32_t* bin_start, uint32_t c, uint32_t nb, uint32_t qsub,
                                            uint32_t& s, uint32_t& n) {
  s = bin_start[c * qsub];
  const uint32_t e = (c == nb) ? bin_start[nb * qsub + 1] : bin_start[(c + 1) * qsub];
  n = e - s;
}

// Work items in EF_ITEM_CLASSES cost classes, in one exclusive scan: slot k (nb + 1) + c holds brick
// c's item count if the brick is in class k, else 0; slot K (nb + 1) = 0 (-> the item count).
// Class 0: the brick list is longer than the average (or overflowed, or the out-of-domain bin);
// class k < K - 1: longer than 2^-k of the average; the last class: the rest. Heavy items come
// first and the lightest (volume) items last, each class in Morton order, so the persistent
// kernels' tail is made of short items (bl_n = null: everything in class 0).
__device__ __forceinline__ uint32_t item_class(const uint32_t* bl_n, const DevScalars* ds, uint32_t c, uint32_t nb) {
  if (!bl_n || c == nb) return 0;
  const uint32_t l = bl_n[c];
  if (l == BL_OVERFLOW) return 0;
  const float r = (float)l * (float)nb / fmaxf((float)ds->pool_used, 1.0f);  // list length / average
  uint32_t k = 0;
  float t = 1.0f;
  while (k + 1 < (uint32_t)EF_ITEM_CLASSES && !(r > t)) {
    ++k;
    t *= 0.5f;
  }
  return k;
}

__global__ void k_items_count(const uint32_t* __restrict__ bin_start, uint32_t nb, uint32_t qsub,
                              const uint32_t* __restrict__ bl_n, const DevScalars* ds, uint32_t* __restrict__ cnt) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= nb + 1; c += gridDim.x * blockDim.x) {
    if (c == nb + 1) {
      cnt[ITEMS_N_AT(nb)] = 0;
      continue;
    }
    uint32_t s, n;
    brick_range(bin_start, c, nb, qsub, s, n);
    const uint32_t m = (n + IQ - 1) / IQ;
    const uint32_t k = item_class(bl_n, ds, c, nb);
    for (uint32_t j = 0; j < (uint32_t)EF_ITEM_CLASSES; ++j) cnt[j * (nb + 1) + c] = j == k ? m : 0u;
  }
}

__global__ void k_items_write(const uint32_t* __restrict__ bin_start, uint32_t nb, uint32_t qsub,
                              const uint32_t* __restrict__ bl_n, const DevScalars* ds,
                              const uint32_t* __restrict__ off, int4* __restrict__ items) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= nb; c += gridDim.x * blockDim.x) {
    uint32_t s, n;
    brick_range(bin_start, c, nb, qsub, s, n);
    if (n == 0) continue;
    const uint32_t m = (n + IQ - 1) / IQ;
    const uint32_t o = off[item_class(bl_n, ds, c, nb) * (nb + 1) + c];
    const int brick = (c == nb) ? -1 : (int)c;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t a = (uint32_t)(((uint64_t)i * n) / m), b = (uint32_t)(((uint64_t)(i + 1) * n) / m);
      items[o + i] = make_int4((int)(s + a), (int)(b - a), brick, 0);
    }
  }
}

// count + exclusive scan + write of the work items in one single-CTA pass (small brick counts):
// three launches and a three-kernel scan become one
__global__ void __launch_bounds__(1024) k_items_fused(const uint32_t* __restrict__ bin_start, uint32_t nb,
                                                     uint32_t qsub, uint32_t* __restrict__ item_off,
                                                     int4* __restrict__ items) {
  __shared__ uint32_t s_w[33];
  uint32_t carry = 0;
  for (uint32_t c0 = 0; c0 <= nb + 1; c0 += 1024) {
    const uint32_t c = c0 + threadIdx.x;
    uint32_t st = 0, n = 0, m = 0;
    if (c <= nb) {
      brick_range(bin_start, c, nb, qsub, st, n);
      m = (n + IQ - 1) / IQ;
    }
    uint32_t total;
    const uint32_t off = block_excl_scan_1024(m, s_w, &total) + carry;
    if (c <= nb + 1) item_off[c] = off;
    if (c == nb + 1) item_off[ITEMS_N_AT(nb)] = off;  // the number of items
    const int brick = (c == nb) ? -1 : (int)c;
    for (uint32_t i = 0; i < m; ++i) {
      const uint32_t a = (uint32_t)(((uint64_t)i * n) / m), b = (uint32_t)(((uint64_t)(i + 1) * n) / m);
      items[off + i] = make_int4((int)(st + a), (int)(b - a), brick, 0);
    }
    carry += total;
    __syncthreads();
  }
}

int launch_items_fused(const uint32_t* bin_start, uint32_t nb, uint32_t qsub, uint32_t* item_off, int4* items,
                       cudaStream_t s) {
  k_items_fused<<<1, 1024, 0, s>>>(bin_start, nb, qsub, item_off, items);
  return 1;
}

int launch_items_count(const uint32_t* bin_start, uint32_t nb, uint32_t qsub, const uint32_t* bl_n,
                       const DevScalars* ds, uint32_t* cnt, cudaStream_t s) {
  k_items_count<<<grid_for(nb + 2, 256), 256, 0, s>>>(bin_start, nb, qsub, bl_n, ds, cnt);
  return 1;
}

int launch_items_write(const uint32_t* bin_start, uint32_t nb, uint32_t qsub, const uint32_t* bl_n,
                       const DevScalars* ds, const uint32_t* off, int4* items, cudaStream_t s) {
  k_items_write<<<grid_for(nb + 1, 128), 128, 0, s>>>(bin_start, nb, qsub, bl_n, ds, off, items);
  return 1;
}

// Fixed-order sum of per-item loss partials (deterministic).
__global__ void k_sum_partials(const float* __restrict__ part, const uint32_t* __restrict__ np, int mult,
                               float* __restrict__ out) {
  __shared__ double s[1024];
  const uint32_t n = *np * (uint32_t)mult;
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) acc += (double)part[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (float)s[0];
}

int launch_sum_partials(const float* part, const uint32_t* n, int mult, float* out, cudaStream_t s) {
  k_sum_partials<<<1, 1024, 0, s>>>(part, n, mult, out);
  return 1;
}

}  // namespace ef
