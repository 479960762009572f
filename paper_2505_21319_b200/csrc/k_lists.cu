// k_lists.cu — S1 brick candidate lists: per brick of B^3 lattice cells, the ids of
// every key that can reach a query inside the brick within the certified cutoff (DESIGN.md
// reading R-1), with a Verlet skin so the lists survive several AdamW steps.
#include "k_common.cuh"

namespace ef {

// Per brick (one warp each): every key that can reach some query inside the brick. A query in
// cell c has mh <= bl_max(c's corners) * 3h^2/4 (its nearest corner is within sqrt(3) h / 2),
// so thr_brick = bl_max(brick nodes) * 3h^2/4 + T_l bounds every warp threshold of the step.
constexpr int KB_WARPS = 2;
__global__ void __launch_bounds__(32 * KB_WARPS) k_brick_lists(const KeysView kv, const BrickGeom bg, float T_l,
                                                          uint32_t* __restrict__ pool, uint32_t pool_cap,
                                                          uint32_t* __restrict__ off, uint32_t* __restrict__ nout,
                                                          DevScalars* ds, uint32_t* __restrict__ scratch) {
  __shared__ uint8_t own[KB_WARPS][OWN_CAP];
  __shared__ uint32_t rs[KB_WARPS][32], ro[KB_WARPS][32];
  // the warp's staging area: a slot of the handle's per-warp scratch (shared with k_fit, which
  // never runs concurrently), BL_CAP ids, L2-resident
  const uint32_t gw = blockIdx.x * KB_WARPS + (threadIdx.x >> 5);  // two warps per scratch slot
  uint32_t* const stw = scratch + (size_t)(gw >> 1) * SCRATCH_STRIDE + (gw & 1) * SCRATCH_HALF;
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
      if (slot < (uint32_t)BL_CAP) stw[slot] = (uint32_t)__ldg(&kv.kid[kp]);  // key id
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
  for (uint32_t i = lane; i < cnt; i += 32) pool[base + i] = stw[i];
  if (lane == 0) {
    off[code] = base;
    nout[code] = cnt;
  }
  __syncwarp();
  }
}

int launch_brick_lists(const KeysView& kv, const BrickGeom& bg, float T_l, uint32_t* pool, uint32_t pool_cap,
                       uint32_t* off, uint32_t* n, DevScalars* ds, uint32_t* scratch, cudaStream_t s) {
  uint32_t blocks = (bg.n_codes + KB_WARPS - 1) / KB_WARPS;
  const uint32_t cap = (uint32_t)(2 * SCRATCH_WARPS / KB_WARPS);  // two warps per scratch slot
  if (blocks > cap) blocks = cap;
  k_brick_lists<<<blocks, 32 * KB_WARPS, 0, s>>>(kv, bg, T_l, pool, pool_cap, off, n, ds, scratch);
  return 1;
}

}  // namespace ef
