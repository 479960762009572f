// k_adamw.cu — S6 AdamW (torch.optim.AdamW semantics, reading R-10) and the
// mean-shift offset initialisation.
#include "efunc_internal.cuh"

namespace ef {

// Elementwise over theta [R^3][13]; op order follows torch's single-tensor AdamW:
//   p *= 1 - lr*wd (masked channels);  m += (1-b1)(g - m);  v = v*b2 + (1-b2) g*g;
//   p += -step_size * m / (sqrt(v) / sqrt(bc2) + eps),  step_size = lr / bc1
// The step counter t lives on the device (ds->adam_t): every block derives the scalar constants
// for t + 1 in double (rounded to fp32 once), and the last block to finish stores t + 1. So a
// captured CUDA graph replays correct bias corrections.
__global__ void k_adamw(float* __restrict__ theta, const float* __restrict__ grad, float* __restrict__ m,
                        float* __restrict__ v, int64_t n, const AdamWConst hc, DevScalars* ds) {
  __shared__ AdamWScal c;
  __shared__ unsigned long long t_next;
  if (threadIdx.x == 0) {
    t_next = ds->adam_t + 1;
    c = adamw_scal(hc, t_next);
  }
  __syncthreads();
  const AdamWScal cs = c;
  const uint32_t mask = hc.decay_mask;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(i % hc.nch);
    if ((hc.frozen_mask >> ch) & 1u) continue;  // degree 0: g channels stay exactly 0
    float mi = m[i], vi = v[i];
    theta[i] = adamw_elem(theta[i], grad[i], mi, vi, (mask >> ch) & 1u, cs);
    m[i] = mi;
    v[i] = vi;
  }
  // every block has read adam_t (above) before it arrives here: the last one advances it
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ds->adam_done, 1u) == gridDim.x - 1) {
      ds->adam_t = t_next;
      ds->adam_done = 0;
    }
  }
}

// theta[n][c] = 0 for the channels in mask (degree 0: the polynomial gradients g0, g1)
__global__ void k_zero_channels(float* __restrict__ theta, int n_nodes, uint32_t mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n_nodes * EF_NCH;
       i += (int64_t)gridDim.x * blockDim.x)
    if ((mask >> (int)(i % EF_NCH)) & 1u) theta[i] = 0.0f;
}

int launch_zero_channels(float* theta, int n_nodes, uint32_t mask, cudaStream_t s) {
  if (!mask) return 0;
  int blocks = (int)(((int64_t)n_nodes * EF_NCH + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_zero_channels<<<blocks, 256, 0, s>>>(theta, n_nodes, mask);
  return 1;
}

int launch_adamw(float* theta, const float* grad, float* m, float* v, int64_t n, const AdamWConst& hc,
                 DevScalars* ds, cudaStream_t s) {
  // few fat blocks: each block derives the step constants once (a double pow on one thread)
  long blocks = (n + 255) / 256;
  if (blocks > 148 * 2) blocks = 148 * 2;
  if (blocks < 1) blocks = 1;
  k_adamw<<<(unsigned)blocks, 256, 0, s>>>(theta, grad, m, v, n, hc, ds);
  return 1;
}

// Mean shift: one thread per lattice node; surface points staged through shared memory.
// Pass 1: E_min = min_s bw ||k - s||^2 (the max shift); pass 2: weighted mean.
constexpr int MS_TILE = 1024;

__global__ void k_mean_shift(float* __restrict__ theta, int R, const float* __restrict__ surf, int64_t N,
                             float bw) {
  __shared__ float3 sp[MS_TILE];
  const int Nn = R * R * R;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = n < Nn;
  float kx = 0.f, ky = 0.f, kz = 0.f;
  if (act) {
    const int x = n % R, y = (n / R) % R, z = n / (R * R);
    kx = (float)(-1.0 + 2.0 * x / (double)(R - 1));
    ky = (float)(-1.0 + 2.0 * y / (double)(R - 1));
    kz = (float)(-1.0 + 2.0 * z / (double)(R - 1));
  }
  float emin = INFINITY;
  for (int64_t t0 = 0; t0 < N; t0 += MS_TILE) {
    const int cnt = (int)((N - t0) < (int64_t)MS_TILE ? (N - t0) : (int64_t)MS_TILE);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      sp[i] = make_float3(surf[3 * (t0 + i)], surf[3 * (t0 + i) + 1], surf[3 * (t0 + i) + 2]);
    __syncthreads();
    for (int i = 0; i < cnt; ++i) {
      const float dx = kx - sp[i].x, dy = ky - sp[i].y, dz = kz - sp[i].z;
      emin = fminf(emin, bw * fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
    }
  }
  float W = 0.f, Sx = 0.f, Sy = 0.f, Sz = 0.f;
  for (int64_t t0 = 0; t0 < N; t0 += MS_TILE) {
    const int cnt = (int)((N - t0) < (int64_t)MS_TILE ? (N - t0) : (int64_t)MS_TILE);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x)
      sp[i] = make_float3(surf[3 * (t0 + i)], surf[3 * (t0 + i) + 1], surf[3 * (t0 + i) + 2]);
    __syncthreads();
    for (int i = 0; i < cnt; ++i) {
      const float dx = kx - sp[i].x, dy = ky - sp[i].y, dz = kz - sp[i].z;
      const float e = bw * fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float w = expf(emin - e);
      W += w;
      Sx = fmaf(w, sp[i].x, Sx);
      Sy = fmaf(w, sp[i].y, Sy);
      Sz = fmaf(w, sp[i].z, Sz);
    }
  }
  if (act) {
    float* t = theta + (size_t)n * EF_NCH;
    t[5] = Sx / W - kx;
    t[6] = Sy / W - ky;
    t[7] = Sz / W - kz;
  }
}

int launch_mean_shift(float* theta, int R, const float* surf, int64_t N, float bw, cudaStream_t s) {
  const int Nn = R * R * R;
  k_mean_shift<<<(Nn + 127) / 128, 128, 0, s>>>(theta, R, surf, N, bw);
  return 1;
}

}  // namespace ef
