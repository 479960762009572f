// k_cosine.cu — cosine-series stacks (§4.4 "function
// decomposition"): S(q) = sum_{b<B} w_b(q) O_b(q), Eq. cosine-series, with the separable weights
// w_b(q) = cos(b pi x) cos(b pi y) cos(b pi z) (reading R-C). The band models O_b are an
// n_shapes = B handle (variant GRID, degree 1 = Config G-6); these kernels replicate the queries to
// the bands, combine the band values into S and its spatial gradient, and turn the MSE loss of S into
// the bands' upstreams dL/dO_b = w_b dL/dS (chain rule), in the ABI call efunc_cosine_*.
#include <algorithm>

#include "efunc_internal.cuh"

namespace ef {

__global__ void k_cos_replicate(const float* __restrict__ q, int64_t J, int B, float* __restrict__ qr) {
  const int64_t n = 3 * J;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * B; i += (int64_t)gridDim.x * blockDim.x)
    qr[i] = q[i % n];
}

__device__ __forceinline__ void cos_weight(int b, float x, float y, float z, float& w, float& wx, float& wy,
                                           float& wz) {
  float sx, cx, sy, cy, sz, cz;
  const float k = (float)b * 3.14159265358979f;
  sincosf(k * x, &sx, &cx);
  sincosf(k * y, &sy, &cy);
  sincosf(k * z, &sz, &cz);
  w = cx * cy * cz;
  wx = -k * sx * cy * cz;
  wy = -k * cx * sy * cz;
  wz = -k * cx * cy * sz;
}

__global__ void k_cos_combine(const float* __restrict__ q, int64_t J, int B, const float* __restrict__ O,
                              const float* __restrict__ G, const float* __restrict__ o, float inv_J,
                              float* __restrict__ S, float* __restrict__ GS, float* __restrict__ dL_dO) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < J; j += (int64_t)gridDim.x * blockDim.x) {
    const float x = q[3 * j], y = q[3 * j + 1], z = q[3 * j + 2];
    float s = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
    for (int b = 0; b < B; ++b) {
      float w, wx, wy, wz;
      cos_weight(b, x, y, z, w, wx, wy, wz);
      const float ob = O[(size_t)b * J + j];
      s = fmaf(w, ob, s);
      if (G) {  // dS/dq = sum_b (dw_b O_b + w_b G_b)
        const float* gb = G + 3 * ((size_t)b * J + j);
        gx = fmaf(wx, ob, fmaf(w, gb[0], gx));
        gy = fmaf(wy, ob, fmaf(w, gb[1], gy));
        gz = fmaf(wz, ob, fmaf(w, gb[2], gz));
      }
    }
    if (S) S[j] = s;
    if (GS) {
      GS[3 * j] = gx;
      GS[3 * j + 1] = gy;
      GS[3 * j + 2] = gz;
    }
    if (dL_dO) {  // Eq. loss on S, chained to the bands
      const float r = 2.0f * (s - o[j]) * inv_J;
      for (int b = 0; b < B; ++b) {
        float w, wx, wy, wz;
        cos_weight(b, x, y, z, w, wx, wy, wz);
        dL_dO[(size_t)b * J + j] = w * r;
      }
    }
  }
}

// loss = sum_j (S_j - o_j)^2 / J_global in a fixed order (one block: deterministic)
__global__ void k_cos_loss(const float* __restrict__ S, const float* __restrict__ o, int64_t J, float inv_J,
                           float* __restrict__ loss) {
  __shared__ float red[32];
  float acc = 0.f;
  for (int64_t j = threadIdx.x; j < J; j += blockDim.x) {
    const float d = S[j] - o[j];
    acc = fmaf(d * d, inv_J, acc);
  }
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(~0u, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(~0u, acc, s);
    if (threadIdx.x == 0) *loss = acc;
  }
}

static unsigned grid_of(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

int launch_cos_replicate(const float* q, int64_t J, int B, float* qr, cudaStream_t s) {
  k_cos_replicate<<<grid_of(3 * J * B), 256, 0, s>>>(q, J, B, qr);
  return 1;
}

int launch_cos_combine(const float* q, int64_t J, int B, const float* O, const float* G, const float* o, float inv_J,
                       float* S, float* GS, float* dL_dO, float* loss, cudaStream_t s) {
  if (J <= 0) return 0;
  k_cos_combine<<<grid_of(J), 256, 0, s>>>(q, J, B, O, G, o, inv_J, S, GS, dL_dO);
  if (loss) {
    k_cos_loss<<<1, 1024, 0, s>>>(S, o, J, inv_J, loss);
    return 2;
  }
  return 1;
}

}  // namespace ef
