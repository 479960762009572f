// Warp-level tensor-core (mma.sync -> HMMA) throughput on sm_100a, alone and mixed with the
// MUFU.EX2 / FFMA2 work of the RBF pair loops, to decide whether the pair loops' contractions
// can move to the tensor cores without tcgen05/TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_mma tools/ubench_mma.cu && /tmp/ubench_mma
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;
constexpr int CH = 8;  // independent accumulators per warp

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// OP 0: HMMA tf32 only; 1: HMMA bf16 only; 2: per iteration and chain 1 HMMA tf32 + 1 MUFU.EX2
// (x4 chains of ex2); 3: 2 HMMA tf32 + 1 EX2 + 1 FFMA2; 4: EX2 only (reference)
template <int OP>
__global__ void kern(float* out, unsigned s) {
  float d[CH][4];
  unsigned a[4], b[2];
  float x[4];
  unsigned long long p[4];
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    a[i] = s * (threadIdx.x + i);
    x[i] = threadIdx.x * 1e-3f + i;
    p[i] = (unsigned long long)__float_as_uint(x[i]);
  }
  b[0] = s ^ threadIdx.x;
  b[1] = s + threadIdx.x;
  const unsigned long long ps = 0x3f8000003f800000ull, pt = 0x3a83126f3a83126full;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) mma_tf32(d[c], a, b);
      if (OP == 1) mma_bf16(d[c], a, b);
      if (OP == 2) {
        mma_tf32(d[c], a, b);
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c & 3]));
      }
      if (OP == 3) {
        mma_tf32(d[c], a, b);
        if (c & 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c & 3]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c & 3]) : "l"(ps), "l"(pt));
      }
      if (OP == 4) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c & 3]));
    }
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) r += d[c][0] + d[c][1] + d[c][2] + d[c][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) r += x[i] + __uint_as_float((unsigned)p[i]);
  if (r == 1234.5f) out[0] = r;
}

template <int OP>
void run(const char* name, double flop_per_mma, int mma_per_chain, int threads) {
  float* out;
  cudaMalloc(&out, 4);
  int dev;
  cudaGetDevice(&dev);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, dev);
  const int blocks = pr.multiProcessorCount * (2048 / threads);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<OP><<<blocks, threads>>>(out, 0x3f801234u);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<OP><<<blocks, threads>>>(out, 0x3f801234u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warps = 5.0 * blocks * threads / 32.0;
  const double mmas = warps * ITERS * CH * mma_per_chain;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double per_smsp_clk = mmas / (ms * 1e-3) / pr.multiProcessorCount / 4 / (clk * 1e3);
  printf("%-34s %8.3f ms  %8.1f TFLOP/s  %6.3f warp-MMA/clk/SMSP  (%d threads/CTA, %d warps/SM)\n", name, ms,
         mmas * flop_per_mma / (ms * 1e-3) / 1e12, per_smsp_clk, threads, 2048 / 32);
  cudaFree(out);
}

int main() {
  run<0>("HMMA m16n8k8 tf32", 16 * 8 * 8 * 2, 1, 256);
  run<1>("HMMA m16n8k16 bf16", 16 * 8 * 16 * 2, 1, 256);
  run<2>("HMMA tf32 + 1 EX2", 16 * 8 * 8 * 2, 1, 256);
  run<3>("HMMA tf32 + 0.5 EX2 + FFMA2", 16 * 8 * 8 * 2, 1, 256);
  run<4>("EX2 only (per 'MMA' = 1 warp EX2)", 0, 1, 256);
  return 0;
}
