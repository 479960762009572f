// FP32 pipe micro-benchmark (sm_100a): issue throughput of the instruction forms the
// forward/backward inner loops use, so the ALU roofline in DESIGN.md rests on measurements.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_fp32.cu && /tmp/ubench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  return (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
}

template <int OP>
__global__ void kern(float* out, float s, float t) {
  float x[CH];
  unsigned long long p[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = threadIdx.x * 1e-3f + c;
    p[c] = pk(x[c], x[c] + 1.f);
  }
  const unsigned long long ps = pk(s, s + 1e-7f), pt = pk(t, t);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) x[c] = fmaf(x[c], s, t);                 // FFMA 3-reg
      if (OP == 1) x[c] = fmaf(x[c], 0.999f, 1e-4f);        // FFMA imm
      if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(ps), "l"(pt));
      if (OP == 3) x[c] = x[c] + s;                         // FADD
      if (OP == 4) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(ps));
      if (OP == 5) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
      if (OP == 6) { x[c] = fmaf(x[c], s, t); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c])); }
      if (OP == 7) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[c]) : "l"(ps));
      if (OP == 8) { unsigned v = __float_as_uint(x[c]); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(0x9E3779B9u), "r"(7u)); x[c] = __uint_as_float(v); }
      if (OP == 9) {  // 4 FFMA2 + 1 MUFU.EX2 x2 (the forward's packed pair mix: 9 packed FP32 + 2 EX2 per 2 pairs)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(ps), "l"(pt));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(ps), "l"(pt));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(ps), "l"(pt));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[c]) : "l"(ps), "l"(pt));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
      }
    }
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) r += x[c] + __uint_as_float((unsigned)p[c]) + __uint_as_float((unsigned)(p[c] >> 32));
  if (r == 1234.5f) out[0] = r;
}

template <int OP>
void run(const char* name, int lanes_per_instr, int ops_per_iter) {
  float* out;
  cudaMalloc(&out, 4);
  int dev;
  cudaGetDevice(&dev);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, dev);
  const int blocks = pr.multiProcessorCount * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<OP><<<blocks, threads>>>(out, 1.0001f, 1e-5f);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kern<OP><<<blocks, threads>>>(out, 1.0001f, 1e-5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double instr = 5.0 * blocks * threads / 32.0 * ITERS * CH * ops_per_iter;  // warp instructions
  const double lane_ops = instr * 32 * lanes_per_instr;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double per_sm_clk = lane_ops / (ms * 1e-3) / pr.multiProcessorCount / (clk * 1e3);
  printf("%-22s %8.3f ms  %9.2f T lane-op/s  %6.1f lane-op/clk/SM (at %d MHz nominal)\n", name, ms,
         lane_ops / (ms * 1e-3) / 1e12, per_sm_clk, clk / 1000);
  cudaFree(out);
}

// red.global.add.v4.f32 throughput (L2 atomic ALU): every thread adds 16 B to one of n_slots
// 64-B slots (the padded gradient layout: 2 red.v4 per offset key), spread like the backward's keys
__global__ void kred(float* g, int n_slots, int iters) {
  const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    const unsigned slot = (tid * 2654435761u + i * 40503u) % (unsigned)n_slots;
    float* a = g + (size_t)slot * 16;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f)
                 : "memory");
  }
}

void run_red(int n_slots) {
  float* g;
  cudaMalloc(&g, (size_t)n_slots * 64);
  cudaMemset(g, 0, (size_t)n_slots * 64);
  int dev;
  cudaGetDevice(&dev);
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, dev);
  const int blocks = pr.multiProcessorCount * 8, threads = 256, iters = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kred<<<blocks, threads>>>(g, n_slots, iters);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) kred<<<blocks, threads>>>(g, n_slots, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double reds = 5.0 * blocks * threads * iters;
  printf("%-22s %8.3f ms  %9.3f G red.v4/s (%d slots of 64 B)\n", "RED.E.ADD.F32x4", ms, reds / (ms * 1e-3) / 1e9,
         n_slots);
  cudaFree(g);
}

int main() {
  run<0>("FFMA r,r,r", 1, 1);
  run<1>("FFMA r,imm,imm", 1, 1);
  run<2>("FFMA2 (f32x2)", 2, 1);
  run<3>("FADD", 1, 1);
  run<4>("FADD2 (f32x2)", 2, 1);
  run<5>("MUFU.EX2", 1, 1);
  run<6>("FFMA+MUFU.EX2", 1, 2);
  run<7>("FMUL2 (f32x2)", 2, 1);
  run<8>("IMAD", 1, 1);
  run<9>("4 FFMA2 + 1 EX2 (lane-ops)", 9, 1);  // 8 FP32 lane-ops + 1 EX2 per lane per iter; reported as 9
  run_red(65536);
  run_red(32768 * 2);
  run_red(1 << 20);
  return 0;
}
