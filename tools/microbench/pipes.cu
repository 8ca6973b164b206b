// Pipe-rate microbenchmark for the ops the LM kernel leans on (sm_100a):
// F2F.F64.F32, DADD, FMUL/FADD, SHFL, MUFU.RCP, packed FFMA2/FADD2, integer widening.
// Prints thread-ops/clk/SM (a packed op counts 2).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_f2f(float* out, float seed) {
  float a = seed + threadIdx.x; double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  float b = a * 1.0001f, c = a * 0.9999f, d = a + 1.f;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    acc0 += (double)a; acc1 += (double)b; acc2 += (double)c; acc3 += (double)d;
    a = __fadd_rn(a, 1.0f); b = __fadd_rn(b, 1.0f); c = __fadd_rn(c, 1.0f); d = __fadd_rn(d, 1.0f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc0 + acc1 + acc2 + acc3);
}
__global__ void k_f2f_only(float* out, float seed) {
  // conversions whose results are XOR'd as ints (no DADD), to isolate F2F
  float a = seed + threadIdx.x; unsigned long long x0 = 0, x1 = 0, x2 = 0, x3 = 0;
  float b = a * 1.0001f, c = a * 0.9999f, d = a + 1.f;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    x0 ^= __double_as_longlong((double)a); x1 ^= __double_as_longlong((double)b);
    x2 ^= __double_as_longlong((double)c); x3 ^= __double_as_longlong((double)d);
    a = __fadd_rn(a, 1.0f); b = __fadd_rn(b, 1.0f); c = __fadd_rn(c, 1.0f); d = __fadd_rn(d, 1.0f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(x0 ^ x1 ^ x2 ^ x3);
}
__global__ void k_dadd(float* out, float seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  double s = 1e-3;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = __dadd_rn(a0, s); a1 = __dadd_rn(a1, s); a2 = __dadd_rn(a2, s); a3 = __dadd_rn(a3, s);
    a4 = __dadd_rn(a4, s); a5 = __dadd_rn(a5, s); a6 = __dadd_rn(a6, s); a7 = __dadd_rn(a7, s);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7);
}
__global__ void k_fmul(float* out, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  float s = 1.0000001f, t = 0.9999999f;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = __fmul_rn(a0, s); a1 = __fmul_rn(a1, t); a2 = __fmul_rn(a2, s); a3 = __fmul_rn(a3, t);
    a4 = __fmul_rn(a4, s); a5 = __fmul_rn(a5, t); a6 = __fmul_rn(a6, s); a7 = __fmul_rn(a7, t);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_shfl(float* out, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = __shfl_xor_sync(0xffffffffu, a0, 1); a1 = __shfl_xor_sync(0xffffffffu, a1, 2);
    a2 = __shfl_xor_sync(0xffffffffu, a2, 4); a3 = __shfl_xor_sync(0xffffffffu, a3, 8);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
__global__ void k_rcp(float* out, float seed) {
  float a0 = seed + threadIdx.x + 1, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = __frcp_rn(a0); a1 = __frcp_rn(a1); a2 = __frcp_rn(a2); a3 = __frcp_rn(a3);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
__global__ void k_ex2(float* out, float seed) {
  float a0 = -(seed + threadIdx.x)*1e-3f, a1 = a0 - 1, a2 = a0 - 2, a3 = a0 - 3;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = -exp2f(a0); a1 = -exp2f(a1); a2 = -exp2f(a2); a3 = -exp2f(a3);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c){u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b){u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__device__ __forceinline__ u64 pk(float x, float y){return ((u64)__float_as_uint(y) << 32) | __float_as_uint(x);}
// packed FP32: 8 independent FFMA2 chains, all-register operands (2 flops... counted as 2 thread-ops each)
__global__ void k_ffma2(float* out, float seed) {
  float a = seed + threadIdx.x;
  u64 a0 = pk(a, a+1), a1 = pk(a+2, a+3), a2 = pk(a+4,a+5), a3 = pk(a+6,a+7), a4 = pk(a+8,a+9), a5 = pk(a+10,a+11), a6 = pk(a+12,a+13), a7 = pk(a+14,a+15);
  u64 s = pk(1.0000001f + threadIdx.x * 1e-9f, 0.9999999f), t = pk(1e-7f * threadIdx.x, 1e-7f);
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = ffma2(a0, s, t); a1 = ffma2(a1, s, t); a2 = ffma2(a2, s, t); a3 = ffma2(a3, s, t);
    a4 = ffma2(a4, s, t); a5 = ffma2(a5, s, t); a6 = ffma2(a6, s, t); a7 = ffma2(a7, s, t);
  }
  u64 r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((unsigned)r ^ (unsigned)(r >> 32));
}
__global__ void k_fadd2(float* out, float seed) {
  float a = seed + threadIdx.x;
  u64 a0 = pk(a, a+1), a1 = pk(a+2, a+3), a2 = pk(a+4,a+5), a3 = pk(a+6,a+7), a4 = pk(a+8,a+9), a5 = pk(a+10,a+11), a6 = pk(a+12,a+13), a7 = pk(a+14,a+15);
  u64 s = pk(1e-7f * threadIdx.x, 1e-7f);
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = fadd2(a0, s); a1 = fadd2(a1, s); a2 = fadd2(a2, s); a3 = fadd2(a3, s);
    a4 = fadd2(a4, s); a5 = fadd2(a5, s); a6 = fadd2(a6, s); a7 = fadd2(a7, s);
  }
  u64 r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float((unsigned)r ^ (unsigned)(r >> 32));
}
// scalar FFMA with register (non-immediate) operands
__global__ void k_ffma_reg(float* out, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  float s = 1.0000001f + threadIdx.x * 1e-9f, t = 1e-7f * threadIdx.x;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    a0 = __fmaf_rn(a0, s, t); a1 = __fmaf_rn(a1, s, t); a2 = __fmaf_rn(a2, s, t); a3 = __fmaf_rn(a3, s, t);
    a4 = __fmaf_rn(a4, s, t); a5 = __fmaf_rn(a5, s, t); a6 = __fmaf_rn(a6, s, t); a7 = __fmaf_rn(a7, s, t);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
// F2F widen + DADD interleaved with FFMA2 work: do the XU and FMA pipes overlap?
__global__ void k_f2f_ffma2(float* out, float seed) {
  float a = seed + threadIdx.x; double acc0 = 0, acc1 = 0;
  float b = a * 1.0001f;
  u64 a0 = pk(a, a+1), a1 = pk(a+2, a+3), a2 = pk(a+4,a+5), a3 = pk(a+6,a+7);
  u64 s = pk(1.0000001f + threadIdx.x * 1e-9f, 0.9999999f), t = pk(1e-7f * threadIdx.x, 1e-7f);
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    acc0 += (double)a; acc1 += (double)b;
    a = __fadd_rn(a, 1.0f); b = __fadd_rn(b, 1.0f);
    a0 = ffma2(a0, s, t); a1 = ffma2(a1, s, t); a2 = ffma2(a2, s, t); a3 = ffma2(a3, s, t);
  }
  u64 r = a0 ^ a1 ^ a2 ^ a3;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc0 + acc1) + __uint_as_float((unsigned)r ^ (unsigned)(r >> 32));
}
// f32 -> f64 widening by integer ops (normal inputs): hi = (b>>3)+bias | sign, lo = b<<29
__global__ void k_intwiden(float* out, float seed) {
  float a = seed + threadIdx.x; double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  float b = a * 1.0001f, c = a * 0.9999f, d = a + 1.f;
  #pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    unsigned x[4] = {__float_as_uint(a), __float_as_uint(b), __float_as_uint(c), __float_as_uint(d)};
    double w[4];
    #pragma unroll
    for (int k = 0; k < 4; ++k) {
      unsigned hi = (((x[k] & 0x7fffffffu) >> 3) + 0x38000000u) | (x[k] & 0x80000000u);
      hi = (x[k] & 0x7fffffffu) == 0 ? x[k] : hi;
      w[k] = __hiloint2double((int)hi, (int)(x[k] << 29));
    }
    acc0 += w[0]; acc1 += w[1]; acc2 += w[2]; acc3 += w[3];
    a = __fadd_rn(a, 1.0f); b = __fadd_rn(b, 1.0f); c = __fadd_rn(c, 1.0f); d = __fadd_rn(d, 1.0f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc0 + acc1 + acc2 + acc3);
}

typedef void (*kfn)(float*, float);
static void run(const char* name, kfn k, double ops_per_iter, int sms) {
  float* d; cudaMalloc(&d, 148 * 64 * 1024 * sizeof(float));
  int threads = 512, blocks = sms * 4;
  k<<<blocks, threads>>>(d, 1.f); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<blocks, threads>>>(d, 1.f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double total = (double)blocks * threads * ITERS * ops_per_iter;
  double per_sm_clk = total / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("%-10s %8.3f ms  %8.2f thread-ops/clk/SM (at attr clock %d MHz)  err=%s\n", name, ms, per_sm_clk, clk_khz/1000,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  run("f2f+dadd", k_f2f, 4, sms);
  run("f2f_only", k_f2f_only, 4, sms);
  run("dadd", k_dadd, 8, sms);
  run("fmul", k_fmul, 8, sms);
  run("shfl", k_shfl, 4, sms);
  run("rcp_rn", k_rcp, 4, sms);
  run("exp2f", k_ex2, 4, sms);
  run("ffma_reg", k_ffma_reg, 8, sms);
  run("ffma2", k_ffma2, 16, sms);
  run("fadd2", k_fadd2, 16, sms);
  run("f2f|ffma2", k_f2f_ffma2, 2, sms);
  run("intwiden", k_intwiden, 4, sms);
  return 0;
}
