// Pipe-rate microbenchmark for the ops the LM kernel leans on (sm_100a):
// F2F.F64.F32, DADD, FMUL/FADD, SHFL, MUFU.RCP. Prints thread-ops/clk/SM.
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
  return 0;
}
