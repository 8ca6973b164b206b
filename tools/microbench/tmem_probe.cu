// tmem_probe.cu -- does per-thread TMEM storage work the way the fit kernel would use it?
// 4 CTAs x 128 threads per SM; each CTA allocates 128 TMEM columns, every thread stores 8 floats
// per "pair" into its own TMEM lane (tcgen05.st.32x32b.x8) for 14 pairs, waits, reads them back
// (tcgen05.ld.32x32b.x8 + wait::ld) and checks them; times the round trips.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

__global__ void __launch_bounds__(128, 4) probe(int reps, unsigned long long* bad, unsigned long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t t0 = tbase + ((uint32_t)(warp * 32) << 16);  // this warp's lane quarter
  unsigned long long nbad = 0;
  const long long c0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    for (int p = 0; p < 14; ++p) {
      uint32_t r[8];
      for (int k = 0; k < 8; ++k) r[k] = (uint32_t)(threadIdx.x * 1000003u + p * 131u + k + rep * 7u + blockIdx.x);
      tm_st8(t0 + p * 8, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    for (int p = 0; p < 14; ++p) {
      uint32_t r[8];
      tm_ld8(t0 + p * 8, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int k = 0; k < 8; ++k)
        nbad += r[k] != (uint32_t)(threadIdx.x * 1000003u + p * 131u + k + rep * 7u + blockIdx.x);
    }
  }
  const long long c1 = clock64();
  if (nbad) atomicAdd(bad, nbad);
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(c1 - c0));
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tbase));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *bad, *cyc;
  cudaMalloc(&bad, 8);
  cudaMalloc(&cyc, 8);
  for (int blocks_per_sm : {1, 4}) {
    cudaMemset(bad, 0, 8);
    cudaMemset(cyc, 0, 8);
    const int reps = 200;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<<<sms * blocks_per_sm, 128>>>(reps, bad, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long hb = 0, hc = 0;
    cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    const double per_pair = (double)hc / (sms * blocks_per_sm) / reps / 14.0;
    const double bytes = 2.0 * 32.0 * 128 * 14 * reps * sms * blocks_per_sm;
    printf("blocks/SM %d: %s, mismatches %llu, %.3f ms, %.1f cycles per (st + ld) pair per thread, %.0f GB/s TMEM st+ld\n",
           blocks_per_sm, cudaGetErrorString(err), hb, ms, per_pair, bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
