// TMEM as per-thread private storage (probe for the RESIDENT redesign):
// 768 threads (24 warps, 6 per TMEM lane quadrant), 512 columns allocated,
// each warp owns an 80-column block of its quadrant's 32 lanes; every thread
// stores 40 doubles (80 x 32-bit columns) and reads them back.  Checks values
// and times tcgen05.ld / tcgen05.st throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st2(uint32_t taddr, double v) {
  uint32_t lo = (uint32_t)__double_as_longlong(v), hi = (uint32_t)(__double_as_longlong(v) >> 32);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ double tm_ld2(uint32_t taddr) {
  uint32_t lo, hi;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __longlong_as_double(((long long)hi << 32) | lo);
}
template <int N>
__device__ __forceinline__ void tm_ld8(uint32_t taddr, double (&v)[4]) {
  uint32_t a[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7])
               : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = __longlong_as_double(((long long)a[2 * k + 1] << 32) | a[2 * k]);
}

__global__ void __launch_bounds__(768, 1) k_probe(int iters, unsigned long long* cyc, int* bad) {
  __shared__ uint32_t s_base;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = s_base;
  const uint32_t my = base + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)(80 * (w >> 2));
  // store 40 doubles per thread
  for (int j = 0; j < 40; ++j) tm_st2(my + 2 * j, (double)(threadIdx.x * 1000 + j + blockIdx.x * 1e6));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  int nbad = 0;
  for (int j = 0; j < 40; ++j)
    if (tm_ld2(my + 2 * j) != (double)(threadIdx.x * 1000 + j + blockIdx.x * 1e6)) ++nbad;
  // throughput: x2 loads with a wait each, then x8 loads
  double acc = 0.0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int j = 0; j < 40; ++j) acc += tm_ld2(my + 2 * j);
  __syncthreads();
  unsigned long long t1 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int j = 0; j < 40; j += 4) {
      double v[4];
      tm_ld8<8>(my + 2 * j, v);
      acc += v[0] + v[1] + v[2] + v[3];
    }
  __syncthreads();
  unsigned long long t2 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int j = 0; j < 40; ++j) tm_st2(my + 2 * j, acc + j);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncthreads();
  unsigned long long t3 = clock64();
  if (acc == 12345.0) nbad += 1000000;
  atomicAdd(bad, nbad);
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  unsigned long long* cyc;
  int* bad;
  cudaMalloc(&cyc, 24);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  const int iters = 200;
  k_probe<<<148, 768>>>(iters, cyc, bad);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[3];
  int hb;
  cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  const double bytes = 768.0 * 40 * 8 * iters;  // per CTA per pass
  printf("err=%s bad=%d\n", cudaGetErrorString(e), hb);
  printf("ld x2+wait: %llu cyc -> %.1f B/clk/SM\n", h[0], bytes / h[0]);
  printf("ld x8+wait: %llu cyc -> %.1f B/clk/SM\n", h[1], bytes / h[1]);
  printf("st x2     : %llu cyc -> %.1f B/clk/SM\n", h[2], bytes / h[2]);
  return 0;
}
