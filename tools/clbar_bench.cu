// Microbenchmark: per-level cost of the cluster-resident triangular solve's
// synchronisation (k_trsv_cl) on B200 -- barrier.cluster alone and with the
// global store -> barrier -> dependent load chain of one level.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o clbar_bench tools/clbar_bench.cu && ./clbar_bench
// Variants (one "level" = one iteration):
//   0  barrier.cluster.arrive.release + wait.acquire
//   1  arrive.relaxed + wait (no release)
//   2  st.global of one word per thread, then 0
//   3  2 + a load of a word another CTA stored the previous level (ld.global.cg), used in the store
//   4  3 + eight independent DRAM loads per thread issued between arrive and wait (prefetch stand-in)
//   5  4 with the prefetch as cp.async into shared memory (not waited on by the release)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

template <int V>
__global__ void __launch_bounds__(512, 1) kcl(double* buf, const double* big, long long bigmask, int iters,
                                                   unsigned long long* cyc, double* sink) {
  __shared__ double stage[512 * 8];
  const unsigned r = cl_rank(), n = cl_size();
  const int cl = blockIdx.x / n;
  const int t = threadIdx.x;
  double* my = buf + ((size_t)cl * n * 2) * 512;  // [2][n][512] per cluster
  double acc = 0.0, pf = 0.0;
  unsigned long long h = (unsigned long long)(blockIdx.x * 512 + t) * 0x9E3779B97F4A7C15ull;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    if (V >= 3) {
      // a word stored by the next CTA of the cluster in the previous level
      const double v = __ldcg(&my[((size_t)(par ^ 1) * n + (r + 1) % n) * 512 + (t * 37) % 512]);
      acc = acc * 0.5 + v;
    }
    if (V >= 2) __stcg(&my[((size_t)par * n + r) * 512 + t], acc + it);
    if (V == 1)
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    else
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if (V == 4) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        pf += __ldg(&big[(h >> 20) & bigmask]);
      }
    }
    if (V == 5) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(&stage[k * 512 + t])),
                     "l"(&big[(h >> 20) & bigmask])
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (V == 5) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      pf += stage[((it + 3) & 7) * 512 + t];
    }
  }
  unsigned long long t1 = clock64();
  if (V == 5) asm volatile("cp.async.wait_all;" ::: "memory");
  if (t == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc + pf == 12345.678) sink[0] = acc + pf;
}

template <int V>
void run(int csz, int nclusters, double* buf, const double* big, long long mask, unsigned long long* cyc, double* sink) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csz * nclusters);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csz;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int iters = 2000;
  cudaFuncSetAttribute(kcl<V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchKernelEx(&cfg, kcl<V>, buf, big, mask, iters, cyc, sink);  // warm
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kcl<V>, buf, big, mask, iters, cyc, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[16 * 16];
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * csz * nclusters, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < csz * nclusters; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("{\"variant\": %d, \"cluster\": %d, \"clusters\": %d, \"ns_per_level\": %.1f, \"cycles_per_level\": %.1f, \"err\": \"%s\"}\n", V,
         csz, nclusters, 1e6 * ms / iters, (double)mx / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *buf, *big, *sink;
  unsigned long long* cyc;
  const long long nbig = 1ll << 27;  // 1 GB of doubles: the prefetch stand-in misses L2
  cudaMalloc(&buf, sizeof(double) * 16 * 16 * 2 * 512);
  cudaMalloc(&big, sizeof(double) * nbig);
  cudaMemset(big, 0, sizeof(double) * nbig);
  cudaMalloc(&sink, 8);
  cudaMalloc(&cyc, 8 * 256);
  for (int csz : {1, 4, 7, 16})
    for (int ncl : {1, 8}) {
      if (csz == 16 && ncl == 8) ncl = 7;
      run<0>(csz, ncl, buf, big, nbig - 1, cyc, sink);
      run<1>(csz, ncl, buf, big, nbig - 1, cyc, sink);
      run<2>(csz, ncl, buf, big, nbig - 1, cyc, sink);
      run<3>(csz, ncl, buf, big, nbig - 1, cyc, sink);
      run<4>(csz, ncl, buf, big, nbig - 1, cyc, sink);
      run<5>(csz, ncl, buf, big, nbig - 1, cyc, sink);
    }
  return 0;
}
