// Microbenchmark: grid-wide barrier + all-reduce latency on B200 for the
// RESIDENT local-PCG path (k_resident_pcg), 148 CTAs x 512 threads, one per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bar_bench tools/bar_bench.cu && ./bar_bench
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// V: 5 sentinel ring (k_resident_pcg's group_allsum): release-store own slot, poll all slots;
// V: 0 fence+atomicAdd+acquire spin; 1 red.release + relaxed spin + fence; 2 cg grid.sync;
//    3 = 1 with nanosleep backoff; 4 = two-level (groups of 8 CTAs -> leaders)
template <int V>
__global__ void __launch_bounds__(512, 1) kbar(unsigned long long* bar, double* part, int iters, double* out) {
  __shared__ double red[16];
  const int G = gridDim.x, c = blockIdx.x;
  unsigned long long seq = 0;
  double acc = c;
  for (int it = 0; it < iters; ++it) {
    // CTA reduce of a value
    double v = acc + threadIdx.x;
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(~0u, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (V == 14) {  // 3 values per CTA, sum via 8 distributed arrival counters + one read of all slots
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double s = lane < 16 ? red[lane] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
        unsigned long long* ctr = bar;          // 8 counters, one 64-byte line
        double* sl = part;                      // [2][G][4]
        const int par = seq & 1;
        if (lane == 0) {
          for (int j = 0; j < 3; ++j) __stcg(&sl[(par * G + c) * 4 + j], s + j);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          atomicAdd(&ctr[c & 7], 1ull);
        }
        // counter k receives ceil/floor(G / 8) arrivals per reduction
        const unsigned long long need = lane < 8 ? (unsigned long long)((G - lane + 7) / 8) * (seq + 1) : 0ull;
        for (;;) {
          const unsigned long long v = lane < 8 ? ld_rlx(&ctr[lane]) : 0ull;
          if (__all_sync(~0u, v >= need)) break;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        double a2 = 0;
        for (int k = lane; k < G; k += 32)
          for (int j = 0; j < 3; ++j) a2 += __ldcg(&sl[(par * G + k) * 4 + j]);
        for (int o = 16; o; o >>= 1) a2 += __shfl_xor_sync(~0u, a2, o);
        if (lane == 0) red[0] = a2;
      }
      __syncthreads();
      acc = red[0] * 1e-9;
      ++seq;
      continue;
    }
    if (V >= 9) {  // 3 values per CTA (as k_resident_pcg): 9 = 3 release stores + acquire polls; 10 = + nanosleep(64)
                   // 11: 1 fence + relaxed stores, relaxed polls; 12: 1 fence + relaxed stores, acquire polls;
                   // 13: 1 fence + relaxed stores, relaxed polls + 1 reader fence
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double s = lane < 16 ? red[lane] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
        unsigned long long* sl = bar + 64;
        const unsigned ring = seq % 3, nxt = (seq + 1) % 3;
        if (lane == 0) {
          for (int j = 0; j < 3; ++j)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + (nxt * 3 + j) * G + c), "l"(~0ull) : "memory");
          if (V <= 10) {
            for (int j = 0; j < 3; ++j)
              asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(sl + (ring * 3 + j) * G + c),
                           "l"((unsigned long long)__double_as_longlong(s + j)) : "memory");
          } else {
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int j = 0; j < 3; ++j)
              asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + (ring * 3 + j) * G + c),
                           "l"((unsigned long long)__double_as_longlong(s + j)) : "memory");
          }
        }
        unsigned long long u[3][5];
        for (int j = 0; j < 3; ++j)
          for (int t = 0; t < 5; ++t) u[j][t] = lane + 32 * t < G ? ~0ull : 0ull;
        for (;;) {
          bool done = true;
#pragma unroll
          for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int t = 0; t < 5; ++t)
              if (u[j][t] == ~0ull)
                u[j][t] = (V == 11 || V == 13) ? ld_rlx(sl + (ring * 3 + j) * G + lane + 32 * t)
                                               : ld_acq(sl + (ring * 3 + j) * G + lane + 32 * t);
#pragma unroll
          for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int t = 0; t < 5; ++t) done = done && u[j][t] != ~0ull;
          if (__all_sync(~0u, done)) break;
          if (V == 10) __nanosleep(64);
        }
        if (V == 13) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        double a2 = 0;
        for (int j = 0; j < 3; ++j)
          for (int t = 0; t < 5; ++t) a2 += __longlong_as_double(u[j][t]);
        for (int o = 16; o; o >>= 1) a2 += __shfl_xor_sync(~0u, a2, o);
        if (lane == 0) red[0] = a2;
      }
      __syncthreads();
      acc = red[0] * 1e-9;
      ++seq;
      continue;
    }
    if (V >= 6) {  // 6: parallel poll + fence.sc; 7: parallel poll + fence.acq_rel; 8: no fence
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double s = lane < 16 ? red[lane] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
        unsigned long long* sl = bar + 64;
        const unsigned ring = seq % 3, nxt = (seq + 1) % 3;
        if (lane == 0) {
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + nxt * G + c), "l"(~0ull) : "memory");
          if (V == 8)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + ring * G + c),
                         "l"((unsigned long long)__double_as_longlong(s)) : "memory");
          else
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(sl + ring * G + c),
                         "l"((unsigned long long)__double_as_longlong(s)) : "memory");
        }
        unsigned long long u[5];
        for (int t = 0; t < 5; ++t) u[t] = lane + 32 * t < G ? ~0ull : 0ull;
        for (;;) {
          bool done = true;
#pragma unroll
          for (int t = 0; t < 5; ++t)
            if (u[t] == ~0ull) u[t] = ld_rlx(sl + ring * G + lane + 32 * t);
#pragma unroll
          for (int t = 0; t < 5; ++t) done = done && u[t] != ~0ull;
          if (__all_sync(~0u, done)) break;
        }
        if (V == 6) __threadfence();
        if (V == 7) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        double a2 = 0;
        for (int t = 0; t < 5; ++t) a2 += __longlong_as_double(u[t]);
        for (int o = 16; o; o >>= 1) a2 += __shfl_xor_sync(~0u, a2, o);
        if (lane == 0) red[0] = a2;
      }
      __syncthreads();
      acc = red[0] * 1e-9;
      ++seq;
      continue;
    }
    if (V == 5) {
      if (threadIdx.x < 32) {
        double s = threadIdx.x < 16 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
        unsigned long long* sl = bar + 64;  // [3][G]
        const unsigned ring = seq % 3, nxt = (seq + 1) % 3;
        if (threadIdx.x == 0) {
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sl + nxt * G + c), "l"(~0ull) : "memory");
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(sl + ring * G + c),
                       "l"((unsigned long long)__double_as_longlong(s)) : "memory");
        }
        double acc = 0;
        for (int k = threadIdx.x; k < G; k += 32) {
          unsigned long long u;
          while ((u = ld_rlx(sl + ring * G + k)) == ~0ull) {
          }
          acc += __longlong_as_double(u);
        }
        __threadfence();
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
        if (threadIdx.x == 0) red[0] = acc;
      }
      __syncthreads();
      acc = red[0] * 1e-9;
      ++seq;
      continue;
    }
    if (V == 2) {
      if (threadIdx.x == 0) {
        double s = 0;
        for (int k = 0; k < 16; ++k) s += red[k];
        part[(seq & 1) * G + c] = s;
      }
      cg::this_grid().sync();
    } else if (threadIdx.x < 32) {
      double s = threadIdx.x < 16 ? red[threadIdx.x] : 0.0;
      for (int o = 16; o; o >>= 1) s += __shfl_down_sync(~0u, s, o);
      if (threadIdx.x == 0) {
        __stcg(&part[(seq & 1) * G + c], s);
        const unsigned long long target = (seq + 1) * (unsigned long long)G;
        if (V == 0) {
          __threadfence();
          atomicAdd(bar, 1ull);
          while (ld_acq(bar) < target) {
          }
        } else if (V == 1 || V == 3) {
          red_rel(bar, 1ull);
          while (ld_rlx(bar) < target) {
            if (V == 3) __nanosleep(32);
          }
          __threadfence();
        } else {  // V == 4: two level, groups of 8
          const int grp = c >> 3, ngrp = (G + 7) >> 3;
          const int gsz = min(8, G - grp * 8);
          unsigned long long* gb = bar + 16 * (1 + grp);
          red_rel(gb, 1ull);
          if ((c & 7) == 0) {
            while (ld_rlx(gb) < (seq + 1) * gsz) {
            }
            __threadfence();
            red_rel(bar, 1ull);
          }
          while (ld_rlx(bar) < (seq + 1) * ngrp) {
          }
          __threadfence();
        }
      }
    }
    __syncthreads();
    ++seq;
    // everyone sums the partials
    const int lane = threadIdx.x & 31;
    double s = 0;
    for (int k = lane; k < G; k += 32) s += __ldcg(&part[((seq - 1) & 1) * G + k]);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    acc = s * 1e-9;
  }
  if (threadIdx.x == 0 && c == 0) *out = acc;
}

template <int V>
float run(int G, int iters, unsigned long long* bar, double* part, double* out) {
  cudaMemset(bar, 0, 64 * 8);
  void* args[] = {&bar, &part, &iters, &out};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)kbar<V>, G, 512, args, 0, 0);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* bar;
  double *part, *out;
  cudaMalloc(&bar, (64 + 9 * 1024) * 8);
  cudaMalloc(&part, 2 * 1024 * 4 * 8);
  cudaMalloc(&out, 8);
  const int iters = 2000;
  for (int G : {sms, sms / 2, 74, 37, 16}) {
    run<0>(G, 10, bar, part, out);
    float t0 = run<0>(G, iters, bar, part, out);
    float t1 = run<1>(G, iters, bar, part, out);
    float t2 = run<2>(G, iters, bar, part, out);
    float t3 = run<3>(G, iters, bar, part, out);
    float t4 = run<4>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8);
    float t5 = run<5>(G, iters, bar, part, out);
    float t6, t7, t8;
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8);
    t6 = run<6>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8);
    t7 = run<7>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8);
    t8 = run<8>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8 * 3);
    float t9 = run<9>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8 * 3);
    float t10 = run<10>(G, iters, bar, part, out);
    float t11, t12, t13;
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8 * 3);
    t11 = run<11>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8 * 3);
    t12 = run<12>(G, iters, bar, part, out);
    cudaMemset(bar + 64, 0xff, 3 * 1024 * 8 * 3);
    t13 = run<13>(G, iters, bar, part, out);
    cudaMemset(bar, 0, 64 * 8);
    float t14 = run<14>(G, iters, bar, part, out);
    printf("G=%3d 3-value distributed counters (8) + one slot read: %.2f\n", G, t14 * 1e3 / iters);
    printf("G=%3d 3-value ring: 3 st.release + acquire polls %.2f | + nanosleep %.2f | fence+relaxed st: relaxed polls %.2f, acquire polls %.2f, relaxed polls + fence %.2f\n",
           G, t9 * 1e3 / iters, t10 * 1e3 / iters, t11 * 1e3 / iters, t12 * 1e3 / iters, t13 * 1e3 / iters);
    printf("G=%3d parallel-poll ring: fence.sc %.2f | fence.acq_rel %.2f | no fence (unsafe) %.2f\n", G, t6 * 1e3 / iters,
           t7 * 1e3 / iters, t8 * 1e3 / iters);
    printf("G=%3d us/barrier: fence+atom+acq %.2f | red.release+rlx %.2f | cg.sync %.2f | +nanosleep %.2f | 2-level %.2f | sentinel ring %.2f\n", G,
           t0 * 1e3 / iters, t1 * 1e3 / iters, t2 * 1e3 / iters, t3 * 1e3 / iters, t4 * 1e3 / iters, t5 * 1e3 / iters);
  }
  return 0;
}
