// Micro-benchmark: cost of the system-scope release (fence.acq_rel.sys + flag store) that
// publishes a GEMM-RS wire tile, as the number of stores in flight and the publishing warp vary.
// 148 CTAs x (8 storer warps + 1 publisher warp). Each iteration every storer warp stores
// `kb` KiB (16-B stores, coalesced) to its own region, then:
//   mode 0: each storer warp: fence.acq_rel.sys, lane 0 flag store            (per-warp publish)
//   mode 1: storers bar.arrive; publisher warp bar.sync, fence.acq_rel.sys, flag (hand-off)
//   mode 2: as 0 with fence.acq_rel.gpu
//   mode 3: as 1 with fence.acq_rel.gpu
//   mode 4: no fence (stores + flag only)
// Prints mean fence time (ns) and the mean iteration time (ns) seen by the storers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fence_cost fence_cost.cu && ./fence_cost
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int kMode>
__global__ void __launch_bounds__(288, 1) k(uint4* buf, uint32_t* flags, unsigned long long* acc, int iters, int kb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per_warp16 = kb * 1024 / 16;
  uint4* mine = buf + (static_cast<int64_t>(blockIdx.x) * 8 + (warp < 8 ? warp : 0)) * per_warp16;
  unsigned long long fence_ns = 0, iter_ns = 0;
  for (int it = 0; it < iters; ++it) {
    const uint64_t t0 = gt();
    if (warp < 8) {
      for (int i = lane; i < per_warp16; i += 32) mine[i] = make_uint4(it, i, warp, blockIdx.x);
      if (kMode == 0 || kMode == 2 || kMode == 4) {
        const uint64_t f0 = gt();
        if (kMode == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
        if (kMode == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (lane == 0) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 16 + warp), "r"(it) : "memory");
        fence_ns += gt() - f0;
      } else {
        asm volatile("bar.arrive 1, 288;" ::: "memory");
      }
      iter_ns += gt() - t0;
    } else if (kMode == 1 || kMode == 3) {
      asm volatile("bar.sync 1, 288;" ::: "memory");
      const uint64_t f0 = gt();
      if (kMode == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
      if (kMode == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (lane == 0) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 16 + 8), "r"(it) : "memory");
      fence_ns += gt() - f0;
      // storers of the next iteration wait for this (keeps barrier generations apart)
    }
    if (kMode == 1 || kMode == 3) __syncthreads();
  }
  if (lane == 0) {
    if (fence_ns) { atomicAdd(acc + 0, fence_ns); atomicAdd(acc + 2, 1ull); }
    if (warp < 8) { atomicAdd(acc + 1, iter_ns); atomicAdd(acc + 3, 1ull); }
  }
}

int main() {
  const int ctas = 148, iters = 200;
  uint4* buf; uint32_t* flags; unsigned long long* acc;
  cudaMalloc(&buf, static_cast<size_t>(ctas) * 8 * 64 * 1024);
  cudaMalloc(&flags, ctas * 16 * 4);
  cudaMalloc(&acc, 4 * 8);
  const char* names[] = {"per-warp fence.sys", "hand-off fence.sys", "per-warp fence.gpu", "hand-off fence.gpu", "no fence"};
  for (int kb : {2, 8, 16, 32}) {
    for (int mode = 0; mode < 5; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(acc, 0, 32);
        switch (mode) {
          case 0: k<0><<<ctas, 288>>>(buf, flags, acc, iters, kb); break;
          case 1: k<1><<<ctas, 288>>>(buf, flags, acc, iters, kb); break;
          case 2: k<2><<<ctas, 288>>>(buf, flags, acc, iters, kb); break;
          case 3: k<3><<<ctas, 288>>>(buf, flags, acc, iters, kb); break;
          case 4: k<4><<<ctas, 288>>>(buf, flags, acc, iters, kb); break;
        }
        unsigned long long h[4];
        cudaMemcpy(h, acc, 32, cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("kb/warp %2d  %-20s fence %8.0f ns  storer iteration %8.0f ns\n", kb, names[mode],
                 h[2] ? double(h[0]) / h[2] / iters : 0.0, double(h[1]) / h[3] / iters);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
