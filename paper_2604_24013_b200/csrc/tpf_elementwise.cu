// Element-wise glue of the TP-SP MLP block (tpsp_mlp_forward, layers.cpp:140-147):
// SwiGLU on the rank's [gate | up] column shard. HBM-bound: 16 B vector loads/stores,
// grid sized to a multiple of the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>

#include "tpf.h"
#include "tpf_host.h"
#include "tpf_internal.h"
#include "tpf_ptx.cuh"

#include <algorithm>

namespace tpf {
namespace {

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

__global__ void __launch_bounds__(256) swiglu_kernel(const uint4* __restrict__ gu,
                                                     uint4* __restrict__ out, int64_t rows,
                                                     int64_t f_vec) {
  const int64_t total = rows * f_vec;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / f_vec, c = i - r * f_vec;
    const uint4 g = gu[r * 2 * f_vec + c];
    const uint4 u = gu[r * 2 * f_vec + f_vec + c];
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 gf = __bfloat1622float2(g2[k]);
      const float2 uf = __bfloat1622float2(u2[k]);
      o2[k] = __floats2bfloat162_rn(silu(gf.x) * uf.x, silu(gf.y) * uf.y);
    }
    out[i] = o;
  }
}

}  // namespace
}  // namespace tpf

extern "C" int tpf_swiglu(const void* gu, void* out, int64_t rows, int64_t F, void* stream) {
  if (rows < 1 || F < 1 || F % 8) return TPF_E_SHAPE;
  const int sms = tpf::num_sms();
  if (sms <= 0) return TPF_E_CUDA;
  const int64_t f_vec = F / 8;
  const int64_t work = rows * f_vec;
  int64_t blocks = (work + 255) / 256;
  blocks = blocks < static_cast<int64_t>(sms) * 8 ? blocks : static_cast<int64_t>(sms) * 8;
  tpf::swiglu_kernel<<<static_cast<int>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(gu), static_cast<uint4*>(out), rows, f_vec);
  return cudaGetLastError() == cudaSuccess ? TPF_OK : TPF_E_CUDA;
}

// ------------------------------------------------------------ UP attention helpers
namespace tpf {
namespace {

// Row softmax (softmax_rows, tensor.cpp:123-143, max-subtracted) of scale * scores:
// fp32 (rows, cols) -> bf16 P. One CTA per row, three passes over the (L2-resident) row.
__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* __restrict__ s,
                                                           __nv_bfloat16* __restrict__ p,
                                                           int64_t cols, float scale_log2e) {
  __shared__ float red[32];
  const float* row = s + static_cast<int64_t>(blockIdx.x) * cols;
  __nv_bfloat16* out = p + static_cast<int64_t>(blockIdx.x) * cols;
  float mx = -INFINITY;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) mx = fmaxf(mx, row[c]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) sum += exp2f((row[c] - mx) * scale_log2e);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  sum = 0.f;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) sum += red[w];
  const float inv = 1.f / sum;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
    out[c] = __float2bfloat16_rn(exp2f((row[c] - mx) * scale_log2e) * inv);
}

// Wait until every flag[i] >= epoch (bounded; error record on timeout).
// Wait until every flags[i] >= epoch (bounded; error record + blame entry on give-up). Flag i
// was written by source rank (first + i) / per_src.
__device__ __forceinline__ void wait_flag_range(const uint32_t* flags, int64_t n, uint32_t epoch, int64_t timeout_ns,
                                                uint32_t* err, int rank, const Blame& blame, int64_t first,
                                                int64_t per_src) {
  const uint64_t t0 = globaltimer();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    while (ld_relaxed_sys(flags + i) < epoch) {
      const bool abort = ld_relaxed_sys(err + 4) != 0 ||
                         (blame.table[0] && ld_relaxed_sys(blame.table[rank] + kBlameAbort) == epoch);
      if (abort || globaltimer() - t0 > static_cast<uint64_t>(timeout_ns)) {
        if (!abort && atomicCAS(err, 0u, 1u) == 0u) {
          err[1] = static_cast<uint32_t>(rank);
          err[2] = 0xFFFFFFFFu;
          err[3] = static_cast<uint32_t>(i);
        }
        blame_store(blame.table, blame.T, rank, static_cast<int>((first + i) / per_src));
        if (!abort) group_abort_store(blame.table, blame.T, kBlameAbort, epoch);
        atomicExch(err + 4, 1u);
        return;
      }
      __nanosleep(64);
    }
    (void)ld_acquire_sys(flags + i);
  }
}

__global__ void wait_flags_kernel(const uint32_t* flags, int64_t n, uint32_t epoch, int64_t timeout_ns,
                                  uint32_t* err, int rank, const __grid_constant__ Blame blame, int64_t first,
                                  int64_t per_src) {
  wait_flag_range(flags, n, epoch, timeout_ns, err, rank, blame, first, per_src);
}

__global__ void wait_flags2_kernel(const uint32_t* flags0, const uint32_t* flags1, int64_t n,
                                   const uint32_t* epoch_dev, uint32_t epoch_static, int64_t timeout_ns,
                                   uint32_t* err, int rank, const __grid_constant__ Blame blame, int64_t first,
                                   int64_t per_src) {
  const uint32_t epoch = epoch_dev ? epoch_read(epoch_dev, 0) : epoch_static;
  const uint32_t* flags = (epoch_dev && (epoch & 1u)) ? flags1 : flags0;
  wait_flag_range(flags, n, epoch, timeout_ns, err, rank, blame, first, per_src);
}

__global__ void copy_by_parity_kernel(int4* dst, const int4* src0, const int4* src1, int64_t n,
                                      const uint32_t* epoch_dev) {
  const int4* src = (epoch_read(epoch_dev, 0) & 1u) ? src1 : src0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

void launch_wait_flags2(const uint32_t* flags0, const uint32_t* flags1, int64_t n, const uint32_t* epoch_dev,
                        uint32_t epoch, int64_t timeout_ns, uint32_t* err, int rank, const Blame& blame,
                        int64_t first, int64_t per_src, cudaStream_t st) {
  if (n <= 0) return;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, 64));
  wait_flags2_kernel<<<blocks, threads, 0, st>>>(flags0, flags1, n, epoch_dev, epoch, timeout_ns, err, rank, blame,
                                                 first, per_src > 0 ? per_src : 1);
}

void launch_copy_by_parity(void* dst, const void* src0, const void* src1, int64_t bytes, const uint32_t* epoch_dev,
                           cudaStream_t st) {
  const int64_t n = bytes / 16;
  if (n <= 0) return;
  const int threads = 512;
  const int blocks = static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, 4 * 148));
  copy_by_parity_kernel<<<blocks, threads, 0, st>>>(static_cast<int4*>(dst), static_cast<const int4*>(src0),
                                                    static_cast<const int4*>(src1), n, epoch_dev);
}

void launch_softmax(const float* s, void* p, int64_t rows, int64_t cols, float scale, cudaStream_t st) {
  softmax_rows_kernel<<<static_cast<unsigned>(rows), 256, 0, st>>>(s, static_cast<__nv_bfloat16*>(p), cols,
                                                                   scale * 1.4426950408889634f);
}

void launch_wait_flags(const uint32_t* flags, int64_t n, uint32_t epoch, int64_t timeout_ns, uint32_t* err,
                       int rank, const Blame& blame, int64_t first, int64_t per_src, cudaStream_t st) {
  if (n <= 0) return;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, 64));
  wait_flags_kernel<<<blocks, threads, 0, st>>>(flags, n, epoch, timeout_ns, err, rank, blame, first,
                                                per_src > 0 ? per_src : 1);
}

}  // namespace tpf
