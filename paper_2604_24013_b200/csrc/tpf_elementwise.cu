// Element-wise glue of the TP-SP MLP block (tpsp_mlp_forward, layers.cpp:140-147):
// SwiGLU on the rank's [gate | up] column shard. HBM-bound: 16 B vector loads/stores,
// grid sized to a multiple of the SM count.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>

#include "tpf.h"
#include "tpf_host.h"
#include "tpf_internal.h"

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
