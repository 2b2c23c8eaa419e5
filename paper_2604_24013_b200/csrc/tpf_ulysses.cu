// Ulysses first all-to-all: Q/K/V go from the sequence-sharded
// layout (every head, one sequence slice per rank) to the head-sharded layout (one head
// group, the whole sequence), over NVLink peer stores.
//
// Reference: ref_all_to_all (fabric.cpp:183-207) applied to the per-group parts of
// layers_test.cpp:347-397 ("FullFlowFromSequenceShardedLayout"). Source rank r, head group g:
//   src row (b*H + g*hl + hh, s)  ->  rank g's row (b*hl + hh, r*sl + s),  s in [0, sl)
// For a fixed (tensor, b, g, hh) the source block (sl x Dh) and its destination block are both
// contiguous, so the copy is a list of 3*B*H contiguous blocks per source rank. The blocks are
// cut into 64 KiB pieces and the persistent grid strides over them with 16-byte loads and peer
// stores, destination-rotated (peer r+1 first) so every NVLink port is busy from the start.
// Each CTA then publishes one flag per (source rank, CTA) to every destination after a system
// fence; the receiver's wait kernel covers T * ctas flags.
#include <cuda_bf16.h>
#include <cstdint>

#include "tpf_internal.h"
#include "tpf_ptx.cuh"

namespace tpf {
namespace {

constexpr int kPushThreads = 512;
constexpr int kVec = 8;                                   // 16 B loads in flight per thread
constexpr int kPieceBytes = kPushThreads * kVec * 16;         // 64 KiB

__global__ void __launch_bounds__(kPushThreads) ulysses_push_kernel(UlyssesParams p) {
  const int hosted = blockIdx.x / p.ctas_per_rank;
  const int cta = blockIdx.x % p.ctas_per_rank;
  const int rank = p.rank0 + hosted;
  const int T = p.T;
  const int64_t block_bytes = p.sl * p.Dh * 2;
  const int64_t pieces_per_block = (block_bytes + kPieceBytes - 1) / kPieceBytes;
  const int64_t blocks_per_dst = 3 * p.B * p.hl;  // (tensor, b, hh) for one head group
  const int64_t total = static_cast<int64_t>(T) * blocks_per_dst * pieces_per_block;
  // this launch opens the call: epoch = device epoch + 1, heap parity = epoch & 1
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = epoch_read(p.epoch_dev, 1);
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const int par = static_cast<int>(epoch & 1u);
  for (int64_t w = cta; w < total; w += p.ctas_per_rank) {
    const int64_t piece = w % pieces_per_block;
    int64_t rest = w / pieces_per_block;
    const int64_t hh = rest % p.hl;
    rest /= p.hl;
    const int64_t b = rest % p.B;
    rest /= p.B;
    const int tensor = static_cast<int>(rest % 3);
    const int g = static_cast<int>((rank + 1 + rest / 3) % T);  // rotated destination
    const char* src = p.src[tensor] + hosted * p.src_rank_stride +
                      ((b * p.H + g * p.hl + hh) * p.sl) * p.Dh * 2 + piece * kPieceBytes;
    char* dst = p.dst[par][g] + tensor * p.tensor_bytes + ((b * p.hl + hh) * p.S + rank * p.sl) * p.Dh * 2 +
                piece * kPieceBytes;
    const int64_t n = min(static_cast<int64_t>(kPieceBytes), block_bytes - piece * kPieceBytes) / 16;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    int4* d4 = reinterpret_cast<int4*>(dst);
    if (n == kPushThreads * kVec) {
      // all loads first (kVec independent 16 B loads per thread), then the peer stores
      int4 v[kVec];
#pragma unroll
      for (int u = 0; u < kVec; ++u) v[u] = __ldg(s4 + u * kPushThreads + threadIdx.x);
#pragma unroll
      for (int u = 0; u < kVec; ++u) d4[u * kPushThreads + threadIdx.x] = v[u];
    } else {
      for (int64_t i = threadIdx.x; i < n; i += kPushThreads) d4[i] = __ldg(s4 + i);
    }
  }
  __syncthreads();
  if (threadIdx.x < T && rank != p.fault_rank) {
    __threadfence_system();
    st_relaxed_sys(p.flags[par][threadIdx.x] + static_cast<int64_t>(rank) * p.ctas_per_rank + cta, epoch);
  }
  if (threadIdx.x == 0) epoch_publish(p.epoch_dev, epoch, gridDim.x);
}

}  // namespace

void launch_ulysses_push(const UlyssesParams& p, cudaStream_t stream) {
  ulysses_push_kernel<<<p.ctas_per_rank * p.R, kPushThreads, 0, stream>>>(p);
}

}  // namespace tpf
