// UP (Ulysses) attention with the output all-to-all fused: a persistent tcgen05 flash-
// attention forward kernel (non-causal, head_dim 128) whose epilogue pushes every O tile
// straight into the slice owner's buffer -- fuse_all_to_all_attention, Alg. 5,
// reference layers.cpp:174-218.
//
// One CTA per SM, 8 warps:
//   warp 0     TMA producer: Q tile (128 x 128) per work item, K/V tiles (128 x 128 each)
//              through a 2-stage ring
//   warp 1     tcgen05.mma issuer (cta_group::1): S = Q K^T into two ping-pong TMEM buffers
//              (look-ahead one tile), O += P V into a TMEM accumulator
//   warp 2     TMEM allocator
//   warps 4-7  softmax + epilogue, thread = query row: online softmax on S read from TMEM,
//              P written to SMEM as the SWIZZLE_128B K-major operand image, O rescaled in
//              TMEM only when a row max moved; finally O / l -> bf16 -> peer store + flag
// Work items (step i, head g, q-tile) run step-major, so the rank's own slice (step T-1)
// is computed last and no transfer trails it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tpf_internal.h"
#include "tpf_ptx.cuh"

namespace tpf {

namespace {

constexpr int kFTile = 128;                          // q rows / kv rows per tile, head_dim
constexpr int kFAtom = kFTile * 64 * 2;              // one 64-column SW128 atom: 16 KiB
constexpr int kFQBytes = 2 * kFAtom;                 // 32 KiB
constexpr int kFKVBytes = 4 * kFAtom;                // K + V: 64 KiB
constexpr int kFSmem = kFQBytes + 2 * kFKVBytes + kFQBytes /*P*/ + 1024 + 256;

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fmha_wait(const FmhaParams& p, uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait(bar, parity)) {
    if (globaltimer() - t0 > static_cast<uint64_t>(p.timeout_ns) * 2) {
      if (atomicCAS(p.err, 0u, 2u) == 0u) { p.err[1] = 0xFFFFFFFFu; }
      atomicExch(p.err + 4, 1u);
      return;
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(256, 1) tpf_fmha_a2a_kernel(const __grid_constant__ FmhaParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sq = smem;
  uint8_t* skv = smem + kFQBytes;
  uint8_t* sp = skv + 2 * kFKVBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp + kFQBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;    // [2]
  uint64_t* kv_empty = bars + 4;   // [2]
  uint64_t* s_full = bars + 6;     // [2]
  uint64_t* p_ready = bars + 8;
  uint64_t* pv_done = bars + 9;
  uint64_t* o_free = bars + 10;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x / p.ctas_per_rank;
  const int c = blockIdx.x - h * p.ctas_per_rank;
  if (h >= p.R) return;
  const int rank = p.rank0 + h;
  const int C = p.ctas_per_rank;
  const int per_step = p.G * p.nqt;
  const int nitems = p.T * per_step;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tmap_q);
    prefetch_tmap(&p.tmap_k);
    prefetch_tmap(&p.tmap_v);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(kv_full + s, 1);
      mbar_init(kv_empty + s, 1);
      mbar_init(s_full + s, 1);
    }
    mbar_init(p_ready, 4);
    mbar_init(pv_done, 1);
    mbar_init(o_free, 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t t_o = tmem + 2 * kFTile;

  if (warp == 0) {
    // =============================================================== TMA producer
    if (lane == 0) {
      uint32_t kvc = 0, ic = 0;
      for (int it = c; it < nitems; it += C, ++ic) {
        const int step = it / per_step, rem = it - step * per_step;
        const int g = rem / p.nqt, qt = rem - g * p.nqt;
        const int l = p.local ? 0 : (rank + step + 1) % p.T;
        const int row0 = static_cast<int>(static_cast<int64_t>(l) * p.sl + qt * kFTile);
        fmha_wait(p, q_empty, (ic & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, kFQBytes);
        tma_load_4d(sq, &p.tmap_q, q_full, 0, row0, g, h);
        tma_load_4d(sq + kFAtom, &p.tmap_q, q_full, 64, row0, g, h);
        for (int j = 0; j < p.nkv; ++j, ++kvc) {
          const int st = kvc & 1;
          fmha_wait(p, kv_empty + st, ((kvc >> 1) & 1) ^ 1);
          uint8_t* kv = skv + st * kFKVBytes;
          mbar_arrive_expect_tx(kv_full + st, kFKVBytes);
          tma_load_4d(kv, &p.tmap_k, kv_full + st, 0, j * kFTile, g, h);
          tma_load_4d(kv + kFAtom, &p.tmap_k, kv_full + st, 64, j * kFTile, g, h);
          tma_load_4d(kv + 2 * kFAtom, &p.tmap_v, kv_full + st, 0, j * kFTile, g, h);
          tma_load_4d(kv + 3 * kFAtom, &p.tmap_v, kv_full + st, 64, j * kFTile, g, h);
        }
      }
    }
  } else if (warp == 1) {
    // =============================================================== MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(kFTile, kFTile, /*b_mn_major=*/false);
      constexpr uint32_t idesc_o = make_idesc_bf16(kFTile, kFTile, /*b_mn_major=*/true);
      uint32_t kvc = 0, sc = 0, pc = 0, ic = 0;
      const uint32_t qa = smem_u32(sq);
      auto issue_s = [&](uint32_t kv_idx) {
        const int st = kv_idx & 1;
        fmha_wait(p, kv_full + st, (kv_idx >> 1) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(skv + st * kFKVBytes);
        const uint32_t d = tmem + (sc & 1) * kFTile;
#pragma unroll
        for (int k = 0; k < kFTile / 16; ++k) {
          const uint32_t off = (k >> 2) * kFAtom + (k & 3) * 32;
          mma_bf16(d, make_sdesc(qa + off, 0, 1024), make_sdesc(ka + off, 0, 1024), idesc_s, k > 0);
        }
        mma_commit(s_full + (sc & 1));
        ++sc;
      };
      for (int it = c; it < nitems; it += C, ++ic) {
        fmha_wait(p, q_full, ic & 1);
        tc_fence_after();
        issue_s(kvc);
        for (int j = 0; j < p.nkv; ++j) {
          if (j + 1 < p.nkv) issue_s(kvc + 1);  // look-ahead: overlaps softmax of tile j
          fmha_wait(p, p_ready, pc & 1);
          ++pc;
          if (j == 0) fmha_wait(p, o_free, (ic & 1) ^ 1);
          tc_fence_after();
          const int st = kvc & 1;
          const uint32_t va = smem_u32(skv + st * kFKVBytes + 2 * kFAtom);
          const uint32_t pa = smem_u32(sp);
#pragma unroll
          for (int k = 0; k < kFTile / 16; ++k) {
            // A = P (K-major over kv), B = V (MN-major: rows kv, 64-col atoms 16 KiB apart)
            const uint64_t ad = make_sdesc(pa + (k >> 2) * kFAtom + (k & 3) * 32, 0, 1024);
            const uint64_t bd = make_sdesc(va + k * 2048, kFAtom, 1024);
            mma_bf16(t_o, ad, bd, idesc_o, (j | k) != 0);
          }
          mma_commit(pv_done);
          mma_commit(kv_empty + st);
          ++kvc;
        }
        mma_commit(q_empty);
      }
    }
  } else if (warp >= 4) {
    // =============================================================== softmax + epilogue
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    uint32_t sc = 0, pvc = 0;
    for (int it = c; it < nitems; it += C) {
      const int step = it / per_step, rem = it - step * per_step;
      const int g = rem / p.nqt, qt = rem - g * p.nqt;
      const int dst = p.local ? rank : (rank + step + 1) % p.T;
      float m = -INFINITY, lsum = 0.f;
      for (int j = 0; j < p.nkv; ++j, ++sc) {
        fmha_wait(p, s_full + (sc & 1), (sc >> 1) & 1);
        tc_fence_after();
        uint32_t s[4][32];
        const uint32_t sa = tmem + lane_off + (sc & 1) * kFTile;
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld_32x32b_x32(sa + q * 32, s[q]);
        tmem_ld_wait();
        float mx = m;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(s[q][i]) * p.scale_log2);
        const float alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mx);
        float rs = 0.f;
        uint32_t pk[4][16];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a = fast_exp2(__uint_as_float(s[q][2 * i]) * p.scale_log2 - mx);
            const float b = fast_exp2(__uint_as_float(s[q][2 * i + 1]) * p.scale_log2 - mx);
            const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
            // normaliser from the bf16-rounded probabilities P.V actually uses
            const float2 f = __bfloat1622float2(v);
            rs += f.x + f.y;
            pk[q][i] = *reinterpret_cast<const uint32_t*>(&v);
          }
        lsum = lsum * alpha + rs;
        if (j > 0) {  // P.V of the previous tile done: P buffer and O are free
          fmha_wait(p, pv_done, pvc & 1);
          ++pvc;
          tc_fence_after();
        }
        // P row -> SMEM, SWIZZLE_128B K-major image: atom = kv / 64, 16 B chunk ^ (row & 7)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int chunk = (q & 1) * 4 + cc;  // 16 B chunk inside the 128 B atom row
            uint8_t* dstp = sp + (q >> 1) * kFAtom + row * 128 + ((chunk ^ (row & 7)) << 4);
            *reinterpret_cast<uint4*>(dstp) =
                make_uint4(pk[q][cc * 4], pk[q][cc * 4 + 1], pk[q][cc * 4 + 2], pk[q][cc * 4 + 3]);
          }
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          // online-softmax correction of the running O (only rows whose max moved change)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + lane_off + q * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(t_o + lane_off + q * 32, o);
          }
          tmem_st_wait();
        }
        m = mx;
        fence_proxy_async_smem();  // generic SMEM writes of P -> visible to the tensor core
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_ready);
      }
      // ---------------------------------------------------------------- epilogue
      fmha_wait(p, pv_done, pvc & 1);
      ++pvc;
      tc_fence_after();
      const float inv = 1.f / lsum;
      const int b = g / p.heads, hh = g - b * p.heads;
      char* orow = p.recv[dst] +
                   ((static_cast<int64_t>(b) * p.sl + qt * kFTile + row) * p.fw +
                    (static_cast<int64_t>(p.local ? 0 : rank) * p.heads + hh) * kFTile) * 2;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(t_o + lane_off + q * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(o[cc * 8 + 0]) * inv, __uint_as_float(o[cc * 8 + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(o[cc * 8 + 2]) * inv, __uint_as_float(o[cc * 8 + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(o[cc * 8 + 4]) * inv, __uint_as_float(o[cc * 8 + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(o[cc * 8 + 6]) * inv, __uint_as_float(o[cc * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + (q * 32 + cc * 8) * 2) = w;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
      if (dst != rank) {
        fence_sys();
        __syncwarp();
        if (lane == 0 && rank != p.fault_rank)
          st_relaxed_sys(p.flags[dst] + static_cast<int64_t>(rank) * p.nflags_per_src +
                             (static_cast<int64_t>(g) * p.nqt + qt) * 4 + ew,
                         p.epoch);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

void launch_fmha_a2a(const FmhaParams& p, int grid, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tpf_fmha_a2a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
    attr_set = true;
  }
  tpf_fmha_a2a_kernel<<<grid, 256, kFSmem, stream>>>(p);
}

}  // namespace tpf
