// UP (Ulysses) attention with the output all-to-all fused: a persistent tcgen05 flash-
// attention forward kernel (non-causal, head_dim 128) whose epilogue pushes every O tile
// straight into the slice owner's buffer -- fuse_all_to_all_attention, Alg. 5,
// reference layers.cpp:174-218.
//
// One CTA per SM, 12 warps; a work item is a PAIR of 128-row query tiles of one head, so two
// softmax warpgroups ping-pong against the tensor core:
//   warp 0      TMA producer: Q0 | Q1 (2 x 128 x 128) per item, then K_j, V_j through a
//               5-slot ring of 32 KiB tiles
//   warp 1      tcgen05.mma issuer (cta_group::1), per kv block j:
//                 PV0_{j-1}, S0_j = Q0 K_j^T, PV1_{j-1}, S1_j = Q1 K_j^T
//               so softmax 0 works on S0_j while the tensor core runs PV1 / S1 and vice versa
//   warp 2      TMEM allocator (S0 | S1 | O0 | O1: 4 x 128 fp32 columns)
//   warps 4-7   softmax + epilogue of tile 0, thread = query row
//   warps 8-11  softmax + epilogue of tile 1
// Softmax: S row from TMEM, online max/sum (exp2 with the scale folded into one FFMA2, part
// of the exps on the FMA pipe), P written back over S in TMEM as packed bf16 (the A operand
// of the TS-form P.V MMA), O rescaled in TMEM only when a row max jumped past a threshold. Every ordering hazard is covered by MMA issue order: S_w(j+1) is
// issued after PV_w(j), which waits for P_w(j), so one s_full arrival means "S_w(j+1) ready,
// and P_w / O_w free". Epilogue: O / l -> bf16 -> peer store + flag.
// Work items (step i, head g, q-tile pair) run step-major, so the rank's own slice (step
// T-1) is computed last and no transfer trails it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <mutex>

#include "tpf_internal.h"
#include "tpf_ptx.cuh"

namespace tpf {

namespace {

constexpr int kFTile = 128;                          // q rows / kv rows per tile, head_dim
constexpr int kFAtom = kFTile * 64 * 2;              // one 64-column SW128 atom: 16 KiB
constexpr int kFTileBytes = 2 * kFAtom;              // one 128 x 128 bf16 tile: 32 KiB
constexpr int kFRing = 5;                            // K/V ring slots
constexpr int kFSmem = (2 + kFRing) * kFTileBytes + 1024 + 256;  // Q0 Q1 | ring

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 helpers (FFMA2 / FADD2 on sm_100a).
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2_split(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair of x <= 0 on the FMA pipe (offloads the MUFU unit): x = j + f with j the
// nearest integer (1.5 * 2^23 rounding trick), 2^f by a degree-3 minimax polynomial on
// [-0.5, 0.5] (max rel. error 7.5e-5, far below the bf16 rounding of P), 2^j added into the
// exponent field. x is clamped at -127, where the result is below bf16's smallest normal.
__device__ __forceinline__ float2 exp2_poly2(float x0, float x1) {
  const uint64_t x = f2(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
  const uint64_t t = f2_add(x, f2(12582912.f, 12582912.f));
  const uint64_t j = f2_add(t, f2(-12582912.f, -12582912.f));
  const uint64_t fr = f2_fma(j, f2(-1.f, -1.f), x);
  uint64_t pp = f2_fma(fr, f2(0.0551716685f, 0.0551716685f), f2(0.242611155f, 0.242611155f));
  pp = f2_fma(pp, fr, f2(0.693260968f, 0.693260968f));
  pp = f2_fma(pp, fr, f2(0.999928057f, 0.999928057f));
  const float2 pv = f2_split(pp), tv = f2_split(t);
  return make_float2(__int_as_float(__float_as_int(pv.x) + (__float_as_int(tv.x) << 23)),
                     __int_as_float(__float_as_int(pv.y) + (__float_as_int(tv.y) << 23)));
}

// Exps per 8-element P chunk computed on the FMA pipe instead of MUFU (pairs, 0..4).
#ifndef TPF_POLY_PAIRS
#define TPF_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = TPF_POLY_PAIRS;
// Keep a stale running max until the new one exceeds it by this much (log2 units): exps stay
// <= 2^8 and O is rescaled only on a large jump, never on the small moves of later blocks.
constexpr float kRescaleThreshold = 8.0f;

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

// kQSplit: query-split instance (slice order from the RS schedule, per-slice ready counters);
// a compile-time switch so the UP / plain instance carries none of its code.
template <bool kQSplit>
__global__ void __launch_bounds__(384, 1) tpf_fmha_a2a_kernel(const __grid_constant__ FmhaParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sq = smem;                                  // Q0, Q1
  uint8_t* ring = smem + 2 * kFTileBytes;              // kFRing x 32 KiB
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kFRing * kFTileBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* r_full = bars + 2;             // [kFRing]
  uint64_t* r_empty = bars + 2 + kFRing;   // [kFRing]
  uint64_t* s_full = bars + 2 + 2 * kFRing;   // [2]
  uint64_t* p_ready = s_full + 2;             // [2]
  uint64_t* pv_done = s_full + 4;             // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_full + 6);

  // warp index through a shuffle so ptxas treats it (and the role branches) as warp-uniform
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int h = blockIdx.x / p.ctas_per_rank;
  const int c = blockIdx.x - h * p.ctas_per_rank;
  if (h >= p.R) return;
  const int rank = p.rank0 + h;
  const int C = p.ctas_per_rank;
  const int npair = (p.nqt + 1) >> 1;
  const int per_step = p.G * npair;
  const int nitems = p.T * per_step;

  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = p.epoch_dev ? epoch_read(p.epoch_dev, p.epoch_bump) : p.epoch;
  if (warp == 0 && lane == 0) {
    for (int par = 0; par < 2; ++par) {
      prefetch_tmap(&p.tmap_q[par]);
      prefetch_tmap(&p.tmap_k[par]);
      prefetch_tmap(&p.tmap_v[par]);
    }
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kFRing; ++s) {
      mbar_init(r_full + s, 1);
      mbar_init(r_empty + s, 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(s_full + w, 1);
      mbar_init(p_ready + w, 4);
      mbar_init(pv_done + w, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;  // S0 @ 0, S1 @ 128, O0 @ 256, O1 @ 384
  const uint32_t epoch = s_epoch;
  const int par = p.epoch_dev ? static_cast<int>(epoch & 1u) : p.parity;
  const CUtensorMap* tmq = &p.tmap_q[par];
  const CUtensorMap* tmk = &p.tmap_k[par];
  const CUtensorMap* tmv = &p.tmap_v[par];
  // Register split: warps 0-3 (TMA, MMA, TMEM) need few, the softmax warpgroups hold a whole
  // 128-wide S row: 72 * 128 + 216 * 256 = 168 * 384, exactly the pool the CTA launched with.
  // setmaxnreg.inc blocks until the pool can satisfy it, so the sum must not exceed the pool
  // (checked at launch). Each warpgroup executes one setmaxnreg at the top of its branch, so
  // ptxas allocates the branch under that limit.

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
  if (warp == 0) {
    // =============================================================== TMA producer
    if (lane == 0) {
      uint32_t rc = 0, ic = 0;
      for (int it = c; it < nitems; it += C, ++ic) {
        const int step = it / per_step, rem = it - step * per_step;
        const int g = rem / npair, pr = rem - g * npair;
        // query slice of this step: UP sends slice (r+i+1) % T; query-split follows the RS
        // schedule's slice order; plain local attention has a single slice
        const int l = kQSplit ? p.slice_of[h][step] : p.local ? 0 : (rank + step + 1) % p.T;
        const int row0 = static_cast<int>(static_cast<int64_t>(l) * p.sl + pr * 2 * kFTile);
        fmha_wait(p, q_empty, (ic & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, 2 * kFTileBytes);
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          tma_load_4d(sq + w * kFTileBytes, tmq, q_full, 0, row0 + w * kFTile, g, h);
          tma_load_4d(sq + w * kFTileBytes + kFAtom, tmq, q_full, 64, row0 + w * kFTile, g, h);
        }
        for (int j = 0; j < p.nkv; ++j) {
#pragma unroll
          for (int kv = 0; kv < 2; ++kv, ++rc) {  // K_j then V_j
            const int slot = rc % kFRing;
            fmha_wait(p, r_empty + slot, ((rc / kFRing) & 1) ^ 1);
            uint8_t* dst = ring + slot * kFTileBytes;
            const CUtensorMap* tm = kv ? tmv : tmk;
            mbar_arrive_expect_tx(r_full + slot, kFTileBytes);
            tma_load_4d(dst, tm, r_full + slot, 0, j * kFTile, g, h);
            tma_load_4d(dst + kFAtom, tm, r_full + slot, 64, j * kFTile, g, h);
          }
        }
      }
    }
  } else if (warp == 1) {
    // =============================================================== MMA issuer
    {  // the whole warp runs the loop (uniform values); elect.sync issues
      constexpr uint32_t idesc_s = make_idesc_bf16(kFTile, kFTile, /*b_mn_major=*/false);
      constexpr uint32_t idesc_o = make_idesc_bf16(kFTile, kFTile, /*b_mn_major=*/true);
      uint32_t rc = 0, ic = 0, pc = 0;
      const uint32_t qa = smem_u32(sq);
      auto ring_wait = [&](uint32_t idx) {
        fmha_wait(p, r_full + idx % kFRing, (idx / kFRing) & 1);
        tc_fence_after();
        return smem_u32(ring + (idx % kFRing) * kFTileBytes);
      };
      auto issue_s = [&](int w, uint32_t ka) {
        const uint32_t q = qa + w * kFTileBytes;
#pragma unroll
        for (int k = 0; k < kFTile / 16; ++k) {
          const uint32_t off = (k >> 2) * kFAtom + (k & 3) * 32;
          mma_bf16_warp(tmem + w * kFTile, make_sdesc(q + off, 0, 1024), make_sdesc(ka + off, 0, 1024), idesc_s, k > 0);
        }
        mma_commit_warp(s_full + w);
      };
      auto issue_pv = [&](int w, uint32_t va, bool acc) {
#pragma unroll
        for (int k = 0; k < kFTile / 16; ++k) {
          // A = P from TMEM (S_w's first 64 columns, 16 kv per 8 columns), B = V (MN-major:
          // rows kv, 64-col atoms 16 KiB apart)
          const uint64_t bd = make_sdesc(va + k * 2048, kFAtom, 1024);
          mma_bf16_ts_warp(tmem + (2 + w) * kFTile, tmem + w * kFTile + k * 8, bd, idesc_o, acc || k > 0);
        }
      };
      for (int it = c; it < nitems; it += C, ++ic) {
        fmha_wait(p, q_full, ic & 1);
        tc_fence_after();
        const uint32_t base = rc;
        {
          const uint32_t ka = ring_wait(base);
          issue_s(0, ka);
          issue_s(1, ka);
          mma_commit_warp(r_empty + base % kFRing);
          if (p.nkv == 1) mma_commit_warp(q_empty);
        }
        for (int j = 0; j < p.nkv; ++j) {
          const bool more = j + 1 < p.nkv;
          const uint32_t vidx = base + 2 * j + 1, kidx = base + 2 * j + 2;
          const uint32_t va = ring_wait(vidx);
          fmha_wait(p, p_ready + 0, pc & 1);
          tc_fence_after();
          issue_pv(0, va, j > 0);
          if (!more) mma_commit_warp(pv_done + 0);
          uint32_t ka = 0;
          if (more) {
            ka = ring_wait(kidx);
            issue_s(0, ka);
          }
          fmha_wait(p, p_ready + 1, pc & 1);
          ++pc;
          tc_fence_after();
          issue_pv(1, va, j > 0);
          mma_commit_warp(r_empty + vidx % kFRing);
          if (!more) mma_commit_warp(pv_done + 1);
          if (more) {
            issue_s(1, ka);
            mma_commit_warp(r_empty + kidx % kFRing);
            if (j + 2 == p.nkv) mma_commit_warp(q_empty);
          }
        }
        rc = base + 2 * p.nkv;
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
    // =============================================================== softmax + epilogue
    const int w = (warp - 4) >> 2;          // query tile of the pair
    const int ew = warp & 3;                // TMEM lane quarter
    const int row = ew * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const uint32_t t_s = tmem + lane_off + w * kFTile;
    const uint32_t t_o = tmem + lane_off + (2 + w) * kFTile;
    const float scale = p.scale_log2;
    uint32_t sc = 0, ic = 0;
    for (int it = c; it < nitems; it += C, ++ic) {
      const int step = it / per_step, rem = it - step * per_step;
      const int g = rem / npair, pr = rem - g * npair;
      const int qt = pr * 2 + w;
      const int dst = p.local ? rank : (rank + step + 1) % p.T;
      const int l = kQSplit ? p.slice_of[h][step] : 0;
      float m = -INFINITY, lsum = 0.f;
      for (int j = 0; j < p.nkv; ++j, ++sc) {
        fmha_wait(p, s_full + w, sc & 1);
        tc_fence_after();
        // The whole S row in registers (the softmax warpgroups run with 216 registers), one
        // TMEM round trip; the row max as a tree of 8 independent FMNMX3 chains.
        uint32_t s[4][32];
#ifdef TPF_FMHA_EXPERIMENT_NO_LD  // dev experiment: softmax without the TMEM read
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int i = 0; i < 32; ++i) s[q][i] = __float_as_uint(static_cast<float>(i));
#else
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld_32x32b_x32(t_s + q * 32, s[q]);
        tmem_ld_wait();
#endif
        float mxp[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) mxp[t] = fmaxf(__uint_as_float(s[t >> 1][(t & 1) * 16]), m);
#pragma unroll
        for (int t = 0; t < 8; ++t)
#pragma unroll
          for (int i = 1; i < 16; i += 2)
            mxp[t] = fmax3(mxp[t], __uint_as_float(s[t >> 1][(t & 1) * 16 + i]),
                           __uint_as_float(s[t >> 1][(t & 1) * 16 + ((i + 1) & 15)]));
        const float mx = fmaxf(fmax3(fmax3(mxp[0], mxp[1], mxp[2]), fmax3(mxp[3], mxp[4], mxp[5]), mxp[6]), mxp[7]);
        // Raw-score max (scale > 0). Keep the stale max unless it grew past the threshold.
        const bool moved = m == -INFINITY || (mx - m) * scale > kRescaleThreshold;
        const float mu = moved ? mx : m;
        const float alpha = (m == -INFINITY) ? 0.f : (moved ? fast_exp2((m - mx) * scale) : 1.f);
        const uint64_t sc2 = f2(scale, scale), neg2 = f2(-mu * scale, -mu * scale);
        uint64_t rs2a = f2(0.f, 0.f), rs2b = f2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t pq[16];  // 32 probabilities of this chunk, bf16x2 = 16 TMEM columns
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = cc * 8 + 2 * e;
              // exp2(s * scale - mu * scale), one FFMA2 per pair
              const float2 x = f2_split(f2_fma(f2(__uint_as_float(s[q][i]), __uint_as_float(s[q][i + 1])), sc2, neg2));
              float2 y;
#ifdef TPF_FMHA_EXPERIMENT_NO_EXP  // dev experiment: softmax without the exponentials
              if (true) {
                y = x;
              } else
#endif
              if (e >= 4 - kPolyPairs) {
                y = exp2_poly2(x.x, x.y);
              } else {
                y.x = fast_exp2(x.x);
                y.y = fast_exp2(x.y);
              }
              if (e & 1) rs2b = f2_add(rs2b, f2(y.x, y.y));
              else rs2a = f2_add(rs2a, f2(y.x, y.y));
              pq[cc * 4 + e] = pack_bf16x2(y.x, y.y);
            }
          }
          // P overwrites S_w in place (columns q*16 .. q*16+15: already read into registers);
          // S_w(j+1) is issued only after PV_w(j) has consumed it
          tmem_st_32x32b_x16(t_s + q * 16, pq);
        }
        const float2 ra = f2_split(rs2a), rb = f2_split(rs2b);
        const float rs = (ra.x + ra.y) + (rb.x + rb.y);
        lsum = lsum * alpha + rs;
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          // online-softmax correction of the running O (PV_w(j-1) is complete: S_w(j) was
          // issued after it)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + q * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(t_o + q * 32, o);
          }
          tmem_st_wait();
        }
        m = mu;
        tmem_st_wait();  // P in TMEM before the tensor core may read it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_ready + w);
      }
      // ---------------------------------------------------------------- epilogue
      fmha_wait(p, pv_done + w, ic & 1);
      tc_fence_after();
      if (qt < p.nqt) {
        const float inv = 1.f / lsum;
        const int b = g / p.heads, hh = g - b * p.heads;
        char* orow = p.recv[par][dst] +
                     ((static_cast<int64_t>(b) * (kQSplit ? p.S : p.sl) + (kQSplit ? l * p.sl : 0) +
                       qt * kFTile + row) * p.fw +
                      (static_cast<int64_t>(p.local ? 0 : rank) * p.heads + hh) * kFTile) * 2;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(t_o + q * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(o[cc * 8 + 0]) * inv, __uint_as_float(o[cc * 8 + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(o[cc * 8 + 2]) * inv, __uint_as_float(o[cc * 8 + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(o[cc * 8 + 4]) * inv, __uint_as_float(o[cc * 8 + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(o[cc * 8 + 6]) * inv, __uint_as_float(o[cc * 8 + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + (q * 32 + cc * 8) * 2) = v;
          }
        }
        if (dst != rank) {
          fence_sys();
          __syncwarp();
          if (lane == 0 && rank != p.fault_rank)
            st_relaxed_sys(p.flags[par][dst] + static_cast<int64_t>(rank) * p.nflags_per_src +
                               (static_cast<int64_t>(g) * p.nqt + qt) * 4 + ew,
                           epoch);
        }
      }
      if (kQSplit) {
        // query-split: this warp's 32 context rows of slice l are stored; the concurrently
        // running GEMM-RS waits for all of the slice's warps (phantom tiles count too)
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.qs_ready[h] + l, 1u);
      }
      // O_w is read (tcgen05.ld waited) before this warp's next p_ready arrival, and PV_w(0)
      // of the next item is issued only after that arrival.
      tc_fence_before();
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0 && p.epoch_dev && p.epoch_bump) epoch_publish(p.epoch_dev, epoch, gridDim.x);
}

template <bool kQSplit>
cudaError_t launch_fmha_instance(const FmhaParams& p, int grid, cudaStream_t stream) {
  // function attributes are per device: set once per device, thread-safe
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!((done >> dev) & 1ull)) {
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, tpf_fmha_a2a_kernel<kQSplit>);
      if (e != cudaSuccess) return e;
      // the setmaxnreg split above must fit the pool the launch allocates, or the kernel hangs
      if (fa.numRegs * 384 < 72 * 128 + 216 * 256) return cudaErrorInvalidConfiguration;
      e = cudaFuncSetAttribute(tpf_fmha_a2a_kernel<kQSplit>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem);
      if (e != cudaSuccess) return e;
      done |= 1ull << dev;
    }
  }
  tpf_fmha_a2a_kernel<kQSplit><<<grid, 384, kFSmem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fmha_a2a(const FmhaParams& p, int grid, cudaStream_t stream) {
  return p.qsplit ? launch_fmha_instance<true>(p, grid, stream) : launch_fmha_instance<false>(p, grid, stream);
}

}  // namespace tpf
