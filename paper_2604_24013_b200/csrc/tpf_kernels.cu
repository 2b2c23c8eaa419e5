// Persistent, warp-specialised sm_100a kernel family for the CommFuse hot path:
//
//   OP_RS  GEMM + decomposed reduce-scatter (fuse_reduce_scatter + row_parallel_forward,
//          reference collectives.cpp:285-405, layers.cpp:129-138). With T == 1 it is the
//          plain GEMM (collectives.cpp:379).
//   OP_AG  decomposed all-gather + GEMM (fuse_all_gather + column_parallel_forward,
//          reference collectives.cpp:237-279, layers.cpp:120-127).
//
// CTA pairs (cluster of 2, tcgen05 cta_group::2), one CTA per SM, 12 warps each:
//   warp 0      TMA producer: this CTA's 128-row A block (tensor map or AG wire image)
//               and its half of the 256-column B tile; completion lands on the leader's
//               full barrier
//   warp 1      (leader CTA only) tcgen05.mma.cta_group::2, 256x256x16 bf16 -> fp32, two
//               TMEM accumulators; commits multicast to both CTAs' barriers
//   warps 2-3   TMEM allocator (warp 2); AG ring forwarders: copy a share of every step's
//               wire images from global memory (x at step 0, the inbox after its flag
//               later) to the successor's slot over NVLink, independent of the GEMM
//   warps 4-11  two epilogue warpgroups, one per TMEM accumulator: tcgen05.ld of this
//               CTA's 128 rows -> (+ inbox) -> peer / output
// Work is a static, iteration-major tile list (step = pass * T + iteration), so every
// cross-rank dependency points to an earlier step and the persistent grid always makes
// progress. Wire formats are chosen so the consumer does no re-layout:
//   RS wire  = the TMEM 32x32b fragment image (thread-row interleaved by 16 B column
//              groups), so each warp-wide 16 B store/load touches 512 contiguous bytes;
//   AG wire  = the SWIZZLE_128B K-major UMMA operand image of a 128x64 A tile (16 KiB):
//              exactly the bytes of a pipeline stage, so the receiver TMA-loads it
//              straight into a stage and forwarding it onwards is a verbatim copy.
// Flags carry the per-call epoch (monotonic, never reset); slots are double-buffered by
// epoch parity. Every spin is bounded by a %globaltimer deadline and reports into a
// device error record instead of trapping.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "tpf_internal.h"
#include "tpf_ptx.cuh"

namespace tpf {

namespace {

// This launch's epoch / heap parity (from the device epoch when the call is multi-rank).
__shared__ uint32_t s_epoch;
__shared__ int s_parity;

struct Tile {
  int step, mb, nt, b, row0, valid;  // mb: THIS CTA's m-block; valid rows (0: dummy CTA)
  int pair;                          // m-block pair index within the step
};

// Pair-tile raster: step-major; inside a step, group_m m-block pairs sweep the n-tiles.
// With group_n > 0 the roles swap: group_n n-tiles are swept by all m-block pairs (keeps a
// slab of B L2-resident while A streams; narrow-N, long-K shapes).
__device__ __forceinline__ Tile get_tile(const KParams& p, int lin, int cta) {
  const int per_step = p.npairs * p.nnt;
  Tile t;
  t.step = lin / per_step;
  const int rem = lin - t.step * per_step;
  if (p.group_n > 0) {
    const int GN = p.group_n;
    const int g0 = (rem / (GN * p.npairs)) * GN;
    const int gn = min(GN, p.nnt - g0);
    const int r2 = rem - g0 * p.npairs;
    t.nt = g0 + r2 % gn;
    t.pair = r2 / gn;
  } else {
    const int GM = p.group_m;
    const int g0 = (rem / (GM * p.nnt)) * GM;
    const int gm = min(GM, p.npairs - g0);
    const int r2 = rem - g0 * p.nnt;
    // Pairs never straddle a batch: the pair shares one B tile (cta_group::2), and with a
    // per-batch B (attention heads) both CTAs must be in the same batch.
    t.pair = g0 + r2 % gm;
    t.nt = r2 / gm;
  }
  const int ppb = (p.nmb_per_batch + 1) / 2;
  t.b = t.pair / ppb;
  const int j = 2 * (t.pair - t.b * ppb) + cta;
  t.mb = t.b * p.nmb_per_batch + j;
  if (j >= p.nmb_per_batch) {
    t.row0 = 0; t.valid = 0;
    return t;
  }
  t.row0 = j * BM;
  t.valid = static_cast<int>(min(static_cast<int64_t>(BM), p.Sc - t.row0));
  return t;
}

__device__ __forceinline__ void trace_rec(const KParams& p, int kind, int rank, int step,
                                          int64_t index, uint64_t t0, uint64_t t1) {
  if (!p.trace) return;
  const unsigned long long slot = atomicAdd(p.trace, 1ull);
  if (static_cast<int64_t>(slot) >= p.trace_cap) return;
  unsigned long long* r = p.trace + 4 * (slot + 1);
  r[0] = static_cast<unsigned long long>(kind) | (static_cast<unsigned long long>(rank & 0xFF) << 8) |
         (static_cast<unsigned long long>(blockIdx.x & 0xFFFF) << 16) |
         (static_cast<unsigned long long>(static_cast<uint32_t>(step)) << 32);
  r[1] = static_cast<unsigned long long>(index);
  r[2] = t0;
  r[3] = t1;
}

// This launch's error record says abort, or any rank of the group has set the group abort flag
// in this rank's blame table (tpf::kBlameAbort).
__device__ __forceinline__ bool aborted(const KParams& p, int rank, uint32_t epoch) {
  if (ld_relaxed_sys(p.err + 4) != 0) return true;
  return p.blame.table[0] != nullptr && ld_relaxed_sys(p.blame.table[rank] + kBlameAbort) == epoch;
}

__device__ __noinline__ void record_error(const KParams& p, uint32_t code, int rank, int step,
                                          int tile) {
  if (atomicCAS(p.err, 0u, code) == 0u) {
    p.err[1] = static_cast<uint32_t>(rank);
    p.err[2] = static_cast<uint32_t>(step);
    p.err[3] = static_cast<uint32_t>(tile);
  }
  atomicExch(p.err + 4, 1u);
}

// A waiter gives up on rank `awaited`: blame entry for the failing-rank chain (tpf::Blame).
__device__ __noinline__ void give_up(const KParams& p, bool timed_out, int rank, int awaited, int step, int tile,
                                     uint32_t epoch) {
  if (timed_out) record_error(p, 1, rank, step, tile);
  blame_store(p.blame.table, p.blame.T, rank, awaited);
  if (timed_out) group_abort_store(p.blame.table, p.blame.T, kBlameAbort, epoch);
}

// Bounded spin on a flag written by rank `awaited` (value >= epoch). Returns with acquire
// semantics; on timeout / abort returns false (the kernel then drains with garbage
// and the host raises from the error record).
__device__ __forceinline__ bool wait_flag(const KParams& p, const uint32_t* f, int rank, int awaited,
                                          int step, int tile, uint32_t epoch) {
  if (ld_relaxed_sys(f) >= epoch) {
    (void)ld_acquire_sys(f);
    return true;
  }
  const uint64_t t0 = globaltimer();
  while (true) {
#pragma unroll 1
    for (int k = 0; k < 256; ++k) {
      if (ld_relaxed_sys(f) >= epoch) {
        (void)ld_acquire_sys(f);
        return true;
      }
      __nanosleep(32);
    }
    const bool timed_out = globaltimer() - t0 > static_cast<uint64_t>(p.timeout_ns);
    if (aborted(p, rank, epoch) || timed_out) {
      give_up(p, timed_out && !aborted(p, rank, epoch), rank, awaited, step, tile, epoch);
      return false;
    }
  }
}

__device__ __forceinline__ void mbar_wait(const KParams& p, uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait(bar, parity)) {
    if (globaltimer() - t0 > static_cast<uint64_t>(p.timeout_ns) * 2) {
      record_error(p, 2, -1, -1, -1);
      return;
    }
  }
}

__device__ __forceinline__ char* slot_ptr(const KParams& p, int par, int rank, int slot) {
  return p.sym[rank] + p.data_off[par] + static_cast<int64_t>(slot) * p.slot_bytes;
}

__device__ __forceinline__ uint32_t* flag_ptr(const KParams& p, int par, int rank, int slot,
                                              int64_t idx) {
  return reinterpret_cast<uint32_t*>(p.sym[rank] + p.flag_off[par]) +
         static_cast<int64_t>(slot) * p.flags_per_slot + idx;
}

// Store 32 fp32 accumulator columns of one row to a row-major output.
__device__ __forceinline__ void store_out_row(const KParams& p, char* row_ptr, int64_t col0,
                                              const float (&v)[32]) {
  if (p.out_f32) {
#pragma unroll
    for (int g = 0; g < 8; ++g)
      if (col0 + g * 4 < p.N)
        *reinterpret_cast<float4*>(row_ptr + (col0 + g * 4) * 4) =
            make_float4(v[g * 4], v[g * 4 + 1], v[g * 4 + 2], v[g * 4 + 3]);
  } else {
#pragma unroll
    for (int g = 0; g < 4; ++g)
      if (col0 + g * 8 < p.N) {
        uint4 w;
        w.x = pack_bf16x2(v[g * 8 + 0], v[g * 8 + 1]);
        w.y = pack_bf16x2(v[g * 8 + 2], v[g * 8 + 3]);
        w.z = pack_bf16x2(v[g * 8 + 4], v[g * 8 + 5]);
        w.w = pack_bf16x2(v[g * 8 + 6], v[g * 8 + 7]);
        *reinterpret_cast<uint4*>(row_ptr + (col0 + g * 8) * 2) = w;
      }
  }
}

// RS wire (TMEM-fragment image): sub-chunk j (32 columns), 16 B column group g, row.
__device__ __forceinline__ int64_t wire_off(int wire_f32, int j, int g, int row) {
  const int G = wire_f32 ? 8 : 4;
  return (static_cast<int64_t>(j * G + g) * BM + row) * 16;
}

__device__ __forceinline__ void wire_store(int wire_f32, char* tile, int j, int row,
                                           const float (&v)[32]) {
  if (wire_f32) {
#pragma unroll
    for (int g = 0; g < 8; ++g)
      *reinterpret_cast<float4*>(tile + wire_off(1, j, g, row)) =
          make_float4(v[g * 4], v[g * 4 + 1], v[g * 4 + 2], v[g * 4 + 3]);
  } else {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint4 w;
      w.x = pack_bf16x2(v[g * 8 + 0], v[g * 8 + 1]);
      w.y = pack_bf16x2(v[g * 8 + 2], v[g * 8 + 3]);
      w.z = pack_bf16x2(v[g * 8 + 4], v[g * 8 + 5]);
      w.w = pack_bf16x2(v[g * 8 + 6], v[g * 8 + 7]);
      *reinterpret_cast<uint4*>(tile + wire_off(0, j, g, row)) = w;
    }
  }
}

// rs_direct fold of one 32-column sub-chunk, 8 columns at a time: all T-1 received
// contributions are loaded first (memory-level parallelism), then summed in the
// reference order ((c[p0] + c[p1]) + ... + c[p(T-2)]) + own.
__device__ __forceinline__ void direct_fold(const KParams& p, const char* slot0, int j, int row,
                                            float (&v)[32]) {
  const int64_t slot_stride = p.slot_bytes;
  const int nin = p.T - 1;
#pragma unroll
  for (int qt = 0; qt < 4; ++qt) {
    uint4 raw[kMaxRanks - 1][2];
#pragma unroll
    for (int s = 0; s < kMaxRanks - 1; ++s) {
      if (s < nin) {
        const char* tile = slot0 + s * slot_stride;
        if (p.wire_f32) {
          raw[s][0] = *reinterpret_cast<const uint4*>(tile + wire_off(1, j, qt * 2, row));
          raw[s][1] = *reinterpret_cast<const uint4*>(tile + wire_off(1, j, qt * 2 + 1, row));
        } else {
          raw[s][0] = *reinterpret_cast<const uint4*>(tile + wire_off(0, j, qt, row));
        }
      }
    }
    float acc[8];
#pragma unroll
    for (int s = 0; s < kMaxRanks - 1; ++s) {
      if (s < nin) {
        float in[8];
        if (p.wire_f32) {
          in[0] = __uint_as_float(raw[s][0].x); in[1] = __uint_as_float(raw[s][0].y);
          in[2] = __uint_as_float(raw[s][0].z); in[3] = __uint_as_float(raw[s][0].w);
          in[4] = __uint_as_float(raw[s][1].x); in[5] = __uint_as_float(raw[s][1].y);
          in[6] = __uint_as_float(raw[s][1].z); in[7] = __uint_as_float(raw[s][1].w);
        } else {
          in[0] = bf16lo(raw[s][0].x); in[1] = bf16hi(raw[s][0].x);
          in[2] = bf16lo(raw[s][0].y); in[3] = bf16hi(raw[s][0].y);
          in[4] = bf16lo(raw[s][0].z); in[5] = bf16hi(raw[s][0].z);
          in[6] = bf16lo(raw[s][0].w); in[7] = bf16hi(raw[s][0].w);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = s == 0 ? in[c] : acc[c] + in[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) v[qt * 8 + c] = acc[c] + v[qt * 8 + c];
  }
}

}  // namespace

// rs_direct last step: fold the T-1 received partials into the own one, sub-chunk by
// sub-chunk. Inlined: with the epilogue warpgroups at 208 registers it fits without spills,
// and the ABI call of a non-inlined version cost 11% on the per-GPU pairwise GEMM-RS.
__device__ __forceinline__ void rs_epilogue_fold(const KParams& p, uint32_t taddr, const char* in0, char* rp,
                                              int64_t ocol0, int row, bool valid, uint32_t tempty_a) {
  for (int j = 0; j < BN / 32; ++j) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + j * 32, r);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(r[c]);
    if (valid) {
      // rs_direct fold: ((c[p0] + c[p1]) + ... + c[p(T-2)]) + own  (collectives.cpp:326-355)
      direct_fold(p, in0, j, row, v);
      store_out_row(p, rp, ocol0 + j * 32, v);
    }
  }
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(tempty_a);
}

// rs_direct last step of a pair's LAST tile (bf16 wire): the same fold, with the T-1 received
// partials staged through shared memory by bulk copies. The fold reads T-1 partials per output
// element; from L2 with per-thread loads it is latency-bound (~90 us for the final step at
// TP = 8), while the pipeline stages are idle once the pair's last main loop is done. One elected
// thread of the epilogue warpgroup copies sub-chunk j + 1 of every partial (T-1 contiguous
// 8 KiB pieces) into one half of a double buffer while the group sums sub-chunk j from the
// other half in the reference order ((c[p0] + c[p1]) + ...) and adds the own partial last.
__device__ __noinline__ void rs_epilogue_fold_stages(const KParams& p, uint32_t taddr, const char* in0, char* rp,
                                                      int64_t ocol0, int row, bool valid, uint32_t tempty_a,
                                                      uint8_t* sbuf, uint64_t* fbar, int eg, int ew) {
  constexpr uint32_t kUnit = 4 * BM * 16;               // one 32-column sub-chunk of one bf16 partial
  constexpr uint32_t kBuf = (kMaxRanks - 1) * kUnit;    // one half of the double buffer
  const int nin = p.T - 1;
  const bool issuer = ew == 0;  // the whole warp (warp-uniform values); elect.sync issues
  auto issue = [&](int j) {
    uint8_t* dst = sbuf + (j & 1) * kBuf;
    mbar_arrive_expect_tx_warp(fbar + (j & 1), nin * kUnit);
    for (int s = 0; s < nin; ++s)
      bulk_load_warp(dst + s * kUnit, in0 + s * p.slot_bytes + static_cast<int64_t>(j) * kUnit, kUnit, fbar + (j & 1));
  };
  // every warp of the group has acquired its rows' flags of all T-1 partials: the barrier carries
  // those acquires to the issuer, whose proxy fence orders them before the async-proxy copies
  named_bar_sync(1 + eg, 128);
  if (issuer) {
    fence_proxy_async_global();
    issue(0);
  }
  for (int j = 0; j < BN / 32; ++j) {
    if (issuer && j + 1 < BN / 32) issue(j + 1);
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + j * 32, r);
    mbar_wait(p, fbar + (j & 1), (j >> 1) & 1);
    tmem_ld_wait();
    if (valid) {
      const uint8_t* buf = sbuf + (j & 1) * kBuf;
      float acc[32];
#pragma unroll 1
      for (int s = 0; s < nin; ++s) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint4 w = *reinterpret_cast<const uint4*>(buf + s * kUnit + (g * BM + row) * 16);
          const float in[8] = {bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y),
                               bf16lo(w.z), bf16hi(w.z), bf16lo(w.w), bf16hi(w.w)};
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[g * 8 + c] = s == 0 ? in[c] : acc[g * 8 + c] + in[c];
        }
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = acc[c] + __uint_as_float(r[c]);
      store_out_row(p, rp, ocol0 + j * 32, acc);
    }
    named_bar_sync(1 + eg, 128);  // half (j & 1) is read by every warp before sub-chunk j + 2 refills it
  }
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(tempty_a);
}

// rs_direct last step, bf16 wire (MODE_RS_DIRECT): the fold reads T-1 partials per output
// element, which from L2 with per-thread loads is latency-bound (a traced cfg2 TP8 call spent
// ~90 us folding after its last main loop). Instead one elected thread of the epilogue warpgroup
// bulk-copies the T-1 partials' next 8-column word (T-1 contiguous 2 KiB pieces of the wire
// images) into one half of the group's double buffer while the group sums the current word from
// the other half, in the reference order ((c[p0] + c[p1]) + ...), and adds the own partial last.
__device__ __noinline__ void rs_epilogue_fold_smem(const KParams& p, uint32_t taddr, const char* in0, char* rp,
                                                   int64_t ocol0, int row, bool valid, uint32_t tempty_a,
                                                   uint8_t* sbuf, uint64_t* fbar, int eg, int ew) {
  constexpr uint32_t kBuf = (kMaxRanks - 1) * kFoldUnit;  // one half of the double buffer
  constexpr int kWords = BN / 8;                           // 16-B words (8 bf16 columns) per row
  const int nin = p.T - 1;
  const bool issuer = ew == 0;  // the whole warp (warp-uniform values); elect.sync issues
  // word u of every partial: wire_off(0, u / 4, u % 4, 0) = u * BM * 16
  auto issue = [&](int u) {
    uint8_t* dst = sbuf + (u & 1) * kBuf;
    mbar_arrive_expect_tx_warp(fbar + (u & 1), nin * kFoldUnit);
    for (int s = 0; s < nin; ++s)
      bulk_load_warp(dst + s * kFoldUnit, in0 + s * p.slot_bytes + static_cast<int64_t>(u) * kFoldUnit, kFoldUnit,
                     fbar + (u & 1));
  };
  // every warp of the group has acquired its rows' flags of all T-1 partials: the barrier carries
  // those acquires to the issuer, whose proxy fence orders them before the async-proxy copies
  named_bar_sync(1 + eg, 128);
  if (issuer) {
    fence_proxy_async_global();
    issue(0);
  }
  for (int j = 0; j < BN / 32; ++j) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + j * 32, r);
    float v[32];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int u = j * 4 + g;
      if (issuer && u + 1 < kWords) issue(u + 1);
      mbar_wait(p, fbar + (u & 1), (u >> 1) & 1);
      if (g == 0) tmem_ld_wait();
      const uint8_t* buf = sbuf + (u & 1) * kBuf;
      float acc[8];
#pragma unroll 1
      for (int s = 0; s < nin; ++s) {
        const uint4 w = *reinterpret_cast<const uint4*>(buf + s * kFoldUnit + row * 16);
        const float in[8] = {bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y),
                             bf16lo(w.z), bf16hi(w.z), bf16lo(w.w), bf16hi(w.w)};
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = s == 0 ? in[c] : acc[c] + in[c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) v[g * 8 + c] = acc[c] + __uint_as_float(r[g * 8 + c]);
      named_bar_sync(1 + eg, 128);  // half (u & 1) is read by every warp before word u + 2 refills it
    }
    if (valid) store_out_row(p, rp, ocol0 + j * 32, v);
  }
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(tempty_a);
}

// GEMM-RS epilogue of one 128 x 256 accumulator (this thread: one row), pipelined by one
// 32-column sub-chunk: the inbox loads of sub-chunk j+1 are in flight while sub-chunk j is
// read from TMEM, summed and stored (bf16 wire; the fp32 parity wire loads its inbox in
// the same iteration). The accumulator is released as soon as its last columns are in
// registers. kF32 is a template parameter so each instance keeps only its own buffers live.
template <bool kF32, int kDepth>
__device__ __forceinline__ void rs_epilogue_pipelined(const KParams& p, uint32_t taddr, const char* inbox,
                                                      char* dst_tile, char* rp, int64_t ocol0, int row,
                                                      bool valid, bool last, uint32_t tempty_a) {
  constexpr int kW = kF32 ? 8 : 4;  // 16-B inbox words per sub-chunk
  constexpr int kNJ = BN / 32;
  // bf16 wire: kDepth sub-chunks of the inbox in flight (64 B each per thread). The RS ring is a
  // chain of tile epilogues across steps and each link pays these loads' latency: 4 in flight
  // instead of 2 measured -2% on the per-GPU TP8 ring (8: no better, and spills).
  constexpr int kD = kF32 ? 1 : kDepth;
  uint32_t r[32];
  uint4 raw[kD][kW];
  const bool pull = valid && inbox;
  if (pull && kD > 1) {
#pragma unroll
    for (int d = 0; d < kD; ++d)
#pragma unroll
      for (int g = 0; g < kW; ++g) raw[d][g] = *reinterpret_cast<const uint4*>(inbox + wire_off(kF32, d, g, row));
  }
#pragma unroll(kD > 1 ? kNJ : 1)
  for (int j = 0; j < kNJ; ++j) {
    const int c = j % kD;
    if (pull && kD == 1) {
#pragma unroll
      for (int g = 0; g < kW; ++g) raw[0][g] = *reinterpret_cast<const uint4*>(inbox + wire_off(kF32, j, g, row));
    }
    tmem_ld_32x32b_x32(taddr + j * 32, r);
    tmem_ld_wait();
    if (j + 1 == kNJ) {
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(tempty_a);
    }
    if (!valid) continue;
    float v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
    if (inbox) {
      // rs_pipelined: partial += inbox   (collectives.cpp:303)
#pragma unroll
      for (int g = 0; g < kW; ++g) {
        const uint4 w = raw[c][g];
        if (kF32) {
          v[g * 4 + 0] = v[g * 4 + 0] + __uint_as_float(w.x);
          v[g * 4 + 1] = v[g * 4 + 1] + __uint_as_float(w.y);
          v[g * 4 + 2] = v[g * 4 + 2] + __uint_as_float(w.z);
          v[g * 4 + 3] = v[g * 4 + 3] + __uint_as_float(w.w);
        } else {
          v[g * 8 + 0] = v[g * 8 + 0] + bf16lo(w.x); v[g * 8 + 1] = v[g * 8 + 1] + bf16hi(w.x);
          v[g * 8 + 2] = v[g * 8 + 2] + bf16lo(w.y); v[g * 8 + 3] = v[g * 8 + 3] + bf16hi(w.y);
          v[g * 8 + 4] = v[g * 8 + 4] + bf16lo(w.z); v[g * 8 + 5] = v[g * 8 + 5] + bf16hi(w.z);
          v[g * 8 + 6] = v[g * 8 + 6] + bf16lo(w.w); v[g * 8 + 7] = v[g * 8 + 7] + bf16hi(w.w);
        }
      }
      if (kD > 1 && j + kD < kNJ) {
#pragma unroll
        for (int g = 0; g < kW; ++g) raw[c][g] = *reinterpret_cast<const uint4*>(inbox + wire_off(kF32, j + kD, g, row));
      }
    }
    if (last)
      store_out_row(p, rp, ocol0 + j * 32, v);
    else
      wire_store(kF32, dst_tile, j, row, v);
  }
}

// Instances launched with programmatic dependent launch (PDL): the T == 1 GEMM. Its CTAs
// never wait on another grid, so letting the next launch in early cannot starve anything
// (the attention-family and query-split instances wait on other grids of this GPU and must
// keep plain stream order). Measured (tools/ab_env.py, alternating processes): +1.7% on the
// T = 1 MLP block; on the per-GPU TP = 8 fused GEMM-RS PDL cost 5% with every trigger
// placement (after the prologue, after the last TMA load, implicit at exit), and it was
// neutral on the fused AG-GEMM, so the multi-rank instances keep plain stream order.
__host__ __device__ constexpr bool pdl_instance(int mode) {
  return mode == MODE_SINGLE || mode == MODE_STD || mode == MODE_DP_GRAD || mode == MODE_GATHER_B ||
         mode == MODE_RS_DIRECT || mode == MODE_DP_DIRECT;
}

// Operand / epilogue modes are compile-time (one instance per use): runtime flags in the
// single-thread producer / MMA loops cost measurable throughput.
// The kernel body: CTA g of the ctas_per_rank CTAs serving hosted rank h (rank p.rank0 + h).
// exit_ctas = CTAs that read p's device epoch (the last of them to exit publishes it).
template <int kOp, int kMode>
__device__ __forceinline__ void fused_body(const KParams& p, const int h, const int g, const uint32_t exit_ctas) {
  constexpr bool kAMn = kMode == MODE_DP_GRAD || kMode == MODE_DP_DIRECT;  // A MN-major (X^T)
  constexpr bool kGatherB = kMode == MODE_GATHER_B;                    // AG carries B
  constexpr bool kBBatched = kMode == MODE_QK || kMode == MODE_PV;     // B per batch (head)
  constexpr bool kBKMajor = kGatherB || kMode == MODE_QK;              // B stored (N, K)
  constexpr bool kUpEpi = kMode == MODE_PV;                            // merge_heads + push + flags
  constexpr bool kSingle = kMode == MODE_SINGLE;                       // T == 1: no ring at all
  constexpr bool kPdl = pdl_instance(kMode);                           // launched with PDL
  // rs_direct (pairwise) fold: its own instances for the TP and DP operands (folds staged
  // through shared memory); the query-split / UP instances keep the runtime switch
  constexpr bool kDirectInst = kMode == MODE_RS_DIRECT || kMode == MODE_DP_DIRECT;
  const bool direct = kDirectInst || (kMode != MODE_STD && kMode != MODE_DP_GRAD && p.direct);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  constexpr int kSt = kDirectInst ? kStagesDirect : kStages;  // pipeline stages
  uint8_t* smem_b = smem + kSt * kAStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSt * kStageBytes);
  uint64_t* full = bars;                  // leader: 2 arrivals + 2 x stage tx bytes
  uint64_t* empty = bars + kSt;       // per CTA: 1 (leader's multicast commit)
  uint64_t* tfull = bars + 2 * kSt;   // per CTA: 1 (leader's multicast commit)
  uint64_t* tempty = bars + 2 * kSt + 2;  // leader: 8 epilogue warps of the pair
  uint64_t* fold_bar = bars + 4 * kSt + 4;   // [2 groups][2 buffers]: rs_direct fold staging
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * kSt + 8);
  uint64_t* fwd_bar = bars + 4 * kSt + 9;    // [2]: AG forwarder warps, their bulk / tensor loads
  uint8_t* fold_smem = smem + kSt * kStageBytes + 2048;  // pairwise instances: [2 groups][kFoldGroupBytes]
  uint8_t* fwd_smem = smem + kSt * kStageBytes + 1024;   // AG (both kinds): 2 x 16 KiB forwarder buffers

  // warp index through a shuffle so ptxas treats it (and the role branches) as warp-uniform
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int cta = static_cast<int>(cluster_ctarank());
  const bool leader = cta == 0;
  const int rank = p.rank0 + h;
  const int G = p.ctas_per_rank;
  const int gp = g >> 1, GP = G >> 1;  // pair index / pairs per rank
  const int per_step = p.npairs * p.nnt;
  const int ntiles = p.nsteps * per_step;
  const bool active = h < p.n_hosted;  // (grid is sized exactly; kept for safety)
  // AG ring forwarding (warps 2-3, decoupled from the GEMM pipeline: see the forwarder branch)
  const bool fwd = !kSingle && kOp == OP_AG && p.T > 1 && !p.compute_only;
  const int fbatch = min(max(p.ag_batch, 1), 8);  // forwards per fence + flag publication

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.tmap_a);
    prefetch_tmap(&p.tmap_b);
    if (kOp == OP_AG && p.T > 1) {
      prefetch_tmap(&p.tmap_wire[0]);
      prefetch_tmap(&p.tmap_wire[1]);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kSt; ++s) {
      mbar_init(full + s, 2);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);
      mbar_init(fold_bar + a, 1);
      mbar_init(fold_bar + 2 + a, 1);
      mbar_init(fwd_bar + a, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<512>(tmem_holder);
  // PDL: everything above is CTA-local and overlaps the previous kernel's tail; no global
  // memory is touched before the previous grid has completed.
  if (kPdl) griddep_wait();
  if (threadIdx.x == 0) {
    const uint32_t e = p.epoch_dev ? epoch_read(p.epoch_dev, p.epoch_bump) : p.epoch;
    s_epoch = e;
    s_parity = p.epoch_dev ? static_cast<int>(e & 1u) : p.parity;
    // fault injection: the failing rank names itself in the blame tables (its successors
    // time out on its flags and follow the chain to it)
    if (rank == p.fault_rank && g == 0 && h < p.n_hosted && p.T > 1) blame_store(p.blame.table, p.blame.T, rank, rank);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  // The next PDL launch may start its prologue on SMs as this grid's CTAs exit. Only
  // instances whose CTAs never wait on another grid trigger early: a dependent grid must
  // not take SMs a concurrently running kernel (query-split attention) still needs.
  if (kPdl && p.pdl_trigger == 1) griddep_launch_dependents();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t ep = s_epoch;  // this launch's epoch / heap parity, in registers from here on
  const int par = s_parity;
  const CUtensorMap* wmap = &p.tmap_wire[par];

  if (!active) {
  } else if (warp < 4) {
    // Register split (384 threads, pool kRegPool per thread at launch): warps 0-3 (TMA,
    // MMA, TMEM / forwarders) need few; the two epilogue warpgroups hold a 32-column
    // TMEM chunk pipeline each. setmaxnreg.inc blocks until the pool can satisfy it, so
    // the split must fit the pool the launch allocates (checked in launch_instance).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
    if (warp == 0) {
      // ===================================================== TMA producer (both CTAs)
      // The whole warp walks the schedule (warp-uniform values; the AG wire-image flag scan is
      // warp-parallel) and elect.sync issues the barrier arrivals and TMA loads.
      const uint64_t pol_a = l2_policy(p.l2_a), pol_b = l2_policy(p.l2_b);
      int stage = 0;
      uint32_t phase = 0;
      for (int lin = gp; lin < ntiles; lin += GP) {
        const Tile t = get_tile(p, lin, cta);
        const int pass = t.step / p.T, it = t.step - pass * p.T;
        const bool from_wire = !kSingle && (kOp == OP_AG) && it > 0 && !p.compute_only;
        const bool a_from_wire = from_wire && !kGatherB;
        const bool b_from_wire = from_wire && kGatherB;
        int64_t arow;
        if (t.valid == 0)
          arow = p.x_rows;  // whole box out of bounds: TMA zero-fills, bytes still counted
        else if (kOp == OP_RS)
          arow = (kMode == MODE_QK ? p.a_row_off[h] : 0) +
                 (p.T > 1 ? (static_cast<int64_t>(p.sched[rank][it][2]) * p.m + pass) : 0) * p.Sc + t.row0;
        else if (kGatherB)
          arow = t.row0;
        else
          arow = pass * p.Sc + t.row0;
        const int aslot = pass * (p.T - 1) + it - 1;
        // wire images of this CTA's operand for this tile: A rows (m-block) or B half (n-tile)
        const int64_t img0 = kGatherB ? (static_cast<int64_t>(cta) * p.nnt + t.nt) * p.nkb
                                        : static_cast<int64_t>(t.mb) * p.nkb;
        const bool wire_live = a_from_wire ? (t.valid > 0) : b_from_wire;
        const uint32_t* mflags = (a_from_wire || b_from_wire) ? flag_ptr(p, par, rank, aslot, img0) : nullptr;
        int ready = -1;  // wire images [0, ready] of this operand block are known to have landed
        uint64_t t_first = 0;
        if (kMode == MODE_QSPLIT && t.valid > 0 && !p.compute_only) {
          // the A rows of this step's query slice come from the concurrently running attention
          // kernel (generic stores): wait for the slice's counter, then order the TMA reads
          // (every lane acquires and fences: elect.sync picks the issuing lane)
          const int l = p.T > 1 ? p.sched[rank][it][2] : 0;
          const uint32_t* cnt = p.qs_ready[h] + l;
          if (ld_acquire_gpu(cnt) < p.qs_target) {
            const uint64_t tq0 = globaltimer();
            while (ld_acquire_gpu(cnt) < p.qs_target) {
              if (aborted(p, rank, ep)) break;
              if (globaltimer() - tq0 > static_cast<uint64_t>(p.timeout_ns)) {
                record_error(p, 1, rank, t.step, lin);
                break;
              }
              __nanosleep(256);
            }
          }
          fence_proxy_async_global();
        }
        for (int kb = 0; kb < p.nkb; ++kb) {
          if (wire_live && kb > ready) {
            // Claim the run of consecutive landed images from kb on: every lane acquire-loads
            // one flag (image kb + lane, system scope; one round trip per poll) until image
            // kb has landed. The warp barrier carries the acquires to every lane, whose proxy
            // fence orders them before the TMA (async-proxy) reads. Images past the run are
            // claimed when the producer reaches them, mid-tile, behind the buffered stages.
            // (Relaxed polls plus one fence.acq_rel.sys measured 3x slower: the system fence
            // costs more than the round trips it saves.)
            const uint64_t tw0 = p.trace ? globaltimer() : 0;
            uint64_t tspin = 0;
            int run = 0;
            for (int poll = 0;; ++poll) {
              const int k = kb + lane;
              const bool ok = k >= p.nkb || ld_acquire_sys(mflags + k) >= ep;
              const uint32_t m = __ballot_sync(0xffffffffu, ok);
              run = (m == 0xffffffffu) ? 32 : __ffs(~m) - 1;
              if (run > 0) break;
              if (poll == 0) tspin = globaltimer();
              __nanosleep(32);
              if ((poll & 255) == 255) {
                const bool timed_out = globaltimer() - tspin > static_cast<uint64_t>(p.timeout_ns);
                if (aborted(p, rank, ep) || timed_out) {
                  if (lane == 0)
                    give_up(p, timed_out && !aborted(p, rank, ep), rank, p.sched[rank][it - 1][1], t.step, lin, ep);
                  break;
                }
              }
            }
            ready = min(kb + max(run, 1) - 1, p.nkb - 1);
            __syncwarp();
            fence_proxy_async_global();  // every lane: whichever lane elect.sync picks issues the TMA
            if (p.trace && lane == 0) {
              const uint64_t tw1 = globaltimer();
              if (tw1 - tw0 > 1000) trace_rec(p, TR_WAIT_A, rank, t.step, static_cast<int64_t>(lin) * 1024 + kb, tw0, tw1);
            }
          }
          {
            mbar_wait(p, empty + stage, phase ^ 1);
            uint8_t* sa = smem_a + stage * kAStageBytes;
            uint8_t* sb = smem_b + stage * kBStageBytes;
            const uint32_t fb = mapa_shared(smem_u32(full + stage), 0);
            const int img = static_cast<int>(img0) + kb;
            if (leader)
              mbar_arrive_expect_tx_warp(full + stage, 2 * kStageBytes);
            else
              mbar_arrive_cluster_warp(fb);
            if (a_from_wire) {
              tma_load_2sm_5d_warp(sa, wmap, fb, 0, 0, t.valid ? img : p.nmb * p.nkb, aslot, h);
            } else if (kAMn) {
              // MN-major A (e.g. X^T from row-major X): two 64-row x 64-K SW128 atoms
  #pragma unroll
              for (int q = 0; q < BM / 64; ++q)
                tma_load_2sm_4d_warp(sa + q * (64 * BK * 2), &p.tmap_a, fb, static_cast<int>(arow) + q * 64, kb * BK,
                                t.b, h);
            } else {
              tma_load_2sm_4d_hint_warp(sa, &p.tmap_a, fb, kb * BK, static_cast<int>(arow), t.b, h, pol_a);
            }
            if (b_from_wire) {
              tma_load_2sm_5d_warp(sb, wmap, fb, 0, 0, img, aslot, h);
            } else if (kBKMajor) {
              // K-major B (w stored (N, K)): one 128-column x 64-K SW128 box
              if (kBBatched)
                tma_load_2sm_4d_warp(sb, &p.tmap_b, fb, kb * BK, t.nt * BN + cta * (BN / 2), t.b, h);
              else
                tma_load_2sm_3d_warp(sb, &p.tmap_b, fb, kb * BK, t.nt * BN + cta * (BN / 2), h);
            } else {
  #pragma unroll
              for (int q = 0; q < BN / 128; ++q) {
                if (kBBatched)
                  tma_load_2sm_4d_warp(sb + q * (64 * BK * 2), &p.tmap_b, fb, t.nt * BN + cta * (BN / 2) + q * 64,
                                  kb * BK, t.b, h);
                else
                  tma_load_2sm_3d_hint_warp(sb + q * (64 * BK * 2), &p.tmap_b, fb, t.nt * BN + cta * (BN / 2) + q * 64,
                                       kb * BK, h, pol_b);
              }
            }
            if (p.trace && kb == 0) t_first = globaltimer();
          }
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
        if (p.trace && lane == 0) trace_rec(p, TR_MAINLOOP, rank, t.step, lin, t_first, globaltimer());
      }
      if (kPdl && p.pdl_trigger == 2) griddep_launch_dependents();  // all of this CTA's loads issued
    } else if (warp == 1) {
      // ===================================================== MMA issuer (leader CTA)
      // The whole warp runs the loop (warp-uniform values) and elect.sync issues, so the
      // descriptors live in uniform registers.
      if (leader) {
        const uint32_t idesc =
            make_idesc_bf16(2 * BM, BN, /*b_mn_major=*/!kBKMajor, /*a_mn_major=*/kAMn);
        int stage = 0;
        uint32_t phase = 0;
        int lt = 0;
        for (int lin = gp; lin < ntiles; lin += GP, ++lt) {
          const int a = lt & 1;
          const uint32_t use = static_cast<uint32_t>(lt >> 1);
          mbar_wait(p, tempty + a, (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + a * BN;
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(p, full + stage, phase);
            tc_fence_after();
            const uint32_t abase = smem_u32(smem_a + stage * kAStageBytes);
            const uint32_t bbase = smem_u32(smem_b + stage * kBStageBytes);
  #pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // A: K-major SW128, 16 elems = 32 B step inside the atom; SBO = 8 rows x 128 B.
              // MN-major A: like B, 16 K-rows = 2048 B, LBO = 64-row atom (8 KiB), SBO = 1 KiB.
              const uint64_t ad = kAMn ? make_sdesc(abase + k * 2048, 64 * BK * 2, 1024)
                                         : make_sdesc(abase + k * 32, 0, 1024);
              // B: MN-major SW128 (this CTA's 128 columns; the peer holds the other 128 at the
              // same offsets); 16 K-rows = 2048 B; LBO = 64-col atom (64 x 128 B); SBO = 8 K-rows.
              const uint64_t bd = kBKMajor ? make_sdesc(bbase + k * 32, 0, 1024)
                                                             : make_sdesc(bbase + k * 2048, 64 * BK * 2, 1024);
              mma_bf16_2sm_warp(d, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
            mma_commit_2sm_warp(empty + stage, 0x3);
            if (++stage == kSt) { stage = 0; phase ^= 1; }
          }
          mma_commit_2sm_warp(tfull + a, 0x3);
        }
      }
    } else {
      // ===================================================== AG ring forwarders (warps 2-3)
      if (fwd) {
        // The ring forward is decoupled from the GEMM. Every CTA's two forwarder warps take a
        // share of each step's images (round-robin over all CTAs of the rank), step by step:
        // step 0 copies this rank's own operand (A: rows of x; gather_b: a 128-row half of a
        // weight n-tile; a tensor load puts it in the SW128 image layout, zero past the
        // edges), step i > 0 copies the inbox image of slot i-1
        // once the predecessor's flag is seen, into the successor's slot i. No pipeline
        // stage is ever held (gating stage reuse on a forwarder cost 10-18 us per call at
        // TP = 8), the work is spread over all SMs, and step i's sends depend only on the
        // predecessor's step i-1 sends, so the ring runs ahead of the GEMM and cannot wait
        // on it. Each warp fences and publishes its flags per batch and at every step end.
        const int fw = g * 2 + (warp - 2);  // this warp's index among the rank's forwarders
        const int nfw = G * 2;
        // Copies are TMA bulk operations issued by lane 0 through a 16 KiB SMEM bounce buffer
        // per warp: a load into the buffer, then a bulk store into the successor's slot. No
        // registers hold data, so the copy rate is not bounded by the loads in flight that the
        // 88-register control warps can hold (cfg3 TP8 per-GPU AG 308 -> 300 us, wire waits
        // 966 -> 218 per call).
        uint8_t* fbuf = fwd_smem + (warp - 2) * kAStageBytes;
        uint64_t* fbar = fwd_bar + (warp - 2);
        uint32_t fph = 0;
        int unpub[8];  // fbatch <= 8
        int nunpub = 0;
        int cur_slot = 0, cur_dst = 0;
        auto flush = [&]() {
          const uint64_t tf0 = p.trace ? globaltimer() : 0;
          if (lane == 0) {
            bulk_wait<0>();               // this warp's bulk stores have completed
            fence_proxy_async_global();   // ... ordered before the generic flag stores
            fence_sys();
            if (rank != p.fault_rank)
              for (int i = 0; i < nunpub; ++i) st_relaxed_sys(flag_ptr(p, par, cur_dst, cur_slot, unpub[i]), ep);
          }
          __syncwarp();
          if (p.trace && lane == 0) trace_rec(p, TR_FLUSH, rank, 0, nunpub, tf0, globaltimer());
          nunpub = 0;
        };
        // images per slot: A rows per (m-block, k-block); gather_b B halves per (half, n-tile, k-block)
        const int nimg = kGatherB ? 2 * p.nnt * p.nkb : p.nmb * p.nkb;
        for (int pass = 0; pass < p.m; ++pass) {
          for (int it = 0; it < p.T - 1; ++it) {
            const int slot = pass * (p.T - 1) + it;
            cur_slot = slot;
            cur_dst = p.sched[rank][it][0];
            const uint64_t t0 = p.trace ? globaltimer() : 0;
            for (int img = fw; img < nimg; img += nfw) {
              const int mb = img / p.nkb, kb = img - mb * p.nkb;  // gather_b: mb = half * nnt + n-tile
              const int bb = mb / p.nmb_per_batch, j = mb - bb * p.nmb_per_batch;
              const int row0 = j * BM;
              if (!kGatherB && p.Sc - row0 <= 0) continue;  // padding m-block of an odd pair: never read
              if (lane == 0) {
                char* dst = slot_ptr(p, par, cur_dst, slot) + static_cast<int64_t>(img) * kAStageBytes;
                bulk_wait_read<0>();  // the previous store has read the buffer
                if (it == 0) {
                  // rows past this chunk are read as whatever x holds there (their products
                  // are never stored)
                  mbar_arrive_expect_tx(fbar, kAStageBytes);
                  if (kGatherB)  // K-major B: 64 K x 128 N box of half mb / nnt of n-tile mb % nnt
                    tma_load_3d(fbuf, &p.tmap_b, fbar, kb * BK, (mb % p.nnt) * BN + (mb / p.nnt) * (BN / 2), h);
                  else
                    tma_load_4d(fbuf, &p.tmap_a, fbar, kb * BK, pass * static_cast<int>(p.Sc) + row0, bb, h);
                } else {
                  const uint32_t* fsrc = flag_ptr(p, par, rank, slot - 1, img);
                  wait_flag(p, fsrc, rank, p.sched[rank][it - 1][1], pass * p.T + it, img, ep);
                  fence_proxy_async_global();  // the acquired image, read by the async proxy
                  mbar_arrive_expect_tx(fbar, kAStageBytes);
                  bulk_load(fbuf, slot_ptr(p, par, rank, slot - 1) + static_cast<int64_t>(img) * kAStageBytes,
                            kAStageBytes, fbar);
                }
                mbar_wait(p, fbar, fph);
                bulk_store(dst, fbuf, kAStageBytes);
                bulk_commit();
              }
              fph ^= 1;
              unpub[nunpub++] = img;
              if (nunpub == fbatch) flush();
            }
            if (nunpub > 0) flush();
            if (p.trace && lane == 0) trace_rec(p, TR_AG_PIECE, rank, slot, fw, t0, globaltimer());
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
    // ===================================================== epilogue (warps 4..11)
    // Two warpgroups, one per TMEM accumulator: group eg drains accumulator eg, i.e. this
    // pair's tiles lt = eg, eg + 2, ... Each group has two main loops' time for one tile's
    // epilogue (TMEM read, inbox add, wire / output stores, fence + flags), which at short
    // per-rank K (GEMM-RS at TP = 8) is longer than one main loop.
    const int eg = (warp - 4) >> 2;
    const int ew = (warp - 4) & 3;   // TMEM lane quarter this warp may access (warp % 4)
    const int row = ew * 32 + lane;  // row inside this CTA's 128-row block == TMEM lane
    char* out_h = p.out + h * p.out_rank_stride;
    const int64_t esz = p.out_f32 ? 4 : 2;
    const int64_t tile_bytes = static_cast<int64_t>(BM) * BN * (p.wire_f32 ? 4 : 2);
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(tempty), 0);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(tempty + 1), 0);
    // RS flags: one system fence covers the wire stores of up to kPend tiles, and pending
    // flags are always published before any wait that may block (an inbox flag, or an
    // accumulator the other group's progress gates), so the ring can never wait on itself.
    // kPend = 1 (publish every tile): at TP = 8 a step is less than one round of pair
    // tiles, so the successor's next-step tile is often already waiting on this flag; the
    // lazy kPend = 2 cost 9% on the per-GPU cfg2 GEMM-RS under the self-ring model.
    constexpr int kPend = 1;
    uint32_t* pend[kPend];
    int npend = 0;
    auto publish = [&]() {
      if (npend == 0) return;
      const uint64_t tp0 = (p.trace && lane == 0) ? globaltimer() : 0;
      fence_sys();
      __syncwarp();
      if (lane == 0 && rank != p.fault_rank)
        for (int i = 0; i < npend; ++i) st_relaxed_sys(pend[i], ep);
      if (p.trace && lane == 0 && ew == 0) trace_rec(p, TR_PUBLISH, rank, 0, npend, tp0, globaltimer());
      npend = 0;
    };
    const int a = eg;
    int lt = eg;
    for (int lin = gp + eg * GP; lin < ntiles; lin += 2 * GP, lt += 2) {
      const Tile t = get_tile(p, lin, cta);
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      if (npend > 0 && !mbar_try_wait(tfull + a, use & 1)) publish();
      mbar_wait(p, tfull + a, use & 1);
      tc_fence_after();
      const uint64_t t_epi0 = (p.trace && lane == 0) ? globaltimer() : 0;
      const int pass = t.step / p.T, it = t.step - pass * p.T;
      const bool valid = row < t.valid;
      const bool tile_live = t.valid > 0;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + a * BN;
      const int64_t tile_idx = static_cast<int64_t>(t.mb) * p.nnt + t.nt;
      const int64_t fidx = tile_idx * 4 + ew;

      if (kOp == OP_AG) {
        const int l = p.T > 1 ? p.sched[rank][it][2] : 0;
        // gather_b: rows stay local, the step selects the output column block l
        const int64_t orow = kGatherB ? static_cast<int64_t>(t.b) * p.out_rows + t.row0 + row
                                        : static_cast<int64_t>(t.b) * p.out_rows +
                                              (static_cast<int64_t>(l) * p.m + pass) * p.Sc + t.row0 + row;
        char* rp = out_h + (orow * p.out_ld + (kGatherB ? static_cast<int64_t>(l) * p.blk_cols : 0)) * esz;
        if (p.act == ACT_SWIGLU) {
          // Tile-interleaved W: columns [0,128) of the tile are gate, [128,256) the matching
          // up columns -> 128 output columns silu(gate) * up (Llama MLP, fused).
          for (int j = 0; j < BN / 64; ++j) {
            uint32_t rg[32], ru[32];
            tmem_ld_32x32b_x32(taddr + j * 32, rg);
            tmem_ld_32x32b_x32(taddr + BN / 2 + j * 32, ru);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const float gt = __uint_as_float(rg[c]);
              v[c] = __fdividef(gt, 1.0f + __expf(-gt)) * __uint_as_float(ru[c]);
            }
            if (valid) store_out_row(p, rp, static_cast<int64_t>(t.nt) * (BN / 2) + j * 32, v);
          }
        } else {
          for (int j = 0; j < BN / 32; ++j) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + j * 32, r);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const float x = __uint_as_float(r[c]);
              v[c] = p.act == ACT_SQUARE ? x * x : x;
            }
            if (valid) store_out_row(p, rp, static_cast<int64_t>(t.nt) * BN + j * 32, v);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(a ? tempty_leader1 : tempty_leader0);
        if (p.trace && lane == 0 && ew == 0 && tile_live)
          trace_rec(p, TR_TILE, rank, t.step, lin, t_epi0, globaltimer());
        continue;
      }

      // ------------------------------------------------ OP_RS
      const bool last = (it == p.T - 1) || p.compute_only;
      const int slot_send = pass * (p.T - 1) + it;
      const int send_rank = p.T > 1 ? p.sched[rank][it][0] : -1;
      const char* inbox = nullptr;
      if (tile_live && !direct && it > 0 && !p.compute_only) {
        const int slot_in = slot_send - 1;
        const uint64_t tw0 = (p.trace && lane == 0) ? globaltimer() : 0;
        const uint32_t* fin = flag_ptr(p, par, rank, slot_in, fidx);
        if (npend > 0 && ld_relaxed_sys(fin) < ep) publish();
        wait_flag(p, fin, rank, p.sched[rank][it - 1][1], t.step, lin, ep);
        if (p.trace && lane == 0 && ew == 0) {
          const uint64_t tw1 = globaltimer();
          if (tw1 - tw0 > 1000) trace_rec(p, TR_WAIT_IN, rank, t.step, lin, tw0, tw1);
        }
        inbox = slot_ptr(p, par, rank, slot_in) + tile_idx * tile_bytes;
      }
      if (tile_live && direct && last && p.T > 1 && !p.compute_only) {
        publish();
        for (int s = 0; s < p.T - 1; ++s)
          wait_flag(p, flag_ptr(p, par, rank, pass * (p.T - 1) + s, fidx), rank, p.sched[rank][s][1], t.step, lin,
                    ep);
      }
      __syncwarp();
      char* dst_tile =
          (last || !tile_live) ? nullptr : slot_ptr(p, par, send_rank, slot_send) + tile_idx * tile_bytes;
      // heads_merge (UP): batch g = b*heads + hh -> rows of b, columns hh*N (merge_heads fused)
      const int hm = kUpEpi ? p.heads_merge : 0;
      const int64_t ob = hm ? t.b / hm : t.b;
      const int64_t ocol = kUpEpi ? p.out_col_off[h] + (hm ? static_cast<int64_t>(t.b % hm) * p.N : 0) : 0;
      const int64_t orow = ob * p.out_rows + pass * p.Sc + t.row0 + row;
      char* rp = ((kUpEpi && p.out_rank[h]) ? p.out_rank[h] : out_h) + (orow * p.out_ld + ocol) * esz;
      const bool folding = direct && last && p.T > 1 && !p.compute_only;
      if (folding) {
        const char* in0 = slot_ptr(p, par, rank, pass * (p.T - 1)) + tile_idx * tile_bytes;
        // pairwise instance, bf16 wire: stage the fold through shared memory -- the pair's last
        // tile through its idle pipeline stages (8 KiB pieces, 32 columns at a time), every other
        // fold tile through the warpgroup's own buffers (2 KiB pieces, 8 columns at a time)
        if (kDirectInst && !p.wire_f32 && tile_live && lin + GP >= ntiles)
          rs_epilogue_fold_stages(p, taddr, in0, rp, static_cast<int64_t>(t.nt) * BN, row, valid,
                                  a ? tempty_leader1 : tempty_leader0, smem, fold_bar + 2 * eg, eg, ew);
        else if (kDirectInst && !p.wire_f32 && tile_live)
          rs_epilogue_fold_smem(p, taddr, in0, rp, static_cast<int64_t>(t.nt) * BN, row, valid,
                                a ? tempty_leader1 : tempty_leader0, fold_smem + eg * kFoldGroupBytes,
                                fold_bar + 2 * eg, eg, ew);
        else
          rs_epilogue_fold(p, taddr, in0, rp, static_cast<int64_t>(t.nt) * BN, row, valid,
                           a ? tempty_leader1 : tempty_leader0);
      } else {
        // Software-pipelined by one 32-column sub-chunk: the TMEM read and the inbox loads
        // of sub-chunk j+1 are in flight while sub-chunk j is summed and stored, so each
        // latency is paid once per tile instead of once per sub-chunk. The accumulator is
        // released as soon as its last columns are in registers.
        const uint32_t tempty_a = a ? tempty_leader1 : tempty_leader0;
        const int64_t ocol0 = static_cast<int64_t>(t.nt) * BN;
        if (p.wire_f32)
          rs_epilogue_pipelined<true, 1>(p, taddr, inbox, dst_tile, rp, ocol0, row, valid, last, tempty_a);
        else
          rs_epilogue_pipelined<false, (kMode == MODE_STD || kMode == MODE_DP_GRAD) ? 4 : 2>(p, taddr, inbox, dst_tile, rp, ocol0, row, valid,
                                                                 last, tempty_a);
      }
      if (p.trace && lane == 0 && ew == 0 && tile_live)
        trace_rec(p, TR_EPI_LOOP, rank, t.step, lin, t_epi0, globaltimer());
      if (!last && tile_live) {
        pend[npend++] = flag_ptr(p, par, send_rank, slot_send, fidx);
        if (npend == kPend) publish();
        if (p.trace && lane == 0 && ew == 0) trace_rec(p, TR_FLAG, rank, t.step, lin, t_epi0, globaltimer());
      }
      if (kUpEpi && last && tile_live && p.done_rank[h]) {
        // completion flag for a pushed output tile (UP all-to-all)
        fence_sys();
        __syncwarp();
        if (lane == 0 && rank != p.fault_rank) st_relaxed_sys(p.done_rank[h] + fidx, ep);
      }
      if (p.trace && lane == 0 && ew == 0 && tile_live)
        trace_rec(p, TR_TILE, rank, t.step, lin, t_epi0, globaltimer());
    }
    publish();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm<512>(tmem_base);
  if (threadIdx.x == 0 && p.epoch_dev && p.epoch_bump) epoch_publish(p.epoch_dev, ep, exit_ctas);
}

template <int kOp, int kMode>
__global__ void __launch_bounds__(kThreads, 1) tpf_fused_kernel(const __grid_constant__ KParams p) {
  const int h = blockIdx.x / p.ctas_per_rank;  // hosted rank served by this CTA
  fused_body<kOp, kMode>(p, h, blockIdx.x - h * p.ctas_per_rank, gridDim.x);
}

// Split group: CTA block r * ctas_per_rank + g runs rank r's own (per-process) parameters.
template <int kOp, int kMode>
__global__ void __launch_bounds__(kThreads, 1) tpf_fused_group_kernel(const __grid_constant__ GroupParams gp) {
  const int r = blockIdx.x / gp.p[0].ctas_per_rank;
  if (r >= gp.n) return;  // (the grid is sized exactly; both CTAs of a pair share r)
  const KParams& p = gp.p[r];
  fused_body<kOp, kMode>(p, 0, blockIdx.x - r * p.ctas_per_rank, p.ctas_per_rank);
}

namespace {

// Function attributes are per device: set once per (instance, device), thread-safe.
template <typename F>
void once_per_device(uint64_t& done, F&& f) {
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!((done >> dev) & 1ull)) {
    f();
    done |= 1ull << dev;
  }
}

// TPF_PDL (A/B measurement switch): 0 plain stream order (griddepcontrol.wait then returns
// at once); 1 (default) trigger the next launch after the prologue; 2 after this CTA's last
// TMA load; 3 PDL launch without an explicit trigger (the next launch starts at exit).
int pdl_setting() {
  static const int v = [] {
    const char* e = std::getenv("TPF_PDL");
    return (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 1;
  }();
  return v;
}
bool pdl_enabled() { return pdl_setting() != 0; }
// TPF_PDL_FUSED=1 (A/B switch): the multi-rank GEMM instances launch with PDL too. Safe: a
// dependent grid's CTAs pass griddepcontrol.wait only once this grid has completed, so none of
// its cross-CTA waits can start before the whole grid is resident.
bool pdl_fused_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("TPF_PDL_FUSED");
    return e && e[0] == '1';
  }();
  return v;
}

template <int kOp, int kMode, typename Params>
cudaError_t launch_instance(const Params& p, int grid, cudaStream_t stream) {
  constexpr bool kGroup = std::is_same<Params, GroupParams>::value;
  void (*kern)(Params);
  if constexpr (kGroup)
    kern = tpf_fused_group_kernel<kOp, kMode>;
  else
    kern = tpf_fused_kernel<kOp, kMode>;
  static uint64_t attr_done = 0;
  static bool pool_ok[64];
  constexpr int kSmem = (kMode == MODE_RS_DIRECT || kMode == MODE_DP_DIRECT) ? kSmemBytesDirect
                        : (kOp == OP_AG && (kMode == MODE_STD || kMode == MODE_GATHER_B)) ? kSmemBytesFwd
                                                              : kSmemBytes;
  once_per_device(attr_done, [kern] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    // the setmaxnreg split must fit the register pool the launch allocates, or
    // setmaxnreg.inc blocks forever
    cudaFuncAttributes fa;
    int dev = 0;
    cudaGetDevice(&dev);
    pool_ok[dev & 63] = cudaFuncGetAttributes(&fa, kern) == cudaSuccess &&
                        fa.numRegs * kThreads >= 128 * kRegsCtl + 256 * kRegsEpi;
  });
  {
    int dev = 0;
    cudaGetDevice(&dev);
    if (!pool_ok[dev & 63]) return cudaErrorInvalidConfiguration;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // CTA pairs for tcgen05 cta_group::2
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // PDL: the prologue (barrier init, TMEM allocation, tensor-map prefetch) overlaps the
  // previous kernel's tail; the kernel waits (griddepcontrol.wait) before touching memory.
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  if constexpr (kGroup) {
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
  } else {
    const bool pdl = kMode == MODE_SINGLE ? pdl_enabled() : (pdl_instance(kMode) && pdl_fused_enabled());
    cfg.numAttrs = pdl ? 2 : 1;
    KParams q = p;
    q.pdl_trigger = pdl_setting() == 3 ? 0 : pdl_setting();
    return cudaLaunchKernelEx(&cfg, kern, q);
  }
}

}  // namespace

cudaError_t launch_fused(const KParams& p, int grid, cudaStream_t stream) {
  switch (p.mode) {
    case MODE_DP_GRAD: return launch_instance<OP_RS, MODE_DP_GRAD>(p, grid, stream);
    case MODE_GATHER_B: return launch_instance<OP_AG, MODE_GATHER_B>(p, grid, stream);
    case MODE_QK: return launch_instance<OP_RS, MODE_QK>(p, grid, stream);
    case MODE_PV: return launch_instance<OP_RS, MODE_PV>(p, grid, stream);
    case MODE_QSPLIT: return launch_instance<OP_RS, MODE_QSPLIT>(p, grid, stream);
    case MODE_RS_DIRECT: return launch_instance<OP_RS, MODE_RS_DIRECT>(p, grid, stream);
    case MODE_DP_DIRECT: return launch_instance<OP_RS, MODE_DP_DIRECT>(p, grid, stream);
    case MODE_SINGLE:
      return p.op == OP_AG ? launch_instance<OP_AG, MODE_SINGLE>(p, grid, stream)
                           : launch_instance<OP_RS, MODE_SINGLE>(p, grid, stream);
    default:
      return p.op == OP_AG ? launch_instance<OP_AG, MODE_STD>(p, grid, stream)
                           : launch_instance<OP_RS, MODE_STD>(p, grid, stream);
  }
}

cudaError_t launch_fused_group(const GroupParams& gp, int grid, cudaStream_t stream) {
  switch (gp.p[0].mode) {
    case MODE_STD:
      return gp.p[0].op == OP_AG ? launch_instance<OP_AG, MODE_STD>(gp, grid, stream)
                                 : launch_instance<OP_RS, MODE_STD>(gp, grid, stream);
    case MODE_DP_GRAD: return launch_instance<OP_RS, MODE_DP_GRAD>(gp, grid, stream);
    case MODE_GATHER_B: return launch_instance<OP_AG, MODE_GATHER_B>(gp, grid, stream);
    case MODE_RS_DIRECT: return launch_instance<OP_RS, MODE_RS_DIRECT>(gp, grid, stream);
    case MODE_DP_DIRECT: return launch_instance<OP_RS, MODE_DP_DIRECT>(gp, grid, stream);
    default: return cudaErrorInvalidValue;  // other instances are not split-group operations
  }
}

// Largest number of co-resident CTA pairs (all CTAs must be resident: spins on
// other CTAs' progress rely on it). All instances share block size and smem.
int max_pairs() {
  static std::mutex mu;
  static int cached[64];
  static uint64_t have = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if ((have >> dev) & 1ull) return cached[dev];
  cudaFuncSetAttribute(tpf_fused_kernel<OP_RS, MODE_STD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, tpf_fused_kernel<OP_RS, MODE_STD>, &cfg) != cudaSuccess) n = 0;
  if (n > 0) {
    cached[dev] = n;
    have |= 1ull << dev;
  }
  return n;
}

}  // namespace tpf
