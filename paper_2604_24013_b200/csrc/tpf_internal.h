// Internal (non-ABI) definitions shared by the host runtime (tpf_runtime.cu)
// and the sm_100a kernels (tpf_kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace tpf {

constexpr int kMaxRanks = 8;
constexpr int BM = 128;          // rows per CTA; the CTA pair computes 256 x BN (UMMA M = 256)
constexpr int BN = 256;          // UMMA N (each CTA of the pair stages BN/2 columns of B)
constexpr int BK = 64;           // 64 bf16 = one 128 B swizzle atom row
constexpr int kStages = 6;
constexpr int kThreads = 384;    // 12 warps: TMA, MMA, 2x comm, 2 x 4 epilogue (one group per accumulator)
constexpr int kRegPool = 168;    // registers per thread the launch allocates (__launch_bounds__(384, 1))
constexpr int kRegsCtl = 88;     // setmaxnreg: warps 0-3 (the AG producer / forwarders spill below 88)
constexpr int kRegsEpi = 208;    // setmaxnreg: epilogue warpgroups (128 * 88 + 256 * 208 == 384 * 168)
static_assert(128 * kRegsCtl + 256 * kRegsEpi <= kThreads * kRegPool, "setmaxnreg split exceeds the pool");
constexpr int kAStageBytes = BM * BK * 2;        // 16 KiB: also the AG wire "image" unit
constexpr int kBStageBytes = (BN / 2) * BK * 2;  // 16 KiB: this CTA's half of B
constexpr int kStageBytes = kAStageBytes + kBStageBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 512;  // + barriers
// Pairwise (MODE_RS_DIRECT) instance: one pipeline stage fewer, and behind the barriers a fold
// staging area per epilogue warpgroup (two buffers of T-1 <= 7 partials x one 16-B word column
// = 128 rows x 16 B = 2 KiB each).
constexpr int kStagesDirect = kStages - 1;
constexpr int kFoldUnit = BM * 16;                                  // 2 KiB
constexpr int kFoldGroupBytes = 2 * (kMaxRanks - 1) * kFoldUnit;    // 28 KiB per warpgroup
constexpr int kSmemBytesDirect = kStagesDirect * kStageBytes + 2048 + 2 * kFoldGroupBytes + 1024;
static_assert(kSmemBytesDirect <= 227 * 1024, "pairwise instance exceeds the shared-memory limit");
// AG-GEMM instances (MODE_STD, MODE_GATHER_B): two 16 KiB forwarder bounce buffers after 1 KiB of barriers
// (+ 1 KiB alignment slack; the kernel's 1 KiB of static shared memory counts against 227 KiB)
constexpr int kSmemBytesFwd = kStages * kStageBytes + 1024 + 2 * kAStageBytes + 1024;
static_assert(kSmemBytesFwd + 1024 <= 227 * 1024, "AG instance exceeds the shared-memory limit");

enum Op : int { OP_RS = 0, OP_AG = 1 };
enum Act : int { ACT_NONE = 0, ACT_SQUARE = 1, ACT_SWIGLU = 2 };
// Kernel instance (compile-time operand layout / epilogue variant).
enum Mode : int {
  MODE_STD = 0,       // A K-major (x rows), B MN-major (W (K, N)): TP AG-GEMM / GEMM-RS / GEMM
  MODE_DP_GRAD = 1,   // GEMM-RS with A MN-major (X^T from row-major X): DP gradient RS
  MODE_GATHER_B = 2,  // AG carrying B (K-major W rows): DP parameter all-gather
  MODE_QK = 3,        // B K-major, per batch (head); per-rank A row offset: UP scores
  MODE_PV = 4,        // B MN-major, per batch; merge_heads + peer push + flags: UP output
  MODE_SINGLE = 5,    // MODE_STD operands, T == 1 (no ring): the degenerate GEMM (+ epilogue act)
  MODE_QSPLIT = 6,    // GEMM-RS whose A slices are produced concurrently by the attention kernel:
                      // a step's tiles wait for their query slice's ready counter (Alg. 4)
  MODE_RS_DIRECT = 7, // MODE_STD GEMM-RS with the pairwise schedule's rs_direct fold (its own
                      // instance: the ring / circular MODE_STD instance carries no fold code)
  MODE_DP_DIRECT = 8, // MODE_DP_GRAD operands with the pairwise fold (the same split: the ring /
                      // circular DP instance carries no fold code)
};

// Blame table: a waiter that gives up on a peer flag (timeout, or the group aborting) records
// the rank it was blocked on, in every rank's table (system-scope stores into the symmetric
// heaps), so any rank's tpf_comm_sync can follow the chain waiter -> awaited -> ... to the rank
// that failed -- the reference's GroupError::failing_rank (fabric.hpp:22-31, 207-219), not a
// victim. Entry [waiter] = awaited + 1; a rank that failed itself (fault injection) stores its
// own rank + 1. The table sits at the end of the parity-1 flag block.
// Word kBlameAbort of the table is the group abort flag: the first waiter to time out sets it in
// every rank's table, and every rank's waiters give up at once (recording what they waited on)
// -- the reference's "other ranks blocked on receives are woken and unwound" (fabric.hpp:185-189)
// -- instead of each process draining garbage into its successors' waits.
constexpr int64_t kBlameBytes = 256;
constexpr int kBlameAbort = kMaxRanks;
struct Blame {
  uint32_t* table[kMaxRanks];  // every rank's table (peer-mapped); table[0] null: disabled
  int T;
};

// Error record in device memory (first error wins).
//   [0] code (0 ok, 1 peer-flag timeout, 2 mbarrier timeout)
//   [1] rank  [2] step  [3] tile / piece  [4] abort flag
constexpr int kErrWords = 8;

struct KParams {
  CUtensorMap tmap_a;  // A operand source (x), dims (K, rows, B, hosted ranks); MN-major A: (rows, K, B, ranks)
  CUtensorMap tmap_b;  // W, dims (N, K, hosted ranks), N contiguous (MN-major B); K-major B: (K, N, ranks)
  CUtensorMap tmap_wire[2];  // AG wire images per heap parity (128 B, 128 rows, image, slot, rank)
  int op;              // OP_RS (GEMM-RS, also the T == 1 GEMM) or OP_AG
  int mode;            // Mode (kernel instance)
  int T;               // group size
  int m;               // granularity (ring passes)
  int direct;          // 1: pairwise rs_direct fold; 0: pipelined (ring / circular)
  int n_hosted;        // ranks hosted by this launch (1 = one rank per GPU)
  int rank0;           // rank id of hosted rank 0
  int ctas_per_rank;   // CTAs serving one hosted rank (even: CTA pairs)
  int group_m;         // raster: m-block pairs that sweep the n-tiles together
  int group_n;         // raster (when > 0, instead of group_m): n-tiles that the m-block pairs sweep
  int l2_a, l2_b;      // TMA L2 eviction priority of the A / B loads: 0 normal, 1 evict_first, 2 evict_last
  int ag_batch;        // AG: forwarded images per fence + flag publication (clamped to 1..8)
  int act;             // AG epilogue activation (Act)
  int64_t out_ld;      // output row stride (elements)
  int64_t blk_cols;    // MODE_GATHER_B: columns of one rank's weight block (output column offset unit)
  // plain (T == 1) path extensions used by the UP attention pipeline
  int heads_merge;                    // >0: batch g -> (b = g / heads, hh = g % heads), column hh*N
  int64_t a_row_off[kMaxRanks];       // per hosted rank: A row offset (query slice)
  char* out_rank[kMaxRanks];          // per hosted rank: output base (may be a peer pointer)
  int64_t out_col_off[kMaxRanks];     // per hosted rank: output column offset
  uint32_t* done_rank[kMaxRanks];     // per hosted rank: per tile-warp completion flags (peer) or null
  int wire_f32;        // RS wire dtype: 1 fp32, 0 bf16
  int out_f32;         // output dtype: 1 fp32, 0 bf16
  int nmb_per_batch;   // ceil(Sc / BM)
  int nmb, nnt, nkb;   // m-blocks, n-tiles, k-blocks per step
  int npairs;          // ceil(nmb / 2): m-block pairs (one per CTA pair)
  int nsteps;          // T * m (1 when T == 1)
  int64_t Sc;          // rows of one sequence chunk, per batch row
  int64_t N;           // output columns
  int64_t x_rows;      // x rows per batch (RS: S, AG: S/T)
  int64_t out_rows;    // out rows per batch (RS: S/T, AG: S)
  char* out;
  int64_t out_rank_stride;
  char* sym[kMaxRanks];     // symmetric base of every rank, mapped in this process
  int64_t data_off[2];      // per parity: slot data region offset
  int64_t flag_off[2];      // per parity: flag region offset
  int64_t slot_bytes;       // one slot (one (pass, iteration) message)
  int64_t flags_per_slot;
  uint32_t epoch;      // static epoch / parity, used when epoch_dev is null (T == 1 calls)
  int parity;
  const uint32_t* qs_ready[kMaxRanks];  // MODE_QSPLIT: per hosted rank, per query slice counters
  uint32_t qs_target;                   // MODE_QSPLIT: counter value of a finished slice
  uint32_t* epoch_dev; // device epoch [value, exit counter]: read at entry (+ epoch_bump), and
  int epoch_bump;      // the last CTA to exit publishes the value (CUDA-graph replayable)
  int8_t sched[kMaxRanks][kMaxRanks][3];  // [rank][step] (send, recv, slice)
  uint32_t* err;
  int64_t timeout_ns;
  int fault_rank;   // test hook: this rank never publishes its flags (-1: none)
  int compute_only; // measurement: same tiles, no flag waits / wire traffic (exposed-comm baseline)
  int pdl_trigger;  // PDL instances: 1 trigger the next launch after the prologue, 2 after the last TMA load, 0 at exit
  // Optional device trace (%globaltimer ns): records of 4 x u64 appended via trace[0] counter.
  unsigned long long* trace;
  int64_t trace_cap;  // records
  Blame blame;
};

// Split group (tpf_comm_create_split_group): every rank's own per-process launch parameters
// (n_hosted = 1, rank0 = r, its own heap / epoch / error record), run as ONE launch of
// n * ctas_per_rank CTAs. Ranks whose kernels wait on each other must never be separate
// launches on one GPU (nothing makes them co-resident); one launch sized to the resident CTA
// pairs is.
struct GroupParams {
  KParams p[kMaxRanks];
  int n;
};

// trace record: {kind | rank << 8 | cta(block) << 16 | step << 32, index, t0, t1}
enum TraceKind : int {
  TR_TILE = 1,       // index = tile lin; t0 = accumulator ready (epilogue start), t1 = epilogue done
  TR_MAINLOOP = 2,   // index = tile lin; t0 = first stage issued, t1 = last stage issued (producer)
  TR_AG_PIECE = 3,   // index = piece;   t0 = source ready, t1 = flag published
  TR_WAIT_A = 4,     // index = tile lin*1024+kb; producer blocked on an AG wire image (t1-t0)
  TR_WAIT_IN = 5,    // index = tile lin; epilogue blocked on an RS inbox flag
  TR_FLAG = 6,       // index = tile lin; RS flag published to the successor at t1
  TR_FLUSH = 7,      // index = #flags; AG forwarder fence + flag publication (t1-t0)
  TR_EPI_LOOP = 8,   // index = tile lin; RS epilogue: t0 = accumulator ready, t1 = stores issued
  TR_PUBLISH = 9,    // index = #flags; RS epilogue system fence + flag publication (t1-t0)
};

// UP v2: fused flash-attention + output all-to-all (csrc/tpf_attention.cu)
struct FmhaParams {
  CUtensorMap tmap_q[2], tmap_k[2], tmap_v[2];  // per heap parity (a symmetric inbox differs per
                                                // parity; user buffers: both the same)
  int T, R, rank0, heads, G, nqt, nkv, ctas_per_rank;
  int local;                           // 1: plain attention into recv[rank] (no all-to-all)
  int64_t S, sl, fw;                   // fw = T * heads * Dh (output row stride, elements)
  float scale_log2;                    // softmax scale * log2(e)
  char* recv[2][kMaxRanks];            // [parity] every rank's receive buffer (peer-mapped)
  uint32_t* flags[2][kMaxRanks];       // [parity] every rank's flag block (peer-mapped)
  int64_t nflags_per_src;              // G * nqt * 4
  uint32_t epoch;                      // static epoch / parity when epoch_dev is null
  int parity;
  uint32_t* epoch_dev;                 // device epoch (see KParams)
  int epoch_bump;
  int qsplit;                          // query-split: local context in the RS schedule's slice
  int8_t slice_of[kMaxRanks][kMaxRanks];  // order ([hosted rank][step] -> slice), and one
  uint32_t* qs_ready[kMaxRanks];       // counter per (hosted rank, slice) bumped per finished warp
  int fault_rank;
  uint32_t* err;
  int64_t timeout_ns;
};

// Ulysses first all-to-all (tpf_ulysses.cu): sequence-sharded Q/K/V -> head-sharded.
struct UlyssesParams {
  const char* src[3];               // q, k, v of hosted rank 0: (B*H, sl, Dh) bf16
  int64_t src_rank_stride;          // bytes between hosted ranks' inputs
  char* dst[2][kMaxRanks];          // [parity] every rank's inbox: [q | k | v], each (B*hl, S, Dh)
  uint32_t* flags[2][kMaxRanks];    // [parity] every rank's a2a flag block: [src rank][cta]
  int64_t tensor_bytes;             // B*hl*S*Dh*2
  int64_t B, H, hl, S, sl, Dh;
  int T, R, rank0, ctas_per_rank;
  uint32_t* epoch_dev;              // device epoch: this launch opens the call (bump)
  int fault_rank;
};

void launch_ulysses_push(const UlyssesParams& p, cudaStream_t stream);
cudaError_t launch_fused(const KParams& p, int grid, cudaStream_t stream);
cudaError_t launch_fused_group(const GroupParams& gp, int grid, cudaStream_t stream);
cudaError_t launch_fmha_a2a(const FmhaParams& p, int grid, cudaStream_t stream);
void launch_softmax(const float* s, void* p, int64_t rows, int64_t cols, float scale, cudaStream_t st);
// Wait until flags[parity][0..n) >= epoch, epoch / parity read from epoch_dev (the call's
// current device epoch), or the given static epoch / flags[0] when epoch_dev is null.
// Flag i of the waited range belongs to source rank (first + i) / per_src (blame on give-up).
void launch_wait_flags2(const uint32_t* flags0, const uint32_t* flags1, int64_t n, const uint32_t* epoch_dev,
                        uint32_t epoch, int64_t timeout_ns, uint32_t* err, int rank, const Blame& blame,
                        int64_t first, int64_t per_src, cudaStream_t st);
// dst <- src[parity of the call's device epoch], `bytes` a multiple of 16.
void launch_copy_by_parity(void* dst, const void* src0, const void* src1, int64_t bytes, const uint32_t* epoch_dev,
                           cudaStream_t st);
void launch_wait_flags(const uint32_t* flags, int64_t n, uint32_t epoch, int64_t timeout_ns, uint32_t* err,
                       int rank, const Blame& blame, int64_t first, int64_t per_src, cudaStream_t st);
int max_pairs();
int num_sms();

}  // namespace tpf
