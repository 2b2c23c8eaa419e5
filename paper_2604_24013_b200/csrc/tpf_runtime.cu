// C-ABI implementation (include/tpf.h): communicator + symmetric heap over CUDA
// IPC, TMA descriptor construction, argument validation mirroring the
// reference's exceptions, and launch of the persistent fused kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "tpf.h"
#include "tpf_host.h"
#include "tpf_internal.h"

namespace {

thread_local std::string g_last_error;

int fail(const tpf::Status& s) {
  g_last_error = s.msg;
  return s.code;
}

#define TPF_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(tpf::Status::cuda(std::string(#expr) + ": " + cudaGetErrorString(e_))); \
  } while (0)

#define TPF_CUDA_TRY_STATUS(expr)                                                   \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return tpf::Status::cuda(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int64_t kFlagBytesPerParity = 1 << 20;  // 256 Ki flags per parity
// usable flag bytes per parity: the blame table (tpf::Blame) takes the end of the parity-1 block
constexpr int64_t kFlagCapBytes = kFlagBytesPerParity - tpf::kBlameBytes;
constexpr int64_t kBlameOff = 2 * kFlagBytesPerParity - tpf::kBlameBytes;
constexpr int64_t kDefaultTimeoutNs = 10ll * 1000 * 1000 * 1000;

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  const int x = (e && *e) ? std::atoi(e) : dflt;
  return x > 0 ? x : dflt;
}

// Raster: m-block pairs that sweep the n-tiles together (L2 reuse of B). 16 pairs =
// 32 m-blocks = 4096 rows: the 126 MB L2 holds that A panel plus the live B strips.
int env_group_m() {
  static int v = [] {
    const char* e = std::getenv("TPF_GROUP_M");
    const int x = (e && *e) ? std::atoi(e) : 16;
    return x > 0 ? x : 16;
  }();
  return v;
}

int64_t env_timeout_ns() {
  const char* v = std::getenv("TPF_TIMEOUT_MS");
  if (v && *v) return static_cast<int64_t>(std::atoll(v)) * 1000 * 1000;
  return kDefaultTimeoutNs;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// bf16 tensor map with SWIZZLE_128B and zero OOB fill. dims/strides inner -> outer;
// strides (bytes) for dims 1..rank-1.
tpf::Status make_tmap(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                      const uint64_t* strides, const uint32_t* box,
                      CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn enc = get_encode();
  if (!enc) return tpf::Status::cuda("cuTensorMapEncodeTiled unavailable (no CUDA driver)");
  if (reinterpret_cast<uintptr_t>(base) % 16)
    return tpf::Status::shape("tensor base address must be 16-byte aligned");
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i > 0) {
      s[i - 1] = strides[i - 1];
      if (strides[i - 1] % 16)
        return tpf::Status::shape("row pitch must be a multiple of 16 bytes (feature dims % 8 == 0)");
    }
  }
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, s, b,
                   e, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return tpf::Status::cuda("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return tpf::Status::ok();
}

uint32_t* default_err_buffer() {
  static uint32_t* buf = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaMalloc(&buf, tpf::kErrWords * sizeof(uint32_t)) == cudaSuccess)
      cudaMemset(buf, 0, tpf::kErrWords * sizeof(uint32_t));
    else
      buf = nullptr;
  });
  return buf;
}

}  // namespace

// Split group (tpf_comm_create_split_group): the per-rank launch parameters of one collective
// call, collected from every rank's call; the last rank's call launches them all as one grid.
struct SplitGroup {
  int world = 0;
  std::mutex mu;
  tpf::GroupParams gp;
  bool have[tpf::kMaxRanks] = {};
  int npending = 0;
  cudaStream_t stream = nullptr;
};

struct tpf_comm {
  int rank = 0;
  int world = 1;
  int local_group = 0;          // 1: all ranks hosted by this process (single GPU)
  size_t sym_bytes = 0;         // per rank
  char* local = nullptr;        // this process's allocation (all ranks if local_group)
  char* sym[tpf::kMaxRanks] = {};
  bool opened[tpf::kMaxRanks] = {};
  bool peers_ready = false;
  uint32_t* dev_epoch = nullptr;  // device epoch [value, exit counter] (graph-replayable calls)
  uint32_t* qs_ready = nullptr;   // query-split slice counters [hosted rank][slice]
  cudaStream_t side = nullptr;    // query-split: the GEMM-RS runs here, concurrently with attention
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint32_t* err = nullptr;      // device error record
  int64_t timeout_ns = kDefaultTimeoutNs;
  int device = 0;
  int fault_rank = -1;
  int compute_only = 0;
  char* scratch = nullptr;
  size_t scratch_bytes = 0;
  // Scratch buffers outgrown by a later call. A CUDA graph that captured an earlier call keeps
  // that call's scratch pointer, so an outgrown buffer is never freed before tpf_comm_destroy.
  std::vector<char*> retired;
  unsigned long long* trace = nullptr;
  int64_t trace_cap = 0;
  int is_virtual = 0;            // tpf_comm_create_virtual (peers alias the own heap: no blame)
  int failing_rank = -1;         // resolved by the last tpf_comm_sync that reported TPF_E_PEER
  std::shared_ptr<SplitGroup> group;  // tpf_comm_create_split_group: shared deferred launch
};

namespace {

struct Geometry {
  int nmb_per_batch, nmb, nnt, nkb, npairs;
  int64_t Sc;
};

Geometry geometry(int64_t B, int64_t Sc, int64_t K, int64_t N) {
  Geometry g;
  g.Sc = Sc;
  g.nmb_per_batch = static_cast<int>(ceil_div(Sc, tpf::BM));
  g.nmb = static_cast<int>(B) * g.nmb_per_batch;
  g.nnt = static_cast<int>(ceil_div(N, tpf::BN));
  g.nkb = static_cast<int>(ceil_div(K, tpf::BK));
  g.npairs = static_cast<int>(B) * ((g.nmb_per_batch + 1) / 2);  // pairs stay within a batch
  return g;
}

int64_t data_bytes_per_parity(size_t sym_bytes) {
  return (static_cast<int64_t>(sym_bytes) - 2 * kFlagBytesPerParity) / 2;
}

// The unfused attention fallback reads the device epoch back to the host to build its
// multi-launch pointers, which a captured CUDA graph cannot replay. It refuses capture
// loudly (everything else keeps the epoch on the device and is graph-replayable).
tpf::Status check_not_capturing(const tpf_comm* c, cudaStream_t stream) {
  if (!c || c->world <= 1) return tpf::Status::ok();
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone)
    return tpf::Status::invalid("the unfused attention fallback (head_dim != 128) cannot be captured into a "
                                "CUDA graph (host-side epoch read); use head_dim 128 or call it eagerly");
  return tpf::Status::ok();
}

struct Call {
  int op, T, m, direct, act, wire_f32, out_f32, n_hosted, rank0;
  int64_t B, Sc, K, N, x_rows, out_rows;
  int64_t N_gemm;  // columns of W (B operand); == N unless the epilogue narrows (SwiGLU)
  int a_mn;        // x is stored (K, rows): A = x^T read MN-major (DP: X^T dY without a transpose)
  int b_kmajor;    // w is stored (N, K) (PyTorch Linear layout): K-major B
  int gather_b;    // AG ring carries weight column blocks (DP param all-gather)
  int64_t out_ld;  // output row stride (0: N)
  int b_batched;   // w is per batch block: (R, B, rowsW, colsW)
  int heads_merge;
  int64_t a_row_off[tpf::kMaxRanks];
  char* out_rank[tpf::kMaxRanks];
  int64_t out_col_off[tpf::kMaxRanks];
  uint32_t* done_rank[tpf::kMaxRanks];
  bool no_epoch;   // do not advance the epoch (steps of one multi-launch collective)
  int max_pairs_per_rank;                        // 0: all resident CTA pairs
  const uint32_t* qs_ready[tpf::kMaxRanks];      // non-null: MODE_QSPLIT (A slices from the attention)
  uint32_t qs_target;
  const void* x;
  const void* w;
  void* out;
  const int32_t* sched;  // T*T*3 or null (T == 1)
};

// Split group: record rank c->rank's launch parameters; the call of the group's last rank
// launches every rank's parameters as one grid (n * ctas_per_rank CTAs, all resident).
tpf::Status group_submit(tpf_comm* c, const tpf::KParams& p, cudaStream_t stream) {
  SplitGroup& G = *c->group;
  std::lock_guard<std::mutex> lock(G.mu);
  auto reset = [&G] {
    for (int r = 0; r < tpf::kMaxRanks; ++r) G.have[r] = false;
    G.npending = 0;
  };
  if (G.have[c->rank]) {
    reset();
    return tpf::Status::invalid("split group: rank " + std::to_string(c->rank) +
                                " made a second call before every rank made the first (calls are collective)");
  }
  if (G.npending > 0) {
    int first = 0;
    while (!G.have[first]) ++first;
    const tpf::KParams& f = G.gp.p[first];
    if (f.op != p.op || f.mode != p.mode || f.T != p.T || f.m != p.m || f.nmb != p.nmb || f.nnt != p.nnt ||
        f.nkb != p.nkb || f.direct != p.direct || f.wire_f32 != p.wire_f32 || f.ctas_per_rank != p.ctas_per_rank) {
      reset();
      return tpf::Status::invalid("split group: rank " + std::to_string(c->rank) +
                                  " made a different collective call than rank " + std::to_string(first));
    }
    if (stream != G.stream) {
      reset();
      return tpf::Status::invalid("split group: every rank must issue the call on the same stream");
    }
  }
  G.gp.p[c->rank] = p;
  G.have[c->rank] = true;
  G.stream = stream;
  if (++G.npending < G.world) return tpf::Status::ok();
  G.gp.n = G.world;
  reset();
  cudaError_t e = tpf::launch_fused_group(G.gp, p.ctas_per_rank * G.world, stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return tpf::Status::cuda(std::string("split-group launch: ") + cudaGetErrorString(e));
  return tpf::Status::ok();
}

tpf::Status launch(tpf_comm* c, const Call& k, cudaStream_t stream) {
  tpf::KParams p;
  std::memset(&p, 0, sizeof(p));
  const int64_t NG = k.N_gemm > 0 ? k.N_gemm : k.N;
  const Geometry g = geometry(k.B, k.Sc, k.K, NG);
  const int R = k.n_hosted;
  const int64_t x_rank_stride = k.B * k.x_rows * k.K * 2;
  const int64_t w_rank_stride = k.K * NG * 2 * (k.b_batched ? k.B : 1);
  const int64_t esz = k.out_f32 ? 4 : 2;
  if (k.a_mn) {
    const uint64_t dims[4] = {static_cast<uint64_t>(k.x_rows), static_cast<uint64_t>(k.K),
                              static_cast<uint64_t>(k.B), static_cast<uint64_t>(R)};
    const uint64_t strides[3] = {static_cast<uint64_t>(k.x_rows * 2),
                                 static_cast<uint64_t>(k.x_rows * k.K * 2),
                                 static_cast<uint64_t>(x_rank_stride)};
    const uint32_t box[4] = {64, tpf::BK, 1, 1};
    tpf::Status s = make_tmap(&p.tmap_a, k.x, 4, dims, strides, box);
    if (!s.good()) return s;
  } else {
    const uint64_t dims[4] = {static_cast<uint64_t>(k.K), static_cast<uint64_t>(k.x_rows),
                              static_cast<uint64_t>(k.B), static_cast<uint64_t>(R)};
    const uint64_t strides[3] = {static_cast<uint64_t>(k.K * 2),
                                 static_cast<uint64_t>(k.x_rows * k.K * 2),
                                 static_cast<uint64_t>(x_rank_stride)};
    const uint32_t box[4] = {tpf::BK, tpf::BM, 1, 1};
    tpf::Status s = make_tmap(&p.tmap_a, k.x, 4, dims, strides, box);
    if (!s.good()) return s;
  }
  const int64_t out_ld = k.out_ld > 0 ? k.out_ld : k.N;
  if (k.b_batched) {
    const bool km = k.b_kmajor != 0;
    const uint64_t d0 = km ? k.K : NG, d1 = km ? NG : k.K;
    const uint64_t dims[4] = {d0, d1, static_cast<uint64_t>(k.B), static_cast<uint64_t>(R)};
    const uint64_t strides[3] = {d0 * 2, d0 * d1 * 2, static_cast<uint64_t>(w_rank_stride)};
    const uint32_t box[4] = {km ? static_cast<uint32_t>(tpf::BK) : 64u, km ? static_cast<uint32_t>(tpf::BN / 2) : static_cast<uint32_t>(tpf::BK), 1, 1};
    tpf::Status s = make_tmap(&p.tmap_b, k.w, 4, dims, strides, box);
    if (!s.good()) return s;
  } else if (k.b_kmajor || k.gather_b) {
    const uint64_t dims[3] = {static_cast<uint64_t>(k.K), static_cast<uint64_t>(NG),
                              static_cast<uint64_t>(R)};
    const uint64_t strides[2] = {static_cast<uint64_t>(k.K * 2), static_cast<uint64_t>(w_rank_stride)};
    const uint32_t box[3] = {tpf::BK, tpf::BN / 2, 1};
    tpf::Status s = make_tmap(&p.tmap_b, k.w, 3, dims, strides, box);
    if (!s.good()) return s;
  } else {
    const uint64_t dims[3] = {static_cast<uint64_t>(NG), static_cast<uint64_t>(k.K),
                              static_cast<uint64_t>(R)};
    const uint64_t strides[2] = {static_cast<uint64_t>(NG * 2),
                                 static_cast<uint64_t>(w_rank_stride)};
    const uint32_t box[3] = {64, tpf::BK, 1};
    tpf::Status s = make_tmap(&p.tmap_b, k.w, 3, dims, strides, box);
    if (!s.good()) return s;
  }
  p.op = k.op;
  p.mode = k.a_mn ? tpf::MODE_DP_GRAD
         : k.gather_b ? tpf::MODE_GATHER_B
         : (k.b_batched && k.b_kmajor) ? tpf::MODE_QK
         : k.b_batched ? tpf::MODE_PV
         : k.qs_ready[0] ? tpf::MODE_QSPLIT
         : k.T == 1 ? tpf::MODE_SINGLE
         : tpf::MODE_STD;
  if (p.mode == tpf::MODE_STD && k.op == tpf::OP_RS && k.direct) p.mode = tpf::MODE_RS_DIRECT;
  if (p.mode == tpf::MODE_DP_GRAD && k.direct) p.mode = tpf::MODE_DP_DIRECT;
  if ((p.mode == tpf::MODE_STD || p.mode == tpf::MODE_SINGLE) && k.b_kmajor)
    return tpf::Status::invalid("internal: K-major B is only instantiated for the DP / UP modes");
  p.T = k.T;
  p.m = k.m;
  p.direct = k.direct;
  p.n_hosted = R;
  p.rank0 = k.rank0;
  p.act = k.act;
  p.out_ld = out_ld;
  p.blk_cols = k.N;
  p.heads_merge = k.heads_merge;
  for (int r = 0; r < tpf::kMaxRanks; ++r) {
    p.a_row_off[r] = k.a_row_off[r];
    p.out_rank[r] = k.out_rank[r];
    p.out_col_off[r] = k.out_col_off[r];
    p.done_rank[r] = k.done_rank[r];
  }
  p.wire_f32 = k.wire_f32;
  p.out_f32 = k.out_f32;
  p.nmb_per_batch = g.nmb_per_batch;
  p.nmb = g.nmb;
  p.nnt = g.nnt;
  p.nkb = g.nkb;
  p.npairs = g.npairs;
  for (int h = 0; h < R; ++h) p.qs_ready[h] = k.qs_ready[h];
  p.qs_target = k.qs_target;
  // Raster and L2 residency. Multi-rank instances: groups of 16 m-block pairs sweep the
  // n-tiles. T == 1 GEMMs (measured on the bench block, tools/l2_probe.py, profiles/r02_l2_raster.txt):
  // narrow N (fewer n-tiles than m-block pairs, e.g. the 8192x14336x4096 down projection):
  // half the n-tiles are swept by every m-block pair with that B slab marked evict_last
  // (-3.5% time, -22% DRAM bytes); otherwise the m-group's A panels are marked evict_last.
  p.group_m = env_group_m();
  p.group_n = 0;
  p.l2_a = p.l2_b = 0;
  if (p.mode == tpf::MODE_SINGLE) {
    if (g.nnt < g.npairs) {
      p.group_n = std::max(1, g.nnt / 2);
      p.l2_b = 2;
    } else {
      p.l2_a = 2;
    }
  }
  if (const char* e = std::getenv("TPF_GROUP_N")) p.group_n = std::atoi(e);  // dev A/B overrides
  if (const char* e = std::getenv("TPF_L2_A")) p.l2_a = std::atoi(e);
  if (const char* e = std::getenv("TPF_L2_B")) p.l2_b = std::atoi(e);
  p.ag_batch = env_int("TPF_AG_BATCH", 4);
  p.nsteps = k.T * k.m;
  p.Sc = k.Sc;
  p.N = k.N;
  p.x_rows = k.x_rows;
  p.out_rows = k.out_rows;
  p.out = static_cast<char*>(k.out);
  p.out_rank_stride = k.B * k.out_rows * out_ld * esz;
  p.timeout_ns = c ? c->timeout_ns : kDefaultTimeoutNs;
  p.fault_rank = c ? c->fault_rank : -1;
  p.compute_only = c ? c->compute_only : 0;
  p.trace = c ? c->trace : nullptr;
  p.trace_cap = c ? c->trace_cap : 0;
  if (k.T > 1) {
    for (int r = 0; r < k.T; ++r)
      for (int i = 0; i < k.T; ++i)
        for (int f = 0; f < 3; ++f)
          p.sched[r][i][f] = static_cast<int8_t>(k.sched[(r * k.T + i) * 3 + f]);
    const int nslots = k.m * (k.T - 1);
    int64_t slot_bytes, flags_per_slot;
    if (k.op == tpf::OP_RS) {
      slot_bytes = static_cast<int64_t>(g.nmb) * g.nnt * tpf::BM * tpf::BN * (k.wire_f32 ? 4 : 2);
      flags_per_slot = static_cast<int64_t>(g.nmb) * g.nnt * 4;
    } else {
      // AG wire images: A rows per (m-block, k-block), or (gather_b) B halves per (half, n-tile, k-block)
      const int64_t nimg = k.gather_b ? 2ll * g.nnt * g.nkb : static_cast<int64_t>(g.nmb) * g.nkb;
      slot_bytes = nimg * tpf::kAStageBytes;
      flags_per_slot = nimg;
    }
    const int64_t data_cap = data_bytes_per_parity(c->sym_bytes);
    if (nslots * slot_bytes > data_cap)
      return tpf::Status::capacity("symmetric heap too small: call needs " +
                                   std::to_string(2 * (nslots * slot_bytes) + 2 * kFlagBytesPerParity) +
                                   " bytes per rank, communicator has " + std::to_string(c->sym_bytes));
    if (nslots * flags_per_slot * 4 > kFlagCapBytes)
      return tpf::Status::capacity("too many flags for one call");
    for (int r = 0; r < k.T; ++r) p.sym[r] = c->sym[r];
    p.flag_off[0] = 0;
    p.flag_off[1] = kFlagBytesPerParity;
    p.data_off[0] = 2 * kFlagBytesPerParity;
    p.data_off[1] = 2 * kFlagBytesPerParity + data_cap;
    p.slot_bytes = slot_bytes;
    p.flags_per_slot = flags_per_slot;
    if (k.op == tpf::OP_AG) {
      // AG wire images of the hosted ranks' local slots: (128 B, 128 rows, image, slot, rank),
      // one map per heap parity (the kernel picks by the device epoch)
      const int64_t rank_stride = R > 1 ? static_cast<int64_t>(c->sym_bytes) : nslots * slot_bytes;
      const uint64_t dims[5] = {64, tpf::BM, static_cast<uint64_t>(flags_per_slot),
                                static_cast<uint64_t>(nslots), static_cast<uint64_t>(R)};
      const uint64_t strides[4] = {128, tpf::kAStageBytes, static_cast<uint64_t>(slot_bytes),
                                   static_cast<uint64_t>(rank_stride)};
      const uint32_t box[5] = {64, tpf::BM, 1, 1, 1};
      for (int par = 0; par < 2; ++par) {
        tpf::Status s = make_tmap(&p.tmap_wire[par], c->sym[k.rank0] + p.data_off[par], 5, dims, strides, box,
                                  CU_TENSOR_MAP_SWIZZLE_NONE);
        if (!s.good()) return s;
      }
    }
    if (!c->is_virtual) {
      p.blame.T = k.T;
      for (int x = 0; x < k.T; ++x) p.blame.table[x] = reinterpret_cast<uint32_t*>(c->sym[x] + kBlameOff);
    }
    // epoch: in device memory, advanced by the launch that opens the call
    p.epoch_dev = c->dev_epoch;
    p.epoch_bump = k.no_epoch ? 0 : 1;
    p.epoch = 0;
    p.parity = 0;
  } else {
    p.sched[0][0][0] = -1;
    p.sched[0][0][1] = -1;
    p.sched[0][0][2] = 0;
    // single-rank step: no ring flags; a step of a multi-launch collective (UP fallback)
    // publishes done flags with the call's current device epoch
    p.epoch_dev = (c && k.no_epoch) ? c->dev_epoch : nullptr;
    p.epoch_bump = 0;
    p.epoch = 1;
    p.parity = 0;
  }
  p.err = c ? c->err : default_err_buffer();
  if (!p.err) return tpf::Status::cuda("no device error buffer (CUDA unavailable)");

  const int sms = tpf::num_sms();
  if (sms <= 0) return tpf::Status::cuda("no CUDA device");
  int pairs = tpf::max_pairs();
  if (pairs <= 0) return tpf::Status::cuda("kernel cannot be resident (cluster occupancy 0)");
  pairs = std::min(pairs, sms / 2);
  // a split group's ranks share this GPU's SMs like a local group's hosted ranks
  const int share = (c && c->group) ? c->world : R;
  int pairs_per_rank = pairs / share;
  if (k.max_pairs_per_rank > 0) pairs_per_rank = std::min(pairs_per_rank, k.max_pairs_per_rank);
  if (pairs_per_rank < 1)
    return tpf::Status::invalid("local group of " + std::to_string(share) + " ranks needs " +
                                std::to_string(share) + " resident CTA pairs, device has " +
                                std::to_string(pairs));
  p.ctas_per_rank = 2 * pairs_per_rank;
  if (c && c->group && k.T > 1) return group_submit(c, p, stream);
  cudaError_t e = tpf::launch_fused(p, p.ctas_per_rank * R, stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return tpf::Status::cuda(std::string("kernel launch: ") + cudaGetErrorString(e));
  return tpf::Status::ok();
}

int hosted(const tpf_comm* c) { return c->local_group ? c->world : 1; }

// Blame tables of every rank of c's group (disabled for T == 1 and the virtual group).
tpf::Blame blame_of(const tpf_comm* c) {
  tpf::Blame b;
  std::memset(&b, 0, sizeof(b));
  if (!c || c->world <= 1 || c->is_virtual) return b;
  b.T = c->world;
  for (int x = 0; x < c->world; ++x) b.table[x] = reinterpret_cast<uint32_t*>(c->sym[x] + kBlameOff);
  return b;
}

// The attention paths are multi-launch sequences; a split group defers single launches only.
tpf::Status check_not_split(const tpf_comm* c, const char* what) {
  if (c && c->group && c->world > 1)
    return tpf::Status::invalid(std::string(what) + " is not available on a split group (fused GEMM ops only)");
  return tpf::Status::ok();
}

tpf::Status check_ready(const tpf_comm* c) {
  if (!c) return tpf::Status::invalid("null communicator");
  int dev = -1;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != c->device)
    return tpf::Status::invalid("communicator was created on device " + std::to_string(c->device) +
                                " but the current device is " + std::to_string(dev));
  if (c->world > 1 && !c->peers_ready)
    return tpf::Status::invalid("communicator peers not opened (call tpf_comm_open_peers)");
  return tpf::Status::ok();
}

// Device resources of a communicator: the symmetric heap (heap_bytes, zeroed), the error
// record, the device epoch, the query-split counters, the side stream and its fork / join
// events. On failure the caller releases what was allocated with tpf_comm_destroy.
cudaError_t alloc_comm_resources(tpf_comm* c, size_t heap_bytes) {
  cudaGetDevice(&c->device);
  cudaError_t e = cudaMalloc(&c->local, heap_bytes);
  if (e == cudaSuccess) e = cudaMemset(c->local, 0, heap_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->err, tpf::kErrWords * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(c->err, 0, tpf::kErrWords * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->dev_epoch, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(c->dev_epoch, 0, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->qs_ready, tpf::kMaxRanks * tpf::kMaxRanks * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e;
}

// Make c->scratch at least `bytes`. An outgrown buffer is retired, not freed: a CUDA graph that
// captured an earlier call still addresses it, and replays may interleave with eager calls of
// other shapes. Growing inside a stream capture is refused (cudaMalloc is not a
// capturable operation): make one eager call of the largest shape before capturing.
tpf::Status grow_scratch(tpf_comm* c, size_t bytes, cudaStream_t stream) {
  if (c->scratch_bytes >= bytes) return tpf::Status::ok();
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone)
    return tpf::Status::invalid("attention scratch must grow to " + std::to_string(bytes) +
                                " bytes inside a CUDA graph capture; make one eager call of this shape first");
  char* p = nullptr;
  TPF_CUDA_TRY_STATUS(cudaMalloc(&p, bytes));
  if (c->scratch) c->retired.push_back(c->scratch);
  c->scratch = p;
  c->scratch_bytes = bytes;
  return tpf::Status::ok();
}

}  // namespace

namespace tpf {
int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}
}  // namespace tpf

extern "C" {

int tpf_version(void) { return 1; }

const char* tpf_last_error(void) { return g_last_error.c_str(); }

int tpf_device_sms(void) { return tpf::num_sms(); }

int tpf_ring_indices(int rs, int r, int i, int n, int32_t out[3]) {
  tpf::Status s = tpf::ring_indices(rs != 0, r, i, n, out);
  return s.good() ? TPF_OK : fail(s);
}

int tpf_schedule_build(int kind, int n, int32_t* out) {
  std::vector<int32_t> t;
  tpf::Status s = tpf::build_schedule(kind, n, t);
  if (!s.good()) return fail(s);
  if (!t.empty()) std::memcpy(out, t.data(), t.size() * sizeof(int32_t));
  return TPF_OK;
}

int tpf_schedule_check(int kind, int n, const int32_t* table) {
  tpf::Status s = tpf::check_schedule(kind, n, table);
  return s.good() ? TPF_OK : fail(s);
}

int tpf_comm_create(int rank, int world, size_t sym_bytes, tpf_comm** out) {
  if (!out) return fail(tpf::Status::invalid("null output pointer"));
  if (world < 1 || world > tpf::kMaxRanks || rank < 0 || rank >= world)
    return fail(tpf::Status::invalid("tpf_comm_create: rank " + std::to_string(rank) +
                                     " / world " + std::to_string(world) + " out of range (world <= 8)"));
  if (static_cast<int64_t>(sym_bytes) < 2 * kFlagBytesPerParity + 2 * 4096)
    sym_bytes = 2 * kFlagBytesPerParity + 2 * 4096;
  sym_bytes = (sym_bytes + 4095) & ~static_cast<size_t>(4095);
  tpf_comm* c = new tpf_comm();
  c->rank = rank;
  c->world = world;
  c->sym_bytes = sym_bytes;
  c->timeout_ns = env_timeout_ns();
  const cudaError_t e = alloc_comm_resources(c, sym_bytes);
  if (e != cudaSuccess) {
    tpf_comm_destroy(c);  // releases whatever was allocated so far
    return fail(tpf::Status::cuda(std::string("tpf_comm_create: ") + cudaGetErrorString(e)));
  }
  c->sym[rank] = c->local;
  c->peers_ready = (world == 1);
  *out = c;
  return TPF_OK;
}

int tpf_comm_ipc_handle(tpf_comm* c, void* handle_out) {
  if (!c || c->local_group) return fail(tpf::Status::invalid("ipc handle: not a per-process communicator"));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == TPF_IPC_HANDLE_BYTES, "IPC handle size");
  TPF_CUDA_TRY(cudaIpcGetMemHandle(&h, c->local));
  std::memcpy(handle_out, &h, sizeof(h));
  return TPF_OK;
}

int tpf_comm_open_peers(tpf_comm* c, const void* handles) {
  if (!c || c->local_group) return fail(tpf::Status::invalid("open peers: not a per-process communicator"));
  const char* hb = static_cast<const char*>(handles);
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank || c->opened[r]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + r * TPF_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    TPF_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->sym[r] = static_cast<char*>(p);
    c->opened[r] = true;
  }
  c->peers_ready = true;
  return TPF_OK;
}

int tpf_comm_create_local_group(int world, size_t sym_bytes_per_rank, tpf_comm** out) {
  if (!out) return fail(tpf::Status::invalid("null output pointer"));
  if (world < 1 || world > tpf::kMaxRanks)
    return fail(tpf::Status::invalid("tpf_comm_create_local_group: world out of range (1..8)"));
  size_t per = std::max<size_t>(sym_bytes_per_rank, 2 * kFlagBytesPerParity + 2 * 4096);
  per = (per + 4095) & ~static_cast<size_t>(4095);
  tpf_comm* c = new tpf_comm();
  c->rank = 0;
  c->world = world;
  c->local_group = 1;
  c->sym_bytes = per;
  c->timeout_ns = env_timeout_ns();
  const cudaError_t e = alloc_comm_resources(c, per * world);
  if (e != cudaSuccess) {
    tpf_comm_destroy(c);  // releases whatever was allocated so far
    return fail(tpf::Status::cuda(std::string("tpf_comm_create_local_group: ") + cudaGetErrorString(e)));
  }
  for (int r = 0; r < world; ++r) c->sym[r] = c->local + per * r;
  c->peers_ready = true;
  *out = c;
  return TPF_OK;
}

int tpf_comm_create_virtual(int world, size_t sym_bytes, tpf_comm** out) {
  // Measurement tool: rank 0 of a `world`-rank group on this GPU, with every peer virtual.
  // Peer heaps alias this rank's own heap (a self-ring), so a send lands in this rank's inbox
  // slot of the same index -- the slot the real successor would fill -- and is read one step
  // later while still L2-resident, as data arriving over NVLink would be. Every flag a step
  // waits on is written by this rank's own previous-step send in the same call, so every
  // wait is real from the first call on (flags start at zero like any communicator's). The
  // kernels run the real protocol instructions at full-GPU scale, which measures what one GPU
  // of a TP group computes; the results are well defined (tests/test_gpu_virtual.py): the AG
  // gathers the own slice at every step, the GEMM-RS sums the GEMMs of every row slice.
  tpf_comm* c = nullptr;
  int rc = tpf_comm_create(0, world, sym_bytes, &c);
  if (rc != TPF_OK) return rc;
  c->is_virtual = 1;
  for (int r = 1; r < world; ++r) c->sym[r] = c->local;
  c->peers_ready = true;
  *out = c;
  return TPF_OK;
}

int tpf_comm_create_split_group(int world, size_t sym_bytes, tpf_comm** comms) {
  if (!comms) return fail(tpf::Status::invalid("null output pointer"));
  if (world < 1 || world > tpf::kMaxRanks)
    return fail(tpf::Status::invalid("tpf_comm_create_split_group: world out of range (1..8)"));
  auto group = std::make_shared<SplitGroup>();
  group->world = world;
  for (int r = 0; r < world; ++r) {
    comms[r] = nullptr;
    const int rc = tpf_comm_create(r, world, sym_bytes, &comms[r]);
    if (rc != TPF_OK) {
      const std::string msg = g_last_error;
      for (int q = 0; q < r; ++q) tpf_comm_destroy(comms[q]);
      g_last_error = msg;
      return rc;
    }
    comms[r]->group = group;
  }
  // peers: the other communicators' heaps, as tpf_comm_open_peers maps them over CUDA IPC
  for (int r = 0; r < world; ++r) {
    for (int x = 0; x < world; ++x) comms[r]->sym[x] = comms[x]->local;
    comms[r]->peers_ready = true;
  }
  return TPF_OK;
}

int tpf_comm_destroy(tpf_comm* c) {
  if (!c) return TPF_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (c->opened[r]) cudaIpcCloseMemHandle(c->sym[r]);
  if (c->local) cudaFree(c->local);
  if (c->err) cudaFree(c->err);
  if (c->dev_epoch) cudaFree(c->dev_epoch);
  if (c->qs_ready) cudaFree(c->qs_ready);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->scratch) cudaFree(c->scratch);
  for (char* r : c->retired) cudaFree(r);
  delete c;
  return TPF_OK;
}

int tpf_comm_rank(const tpf_comm* c) { return c ? c->rank : -1; }
int tpf_comm_failing_rank(const tpf_comm* c) { return c ? c->failing_rank : -1; }
int tpf_comm_world(const tpf_comm* c) { return c ? c->world : -1; }

int tpf_comm_device(const tpf_comm* c) { return c ? c->device : -1; }

int tpf_comm_set_timeout_ns(tpf_comm* c, int64_t ns) {
  if (!c) return fail(tpf::Status::invalid("null communicator"));
  c->timeout_ns = ns > 0 ? ns : env_timeout_ns();
  return TPF_OK;
}

int tpf_comm_set_trace(tpf_comm* c, void* buffer, int64_t capacity_records) {
  if (!c) return fail(tpf::Status::invalid("null communicator"));
  c->trace = static_cast<unsigned long long*>(buffer);
  c->trace_cap = buffer ? capacity_records : 0;
  return TPF_OK;
}

int tpf_comm_set_compute_only(tpf_comm* c, int on) {
  if (!c) return fail(tpf::Status::invalid("null communicator"));
  c->compute_only = on ? 1 : 0;
  return TPF_OK;
}

int tpf_comm_inject_fault(tpf_comm* c, int rank) {
  if (!c) return fail(tpf::Status::invalid("null communicator"));
  if (rank < -1 || rank >= c->world) return fail(tpf::Status::invalid("inject_fault: rank out of range"));
  c->fault_rank = rank;
  return TPF_OK;
}

int tpf_comm_sync(tpf_comm* c, void* stream) {
  if (!c) return fail(tpf::Status::invalid("null communicator"));
  if (c->group) {
    // Ranks may run on their own threads (spawn_group): wait, bounded by the peer timeout, until
    // every rank has made the pending call and the group launch has been issued.
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
      int pending;
      {
        std::lock_guard<std::mutex> lock(c->group->mu);
        pending = c->group->npending;
      }
      if (pending == 0) break;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(c->timeout_ns))
        return fail(tpf::Status::invalid("split group: a collective call is still waiting for " +
                                         std::to_string(c->world - pending) + " rank(s) to make it"));
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  TPF_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  uint32_t rec[tpf::kErrWords];
  TPF_CUDA_TRY(cudaMemcpy(rec, c->err, sizeof(rec), cudaMemcpyDeviceToHost));
  if (rec[0] == 0 && c->world > 1 && !c->is_virtual) {
    // A rank that did not fail this call may still hold blame entries or the group abort flag
    // written by the others (or its own fault-injection mark): clear them for the next call.
    char* own = c->local_group ? c->local : c->sym[c->rank];
    uint32_t tab[tpf::kBlameBytes / 4];
    TPF_CUDA_TRY(cudaMemcpy(tab, own + kBlameOff, sizeof(tab), cudaMemcpyDeviceToHost));
    bool dirty = false;
    for (uint32_t v : tab) dirty |= v != 0;
    if (dirty) {
      const int nheaps = c->local_group ? c->world : 1;
      for (int h = 0; h < nheaps; ++h)
        TPF_CUDA_TRY(cudaMemset((c->local_group ? c->sym[h] : own) + kBlameOff, 0, tpf::kBlameBytes));
    }
  }
  if (rec[0] != 0) {
    TPF_CUDA_TRY(cudaMemset(c->err, 0, sizeof(rec)));
    const int waiter = static_cast<int>(rec[1]);
    // Follow the blame chain (tpf::Blame) from the rank that timed out to the rank that failed:
    // waiter -> the rank it waited on -> ... until a rank that was not blocked (it failed
    // without recording, e.g. a dead process) or that named itself. Peers in other processes
    // record their give-ups within microseconds of ours; a short grace covers the race.
    int culprit = waiter;
    uint32_t tab[tpf::kMaxRanks] = {};
    const bool have_tables = c->world > 1 && !c->is_virtual;
    if (have_tables) {
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
      char* own = c->local_group ? c->local : c->sym[c->rank];
      TPF_CUDA_TRY(cudaMemcpy(tab, own + kBlameOff, sizeof(tab), cudaMemcpyDeviceToHost));
      int r = waiter;  // -1: a pipeline-barrier timeout, no waiter to start the chain from
      for (int n = 0; r >= 0 && r < c->world && n <= c->world && tab[r] != 0; ++n) {
        const int a = static_cast<int>(tab[r]) - 1;
        if (a == r || a < 0 || a >= c->world) break;
        r = a;
      }
      // A rank that marked itself failed is the failing rank, whatever the waiters' links say
      // (they are recorded as each waiter gives up, and a late give-up can leave a gap).
      for (int x = 0; x < c->world; ++x)
        if (tab[x] == static_cast<uint32_t>(x + 1)) r = x;
      culprit = r;
      const int nheaps = c->local_group ? c->world : 1;
      for (int h = 0; h < nheaps; ++h)
        TPF_CUDA_TRY(cudaMemset((c->local_group ? c->sym[h] : own) + kBlameOff, 0, tpf::kBlameBytes));
    }
    c->failing_rank = culprit;
    std::string what = rec[0] == 1 ? "peer flag wait timed out" : "pipeline barrier timed out";
    return fail(tpf::Status::peer("rank " + std::to_string(culprit) + " failed: " + what + " (rank " +
                                  std::to_string(waiter) + " gave up at step " +
                                  std::to_string(static_cast<int>(rec[2])) + ", tile " +
                                  std::to_string(static_cast<int>(rec[3])) + ")"));
  }
  return TPF_OK;
}

int64_t tpf_sym_bytes_ag(int world, int64_t B, int64_t S, int64_t K, int64_t N_local, int m) {
  if (world <= 1) return 0;
  const Geometry g = geometry(B, S / world / std::max(m, 1), K, N_local);
  const int64_t slot = static_cast<int64_t>(g.nmb) * g.nkb * tpf::kAStageBytes;
  return 2 * kFlagBytesPerParity + 2 * static_cast<int64_t>(m) * (world - 1) * slot;
}

int64_t tpf_sym_bytes_dp_ag(int world, int64_t K, int64_t N_local) {
  if (world <= 1) return 0;
  const int64_t slot = 2 * ceil_div(N_local, tpf::BN) * ceil_div(K, tpf::BK) * tpf::kAStageBytes;
  return 2 * kFlagBytesPerParity + 2 * static_cast<int64_t>(world - 1) * slot;
}

int64_t tpf_sym_bytes_ulysses(int world, int64_t batch, int64_t heads_total, int64_t S, int64_t Dh) {
  // attention output area (every rank's (batch, S/T, heads_total*Dh) bf16 inbox), then the
  // first all-to-all inbox [q | k | v] of this rank's head group, per parity
  if (world < 1 || S % world || heads_total % world) return -1;
  const int64_t sl = S / world, hl = heads_total / world;
  const int64_t out_area = batch * sl * heads_total * Dh * 2;
  const int64_t inbox = 3 * batch * hl * S * Dh * 2;
  return 2 * (((out_area + 4095) / 4096) * 4096 + inbox) + 2 * kFlagBytesPerParity + 8192;
}

int64_t tpf_sym_bytes_rs(int world, int64_t B, int64_t S, int64_t K_local, int64_t N, int m,
                         int wire_dtype) {
  if (world <= 1) return 0;
  const Geometry g = geometry(B, S / world / std::max(m, 1), K_local, N);
  const int64_t slot =
      static_cast<int64_t>(g.nmb) * g.nnt * tpf::BM * tpf::BN * (wire_dtype == TPF_F32 ? 4 : 2);
  return 2 * kFlagBytesPerParity + 2 * static_cast<int64_t>(m) * (world - 1) * slot;
}

int tpf_dp_grad_rs(tpf_comm* c, const void* X, const void* dY, void* dW, int64_t M_local, int64_t K,
                   int64_t N, int kind, int m, int wire_dtype, int out_dtype, void* stream) {
  tpf::Status s = check_ready(c);
  if (!s.good()) return fail(s);
  const int T = c->world;
  if (m < 1) return fail(tpf::Status::invalid("fuse_reduce_scatter: granularity must be >= 1"));
  if (m > 1 && kind != TPF_RING)
    return fail(tpf::Status::invalid(
        "fuse_reduce_scatter: granularity > 1 is supported for the ring schedule only"));
  std::vector<int32_t> sched;
  s = tpf::build_schedule(kind, T, sched);
  if (!s.good()) return fail(s);
  if (M_local < 1 || K < 1 || N < 1)
    return fail(tpf::Status::shape("dp_grad_rs: dimensions must be positive"));
  if (T > 1 && K % (static_cast<int64_t>(T) * m))
    return fail(tpf::Status::invalid("fuse_reduce_scatter: sequence length " + std::to_string(K) +
                                     " is not divisible by " + std::to_string(T * m) + " (group size " +
                                     std::to_string(T) + " x granularity " + std::to_string(m) + ")"));
  if (K % 8 || N % 8) return fail(tpf::Status::shape("dp_grad_rs: K and N must be multiples of 8"));
  Call k{};
  k.op = tpf::OP_RS;
  k.T = T;
  k.m = T > 1 ? m : 1;
  k.direct = kind == TPF_PAIRWISE;
  k.wire_f32 = wire_dtype == TPF_F32;
  k.out_f32 = out_dtype == TPF_F32;
  k.n_hosted = hosted(c);
  k.rank0 = c->local_group ? 0 : c->rank;
  k.a_mn = 1;
  // x = X_r^T seen as (1, K, M_local): "sequence" rows = K (dW rows), reduction = M_local
  k.B = 1; k.Sc = K / (static_cast<int64_t>(T) * k.m); k.K = M_local; k.N = N;
  k.x_rows = K; k.out_rows = K / T;
  k.x = X; k.w = dY; k.out = dW;
  k.sched = T > 1 ? sched.data() : nullptr;
  s = launch(c, k, static_cast<cudaStream_t>(stream));
  return s.good() ? TPF_OK : fail(s);
}

int tpf_dp_param_ag_gemm(tpf_comm* c, const void* x, const void* w_rows, void* out, int64_t M_local,
                         int64_t K, int64_t N_local, int out_dtype, void* stream) {
  tpf::Status s = check_ready(c);
  if (!s.good()) return fail(s);
  const int T = c->world;
  if (M_local < 1 || K < 1 || N_local < 1)
    return fail(tpf::Status::shape("dp_param_ag_gemm: dimensions must be positive"));
  if (K % 8 || N_local % 8) return fail(tpf::Status::shape("dp_param_ag_gemm: K and N_local must be multiples of 8"));
  std::vector<int32_t> sched;
  Call k{};
  k.op = tpf::OP_AG;
  k.T = T;
  k.m = 1;
  k.out_f32 = out_dtype == TPF_F32;
  k.n_hosted = hosted(c);
  k.rank0 = c->local_group ? 0 : c->rank;
  k.gather_b = 1;
  k.b_kmajor = 1;
  k.B = 1; k.Sc = M_local; k.K = K; k.N = N_local; k.x_rows = M_local; k.out_rows = M_local;
  k.out_ld = N_local * T;
  k.x = x; k.w = w_rows; k.out = out;
  if (T > 1) {
    sched.resize(static_cast<size_t>(T) * T * 3);
    for (int r = 0; r < T; ++r)
      for (int i = 0; i < T; ++i) tpf::ring_indices(false, r, i, T, &sched[(r * T + i) * 3]);
    k.sched = sched.data();
  }
  s = launch(c, k, static_cast<cudaStream_t>(stream));
  return s.good() ? TPF_OK : fail(s);
}

// Fused flash attention + output all-to-all (UP v2, Dh = 128). q/k/v: (G, S, 128) bf16 per hosted
// rank, hosted ranks `rstride` bytes apart; qkv1 (may equal qkv) are the inputs to use when the
// call's heap parity is 1 (a symmetric inbox). `bump`: this launch opens the call (advances the
// device epoch); otherwise an earlier launch of the call did.
static tpf::Status fmha_a2a_v2(tpf_comm* c, const void* const qkv[3], const void* const qkv1[3], uint64_t rstride,
                               void* out, int64_t batch, int64_t heads, int64_t S, int bump, int scale,
                               cudaStream_t stream) {
  const int T = c->world;
  const int R = hosted(c);
  const int r0 = c->local_group ? 0 : c->rank;
  const int64_t Dh = 128, G = batch * heads, sl = S / T, fw = static_cast<int64_t>(T) * heads * Dh;
  const int64_t recv_bytes = batch * sl * fw * 2;
  const int64_t nflags2 = G * (sl / 128) * 4;
  if (nflags2 * T * 4 > kFlagCapBytes || recv_bytes > data_bytes_per_parity(c->sym_bytes))
    return tpf::Status::capacity("symmetric heap too small for the attention all-to-all");
  auto recv_at = [&](int rank, int par) {
    return c->sym[rank] + 2 * kFlagBytesPerParity + par * data_bytes_per_parity(c->sym_bytes);
  };
  auto flags_at = [&](int rank, int par) {
    return reinterpret_cast<uint32_t*>(c->sym[rank] + par * kFlagBytesPerParity);
  };
  tpf::FmhaParams fp;
  std::memset(&fp, 0, sizeof(fp));
  const uint64_t dims[4] = {static_cast<uint64_t>(Dh), static_cast<uint64_t>(S), static_cast<uint64_t>(G),
                            static_cast<uint64_t>(R)};
  const uint64_t strides[3] = {static_cast<uint64_t>(Dh * 2), static_cast<uint64_t>(S * Dh * 2), rstride};
  const uint32_t box[4] = {64, 128, 1, 1};
  tpf::Status s;
  for (int par = 0; par < 2 && s.good(); ++par) {
    const void* const* in = par ? qkv1 : qkv;
    s = make_tmap(&fp.tmap_q[par], in[0], 4, dims, strides, box);
    if (s.good()) s = make_tmap(&fp.tmap_k[par], in[1], 4, dims, strides, box);
    if (s.good()) s = make_tmap(&fp.tmap_v[par], in[2], 4, dims, strides, box);
  }
  if (!s.good()) return s;
  fp.T = T; fp.R = R; fp.rank0 = r0; fp.heads = static_cast<int>(heads); fp.G = static_cast<int>(G);
  fp.nqt = static_cast<int>(sl / 128); fp.nkv = static_cast<int>(S / 128);
  fp.S = S; fp.sl = sl; fp.fw = fw;
  fp.scale_log2 = (scale ? 1.0f / std::sqrt(static_cast<float>(Dh)) : 1.0f) * 1.4426950408889634f;
  for (int par = 0; par < 2; ++par)
    for (int x = 0; x < T; ++x) {
      fp.recv[par][x] = recv_at(x, par);
      fp.flags[par][x] = flags_at(x, par);
    }
  fp.nflags_per_src = nflags2;
  fp.epoch_dev = c->dev_epoch;
  fp.epoch_bump = bump;
  fp.fault_rank = c->fault_rank;
  fp.err = c->err;
  fp.timeout_ns = c->timeout_ns;
  const int sms = tpf::num_sms();
  fp.ctas_per_rank = std::max(1, sms / R);
  TPF_CUDA_TRY_STATUS(tpf::launch_fmha_a2a(fp, fp.ctas_per_rank * R, stream));
  for (int hh = 0; hh < R; ++hh) {
    const int rank = r0 + hh;
    uint32_t* f0 = flags_at(rank, 0);
    uint32_t* f1 = flags_at(rank, 1);
    if (!c->is_virtual) {  // virtual group: the only source is this rank (self-ring), nothing comes in
      tpf::launch_wait_flags2(f0, f1, static_cast<int64_t>(rank) * nflags2, c->dev_epoch, 0, c->timeout_ns, c->err,
                              rank, blame_of(c), 0, nflags2, stream);
      const int64_t off = static_cast<int64_t>(rank + 1) * nflags2;
      tpf::launch_wait_flags2(f0 + off, f1 + off, static_cast<int64_t>(T - 1 - rank) * nflags2, c->dev_epoch, 0,
                              c->timeout_ns, c->err, rank, blame_of(c), off, nflags2, stream);
    }
    tpf::launch_copy_by_parity(static_cast<char*>(out) + hh * recv_bytes, recv_at(rank, 0), recv_at(rank, 1),
                               recv_bytes, c->dev_epoch, stream);
  }
  TPF_CUDA_TRY_STATUS(cudaGetLastError());
  return tpf::Status::ok();
}

int tpf_attention_a2a(tpf_comm* c, const void* q, const void* k, const void* v, void* out, int64_t batch,
                      int64_t heads, int64_t S, int64_t Dh, int scale, void* stream_v) {
  // fuse_all_to_all_attention (Alg. 5, layers.cpp:174-218) on the GEMM kernel family.
  tpf::Status s = check_ready(c);
  if (s.good()) s = check_not_split(c, "tpf_attention_a2a");
  if (!s.good()) return fail(s);
  const int T = c->world;
  if (batch < 1 || heads < 1 || S < 1 || Dh < 1)
    return fail(tpf::Status::invalid("attention inputs need batch >= 1, heads >= 1"));
  if (S % T)
    return fail(tpf::Status::invalid("fuse_all_to_all_attention: sequence length " + std::to_string(S) +
                                     " is not divisible by group size " + std::to_string(T)));
  if (Dh % 8 || S % 8) return fail(tpf::Status::shape("attention: head_dim and seq must be multiples of 8"));
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const int R = hosted(c);
  const int r0 = c->local_group ? 0 : c->rank;
  const int64_t G = batch * heads, sl = S / T, fw = static_cast<int64_t>(T) * heads * Dh;
  const Geometry gpv = geometry(G, sl, S, Dh);
  const int64_t nflags = static_cast<int64_t>(gpv.nmb) * gpv.nnt * 4;  // per source rank
  const int64_t recv_bytes = batch * sl * fw * 2;
  if (nflags * T * 4 > kFlagCapBytes || recv_bytes > data_bytes_per_parity(c->sym_bytes))
    return fail(tpf::Status::capacity("symmetric heap too small for the attention all-to-all"));
  auto recv_at = [&](int rank, int par) {
    return c->sym[rank] + 2 * kFlagBytesPerParity + par * data_bytes_per_parity(c->sym_bytes);
  };
  auto flags_at = [&](int rank, int par) {
    return reinterpret_cast<uint32_t*>(c->sym[rank] + par * kFlagBytesPerParity);
  };
  if (Dh == 128 && sl % 128 == 0) {
    // v2: one persistent fused flash-attention launch for all steps / heads / hosted ranks
    const void* qkv[3] = {q, k, v};
    s = fmha_a2a_v2(c, qkv, qkv, static_cast<uint64_t>(G * S * Dh * 2), out, batch, heads, S, /*bump=*/1, scale,
                    stream);
    return s.good() ? TPF_OK : fail(s);
  }
  // v1 (any head_dim): scores fp32 (R, G, sl, S), probabilities bf16 (R, G, sl, S).
  // Not graph-capturable (host-side epoch read, scratch allocation): refuse before any work.
  {
    const tpf::Status cs = check_not_capturing(c, stream);
    if (!cs.good()) return fail(cs);
  }
  const size_t sc_bytes = static_cast<size_t>(R) * G * sl * S * 4, pb_bytes = sc_bytes / 2;
  s = grow_scratch(c, sc_bytes + pb_bytes, stream);
  if (!s.good()) return fail(s);
  float* scores = reinterpret_cast<float*>(c->scratch);
  char* probs = c->scratch + sc_bytes;
  // This multi-launch fallback computes parity-specific pointers on the host, so it opens
  // the call by reading and advancing the device epoch synchronously (not graph-capturable).
  uint32_t epoch = 0;
  TPF_CUDA_TRY(cudaStreamSynchronize(stream));
  TPF_CUDA_TRY(cudaMemcpy(&epoch, c->dev_epoch, sizeof(epoch), cudaMemcpyDeviceToHost));
  epoch += 1;
  TPF_CUDA_TRY(cudaMemcpy(c->dev_epoch, &epoch, sizeof(epoch), cudaMemcpyHostToDevice));
  const int par = static_cast<int>(epoch & 1u);
  auto recv_of = [&](int rank) { return c->sym[rank] + 2 * kFlagBytesPerParity + par * data_bytes_per_parity(c->sym_bytes); };
  auto flags_of = [&](int rank) {
    return reinterpret_cast<uint32_t*>(c->sym[rank] + par * kFlagBytesPerParity);
  };
  for (int i = 0; i < T; ++i) {
    // 1) scores = Q[slice l] K^T for every head (K-major B = K itself, batched per head)
    Call qk{};
    qk.op = tpf::OP_RS; qk.T = 1; qk.m = 1; qk.out_f32 = 1; qk.n_hosted = R; qk.rank0 = r0;
    qk.B = G; qk.Sc = sl; qk.K = Dh; qk.N = S; qk.x_rows = S; qk.out_rows = sl;
    qk.x = q; qk.w = k; qk.out = scores; qk.b_kmajor = 1; qk.b_batched = 1; qk.no_epoch = true;
    for (int h = 0; h < R; ++h) qk.a_row_off[h] = static_cast<int64_t>((r0 + h + i + 1) % T) * sl;
    s = launch(c, qk, stream);
    if (!s.good()) return fail(s);
    // 2) P = softmax(scale * scores) rows
    tpf::launch_softmax(scores, probs, static_cast<int64_t>(R) * G * sl, S,
                        scale ? 1.0f / std::sqrt(static_cast<float>(Dh)) : 1.0f, stream);
    // 3) O = P V, epilogue pushes each tile to the slice owner's receive buffer at the
    //    source rank's feature block (merge_heads + concat_feat fused) and flags it.
    Call pv{};
    pv.op = tpf::OP_RS; pv.T = 1; pv.m = 1; pv.out_f32 = 0; pv.n_hosted = R; pv.rank0 = r0;
    pv.B = G; pv.Sc = sl; pv.K = S; pv.N = Dh; pv.x_rows = sl; pv.out_rows = sl;
    pv.x = probs; pv.w = v; pv.out = out; pv.b_batched = 1; pv.heads_merge = static_cast<int>(heads);
    pv.out_ld = fw; pv.no_epoch = true;
    for (int h = 0; h < R; ++h) {
      const int rank = r0 + h, dst = (rank + i + 1) % T;
      pv.out_rank[h] = recv_of(dst);
      pv.out_col_off[h] = static_cast<int64_t>(rank) * heads * Dh;
      pv.done_rank[h] = dst == rank ? nullptr : flags_of(dst) + rank * nflags;
    }
    s = launch(c, pv, stream);
    if (!s.good()) return fail(s);
  }
  // 4) wait for the T-1 incoming parts (flags are indexed by source rank; the own part
  //    was written locally in the last step), then hand the assembled slice to the caller.
  for (int h = 0; h < R; ++h) {
    const int rank = r0 + h;
    uint32_t* f = flags_of(rank);
    if (!c->is_virtual) {  // virtual group: the only source is this rank (self-ring), nothing comes in
      tpf::launch_wait_flags(f, static_cast<int64_t>(rank) * nflags, epoch, c->timeout_ns, c->err, rank, blame_of(c),
                             0, nflags, stream);
      tpf::launch_wait_flags(f + static_cast<int64_t>(rank + 1) * nflags, static_cast<int64_t>(T - 1 - rank) * nflags,
                             epoch, c->timeout_ns, c->err, rank, blame_of(c), static_cast<int64_t>(rank + 1) * nflags,
                             nflags, stream);
    }
    TPF_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(out) + h * recv_bytes, recv_of(rank), recv_bytes,
                                 cudaMemcpyDeviceToDevice, stream));
  }
  TPF_CUDA_TRY(cudaGetLastError());
  return TPF_OK;
}

int tpf_query_split_attention(tpf_comm* c, const void* q, const void* k, const void* v, const void* w_o,
                              void* out, int64_t batch, int64_t heads, int64_t S, int64_t Dh, int64_t D, int kind,
                              int wire_dtype, int out_dtype, int scale, void* stream_v) {
  // query_split_attention (Alg. 4, layers.cpp:149-172): context = merge_heads(attention(q, k, v))
  // for every query slice (fused tcgen05 flash attention, local output), then the fused
  // GEMM-RS over the row-sharded output projection with the schedule's reduction order.
  tpf::Status s = check_ready(c);
  if (s.good()) s = check_not_split(c, "tpf_query_split_attention");
  if (!s.good()) return fail(s);
  const int T = c->world;
  std::vector<int32_t> sched;
  s = tpf::build_schedule(kind, T, sched);
  if (!s.good()) return fail(s);
  if (batch < 1 || heads < 1 || S < 1 || D < 1)
    return fail(tpf::Status::invalid("attention inputs need batch >= 1, heads >= 1"));
  if (T > 1 && S % T)
    return fail(tpf::Status::invalid("fuse_reduce_scatter: sequence length " + std::to_string(S) +
                                     " is not divisible by " + std::to_string(T) + " (group size " +
                                     std::to_string(T) + " x granularity 1)"));
  if (Dh != 128 || S % 128 || D % 8)
    return fail(tpf::Status::shape("query_split_attention: needs head_dim 128, seq % 128 == 0, d % 8 == 0"));
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const int R = hosted(c);
  const int r0 = c->local_group ? 0 : c->rank;
  const int64_t G = batch * heads, hd = heads * Dh;
  const size_t ctx_bytes = static_cast<size_t>(R) * batch * S * hd * 2;
  s = grow_scratch(c, ctx_bytes, stream);
  if (!s.good()) return fail(s);
  tpf::FmhaParams fp;
  std::memset(&fp, 0, sizeof(fp));
  const uint64_t dims[4] = {static_cast<uint64_t>(Dh), static_cast<uint64_t>(S), static_cast<uint64_t>(G),
                            static_cast<uint64_t>(R)};
  const uint64_t strides[3] = {static_cast<uint64_t>(Dh * 2), static_cast<uint64_t>(S * Dh * 2),
                               static_cast<uint64_t>(G * S * Dh * 2)};
  const uint32_t box[4] = {64, 128, 1, 1};
  for (int par = 0; par < 2 && s.good(); ++par) {  // user buffers: both parities the same
    s = make_tmap(&fp.tmap_q[par], q, 4, dims, strides, box);
    if (s.good()) s = make_tmap(&fp.tmap_k[par], k, 4, dims, strides, box);
    if (s.good()) s = make_tmap(&fp.tmap_v[par], v, 4, dims, strides, box);
  }
  if (!s.good()) return fail(s);
  fp.R = R; fp.rank0 = r0; fp.heads = static_cast<int>(heads); fp.G = static_cast<int>(G);
  fp.local = 1;
  fp.nkv = static_cast<int>(S / 128);
  fp.S = S; fp.fw = hd;
  fp.scale_log2 = (scale ? 1.0f / std::sqrt(static_cast<float>(Dh)) : 1.0f) * 1.4426950408889634f;
  for (int hh = 0; hh < R; ++hh)
    fp.recv[0][r0 + hh] = fp.recv[1][r0 + hh] = c->scratch + static_cast<size_t>(hh) * batch * S * hd * 2;
  fp.epoch_dev = nullptr;  // local attention: no flags; the GEMM-RS below opens the call
  fp.err = c->err;
  fp.timeout_ns = c->timeout_ns;
  fp.fault_rank = -1;
  Call kc{};
  kc.op = tpf::OP_RS;
  kc.T = T;
  kc.m = 1;
  kc.direct = kind == TPF_PAIRWISE;
  kc.wire_f32 = wire_dtype == TPF_F32;
  kc.out_f32 = out_dtype == TPF_F32;
  kc.n_hosted = R;
  kc.rank0 = r0;
  kc.B = batch; kc.Sc = S / T; kc.K = hd; kc.N = D; kc.x_rows = S; kc.out_rows = S / T;
  kc.x = c->scratch; kc.w = w_o; kc.out = out;
  kc.sched = T > 1 ? sched.data() : nullptr;
  const int sms = tpf::num_sms();
  const int64_t sl = S / T;
  // Alg. 4 proper: the attention produces the query slices in the RS schedule's order on part
  // of the SMs while the GEMM-RS consumes them on the rest, so each step's projection and
  // transfer ride under the attention of the next slices. The split follows the work ratio.
  const double attn_t = 4.0 * G * S * S * Dh * 1.15, proj_t = 2.0 * batch * S * hd * D;
  const int per_rank = sms / R;
  int rs_pairs = static_cast<int>(std::lround(proj_t / (attn_t + proj_t) * per_rank / 2.0));
  rs_pairs = std::max(1, std::min(rs_pairs, per_rank / 2 - 1));
  const int fmha_ctas = per_rank - 2 * rs_pairs;
  const bool concurrent = T > 1 && sl % 128 == 0 && fmha_ctas >= 1 && env_int("TPF_QSPLIT_CONCURRENT", 1) != 0;
  if (!concurrent) {
    fp.T = 1; fp.sl = S; fp.nqt = static_cast<int>(S / 128);
    fp.ctas_per_rank = std::max(1, per_rank);
    TPF_CUDA_TRY(tpf::launch_fmha_a2a(fp, fp.ctas_per_rank * R, stream));
    s = launch(c, kc, stream);
    return s.good() ? TPF_OK : fail(s);
  }
  fp.T = T; fp.sl = sl; fp.nqt = static_cast<int>(sl / 128);
  fp.qsplit = 1;
  for (int hh = 0; hh < R; ++hh) {
    for (int i = 0; i < T; ++i) fp.slice_of[hh][i] = static_cast<int8_t>(sched[((r0 + hh) * T + i) * 3 + 2]);
    fp.qs_ready[hh] = c->qs_ready + hh * tpf::kMaxRanks;
    kc.qs_ready[hh] = fp.qs_ready[hh];
  }
  kc.qs_target = static_cast<uint32_t>(G * ((fp.nqt + 1) / 2) * 8);  // items x 2 tiles x 4 warps
  kc.max_pairs_per_rank = rs_pairs;
  fp.ctas_per_rank = fmha_ctas;
  TPF_CUDA_TRY(cudaMemsetAsync(c->qs_ready, 0, tpf::kMaxRanks * tpf::kMaxRanks * sizeof(uint32_t), stream));
  TPF_CUDA_TRY(cudaEventRecord(c->ev_fork, stream));
  TPF_CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  TPF_CUDA_TRY(tpf::launch_fmha_a2a(fp, fp.ctas_per_rank * R, stream));
  // Deadlock-free by construction: the attention never waits on the GEMM-RS, so every CTA of
  // it finishes even if some GEMM-RS clusters only become resident after it.
  s = launch(c, kc, c->side);
  if (!s.good()) return fail(s);
  TPF_CUDA_TRY(cudaEventRecord(c->ev_join, c->side));
  TPF_CUDA_TRY(cudaStreamWaitEvent(stream, c->ev_join, 0));
  return TPF_OK;
}

int tpf_gemm(const void* a, const void* b, void* out, int64_t M, int64_t K, int64_t N,
             int out_dtype, void* stream) {
  if (M < 1 || K < 1 || N < 1) return fail(tpf::Status::shape("tpf_gemm: dimensions must be positive"));
  if (K % 8 || N % 8) return fail(tpf::Status::shape("tpf_gemm: K and N must be multiples of 8"));
  Call k{};
  k.op = tpf::OP_RS;
  k.T = 1; k.m = 1; k.n_hosted = 1;
  k.out_f32 = out_dtype == TPF_F32;
  k.B = 1; k.Sc = M; k.K = K; k.N = N; k.x_rows = M; k.out_rows = M;
  k.x = a; k.w = b; k.out = out;
  tpf::Status s = launch(nullptr, k, static_cast<cudaStream_t>(stream));
  return s.good() ? TPF_OK : fail(s);
}

int tpf_ag_gemm(tpf_comm* c, const void* x, const void* w, void* out, int64_t B, int64_t S,
                int64_t K, int64_t N_local, int m, int act, int out_dtype, void* stream) {
  // fuse_all_gather argument checks (collectives.cpp:239-248), in reference order.
  if (m < 1) return fail(tpf::Status::invalid("fuse_all_gather: granularity must be >= 1"));
  tpf::Status s = check_ready(c);
  if (!s.good()) return fail(s);
  const int T = c->world;
  if (B < 1 || S < 1 || K < 1 || N_local < 1)
    return fail(tpf::Status::shape("column_parallel_forward: dimensions must be positive"));
  if (S % T)
    return fail(tpf::Status::invalid("column_parallel_forward: sequence length " + std::to_string(S) +
                                     " is not divisible by group size " + std::to_string(T)));
  const int64_t sl = S / T;
  if (T > 1 && sl % m)
    return fail(tpf::Status::invalid("fuse_all_gather: slice length " + std::to_string(sl) +
                                     " is not divisible by granularity " + std::to_string(m)));
  if (K % 8 || N_local % 8)
    return fail(tpf::Status::shape("column_parallel_forward: K and N_local must be multiples of 8"));
  if (act < TPF_ACT_NONE || act > TPF_ACT_SWIGLU)
    return fail(tpf::Status::invalid("column_parallel_forward: unknown activation"));
  if (act == TPF_ACT_SWIGLU && N_local % tpf::BN)
    return fail(tpf::Status::shape("SwiGLU epilogue needs the tile-interleaved gate||up shard with "
                                   "N_local a multiple of 256"));
  std::vector<int32_t> sched;
  Call k{};
  k.op = tpf::OP_AG;
  k.T = T;
  k.m = T > 1 ? m : 1;
  k.act = act;
  k.out_f32 = out_dtype == TPF_F32;
  k.n_hosted = hosted(c);
  k.rank0 = c->local_group ? 0 : c->rank;
  k.B = B; k.Sc = T > 1 ? sl / m : S; k.K = K; k.x_rows = sl; k.out_rows = S;
  k.N_gemm = N_local;
  k.N = act == TPF_ACT_SWIGLU ? N_local / 2 : N_local;
  k.x = x; k.w = w; k.out = out;
  if (T > 1) {
    sched.resize(static_cast<size_t>(T) * T * 3);
    for (int r = 0; r < T; ++r)
      for (int i = 0; i < T; ++i) tpf::ring_indices(false, r, i, T, &sched[(r * T + i) * 3]);
    k.sched = sched.data();
  }
  s = launch(c, k, static_cast<cudaStream_t>(stream));
  return s.good() ? TPF_OK : fail(s);
}

int tpf_gemm_rs(tpf_comm* c, const void* x, const void* w, void* out, int64_t B, int64_t S,
                int64_t K_local, int64_t N, int kind, int m, int wire_dtype, int out_dtype,
                void* stream) {
  tpf::Status s = check_ready(c);
  if (!s.good()) return fail(s);
  const int T = c->world;
  // fuse_reduce_scatter argument checks (collectives.cpp:365-386), in reference order.
  if (m < 1) return fail(tpf::Status::invalid("fuse_reduce_scatter: granularity must be >= 1"));
  if (m > 1 && kind != TPF_RING)
    return fail(tpf::Status::invalid(
        "fuse_reduce_scatter: granularity > 1 is supported for the ring schedule only"));
  std::vector<int32_t> sched;
  s = tpf::build_schedule(kind, T, sched);
  if (!s.good()) return fail(s);
  if (B < 1 || S < 1 || K_local < 1 || N < 1)
    return fail(tpf::Status::shape("row_parallel_forward: dimensions must be positive"));
  if (T > 1 && S % (static_cast<int64_t>(T) * m))
    return fail(tpf::Status::invalid("fuse_reduce_scatter: sequence length " + std::to_string(S) +
                                     " is not divisible by " + std::to_string(T * m) + " (group size " +
                                     std::to_string(T) + " x granularity " + std::to_string(m) + ")"));
  if (K_local % 8 || N % 8)
    return fail(tpf::Status::shape("row_parallel_forward: K_local and N must be multiples of 8"));
  Call k{};
  k.op = tpf::OP_RS;
  k.T = T;
  k.m = T > 1 ? m : 1;
  k.direct = kind == TPF_PAIRWISE;
  k.wire_f32 = wire_dtype == TPF_F32;
  k.out_f32 = out_dtype == TPF_F32;
  k.n_hosted = hosted(c);
  k.rank0 = c->local_group ? 0 : c->rank;
  k.B = B; k.Sc = S / (static_cast<int64_t>(T) * k.m); k.K = K_local; k.N = N;
  k.x_rows = S; k.out_rows = S / T;
  k.x = x; k.w = w; k.out = out;
  k.sched = T > 1 ? sched.data() : nullptr;
  s = launch(c, k, static_cast<cudaStream_t>(stream));
  return s.good() ? TPF_OK : fail(s);
}

}  // extern "C"

// ---------------------------------------------------------------- Ulysses (UP end to end)
// First all-to-all (sequence-sharded -> head-sharded Q/K/V, peer stores into every rank's
// symmetric inbox), then the fused flash attention whose epilogue performs the second
// all-to-all (fuse_all_to_all_attention). Inbox layout per parity, after the attention's
// output area: [q | k | v], each (batch*heads_local, S, Dh) bf16. The a2a flags sit after
// the attention's flags in the same parity block: [source rank][cta].
// Opens the call (the push kernel advances the device epoch). inbox_local[par] receives this
// process's hosted rank 0 inbox for heap parity par.
static tpf::Status ulysses_first_a2a(tpf_comm* c, const void* q, const void* k, const void* v, int64_t batch,
                                     int64_t heads_total, int64_t S, int64_t Dh, int64_t out_area_bytes,
                                     int64_t flag_off, char* inbox_local[2], cudaStream_t stream) {
  const int T = c->world;
  const int R = hosted(c);
  const int r0 = c->local_group ? 0 : c->rank;
  const int64_t hl = heads_total / T, sl = S / T;
  const int64_t tensor_bytes = batch * hl * S * Dh * 2;
  const int64_t inbox_off = (out_area_bytes + 4095) & ~int64_t{4095};
  if (inbox_off + 3 * tensor_bytes > data_bytes_per_parity(c->sym_bytes))
    return tpf::Status::capacity("symmetric heap too small for the Ulysses all-to-all (need " +
                                 std::to_string(2 * (inbox_off + 3 * tensor_bytes) + 2 * kFlagBytesPerParity) +
                                 " bytes per rank)");
  tpf::UlyssesParams up;
  std::memset(&up, 0, sizeof(up));
  up.src[0] = static_cast<const char*>(q);
  up.src[1] = static_cast<const char*>(k);
  up.src[2] = static_cast<const char*>(v);
  up.src_rank_stride = batch * heads_total * sl * Dh * 2;
  up.tensor_bytes = tensor_bytes;
  up.B = batch; up.H = heads_total; up.hl = hl; up.S = S; up.sl = sl; up.Dh = Dh;
  up.T = T; up.R = R; up.rank0 = r0;
  up.ctas_per_rank = std::max(1, std::min(tpf::num_sms() / R, 132));
  if ((flag_off + static_cast<int64_t>(T) * up.ctas_per_rank) * 4 > kFlagCapBytes)
    return tpf::Status::capacity("flag block too small for the Ulysses all-to-all");
  for (int par = 0; par < 2; ++par)
    for (int x = 0; x < T; ++x) {
      up.dst[par][x] = c->sym[x] + 2 * kFlagBytesPerParity + par * data_bytes_per_parity(c->sym_bytes) + inbox_off;
      up.flags[par][x] = reinterpret_cast<uint32_t*>(c->sym[x] + par * kFlagBytesPerParity) + flag_off;
    }
  up.epoch_dev = c->dev_epoch;
  up.fault_rank = c->fault_rank;
  tpf::launch_ulysses_push(up, stream);
  TPF_CUDA_TRY_STATUS(cudaGetLastError());
  for (int hh = 0; hh < R && !c->is_virtual; ++hh) {  // virtual group: no other sources (the own part is
    const int rank = r0 + hh;                          // stream-ordered after the push)
    tpf::launch_wait_flags2(up.flags[0][rank], up.flags[1][rank], static_cast<int64_t>(T) * up.ctas_per_rank,
                            c->dev_epoch, 0, c->timeout_ns, c->err, rank, blame_of(c), 0, up.ctas_per_rank, stream);
  }
  inbox_local[0] = up.dst[0][r0];
  inbox_local[1] = up.dst[1][r0];
  return tpf::Status::ok();
}

static tpf::Status check_ulysses(tpf_comm* c, int64_t batch, int64_t heads_total, int64_t S, int64_t Dh) {
  const int T = c->world;
  if (batch < 1 || heads_total < 1 || S < 1 || Dh < 1)
    return tpf::Status::invalid("Ulysses inputs need batch >= 1, heads >= 1, seq >= 1, head_dim >= 1");
  if (S % T)
    return tpf::Status::invalid("Ulysses: sequence length " + std::to_string(S) +
                                " is not divisible by group size " + std::to_string(T));
  if (heads_total % T)
    return tpf::Status::invalid("Ulysses: head count " + std::to_string(heads_total) +
                                " is not divisible by group size " + std::to_string(T));
  if (Dh % 8) return tpf::Status::shape("Ulysses: head_dim must be a multiple of 8");
  return tpf::Status::ok();
}

int tpf_ulysses_a2a(tpf_comm* c, const void* q, const void* k, const void* v, void* q_out, void* k_out, void* v_out,
                    int64_t batch, int64_t heads_total, int64_t S, int64_t Dh, void* stream_v) {
  tpf::Status s = check_ready(c);
  if (s.good()) s = check_not_split(c, "tpf_ulysses_a2a");
  if (s.good()) s = check_ulysses(c, batch, heads_total, S, Dh);
  if (!s.good()) return fail(s);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  char* inbox[2] = {nullptr, nullptr};
  s = ulysses_first_a2a(c, q, k, v, batch, heads_total, S, Dh, 0, 0, inbox, stream);
  if (!s.good()) return fail(s);
  const int64_t tb = batch * (heads_total / c->world) * S * Dh * 2;
  void* outs[3] = {q_out, k_out, v_out};
  for (int hh = 0; hh < hosted(c); ++hh)
    for (int t = 0; t < 3; ++t)
      tpf::launch_copy_by_parity(static_cast<char*>(outs[t]) + hh * tb, inbox[0] + hh * c->sym_bytes + t * tb,
                                 inbox[1] + hh * c->sym_bytes + t * tb, tb, c->dev_epoch, stream);
  TPF_CUDA_TRY(cudaGetLastError());
  return TPF_OK;
}

int tpf_ulysses_attention(tpf_comm* c, const void* q, const void* k, const void* v, void* out, int64_t batch,
                          int64_t heads_total, int64_t S, int64_t Dh, int scale, void* stream_v) {
  tpf::Status s = check_ready(c);
  if (s.good()) s = check_not_split(c, "tpf_ulysses_attention");
  if (s.good()) s = check_ulysses(c, batch, heads_total, S, Dh);
  if (!s.good()) return fail(s);
  const int T = c->world;
  const int64_t hl = heads_total / T, sl = S / T;
  if (Dh != 128 || sl % 128)
    return fail(tpf::Status::shape("tpf_ulysses_attention: the fused path needs head_dim 128 and S/T % 128 == 0"));
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const int64_t out_area = batch * sl * heads_total * Dh * 2;
  const int64_t attn_flags = batch * hl * (sl / 128) * 4 * T;
  char* inbox[2] = {nullptr, nullptr};
  s = ulysses_first_a2a(c, q, k, v, batch, heads_total, S, Dh, out_area, (attn_flags + 31) & ~int64_t{31}, inbox,
                        stream);
  if (!s.good()) return fail(s);
  const int64_t tb = batch * hl * S * Dh * 2;
  const void* qkv0[3] = {inbox[0], inbox[0] + tb, inbox[0] + 2 * tb};
  const void* qkv1[3] = {inbox[1], inbox[1] + tb, inbox[1] + 2 * tb};
  // the push kernel opened the call; the attention reads that epoch
  s = fmha_a2a_v2(c, qkv0, qkv1, static_cast<uint64_t>(c->sym_bytes), out, batch, hl, S, /*bump=*/0, scale, stream);
  return s.good() ? TPF_OK : fail(s);
}
