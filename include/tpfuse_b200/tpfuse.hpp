// tpfuse_b200 — C++ host mirror of the reference's operator API for the fused
// AG-GEMM / GEMM-RS path, over the C ABI in include/tpf.h (libtpfuse_b200.so).
//
// Same names, argument meaning and error behaviour as
// /root/reference/proj/include/tpfuse/{tensor,collectives,layers,fabric}.hpp:
//   ScheduleKind / ScheduleStep / Schedule / RingIndices      collectives.hpp:19-49
//   ring_indices_ag / ring_indices_rs / build_schedule /
//   check_schedule                                           collectives.hpp:51-64
//   Tensor / Matrix / ShapeError (host, double)              tensor.hpp:13-85
//   ShardedLinear::split_rows / split_columns                layers.hpp:15-38
//   column_parallel_forward / row_parallel_forward /
//   tpsp_mlp_forward                                         layers.hpp:68-84
//   GroupError                                               fabric.hpp:23-32
//
// Two ways to run a group:
//   * RankEndpoint — one rank per process (per GPU): the production path; operates on
//     device tensors (bf16 operands) and streams, no host copies.
//   * LocalGroup   — all T ranks of a group on the current GPU, one persistent launch
//     per op (the analogue of the reference's in-process spawn_group); takes host
//     Tensors like the reference's tests do. Operands are staged as bf16 (exact for
//     the reference's integer test data), results come back from fp32.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "tpf.h"

namespace tpfuse_b200 {

// ------------------------------------------------------------------ errors
class ShapeError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

class GroupError : public std::runtime_error {
 public:
  GroupError(int rank, const std::string& what) : std::runtime_error(what), rank_(rank) {}
  int failing_rank() const { return rank_; }

 private:
  int rank_ = -1;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {

[[noreturn]] inline void raise(int code) {
  const std::string msg = tpf_last_error();
  switch (code) {
    case TPF_E_INVALID: throw std::invalid_argument(msg);
    case TPF_E_SHAPE: throw ShapeError(msg);
    case TPF_E_LOGIC: throw std::logic_error(msg);
    case TPF_E_PEER: {
      int rank = -1;
      if (msg.rfind("rank ", 0) == 0) rank = std::atoi(msg.c_str() + 5);
      throw GroupError(rank, msg);
    }
    default: throw DeviceError(msg);
  }
}

inline void check(int rc) {
  if (rc != TPF_OK) raise(rc);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

inline uint16_t to_bf16(double v) {  // round-to-nearest-even
  float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

}  // namespace detail

// --------------------------------------------------------------- schedules
enum class ScheduleKind { Ring = TPF_RING, PairwiseBidirectional = TPF_PAIRWISE, CircularSlices = TPF_CIRCULAR };

inline std::string to_string(ScheduleKind k) {
  switch (k) {
    case ScheduleKind::Ring: return "ring";
    case ScheduleKind::PairwiseBidirectional: return "pairwise";
    case ScheduleKind::CircularSlices: return "circular-slices";
  }
  return "unknown";
}

struct ScheduleStep {
  int send_peer = -1;
  int recv_peer = -1;
  int compute_slice = 0;
  bool has_comm() const { return send_peer >= 0; }
};

struct Schedule {
  ScheduleKind kind = ScheduleKind::Ring;
  int group_size = 1;
  std::vector<std::vector<ScheduleStep>> steps;  // [rank][iteration]
  int iterations() const { return steps.empty() ? 0 : static_cast<int>(steps[0].size()); }
};

struct RingIndices {
  int send_peer;
  int recv_peer;
  int compute_slice;
};

inline RingIndices ring_indices_ag(int r, int i, int n) {
  int32_t o[3];
  detail::check(tpf_ring_indices(0, r, i, n, o));
  return {o[0], o[1], o[2]};
}

inline RingIndices ring_indices_rs(int r, int i, int n) {
  int32_t o[3];
  detail::check(tpf_ring_indices(1, r, i, n, o));
  return {o[0], o[1], o[2]};
}

inline std::vector<int32_t> flatten(const Schedule& s) {
  std::vector<int32_t> t;
  for (const auto& row : s.steps)
    for (const auto& st : row) {
      t.push_back(st.send_peer);
      t.push_back(st.recv_peer);
      t.push_back(st.compute_slice);
    }
  return t;
}

inline void check_schedule(const Schedule& s) {
  std::vector<int32_t> t = flatten(s);
  const int n = s.group_size;
  if (static_cast<int>(s.steps.size()) != n)
    throw std::logic_error("check_schedule: step table must cover every rank");
  for (const auto& row : s.steps)
    if (n > 1 && static_cast<int>(row.size()) != n)
      throw std::logic_error("check_schedule: every rank must have n iterations");
  if (t.empty()) t.push_back(0);
  detail::check(tpf_schedule_check(static_cast<int>(s.kind), n, t.data()));
}

inline Schedule build_schedule(ScheduleKind kind, int n) {
  std::vector<int32_t> t(static_cast<size_t>(n > 0 ? n * n * 3 : 1));
  detail::check(tpf_schedule_build(static_cast<int>(kind), n, t.data()));
  Schedule s;
  s.kind = kind;
  s.group_size = n;
  s.steps.assign(static_cast<size_t>(n), {});
  if (n == 1) return s;
  for (int r = 0; r < n; ++r)
    for (int i = 0; i < n; ++i) {
      const int32_t* e = &t[(static_cast<size_t>(r) * n + i) * 3];
      s.steps[r].push_back({e[0], e[1], e[2]});
    }
  return s;
}

// ----------------------------------------------------------- host tensors
class Tensor {
 public:
  Tensor() = default;
  Tensor(int64_t b, int64_t s, int64_t d) : b_(b), s_(s), d_(d) {
    if (b < 1 || s < 1 || d < 1)
      throw ShapeError("tensor dimensions must be positive, got (" + std::to_string(b) + "," +
                       std::to_string(s) + "," + std::to_string(d) + ")");
    data_.assign(static_cast<size_t>(b * s * d), 0.0);
  }
  int64_t batch() const { return b_; }
  int64_t seq() const { return s_; }
  int64_t feat() const { return d_; }
  double& operator()(int64_t b, int64_t s, int64_t d) { return data_[(b * s_ + s) * d_ + d]; }
  double operator()(int64_t b, int64_t s, int64_t d) const { return data_[(b * s_ + s) * d_ + d]; }
  std::vector<double>& raw() { return data_; }
  const std::vector<double>& raw() const { return data_; }
  std::string shape_str() const {
    return "(" + std::to_string(b_) + "," + std::to_string(s_) + "," + std::to_string(d_) + ")";
  }
  bool same_shape(const Tensor& o) const { return b_ == o.b_ && s_ == o.s_ && d_ == o.d_; }
  friend bool operator==(const Tensor& a, const Tensor& b) { return a.same_shape(b) && a.data_ == b.data_; }

 private:
  int64_t b_ = 0, s_ = 0, d_ = 0;
  std::vector<double> data_;
};

class Matrix {
 public:
  Matrix() = default;
  Matrix(int64_t r, int64_t c) : r_(r), c_(c) {
    if (r < 1 || c < 1) throw ShapeError("matrix dimensions must be positive");
    data_.assign(static_cast<size_t>(r * c), 0.0);
  }
  int64_t rows() const { return r_; }
  int64_t cols() const { return c_; }
  double& operator()(int64_t r, int64_t c) { return data_[r * c_ + c]; }
  double operator()(int64_t r, int64_t c) const { return data_[r * c_ + c]; }
  std::vector<double>& raw() { return data_; }
  const std::vector<double>& raw() const { return data_; }

 private:
  int64_t r_ = 0, c_ = 0;
  std::vector<double> data_;
};

class ShardedLinear {
 public:
  enum class Kind { RowShard, ColumnShard };

  static ShardedLinear split_rows(Matrix full, int world) {
    if (world < 1 || full.rows() % world)
      throw ShapeError("split_rows: " + std::to_string(full.rows()) + " rows cannot be split across " +
                       std::to_string(world) + " ranks");
    const int64_t rows = full.rows() / world;
    std::vector<Matrix> sh;
    for (int r = 0; r < world; ++r) {
      Matrix m(rows, full.cols());
      for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < full.cols(); ++j) m(i, j) = full(r * rows + i, j);
      sh.push_back(std::move(m));
    }
    return ShardedLinear(Kind::RowShard, std::move(full), std::move(sh));
  }

  static ShardedLinear split_columns(Matrix full, int world) {
    if (world < 1 || full.cols() % world)
      throw ShapeError("split_columns: " + std::to_string(full.cols()) + " columns cannot be split across " +
                       std::to_string(world) + " ranks");
    const int64_t cols = full.cols() / world;
    std::vector<Matrix> sh;
    for (int r = 0; r < world; ++r) {
      Matrix m(full.rows(), cols);
      for (int64_t i = 0; i < full.rows(); ++i)
        for (int64_t j = 0; j < cols; ++j) m(i, j) = full(i, r * cols + j);
      sh.push_back(std::move(m));
    }
    return ShardedLinear(Kind::ColumnShard, std::move(full), std::move(sh));
  }

  Kind kind() const { return kind_; }
  int world() const { return static_cast<int>(shards_.size()); }
  const Matrix& full() const { return full_; }
  const Matrix& shard(int r) const { return shards_.at(static_cast<size_t>(r)); }
  Matrix& shard(int r) { return shards_.at(static_cast<size_t>(r)); }

 private:
  ShardedLinear(Kind k, Matrix f, std::vector<Matrix> s) : kind_(k), full_(std::move(f)), shards_(std::move(s)) {}
  Kind kind_;
  Matrix full_;
  std::vector<Matrix> shards_;
};

enum class Activation { None = TPF_ACT_NONE, Square = TPF_ACT_SQUARE };

// ------------------------------------------------------- device tensor view
struct DeviceTensor {
  void* data = nullptr;
  int64_t batch = 0, seq = 0, feat = 0;
  int dtype = TPF_BF16;
};

// ---------------------------------------------------- one rank per process
class RankEndpoint {
 public:
  RankEndpoint(int rank, int world, size_t sym_bytes) {
    detail::check(tpf_comm_create(rank, world, sym_bytes, &c_));
    // The library links its own CUDA runtime: it must see the device this process made current.
    int dev = -1;
    if (cudaGetDevice(&dev) == cudaSuccess && dev != tpf_comm_device(c_)) {
      const int lib_dev = tpf_comm_device(c_);
      tpf_comm_destroy(c_);
      c_ = nullptr;
      throw std::runtime_error("tpfuse: communicator created on device " + std::to_string(lib_dev) +
                               " but the current device is " + std::to_string(dev));
    }
  }
  ~RankEndpoint() {
    if (c_) tpf_comm_destroy(c_);
  }
  RankEndpoint(const RankEndpoint&) = delete;
  RankEndpoint& operator=(const RankEndpoint&) = delete;

  int rank() const { return tpf_comm_rank(c_); }
  int group_size() const { return tpf_comm_world(c_); }

  // Bootstrap: export this rank's IPC handle, exchange out of band (MPI / sockets /
  // torch.distributed), then open every peer's.
  std::vector<uint8_t> ipc_handle() const {
    std::vector<uint8_t> h(TPF_IPC_HANDLE_BYTES);
    if (group_size() > 1) detail::check(tpf_comm_ipc_handle(c_, h.data()));
    return h;
  }
  void open_peers(const std::vector<uint8_t>& all_handles) {
    if (group_size() > 1) detail::check(tpf_comm_open_peers(c_, all_handles.data()));
  }
  void sync(cudaStream_t s = nullptr) { detail::check(tpf_comm_sync(c_, s)); }
  tpf_comm* handle() { return c_; }

 private:
  friend class SplitGroup;
  explicit RankEndpoint(tpf_comm* adopted) : c_(adopted) {}
  tpf_comm* c_ = nullptr;
};

// ------------------------------------------- one GPU, the per-rank path (split group)
// T endpoints built exactly like T processes' RankEndpoints (own symmetric heap, device epoch,
// error record), peers mapped directly instead of through CUDA IPC (tpf_comm_create_split_group).
// Device-level calls on every endpoint (any order, any threads, one stream) run as one launch
// once the last rank has made its call; ep.sync() waits for that launch.
class SplitGroup {
 public:
  explicit SplitGroup(int world, size_t sym_bytes) {
    std::vector<tpf_comm*> cs(static_cast<size_t>(world), nullptr);
    detail::check(tpf_comm_create_split_group(world, sym_bytes, cs.data()));
    for (tpf_comm* c : cs) eps_.emplace_back(new RankEndpoint(c));
  }
  SplitGroup(const SplitGroup&) = delete;
  SplitGroup& operator=(const SplitGroup&) = delete;
  int size() const { return static_cast<int>(eps_.size()); }
  RankEndpoint& endpoint(int r) { return *eps_.at(static_cast<size_t>(r)); }

 private:
  std::vector<std::unique_ptr<RankEndpoint>> eps_;
};

// spawn_group (fabric.hpp:185-226) over a split group: body(endpoint(r)) on one worker thread
// per rank; results in rank order; the first failing rank is rethrown as GroupError naming it.
template <typename Body>
auto spawn_group(SplitGroup& group, Body&& body) {
  using Result = std::invoke_result_t<Body&, RankEndpoint&>;
  const int t = group.size();
  std::vector<std::exception_ptr> errors(static_cast<size_t>(t));
  std::vector<std::optional<std::conditional_t<std::is_void_v<Result>, int, Result>>> results(static_cast<size_t>(t));
  std::vector<std::thread> workers;
  for (int r = 0; r < t; ++r)
    workers.emplace_back([&, r] {
      try {
        if constexpr (std::is_void_v<Result>) {
          body(group.endpoint(r));
          results[static_cast<size_t>(r)] = 0;
        } else {
          results[static_cast<size_t>(r)] = body(group.endpoint(r));
        }
      } catch (...) {
        errors[static_cast<size_t>(r)] = std::current_exception();
      }
    });
  for (std::thread& w : workers) w.join();
  // A rank's GroupError already names the rank that failed (blame chain); any other failure
  // names the rank that raised it.
  for (int r = 0; r < t; ++r) {
    if (!errors[static_cast<size_t>(r)]) continue;
    try {
      std::rethrow_exception(errors[static_cast<size_t>(r)]);
    } catch (const GroupError&) {
      throw;
    } catch (const std::exception& e) {
      throw GroupError(r, "rank " + std::to_string(r) + " failed: " + e.what());
    }
  }
  if constexpr (std::is_void_v<Result>) {
    return;
  } else {
    std::vector<Result> out;
    for (auto& v : results) out.push_back(std::move(*v));
    return out;
  }
}

// Device-level drop-ins (layers.hpp:68-76). x/w bf16; out bf16 or fp32.
inline void column_parallel_forward(RankEndpoint& ep, const DeviceTensor& x, const DeviceTensor& w_shard,
                                    DeviceTensor& out, int m = 1, Activation act = Activation::None,
                                    cudaStream_t stream = nullptr) {
  detail::check(tpf_ag_gemm(ep.handle(), x.data, w_shard.data, out.data, x.batch,
                            x.seq * ep.group_size(), x.feat, w_shard.feat, m, static_cast<int>(act),
                            out.dtype, stream));
}

inline void row_parallel_forward(RankEndpoint& ep, const DeviceTensor& x, const DeviceTensor& w_shard,
                                 const Schedule& schedule, DeviceTensor& out, int m = 1, int wire = TPF_F32,
                                 cudaStream_t stream = nullptr) {
  if (schedule.group_size != ep.group_size())
    throw std::invalid_argument("fuse_reduce_scatter: schedule built for " +
                                std::to_string(schedule.group_size) + " ranks, group has " +
                                std::to_string(ep.group_size()));
  detail::check(tpf_gemm_rs(ep.handle(), x.data, w_shard.data, out.data, x.batch, x.seq, x.feat, w_shard.feat,
                            static_cast<int>(schedule.kind), m, wire, out.dtype, stream));
}

// UP: fuse_all_to_all_attention (layers.hpp:100-101). q/k/v bf16 (batch*heads, S, Dh) for this
// rank's head group; out bf16 (batch, S/T, T*heads*Dh). Dh == 128 runs the fused tcgen05
// flash-attention kernel; other head dims run the GEMM-family pipeline.
inline void fuse_all_to_all_attention(RankEndpoint& ep, const void* q, const void* k, const void* v, void* out,
                                      int64_t batch, int64_t heads, int64_t S, int64_t Dh, bool scale_scores = true,
                                      cudaStream_t stream = nullptr) {
  detail::check(tpf_attention_a2a(ep.handle(), q, k, v, out, batch, heads, S, Dh, scale_scores ? 1 : 0, stream));
}

// Ulysses first all-to-all (ref_all_to_all of fabric.cpp:183-207 as layers_test.cpp:347-397
// drives it): q/k/v (batch*heads_total, S/T, Dh) sequence-sharded -> (batch*heads_total/T, S, Dh).
inline void ulysses_all_to_all(RankEndpoint& ep, const void* q, const void* k, const void* v, void* q_out,
                               void* k_out, void* v_out, int64_t batch, int64_t heads_total, int64_t S, int64_t Dh,
                               cudaStream_t stream = nullptr) {
  detail::check(tpf_ulysses_a2a(ep.handle(), q, k, v, q_out, k_out, v_out, batch, heads_total, S, Dh, stream));
}

// The whole UP attention from the sequence-sharded layout: first all-to-all + fused attention
// with the output all-to-all. out (batch, S/T, heads_total*128) bf16.
inline void ulysses_attention(RankEndpoint& ep, const void* q, const void* k, const void* v, void* out,
                              int64_t batch, int64_t heads_total, int64_t S, bool scale_scores = true,
                              cudaStream_t stream = nullptr) {
  detail::check(tpf_ulysses_attention(ep.handle(), q, k, v, out, batch, heads_total, S, 128, scale_scores ? 1 : 0,
                                      stream));
}

// query_split_attention (layers.hpp:88-91): w_o is this rank's (heads*128, D) row shard.
inline void query_split_attention(RankEndpoint& ep, const void* q, const void* k, const void* v, const void* w_o,
                                  DeviceTensor& out, int64_t batch, int64_t heads, int64_t S,
                                  const Schedule& schedule, int wire = TPF_F32, bool scale_scores = true,
                                  cudaStream_t stream = nullptr) {
  detail::check(tpf_query_split_attention(ep.handle(), q, k, v, w_o, out.data, batch, heads, S, 128, out.feat,
                                          static_cast<int>(schedule.kind), wire, out.dtype, scale_scores ? 1 : 0,
                                          stream));
}

// DP gradient sync (cfg 4): dW rows [r*K/T, (r+1)*K/T) of sum_q X_q^T dY_q.
inline void dp_grad_reduce_scatter(RankEndpoint& ep, const void* X, const void* dY, DeviceTensor& dW,
                                   int64_t M_local, int64_t K, const Schedule& schedule, int m = 1,
                                   int wire = TPF_F32, cudaStream_t stream = nullptr) {
  detail::check(tpf_dp_grad_rs(ep.handle(), X, dY, dW.data, M_local, K, dW.feat, static_cast<int>(schedule.kind), m,
                               wire, dW.dtype, stream));
}

// DP parameter all-gather fused into the forward GEMM (cfg 4): out = x . W^T, W row-sharded.
inline void dp_param_all_gather_gemm(RankEndpoint& ep, const void* x, const void* w_rows, DeviceTensor& out,
                                     int64_t M_local, int64_t K, int64_t N_local, cudaStream_t stream = nullptr) {
  detail::check(tpf_dp_param_ag_gemm(ep.handle(), x, w_rows, out.data, M_local, K, N_local, out.dtype, stream));
}

// ------------------------------------------ single-GPU group (spawn_group analogue)
// Per-rank attention operands, folded (batch*heads, seq, head_dim): layers.hpp:40-56.
struct AttentionInputs {
  int batch = 0;
  int heads = 0;  // heads held by this rank
  Tensor q, k, v;
  int64_t head_dim() const { return q.feat(); }
  int64_t seq() const { return q.seq(); }
};

inline AttentionInputs make_attention_inputs(int batch, int heads, Tensor q, Tensor k, Tensor v) {
  if (batch < 1 || heads < 1) throw std::invalid_argument("attention inputs need batch >= 1 and heads >= 1");
  if (q.batch() != static_cast<int64_t>(batch) * heads)
    throw ShapeError("attention inputs: q " + q.shape_str() + " is not folded as (batch*heads, seq, head_dim)");
  if (!k.same_shape(v) || k.batch() != q.batch() || k.feat() != q.feat())
    throw ShapeError("attention inputs: k " + k.shape_str() + " / v " + v.shape_str() + " do not match q " +
                     q.shape_str());
  return AttentionInputs{batch, heads, std::move(q), std::move(k), std::move(v)};
}

struct AttentionOptions {
  bool scale_scores = true;  // scale scores by 1/sqrt(head_dim) before the softmax
};

class LocalGroup {
 public:
  explicit LocalGroup(int world, size_t sym_bytes_per_rank = size_t(64) << 20) : world_(world) {
    detail::check(tpf_comm_create_local_group(world, sym_bytes_per_rank, &c_));
  }
  ~LocalGroup() {
    for (void* p : bufs_) cudaFree(p);
    if (c_) tpf_comm_destroy(c_);
  }
  LocalGroup(const LocalGroup&) = delete;
  LocalGroup& operator=(const LocalGroup&) = delete;
  int size() const { return world_; }
  tpf_comm* handle() { return c_; }

  // column_parallel_forward on every rank: xs[r] is rank r's (B, S/T, K) slice.
  std::vector<Tensor> column_parallel_forward(const std::vector<Tensor>& xs, const ShardedLinear& w, int m = 1,
                                              Activation act = Activation::None) {
    require_kind(w, ShardedLinear::Kind::ColumnShard, "column_parallel_forward");
    check_ranks(xs, "column_parallel_forward");
    const Tensor& x0 = xs[0];
    const int64_t K = x0.feat(), N = w.shard(0).cols(), Kp = up8(K), Np = up8(N);
    if (w.shard(0).rows() != K)
      throw ShapeError("matmul: feature width of x " + x0.shape_str() + " does not match rows of w");
    void* dx = stage_x(xs, Kp, 0, K);
    void* dw = stage_w(w, Kp, Np, 0, K);
    const int64_t S = x0.seq() * world_;
    const int64_t out_elems = x0.batch() * S * Np;
    float* dout = static_cast<float*>(alloc(sizeof(float) * out_elems * world_));
    detail::check(tpf_ag_gemm(c_, dx, dw, dout, x0.batch(), S, Kp, Np, m, static_cast<int>(act), TPF_F32, nullptr));
    detail::check(tpf_comm_sync(c_, nullptr));
    return fetch(dout, x0.batch(), S, Np, N);
  }

  // row_parallel_forward on every rank: xs[r] is rank r's (B, S, K/T) feature shard.
  std::vector<Tensor> row_parallel_forward(const std::vector<Tensor>& xs, const ShardedLinear& w,
                                           const Schedule& schedule, int m = 1, int wire = TPF_F32) {
    require_kind(w, ShardedLinear::Kind::RowShard, "row_parallel_forward");
    check_ranks(xs, "row_parallel_forward");
    if (schedule.group_size != world_)
      throw std::invalid_argument("fuse_reduce_scatter: schedule built for " +
                                  std::to_string(schedule.group_size) + " ranks, group has " +
                                  std::to_string(world_));
    const Tensor& x0 = xs[0];
    const int64_t K = x0.feat(), N = w.shard(0).cols(), Kp = up8(K), Np = up8(N);
    if (w.shard(0).rows() != K)
      throw ShapeError("matmul: feature width of x " + x0.shape_str() + " does not match rows of w");
    void* dx = stage_x(xs, Kp, 0, K);
    void* dw = stage_w(w, Kp, Np, 0, K);
    const int64_t S = x0.seq();
    if (world_ > 1 && S % world_)
      throw std::invalid_argument("fuse_reduce_scatter: sequence length " + std::to_string(S) +
                                  " is not divisible by " + std::to_string(world_));
    const int64_t So = S / world_;
    float* dout = static_cast<float*>(alloc(sizeof(float) * x0.batch() * So * Np * world_));
    detail::check(tpf_gemm_rs(c_, dx, dw, dout, x0.batch(), S, Kp, Np, static_cast<int>(schedule.kind), m, wire,
                              TPF_F32, nullptr));
    detail::check(tpf_comm_sync(c_, nullptr));
    return fetch(dout, x0.batch(), So, Np, N);
  }

  // tpsp_mlp_forward (layers.cpp:140-147) with the activation fused into the AG-GEMM
  // epilogue; the hidden activation is the bf16 operand of the second GEMM.
  std::vector<Tensor> tpsp_mlp_forward(const std::vector<Tensor>& xs, const ShardedLinear& up,
                                       const ShardedLinear& down, Activation act, const Schedule& schedule,
                                       int m = 1) {
    require_kind(up, ShardedLinear::Kind::ColumnShard, "column_parallel_forward");
    require_kind(down, ShardedLinear::Kind::RowShard, "row_parallel_forward");
    check_ranks(xs, "tpsp_mlp_forward");
    const Tensor& x0 = xs[0];
    const int64_t D = x0.feat(), H = up.shard(0).cols(), Dp = up8(D), Hp = up8(H), No = down.shard(0).cols(),
                  Nop = up8(No);
    const int64_t S = x0.seq() * world_;
    void* dx = stage_x(xs, Dp, 0, D);
    void* dup = stage_w(up, Dp, Hp, 0, D);
    void* ddown = stage_w(down, Hp, Nop, 0, H);
    void* hid = alloc(2 * x0.batch() * S * Hp * world_);
    detail::check(tpf_ag_gemm(c_, dx, dup, hid, x0.batch(), S, Dp, Hp, m, static_cast<int>(act), TPF_BF16, nullptr));
    float* dout = static_cast<float*>(alloc(sizeof(float) * x0.batch() * x0.seq() * Nop * world_));
    detail::check(tpf_gemm_rs(c_, hid, ddown, dout, x0.batch(), S, Hp, Nop, static_cast<int>(schedule.kind), m,
                              TPF_F32, TPF_F32, nullptr));
    detail::check(tpf_comm_sync(c_, nullptr));
    return fetch(dout, x0.batch(), x0.seq(), Nop, No);
  }

  // fuse_all_to_all_attention (layers.cpp:174-218) on every rank: qkv[r] is rank r's head
  // group over the whole sequence; returns (batch, S/T, T*heads*Dh) per rank.
  std::vector<Tensor> fuse_all_to_all_attention(const std::vector<AttentionInputs>& qkv,
                                                const AttentionOptions& options = {}) {
    check_attention(qkv, "fuse_all_to_all_attention");
    const AttentionInputs& a0 = qkv[0];
    const int64_t S = a0.seq(), Dh = a0.head_dim();
    if (S % world_)
      throw std::invalid_argument("fuse_all_to_all_attention: sequence length " + std::to_string(S) +
                                  " is not divisible by group size " + std::to_string(world_));
    void* dq = stage_folded(qkv, 0);
    void* dk = stage_folded(qkv, 1);
    void* dv = stage_folded(qkv, 2);
    const int64_t F = static_cast<int64_t>(world_) * a0.heads * Dh;
    void* dout = alloc(2 * static_cast<size_t>(world_) * a0.batch * (S / world_) * F);
    detail::check(tpf_attention_a2a(c_, dq, dk, dv, dout, a0.batch, a0.heads, S, Dh, options.scale_scores ? 1 : 0,
                                    nullptr));
    detail::check(tpf_comm_sync(c_, nullptr));
    return fetch_bf16(dout, a0.batch, S / world_, F);
  }

  // query_split_attention (layers.cpp:149-172): out_proj is row-sharded ((T*heads*Dh) x D).
  std::vector<Tensor> query_split_attention(const std::vector<AttentionInputs>& qkv, const ShardedLinear& out_proj,
                                            const Schedule& schedule, const AttentionOptions& options = {}) {
    check_attention(qkv, "query_split_attention");
    require_kind(out_proj, ShardedLinear::Kind::RowShard, "query_split_attention");
    const AttentionInputs& a0 = qkv[0];
    const int64_t S = a0.seq(), Dh = a0.head_dim(), D = out_proj.shard(0).cols(), Dp = up8(D);
    if (out_proj.shard(0).rows() != a0.heads * Dh)
      throw ShapeError("query_split_attention: out_proj shard rows do not match heads * head_dim");
    void* dq = stage_folded(qkv, 0);
    void* dk = stage_folded(qkv, 1);
    void* dv = stage_folded(qkv, 2);
    void* dw = stage_w(out_proj, a0.heads * Dh, Dp, 0, a0.heads * Dh);
    float* dout = static_cast<float*>(alloc(sizeof(float) * world_ * a0.batch * (S / world_) * Dp));
    detail::check(tpf_query_split_attention(c_, dq, dk, dv, dw, dout, a0.batch, a0.heads, S, Dh, Dp,
                                            static_cast<int>(schedule.kind), TPF_F32, TPF_F32,
                                            options.scale_scores ? 1 : 0, nullptr));
    detail::check(tpf_comm_sync(c_, nullptr));
    return fetch(dout, a0.batch, S / world_, Dp, D);
  }

 private:
  void check_attention(const std::vector<AttentionInputs>& qkv, const char* op) const {
    if (static_cast<int>(qkv.size()) != world_)
      throw std::invalid_argument(std::string(op) + ": expected one input per rank");
    for (const AttentionInputs& a : qkv)
      if (a.batch != qkv[0].batch || a.heads != qkv[0].heads || !a.q.same_shape(qkv[0].q) ||
          !a.k.same_shape(qkv[0].k))
        throw ShapeError(std::string(op) + ": ranks disagree on attention shapes");
  }

  // rank-stacked bf16 (T, batch*heads, S, Dh) of q (which = 0), k (1) or v (2)
  void* stage_folded(const std::vector<AttentionInputs>& qkv, int which) {
    const Tensor& t0 = which == 0 ? qkv[0].q : which == 1 ? qkv[0].k : qkv[0].v;
    const size_t n = t0.raw().size();
    std::vector<uint16_t> h(static_cast<size_t>(world_) * n);
    for (int r = 0; r < world_; ++r) {
      const Tensor& t = which == 0 ? qkv[r].q : which == 1 ? qkv[r].k : qkv[r].v;
      for (size_t i = 0; i < n; ++i) h[r * n + i] = detail::to_bf16(t.raw()[i]);
    }
    void* d = alloc(h.size() * 2);
    detail::cuda_check(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
    return d;
  }

  std::vector<Tensor> fetch_bf16(const void* d, int64_t B, int64_t S, int64_t N) {
    std::vector<uint16_t> h(static_cast<size_t>(world_ * B * S * N));
    detail::cuda_check(cudaMemcpy(h.data(), d, h.size() * 2, cudaMemcpyDeviceToHost), "cudaMemcpy");
    std::vector<Tensor> out;
    for (int r = 0; r < world_; ++r) {
      Tensor t(B, S, N);
      for (int64_t i = 0; i < B * S * N; ++i) {
        const uint32_t u = static_cast<uint32_t>(h[r * B * S * N + i]) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        t.raw()[i] = f;
      }
      out.push_back(std::move(t));
    }
    for (void* p : bufs_) cudaFree(p);
    bufs_.clear();
    return out;
  }

  static int64_t up8(int64_t v) { return (v + 7) / 8 * 8; }

  void require_kind(const ShardedLinear& w, ShardedLinear::Kind k, const char* op) const {
    if (w.kind() != k)
      throw std::invalid_argument(std::string(op) + ": wrong shard kind (need " +
                                  (k == ShardedLinear::Kind::RowShard ? "row" : "column") + " shards)");
    if (w.world() != world_)
      throw std::invalid_argument(std::string(op) + ": weight sharded for " + std::to_string(w.world()) +
                                  " ranks, group has " + std::to_string(world_));
  }

  void check_ranks(const std::vector<Tensor>& xs, const char* op) const {
    if (static_cast<int>(xs.size()) != world_)
      throw std::invalid_argument(std::string(op) + ": expected one input per rank");
    for (const Tensor& x : xs)
      if (!x.same_shape(xs[0])) throw ShapeError(std::string(op) + ": ranks disagree on input shape");
  }

  void* alloc(size_t bytes) {
    void* p = nullptr;
    detail::cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    bufs_.push_back(p);
    return p;
  }

  // rank-stacked bf16 (T, B, S, Kp) with zero padding of the feature axis
  void* stage_x(const std::vector<Tensor>& xs, int64_t Kp, int64_t k0, int64_t K) {
    const Tensor& x0 = xs[0];
    const int64_t rows = x0.batch() * x0.seq();
    std::vector<uint16_t> h(static_cast<size_t>(world_ * rows * Kp), 0);
    for (int r = 0; r < world_; ++r)
      for (int64_t i = 0; i < rows; ++i)
        for (int64_t k = 0; k < K; ++k)
          h[(r * rows + i) * Kp + k] = detail::to_bf16(xs[r].raw()[i * x0.feat() + k0 + k]);
    void* d = alloc(h.size() * 2);
    detail::cuda_check(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
    return d;
  }

  // rank-stacked bf16 shards (T, Kp, Np), zero padded
  void* stage_w(const ShardedLinear& w, int64_t Kp, int64_t Np, int64_t k0, int64_t K) {
    const int64_t N = w.shard(0).cols();
    std::vector<uint16_t> h(static_cast<size_t>(world_ * Kp * Np), 0);
    for (int r = 0; r < world_; ++r)
      for (int64_t k = 0; k < K; ++k)
        for (int64_t n = 0; n < N; ++n) h[(r * Kp + k) * Np + n] = detail::to_bf16(w.shard(r)(k0 + k, n));
    void* d = alloc(h.size() * 2);
    detail::cuda_check(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
    return d;
  }

  std::vector<Tensor> fetch(const float* d, int64_t B, int64_t S, int64_t Np, int64_t N) {
    std::vector<float> h(static_cast<size_t>(world_ * B * S * Np));
    detail::cuda_check(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
    std::vector<Tensor> out;
    for (int r = 0; r < world_; ++r) {
      Tensor t(B, S, N);
      for (int64_t i = 0; i < B * S; ++i)
        for (int64_t n = 0; n < N; ++n) t.raw()[i * N + n] = h[(r * B * S + i) * Np + n];
      out.push_back(std::move(t));
    }
    for (void* p : bufs_) cudaFree(p);
    bufs_.clear();
    return out;
  }

  int world_;
  tpf_comm* c_ = nullptr;
  std::vector<void*> bufs_;
};

}  // namespace tpfuse_b200
