// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// C-ABI bridge over the UNMODIFIED reference library (`tpfuse`, compiled by
// oracle/Makefile straight from /root/reference/proj/src/*.cpp into
// oracle/_ref/libtpfuse_ref.so). It lets the Python tests and bench.py's
// CPU-baseline leg drive the reference's own code path:
//   * schedule tables      -> tpfuse::build_schedule / ring_indices_*  (collectives.cpp:47-107)
//   * test-data recipes    -> tpfuse::randint_fill / randint_matrix     (tensor.cpp:234-266)
//   * fused layers         -> tpfuse::column_parallel_forward / row_parallel_forward /
//                             tpsp_mlp_forward under tpfuse::spawn_group (layers.cpp:120-147,
//                             fabric.hpp:185-226)
// Every entry returns 0 on success, -1 on a reference exception (message via
// ref_last_error()).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tpfuse/collectives.hpp"
#include "tpfuse/experiment.hpp"
#include "tpfuse/fabric.hpp"
#include "tpfuse/layers.hpp"
#include "tpfuse/tensor.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

tpfuse::ScheduleKind kind_of(int k) {
  switch (k) {
    case 0: return tpfuse::ScheduleKind::Ring;
    case 1: return tpfuse::ScheduleKind::PairwiseBidirectional;
    case 2: return tpfuse::ScheduleKind::CircularSlices;
  }
  throw std::invalid_argument("bad schedule kind");
}

tpfuse::Tensor tensor_from(const double* p, int64_t b, int64_t s, int64_t d) {
  tpfuse::Tensor t(b, s, d);
  std::memcpy(t.raw().data(), p, sizeof(double) * static_cast<size_t>(b * s * d));
  return t;
}

tpfuse::Matrix matrix_from(const double* p, int64_t r, int64_t c) {
  tpfuse::Matrix m(r, c);
  std::memcpy(m.raw().data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

void copy_out(const tpfuse::Tensor& t, double* out) {
  std::memcpy(out, t.raw().data(), sizeof(double) * t.raw().size());
}

// (B,S,D) -> feature columns [begin, begin+len)
tpfuse::Tensor feat_block(const tpfuse::Tensor& x, int64_t begin, int64_t len) {
  tpfuse::Tensor out(x.batch(), x.seq(), len);
  for (int64_t b = 0; b < x.batch(); ++b)
    for (int64_t s = 0; s < x.seq(); ++s)
      for (int64_t d = 0; d < len; ++d) out(b, s, d) = x(b, s, begin + d);
  return out;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// out: n*n*3 int32 (send, recv, slice) — empty (nothing written) for n == 1.
int ref_build_schedule(int kind, int n, int32_t* out) {
  return guarded([&] {
    const tpfuse::Schedule s = tpfuse::build_schedule(kind_of(kind), n);
    for (int r = 0; r < n; ++r)
      for (int i = 0; i < s.iterations(); ++i) {
        const auto& st = s.steps[r][i];
        out[(r * n + i) * 3 + 0] = st.send_peer;
        out[(r * n + i) * 3 + 1] = st.recv_peer;
        out[(r * n + i) * 3 + 2] = st.compute_slice;
      }
  });
}

int ref_ring_indices(int rs, int r, int i, int n, int32_t* out) {
  return guarded([&] {
    const tpfuse::RingIndices idx =
        rs ? tpfuse::ring_indices_rs(r, i, n) : tpfuse::ring_indices_ag(r, i, n);
    out[0] = idx.send_peer;
    out[1] = idx.recv_peer;
    out[2] = idx.compute_slice;
  });
}

int ref_randint_fill(int64_t b, int64_t s, int64_t d, int lo, int hi, uint64_t seed,
                     double* out) {
  return guarded([&] { copy_out(tpfuse::randint_fill(b, s, d, lo, hi, seed), out); });
}

int ref_randint_matrix(int64_t r, int64_t c, int lo, int hi, uint64_t seed, double* out) {
  return guarded([&] {
    const tpfuse::Matrix m = tpfuse::randint_matrix(r, c, lo, hi, seed);
    std::memcpy(out, m.raw().data(), sizeof(double) * m.raw().size());
  });
}

// AG-GEMM through the reference: x_full (B,S,K) is split into T sequence
// slices (rank r gets slice r); w_full (K,N) column-sharded.
// out: T consecutive (B,S,N/T) per-rank outputs.
int ref_column_parallel(int t, int m, int64_t b, int64_t s, int64_t k, int64_t n,
                        const double* x_full, const double* w_full, double* out) {
  return guarded([&] {
    const tpfuse::Tensor x = tensor_from(x_full, b, s, k);
    const tpfuse::ShardedLinear w =
        tpfuse::ShardedLinear::split_columns(matrix_from(w_full, k, n), t);
    const auto slices = tpfuse::split_seq(x, t);
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      return tpfuse::column_parallel_forward(ep, slices[ep.rank()], w, m);
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}

// GEMM-RS through the reference: x_full (B,S,K) is feature-sharded (rank r
// gets columns [r*K/T,(r+1)*K/T)); w_full (K,N) row-sharded.
// out: T consecutive (B,S/T,N) per-rank outputs.
int ref_row_parallel(int t, int kind, int m, int64_t b, int64_t s, int64_t k, int64_t n,
                     const double* x_full, const double* w_full, double* out) {
  return guarded([&] {
    const tpfuse::Tensor x = tensor_from(x_full, b, s, k);
    const tpfuse::ShardedLinear w =
        tpfuse::ShardedLinear::split_rows(matrix_from(w_full, k, n), t);
    const tpfuse::Schedule sched = tpfuse::build_schedule(kind_of(kind), t);
    const int64_t kl = k / t;
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      return tpfuse::row_parallel_forward(ep, feat_block(x, ep.rank() * kl, kl), w, sched, m);
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}

// FuseRS with identity f on explicit per-rank inputs (T x (B,S,D) stacked).
int ref_fuse_rs_identity(int t, int kind, int m, int64_t b, int64_t s, int64_t d,
                         const double* inputs, double* out) {
  return guarded([&] {
    std::vector<tpfuse::Tensor> xs;
    for (int r = 0; r < t; ++r) xs.push_back(tensor_from(inputs + r * b * s * d, b, s, d));
    const tpfuse::Schedule sched = tpfuse::build_schedule(kind_of(kind), t);
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      return tpfuse::fuse_reduce_scatter(
          ep, xs[ep.rank()], [](const tpfuse::Tensor& c) { return c; }, sched, m);
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}

// TP-SP MLP block with the square activation (verify_mlp recipe,
// experiment.cpp:302-330). x_full (B,S,D); up (D,H); down (H,D).
// out: T consecutive (B,S/T,D).
int ref_mlp_square(int t, int kind, int m, int64_t b, int64_t s, int64_t d, int64_t h,
                   const double* x_full, const double* up_full, const double* down_full,
                   double* out) {
  return guarded([&] {
    const tpfuse::Tensor x = tensor_from(x_full, b, s, d);
    const tpfuse::ShardedLinear up =
        tpfuse::ShardedLinear::split_columns(matrix_from(up_full, d, h), t);
    const tpfuse::ShardedLinear down =
        tpfuse::ShardedLinear::split_rows(matrix_from(down_full, h, d), t);
    const tpfuse::Schedule sched = tpfuse::build_schedule(kind_of(kind), t);
    const auto slices = tpfuse::split_seq(x, t);
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      return tpfuse::tpsp_mlp_forward(ep, slices[ep.rank()], up, down,
                                      [](double v) { return v * v; }, sched, m);
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}

// Timing leg for the CPU baseline / reference arm: runs the reference's
// column_parallel_forward (AG-GEMM, K_ag x N_ag) and row_parallel_forward
// (GEMM-RS, K_rs x N_rs, ring) on integer data with T rank threads (the
// reference's own concurrency: one worker per rank, fabric.hpp:196-213).
// Inputs are generated once, outside the timed region; each of `reps`
// repetitions is timed with steady_clock around spawn_group (the reference's
// own bench pattern, experiment.cpp:755-763). ag_secs/rs_secs: reps entries.
int ref_time_ops(int t, int64_t b, int64_t s, int64_t k_ag, int64_t n_ag, int64_t k_rs,
                 int64_t n_rs, int reps, double* ag_secs, double* rs_secs) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const tpfuse::Tensor x_ag = tpfuse::randint_fill(b, s, k_ag, 0, 5, 2);
    const tpfuse::ShardedLinear w_ag = tpfuse::ShardedLinear::split_columns(
        tpfuse::randint_matrix(k_ag, n_ag, -2, 2, 1), t);
    const auto slices = tpfuse::split_seq(x_ag, t);
    const int64_t kl = k_rs / t;
    std::vector<tpfuse::Tensor> xs;
    for (int r = 0; r < t; ++r) xs.push_back(tpfuse::randint_fill(b, s, kl, 0, 5, 10 + r));
    const tpfuse::ShardedLinear w_rs = tpfuse::ShardedLinear::split_rows(
        tpfuse::randint_matrix(k_rs, n_rs, -2, 2, 3), t);
    const tpfuse::Schedule ring = tpfuse::build_schedule(tpfuse::ScheduleKind::Ring, t);
    for (int i = 0; i < reps; ++i) {
      auto t0 = clk::now();
      tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
        return tpfuse::column_parallel_forward(ep, slices[ep.rank()], w_ag, 1);
      });
      auto t1 = clk::now();
      tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
        return tpfuse::row_parallel_forward(ep, xs[ep.rank()], w_rs, ring, 1);
      });
      auto t2 = clk::now();
      ag_secs[i] = std::chrono::duration<double>(t1 - t0).count();
      rs_secs[i] = std::chrono::duration<double>(t2 - t1).count();
    }
  });
}

}  // extern "C"

extern "C" int ref_attention_a2a(int t, int batch, int heads, int64_t s, int64_t dh, int scale,
                                 const double* q, const double* k, const double* v, double* out) {
  return guarded([&] {
    const int64_t bh = static_cast<int64_t>(batch) * heads, per = bh * s * dh;
    std::vector<tpfuse::AttentionInputs> in;
    for (int r = 0; r < t; ++r)
      in.push_back(tpfuse::make_attention_inputs(batch, heads, tensor_from(q + r * per, bh, s, dh),
                                                 tensor_from(k + r * per, bh, s, dh),
                                                 tensor_from(v + r * per, bh, s, dh)));
    tpfuse::AttentionOptions opt;
    opt.scale_scores = scale != 0;
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      return tpfuse::fuse_all_to_all_attention(ep, in[ep.rank()], opt);
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}

extern "C" int ref_query_split_attention(int t, int kind, int batch, int heads, int64_t s, int64_t dh,
                                         int64_t d, int scale, const double* q, const double* k,
                                         const double* v, const double* w_o, double* out) {
  return guarded([&] {
    const int64_t bh = static_cast<int64_t>(batch) * heads, per = bh * s * dh;
    std::vector<tpfuse::AttentionInputs> in;
    for (int r = 0; r < t; ++r)
      in.push_back(tpfuse::make_attention_inputs(batch, heads, tensor_from(q + r * per, bh, s, dh),
                                                 tensor_from(k + r * per, bh, s, dh),
                                                 tensor_from(v + r * per, bh, s, dh)));
    const tpfuse::ShardedLinear wo =
        tpfuse::ShardedLinear::split_rows(matrix_from(w_o, static_cast<int64_t>(t) * heads * dh, d), t);
    const tpfuse::Schedule sched = tpfuse::build_schedule(kind_of(kind), t);
    tpfuse::AttentionOptions opt;
    opt.scale_scores = scale != 0;
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      return tpfuse::query_split_attention(ep, in[ep.rank()], wo, sched, opt);
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}

// Bench CSV wire format (experiment.cpp:838-860): runs the reference's own run_bench on a
// small config and returns its CSV text, so the GPU bench's rows can be checked field by
// field against the reference's formatting.
extern "C" int ref_bench_csv(const char* layer, int tp, int64_t batch, int64_t seq, int64_t d_model, int heads,
                             int granularity, const char* schedule, uint64_t seed, int reps, char* buf,
                             int64_t cap) {
  return guarded([&] {
    tpfuse::ExperimentConfig cfg;
    cfg.layer = tpfuse::layer_kind_from_string(layer);
    cfg.schedule = tpfuse::schedule_kind_from_string(schedule);
    cfg.tp_size = tp;
    cfg.batch = batch;
    cfg.seq = seq;
    cfg.d_model = d_model;
    cfg.heads = heads;
    cfg.granularity = granularity;
    cfg.seed = seed;
    cfg.reps = reps;
    std::ostringstream csv;
    tpfuse::run_bench(cfg, csv);
    const std::string s = csv.str();
    if (static_cast<int64_t>(s.size()) + 1 > cap) throw std::length_error("ref_bench_csv: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// Ulysses first all-to-all exactly as layers_test.cpp:347-397 drives it: per-group parts of
// this rank's sequence slice, tpfuse::ref_all_to_all, tpfuse::concat_seq.
extern "C" int ref_ulysses_a2a(int t, int batch, int heads, int64_t s, int64_t dh, const double* in, double* out) {
  return guarded([&] {
    const int64_t sl = s / t, hl = heads / t, bh = static_cast<int64_t>(batch) * heads;
    auto outs = tpfuse::spawn_group(t, [&](tpfuse::RankEndpoint& ep) {
      const int r = ep.rank();
      const tpfuse::Tensor slice = tensor_from(in + r * bh * sl * dh, bh, sl, dh);
      std::vector<tpfuse::Tensor> parts;
      for (int g = 0; g < t; ++g) {
        tpfuse::Tensor p(static_cast<int64_t>(batch) * hl, sl, dh);
        for (int64_t b = 0; b < batch; ++b)
          for (int64_t h = 0; h < hl; ++h)
            for (int64_t i = 0; i < sl; ++i)
              for (int64_t d = 0; d < dh; ++d) p(b * hl + h, i, d) = slice(b * heads + g * hl + h, i, d);
        parts.push_back(std::move(p));
      }
      return tpfuse::concat_seq(tpfuse::ref_all_to_all(ep, parts));
    });
    size_t off = 0;
    for (auto& o : outs) {
      copy_out(o, out + off);
      off += o.raw().size();
    }
  });
}
