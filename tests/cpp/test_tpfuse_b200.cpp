// C++ parity tests for the tpfuse_b200 host mirror (include/tpfuse_b200/tpfuse.hpp),
// written like the reference's GoogleTest suites (collectives_test.cpp, layers_test.cpp,
// acceptance_test.cpp C1/C3/C7): integer data from the reference's randint recipe
// (std::mt19937_64() % span, tensor.cpp:234-250), central / single-device oracles,
// exact equality. GTest is not in the image, so this is a minimal self-contained runner.
//
//   test_tpfuse_b200 --cpu   schedule / error tests only (no GPU needed)
//   test_tpfuse_b200         everything (needs an sm_100 GPU)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "tpfuse_b200/tpfuse.hpp"

using namespace tpfuse_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                             \
  do {                                                                          \
    if (!(cond)) {                                                              \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);             \
      ++g_fail;                                                                 \
      return;                                                                   \
    }                                                                           \
  } while (0)
#define CHECK_THROWS(stmt, Exc)                                                 \
  do {                                                                          \
    bool thrown_ = false;                                                       \
    try {                                                                       \
      stmt;                                                                     \
    } catch (const Exc&) {                                                      \
      thrown_ = true;                                                           \
    }                                                                           \
    if (!thrown_) {                                                             \
      std::printf("  FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__,   \
                  #stmt, #Exc);                                                 \
      ++g_fail;                                                                 \
      return;                                                                   \
    }                                                                           \
  } while (0)

static void run(const char* name, const std::function<void()>& f) {
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception& e) {
    std::printf("  FAIL %s: unexpected exception: %s\n", name, e.what());
    ++g_fail;
  }
  if (g_fail == before) {
    ++g_pass;
    std::printf("[PASS] %s\n", name);
  } else {
    std::printf("[FAIL] %s\n", name);
  }
}

// ---- reference data recipe and central oracles
static Tensor randint_fill(int64_t b, int64_t s, int64_t d, int lo, int hi, uint64_t seed) {
  std::mt19937_64 e(seed);
  const uint64_t span = static_cast<uint64_t>(hi - lo);
  Tensor t(b, s, d);
  for (double& v : t.raw()) v = static_cast<double>(lo + static_cast<int64_t>(e() % span));
  return t;
}

static Matrix randint_matrix(int64_t r, int64_t c, int lo, int hi, uint64_t seed) {
  std::mt19937_64 e(seed);
  const uint64_t span = static_cast<uint64_t>(hi - lo);
  Matrix m(r, c);
  for (double& v : m.raw()) v = static_cast<double>(lo + static_cast<int64_t>(e() % span));
  return m;
}

static Tensor matmul(const Tensor& x, const Matrix& w) {
  Tensor o(x.batch(), x.seq(), w.cols());
  for (int64_t b = 0; b < x.batch(); ++b)
    for (int64_t s = 0; s < x.seq(); ++s)
      for (int64_t c = 0; c < w.cols(); ++c) {
        double acc = 0;
        for (int64_t k = 0; k < x.feat(); ++k) acc += x(b, s, k) * w(k, c);
        o(b, s, c) = acc;
      }
  return o;
}

static Tensor seq_slice(const Tensor& x, int n, int i) {
  const int64_t p = x.seq() / n;
  Tensor o(x.batch(), p, x.feat());
  for (int64_t b = 0; b < x.batch(); ++b)
    for (int64_t s = 0; s < p; ++s)
      for (int64_t d = 0; d < x.feat(); ++d) o(b, s, d) = x(b, i * p + s, d);
  return o;
}

static Tensor feat_block(const Tensor& x, int64_t k0, int64_t len) {
  Tensor o(x.batch(), x.seq(), len);
  for (int64_t b = 0; b < x.batch(); ++b)
    for (int64_t s = 0; s < x.seq(); ++s)
      for (int64_t d = 0; d < len; ++d) o(b, s, d) = x(b, s, k0 + d);
  return o;
}

static uint64_t mix_seed(uint64_t seed, uint64_t salt) {  // experiment.cpp:163-168
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------- CPU tests
static void schedule_tests() {
  run("RingIndices.Formulas", [] {
    const RingIndices ag = ring_indices_ag(0, 1, 4);
    CHECK(ag.send_peer == 1 && ag.recv_peer == 3 && ag.compute_slice == 3);
    const RingIndices rs = ring_indices_rs(0, 0, 4);
    CHECK(rs.send_peer == 1 && rs.recv_peer == 3 && rs.compute_slice == 3);
    for (int n = 1; n <= 8; ++n)
      for (int r = 0; r < n; ++r) {
        CHECK(ring_indices_ag(r, 0, n).compute_slice == r);
        CHECK(ring_indices_rs(r, n - 1, n).compute_slice == r);
      }
    CHECK_THROWS(ring_indices_ag(4, 0, 4), std::invalid_argument);
  });
  run("Schedule.PairwiseRoundsN4", [] {
    const Schedule s = build_schedule(ScheduleKind::PairwiseBidirectional, 4);
    const int want[3][4] = {{1, 0, 3, 2}, {2, 3, 0, 1}, {3, 2, 1, 0}};
    for (int i = 0; i < 3; ++i)
      for (int r = 0; r < 4; ++r) CHECK(s.steps[r][i].send_peer == want[i][r]);
  });
  run("Schedule.InvariantsAllKinds", [] {
    for (int n : {2, 4, 6, 8})
      for (ScheduleKind k : {ScheduleKind::Ring, ScheduleKind::PairwiseBidirectional, ScheduleKind::CircularSlices}) {
        const Schedule s = build_schedule(k, n);
        check_schedule(s);
        for (int r = 0; r < n; ++r) {
          CHECK(s.steps[r].back().compute_slice == r);
          CHECK(!s.steps[r].back().has_comm());
        }
      }
  });
  run("Schedule.Rejections", [] {
    CHECK_THROWS(build_schedule(ScheduleKind::PairwiseBidirectional, 3), std::invalid_argument);
    CHECK_THROWS(build_schedule(ScheduleKind::Ring, 0), std::invalid_argument);
    Schedule s = build_schedule(ScheduleKind::Ring, 4);
    s.steps[1][3].compute_slice = 0;
    CHECK_THROWS(check_schedule(s), std::logic_error);
    CHECK(build_schedule(ScheduleKind::Ring, 1).iterations() == 0);
  });
  run("ShardedLinear.SplitErrors", [] {
    CHECK_THROWS(ShardedLinear::split_rows(Matrix(6, 4), 4), ShapeError);
    CHECK_THROWS(ShardedLinear::split_columns(Matrix(4, 6), 4), ShapeError);
  });
}

// ------------------------------------------------------------- GPU tests
// Single-device attention in double (reference_attention, layers.cpp:107-118 semantics):
// folded (batch*heads, S, Dh), rows [q0, q0+nq) of the queries; returns (batch*heads, nq, Dh).
static Tensor attention_ref(const Tensor& q, const Tensor& k, const Tensor& v, int64_t q0, int64_t nq, bool scale) {
  const int64_t G = q.batch(), S = k.seq(), Dh = q.feat();
  Tensor out(G, nq, Dh);
  std::vector<double> sc(static_cast<size_t>(S));
  const double f = scale ? 1.0 / std::sqrt(static_cast<double>(Dh)) : 1.0;
  for (int64_t g = 0; g < G; ++g)
    for (int64_t i = 0; i < nq; ++i) {
      double mx = -1e300;
      for (int64_t j = 0; j < S; ++j) {
        double d = 0;
        for (int64_t c = 0; c < Dh; ++c) d += q(g, q0 + i, c) * k(g, j, c);
        sc[j] = d * f;
        mx = std::max(mx, sc[j]);
      }
      double sum = 0;
      for (int64_t j = 0; j < S; ++j) sum += (sc[j] = std::exp(sc[j] - mx));
      for (int64_t c = 0; c < Dh; ++c) {
        double a = 0;
        for (int64_t j = 0; j < S; ++j) a += sc[j] * v(g, j, c);
        out(g, i, c) = a / sum;
      }
    }
  return out;
}

static double rel_dev(const Tensor& a, const Tensor& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.raw().size(); ++i) {
    num = std::max(num, std::fabs(a.raw()[i] - b.raw()[i]));
    den = std::max(den, std::fabs(b.raw()[i]));
  }
  return den > 0 ? num / den : num;
}

static Tensor uniform_bf16(int64_t b, int64_t s, int64_t d, uint64_t seed) {
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  Tensor t(b, s, d);
  for (double& x : t.raw()) {
    float f = static_cast<float>(u(gen));
    uint32_t bits;
    std::memcpy(&bits, &f, 4);
    bits &= 0xffff0000u;  // exactly representable in bf16
    std::memcpy(&f, &bits, 4);
    x = f;
  }
  return t;
}

// bf16 device copy of host values (all exactly representable: integer test data)
static void* to_device_bf16(const std::vector<double>& v) {
  std::vector<uint16_t> h(v.size());
  for (size_t i = 0; i < v.size(); ++i) h[i] = detail::to_bf16(v[i]);
  void* d = nullptr;
  detail::cuda_check(cudaMalloc(&d, h.size() * 2), "cudaMalloc");
  detail::cuda_check(cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "cudaMemcpy");
  return d;
}

static Tensor from_device_f32(const void* d, int64_t b, int64_t s, int64_t n) {
  std::vector<float> h(static_cast<size_t>(b * s * n));
  detail::cuda_check(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  Tensor t(b, s, n);
  for (size_t i = 0; i < h.size(); ++i) t.raw()[i] = h[i];
  return t;
}

// The reference's threading model on the per-rank path: one worker thread per rank
// (spawn_group), each calling the device-level drop-ins on its own RankEndpoint of a split group.
static void split_group_tests() {
  run("SplitGroup.SpawnGroupRowAndColumnParallelExact", [] {
    const int t = 4, B = 1, S = 256, K = 128, N = 256;
    const Tensor x = randint_fill(B, S, K, 0, 5, 31);
    const Matrix wm = randint_matrix(K, N, -2, 2, 32);
    const Tensor full = matmul(x, wm);
    SplitGroup g(t, tpf_sym_bytes_rs(t, B, S, K / t, N, 1, TPF_F32) + tpf_sym_bytes_ag(t, B, S, K, N / t, 1));
    const ShardedLinear rows = ShardedLinear::split_rows(wm, t), cols = ShardedLinear::split_columns(wm, t);
    for (ScheduleKind k : {ScheduleKind::Ring, ScheduleKind::PairwiseBidirectional, ScheduleKind::CircularSlices}) {
      const auto got = spawn_group(g, [&](RankEndpoint& ep) {
        const int r = ep.rank();
        DeviceTensor xd{to_device_bf16(feat_block(x, r * (K / t), K / t).raw()), B, S, K / t, TPF_BF16};
        DeviceTensor wd{to_device_bf16(rows.shard(r).raw()), 1, K / t, N, TPF_BF16};
        DeviceTensor yd{nullptr, B, S / t, N, TPF_F32};
        detail::cuda_check(cudaMalloc(&yd.data, sizeof(float) * B * (S / t) * N), "cudaMalloc");
        row_parallel_forward(ep, xd, wd, build_schedule(k, t), yd);
        ep.sync();
        Tensor y = from_device_f32(yd.data, B, S / t, N);
        cudaFree(xd.data); cudaFree(wd.data); cudaFree(yd.data);
        return y;
      });
      for (int r = 0; r < t; ++r) CHECK(got[r] == seq_slice(full, t, r));
    }
    const auto col = spawn_group(g, [&](RankEndpoint& ep) {
      const int r = ep.rank();
      DeviceTensor xd{to_device_bf16(seq_slice(x, t, r).raw()), B, S / t, K, TPF_BF16};
      DeviceTensor wd{to_device_bf16(cols.shard(r).raw()), 1, K, N / t, TPF_BF16};
      DeviceTensor yd{nullptr, B, S, N / t, TPF_F32};
      detail::cuda_check(cudaMalloc(&yd.data, sizeof(float) * B * S * (N / t)), "cudaMalloc");
      column_parallel_forward(ep, xd, wd, yd);
      ep.sync();
      Tensor y = from_device_f32(yd.data, B, S, N / t);
      cudaFree(xd.data); cudaFree(wd.data); cudaFree(yd.data);
      return y;
    });
    for (int r = 0; r < t; ++r) CHECK(col[r] == feat_block(full, r * (N / t), N / t));
  });
  // fabric_test.cpp:44-58: a failing rank surfaces as GroupError naming it
  run("SplitGroup.SpawnGroupFailingRankIsNamed", [] {
    const int t = 4, B = 1, S = 256, K = 128, N = 256;
    SplitGroup g(t, tpf_sym_bytes_rs(t, B, S, K / t, N, 1, TPF_F32));
    for (int r = 0; r < t; ++r) {
      tpf_comm_set_timeout_ns(g.endpoint(r).handle(), 200ll * 1000 * 1000);
      tpf_comm_inject_fault(g.endpoint(r).handle(), 2);
    }
    int failing = -1;
    try {
      spawn_group(g, [&](RankEndpoint& ep) {
        DeviceTensor xd{nullptr, B, S, K / t, TPF_BF16}, wd{nullptr, 1, K / t, N, TPF_BF16},
            yd{nullptr, B, S / t, N, TPF_F32};
        cudaMalloc(&xd.data, 2 * B * S * (K / t));
        cudaMemset(xd.data, 0, 2 * B * S * (K / t));
        cudaMalloc(&wd.data, 2 * (K / t) * N);
        cudaMemset(wd.data, 0, 2 * (K / t) * N);
        cudaMalloc(&yd.data, 4 * B * (S / t) * N);
        row_parallel_forward(ep, xd, wd, build_schedule(ScheduleKind::Ring, t), yd);
        try {
          ep.sync();
        } catch (...) {
          cudaFree(xd.data); cudaFree(wd.data); cudaFree(yd.data);
          throw;
        }
        cudaFree(xd.data); cudaFree(wd.data); cudaFree(yd.data);
      });
    } catch (const GroupError& e) {
      failing = e.failing_rank();
    }
    CHECK(failing == 2);
  });
}

static void gpu_tests() {
  split_group_tests();
  // SPEC acceptance C1: T in {1,2,4,8}, m in {1,2}, every applicable schedule, seeds 0-4,
  // B=2, S=64, D=32, hidden 64; exact equality with the single-device oracle.
  run("Acceptance.C1.ExactOracleEquivalence", [] {
    for (int t : {1, 2, 4, 8})
      for (uint64_t seed = 0; seed < 5; ++seed) {
        LocalGroup g(t);
        const int B = 2, S = 64, D = 32, H = 64;
        const Tensor x = randint_fill(B, S, D, 0, 5, mix_seed(seed, 0));
        const Matrix upm = randint_matrix(D, H, -2, 2, mix_seed(seed, 1));
        const Matrix w2m = randint_matrix(D, D, -2, 2, mix_seed(seed, 4));
        const ShardedLinear up = ShardedLinear::split_columns(upm, t);
        const ShardedLinear w2 = ShardedLinear::split_rows(w2m, t);
        const Tensor col_full = matmul(x, upm);
        const Tensor x2 = randint_fill(B, S, D, 0, 5, mix_seed(seed, 3));
        const Tensor row_full = matmul(x2, w2m);
        std::vector<Tensor> slices, feats;
        for (int r = 0; r < t; ++r) {
          slices.push_back(seq_slice(x, t, r));
          feats.push_back(feat_block(x2, r * (D / t), D / t));
        }
        for (int m : {1, 2}) {
          const auto col = g.column_parallel_forward(slices, up, m);
          for (int r = 0; r < t; ++r) CHECK(col[r] == feat_block(col_full, r * (H / t), H / t));
          for (ScheduleKind k : {ScheduleKind::Ring, ScheduleKind::PairwiseBidirectional, ScheduleKind::CircularSlices}) {
            if (k == ScheduleKind::PairwiseBidirectional && t % 2 && t != 1) continue;
            if (m > 1 && k != ScheduleKind::Ring) continue;
            const auto row = g.row_parallel_forward(feats, w2, build_schedule(k, t), m);
            for (int r = 0; r < t; ++r) CHECK(row[r] == seq_slice(row_full, t, r));
          }
        }
      }
  });
  // C7: byte-identical results across schedules (integer data).
  run("Acceptance.C7.CrossScheduleByteIdentity", [] {
    const int t = 4;
    LocalGroup g(t);
    const Tensor x = randint_fill(2, 64, 64, -4, 5, 11);
    const ShardedLinear w = ShardedLinear::split_rows(randint_matrix(64, 48, -2, 2, 12), t);
    std::vector<Tensor> feats;
    for (int r = 0; r < t; ++r) feats.push_back(feat_block(x, r * 16, 16));
    const auto a = g.row_parallel_forward(feats, w, build_schedule(ScheduleKind::Ring, t));
    const auto b = g.row_parallel_forward(feats, w, build_schedule(ScheduleKind::PairwiseBidirectional, t));
    const auto c = g.row_parallel_forward(feats, w, build_schedule(ScheduleKind::CircularSlices, t));
    for (int r = 0; r < t; ++r) CHECK(a[r] == b[r] && a[r] == c[r]);
  });
  // layers_test.cpp MLP with the square activation (hidden kept in bf16: exact while
  // hidden^2 stays a bf16-representable integer -> small data).
  run("Layers.TpspMlpSquareExact", [] {
    const int t = 4;
    LocalGroup g(t);
    const Tensor x = randint_fill(2, 32, 16, 0, 2, 21);
    const Matrix upm = randint_matrix(16, 32, -1, 2, 22);
    const Matrix downm = randint_matrix(32, 16, -2, 2, 23);
    Tensor hid = matmul(x, upm);
    for (double& v : hid.raw()) v = v * v;
    const Tensor want = matmul(hid, downm);
    std::vector<Tensor> slices;
    for (int r = 0; r < t; ++r) slices.push_back(seq_slice(x, t, r));
    const auto out = g.tpsp_mlp_forward(slices, ShardedLinear::split_columns(upm, t),
                                        ShardedLinear::split_rows(downm, t), Activation::Square,
                                        build_schedule(ScheduleKind::Ring, t));
    for (int r = 0; r < t; ++r) CHECK(out[r] == seq_slice(want, t, r));
  });
  // layers_test.cpp FuseAllToAllAttention: rank l receives, from every source rank q,
  // merge_heads(attention(q's head group, query slice l)) at feature block q.
  run("Layers.FuseAllToAllAttentionMatchesReference", [] {
    for (int t : {2, 4})
      for (int64_t dh : {int64_t(128), int64_t(32)}) {  // fused flash kernel / GEMM family
        LocalGroup g(t);
        const int batch = 2, heads = 2;
        const int64_t S = 128 * t;
        std::vector<AttentionInputs> in;
        for (int r = 0; r < t; ++r)
          in.push_back(make_attention_inputs(batch, heads, uniform_bf16(batch * heads, S, dh, 100 + r),
                                             uniform_bf16(batch * heads, S, dh, 200 + r),
                                             uniform_bf16(batch * heads, S, dh, 300 + r)));
        const auto out = g.fuse_all_to_all_attention(in);
        const int64_t sl = S / t;
        for (int l = 0; l < t; ++l) {
          Tensor want(batch, sl, static_cast<int64_t>(t) * heads * dh);
          for (int q = 0; q < t; ++q) {
            const Tensor ctx = attention_ref(in[q].q, in[q].k, in[q].v, l * sl, sl, true);
            for (int b = 0; b < batch; ++b)
              for (int hh = 0; hh < heads; ++hh)
                for (int64_t i = 0; i < sl; ++i)
                  for (int64_t c = 0; c < dh; ++c)
                    want(b, i, (static_cast<int64_t>(q) * heads + hh) * dh + c) = ctx(b * heads + hh, i, c);
          }
          CHECK(rel_dev(out[l], want) <= 2e-2);
        }
      }
  });
  // query_split_attention (layers.cpp:149-172): fuse_reduce_scatter of
  // merge_heads(attention(q_slice)) . W_o[r] over the query sequence, every schedule.
  run("Layers.QuerySplitAttentionMatchesReference", [] {
    const int t = 2, batch = 1, heads = 2;
    const int64_t S = 256 * t, dh = 128, D = 64;
    LocalGroup g(t);
    std::vector<AttentionInputs> in;
    for (int r = 0; r < t; ++r)
      in.push_back(make_attention_inputs(batch, heads, uniform_bf16(batch * heads, S, dh, 400 + r),
                                         uniform_bf16(batch * heads, S, dh, 500 + r),
                                         uniform_bf16(batch * heads, S, dh, 600 + r)));
    Matrix wo(static_cast<int64_t>(t) * heads * dh, D);
    {
      const Tensor w = uniform_bf16(1, t * heads * dh, D, 700);
      for (int64_t i = 0; i < wo.rows(); ++i)
        for (int64_t c = 0; c < D; ++c) wo(i, c) = w(0, i, c) / 16;
    }
    const ShardedLinear wos = ShardedLinear::split_rows(wo, t);
    // central: y = sum_r merge_heads(attention_r) . W_o[r], sequence-sliced
    Tensor y(batch, S, D);
    for (int r = 0; r < t; ++r) {
      const Tensor ctx = attention_ref(in[r].q, in[r].k, in[r].v, 0, S, true);
      for (int b = 0; b < batch; ++b)
        for (int64_t i = 0; i < S; ++i)
          for (int64_t c = 0; c < D; ++c) {
            double a = 0;
            for (int hh = 0; hh < heads; ++hh)
              for (int64_t e = 0; e < dh; ++e) a += ctx(b * heads + hh, i, e) * wos.shard(r)(hh * dh + e, c);
            y(b, i, c) += a;
          }
    }
    for (ScheduleKind k : {ScheduleKind::Ring, ScheduleKind::PairwiseBidirectional, ScheduleKind::CircularSlices}) {
      const auto out = g.query_split_attention(in, wos, build_schedule(k, t));
      for (int r = 0; r < t; ++r) CHECK(rel_dev(out[r], seq_slice(y, t, r)) <= 2e-2);
    }
  });
  run("Layers.AttentionErrorBehaviour", [] {
    LocalGroup g(2);
    CHECK_THROWS(make_attention_inputs(1, 2, Tensor(3, 8, 8), Tensor(3, 8, 8), Tensor(3, 8, 8)), ShapeError);
    std::vector<AttentionInputs> in;
    for (int r = 0; r < 2; ++r)
      in.push_back(make_attention_inputs(1, 1, Tensor(1, 129, 8), Tensor(1, 129, 8), Tensor(1, 129, 8)));
    CHECK_THROWS(g.fuse_all_to_all_attention(in), std::invalid_argument);  // 129 % 2
  });
  run("Layers.ErrorBehaviour", [] {
    LocalGroup g(4);
    std::vector<Tensor> xs(4, Tensor(1, 64, 16));
    const ShardedLinear rows = ShardedLinear::split_rows(Matrix(64, 16), 4);
    const ShardedLinear cols = ShardedLinear::split_columns(Matrix(16, 16), 4);
    CHECK_THROWS(g.row_parallel_forward(xs, cols, build_schedule(ScheduleKind::Ring, 4)), std::invalid_argument);
    CHECK_THROWS(g.row_parallel_forward(xs, ShardedLinear::split_rows(Matrix(64, 16), 2),
                                        build_schedule(ScheduleKind::Ring, 4)),
                 std::invalid_argument);
    std::vector<Tensor> xr(4, Tensor(1, 64, 16));
    const ShardedLinear r4 = ShardedLinear::split_rows(Matrix(64, 16), 4);
    CHECK_THROWS(g.row_parallel_forward(xr, r4, build_schedule(ScheduleKind::PairwiseBidirectional, 4), 2),
                 std::invalid_argument);
    CHECK_THROWS(g.row_parallel_forward(xr, r4, build_schedule(ScheduleKind::Ring, 2)), std::invalid_argument);
    std::vector<Tensor> odd(4, Tensor(1, 6, 16));
    CHECK_THROWS(g.row_parallel_forward(odd, r4, build_schedule(ScheduleKind::Ring, 4)), std::invalid_argument);
  });
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  schedule_tests();
  if (!cpu_only) gpu_tests();
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
