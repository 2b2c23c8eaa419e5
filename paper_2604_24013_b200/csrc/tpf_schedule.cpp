// Host schedule module: per-rank, per-iteration (send_peer, recv_peer,
// compute_slice) tables for the decomposed collectives. Tables are bit-exact
// with the reference (collectives.cpp:37-235; pinned by tests/test_schedule.py
// against the compiled reference and the golden fixtures) and are uploaded
// verbatim into the fused kernel's parameter block.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "tpf_host.h"

namespace tpf {

namespace {

// Round-robin tournament (circle method): rank n-1 stays fixed, the other n-1
// ranks rotate; round `round` pairs the fixed rank with u = n-2-round and the
// remaining ranks as reflections around u (mod n-1). (collectives.cpp:37-43)
int tournament_partner(int r, int round, int n) {
  const int fixed = n - 1;
  const int u = n - 2 - round;
  if (r == fixed) return u;
  if (r == u) return fixed;
  const int ring = n - 1;
  const int v = (2 * u - r) % ring;
  return v < 0 ? v + ring : v;
}

int mod(int a, int n) {
  const int v = a % n;
  return v < 0 ? v + n : v;
}

}  // namespace

Status ring_indices(bool rs, int r, int i, int n, int32_t out[3]) {
  if (n < 1) return Status::invalid(rs ? "ring_indices_rs: n must be >= 1" : "ring_indices_ag: n must be >= 1");
  if (r < 0 || r >= n || i < 0 || i >= n)
    return Status::invalid(std::string(rs ? "ring_indices_rs" : "ring_indices_ag") + ": rank " +
                           std::to_string(r) + " or iteration " + std::to_string(i) +
                           " outside [0," + std::to_string(n) + ")");
  out[0] = mod(r + 1, n);                   // Alg. 1/2: j = (r+1) mod N
  out[1] = mod(r - 1, n);                   //           k = (r-1+N) mod N
  out[2] = rs ? mod(r - i - 1, n) : mod(r - i, n);  // l: RS offset leaves own slice last
  return Status::ok();
}

Status build_schedule(int kind, int n, std::vector<int32_t>& table) {
  if (n < 1) return Status::invalid("build_schedule: n must be >= 1");
  if (kind < 0 || kind > 2) return Status::invalid("build_schedule: unknown schedule kind");
  if (kind == kPairwise && n % 2 != 0 && n != 1)
    return Status::invalid("build_schedule: pairwise schedule requires an even rank count, got " +
                           std::to_string(n));
  table.assign(static_cast<size_t>(n) * n * 3, -1);
  if (n == 1) {
    table.clear();
    return Status::ok();
  }
  for (int r = 0; r < n; ++r) {
    for (int i = 0; i < n; ++i) {
      int32_t* st = &table[(static_cast<size_t>(r) * n + i) * 3];
      const bool comm = i < n - 1;  // final iteration: own slice, no transfer
      int send = -1, recv = -1, slice = r;
      if (kind == kRing) {
        int32_t idx[3];
        ring_indices(true, r, i, n, idx);
        send = idx[0]; recv = idx[1]; slice = idx[2];
      } else if (kind == kCircular) {
        send = mod(r - 1, n); recv = mod(r + 1, n); slice = mod(r + i + 1, n);
      } else if (comm) {
        send = recv = slice = tournament_partner(r, i, n);
      }
      st[0] = comm ? send : -1;
      st[1] = comm ? recv : -1;
      st[2] = slice;
    }
  }
  return check_schedule(kind, n, table.data());
}

namespace {

// Symbolic replay: which (source rank, slice) contributions end up on each
// rank. Pipelined kinds forward a growing set; pairwise delivers one
// contribution per round (collectives.cpp:118-178).
bool delivery_exactly_once(int kind, int n, const int32_t* t, std::string& why) {
  auto at = [&](int r, int i, int f) { return t[(static_cast<size_t>(r) * n + i) * 3 + f]; };
  // count[r][src * n + slice]
  std::vector<std::vector<int>> final_set(n, std::vector<int>(n * n, 0));
  if (kind == kPairwise) {
    for (int i = 0; i < n; ++i)
      for (int r = 0; r < n; ++r) {
        const int dst = at(r, i, 0) >= 0 ? at(r, i, 0) : r;
        if (dst < 0 || dst >= n) { why = "peer out of range"; return false; }
        final_set[dst][r * n + at(r, i, 2)] += 1;
      }
  } else {
    std::vector<std::vector<int>> carry(n, std::vector<int>(n * n, 0));
    for (int i = 0; i < n; ++i) {
      std::vector<std::vector<int>> next(n, std::vector<int>(n * n, 0));
      for (int r = 0; r < n; ++r) {
        std::vector<int> part = i > 0 ? carry[r] : std::vector<int>(n * n, 0);
        part[r * n + at(r, i, 2)] += 1;
        const int dst = at(r, i, 0);
        if (dst >= n) { why = "peer out of range"; return false; }
        if (dst >= 0) next[dst] = part;
        else final_set[r] = part;
      }
      carry.swap(next);
    }
  }
  for (int r = 0; r < n; ++r) {
    int total = 0;
    for (int v : final_set[r]) total += v;
    if (total != n) {
      why = "rank " + std::to_string(r) + " accumulated " + std::to_string(total) +
            " contributions, expected " + std::to_string(n);
      return false;
    }
    for (int q = 0; q < n; ++q)
      if (final_set[r][q * n + r] != 1) {
        why = "contribution of rank " + std::to_string(q) + " for slice " + std::to_string(r) +
              " not delivered exactly once";
        return false;
      }
  }
  return true;
}

}  // namespace

Status check_schedule(int kind, int n, const int32_t* t) {
  auto fail = [](const std::string& why) { return Status::logic("check_schedule: " + why); };
  if (n < 1) return fail("group size must be >= 1");
  if (n == 1) return Status::ok();
  for (int r = 0; r < n; ++r) {
    int sends = 0, recvs = 0;
    for (int i = 0; i < n; ++i) {
      const int32_t* st = t + (static_cast<size_t>(r) * n + i) * 3;
      sends += st[0] >= 0;
      recvs += st[1] >= 0;
      if (st[2] < 0 || st[2] >= n) return fail("compute slice out of range");
    }
    if (sends != n - 1 || recvs != n - 1)
      return fail("rank " + std::to_string(r) + " posts " + std::to_string(sends) + " sends / " +
                  std::to_string(recvs) + " recvs, expected " + std::to_string(n - 1) + " each");
    if (t[(static_cast<size_t>(r) * n + n - 1) * 3 + 2] != r)
      return fail("rank " + std::to_string(r) + " must compute its own slice last");
  }
  if (kind == kPairwise) {
    for (int i = 0; i < n - 1; ++i) {
      std::vector<int> seen(n, 0);
      for (int r = 0; r < n; ++r) {
        const int32_t* st = t + (static_cast<size_t>(r) * n + i) * 3;
        if (st[0] != st[1]) return fail("pairwise exchange must be bidirectional");
        if (st[0] < 0 || st[0] >= n) return fail("pairwise partner out of range");
        if (t[(static_cast<size_t>(st[0]) * n + i) * 3] != r)
          return fail("pairwise partners disagree in round " + std::to_string(i));
        if (seen[r]++) return fail("rank appears in two pairs of one round");
      }
    }
  }
  std::string why;
  if (!delivery_exactly_once(kind, n, t, why)) return fail(why);
  return Status::ok();
}

}  // namespace tpf
