// Host-side internal API of libtpfuse_b200 (schedule module + status type).
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "tpf.h"

namespace tpf {

constexpr int kRing = TPF_RING;
constexpr int kPairwise = TPF_PAIRWISE;
constexpr int kCircular = TPF_CIRCULAR;

struct Status {
  int code = TPF_OK;
  std::string msg;
  static Status ok() { return {}; }
  static Status invalid(std::string m) { return {TPF_E_INVALID, std::move(m)}; }
  static Status shape(std::string m) { return {TPF_E_SHAPE, std::move(m)}; }
  static Status logic(std::string m) { return {TPF_E_LOGIC, std::move(m)}; }
  static Status cuda(std::string m) { return {TPF_E_CUDA, std::move(m)}; }
  static Status peer(std::string m) { return {TPF_E_PEER, std::move(m)}; }
  static Status capacity(std::string m) { return {TPF_E_CAPACITY, std::move(m)}; }
  bool good() const { return code == TPF_OK; }
};

Status ring_indices(bool rs, int r, int i, int n, int32_t out[3]);
Status build_schedule(int kind, int n, std::vector<int32_t>& table);
Status check_schedule(int kind, int n, const int32_t* table);

}  // namespace tpf
