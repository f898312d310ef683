// Seeded helpers used by the reference storage suite (the subset of its
// tests/generators.h:13-38 that test_storage.cpp needs), restated here so the
// suite builds without the out-of-scope notation module.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <set>
#include <vector>

#include "stam/storage.h"

namespace stam::testing {

using Rng = std::mt19937_64;

inline double uniformValue(Rng& rng) { return (double)(rng() >> 11) * (1.0 / 9007199254740992.0); }
inline int64_t uniformInt(Rng& rng, int64_t n) { return (int64_t)(rng() % (uint64_t)n); }

// Random COO entries at the given density, values in [0,1).
inline std::vector<std::pair<std::vector<int64_t>, double>> randomEntries(
    const std::vector<int64_t>& dims, double density, Rng& rng) {
  int64_t total = 1;
  for (int64_t d : dims) total *= d;
  const int64_t want = std::min<int64_t>(total, (int64_t)std::llround(density * (double)total));
  std::set<int64_t> picked;
  if (want == total) {
    for (int64_t p = 0; p < total; p++) picked.insert(p);
  } else {
    while ((int64_t)picked.size() < want) picked.insert(uniformInt(rng, total));
  }
  std::vector<std::pair<std::vector<int64_t>, double>> out;
  for (int64_t p : picked) {
    std::vector<int64_t> c(dims.size());
    for (int d = (int)dims.size() - 1; d >= 0; d--) {
      c[(size_t)d] = p % dims[(size_t)d];
      p /= dims[(size_t)d];
    }
    out.emplace_back(std::move(c), uniformValue(rng));
  }
  return out;
}

}  // namespace stam::testing
