// stam/workspace.h — the paper's dense workspace (source-compatible with the
// reference include/stam/workspace.h:14-60): values, guard flags and the list
// of inserted coordinates; reset costs O(insertions).  The GPU kernels
// reproduce exactly these semantics (insert-assign, insert-accumulate into
// 0.0, presence checks, sorted drain).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "stam/error.h"

namespace stam {

class Workspace {
 public:
  explicit Workspace(std::vector<int64_t> dimensions);

  int64_t size() const { return (int64_t)values_.size(); }
  int64_t nnz() const { return (int64_t)inserted_.size(); }
  const std::vector<int64_t>& dimensions() const { return dims_; }
  const std::vector<int64_t>& insertedCoords() const { return inserted_; }

  int64_t linearize(const std::vector<int64_t>& coords) const;
  void insert(int64_t coord, double value, bool accumulate);
  void mark(int64_t coord);
  double value(int64_t coord) const;
  bool present(int64_t coord) const { return guard_[(size_t)coord] != 0; }
  std::vector<std::pair<int64_t, double>> drain(bool sort);
  void reset();
  int64_t touchedEntries() const { return touched_; }
  void checkClean() const;

 private:
  void check(int64_t coord) const;

  std::vector<int64_t> dims_;
  std::vector<double> values_;
  std::vector<unsigned char> guard_;
  std::vector<int64_t> inserted_;
  int64_t touched_ = 0;
};

}  // namespace stam
