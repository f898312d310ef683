// stam/io.h — exchange formats (the reference's src/io.cpp is
// a placeholder): Matrix Market coordinate files and FROSTT .tns files.
#pragma once

#include <string>

#include "stam/storage.h"

namespace stam {

/// Matrix Market coordinate file -> csr() with sorted columns.  Fields real,
/// integer and pattern (pattern entries get 1.0); symmetric and
/// skew-symmetric files are expanded to general; duplicate coordinates are
/// summed in file order.  Malformed input throws Error(Io) naming the line;
/// coordinates outside [1, dim] throw Error(OutOfRange).
TensorStorage loadMatrixMarket(const std::string& path);

/// FROSTT .tns file (whitespace-separated 1-based coordinates then the value;
/// '#' comments) -> {dense, compressed, ...} storage (csf(order); csr() for
/// order 2).  The order comes from the first entry line; dimensions are the
/// largest coordinate of each mode unless `dims` is given.  Duplicates are
/// summed in file order; coordinate 0 throws Error(OutOfRange).
TensorStorage loadTns(const std::string& path, const std::vector<int64_t>& dims = {});

/// Writes `t` to `path`: "matrix coordinate real general" Matrix Market when
/// the path ends in .mtx (order 2), FROSTT .tns otherwise; 1-based, values
/// with 17 significant digits, so load(store(x)) == x for ordered storage.
void store(const std::string& path, const TensorStorage& t);

}  // namespace stam
