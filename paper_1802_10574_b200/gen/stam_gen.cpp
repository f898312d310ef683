// stam_gen.cpp — seeded synthetic inputs with BASELINE.json's shapes.
//
// The reference's generators (tests/generators.h:13-38) use mt19937_64 and
// map a 64-bit draw to [0,1) as (x >> 11) * 2^-53.  This library keeps that
// value mapping and the `x % n` integer draw, but draws from one SplitMix64
// stream per row / slice so generation parallelises over host threads and is
// identical for any thread count.  Column sets are sampled without replacement
// and sorted, as BASELINE's configs require.  Parametrisations follow SURVEY
// Appendix B (documented in DESIGN.md §Inputs).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#define GEN_API extern "C" __attribute__((visibility("default")))

namespace {

// SplitMix64 finaliser: a bijective 64-bit mix.
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// One SplitMix64 stream per (seed, id).  The start state is a hash of both
// (not seed*C + id*G, which put stream id+1 one draw behind stream id on the
// same Weyl sequence and made neighbouring rows / slices shifted copies of each
// other), so streams of different ids start at unrelated points of the 2^64
// cycle.
struct Stream {
  uint64_t s;
  Stream(uint64_t seed, uint64_t id) {
    s = mix64(mix64(seed ^ 0x6A09E667F3BCC909ull) ^ mix64(id + 0x3C6EF372FE94F82Bull));
  }
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
  uint64_t below(uint64_t n) { return next() % n; }
};

template <typename F>
void parallel_dynamic(int64_t n, int nthreads, int64_t chunk, F f) {
  if (nthreads < 1) nthreads = 1;
  std::atomic<int64_t> next{0};
  auto work = [&]() {
    while (true) {
      const int64_t b = next.fetch_add(chunk);
      if (b >= n) break;
      const int64_t e = std::min(n, b + chunk);
      for (int64_t i = b; i < e; i++) f(i);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; t++) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
}

// `count` distinct keys uniform in [0, n), sorted ascending, into out.
void sample_distinct_sorted(Stream& rng, uint64_t n, int64_t count, std::vector<uint64_t>& out,
                            std::vector<uint64_t>& bitmap) {
  out.clear();
  if (count <= 0) return;
  if ((uint64_t)count * 32 >= n) {
    // dense: bitmap of n bits
    const size_t words = (size_t)((n + 63) / 64);
    bitmap.assign(words, 0);
    int64_t have = 0;
    if ((uint64_t)count * 2 > n) {
      // choose the complement
      std::fill(bitmap.begin(), bitmap.end(), ~0ull);
      if (n % 64) bitmap[words - 1] = (1ull << (n % 64)) - 1;
      int64_t drop = (int64_t)n - count;
      while (drop > 0) {
        const uint64_t k = rng.below(n);
        if (bitmap[k >> 6] >> (k & 63) & 1ull) {
          bitmap[k >> 6] &= ~(1ull << (k & 63));
          drop--;
        }
      }
    } else {
      while (have < count) {
        const uint64_t k = rng.below(n);
        if (!(bitmap[k >> 6] >> (k & 63) & 1ull)) {
          bitmap[k >> 6] |= 1ull << (k & 63);
          have++;
        }
      }
    }
    out.reserve((size_t)count);
    for (size_t w = 0; w < words; w++) {
      uint64_t m = bitmap[w];
      while (m) {
        const int b = __builtin_ctzll(m);
        out.push_back((uint64_t)w * 64 + b);
        m &= m - 1;
      }
    }
    return;
  }
  // sparse: draw, sort, dedup, top up
  out.reserve((size_t)count);
  while ((int64_t)out.size() < count) {
    const int64_t need = count - (int64_t)out.size();
    for (int64_t t = 0; t < need; t++) out.push_back(rng.below(n));
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
  }
}

}  // namespace

// Row lengths P(L) ∝ (L + q)^-a on [lmin, lmax], i.i.d. per row; writes the
// CSR pos array (nrows + 1).  Returns total nnz.
GEN_API int64_t gen_powerlaw_pos(int64_t nrows, double a, double q, int64_t lmin, int64_t lmax,
                                 uint64_t seed, int64_t* pos) {
  std::vector<double> cdf((size_t)(lmax - lmin + 1));
  double acc = 0;
  for (int64_t L = lmin; L <= lmax; L++) {
    acc += std::pow((double)L + q, -a);
    cdf[(size_t)(L - lmin)] = acc;
  }
  for (auto& c : cdf) c /= acc;
  Stream rng(seed, (1ull << 62) + 0x5eed);  // disjoint from the per-row ids
  pos[0] = 0;
  for (int64_t i = 0; i < nrows; i++) {
    const double u = rng.uniform();
    const int64_t L = lmin + (int64_t)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    pos[i + 1] = pos[i] + std::min(L, lmax);
  }
  return pos[nrows];
}

// Fills CSR rows whose lengths are given by pos: distinct uniform columns in
// [0, ncols), sorted; values lo + (hi - lo) * u.
GEN_API int gen_csr_fill(int64_t nrows, int64_t ncols, uint64_t seed, double lo, double hi,
                         const int64_t* pos, int64_t* idx, double* vals, int nthreads) {
  for (int64_t i = 0; i < nrows; i++)
    if (pos[i + 1] - pos[i] > ncols) return -1;
  parallel_dynamic(nrows, nthreads, 256, [&](int64_t i) {
    thread_local std::vector<uint64_t> keys, bitmap;
    Stream rng(seed, (uint64_t)i);
    const int64_t b = pos[i], n = pos[i + 1] - pos[i];
    sample_distinct_sorted(rng, (uint64_t)ncols, n, keys, bitmap);
    for (int64_t t = 0; t < n; t++) {
      idx[b + t] = (int64_t)keys[(size_t)t];
      vals[b + t] = lo + (hi - lo) * rng.uniform();
    }
  });
  return 0;
}

// Slice sizes for `nslices` drawn i.i.d. uniform per nonzero (multinomial).
GEN_API int gen_uniform_slice_counts(int64_t nslices, int64_t nnz, uint64_t seed, int64_t* counts,
                                     int nthreads) {
  if (nthreads < 1) nthreads = 1;
  std::memset(counts, 0, sizeof(int64_t) * (size_t)nslices);
  const int64_t chunk = 1 << 22;
  const int64_t nchunks = (nnz + chunk - 1) / chunk;
  std::vector<std::vector<int64_t>> part((size_t)nthreads);
  std::atomic<int64_t> next{0};
  auto work = [&](int t) {
    auto& h = part[(size_t)t];
    h.assign((size_t)nslices, 0);
    while (true) {
      const int64_t c = next.fetch_add(1);
      if (c >= nchunks) break;
      Stream rng(seed, (1ull << 61) + (uint64_t)c);
      const int64_t e = std::min(nnz, (c + 1) * chunk);
      for (int64_t p = c * chunk; p < e; p++) h[(size_t)rng.below((uint64_t)nslices)]++;
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; t++) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (auto& h : part)
    for (int64_t i = 0; i < nslices; i++) counts[i] += h[(size_t)i];
  return 0;
}

// CSF(3) with given nnz per i-slice; (j,k) distinct uniform over J x K per
// slice, stored sorted (fibers = distinct j).  Two phases so the caller can
// allocate: gen_csf3_plan computes fibers per slice (pass nullptr outputs),
// gen_csf3_fill regenerates the same pairs and fills the arrays.
namespace {
template <typename Emit>
void csf3_slices(int64_t I, int64_t J, int64_t K, const int64_t* slice_nnz, uint64_t seed,
                 int nthreads, Emit emit) {
  parallel_dynamic(I, nthreads, 1, [&](int64_t i) {
    thread_local std::vector<uint64_t> keys, bitmap;
    Stream rng(seed, (uint64_t)i);
    sample_distinct_sorted(rng, (uint64_t)J * (uint64_t)K, slice_nnz[i], keys, bitmap);
    emit(i, keys, rng);
  });
}
}  // namespace

GEN_API int gen_csf3_plan(int64_t I, int64_t J, int64_t K, const int64_t* slice_nnz, uint64_t seed,
                          int64_t* slice_fibers, int nthreads) {
  for (int64_t i = 0; i < I; i++)
    if (slice_nnz[i] < 0 || (uint64_t)slice_nnz[i] > (uint64_t)J * (uint64_t)K) return -1;
  csf3_slices(I, J, K, slice_nnz, seed, nthreads,
              [&](int64_t i, const std::vector<uint64_t>& keys, Stream&) {
                int64_t f = 0;
                uint64_t last = ~0ull;
                for (uint64_t key : keys) {
                  const uint64_t j = key / (uint64_t)K;
                  if (j != last) {
                    f++;
                    last = j;
                  }
                }
                slice_fibers[i] = f;
              });
  return 0;
}

// pos1 [I+1] and pos2 offsets must be derivable: the caller passes pos1 (from
// prefix sums of slice_fibers) and nz_off (prefix sums of slice_nnz).
GEN_API int gen_csf3_fill(int64_t I, int64_t J, int64_t K, const int64_t* slice_nnz, uint64_t seed,
                          const int64_t* pos1, const int64_t* nz_off, int64_t* idx1, int64_t* pos2,
                          int64_t* idx2, double* vals, double lo, double hi, int nthreads) {
  csf3_slices(I, J, K, slice_nnz, seed, nthreads,
              [&](int64_t i, const std::vector<uint64_t>& keys, Stream& rng) {
                int64_t f = pos1[i];
                int64_t p = nz_off[i];
                uint64_t last = ~0ull;
                for (uint64_t key : keys) {
                  const uint64_t j = key / (uint64_t)K, k = key % (uint64_t)K;
                  if (j != last) {
                    idx1[f] = (int64_t)j;
                    pos2[f] = p;
                    f++;
                    last = j;
                  }
                  idx2[p] = (int64_t)k;
                  vals[p] = lo + (hi - lo) * rng.uniform();
                  p++;
                }
              });
  if (I > 0) pos2[pos1[I]] = nz_off[I];
  return 0;
}

// Dense row-major matrix with values lo + (hi - lo) * u (one stream per row).
GEN_API int gen_dense(int64_t nrows, int64_t ncols, uint64_t seed, double lo, double hi,
                      double* out, int nthreads) {
  parallel_dynamic(nrows, nthreads, 1024, [&](int64_t i) {
    Stream rng(seed, (uint64_t)i);
    for (int64_t r = 0; r < ncols; r++) out[i * ncols + r] = lo + (hi - lo) * rng.uniform();
  });
  return 0;
}
