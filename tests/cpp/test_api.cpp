// C++ API tests: the stam storage/workspace surface and the stam::spgemm /
// spadd / mttkrp entry points (GPU cases run only with STAM_TEST_GPU=1).
#define SHIM_MAIN
#include "doctest.h"

#include <cstdlib>
#include <cstring>
#include <vector>

#include "stam/kernels.h"
#include "stam/storage.h"
#include "stam/workspace.h"

using namespace stam;

static bool g_gpu = false;

static TensorStorage csrOf(int64_t rows, int64_t cols, std::vector<int64_t> pos,
                           std::vector<int64_t> idx, std::vector<double> vals) {
  std::vector<TensorStorage::Level> levels(2);
  levels[1].pos = std::move(pos);
  levels[1].idx = std::move(idx);
  return TensorStorage::fromArrays({rows, cols}, csr(), std::move(levels), std::move(vals));
}

TEST_CASE("fromArrays adopts and validates") {
  TensorStorage t = csrOf(2, 3, {0, 1, 3}, {2, 0, 1}, {1.0, 2.0, 3.0});
  CHECK(t.storedCount() == 3);
  CHECK(t.locate({1, 1}) == 2);
  CHECK_THROWS_AS(csrOf(2, 3, {0, 2, 3}, {2, 0, 1}, {1.0, 2.0, 3.0}), Error);  // unordered
  CHECK_THROWS_AS(csrOf(2, 3, {0, 1, 3}, {2, 0, 5}, {1.0, 2.0, 3.0}), Error);  // out of range
}

TEST_CASE("builder appends rows, closes trailing rows and sums duplicates") {
  TensorBuilder b({3, 4}, csr());
  b.appendRow({0}, {{1, 1.0}, {3, 2.0}});
  b.append({0, 3}, 5.0);  // duplicate adds
  b.appendRow({2}, {{0, 4.0}});
  TensorStorage t = b.finalize();
  CHECK(t.level(1).pos == std::vector<int64_t>{0, 2, 2, 3});
  CHECK(t.level(1).idx == std::vector<int64_t>{1, 3, 0});
  CHECK(t.vals() == std::vector<double>{1.0, 7.0, 4.0});
  TensorBuilder c({2, 2}, csr());
  c.appendRow({1}, {{0, 1.0}});
  CHECK_THROWS_AS(c.appendRow({0}, {{0, 1.0}}), Error);
}

TEST_CASE("csf(3) storage and iteration") {
  TensorStorage t = fromCoo({2, 3, 4}, csf(3), {{{1, 2, 3}, 1.0}, {{0, 1, 0}, 2.0}, {{1, 2, 1}, 3.0}});
  CHECK(t.level(1).pos == std::vector<int64_t>{0, 1, 2});
  CHECK(t.level(2).pos == std::vector<int64_t>{0, 1, 3});
  CHECK(t.level(2).idx == std::vector<int64_t>{0, 1, 3});
  CHECK(t.vals() == std::vector<double>{2.0, 3.0, 1.0});
}

TEST_CASE("workspace insert / present / drain / reset") {
  Workspace w({8});
  w.insert(5, 1.0, true);
  w.insert(2, 2.0, false);
  w.insert(5, 0.5, true);
  CHECK(w.present(5));
  CHECK(!w.present(0));
  auto d = w.drain(true);
  REQUIRE(d.size() == 2);
  CHECK(d[0] == std::pair<int64_t, double>{2, 2.0});
  CHECK(d[1] == std::pair<int64_t, double>{5, 1.5});
  w.checkClean();
  CHECK(w.touchedEntries() == 5);
}

TEST_CASE("gpu: spgemm identity and a known product") {
  if (!g_gpu) return;
  TensorStorage I = csrOf(3, 3, {0, 1, 2, 3}, {0, 1, 2}, {1, 1, 1});
  ExecutionStats st;
  TensorStorage C = spgemm(I, I, {}, &st);
  CHECK(C.level(1).idx == I.level(1).idx);
  CHECK(C.vals() == I.vals());
  CHECK(st.mults == 3);
  // [[1,2],[0,3]] x [[4,0],[5,6]] = [[14,12],[15,18]]
  TensorStorage A = csrOf(2, 2, {0, 2, 3}, {0, 1, 1}, {1, 2, 3});
  TensorStorage B = csrOf(2, 2, {0, 1, 3}, {0, 0, 1}, {4, 5, 6});
  TensorStorage P = spgemm(A, B);
  CHECK(P.level(1).pos == std::vector<int64_t>{0, 2, 4});
  CHECK(P.vals() == std::vector<double>{14, 12, 15, 18});
}

TEST_CASE("gpu: spadd of three operands") {
  if (!g_gpu) return;
  TensorStorage a = csrOf(2, 4, {0, 2, 2}, {0, 3}, {1, 2});
  TensorStorage b = csrOf(2, 4, {0, 1, 2}, {3, 1}, {10, 20});
  TensorStorage c = csrOf(2, 4, {0, 0, 2}, {1, 2}, {100, 200});
  const TensorStorage* ops[] = {&a, &b, &c};
  TensorStorage d = spadd(ops);
  CHECK(d.level(1).pos == std::vector<int64_t>{0, 2, 4});
  CHECK(d.level(1).idx == std::vector<int64_t>{0, 3, 1, 2});
  CHECK(d.vals() == std::vector<double>{1, 12, 120, 200});
  CHECK_THROWS_AS(spgemm(a, a), Error);  // 2x4 * 2x4: dimension mismatch
}

TEST_CASE("gpu: mttkrp dense and sparse") {
  if (!g_gpu) return;
  // B(0,0,0)=1, B(0,1,1)=2, B(1,1,0)=3 ; R = 2
  TensorStorage B = fromCoo({2, 2, 2}, csf(3), {{{0, 0, 0}, 1.0}, {{0, 1, 1}, 2.0}, {{1, 1, 0}, 3.0}});
  TensorStorage Cd({2, 2}, denseFormat(2)), Dd({2, 2}, denseFormat(2));
  Cd.vals() = {1, 2, 3, 4};
  Dd.vals() = {5, 6, 7, 8};
  TensorStorage A = mttkrp(B, Cd, Dd);
  // A(0,:) = 1*C0*D0 + 2*C1*D1 = [5,12] + [42,64]; A(1,:) = 3*C1*D0 = [45,72]
  CHECK(A.vals() == std::vector<double>{47, 76, 45, 72});
  TensorStorage Cs = csrOf(2, 2, {0, 1, 3}, {0, 0, 1}, {1, 3, 4});
  TensorStorage Ds = csrOf(2, 2, {0, 2, 3}, {0, 1, 1}, {5, 6, 8});
  TensorStorage As = mttkrp(B, Cs, Ds);
  // present-checked: A(0,0)=1*1*5 ; A(0,1)=2*4*8 ; A(1,0)=3*3*5 ; A(1,1)=3*4*6
  CHECK(As.level(1).pos == std::vector<int64_t>{0, 2, 4});
  CHECK(As.vals() == std::vector<double>{5, 64, 45, 72});
}

static int g_init = [] {
  const char* v = std::getenv("STAM_TEST_GPU");
  g_gpu = v && std::strcmp(v, "1") == 0;
  return 0;
}();
