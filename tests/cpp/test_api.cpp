// C++ API tests: the stam storage/workspace surface and the stam::spgemm /
// spadd / mttkrp entry points (GPU cases run only with STAM_TEST_GPU=1).
#define SHIM_MAIN
#include "doctest.h"

#include <cstdlib>
#include <cstring>
#include <vector>

#include <cstdio>
#include <fstream>
#include <map>
#include <string>

#include "stam/execute.h"
#include "stam/io.h"
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

static std::string tmpFile(const char* name, const char* text) {
  std::string path = std::string("/tmp/stam_io_") + name;
  std::ofstream(path) << text;
  return path;
}

TEST_CASE("io: matrix market identity, symmetric expansion, errors") {
  TensorStorage I = loadMatrixMarket(
      tmpFile("id.mtx", "%%MatrixMarket matrix coordinate real general\n% c\n2 2 2\n1 1 1\n2 2 1\n"));
  CHECK(I.format() == csr());
  CHECK(I.level(1).pos == std::vector<int64_t>{0, 1, 2});
  CHECK(I.level(1).idx == std::vector<int64_t>{0, 1});
  CHECK(I.vals() == std::vector<double>{1, 1});
  TensorStorage S = loadMatrixMarket(
      tmpFile("sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 5\n3 3 1\n"));
  CHECK(S.storedCount() == 3);  // (2,1) expanded to (1,2)
  CHECK(S.locate({0, 1}).has_value());
  TensorStorage Pt = loadMatrixMarket(
      tmpFile("pat.mtx", "%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 3\n1 3\n"));
  CHECK(Pt.vals() == std::vector<double>{2.0});  // duplicates summed (1.0 each)
  CHECK_THROWS_AS(loadMatrixMarket(tmpFile("bad.mtx", "%%MatrixMarket tensor coordinate real general\n")),
                  Error);
  CHECK_THROWS_AS(loadMatrixMarket(tmpFile("oob.mtx",
                                           "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")),
                  Error);
}

TEST_CASE("io: tns order 3, duplicates summed, 0-based rejected, round trip") {
  TensorStorage T = loadTns(tmpFile("t.tns", "# c\n1 1 1 1.5\n2 3 1 2\n1 1 1 0.5\n1 2 2 3\n"));
  CHECK(T.format() == csf(3));
  CHECK(T.storedCount() == 3);
  CHECK(T.dimensions() == std::vector<int64_t>{2, 3, 2});
  CHECK(*T.locate({0, 0, 0}) == 0);
  CHECK(T.vals()[0] == 2.0);
  CHECK_THROWS_AS(loadTns(tmpFile("z.tns", "0 1 1 1\n")), Error);
  const std::string p = "/tmp/stam_io_rt.tns";
  store(p, T);
  TensorStorage U = loadTns(p, T.dimensions());
  CHECK(U.level(1).pos == T.level(1).pos);
  CHECK(U.level(2).idx == T.level(2).idx);
  CHECK(U.vals() == T.vals());
  TensorStorage A = csrOf(3, 4, {0, 2, 2, 3}, {0, 3, 1}, {0.1, -2.5e-300, 1.0 / 3.0});
  store("/tmp/stam_io_rt.mtx", A);
  TensorStorage B = loadMatrixMarket("/tmp/stam_io_rt.mtx");
  CHECK(B.level(1).pos == A.level(1).pos);
  CHECK(B.level(1).idx == A.level(1).idx);
  CHECK(B.vals() == A.vals());  // 17 significant digits: exact
}

TEST_CASE("gpu: assemble / compute modes and unsorted output") {
  if (!g_gpu) return;
  TensorStorage A = csrOf(2, 2, {0, 2, 3}, {0, 1, 1}, {1, 2, 3});
  TensorStorage B = csrOf(2, 2, {0, 1, 3}, {0, 0, 1}, {4, 5, 6});
  KernelOptions asm_opts;
  asm_opts.mode = ExecutionMode::Assemble;
  TensorStorage idx = spgemm(A, B, asm_opts);
  CHECK(idx.level(1).pos == std::vector<int64_t>{0, 2, 4});
  CHECK(idx.vals() == std::vector<double>{0, 0, 0, 0});
  TensorStorage C = spgemmCompute(A, B, idx);
  CHECK(C.vals() == std::vector<double>{14, 12, 15, 18});
  KernelOptions cmp;
  cmp.mode = ExecutionMode::Compute;
  CHECK_THROWS_AS(spgemm(A, B, cmp), Error);
  KernelOptions uns;
  uns.sort = false;
  TensorStorage Cu = spgemm(A, B, uns);
  CHECK(!Cu.format().levelFormat(1).ordered);
  CHECK(Cu.storedCount() == 4);
  const TensorStorage* ops[] = {&A, &B};
  TensorStorage sidx = spadd(ops, asm_opts);
  TensorStorage S = spaddCompute(ops, sidx);
  CHECK(S.vals() == std::vector<double>{5, 2, 5, 9});
}

TEST_CASE("execute: CIN parse errors and unsupported plans (host)") {
  std::map<std::string, const TensorStorage*> none;
  CHECK_THROWS_AS(execute("forall(i) (A(i) = ", none), Error);
  try {
    execute("forall(i,j) A(i,j) = B(i,j) + C(i,j) + D(i,j)", none);
    FAIL("expected UnsupportedMerge");
  } catch (const Error& e) {
    CHECK(e.code() == ErrorCode::UnsupportedMerge);
  }
  try {
    execute("forall(i,k,j) A(i,j) += B(i,k)*C(k,j)", none);
    FAIL("expected UnplannableResult");
  } catch (const Error& e) {
    CHECK(e.code() == ErrorCode::UnplannableResult);
  }
  try {
    execute("forall(i) ((forall(j) A(i,j) = w0(j)) where (forall(k,j) w0(j) += B(i,k)*C(k,j)))",
            none);
    FAIL("expected MissingBinding");
  } catch (const Error& e) {
    CHECK(e.code() == ErrorCode::MissingBinding);
  }
}

TEST_CASE("gpu: execute dispatches the golden CIN plans") {
  if (!g_gpu) return;
  TensorStorage B = csrOf(2, 2, {0, 2, 3}, {0, 1, 1}, {1, 2, 3});
  TensorStorage C = csrOf(2, 2, {0, 1, 3}, {0, 0, 1}, {4, 5, 6});
  TensorStorage D = csrOf(2, 2, {0, 1, 1}, {1}, {10});
  // test_transform.cpp:141-147 printed form
  ExecuteResult g = execute(
      "forall(i) ((forall(j) A(i,j) = w0(j)) where (forall(k,j) w0(j) += B(i,k)*C(k,j)))",
      {{"B", &B}, {"C", &C}});
  CHECK(g.plan == "spgemm");
  CHECK(g.tensor == "A");
  CHECK(g.result.vals() == std::vector<double>{14, 12, 15, 18});
  // test_transform.cpp:275-284 printed form
  ExecuteResult a = execute(
      "forall(i) ((forall(j) A(i,j) = w0(j)) where ((forall(j) w0(j) = B(i,j) ; forall(j) w0(j) "
      "+= C(i,j) ; forall(j) w0(j) += D(i,j))))",
      {{"B", &B}, {"C", &C}, {"D", &D}});
  CHECK(a.plan == "spadd");
  CHECK(a.result.vals() == std::vector<double>{5, 12, 5, 9});
  ExecuteResult m = execute("forall(i,j) A(i,j) = B(i,j) + C(i,j)", {{"B", &B}, {"C", &C}});
  CHECK(m.plan == "spadd_merge");
  CHECK(m.result.vals() == std::vector<double>{5, 2, 5, 9});
  ExecuteResult rd = execute("forall(i,j) a(i) += B(i,j)*C(i,j)", {{"B", &B}, {"C", &C}});
  CHECK(rd.plan == "rowdot");
  CHECK(rd.result.vals() == std::vector<double>{4, 18});
  // MTTKRP, golden naming (test_transform.cpp:166-184): B(i,k,l), C(l,j), D(k,j)
  TensorStorage T = fromCoo({2, 2, 2}, csf(3), {{{0, 0, 0}, 1.0}, {{0, 1, 1}, 2.0}, {{1, 1, 0}, 3.0}});
  TensorStorage Cd({2, 2}, denseFormat(2)), Dd({2, 2}, denseFormat(2));
  Cd.vals() = {5, 6, 7, 8};  // C(l,j): indexed by the innermost mode
  Dd.vals() = {1, 2, 3, 4};  // D(k,j): indexed by the middle mode
  ExecuteResult md = execute(
      "forall(i,k) ((forall(j) A(i,j) += w0(j)*D(k,j)) where (forall(l,j) w0(j) += "
      "B(i,k,l)*C(l,j)))",
      {{"B", &T}, {"C", &Cd}, {"D", &Dd}});
  CHECK(md.plan == "mttkrp_dense");
  CHECK(md.result.vals() == std::vector<double>{47, 76, 45, 72});
  TensorStorage Cs = csrOf(2, 2, {0, 2, 3}, {0, 1, 1}, {5, 6, 8});
  TensorStorage Ds = csrOf(2, 2, {0, 1, 3}, {0, 0, 1}, {1, 3, 4});
  ExecuteResult ms = execute(
      "forall(i) ((forall(j) A(i,j) = w1(j)) where (forall(k) ((forall(j) w1(j) += w0(j)*D(k,j)) "
      "where (forall(l,j) w0(j) += B(i,k,l)*C(l,j)))))",
      {{"B", &T}, {"C", &Cs}, {"D", &Ds}});
  CHECK(ms.plan == "mttkrp_sparse");
  CHECK(ms.result.vals() == std::vector<double>{5, 64, 45, 72});
  TensorStorage c({2}, denseFormat(1));
  c.vals() = {2, 3};
  ExecuteResult tv = execute("forall(i,j,k) A(i,j) += B(i,j,k)*c(k)", {{"B", &T}, {"c", &c}});
  CHECK(tv.plan == "ttv");
  CHECK(tv.result.vals() == std::vector<double>{2, 6, 6});
}

static int g_init = [] {
  const char* v = std::getenv("STAM_TEST_GPU");
  g_gpu = v && std::strcmp(v, "1") == 0;
  return 0;
}();
