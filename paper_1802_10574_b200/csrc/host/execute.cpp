// execute.cpp — CIN-driven dispatch (stam/execute.h): a parser for the
// concrete index notation schedule() prints (forall / where / ';' sequences /
// '=' and '+=' assignments over products or sums of accesses) and structural
// matchers for the plans the GPU kernels implement.
#include "stam/execute.h"

#include <cctype>
#include <memory>
#include <vector>

#include "stam/error.h"

namespace stam {
namespace {

// ---------------------------------------------------------------- AST
struct Access {
  std::string name;
  std::vector<std::string> idx;
};

struct Stmt {
  enum Kind { Forall, Where, Seq, Assign } kind = Assign;
  std::vector<std::string> vars;  // Forall
  std::vector<Stmt> kids;         // Forall: body; Where: consumer, producer; Seq: items
  Access lhs;                     // Assign
  bool accumulate = false;        // '+='
  char op = 0;                    // '*' product, '+' sum, 0 single access
  std::vector<Access> terms;      // Assign right-hand side
};

// ---------------------------------------------------------------- parser
class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}

  Stmt parse() {
    Stmt st = stmt();
    skip();
    if (p_ != s_.size()) error("unexpected '" + s_.substr(p_, 12) + "'");
    return st;
  }

 private:
  [[noreturn]] void error(const std::string& what) {
    fail(ErrorCode::Parse, "CIN, column " + std::to_string(p_ + 1) + ": " + what);
  }
  void skip() {
    while (p_ < s_.size() && std::isspace((unsigned char)s_[p_])) p_++;
  }
  bool peek(const char* tok) {
    skip();
    return s_.compare(p_, std::char_traits<char>::length(tok), tok) == 0;
  }
  bool accept(const char* tok) {
    if (!peek(tok)) return false;
    p_ += std::char_traits<char>::length(tok);
    return true;
  }
  void expect(const char* tok) {
    if (!accept(tok)) error(std::string("expected '") + tok + "'");
  }
  bool keyword(const char* kw) {
    skip();
    const size_t n = std::char_traits<char>::length(kw);
    if (s_.compare(p_, n, kw) != 0) return false;
    if (p_ + n < s_.size() && (std::isalnum((unsigned char)s_[p_ + n]) || s_[p_ + n] == '_'))
      return false;
    p_ += n;
    return true;
  }
  std::string ident() {
    skip();
    const size_t b = p_;
    while (p_ < s_.size() && (std::isalnum((unsigned char)s_[p_]) || s_[p_] == '_')) p_++;
    if (b == p_ || std::isdigit((unsigned char)s_[b])) error("expected a name");
    return s_.substr(b, p_ - b);
  }
  std::vector<std::string> names() {
    std::vector<std::string> v;
    expect("(");
    if (accept(")")) return v;
    v.push_back(ident());
    while (accept(",")) v.push_back(ident());
    expect(")");
    return v;
  }
  Access access() {
    Access a;
    a.name = ident();
    a.idx = names();
    return a;
  }
  Stmt stmt() {
    if (keyword("forall")) {
      Stmt f;
      f.kind = Stmt::Forall;
      f.vars = names();
      if (f.vars.empty()) error("forall without index variables");
      f.kids.push_back(stmt());
      return f;
    }
    if (accept("(")) {
      Stmt first = stmt();
      if (keyword("where")) {
        Stmt w;
        w.kind = Stmt::Where;
        w.kids.push_back(std::move(first));
        w.kids.push_back(stmt());
        expect(")");
        return w;
      }
      if (peek(";")) {
        Stmt q;
        q.kind = Stmt::Seq;
        q.kids.push_back(std::move(first));
        while (accept(";")) q.kids.push_back(stmt());
        expect(")");
        return q;
      }
      expect(")");
      return first;
    }
    Stmt a;
    a.kind = Stmt::Assign;
    a.lhs = access();
    if (accept("+=")) {
      a.accumulate = true;
    } else {
      expect("=");
    }
    a.terms.push_back(access());
    while (peek("*") || peek("+")) {
      const char op = s_[p_];
      if (a.op && a.op != op) error("mixed '*' and '+' on one right-hand side");
      a.op = op;
      p_++;
      a.terms.push_back(access());
    }
    return a;
  }

  const std::string& s_;
  size_t p_ = 0;
};

// ---------------------------------------------------------------- matching
using Names = std::vector<std::string>;

bool is(const Stmt& s, Stmt::Kind k) { return s.kind == k; }
bool forall(const Stmt& s, const Names& vars) { return s.kind == Stmt::Forall && s.vars == vars; }
bool acc(const Access& a, const Names& idx) { return a.idx == idx; }

// Forall([v...]) whose single body is an assignment: returns it or nullptr.
const Stmt* loop_assign(const Stmt& s, size_t nvars) {
  if (s.kind != Stmt::Forall || s.vars.size() != nvars) return nullptr;
  const Stmt& b = s.kids[0];
  return b.kind == Stmt::Assign ? &b : nullptr;
}

// product a*b with one access named `w` over `widx`: returns the other one
const Access* product_with(const Stmt& a, const std::string& w, const Names& widx) {
  if (a.op != '*' || a.terms.size() != 2) return nullptr;
  for (int t = 0; t < 2; t++)
    if (a.terms[(size_t)t].name == w && acc(a.terms[(size_t)t], widx)) return &a.terms[(size_t)(1 - t)];
  return nullptr;
}

const TensorStorage& bound(const std::map<std::string, const TensorStorage*>& in,
                           const std::string& name) {
  auto it = in.find(name);
  if (it == in.end() || !it->second)
    fail(ErrorCode::MissingBinding, "execute: no tensor bound to '" + name + "'");
  return *it->second;
}

}  // namespace

ExecuteResult execute(const std::string& cin,
                      const std::map<std::string, const TensorStorage*>& in,
                      const KernelOptions& o) {
  const Stmt S = Parser(cin).parse();
  ExecuteResult r;
  // ---- single loop nests without workspaces
  if (const Stmt* a = loop_assign(S, 3)) {
    // TTV: forall(i,j,k) A(i,j) += B(i,j,k)*c(k)
    const Names& v = S.vars;
    if (a->accumulate && a->op == '*' && a->terms.size() == 2 && acc(a->lhs, {v[0], v[1]}) &&
        acc(a->terms[0], {v[0], v[1], v[2]}) && acc(a->terms[1], {v[2]})) {
      r.plan = "ttv";
      r.tensor = a->lhs.name;
      r.result = ttv(bound(in, a->terms[0].name), bound(in, a->terms[1].name), o, &r.stats);
      return r;
    }
    if (a->accumulate && a->op == '*' && a->terms.size() == 2 && a->lhs.idx.size() == 2)
      fail(ErrorCode::UnplannableResult,
           "execute: a sparse result written by scattered inserts has no plan; apply a "
           "workspace (e.g. workspace(B(i,k)*C(k,j), {j}, dense))");
  }
  if (const Stmt* a = loop_assign(S, 2)) {
    const Names& v = S.vars;
    // row-dot: forall(i,j) a(i) += B(i,j)*C(i,j)
    if (a->accumulate && a->op == '*' && a->terms.size() == 2 && acc(a->lhs, {v[0]}) &&
        acc(a->terms[0], v) && acc(a->terms[1], v)) {
      r.plan = "rowdot";
      r.tensor = a->lhs.name;
      r.result = rowdot(bound(in, a->terms[0].name), bound(in, a->terms[1].name), o, &r.stats);
      return r;
    }
    // two-way union: forall(i,j) A(i,j) = B(i,j) + C(i,j)
    if (!a->accumulate && a->op == '+' && acc(a->lhs, v)) {
      for (const Access& t : a->terms)
        if (!acc(t, v)) fail(ErrorCode::UnsupportedMerge, "execute: operand indices differ");
      if (a->terms.size() > 2)
        fail(ErrorCode::UnsupportedMerge,
             "execute: a merge of 3 or more sparse operands needs a workspace (apply "
             "workspace(...) and workspace_reuse(...), PAPER §6.1-case-spadd)");
      std::vector<const TensorStorage*> ops{&bound(in, a->terms[0].name), &bound(in, a->terms[1].name)};
      r.plan = "spadd_merge";
      r.tensor = a->lhs.name;
      r.result = spaddMerge(ops, o, &r.stats);
      return r;
    }
  }
  // ---- workspace plans: forall(i) ((consumer) where (producer))
  if (S.kind == Stmt::Forall && S.kids[0].kind == Stmt::Where) {
    const Stmt& W = S.kids[0];
    const Stmt& cons = W.kids[0];
    const Stmt& prod = W.kids[1];
    if (S.vars.size() == 1) {
      const std::string i = S.vars[0];
      const Stmt* c = loop_assign(cons, 1);
      if (c && !c->accumulate && c->op == 0 && c->lhs.idx.size() == 2 && c->lhs.idx[0] == i &&
          c->terms.size() == 1 && c->terms[0].idx.size() == 1 &&
          c->terms[0].idx[0] == c->lhs.idx[1] && cons.vars[0] == c->lhs.idx[1]) {
        const std::string j = c->lhs.idx[1], w = c->terms[0].name;
        // SpGEMM: forall(k,j) w(j) += A(i,k)*B(k,j)
        if (const Stmt* p = loop_assign(prod, 2)) {
          const std::string k = prod.vars[0];
          if (prod.vars[1] == j && p->accumulate && p->op == '*' && p->terms.size() == 2 &&
              p->lhs.name == w && acc(p->lhs, {j}) && acc(p->terms[0], {i, k}) &&
              acc(p->terms[1], {k, j})) {
            r.plan = "spgemm";
            r.tensor = c->lhs.name;
            r.result = spgemm(bound(in, p->terms[0].name), bound(in, p->terms[1].name), o, &r.stats);
            return r;
          }
        }
        // SpAdd: (forall(j) w(j) = X1(i,j) ; forall(j) w(j) += X2(i,j) ; ...)
        if (prod.kind == Stmt::Seq && prod.kids.size() >= 2) {
          std::vector<const TensorStorage*> ops;
          bool ok = true;
          for (size_t t = 0; t < prod.kids.size() && ok; t++) {
            const Stmt* s = loop_assign(prod.kids[t], 1);
            ok = s && prod.kids[t].vars[0] == j && s->lhs.name == w && acc(s->lhs, {j}) &&
                 s->op == 0 && s->terms.size() == 1 && acc(s->terms[0], {i, j}) &&
                 s->accumulate == (t > 0);
            if (ok) ops.push_back(&bound(in, s->terms[0].name));
          }
          if (ok) {
            r.plan = "spadd";
            r.tensor = c->lhs.name;
            r.result = spadd(ops, o, &r.stats);
            return r;
          }
        }
        // MTTKRP, sparse result: forall(k) ((forall(j) w1(j) += w0(j)*D(k,j))
        //                                   where (forall(l,j) w0(j) += B(i,k,l)*C(l,j)))
        if (prod.kind == Stmt::Forall && prod.vars.size() == 1 && prod.kids[0].kind == Stmt::Where) {
          const std::string k = prod.vars[0];
          const Stmt& inner = prod.kids[0];
          const Stmt* c2 = loop_assign(inner.kids[0], 1);
          const Stmt* p2 = loop_assign(inner.kids[1], 2);
          if (c2 && p2 && inner.kids[0].vars[0] == j && c2->accumulate && c2->lhs.name == w &&
              acc(c2->lhs, {j}) && inner.kids[1].vars[1] == j && p2->accumulate &&
              p2->op == '*' && p2->terms.size() == 2 && acc(p2->lhs, {j})) {
            const std::string l = inner.kids[1].vars[0];
            const Access* Dk = product_with(*c2, p2->lhs.name, {j});
            if (Dk && acc(*Dk, {k, j}) && acc(p2->terms[0], {i, k, l}) && acc(p2->terms[1], {l, j})) {
              r.plan = "mttkrp_sparse";
              r.tensor = c->lhs.name;
              // B(i,k,l): the factor indexed by the middle mode is the API's C
              r.result = mttkrp(bound(in, p2->terms[0].name), bound(in, Dk->name),
                                bound(in, p2->terms[1].name), o, &r.stats);
              return r;
            }
          }
        }
      }
    }
    // MTTKRP, dense result: forall(i,k) ((forall(j) A(i,j) += w(j)*D(k,j))
    //                                    where (forall(l,j) w(j) += B(i,k,l)*C(l,j)))
    if (S.vars.size() == 2) {
      const std::string i = S.vars[0], k = S.vars[1];
      const Stmt* c = loop_assign(cons, 1);
      const Stmt* p = loop_assign(prod, 2);
      if (c && p && c->accumulate && p->accumulate && p->op == '*' && p->terms.size() == 2) {
        const std::string j = cons.vars[0], l = prod.vars[0];
        const Access* Dk = product_with(*c, p->lhs.name, {j});
        if (prod.vars[1] == j && acc(c->lhs, {i, j}) && acc(p->lhs, {j}) && Dk &&
            acc(*Dk, {k, j}) && acc(p->terms[0], {i, k, l}) && acc(p->terms[1], {l, j})) {
          r.plan = "mttkrp_dense";
          r.tensor = c->lhs.name;
          r.result = mttkrp(bound(in, p->terms[0].name), bound(in, Dk->name),
                            bound(in, p->terms[1].name), o, &r.stats);
          return r;
        }
      }
    }
  }
  fail(ErrorCode::UnsupportedMerge,
       "execute: the statement matches none of the GPU plans (SpGEMM, SpAdd, MTTKRP dense/"
       "sparse, TTV, row-dot, two-way merge): " + cin);
}

}  // namespace stam
