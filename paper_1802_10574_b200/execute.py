"""CIN-driven dispatch, mirroring ``include/stam/execute.h``: SPEC's
``execute(plan, inputs, mode)`` for the concrete index
notation ``schedule()`` prints.  The statement is parsed (forall / where /
``;`` sequences / ``=`` and ``+=`` assignments over products or sums of
accesses) and matched structurally — any tensor and index-variable names —
against the plans the GPU kernels implement (SpGEMM, k-operand SpAdd, MTTKRP
with dense or sparse factors, TTV, row-dot, two-way merge), then run through a
``Context``.  Errors raise ``StamError`` with the reference codes (``Parse``,
``UnsupportedMerge``, ``UnplannableResult``, ``MissingBinding``)."""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Any, Dict, List, Optional

from ._native import StamError
from .storage import Dense

_PARSE, _UNSUPPORTED, _UNPLANNABLE, _MISSING = 1, 15, 16, 17


@dataclass
class Access:
    name: str
    idx: List[str]


@dataclass
class Stmt:
    kind: str  # forall | where | seq | assign
    vars: List[str] = field(default_factory=list)
    kids: List["Stmt"] = field(default_factory=list)
    lhs: Optional[Access] = None
    accumulate: bool = False
    op: str = ""
    terms: List[Access] = field(default_factory=list)


_TOK = re.compile(r"\s*(forall\b|where\b|\+=|[A-Za-z_][A-Za-z0-9_]*|[(),;=*+])")


class _Parser:
    def __init__(self, text: str):
        self.toks, pos = [], 0
        while pos < len(text):
            m = _TOK.match(text, pos)
            if not m:
                if text[pos:].strip() == "":
                    break
                raise StamError(_PARSE, f"CIN, column {pos + 1}: unexpected character")
            self.toks.append(m.group(1))
            pos = m.end()
        self.i = 0

    def peek(self):
        return self.toks[self.i] if self.i < len(self.toks) else None

    def take(self, tok=None):
        t = self.peek()
        if t is None or (tok is not None and t != tok):
            raise StamError(_PARSE, f"CIN: expected {tok or 'a token'}, found {t!r}")
        self.i += 1
        return t

    def names(self):
        self.take("(")
        out = []
        if self.peek() != ")":
            out.append(self.ident())
            while self.peek() == ",":
                self.take(",")
                out.append(self.ident())
        self.take(")")
        return out

    def ident(self):
        t = self.take()
        if not re.match(r"[A-Za-z_]", t) or t in ("forall", "where"):
            raise StamError(_PARSE, f"CIN: expected a name, found {t!r}")
        return t

    def access(self):
        return Access(self.ident(), self.names())

    def stmt(self) -> Stmt:
        t = self.peek()
        if t == "forall":
            self.take()
            vs = self.names()
            return Stmt("forall", vars=vs, kids=[self.stmt()])
        if t == "(":
            self.take()
            first = self.stmt()
            if self.peek() == "where":
                self.take()
                s = Stmt("where", kids=[first, self.stmt()])
                self.take(")")
                return s
            if self.peek() == ";":
                kids = [first]
                while self.peek() == ";":
                    self.take()
                    kids.append(self.stmt())
                self.take(")")
                return Stmt("seq", kids=kids)
            self.take(")")
            return first
        a = Stmt("assign", lhs=self.access())
        if self.peek() == "+=":
            self.take()
            a.accumulate = True
        else:
            self.take("=")
        a.terms.append(self.access())
        while self.peek() in ("*", "+"):
            op = self.take()
            if a.op and a.op != op:
                raise StamError(_PARSE, "CIN: mixed '*' and '+' on one right-hand side")
            a.op = op
            a.terms.append(self.access())
        return a


def parse(cin: str) -> Stmt:
    p = _Parser(cin)
    s = p.stmt()
    if p.peek() is not None:
        raise StamError(_PARSE, f"CIN: unexpected {p.peek()!r}")
    return s


def _loop_assign(s: Stmt, n: int) -> Optional[Stmt]:
    if s.kind != "forall" or len(s.vars) != n or s.kids[0].kind != "assign":
        return None
    return s.kids[0]


def _product_with(a: Stmt, w: str, widx) -> Optional[Access]:
    if a.op != "*" or len(a.terms) != 2:
        return None
    for t in (0, 1):
        if a.terms[t].name == w and a.terms[t].idx == widx:
            return a.terms[1 - t]
    return None


@dataclass
class Plan:
    plan: str
    tensor: str
    args: tuple


def match(s: Stmt) -> Plan:
    """The GPU plan of a parsed statement (names of its input tensors)."""
    a = _loop_assign(s, 3)
    if a is not None:
        v = s.vars
        if (a.accumulate and a.op == "*" and len(a.terms) == 2 and a.lhs.idx == v[:2]
                and a.terms[0].idx == v and a.terms[1].idx == [v[2]]):
            return Plan("ttv", a.lhs.name, (a.terms[0].name, a.terms[1].name))
        if a.accumulate and a.op == "*" and len(a.terms) == 2 and len(a.lhs.idx) == 2:
            raise StamError(_UNPLANNABLE, "execute: a sparse result written by scattered inserts "
                                          "has no plan; apply a workspace")
    a = _loop_assign(s, 2)
    if a is not None:
        v = s.vars
        if (a.accumulate and a.op == "*" and len(a.terms) == 2 and a.lhs.idx == [v[0]]
                and a.terms[0].idx == v and a.terms[1].idx == v):
            return Plan("rowdot", a.lhs.name, (a.terms[0].name, a.terms[1].name))
        if not a.accumulate and a.op == "+" and a.lhs.idx == v:
            if any(t.idx != v for t in a.terms):
                raise StamError(_UNSUPPORTED, "execute: operand indices differ")
            if len(a.terms) > 2:
                raise StamError(_UNSUPPORTED, "execute: a merge of 3 or more sparse operands "
                                              "needs a workspace")
            return Plan("spadd_merge", a.lhs.name, ([t.name for t in a.terms],))
    if s.kind == "forall" and s.kids[0].kind == "where":
        cons, prod = s.kids[0].kids
        if len(s.vars) == 1:
            i = s.vars[0]
            c = _loop_assign(cons, 1)
            if (c is not None and not c.accumulate and not c.op and len(c.lhs.idx) == 2
                    and c.lhs.idx[0] == i and len(c.terms) == 1
                    and c.terms[0].idx == [c.lhs.idx[1]] and cons.vars == [c.lhs.idx[1]]):
                j, w = c.lhs.idx[1], c.terms[0].name
                p = _loop_assign(prod, 2)
                if p is not None:
                    k = prod.vars[0]
                    if (prod.vars[1] == j and p.accumulate and p.op == "*" and len(p.terms) == 2
                            and p.lhs.name == w and p.lhs.idx == [j]
                            and p.terms[0].idx == [i, k] and p.terms[1].idx == [k, j]):
                        return Plan("spgemm", c.lhs.name, (p.terms[0].name, p.terms[1].name))
                if prod.kind == "seq" and len(prod.kids) >= 2:
                    names = []
                    for t, ks in enumerate(prod.kids):
                        q = _loop_assign(ks, 1)
                        if not (q is not None and ks.vars == [j] and q.lhs.name == w
                                and q.lhs.idx == [j] and not q.op and len(q.terms) == 1
                                and q.terms[0].idx == [i, j] and q.accumulate == (t > 0)):
                            names = None
                            break
                        names.append(q.terms[0].name)
                    if names:
                        return Plan("spadd", c.lhs.name, (names,))
                if prod.kind == "forall" and len(prod.vars) == 1 and prod.kids[0].kind == "where":
                    k = prod.vars[0]
                    ic, ip = prod.kids[0].kids
                    c2, p2 = _loop_assign(ic, 1), _loop_assign(ip, 2)
                    if (c2 is not None and p2 is not None and ic.vars == [j] and c2.accumulate
                            and c2.lhs.name == w and c2.lhs.idx == [j] and ip.vars[1] == j
                            and p2.accumulate and p2.op == "*" and len(p2.terms) == 2
                            and p2.lhs.idx == [j]):
                        l = ip.vars[0]
                        dk = _product_with(c2, p2.lhs.name, [j])
                        if (dk is not None and dk.idx == [k, j] and p2.terms[0].idx == [i, k, l]
                                and p2.terms[1].idx == [l, j]):
                            return Plan("mttkrp_sparse", c.lhs.name,
                                        (p2.terms[0].name, dk.name, p2.terms[1].name))
        if len(s.vars) == 2:
            i, k = s.vars
            c, p = _loop_assign(cons, 1), _loop_assign(prod, 2)
            if (c is not None and p is not None and c.accumulate and p.accumulate
                    and p.op == "*" and len(p.terms) == 2):
                j, l = cons.vars[0], prod.vars[0]
                dk = _product_with(c, p.lhs.name, [j])
                if (prod.vars[1] == j and c.lhs.idx == [i, j] and p.lhs.idx == [j]
                        and dk is not None and dk.idx == [k, j] and p.terms[0].idx == [i, k, l]
                        and p.terms[1].idx == [l, j]):
                    return Plan("mttkrp_dense", c.lhs.name,
                                (p.terms[0].name, dk.name, p.terms[1].name))
    raise StamError(_UNSUPPORTED, "execute: the statement matches none of the GPU plans")


def execute(cin: str, inputs: Dict[str, Any], ctx=None, **kw):
    """Runs `cin` with its inputs bound by name; returns (tensor name, plan, result)."""
    from .kernels import default_context

    ctx = ctx or default_context()
    pl = match(parse(cin))

    def get(n):
        if n not in inputs:
            raise StamError(_MISSING, f"execute: no tensor bound to '{n}'")
        return inputs[n]

    if pl.plan == "spgemm":
        out = ctx.spgemm(get(pl.args[0]), get(pl.args[1]), **kw)
    elif pl.plan == "spadd":
        out = ctx.spadd([get(n) for n in pl.args[0]], **kw)
    elif pl.plan == "spadd_merge":
        out = ctx.spadd_merge([get(n) for n in pl.args[0]], **kw)
    elif pl.plan == "rowdot":
        out = ctx.rowdot(get(pl.args[0]), get(pl.args[1]), **kw)
    elif pl.plan == "ttv":
        c = get(pl.args[1])
        out = ctx.ttv(get(pl.args[0]), c.vals.reshape(-1) if isinstance(c, Dense) else c, **kw)
    else:  # mttkrp: B(i,k,l); the middle-mode factor is the API's C
        out = ctx.mttkrp(get(pl.args[0]), get(pl.args[1]), get(pl.args[2]), **kw)
    return pl.tensor, pl.plan, out
