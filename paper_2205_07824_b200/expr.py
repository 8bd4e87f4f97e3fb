"""Pointwise model expressions: parse, compile to flat plans, evaluate.

Host-side setup.  Restates the reference's expression language and plan
format (``ldgkit/expr.py``): the grammar at ``expr.py:10-20``, constant
folding + integer-power strength reduction + CSE at ``expr.py:386-486``, and
the batch evaluator at ``expr.py:519-545``.  Plans produced here are
``Plan(instructions, outputs, symbols)`` with the reference's instruction
tuples, so a reference ``KernelPlan`` and a ``Plan`` are interchangeable
inputs to :mod:`.plans` (which lowers them to device coefficient tables).

The evaluator here is used only for data that do not depend on the state
(Dirichlet/Neumann data, sources that depend on x and t, initial data);
state-dependent pointwise work runs inside the CUDA kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

UNARY = ("sin", "cos", "tan", "exp", "log", "sqrt", "abs", "tanh")
BINARY = ("min", "max", "pow")
ARITH = ("add", "sub", "mul", "div", "pow")


class ExprError(ValueError):
    pass


class ExprSyntaxError(ExprError):
    def __init__(self, message, position):
        super().__init__(f"{message} (at offset {position})")
        self.position = position


class UnknownSymbolError(ExprSyntaxError):
    pass


class EvalError(ExprError):
    pass


@dataclass
class Plan:
    instructions: tuple
    outputs: tuple
    symbols: tuple

    @property
    def n_outputs(self):
        return len(self.outputs)

    def used_symbols(self):
        return {ins[1] for ins in self.instructions if ins[0] == "sym"}


# ---------------------------------------------------------------------------
# parsing to hash-consed DAG nodes
# ---------------------------------------------------------------------------


class _Nodes:
    def __init__(self):
        self.nodes, self.index = [], {}

    def add(self, node):
        i = self.index.get(node)
        if i is None:
            i = self.index[node] = len(self.nodes)
            self.nodes.append(node)
        return i


def _lex(text):
    """Token list [(kind, text, pos)] with a trailing ('end', '', len)."""
    out, i, n = [], 0, len(text)
    while True:
        while i < n and text[i] in " \t\r\n":
            i += 1
        if i >= n:
            out.append(("end", "", i))
            return out
        c = text[i]
        if c in "+-*/^(),=;":
            out.append(("op", c, i))
            i += 1
        elif c.isdigit() or c == ".":
            j, seen_e = i, False
            while j < n:
                ch = text[j]
                if ch.isdigit() or ch == ".":
                    j += 1
                elif ch in "eE" and not seen_e and j + 1 < n and (
                        text[j + 1].isdigit() or text[j + 1] in "+-"):
                    seen_e = True
                    j += 2 if text[j + 1] in "+-" else 1
                else:
                    break
            out.append(("num", text[i:j], i))
            i = j
        elif c.isalpha() or c == "_":
            j = i
            while j < n and (text[j].isalnum() or text[j] == "_"):
                j += 1
            out.append(("name", text[i:j], i))
            i = j
        else:
            raise ExprSyntaxError(f"unexpected character {c!r}", i)


class _Parser:
    """sum := term (+|- term)*; term := unary (*|/ unary)*;
    unary := - unary | power; power := primary [^ unary]."""

    def __init__(self, text, symbols, store, local=None):
        self.t = _lex(text)
        self.k = 0
        self.syms = set(symbols)
        self.s = store
        self.local = local or {}

    def peek(self):
        return self.t[self.k]

    def take(self):
        tok = self.t[self.k]
        if tok[0] != "end":
            self.k += 1
        return tok

    def run(self):
        root = self.sum()
        kind, val, pos = self.peek()
        if kind != "end":
            raise ExprSyntaxError(f"unexpected trailing input {val!r}", pos)
        return root

    def sum(self):
        a = self.term()
        while self.peek()[0] == "op" and self.peek()[1] in "+-":
            op = self.take()[1]
            a = self.s.add(("add" if op == "+" else "sub", a, self.term()))
        return a

    def term(self):
        a = self.unary()
        while self.peek()[0] == "op" and self.peek()[1] in "*/":
            op = self.take()[1]
            a = self.s.add(("mul" if op == "*" else "div", a, self.unary()))
        return a

    def unary(self):
        if self.peek()[:2] == ("op", "-"):
            self.take()
            return self.s.add(("neg", self.unary()))
        base = self.primary()
        if self.peek()[:2] == ("op", "^"):
            self.take()
            return self.s.add(("pow", base, self.unary()))
        return base

    def primary(self):
        kind, val, pos = self.take()
        if kind == "num":
            try:
                return self.s.add(("const", float(val)))
            except ValueError:
                raise ExprSyntaxError(f"bad numeric literal {val!r}", pos) from None
        if (kind, val) == ("op", "("):
            inner = self.sum()
            k2, v2, p2 = self.take()
            if (k2, v2) != ("op", ")"):
                raise ExprSyntaxError("expected ')'", p2)
            return inner
        if kind == "name":
            if self.peek()[:2] == ("op", "("):
                return self.call(val, pos)
            if val == "pi":
                return self.s.add(("const", math.pi))
            if val in self.local:
                return self.local[val]
            if val not in self.syms:
                raise UnknownSymbolError(f"unknown symbol '{val}'", pos)
            return self.s.add(("sym", val))
        if kind == "end":
            raise ExprSyntaxError("unexpected end of input", pos)
        raise ExprSyntaxError(f"unexpected token {val!r}", pos)

    def call(self, fn, pos):
        if fn not in UNARY and fn not in BINARY:
            raise ExprSyntaxError(f"unknown function '{fn}'", pos)
        self.take()
        args = [self.sum()]
        while True:
            kind, val, p = self.take()
            if (kind, val) == ("op", ")"):
                break
            if (kind, val) == ("op", ","):
                args.append(self.sum())
            elif kind == "end":
                raise ExprSyntaxError("unexpected end of input in call", p)
            else:
                raise ExprSyntaxError(f"expected ',' or ')', got {val!r}", p)
        want = 1 if fn in UNARY else 2
        if len(args) != want:
            raise ExprSyntaxError(f"'{fn}' takes {want} argument(s), got "
                                  f"{len(args)}", pos)
        return self.s.add(("call", fn, tuple(args)))


@dataclass
class Graph:
    nodes: list
    roots: list
    symbols: tuple

    def used_symbols(self):
        return {n[1] for n in self.nodes if n[0] == "sym"}


def parse_expressions(texts, symbols):
    store = _Nodes()
    roots = []
    for t in texts:
        if not t or not str(t).strip():
            raise ExprSyntaxError("empty expression", 0)
        roots.append(_Parser(str(t), symbols, store).run())
    return Graph(store.nodes, roots, tuple(symbols))


def parse_expression(text, symbols):
    return parse_expressions([text], symbols)


# ---------------------------------------------------------------------------
# compile: fold, reduce small integer powers, deduplicate
# ---------------------------------------------------------------------------


def _fn(fn, args):
    if fn == "abs":
        return np.abs(args[0])
    if fn == "min":
        return np.minimum(args[0], args[1])
    if fn == "max":
        return np.maximum(args[0], args[1])
    if fn == "pow":
        return args[0] ** args[1]
    return getattr(np, fn)(args[0])


def _binop(op, a, b):
    if op == "add":
        return a + b
    if op == "sub":
        return a - b
    if op == "mul":
        return a * b
    if op == "div":
        return a / b
    return a ** b


def compile_plan(graphs):
    """Graph(s) -> Plan with the reference's folding and CSE rules
    (expr.py:404-486)."""
    if isinstance(graphs, Graph):
        graphs = [graphs]
    symbols = graphs[0].symbols
    ins, index = [], {}

    def emit(t):
        i = index.get(t)
        if i is None:
            i = index[t] = len(ins)
            ins.append(t)
        return i

    def cval(i):
        return ins[i][1] if ins[i][0] == "const" else None

    def power(b, e):
        bv, ev = cval(b), cval(e)
        if bv is not None and ev is not None:
            with np.errstate(all="ignore"):
                return emit(("const", float(bv ** ev)))
        if ev is not None and ev == int(ev) and 0 <= int(ev) <= 4:
            n = int(ev)
            if n == 0:
                return emit(("const", 1.0))
            if n == 1:
                return b
            sq = emit(("mul", b, b))
            if n == 2:
                return sq
            return emit(("mul", sq, b)) if n == 3 else emit(("mul", sq, sq))
        return emit(("pow", b, e))

    outputs = []
    for g in graphs:
        memo = {}

        def lower(nid):
            if nid in memo:
                return memo[nid]
            nd = g.nodes[nid]
            tag = nd[0]
            if tag == "const":
                r = emit(("const", float(nd[1])))
            elif tag == "sym":
                r = emit(("sym", nd[1]))
            elif tag == "neg":
                c = lower(nd[1])
                v = cval(c)
                r = emit(("const", -v)) if v is not None else emit(("neg", c))
            elif tag == "call":
                args = tuple(lower(a) for a in nd[2])
                vals = [cval(a) for a in args]
                if nd[1] == "pow":
                    r = power(args[0], args[1])
                elif all(v is not None for v in vals):
                    with np.errstate(all="ignore"):
                        r = emit(("const", float(_fn(nd[1], vals))))
                else:
                    r = emit(("call", nd[1], args))
            else:
                a, b = lower(nd[1]), lower(nd[2])
                if tag == "pow":
                    r = power(a, b)
                else:
                    av, bv = cval(a), cval(b)
                    if av is not None and bv is not None:
                        with np.errstate(all="ignore"):
                            r = emit(("const", float(_binop(tag, av, bv))))
                    else:
                        r = emit((tag, a, b))
            memo[nid] = r
            return r

        for root in g.roots:
            outputs.append(lower(root))
    return Plan(tuple(ins), tuple(outputs), symbols)


def compile_texts(texts, symbols):
    return compile_plan(parse_expressions(list(texts), symbols))


# ---------------------------------------------------------------------------
# host evaluation (state-independent data only)
# ---------------------------------------------------------------------------


def evaluate(plan, bindings):
    """(n_outputs, B) values of a plan over equal-length bindings
    (expr.py:494-545)."""
    used = plan.used_symbols()
    missing = used - set(bindings)
    if missing:
        raise EvalError(f"missing bindings: {sorted(missing)}")
    arrs, batch = {}, None
    for s in used:
        a = np.asarray(bindings[s], dtype=float)
        if a.ndim > 1:
            a = a.ravel()
        if a.ndim == 1:
            if batch is None:
                batch = a.shape[0]
            elif a.shape[0] != batch:
                raise EvalError(f"binding '{s}' has length {a.shape[0]}, "
                                f"expected {batch}")
        arrs[s] = a
    batch = 1 if batch is None else batch
    if batch < 1:
        raise EvalError("empty batch")
    vals = []
    with np.errstate(all="ignore"):
        for t in plan.instructions:
            tag = t[0]
            if tag == "const":
                v = np.full(1, t[1])
            elif tag == "sym":
                v = arrs[t[1]]
            elif tag == "neg":
                v = -vals[t[1]]
            elif tag == "call":
                v = _fn(t[1], [vals[a] for a in t[2]])
            else:
                v = _binop(tag, vals[t[1]], vals[t[2]])
            vals.append(v)
    out = np.empty((len(plan.outputs), batch))
    for k, r in enumerate(plan.outputs):
        out[k] = vals[r]
    return out
