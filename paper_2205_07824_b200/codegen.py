"""Lower pointwise model plans to CUDA device functions.

The reference evaluates a model's flux / source / wavespeed / mass plans
(``expr.py`` ``KernelPlan``: a topologically ordered instruction list,
``expr.py:363-373``) pointwise over numpy batches with an interpreter
(``evaluate`` ``expr.py:519-545``) and a forward-mode dual evaluator for the
Jacobian-vector product (``evaluate_with_tangent`` ``expr.py:553-608``).  The
paper's Exasim generates C++/CUDA from the same symbolic model
(``PAPER.md:183``); this module does that for the B200 path: every plan
becomes one straight-line ``__device__`` function (value) and one dual
function (value + directional derivative), which ``nonlinear.py`` splices
into the kernel template ``csrc/ldg_nl.cuh`` and compiles with NVRTC.

Dual rules follow the reference exactly (``expr.py:591-651``): mul/div/pow
product and quotient rules with the log term of ``pow`` only where the
exponent's tangent is nonzero, ``d|a| = sign(a) da`` (0 at 0), and min/max
taking the left argument's tangent on ties (``<=`` / ``>=``).  Constants
(including substituted parameters mu) are emitted as exact hexadecimal
literals so the device sees bit-identical coefficients.
"""

from __future__ import annotations

import math
import struct

UNARY_CUDA = {"sin": "sin", "cos": "cos", "tan": "tan", "exp": "exp", "log": "log",
              "sqrt": "sqrt", "abs": "fabs", "tanh": "tanh"}


class CodegenError(ValueError):
    pass


def literal(v):
    """Exact C literal of a double."""
    v = float(v)
    if math.isfinite(v):
        return f"({v.hex()})" if v < 0 else v.hex()
    bits = struct.unpack("<q", struct.pack("<d", v))[0]
    return f"__longlong_as_double({bits}LL)"


def symbol_ref(name, nd, mu):
    """Device expression of a reserved symbol (model.py:48-57 spelling);
    returns (code, seed kind) with seed kind 'u'|'q'|'w'|None."""
    if name == "t":
        return "t", None
    if name[0] == "x" and name[1:].isdigit():
        return f"x[{int(name[1:]) - 1}]", None
    if name[0] == "n" and name[1:].isdigit():
        return f"n[{int(name[1:]) - 1}]", None
    if name.startswith("mu") and name[2:].isdigit():
        key = name
        if key not in mu:
            raise CodegenError(f"parameter {name} has no value")
        return literal(mu[key]), None
    if name[0] == "u" and name[1:].isdigit():
        k = int(name[1:]) - 1
        return f"u[{k}]", ("u", k)
    if name[0] == "w" and name[1:].isdigit():
        k = int(name[1:]) - 1
        return f"w[{k}]", ("w", k)
    if name[0] == "q" and "_" in name:
        i, j = name[1:].split("_")
        k = (int(i) - 1) * nd + int(j) - 1
        return f"q[{k}]", ("q", k)
    raise CodegenError(f"symbol {name!r} is not available to device plans")


def plan_symbols(plan):
    return {ins[1] for ins in plan.instructions if ins[0] == "sym"}


def uses(plan, prefix):
    """True if the plan reads any symbol of the given family ('u', 'q', 'w',
    'x', 'n', 't')."""
    out = False
    for s in plan_symbols(plan):
        if prefix == "t":
            out |= s == "t"
        elif prefix == "q":
            out |= s.startswith("q") and "_" in s
        elif prefix in ("u", "w", "x", "n"):
            out |= s[0] == prefix and s[1:].isdigit()
    return out


# helpers the emitted plans call (numpy semantics: sign(0) = 0, sign(nan) =
# nan; minimum / maximum propagate NaN)
DEVICE_HELPERS = """__device__ __forceinline__ double ldg_sign(double a) {
  return a > 0.0 ? 1.0 : (a < 0.0 ? -1.0 : (a == 0.0 ? 0.0 : a));
}
__device__ __forceinline__ double ldg_min(double a, double b) {
  return (a != a || b != b) ? a + b : (a <= b ? a : b);
}
__device__ __forceinline__ double ldg_max(double a, double b) {
  return (a != a || b != b) ? a + b : (a >= b ? a : b);
}
"""

SIG = ("const double* __restrict__ x, double t, const double* __restrict__ u, "
       "const double* __restrict__ q, const double* __restrict__ w, "
       "const double* __restrict__ n")
# helpers the emitted plans call (numpy semantics: sign(0) = 0, sign(nan) =
# nan; minimum / maximum propagate NaN)
DEVICE_HELPERS = """__device__ __forceinline__ double ldg_sign(double a) {
  return a > 0.0 ? 1.0 : (a < 0.0 ? -1.0 : (a == 0.0 ? 0.0 : a));
}
__device__ __forceinline__ double ldg_min(double a, double b) {
  return (a != a || b != b) ? a + b : (a <= b ? a : b);
}
__device__ __forceinline__ double ldg_max(double a, double b) {
  return (a != a || b != b) ? a + b : (a >= b ? a : b);
}
"""

DSIG = ("const double* __restrict__ du, const double* __restrict__ dq, "
        "const double* __restrict__ dw")


def face_symbol_ref(name, nd, mu):
    """Device expression of a face-override symbol (model.py:61-73 spelling:
    ul / ur / ql / qr over the LEFT / RIGHT traces, x, t, mu, n)."""
    for pre, arr in (("ul", "uL"), ("ur", "uR")):
        if name.startswith(pre) and name[2:].isdigit():
            k = int(name[2:]) - 1
            return f"{arr}[{k}]", (f"{arr}", k)
    for pre, arr in (("ql", "qL"), ("qr", "qR")):
        if name.startswith(pre) and "_" in name:
            i, j = name[2:].split("_")
            k = (int(i) - 1) * nd + int(j) - 1
            return f"{arr}[{k}]", (f"{arr}", k)
    if name[0] in "uqw" and not name.startswith("mu"):
        raise CodegenError(f"symbol {name!r} is not available to face override plans")
    return symbol_ref(name, nd, mu)


FSIG = ("const double* __restrict__ x, double t, const double* __restrict__ uL, "
        "const double* __restrict__ uR, const double* __restrict__ qL, "
        "const double* __restrict__ qR, const double* __restrict__ n")
FDSIG = ("const double* __restrict__ duL, const double* __restrict__ duR, "
         "const double* __restrict__ dqL, const double* __restrict__ dqR")


def emit_face_plan(plan, name, nd, mu):
    """``name(x,t,uL,uR,qL,qR,n,out)`` and its dual for a u^ / f^ override
    plan over the face symbols (disc.py:516-547)."""
    return emit_plan(plan, name, nd, mu, resolver=face_symbol_ref, sig=FSIG, dsig=FDSIG,
                     unused="  (void)x; (void)t; (void)uL; (void)uR; (void)qL; (void)qR; (void)n;",
                     dunused="  (void)duL; (void)duR; (void)dqL; (void)dqR;")


def emit_plan(plan, name, nd, mu, resolver=None, sig=None, dsig=None, unused=None,
              dunused=None):
    """CUDA source of ``name(x,t,u,q,w,n,out)`` and
    ``name_d(x,t,u,q,w,n,du,dq,dw,out,dout)`` for a plan (one output slot per
    plan output).  Unused pointer arguments may be null."""
    resolver = resolver or symbol_ref
    sig, dsig = sig or SIG, dsig or DSIG
    ins_list = plan.instructions
    val, dual = [], []          # code expressions per instruction; dual None = 0
    lines_v, lines_d = [], []
    for i, ins in enumerate(ins_list):
        tag = ins[0]
        if tag == "const":
            val.append(literal(ins[1]))
            dual.append(None)
            continue
        if tag == "sym":
            code, seed = resolver(ins[1], nd, mu)
            val.append(code)
            dual.append(None if seed is None else f"d{seed[0]}[{seed[1]}]")
            continue
        v, d = f"v{i}", f"g{i}"
        if tag == "neg":
            a, da = val[ins[1]], dual[ins[1]]
            expr_v = f"-{a}"
            expr_d = None if da is None else f"-{da}"
        elif tag in ("add", "sub"):
            a, b = val[ins[1]], val[ins[2]]
            da, db = dual[ins[1]], dual[ins[2]]
            op = "+" if tag == "add" else "-"
            expr_v = f"{a} {op} {b}"
            if da is None and db is None:
                expr_d = None
            elif db is None:
                expr_d = da
            elif da is None:
                expr_d = db if tag == "add" else f"-{db}"
            else:
                expr_d = f"{da} {op} {db}"
        elif tag == "mul":
            a, b = val[ins[1]], val[ins[2]]
            da, db = dual[ins[1]], dual[ins[2]]
            expr_v = f"{a} * {b}"
            terms = []
            if da is not None:
                terms.append(f"{da} * {b}")
            if db is not None:
                terms.append(f"{a} * {db}")
            expr_d = " + ".join(terms) if terms else None
        elif tag == "div":
            a, b = val[ins[1]], val[ins[2]]
            da, db = dual[ins[1]], dual[ins[2]]
            expr_v = f"{a} / {b}"
            if da is None and db is None:
                expr_d = None
            elif db is None:
                expr_d = f"{da} / {b}"
            elif da is None:
                expr_d = f"(-({v} * {db})) / {b}"
            else:
                expr_d = f"({da} - {v} * {db}) / {b}"
        elif tag == "pow" or (tag == "call" and ins[1] == "pow"):
            ai, bi = (ins[1], ins[2]) if tag == "pow" else ins[2]
            a, b, da, db = val[ai], val[bi], dual[ai], dual[bi]
            expr_v = f"pow({a}, {b})"
            terms = []
            if da is not None:
                terms.append(f"{b} * pow({a}, {b} - 1.0) * {da}")
            if db is not None:
                # expr.py:611-617: the log term only where db != 0
                terms.append(f"(({db}) == 0.0 ? 0.0 : {v} * log({a}) * {db})")
            expr_d = " + ".join(terms) if terms else None
        elif tag == "call":
            fn = ins[1]
            if fn in ("min", "max"):
                ai, bi = ins[2]
                a, b, da, db = val[ai], val[bi], dual[ai], dual[bi]
                expr_v = f"ldg_{fn}({a}, {b})"
                cmp = "<=" if fn == "min" else ">="
                if da is None and db is None:
                    expr_d = None
                else:
                    expr_d = f"(({a}) {cmp} ({b}) ? {da or '0.0'} : {db or '0.0'})"
            elif fn in UNARY_CUDA:
                (ai,) = ins[2]
                a, da = val[ai], dual[ai]
                expr_v = f"{UNARY_CUDA[fn]}({a})"
                if da is None:
                    expr_d = None
                elif fn == "sin":
                    expr_d = f"cos({a}) * {da}"
                elif fn == "cos":
                    expr_d = f"-sin({a}) * {da}"
                elif fn == "tan":
                    expr_d = f"(1.0 + {v} * {v}) * {da}"
                elif fn == "exp":
                    expr_d = f"{v} * {da}"
                elif fn == "log":
                    expr_d = f"{da} / {a}"
                elif fn == "sqrt":
                    expr_d = f"{da} / (2.0 * {v})"
                elif fn == "abs":
                    expr_d = f"ldg_sign({a}) * {da}"
                else:  # tanh
                    expr_d = f"(1.0 - {v} * {v}) * {da}"
            else:
                raise CodegenError(f"unknown function {fn!r}")
        else:
            raise CodegenError(f"unknown instruction {tag!r}")
        lines_v.append(f"  const double {v} = {expr_v};")
        lines_d.append(f"  const double {v} = {expr_v};")
        if expr_d is not None:
            lines_d.append(f"  const double {d} = {expr_d};")
            dual.append(d)
        else:
            dual.append(None)
        val.append(v)
    outs_v = [f"  out[{k}] = {val[r]};" for k, r in enumerate(plan.outputs)]
    outs_d = [f"  out[{k}] = {val[r]};\n  dout[{k}] = {dual[r] or '0.0'};"
              for k, r in enumerate(plan.outputs)]
    unused = unused or "  (void)x; (void)t; (void)u; (void)q; (void)w; (void)n;"
    dunused = dunused or "  (void)du; (void)dq; (void)dw;"
    src = [f"__device__ __forceinline__ void {name}({sig}, double* __restrict__ out) {{",
           unused, *lines_v, *outs_v, "}",
           f"__device__ __forceinline__ void {name}_d({sig}, {dsig},",
           "    double* __restrict__ out, double* __restrict__ dout) {",
           unused, dunused, *lines_d, *outs_d, "}"]
    return "\n".join(src) + "\n"
