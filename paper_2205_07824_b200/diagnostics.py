"""Error norms and integral functionals on the device (diagnostics.py:35-89).

The reference interpolates the state to every volume quadrature point with
numpy and evaluates the exact-solution / integrand plans there — the
accuracy check of every run, ~seconds at 10M DOFs on the host.  Here the
plans are lowered to device functions (codegen.emit_plan) and one block per
element interpolates u (and q, w) with the master tabulation phi, evaluates
the plan at x_q = x0 + J xi_q and writes the element's weighted partial
sums; the host adds the per-element partials in element order (float64,
deterministic).  Same entry points, arguments and results as the reference:

  compute_l2_error(system, state, exact_u, exact_q=None) -> ErrorNorms
  compute_functional(system, state, integrand) -> float
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib, codegen
from .expr import compile_texts


@dataclass
class ErrorNorms:
    """diagnostics.py:13-18."""
    error_u: float
    error_q: float | None = None
    absolute_u: bool = False      # exact solution had zero norm
    absolute_q: bool = False


class DiagParams(C.Structure):
    _fields_ = [("ne", C.c_int32), ("nq", C.c_int32), ("nb", C.c_int32), ("mode", C.c_int32),
                ("t", C.c_double)] + [(k, C.c_void_p) for k in (
                    "x0", "J", "detj", "qp", "qw", "phi", "u", "q", "w", "out", "xq", "wdq")]


_MODULES = {}


def _source(model, nd, plan, nf, mode, curved=False):
    """mode 0: L2 partials of nf fields (state field f vs plan output f);
    mode 1: functional (plan output 0 at (x, t, u~, q~, w~))."""
    ncu, nw = model.ncu, model.nw
    nq_ = ncu * nd
    L = [codegen.DEVICE_HELPERS,
         codegen.emit_plan(plan, "plan_g", nd, model.mu_bindings()),
         "struct DiagParams { int ne, nq, nb, mode; double t; const double *x0, *J, *detj, *qp,"
         " *qw, *phi, *u, *q, *w; double* out; const double *xq, *wdq; };",
         f"#define ND {nd}\n#define NCU {ncu}\n#define NQV {nq_}\n#define NW {max(nw, 1)}\n"
         f"#define NFLD {nf}\n#define MODE {mode}\n#define CURVED {int(curved)}",
         'extern "C" __global__ void __launch_bounds__(128) diag_kernel(const DiagParams P) {',
         "  __shared__ double red[2][128];",
         "  const int e = blockIdx.x;",
         "  const double dj = P.detj[e];",
         "  double s0 = 0.0, s1 = 0.0;",
         "  for (int q = threadIdx.x; q < P.nq; q += blockDim.x) {",
         "    double x[ND];",
         "    for (int d = 0; d < ND; ++d) {",
         "#if CURVED",
         "      x[d] = P.xq[((size_t)e * P.nq + q) * ND + d];",   # per-point geometry map
         "#else",
         "      double v = P.x0[e * ND + d];",
         "      for (int r = 0; r < ND; ++r) v += P.J[(e * ND + d) * ND + r] * P.qp[q * ND + r];",
         "      x[d] = v;",
         "#endif",
         "    }",
         "    const double* ph = P.phi + (size_t)q * P.nb;",
         "    double uq[NCU], qq[NQV], wq[NW];",
         "    for (int c = 0; c < NCU; ++c) uq[c] = 0.0;",
         "    for (int c = 0; c < NQV; ++c) qq[c] = 0.0;",
         "    for (int c = 0; c < NW; ++c) wq[c] = 0.0;",
         "    for (int a = 0; a < P.nb; ++a) {",
         "      const double f = ph[a];",
         "      for (int c = 0; c < NCU; ++c) uq[c] = fma(f, P.u[((size_t)e * P.nb + a) * NCU + c], uq[c]);",
         "      if (P.q) for (int c = 0; c < NQV; ++c) qq[c] = fma(f, P.q[((size_t)e * P.nb + a) * NQV + c], qq[c]);",
         "      if (P.w) for (int c = 0; c < NW; ++c) wq[c] = fma(f, P.w[((size_t)e * P.nb + a) * NW + c], wq[c]);",
         "    }",
         "#if CURVED",
         "    const double wd = P.wdq[(size_t)e * P.nq + q];",
         "#else",
         "    const double wd = dj * P.qw[q];",
         "#endif",
         "    double g[NFLD];",
         "    plan_g(x, P.t, uq, qq, wq, nullptr, g);",
         "#if MODE == 0",
         "    for (int f = 0; f < NFLD; ++f) {",
         "      const double h = NFLD == NCU ? uq[f] : qq[f];",
         "      s0 = fma(wd, (h - g[f]) * (h - g[f]), s0);",
         "      s1 = fma(wd, g[f] * g[f], s1);",
         "    }",
         "#else",
         "    s0 = fma(wd, g[0], s0);",
         "    if (!isfinite(g[0])) s1 = __longlong_as_double(0x7ff8000000000000LL);",
         "#endif",
         "  }",
         "  red[0][threadIdx.x] = s0;",
         "  red[1][threadIdx.x] = s1;",
         "  __syncthreads();",
         "  for (int h = 64; h > 0; h >>= 1) {",
         "    if (threadIdx.x < h) {",
         "      red[0][threadIdx.x] += red[0][threadIdx.x + h];",
         "      red[1][threadIdx.x] += red[1][threadIdx.x + h];",
         "    }",
         "    __syncthreads();",
         "  }",
         "  if (threadIdx.x == 0) { P.out[2 * e] = red[0][0]; P.out[2 * e + 1] = red[1][0]; }",
         "}"]
    return "\n".join(L) + "\n"


def _module(src):
    from .nonlinear import compile_source
    if src not in _MODULES:
        lib = _lib.load()
        cubin = compile_source(src)
        h = C.c_void_p()
        _lib.check(lib.ldg_jit_load(cubin, len(cubin), C.byref(h)), "ldg_jit_load", jit=True)
        _MODULES[src] = h
    return _MODULES[src]


def _dev(system, name, arr):
    import torch
    cache = system.__dict__.setdefault("_diag_tabs", {})
    if name not in cache:
        cache[name] = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64),
                                      device=system.device)
    return cache[name]


def _as_dev(system, a):
    import torch
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=system.device, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=system.device)


def _partials(system, plan, nf, mode, t, u, q=None, w=None):
    import torch
    tab = system.tab
    m = tab.master
    curved = bool(getattr(tab, "curved", False))
    src = _source(system.model, system.nd, plan, nf, mode, curved)
    mod = _module(src)
    out = torch.empty(2 * tab.ne, dtype=torch.float64, device=system.device)
    P = DiagParams()
    P.ne, P.nq, P.nb, P.mode, P.t = tab.ne, int(m.quad_pts.shape[0]), int(m.n_nodes), mode, float(t)
    P.x0 = _dev(system, "x0", tab.x0).data_ptr()
    P.J = _dev(system, "J", tab.J).data_ptr()
    P.detj = _dev(system, "detj", tab.detj).data_ptr()
    P.qp = _dev(system, "qp", m.quad_pts).data_ptr()
    P.qw = _dev(system, "qw", m.quad_wts).data_ptr()
    P.phi = _dev(system, "phi", m.phi).data_ptr()
    if curved:                  # disc.py:91-104: x and w detJ per volume point
        P.xq = _dev(system, "xq", tab.xq_q).data_ptr()
        P.wdq = _dev(system, "wdq", tab.wdetj_q).data_ptr()
    keep = [_as_dev(system, u), _as_dev(system, q), _as_dev(system, w)]
    P.u = keep[0].data_ptr()
    P.q = None if keep[1] is None else keep[1].data_ptr()
    P.w = None if keep[2] is None else keep[2].data_ptr()
    P.out = out.data_ptr()
    lib = _lib.load()
    if tab.ne:
        _lib.check(lib.ldg_jit_launch(mod, b"diag_kernel", tab.ne, 1, 128, 0, C.byref(P),
                                      C.sizeof(P), _lib.stream_ptr()), "diag_kernel", jit=True)
    part = out.reshape(-1, 2).cpu().numpy()
    del keep
    return part


def compute_l2_error(system, state, exact_u, exact_q=None) -> ErrorNorms:
    """Relative L2 errors by quadrature over all elements (diagnostics.py:
    35-65): exact_u has ncu expressions, exact_q optional ncu*nd (row-major)
    for the mixed variable of diffusion / wave models; a zero-norm exact
    solution gives the absolute norm with a flag."""
    model = system.model
    plan = compile_texts(list(exact_u), model.symbols)
    p = _partials(system, plan, system.ncu, 0, state.t, state.u)
    num, den = float(np.sum(p[:, 0])), float(np.sum(p[:, 1]))
    abs_u = den == 0.0
    err_u = np.sqrt(num) if abs_u else np.sqrt(num / den)
    err_q, abs_q = None, False
    if exact_q is not None and system.kind in ("D", "W"):
        q = state.q if system.kind == "W" else system.compute_mixed(state.u, state.t)
        plan_q = compile_texts(list(exact_q), model.symbols)
        p = _partials(system, plan_q, system.ncu * system.nd, 0, state.t, state.u, q=q)
        num, den = float(np.sum(p[:, 0])), float(np.sum(p[:, 1]))
        abs_q = den == 0.0
        err_q = float(np.sqrt(num) if abs_q else np.sqrt(num / den))
    return ErrorNorms(error_u=float(err_u), error_q=err_q, absolute_u=abs_u, absolute_q=abs_q)


def compute_functional(system, state, integrand: str) -> float:
    """Integral of g(u~, x, t) over the domain by quadrature
    (diagnostics.py:68-89); u~ = (u, q, w) with q = compute_mixed(u) for
    kind D and the state's q for kind W."""
    model = system.model
    q = None
    if system.kind == "W" and state.q is not None:
        q = state.q
    elif system.kind == "D":
        q = system.compute_mixed(state.u, state.t)
    plan = compile_texts([integrand], model.symbols)
    p = _partials(system, plan, 1, 1, state.t, state.u, q=q, w=state.w)
    if not np.isfinite(p[:, 1]).all():
        raise ValueError("functional integrand produced non-finite values")
    return float(np.sum(p[:, 0]))
