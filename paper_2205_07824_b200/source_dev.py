"""Volume source load on the device: b = -int s(x, t) phi (disc.py:621-629).

The host restatement (tables.TensorTables.source_load) evaluates the source
plan with numpy at every volume quadrature point of every element — ~2 s on
the host at 10M DOFs, paid inside the first residual of a solve.  Here the
model's source plan is lowered to a device function (codegen.emit_plan, the
same lowering the generated kernels use) and one block per element
evaluates it at the element's quadrature points x_q = x0 + J xi_q and
contracts with the master tabulation: b_a = -sum_q detJ w_q s(x_q) phi_q(a).
Compiled once per model with NVRTC through the C ABI (ldg_jit_*)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib, codegen
from .tables import KernelNanError


class SrcParams(C.Structure):
    _fields_ = [("ne", C.c_int32), ("nq", C.c_int32), ("nb", C.c_int32), ("pad_", C.c_int32),
                ("t", C.c_double)] + [(k, C.c_void_p) for k in (
                    "x0", "J", "detj", "qp", "qw", "phi", "out", "bad")]


def generate_source(model, nd):
    ncu = model.ncu
    L = [codegen.DEVICE_HELPERS,
         codegen.emit_plan(model.source_plan(), "plan_src", nd, model.mu_bindings()),
         "struct SrcParams { int ne, nq, nb, pad_; double t; const double *x0, *J, *detj, *qp,"
         " *qw, *phi; double* out; unsigned long long* bad; };",
         f"#define ND {nd}\n#define NCU {ncu}",
         'extern "C" __global__ void __launch_bounds__(128) src_load(const SrcParams P) {',
         "  extern __shared__ double sv[];                 // detJ w_q s(x_q), (nq, ncu)",
         "  const int e = blockIdx.x;",
         "  const double dj = P.detj[e];",
         "  for (int q = threadIdx.x; q < P.nq; q += blockDim.x) {",
         "    double x[ND], s[NCU];",
         "    for (int d = 0; d < ND; ++d) {",
         "      double v = P.x0[e * ND + d];",
         "      for (int r = 0; r < ND; ++r) v += P.J[(e * ND + d) * ND + r] * P.qp[q * ND + r];",
         "      x[d] = v;",
         "    }",
         "    plan_src(x, P.t, nullptr, nullptr, nullptr, nullptr, s);",
         "    for (int c = 0; c < NCU; ++c) {",
         "      if (!isfinite(s[c])) atomicMin(P.bad, (unsigned long long)e);",
         "      sv[q * NCU + c] = dj * P.qw[q] * s[c];",
         "    }",
         "  }",
         "  __syncthreads();",
         "  for (int a = threadIdx.x; a < P.nb; a += blockDim.x)",
         "    for (int c = 0; c < NCU; ++c) {",
         "      double acc = 0.0;",
         "      for (int q = 0; q < P.nq; ++q) acc = fma(sv[q * NCU + c], P.phi[q * P.nb + a], acc);",
         "      P.out[((size_t)e * P.nb + a) * NCU + c] = -acc;",
         "    }",
         "}"]
    return "\n".join(L) + "\n"


class DeviceSource:
    """Source load of one system on the device (tensor or simplex tables:
    affine maps x0 + J xi, detJ, and the master's volume rule / tabulation)."""

    def __init__(self, tab, device):
        import torch
        from .nonlinear import compile_source
        self.tab, self.device = tab, device
        m = tab.master
        self.nd, self.ncu = tab.nd, tab.ncu
        self.src = generate_source(tab.model, tab.nd)
        self.cubin = compile_source(self.src)
        self.lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self.lib.ldg_jit_load(self.cubin, len(self.cubin), C.byref(h)),
                   "ldg_jit_load", jit=True)
        self._mod = h

        def dev(a):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)
        self.x0, self.J, self.detj = dev(tab.x0), dev(tab.J), dev(tab.detj)
        self.qp, self.qw, self.phi = dev(m.quad_pts), dev(m.quad_wts), dev(m.phi)
        self.nq, self.nb = int(m.quad_pts.shape[0]), int(m.n_nodes)
        self.bad = torch.full((1,), -1, dtype=torch.int64, device=device)

    def __del__(self):
        try:
            if getattr(self, "_mod", None):
                self.lib.ldg_jit_unload(self._mod)
        except Exception:
            pass

    def load(self, t):
        import torch
        out = torch.empty((self.tab.ne, self.nb, self.ncu), dtype=torch.float64,
                          device=self.device)
        P = SrcParams()
        P.ne, P.nq, P.nb, P.t = self.tab.ne, self.nq, self.nb, float(t)
        for k in ("x0", "J", "detj", "qp", "qw", "phi", "bad"):
            setattr(P, k, getattr(self, k).data_ptr())
        P.out = out.data_ptr()
        if self.tab.ne:
            _lib.check(self.lib.ldg_jit_launch(self._mod, b"src_load", self.tab.ne, 1, 128,
                                               8 * self.nq * self.ncu, C.byref(P), C.sizeof(P),
                                               _lib.stream_ptr()), "src_load", jit=True)
        bad = int(self.bad.item())
        if bad != -1:
            self.bad.fill_(-1)
            raise KernelNanError(f"source kernel produced non-finite values (first at element {bad})")
        return out


# ---------------------------------------------------------------------------
# initial state on the device (disc.py:420-432)
# ---------------------------------------------------------------------------


class InitParams(C.Structure):
    _fields_ = [("ne", C.c_int32), ("nb", C.c_int32), ("ng", C.c_int32), ("affine", C.c_int32)] + \
        [(k, C.c_void_p) for k in ("x0", "J", "xi", "gphi", "ho", "out", "bad")]


def generate_init(model, nd, nout):
    """init_nodes: one thread per (element, node) evaluates the model's init
    plan at the node's physical point -- x0 + J xi on affine elements, the
    geometry map sum_g N_g(xi) x_g (disc.py:105) on curved ones."""
    L = [codegen.DEVICE_HELPERS,
         codegen.emit_plan(model.init_plan(), "plan_init", nd, model.mu_bindings()),
         "struct InitParams { int ne, nb, ng, affine; const double *x0, *J, *xi, *gphi, *ho;"
         " double* out; unsigned long long* bad; };",
         f"#define ND {nd}\n#define NOUT {nout}",
         'extern "C" __global__ void __launch_bounds__(256) init_nodes(const InitParams P) {',
         "  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;",
         "  if (idx >= (long long)P.ne * P.nb) return;",
         "  const int e = (int)(idx / P.nb), n = (int)(idx % P.nb);",
         "  double x[ND], v[NOUT];",
         "  for (int d = 0; d < ND; ++d) {",
         "    double a;",
         "    if (P.affine) {",
         "      a = P.x0[e * ND + d];",
         "      for (int r = 0; r < ND; ++r) a += P.J[((size_t)e * ND + d) * ND + r] * P.xi[n * ND + r];",
         "    } else {",
         "      a = 0.0;",
         "      for (int g = 0; g < P.ng; ++g) a += P.gphi[n * P.ng + g] * P.ho[((size_t)e * P.ng + g) * ND + d];",
         "    }",
         "    x[d] = a;",
         "  }",
         "  plan_init(x, 0.0, nullptr, nullptr, nullptr, nullptr, v);",
         "  for (int c = 0; c < NOUT; ++c) {",
         "    if (!isfinite(v[c])) atomicMin(P.bad, (unsigned long long)e);",
         "    P.out[idx * NOUT + c] = v[c];",
         "  }",
         "}"]
    return "\n".join(L) + "\n"


def device_initial_values(tab, model, device):
    """(ne, nb, nout) device tensor of the init plan at every solution node
    (the values interpolate_initial splits into u | q | w)."""
    import torch
    from .nonlinear import compile_source
    nd = tab.nd
    m = tab.master
    nout = len(model.init_plan().outputs)
    src = generate_init(model, nd, nout)
    lib = _lib.load()
    h = C.c_void_p()
    cubin = compile_source(src)
    _lib.check(lib.ldg_jit_load(cubin, len(cubin), C.byref(h)), "ldg_jit_load", jit=True)

    def dev(a):
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)
    try:
        nb = int(m.n_nodes)
        xi = np.asarray(m.nodes, dtype=np.float64).reshape(nb, -1)[:, :nd]
        affine = not getattr(tab, "curved", False)
        keep = []
        P = InitParams()
        P.ne, P.nb, P.affine = tab.ne, nb, int(affine)
        if affine:
            x0, J, xid = dev(tab.x0), dev(tab.J), dev(xi)
            keep += [x0, J, xid]
            P.x0, P.J, P.xi = x0.data_ptr(), J.data_ptr(), xid.data_ptr()
            P.ng = 0
        else:
            gphi = dev(tab.geom_master.eval_basis(np.asarray(m.nodes)))
            ho = dev(tab.mesh.ho_nodes)
            keep += [gphi, ho]
            P.ng, P.gphi, P.ho = int(gphi.shape[1]), gphi.data_ptr(), ho.data_ptr()
        out = torch.empty((tab.ne, nb, nout), dtype=torch.float64, device=device)
        bad = torch.full((1,), -1, dtype=torch.int64, device=device)
        P.out, P.bad = out.data_ptr(), bad.data_ptr()
        total = tab.ne * nb
        if total:
            _lib.check(lib.ldg_jit_launch(h, b"init_nodes", (total + 255) // 256, 1, 256, 0,
                                          C.byref(P), C.sizeof(P), _lib.stream_ptr()),
                       "init_nodes", jit=True)
        b = int(bad.item())
        if b != -1:
            raise KernelNanError("initial kernel produced non-finite values "
                                 f"(first at element {b})")
        return out
    finally:
        lib.ldg_jit_unload(h)
