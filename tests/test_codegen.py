"""CPU checks of the generated-kernel path: plan -> CUDA lowering, host
tables of the nonlinear path, and NVRTC compilation for sm_100a (compiling
needs no GPU)."""

import math

import numpy as np
import pytest

from cases import MB_CASES, NL_CASES, b200_setup, build_case


def test_literals_are_exact():
    from paper_2205_07824_b200.codegen import literal
    for v in (0.1, -1.4, 1e-300, 3.0, -0.0, 2.0 ** -1074):
        s = literal(v)
        assert float.fromhex(s.strip("()")) == v
    assert "longlong" in literal(math.inf) and "longlong" in literal(math.nan)


def test_dual_rules_follow_reference():
    """abs -> sign rule, min/max tie rules, pow log term only where the
    exponent's tangent is nonzero (expr.py:611-651)."""
    from paper_2205_07824_b200 import codegen
    from paper_2205_07824_b200.expr import compile_texts
    from paper_2205_07824_b200.model import reserved_symbols
    syms = reserved_symbols(2, 2, 0, 1)
    plan = compile_texts(["abs(u1) + min(u1, u2) + max(u2, 0.5)", "pow(u1, u2) + pow(2, u1)"],
                         syms)
    src = codegen.emit_plan(plan, "p", 2, {"mu1": 1.0})
    assert "ldg_sign(" in src and "<=" in src and ">=" in src
    assert "== 0.0 ? 0.0 :" in src and "log(" in src
    assert "void p(" in src and "void p_d(" in src


@pytest.mark.parametrize("name", sorted(NL_CASES))
def test_nonlinear_tables_and_routing(name):
    from paper_2205_07824_b200.nonlinear import NlTables, generate_source, linear_path_reason
    model, mesh, topo, master = build_case(NL_CASES[name], *b200_setup())
    assert linear_path_reason(model) is not None or mesh.nd == 1   # 1D: always generated
    tab = NlTables(model, mesh, topo, master)
    # face Gauss points matched to the reference rule, weights reproduce the face area
    nqf = tab.fxi.shape[1]
    assert tab.fw.shape == (tab.nf, nqf)
    assert np.allclose(tab.fw.sum(axis=1), [f.weights.sum() for f in master.faces])
    src, shape = generate_source(tab)
    assert "plan_flux_d" in src and shape["NB"] == (master.p + 1) ** mesh.nd


@pytest.mark.parametrize("name", ["euler2d_quad_dirichlet_p2", "ns3d_hex_periodic_p2",
                                  "nonlin_diff2d_quad_p2", "wave2d_quad_absorbing_p3",
                                  "reactode2d_quad_p2"])
def test_nvrtc_compiles_generated_source(name):
    from paper_2205_07824_b200.nonlinear import NlTables, compile_source, generate_source
    model, mesh, topo, master = build_case({**NL_CASES, **MB_CASES}[name], *b200_setup())
    src, _ = generate_source(NlTables(model, mesh, topo, master))
    cubin = compile_source(src)
    assert cubin[:4] == b"\x7fELF" and len(cubin) > 10000


def test_linear_models_keep_the_fused_path():
    from paper_2205_07824_b200 import model
    from paper_2205_07824_b200.nonlinear import linear_path_reason
    assert linear_path_reason(model.builtin_model("poisson", nd=3)) is None
    assert linear_path_reason(model.builtin_model("convection_diffusion", nd=3)) is None
    assert linear_path_reason(model.builtin_model("euler", nd=2)) == "kind C"


def test_device_source_compiles():
    from paper_2205_07824_b200 import model
    from paper_2205_07824_b200.nonlinear import compile_source
    from paper_2205_07824_b200.source_dev import generate_source
    m = model.load_model(str(__import__("cases").GOLDEN / "poisson3d.model"))
    cubin = compile_source(generate_source(m, 3))
    assert cubin[:4] == b"\x7fELF"


def test_device_diagnostics_compile():
    from cases import CASES
    from paper_2205_07824_b200.diagnostics import _source
    from paper_2205_07824_b200.expr import compile_texts
    from paper_2205_07824_b200.nonlinear import compile_source
    model = build_case(CASES["poisson2d_quad_p3"], *b200_setup())[0]
    for texts, nf, mode in ((["sin(x1)*x2"], 1, 0), (["u1*u1 + q1_2"], 1, 1)):
        src = _source(model, 2, compile_texts(texts, model.symbols), nf, mode)
        assert compile_source(src)[:4] == b"\x7fELF"
