"""Device diagnostics (paper_2205_07824_b200.diagnostics) vs the reference's
compute_l2_error / compute_functional (diagnostics.py:35-89) on the golden
values of tests/golden/gen_diagnostics.py."""

import json

import numpy as np
import pytest

from cases import CASES, DIAG, GOLDEN, NL_CASES, b200_setup, build_case, case_state, seeded_state

pytestmark = pytest.mark.gpu
G = json.loads((GOLDEN / "diagnostics.json").read_text())
TOL = 1e-12


@pytest.mark.parametrize("name", sorted(G))
def test_diagnostics_match_reference(name):
    from paper_2205_07824_b200.diagnostics import compute_functional, compute_l2_error
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    eu, eq, g, t = DIAG[name]
    spec = {**CASES, **NL_CASES}[name]
    s = LdgSystem(*build_case(spec, *b200_setup()))
    shape = (s.n_elements, s.n_nodes, s.ncu)
    u = case_state(spec, *shape, 1) if "state" in spec else seeded_state(*shape, 1)
    st = SolverState(u=u, q=None, w=None, t=t)
    n = compute_l2_error(s, st, eu, eq)
    ref = G[name]
    assert abs(n.error_u - ref["error_u"]) <= TOL * abs(ref["error_u"])
    assert n.absolute_u == ref["absolute_u"]
    if ref["error_q"] is None:
        assert n.error_q is None
    else:
        assert abs(n.error_q - ref["error_q"]) <= TOL * abs(ref["error_q"])
    f = compute_functional(s, st, g)
    assert abs(f - ref["functional"]) <= TOL * max(abs(ref["functional"]), 1e-300)


def test_functional_rejects_non_finite():
    from paper_2205_07824_b200.diagnostics import compute_functional
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    s = LdgSystem(*build_case(CASES["poisson2d_quad_p3"], *b200_setup()))
    u = np.zeros((s.n_elements, s.n_nodes, 1))
    with pytest.raises(ValueError, match="non-finite"):
        compute_functional(s, SolverState(u=u, q=None, w=None, t=0.0), "1/u1")
