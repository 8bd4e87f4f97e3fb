"""The oracle (oracle/) against golden vectors of the unmodified reference."""

import numpy as np
import pytest

from cases import CASES, GOLDEN, NL_CASES, b200_setup, build_case
from oracle import make_oracle


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(name):
    g = np.load(GOLDEN / f"{name}.npz")
    model, mesh, topo, master = build_case(CASES[name], *b200_setup())
    o = make_oracle(model, mesh, topo, master)
    assert np.array_equal(o.switch, g["switch"])
    R = o.residual(g["u"])
    J = o.residual_tangent(g["u"], g["du"])
    assert rel(R, g["R"]) < 1e-13
    assert rel(J, g["Jdu"]) < 1e-13
    if "q" in g:
        assert rel(o.compute_mixed(g["u"], 0.0), g["q"]) < 1e-13
        assert rel(o.compute_mixed(g["du"], 0.0, True), g["dq"]) < 1e-13
    assert rel(o.d.fi_h, g["fi_h"]) < 1e-14


@pytest.mark.parametrize("name", sorted(NL_CASES))
def test_oracle_matches_reference_golden_nonlinear(name):
    """Kind C (LLF) and nonlinear kind D cases: residual, tangent, mixed,
    mass and mass tangent extra at a physical base state."""
    g = np.load(GOLDEN / f"{name}.npz")
    model, mesh, topo, master = build_case(NL_CASES[name], *b200_setup())
    o = make_oracle(model, mesh, topo, master)
    t = float(g["t"])
    assert np.array_equal(o.switch, g["switch"])
    assert rel(o.residual(g["u"], t), g["R"]) < 1e-13
    assert rel(o.residual_tangent(g["u"], g["du"], t), g["Jdu"]) < 1e-13
    assert rel(o.mass_apply(g["u"], g["y"], t), g["M"]) < 1e-13
    if "Mx" in g:
        assert rel(o.mass_tangent_extra(g["u"], g["y"], g["du"], t), g["Mx"]) < 1e-13
    if "q" in g:
        assert rel(o.compute_mixed(g["u"], t), g["q"]) < 1e-13
        assert rel(o.compute_mixed(g["du"], t, True), g["dq"]) < 1e-13
