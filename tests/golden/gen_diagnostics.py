"""Golden values of the reference's diagnostics (diagnostics.py:35-89) on
seeded states of a few cases, from the UNMODIFIED reference package:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/gen_diagnostics.py

Writes tests/golden/diagnostics.json (compute_l2_error with exact u and q,
compute_functional) -- what pins paper_2205_07824_b200.diagnostics."""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

from ldgkit import master as R_master  # noqa: E402
from ldgkit import mesh as R_mesh  # noqa: E402
from ldgkit import model as R_model  # noqa: E402
from ldgkit.diagnostics import compute_functional, compute_l2_error  # noqa: E402
from ldgkit.disc import LdgSystem, SolverState  # noqa: E402

from cases import CASES, DIAG, NL_CASES, build_case, case_state, seeded_state  # noqa: E402

def main():
    out = {}
    for name, (eu, eq, g, t) in DIAG.items():
        spec = {**CASES, **NL_CASES}[name]
        model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
        s = LdgSystem(model, mesh, topo, master)
        shape = (s.n_elements, s.n_nodes, s.ncu)
        u = case_state(spec, *shape, 1) if "state" in spec else seeded_state(*shape, 1)
        st = SolverState(u=u, q=None, w=None, t=t)
        n = compute_l2_error(s, st, eu, eq)
        f = compute_functional(s, st, g)
        out[name] = {"error_u": n.error_u, "error_q": n.error_q, "absolute_u": n.absolute_u,
                     "absolute_q": n.absolute_q, "functional": f}
        print(name, out[name])
    (HERE / "diagnostics.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
