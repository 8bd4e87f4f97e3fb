"""ORACLE -- test infrastructure only.

CPU restatement of the reference (``ldgkit``) LDG residual / tangent and
Newton-GMRES path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs may import this package; the product
package ``paper_2205_07824_b200`` never does.
"""

from .ldg_oracle import OracleLdg, run_plan, scatter_add  # noqa: F401


def make_oracle(model, mesh, topo, master):
    """Oracle system over setup objects (reference or B200-package ones)."""
    from paper_2205_07824_b200.refelem import build_geom_master, face_map
    geom = build_geom_master(mesh.elem_kind, mesh.p_geom)
    return OracleLdg(model, mesh, topo, master, geom, face_map)
