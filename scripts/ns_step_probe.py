import sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "scripts")); sys.path.insert(0, str(ROOT / "tests"))
import nl_bench
from cases import TRANSIENT_CASES
ns = dict(TRANSIENT_CASES["ns3d_tgv_hex_p2_dirk11"], p=3, stages=1, order=1)
for n, dt, flags in ((16, 0.005, None), (16, 0.002, None), (16, 0.01, {"restart": 200, "gmres_max_iter": 2000})):
    r = nl_bench.run_transient(dict(ns, counts=[n] * 3), 1, dt, flags=flags)
    print(n, dt, flags, json.dumps(r))
