"""Parity error budget (development aid): rel_bulk / rel_tail of one fixed-K
sweep vs the oracle for several configs, size-class settings and builds
(DD_LIB_PATH selects the build; DD_H_CLUSTER the huge-class path)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
from parity import CONFIGS, compare_states, gpu_ctx, oracle_state

K = 20
for cfg in ["cfg1_gm", "cfg2_gm", "cfg2_bumps", "cfg3_gm_eps2"]:
    p = CONFIGS[cfg]()
    for part in "AB":
        st = oracle_state(p)
        O.domdec_sweep(st, part, fixed_iter=K)
        row = {"lib": os.environ.get("DD_LIB_PATH", "new"), "cl": os.environ.get("DD_H_CLUSTER", "8"), "cfg": cfg,
               "part": part}
        for cap in (0, 8):
            dd = gpu_ctx(p, fixed_iter=K, comp_cap=cap)
            dd.sweep(part)
            c = compare_states(dd.boxes(), st.boxes)
            row[f"cap{cap}"] = [round(c["rel_bulk"] * 1e5, 3), round(c["rel_tail"] * 1e3, 3), c["unexplained"]]
            dd.close()
        print(json.dumps(row), flush=True)
