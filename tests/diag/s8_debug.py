"""s = 8 parity debug (development aid): per basic cell, the worst bulk
entry GPU vs oracle after one fixed-K A sweep; the composite cell, member,
position relative to the X-block and the values; K = 1, 2, 5, 20."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from parity import compare_cell, gpu_ctx, oracle_state
from synth import make_problem

p = make_problem("gm", 64, 8, eps_factor=2.0, theta_deg=20, seed=2)
for K in (1, 2, 5, 20):
    for part in "AB":
        st = oracle_state(p)
        ost = O.domdec_sweep(st, part, fixed_iter=K)
        dd = gpu_ctx(p, fixed_iter=K)
        gst = dd.sweep(part, stats=True)
        gb = dd.boxes()
        worst = []
        for i in range(len(st.boxes)):
            c = compare_cell(gb[i], st.boxes[i])
            worst.append((c["rel_bulk"], i, c["box_equal"]))
        worst.sort(reverse=True)
        rows = []
        for rb, i, be in worst[:4]:
            gr, gc, ga = gb[i]; orr, oc, oa = st.boxes[i]
            if ga.shape == oa.shape:
                rel = np.abs(ga - oa) / np.maximum(oa, 1e-300)
                mask = oa >= 1e-6 * oa.max()
                k = np.argmax(np.where(mask, rel, 0))
                r, cc = divmod(k, oa.shape[1])
                rows.append({"i": i, "rel": float(rb), "box": [gr, gc, list(ga.shape)], "at": [int(r), int(cc)],
                             "g": float(ga[r, cc]), "o": float(oa[r, cc]), "o_max": float(oa.max()),
                             "mass_g": float(ga.sum()), "mass_o": float(oa.sum()), "m": float(st.m[i])})
            else:
                rows.append({"i": i, "rel": float(rb), "box_g": [gr, gc, list(ga.shape)], "box_o": [orr, oc, list(oa.shape)]})
        print(json.dumps({"K": K, "part": part, "l1x_g": gst["l1x_final"], "l1x_o": ost["e_sum"],
                          "worst": rows}), flush=True)
        dd.close()
