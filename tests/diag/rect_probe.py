"""Product-coupling first sweeps on rectangular and square grids vs the oracle
(development aid): rel_bulk / rel_tail per shape and pass count."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from oracle import multiscale as M
from parity import compare_states
from test_gpu_rectangular import _dyadic
from paper_2405_09400_b200 import DomDec

E, s, eps_p = 18, 2, 4.0
for shape in [(24, 40), (40, 24), (32, 32), (24, 24), (40, 40)]:
    for K in (2, 5, 10):
        mu, nu = _dyadic(shape, E, 1), _dyadic(shape, E, 2)
        h = 2.0 / shape[0]
        row = {"shape": shape, "K": K}
        for part in "AB":
            st = M.product_state(mu, nu, s, eps_p, h)
            O.domdec_sweep(st, part, fixed_iter=K)
            dd = DomDec.product(mu, nu, s, eps_p * h * h, h, E, fixed_iter=K)
            dd.sweep(part)
            c = compare_states(dd.boxes(), st.boxes)
            row[part] = [round(c["rel_bulk"] * 1e5, 2), round(c["rel_tail"] * 1e3, 2), c["unexplained"]]
            dd.close()
        print(json.dumps(row), flush=True)
