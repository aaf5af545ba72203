"""Debug aid: pure domdec parity trajectory on a config, report the first
sweep/cell whose comparison with the oracle fails."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from parity import CONFIGS, compare_cell, gpu_ctx, oracle_state

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2_bumps"
p = CONFIGS[cfg]()
K = 20
st = oracle_state(p)
dd = gpu_ctx(p, fixed_iter=K)
for k in range(8):
    part = "AB"[k % 2]
    O.domdec_sweep(st, part, fixed_iter=K)
    dd.sweep(part)
    gb = dd.boxes()
    bad = []
    for i in range(len(gb)):
        c = compare_cell(gb[i], st.boxes[i])
        if not c["guard_ok"] or c["rel_bulk"] > 4e-5:
            bad.append((i, c))
    bad.sort(key=lambda t: (t[1]["guard_ok"], -t[1]["rel_bulk"]))
    print("sweep", k, part, "bad", len(bad), bad[:3], flush=True)
    if bad and (k == 7 or not bad[0][1]["guard_ok"] or bad[0][1]["rel_bulk"] > 1e-3):
        i = bad[0][0]
        g, o = gb[i], st.boxes[i]
        print("gpu box", g[0], g[1], g[2].shape, "oracle", o[0], o[1], o[2].shape)
        np.set_printoptions(precision=3, linewidth=200)
        G, Ov = g[2], o[2]
        if G.shape == Ov.shape:
            rel = np.abs(G - Ov) / np.maximum(Ov, 1e-300)
            idx = np.unravel_index(np.argmax(np.where(Ov >= 1e-6 * Ov.max(), rel, 0)), G.shape)
            print("worst", idx, G[idx], Ov[idx], "max", Ov.max(), "sumG", G.sum(), "sumO", Ov.sum())
            only = (G > 0) != (Ov > 0)
            print("only-one-side entries", [(tuple(x), G[tuple(x)], Ov[tuple(x)]) for x in np.argwhere(only)[:5]])
        else:
            print("G", G, "O", Ov)
