"""A/B: hybrid cycles launched eagerly (domdec_sweep / flow_update, no host
sync) vs domdec_run_cycles (CUDA-graph units).  Prints one JSON line per
configuration with ms per cycle of each."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2405_09400_b200 import DomDec  # noqa: E402
from synth import make_problem  # noqa: E402


def main():
    for N, s, fe, cyc in [(256, 4, 1, 40), (256, 4, 0, 40), (1024, 4, 0, 20), (1024, 4, 8, 16)]:
        p = make_problem("gm", N, s, eps_factor=4.0, theta_deg=5.0, seed=0)
        out = {"N": N, "s": s, "flow_every": fe, "cycles": cyc}
        for mode in ("eager", "graph"):
            dd = DomDec.from_problem(p)
            G = 2 if fe == 0 else 2 * fe
            dd.run_cycles(G, flow_every=fe, conv=0.0) if mode == "graph" else None
            if mode == "eager":
                for k in range(G):
                    dd.sweep("A"); dd.sweep("B")
                    if fe and k % fe == fe - 1:
                        dd.flow_update()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if mode == "graph":
                n, e, mv = dd.run_cycles(cyc, flow_every=fe, conv=0.0)
            else:
                for k in range(cyc):
                    dd.sweep("A"); dd.sweep("B")
                    if fe and k % fe == fe - 1:
                        dd.flow_update()
                dd.marginal_error()
            torch.cuda.synchronize()
            out[mode + "_ms_per_cycle"] = 1e3 * (time.perf_counter() - t0) / cyc
            dd.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
