#!/usr/bin/env python
"""Benchmark of the B200 hot path of arXiv 2405.09400.

Workload (BASELINE.json configs[3]): 1024x1024 -> 1024x1024 grid, cell size 4,
eps = (2h)^2, Gaussian-mixture marginals GM(seed) pushed by a 20 degree
rotation+contraction (synthetic, seeded, exact dyadic values).  A *step* is
one hybrid cycle of Alg. 3: sweep A, sweep B, flow update
— every row of SURVEY §8(a).  The metric is domdec sweeps/s (two sweeps per
step; flow updates take no trajectory time).

Multi-GPU (torchrun): one independent problem per rank (GM seed = rank; the
paper's benchmark is a set of independent pairs), weak
scaling; the only collectives are the barrier/max-time reductions of the
timing protocol and the per-cycle L1-error allreduce of the convergence
check.

--impl reference times the fp64 CPU oracle (the reference arm of this tier)
on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "domdec sweeps/sec and time-to-L1-marginal-error 1e-4 at NxN grid, 1/2/4/8 B200"
CFG = {"N": 1024, "s": 4, "eps_factor": 2.0, "theta": 20.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--N", type=int, default=CFG["N"])
    ap.add_argument("--s", type=int, default=CFG["s"])
    ap.add_argument("--no-ttc", action="store_true", help="skip the time-to-1e-4 run")
    ap.add_argument("--ttc-cycles", type=int, default=3000)
    ap.add_argument("--ttc-seconds", type=float, default=150.0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--parallelism", default="independent", choices=["independent", "stripes"],
                    help="N>1: one problem per rank (weak scaling, default) or one problem in row stripes "
                         "(strong scaling, SURVEY 8(e); the min-cost flow is replicated)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make(seed, N, s):
    from synth import make_problem
    return make_problem("gm", N, s, eps_factor=CFG["eps_factor"], theta_deg=CFG["theta"], seed=seed)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, dev):
        self.dev = dev
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline(p, seconds):
    """The fp64 oracle as it stands (tests' reference implementation) on a
    bounded sample of the same workload: composite cells of the first A sweep
    of the same problem, processed one by one until `seconds` elapse."""
    import oracle as O
    st = O.init_state(p.mu, p.nu, p.s, p.eps_prime, p.h, p.init_off, p.init_ext, p.init_pos, p.init_data)
    ncomp = len(O.composite_partition(st.n1, st.n2, "A"))
    rng = np.random.default_rng(0)
    order = rng.permutation(ncomp)
    done = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds and done < ncomp:
        O.domdec_sweep(st, "A", err=1e-4, cells=[int(x) for x in order[done:done + 8]])
        done += 8
    dt = time.perf_counter() - t0
    return {"value": done / dt / ncomp, "unit": "sweeps/s", "cores": 1, "kind": "oracle",
            "sample": f"{done} of {ncomp} composite cells of the first A sweep of GM(0) {p.N}^2 s={p.s} "
                      f"(fp64 dense log-domain Sinkhorn, Err=1e-4), {dt:.1f} s, extrapolated to one sweep"}


def bench_config(a, world):
    """The workload both arms report (the reference arm adds its sample)."""
    return {"workload": f"GM(rank) {a.N}x{a.N} -> {a.N}x{a.N}, s={a.s}, eps=(2h)^2, theta=20deg; "
                        "step = hybrid cycle (sweep A, sweep B, flow update)",
            "grid": a.N, "cell_size": a.s, "eps": "(2h)^2", "parallelism": f"independent problems x{world}",
            "l2": "flushed between timed steps (256 MB write)",
            "precision": "log-domain fp32 (local gauge), marginals fp64"}


def run_reference(a):
    world, rank, local = dist_env()
    if rank != 0:
        return
    p = make(0, a.N, a.s)
    per = max(1.0, a.cpu_seconds / max(1, a.steps + a.warmup))
    for _ in range(a.warmup):
        cpu_baseline(p, per / 4)
    vals = []
    t0 = time.perf_counter()
    for _ in range(a.steps):
        vals.append(cpu_baseline(p, per))
    dt = time.perf_counter() - t0
    v = float(np.mean([x["value"] for x in vals]))
    out = {"metric": METRIC, "value": v, "unit": "sweeps/s", "n_gpus": a.gpus, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": dt * 1e3 / a.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": dict(bench_config(a, a.gpus), sample=vals[-1]["sample"],
                                precision="fp64 oracle (log-domain Sinkhorn)"),
           "impl": "reference",
           "cpu_baseline": {"value": v, "unit": "sweeps/s", "cores": 1, "kind": "oracle",
                            "sample": vals[-1]["sample"]},
           "e2e": {"value": v, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_stripes(a):
    """One problem sharded in row stripes over the ranks (stripes.py):
    strong scaling; the timed step is one hybrid cycle of the whole problem."""
    import torch
    import torch.distributed as dist
    from paper_2405_09400_b200.stripes import GpuEngine, cycle_program, run_distributed, stripe_rows

    world, rank, local = dist_env()
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = make(0, a.N, a.s)
    rows = stripe_rows(a.N // a.s, world)
    eng = GpuEngine(p, rows[rank], rows[rank + 1], device=local)
    n1, n2 = eng.n1, eng.n2
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def cycle():
        run_distributed(cycle_program(eng, rank, world, rows, n1, n2), rank, world, device=dev)

    for _ in range(a.warmup):
        cycle()
    torch.cuda.synchronize()
    dist.barrier()
    ms = []
    with ClockSampler(local) as clk:
        for k in range(a.steps):
            flush.fill_(float(k))
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cycle()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(ms) / 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_s = float(t.item())
    if rank == 0:
        out = {"metric": METRIC, "value": 2 * a.steps / total_s, "unit": "sweeps/s", "n_gpus": world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_s * 1e3 / a.steps,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic",
               "config": {"workload": f"GM(0) {a.N}x{a.N}, s={a.s}, eps=(2h)^2, theta=20deg; step = hybrid cycle",
                          "parallelism": f"row stripes x{world} (halo rows over NCCL, replicated min-cost flow)",
                          "l2": "flushed between timed steps (256 MB write)"},
               "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2405_09400_b200 import DomDec, mufu_peak

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    p = make(rank, a.N, a.s)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(stream):
        dd = DomDec.from_problem(p, stream=stream.cuda_stream, device=local)
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

        def cycle(sweep_events=None):
            for part in ("A", "B"):
                if sweep_events is not None:
                    e0, e1 = ev(), ev()
                    e0.record(stream)
                    dd.sweep(part)
                    e1.record(stream)
                    sweep_events.append((e0, e1))
                else:
                    dd.sweep(part)
            dd.flow_update()

        for _ in range(a.warmup):
            cycle()
        barrier()
        dd.reset_counters()
        step_ev, sweep_ev = [], []
        with ClockSampler(local) as clk:
            barrier()
            for k in range(a.steps):
                flush.fill_(float(k))          # L2 flush between timed steps (outside the events)
                e0, e1 = ev(), ev()
                e0.record(stream)
                cycle(sweep_ev)
                e1.record(stream)
                step_ev.append((e0, e1))
            barrier()
        step_ms = [x.elapsed_time(y) for x, y in step_ev]
        sweep_ms = [x.elapsed_time(y) for x, y in sweep_ev]
        cnt = dd.counters()
        # one more (untimed) cycle for the flow-update statistics
        dd.sweep("A")
        dd.sweep("B")
        fstats = dd.flow_update(stats=True)
        total_s = allmax(sum(step_ms) / 1e3)
        sweeps_done = 2 * a.steps * world
        value = sweeps_done / total_s
        ex, ey = dd.marginal_error()

        # roofline of the dominant kernel (the fused sweep): algorithmic MUFU ops
        sweep_s = sum(sweep_ms) / 1e3
        achieved = cnt["mufu_ops"] / sweep_s
        import json as _j
        mp = {}
        try:
            mp = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        sm_max = float(mp.get("sm_max_mhz", 1965.0))
        peak_nominal = 148 * 16 * sm_max * 1e6        # MUFU ex2/lg2 per s
        measured_mufu = mufu_peak(local)
        hbm_peak = float(mp.get("hbm_gbs", 6650.0)) * 1e9

        # end-to-end through the public API from host buffers
        barrier()
        t0 = time.perf_counter()
        dd2 = DomDec.from_problem(p, stream=stream.cuda_stream, device=local)
        e2e_steps = max(1, min(a.steps, a.e2e_steps))
        for _ in range(e2e_steps):
            dd2.sweep("A")
            dd2.sweep("B")
            dd2.flow_update()
        e2e_err = dd2.marginal_error()
        torch.cuda.synchronize()
        e2e_s = allmax(time.perf_counter() - t0)
        h2d = (p.mu.nbytes + p.nu.nbytes + p.init_off.nbytes + p.init_ext.nbytes + p.init_pos.nbytes +
               p.init_data.nbytes)
        dd2.close()

        # time to L1 marginal error 1e-4 (reading R14): wall time from the
        # end of domdec_init to the first hybrid cycle whose A and B
        # sweep-entry errors are both <= 1e-4, synchronising at cycle ends
        # only.  Measured on config 3 (256^2, s = 4, the "good initial
        # coupling" T_5) and on the bench grid with T_5.
        def ttc_run(N, s, theta, cap_s, cap_cycles):
            from synth import make_problem
            q = make_problem("gm", N, s, eps_factor=CFG["eps_factor"], theta_deg=theta, seed=rank)
            barrier()
            dd3 = DomDec.from_problem(q, stream=stream.cuda_stream, device=local)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res, conv, flows = None, float("nan"), 0
            t_sw = t_fl = 0.0   # host time per phase (each stats call synchronises)
            for c in range(cap_cycles):
                t1 = time.perf_counter()
                sa = dd3.sweep("A", stats=True)
                sb = dd3.sweep("B", stats=True)
                t2 = time.perf_counter()
                fs = dd3.flow_update(stats=True)
                t_sw += t2 - t1
                t_fl += time.perf_counter() - t2
                flows += int(fs["stationary"] == 0)
                conv = allmax(max(sa["l1x_entry"], sb["l1x_entry"]))
                if conv <= 1e-4:
                    torch.cuda.synchronize()
                    res = {"seconds": allmax(time.perf_counter() - t0), "cycles": c + 1, "sweeps": 2 * (c + 1),
                           "t": 2 * (c + 1) / q.n, "nonstationary_flows": flows}
                    break
                if allmax(time.perf_counter() - t0) > cap_s:
                    res = {"seconds": None, "reached": False, "cycles_run": c + 1, "last_entry_error": conv,
                           "cap_seconds": cap_s, "nonstationary_flows": flows}
                    break
            if res is None:
                res = {"seconds": None, "reached": False, "cycles_run": cap_cycles, "last_entry_error": conv,
                       "nonstationary_flows": flows}
            res["workload"] = f"GM(rank) {N}^2 s={s} eps=(2h)^2 theta={theta:g}deg, hybrid A/B/flow"
            res["phase_seconds"] = {"sweeps": t_sw, "flow_updates": t_fl}
            dd3.close()
            return res

        sg = None
        if rank == 0 and not a.no_ttc:
            # SinkhornGPU comparator: global separable
            # Sinkhorn on the cfg3 pair (256^2, theta=5), cold start at eps=(2h)^2, to Err=1e-4.
            from paper_2405_09400_b200 import sinkhorn_global
            from synth import make_problem as _mp
            q = _mp("gm", 256, 4, theta_deg=5.0, seed=0)
            _, _, it_sg, e_sg, ms_sg = sinkhorn_global(q.mu, q.nu, q.eps_prime, err=1e-4, max_iter=20000,
                                                       check_every=10)
            sg = {"workload": "GM(0) 256^2 theta=5deg, eps=(2h)^2, cold start, Err=1e-4 (PAPER.md:1264)",
                  "seconds": ms_sg / 1e3, "iterations": it_sg, "l1_x": e_sg, "ms_per_iteration": ms_sg / it_sg,
                  "note": "device time (CUDA events), host copies excluded; fp64 potentials"}
        ttc = None
        if not a.no_ttc:
            ttc = {"cfg3_256": ttc_run(256, 4, 5.0, a.ttc_seconds, a.ttc_cycles),
                   f"cfg4_{a.N}": ttc_run(a.N, a.s, 5.0, a.ttc_seconds, a.ttc_cycles)}

    if rank == 0:
        cpu = cpu_baseline(p, a.cpu_seconds) if world == 1 else None
        out = {
            "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_s * 1e3 / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": bench_config(a, world),
            "e2e": {"value": 2 * e2e_steps * world / e2e_s, "unit": "sweeps/s",
                    "h2d_bytes_per_step": int(h2d / e2e_steps), "d2h_bytes_per_step": int(16 / e2e_steps),
                    "steps": e2e_steps,
                    "note": "domdec_init from host buffers + steps hybrid cycles + marginal_error readback"},
            # per step: 2 sweeps x (solve_kernel + split_kernel in 3 size classes) + flow
            # (k_flow_costs, mcf_kernel, k_apply_flow) -- profiles/ launch list
            "gpu_launches": 15 * a.steps,
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_nominal / 1e12,
                         "unit": "TOP/s (MUFU ex2+lg2)", "frac": achieved / peak_nominal,
                         # dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full
                         # capture of each sweep kernel (profiles/r01_ncu_summary.txt: solve
                         # 199.3 + 9.3 MB, split 195.3 + 154.8 MB, small size class, one sweep)
                         "traffic": 5.59e8, "traffic_unit": "bytes per sweep (solve + split launch)",
                         "traffic_vs_algorithmic": 5.59e8 / max(1.0, cnt["bytes"] / max(1, cnt["sweeps"])),
                         "kernel": "sweep = solve_kernel + split_kernel (a1-a6)",
                         "peak_source": f"148 SM x 16 MUFU/clk x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                         "measured_mufu_peak": measured_mufu / 1e12,
                         "frac_of_measured": achieved / measured_mufu,
                         "mufu_ops_per_sweep": cnt["mufu_ops"] / max(1, cnt["sweeps"]),
                         "sweep_ms": sweep_s * 1e3 / max(1, cnt["sweeps"]),
                         "hbm": {"bytes_per_sweep": cnt["bytes"] / max(1, cnt["sweeps"]),
                                 "achieved_gbs": cnt["bytes"] / sweep_s / 1e9,
                                 "peak_gbs": hbm_peak / 1e9, "frac": cnt["bytes"] / sweep_s / hbm_peak}},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "time_to_l1_1e-4": ttc,
            "sinkhorn_global_cfg3": sg,
            # sweeps/s with A and B separately, flow-update time, cycles/s
            "per_partition": {"sweep_ms_A": float(np.mean(sweep_ms[0::2])), "sweep_ms_B": float(np.mean(sweep_ms[1::2])),
                              "flow_ms": (sum(step_ms) - sum(sweep_ms)) / a.steps,
                              "cycles_per_s": a.steps * world / total_s},
            "state": {"l1_x": ex, "l1_y": ey, "iters_per_cell": cnt["iters"] / max(1, cnt["cells"]),
                      "flow_ms_per_step": (sum(step_ms) - sum(sweep_ms)) / a.steps},
            "step_breakdown": {
                "sweeps_share": sum(sweep_ms) / sum(step_ms),
                "flow_share": 1.0 - sum(sweep_ms) / sum(step_ms),
                "dominant_kernel": "mcf_kernel (exact min-cost flow, a8): latency-bound (grid barriers), "
                                   "no throughput roofline; reported in rounds and ms",
                "mcf_last_cycle": {"solver_ms": fstats["solver_ms"], "tile_phases": fstats["rounds"],
                                   "label_rounds": fstats["label_rounds"], "refines": fstats["refines"],
                                   "objective": fstats["objective"], "changed_cells": fstats["changed_cells"]}},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.parallelism == "stripes" and dist_env()[0] > 1:
        run_stripes(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
