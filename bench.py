#!/usr/bin/env python
"""bench.py -- fluid+IB grid-point updates per second (fp64) of the IB-GM step on B200.

Workload at every N: BASELINE.json configs[4] (3D, 384^3 MAC grid, eight triangulated
ellipsoidal shells of 100k nodes each, random divergence-free initial velocity,
rho=1, mu=0.005, dt=5e-5) -- the configuration BASELINE names for the 8-GPU z-slab
split; it also fits one B200 (~6 GB of fields), so the driver's per-N values form
one strong-scaling curve.  configs[2] (2D, 1024^2) and configs[3] (3D, 128^3) are
reported under "extra" with the same keys.  One "step" = one full IB-GM time step
(Steps 1a-3f) on the whole grid.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

`--gpus N` (N > 1) outside torchrun relaunches itself under torch.distributed.run with
N ranks on 127.0.0.1.  Prints ONE JSON line on rank 0.  value = N^d * steps / (max
over ranks of the device time of the K timed steps).  With N GPUs the same grid is
cut into N z-slabs, one per rank, over NCCL (strong scaling).  The
resident fields (14 fp64 fields: 235 MB at 128^3, 6.3 GB at 384^3) are larger than
the 126 MB L2, so no explicit L2 flush is done between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fluid+IB grid-point updates/sec (fp64)"
UNIT = "grid-point updates/s"

# algorithmic HBM bytes per grid cell of each phase:
# doubles each phase must read + write once, x 8 B.
# steps per segment between restores of the base state (R31)
SEG = 10

ALG_DOUBLES = {
    3: {"s1_rhs_xsweep": 13, "sweep_y": 6, "sweep_z": 9, "div_psi_first": 9, "psi_y": 2, "psi_x_p": 4},
    2: {"s1_rhs_xsweep": 9, "sweep_y": 6, "div_psi_first": 7, "psi_x_p": 4},
}


def alg_doubles(dim, n, world=1):
    """Per-phase doubles per cell for this grid: 3D grids of N >= 256 hand D.u^n from S1
    to the first psi pass (S1 writes one more field, the psi pass reads it instead of the
    three u^n components), on one GPU and on z-slabs alike."""
    a = dict(ALG_DOUBLES[dim])
    if dim == 3 and n >= 256:
        a["s1_rhs_xsweep"], a["div_psi_first"] = 14, 7
    return a


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs[2]/[3] extra lines")
    ap.add_argument("--dry-run", action="store_true", help="launch plumbing only: print each rank's view, exit")
    return ap.parse_args()


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "utilization.gpu"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        # the timed region must not start before nvidia-smi is actually sampling
        t0 = time.time()
        while self.proc is not None and not self.lines and time.time() - t0 < 10.0:
            time.sleep(0.02)
        self.n0 = len(self.lines)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        time.sleep(0.1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, smax, reasons, util, allsm = [], [], set(), [], []
        for l in self.lines[getattr(self, "n0", 0):]:     # samples taken during the timed region
            parts = [x.strip() for x in l.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            u = float(parts[6]) if parts[6].replace(".", "").isdigit() else 0.0
            util.append(u)
            allsm.append(s)
            if u > 0:
                sm.append(s)
            smax.append(m)
            for nm, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        # utilization.gpu is a trailing average and can read 0 in a short region: then
        # every sample of the region counts
        use = sm if sm else allsm
        return {"sm_mhz": statistics.median(use) if use else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(allsm), "samples_under_load": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def arm_config(pr, cfg_idx, world):
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": f"configs[{cfg_idx}]", "grid": f"{pr.n}^{pr.dim}", "ib_points": pr.npts,
            "ib_edges": int(pr.edges.shape[0]) if pr.edges is not None else 0, "mu": pr.mu, "rho": pr.rho, "dt": pr.dt,
            "delta_kernel": "cos4" if pr.kernel == 0 else "peskin4",
            "parallelism": "single-gpu" if world == 1 else f"zslab{world}-nccl",
            "l2": ("inputs larger than L2 (14 resident fp64 fields), no flush"
                   if pr.ncell * 8 * (4 * pr.dim + 2) > 126e6 else
                   "working set fits in L2 (no flush): a latency-bound parity config, not a roofline case")}


def max_over_ranks(x: float) -> float:
    """Max of a per-rank scalar over all ranks (the slowest rank's time); identity
    without a process group.  Uses a CUDA tensor on NCCL, a CPU tensor on gloo."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(cfg):
    """The oracle as it stands, single-threaded, on a bounded sample of the same
    workload: whole time steps (the oracle's unit of work), one untimed step first when
    a step is short; a config-4 step (~1 min) is timed alone."""
    from oracle import oracle as O
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(cfg)
    o = O.Oracle(pr.dim, pr.n, pr.mu, pr.rho, pr.dt, chi=pr.chi, kernel=pr.kernel)
    o.set_fields(*pr.u, p=pr.p) if pr.dim == 3 else o.set_fields(pr.u[0], pr.u[1], None, pr.p)
    o.set_boundary(pr.X, pr.edges, pr.kappa, rest=pr.rest, weight=pr.weight)
    big = pr.ncell > 4_000_000
    steps = 1 if big else 2
    if not big:
        o.step(1)
    t0 = time.perf_counter()
    o.step(steps)
    dt = time.perf_counter() - t0
    return {"value": pr.ncell * steps / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} full oracle time step(s) of configs[{cfg}] ({pr.n}^{pr.dim} cells, "
                      f"{pr.npts} IB points){'' if big else ' after 1 untimed step'}; single-threaded C "
                      f"(oracle/ibgm_oracle.c)",
            "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) timed on the host."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1305_3976_b200 import inputs
    pr = inputs.config(args.config)
    o = O.Oracle(pr.dim, pr.n, pr.mu, pr.rho, pr.dt, chi=pr.chi, kernel=pr.kernel)
    o.set_fields(*pr.u, p=pr.p) if pr.dim == 3 else o.set_fields(pr.u[0], pr.u[1], None, pr.p)
    o.set_boundary(pr.X, pr.edges, pr.kappa, rest=pr.rest, weight=pr.weight)
    t0 = time.perf_counter()
    o.step(1)                       # first step (the oracle has no warm-up effects)
    t1 = time.perf_counter() - t0
    budget = 150.0                  # keep the whole run within a few minutes
    if t1 > 20.0:
        # a long step (config 4: ~1 min) is itself the bounded sample
        k, dt, warm = 1, t1, 0
    else:
        k = max(1, min(args.steps, int(budget / max(t1, 1e-3))))
        t0 = time.perf_counter()
        o.step(k)
        dt = time.perf_counter() - t0
        warm = 1
    v = pr.ncell * k / dt
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": k, "warmup": warm, "ms_per_step": 1e3 * dt / k, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": arm_config(pr, args.config, world),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{k} of the requested {args.steps} oracle steps (bounded to ~{budget:.0f} s)"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: start N ranks on this node with
    torch.distributed.run (127.0.0.1 rendezvous) and return their exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print("bench.py: relaunching under torchrun:", " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def measure(ibgm, inputs, torch, cfg, steps, warmup, rank, world, local, stream, keep_ctx=False, clock=None):
    """Time `steps` graph-replayed steps of configs[cfg] (device time on the library's
    stream, max over ranks), then the same steps with per-phase event pairs for the
    roofline attribution.  Returns (record, ctx or None, problem)."""
    pr = inputs.config(cfg)
    if world > 1:
        # z-slab decomposition over the ranks: NCCL transport, the
        # unique id broadcast over the process group
        nccl_id = ibgm.share_nccl_id()
        ctx = ibgm.from_problem(pr, device=local, stream=stream.cuda_stream, nranks=world, rank=rank,
                                nccl_id=nccl_id)
        print(f"bench.py: rank {rank}/{world} NCCL communicator up (configs[{cfg}], slab of {pr.n // world} planes)",
              file=sys.stderr, flush=True)
    else:
        ctx = ibgm.from_problem(pr, device=local, stream=stream.cuda_stream)
    dim = pr.dim
    ncl = pr.ncell // world          # cells this rank holds

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # Every run of steps starts from one base state (2 steps after the initial data, so
    # the AB2 histories and the IB look-ahead are live) and lasts at most SEG steps:
    # configs[4]'s (sigma, mu, dt, h) lie beyond the explicit IB coupling's time-step
    # restriction (R31) -- its membranes blow up
    # after ~110 steps -- so long runs are cut into segments of real steps that all stay
    # finite.  The restore (ib_set_state, H2D from pinned memory) is outside the timed
    # segments; the timed value is the sum of the segments' device times.
    nb = ctx.state_size()
    base = torch.empty(nb, dtype=torch.uint8, pin_memory=True).numpy()
    ctx.step(2)
    ctx.get_state(base)

    def segments(k):
        out, left = [], k
        while left > 0:
            out.append(min(SEG, left))
            left -= out[-1]
        return out

    for m in segments(warmup):
        ctx.set_state(base)
        ctx.step(m)
    ctx.sync()
    torch.cuda.synchronize()

    # --- timed region A: K steps, device time between event pairs on the library's stream
    l0 = ctx.stats()["kernel_launches"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local) if clock else None
    if clk:
        clk.__enter__()
    tot_ms = 0.0
    restores = 0
    for m in segments(steps):
        ctx.set_state(base)              # untimed: back to the base state
        restores += 1
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.step(m)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        tot_ms += e0.elapsed_time(e1)
    if clk:
        clk.__exit__()
    ctx.sync()                       # also surfaces any device-raised fault
    ms = max_over_ranks(tot_ms)
    launches = ctx.stats()["kernel_launches"] - l0
    # every step updates the whole N^d grid (each rank its slab): strong scaling
    value = float(pr.ncell) * steps / (ms * 1e-3)

    # --- timed region B: the same steps with per-phase event pairs (roofline attribution)
    ctx.set_profiling(True)
    kb = max(10, min(steps, 200))
    for m in segments(kb):
        ctx.set_state(base)
        ctx.step(m)
    ctx.sync()
    ph = ctx.phase_times()
    ctx.set_profiling(False)
    tot_ph = sum(v[0] for v in ph.values())
    AD = alg_doubles(dim, pr.n, world)
    dom = max((k for k in ph if k in AD), key=lambda k: ph[k][0])
    dom_ms = ph[dom][0] / ph[dom][1]
    alg = AD[dom] * 8 * ncl
    peak, peak_src = measured_peaks()
    achieved = alg / (dom_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_cfg{cfg}.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom)
    step_alg = sum(AD[k] for k in AD if k in ph) * 8 * ncl
    phases = {k: {"ms": round(v[0] / v[1], 5), "share": round(v[0] / tot_ph, 4),
                  "alg_gbs": (round(AD[k] * 8 * ncl / (v[0] / v[1] * 1e-3) / 1e9, 1)
                              if k in AD else None),
                  "frac": (round(AD[k] * 8 * ncl / (v[0] / v[1] * 1e-3) / 1e9 / peak, 3)
                           if k in AD else None)} for k, v in ph.items()}
    rec = {"value": value, "unit": UNIT, "ms_per_step": ms / steps, "steps": steps, "warmup": warmup,
           "config": arm_config(pr, cfg, world),
           "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "traffic": traffic,
                        "alg_bytes_per_launch": alg, "peak_source": peak_src,
                        "step_frac": step_alg / (ms / steps * 1e-3) / 1e9 / peak},
           "phases": phases, "gpu_launches": launches,
           "segments": {"steps_per_segment": SEG, "segments": restores,
                        "note": "each segment = up to SEG real steps from one base state (2 steps after the initial "
                                "data), restored untimed by ib_set_state between segments (DESIGN.md R31)"}}
    if clk:
        rec["clocks"] = clk.summary()
    if keep_ctx:
        return rec, ctx, pr, base
    ctx.close()
    return rec, None, pr, None


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.dry_run:
        # launch plumbing only (CPU test of the relaunch): report what this rank sees
        print(json.dumps({"dry_run": True, "impl": args.impl, "rank": rank, "world_size": world,
                          "local_rank": local, "gpus": args.gpus}), flush=True)
        return
    if args.impl == "reference":
        return run_reference(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    from paper_1305_3976_b200 import ibgm, inputs
    # a dedicated (non-default) stream: the library enqueues every kernel on it and the
    # timing events are recorded on the same stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0

    head, ctx, pr, base = measure(ibgm, inputs, torch, args.config, args.steps, args.warmup, rank, world, local, stream,
                            keep_ctx=True, clock=True)
    dim = pr.dim

    # --- e2e through the public API with pinned host buffers: every step uploads the
    # complete solver state (ib_set_state: u, the momentum history, p, p*, X, U -- what
    # the next step reads), advances one step and downloads the new state (ib_get_state),
    # so each e2e step is exactly a regular step of the time integration
    e2e = None
    if not args.no_e2e:
        nb = ctx.state_size()
        blob = base                      # start from the base state of the timed region
        ke = max(3, min(args.steps, SEG - 1))
        ctx.set_state(blob)
        ctx.step(1)
        ctx.get_state(blob)              # untimed warm-up of the copy path
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(ke):
            ctx.set_state(blob)          # H2D of the step's inputs (the state)
            ctx.step(1)
            ctx.get_state(blob)          # D2H of the step's result (the new state)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": float(pr.ncell) * ke / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "steps": ke,
               "note": "per step: ib_set_state (H2D of the full solver state from pinned memory) + ib_step(1) + "
                       "ib_get_state (D2H of the new state to pinned memory); bytes per rank"}
    ctx.close()

    # --- the other 2D/3D configurations as extra lines (north_star: 2D and 3D numbers)
    extra = {}
    if not args.no_extra:
        for c in (2, 3):
            if c == args.config:
                continue
            rec, _, _, _ = measure(ibgm, inputs, torch, c, max(20, min(args.steps, 200)), max(3, args.warmup), rank,
                                world, local, stream)
            extra[f"configs[{c}]"] = rec

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config)

    if rank == 0:
        out = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": head["config"],
            "roofline": head["roofline"],
            "phases": head["phases"],
            "gpu_launches": head["gpu_launches"],
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": head["clocks"],
            "extra": extra,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
