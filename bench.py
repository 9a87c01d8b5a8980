"""Benchmark: MG-PCG DoF-iterations/s on B200 (fp64), BASELINE configs[1] workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

A *step* is one full PCG solve (x0 = 0, tol 1e-8, one V(1,1) cycle per
iteration as preconditioner) on the configuration's finest system.
  value  = sum over ranks of N_dofs * its / (max over ranks of the mean device time per step),
           inputs resident in HBM (igb_pcg_device), CUDA events on the library stream,
           L2 flushed (256 MiB write) before every step;
  e2e    = same metric through the public host API (Context.pcg: pinned-host b -> device,
           solve, x -> host), wall clock per step;
  roofline = dominant kernel class from a separate profiled pass (CUDA events around every
           launch, same K steps) -> algorithmic bytes / mean launch time vs MEASURED_PEAKS.json;
  cpu_baseline = oracle/ (reference-faithful NumPy/SciPy restatement) on a bounded sample.
Multi-GPU (torchrun): independent replicas per GPU (the solve does not shard),
weak scaling, NCCL only for the barrier and the max-over-ranks reduction.
--impl reference: the reference-faithful CPU solve (oracle port; the reference itself is pure
Python and does not travel to the GPU box) on rank 0 with all host threads.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_CLASS_PEAK = "hbm_gbs"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--levels", type=int, default=None)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def max_over_ranks(x, dist=None, device=None):
    """Max of a scalar over all ranks (NCCL on GPU, gloo on CPU); identity when single-process."""
    if dist is None or not dist.is_initialized():
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(world, n_dofs, its, ms_per_step):
    """Whole-job DoF*iterations/s of `world` independent replicas timed by the slowest rank."""
    return world * n_dofs * its / (ms_per_step / 1e3)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_problem(args):
    from paper_1902_01818_b200 import configs, multigrid
    kw = {}
    if args.levels is not None:
        kw["levels"] = args.levels
    if args.p is not None and args.config == "cfg4":
        kw["p"] = args.p
    t = time.perf_counter()
    pr = configs.build(args.config, **kw)
    setup = multigrid.MultigridSetup(pr.hier, pr.config)
    f = pr.rhs(setup.assembled_finest)
    return pr, setup, f, time.perf_counter() - t


def workload_desc(args, pr, setup):
    d = {"workload": f"{args.config}" + (f"_p{args.p}" if args.p else "") +
         (f"_L{args.levels}" if args.levels else ""),
         "n_dofs": int(setup.n_dofs), "levels": int(pr.hier.L), "degree": int(pr.hier.p),
         "patches": int(pr.hier.domain.num_patches), "dim": int(pr.hier.dim),
         "mode": pr.hier.mode, "smoother": pr.config.smoother, "tol": pr.config.tol,
         "nnz_finest": int(setup.A[setup.finest].nnz)}
    return d


class ClockSampler:
    """nvidia-smi sampling during the timed region (SM clock, throttle reasons)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def cpu_oracle_rate(setup, f, seconds, threads):
    """Reference-faithful CPU solve (oracle port) repeated for ~`seconds`: DoF*its/s."""
    from threadpoolctl import threadpool_limits
    from oracle.solve import OracleSolver
    with threadpool_limits(limits=threads):
        orc = OracleSolver(setup.setup_bundle())
        n = setup.n_dofs
        total_dofit, total_t, runs, its = 0.0, 0.0, 0, 0
        while True:
            t = time.perf_counter()
            _, its, _ = orc.solve(f, tol=setup.config.tol, max_iters=setup.config.max_iters)
            dt = time.perf_counter() - t
            total_dofit += n * its
            total_t += dt
            runs += 1
            if total_t >= seconds or runs >= 50:
                break
    return total_dofit / total_t, runs, its, total_t


def run_reference(args, rank, world):
    if rank != 0:
        return
    pr, setup, f, t_setup = build_problem(args)
    cores = len(os.sched_getaffinity(0))
    from threadpoolctl import threadpool_limits
    from oracle.solve import OracleSolver
    with threadpool_limits(limits=cores):
        orc = OracleSolver(setup.setup_bundle())
        for _ in range(args.warmup):
            orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
        times, its = [], 0
        for _ in range(args.steps):
            t = time.perf_counter()
            _, its, _ = orc.solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)
            times.append(time.perf_counter() - t)
    ms = 1e3 * float(np.mean(times))
    value = setup.n_dofs * its / (ms / 1e3)
    line = {
        "metric": "MG-PCG DoF*iterations/s", "value": value, "unit": "DoF*it/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic geometry + source, SURVEY 8d)",
        "config": dict(workload_desc(args, pr, setup), iterations=its, setup_s=round(t_setup, 2)),
        "cpu_baseline": {"value": value, "unit": "DoF*it/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full PCG solves of {args.config} (oracle/solve.py, "
                                   f"reference-faithful SciPy/NumPy restatement), {cores} BLAS threads"},
        "e2e": {"value": value, "unit": "DoF*it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    dist = None
    # IGB_BENCH_ONE_GPU=1: functional test of the multi-rank path on a one-GPU box (every rank on
    # device 0, gloo for the barrier / max reduction); its numbers are not a scaling measurement
    one_gpu = os.environ.get("IGB_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    red_dev = "cpu" if one_gpu else f"cuda:{local}"
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1902_01818_b200 import multigrid

    pr, setup, f, t_setup = build_problem(args)
    solver = multigrid.MultigridSolver(pr.hier, pr.config, device=local, setup=setup)
    ctx = solver.ctx
    n = solver.n_dofs
    cfg = pr.config
    d_b = ctx.device_alloc(8 * n)
    d_x = ctx.device_alloc(8 * n)
    ctx.h2d(d_b, f)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MiB

    def l2_flush():
        flush.fill_(1.0)
        torch.cuda.synchronize(local)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(local)

    for _ in range(args.warmup):
        l2_flush()
        its, hist = ctx.pcg_device(d_b, d_x, cfg.tol, cfg.max_iters)

    # ---- timed region: device-resident inputs, CUDA-event time per solve
    dev_ms = []
    ctx.launch_count(reset=True)
    barrier()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            l2_flush()
            its, hist = ctx.pcg_device(d_b, d_x, cfg.tol, cfg.max_iters)
            dev_ms.append(ctx.last_timing()[0])
    barrier()
    launches = ctx.launch_count(reset=True)
    ms = max_over_ranks(float(np.mean(dev_ms)), dist, red_dev)
    value = replica_value(world, n, its, ms)

    # ---- e2e: public host API (H2D of b from pinned host memory, solve, D2H of x + history into
    # host memory), wall clock
    fh = ctx.pinned(n)
    fh[:] = f
    xh = ctx.pinned(n)
    for _ in range(args.warmup):  # the host-buffer entry point has its own solve graph: warm it too
        l2_flush()
        solver.ctx.pcg(fh, cfg.tol, cfg.max_iters, out=xh)
    e2e_s = []
    for _ in range(max(1, args.steps)):
        l2_flush()
        barrier()
        t = time.perf_counter()
        x, its_e, hist_e = solver.ctx.pcg(fh, cfg.tol, cfg.max_iters, out=xh)
        e2e_s.append(time.perf_counter() - t)
    e2e_t = max_over_ranks(float(np.mean(e2e_s)), dist, red_dev)
    e2e = {"value": replica_value(world, n, its_e, 1e3 * e2e_t), "unit": "DoF*it/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n + 8 * its_e}

    # ---- profiled pass (separate): per-kernel-class CUDA-event times
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(args.steps):
        l2_flush()
        ctx.pcg_device(d_b, d_x, cfg.tol, cfg.max_iters)
    prof = ctx.profile_get()
    ctx.profile(False)
    peaks, peak_kind = measured_peaks()
    dom = max(prof, key=lambda k: prof[k]["ms"])
    P = prof[dom]
    mean_launch_s = P["ms"] / 1e3 / max(1, P["launches"])
    bytes_per_launch = P["bytes"] / max(1, P["launches"])
    achieved = bytes_per_launch / mean_launch_s / 1e9 if mean_launch_s > 0 else 0.0
    traffic, traffic_src = None, None
    tp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    if os.path.exists(tp) and args.config == "cfg2":  # committed ncu capture of the same workload
        t = json.load(open(tp)).get(dom)
        if t:
            traffic, traffic_src = t["bytes_per_launch"], t["source"]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "peak_source": peak_kind,
                "note": "algorithmic bytes per launch / mean CUDA-event launch time, profiled pass",
                "classes": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                                "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else 0.0}
                            for k, v in prof.items()}}

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            rate, runs, cits, tt = cpu_oracle_rate(setup, f, args.cpu_sample_seconds, 1)
            cpu = {"value": rate, "unit": "DoF*it/s", "cores": 1, "kind": "port",
                   "sample": f"{runs} full PCG solves of {args.config} ({tt:.1f} s), oracle/solve.py, 1 thread"}
        out = {
            "metric": "MG-PCG DoF*iterations/s", "value": value, "unit": "DoF*it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic geometry + source, SURVEY 8d)",
            "config": dict(workload_desc(args, pr, setup), iterations=its, l2="flushed (256 MiB write) before every step",
                           setup_s=round(t_setup, 2), upload_s=round(solver.setup_timings["upload"], 2),
                           parallelism=f"replicas x{world}"),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "gpu_launches": int(launches), "clocks": clocks.summary(),
            "final_rel_residual": hist[-1] if hist else None,
        }
        print(json.dumps(out), flush=True)
    solver.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
