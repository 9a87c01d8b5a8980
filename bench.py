"""Benchmark: MG-PCG DoF-iterations/s on B200 (fp64), BASELINE configs[4] workload (cfg5, full size).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg5]

Workload: BASELINE.json names no single config for the metric, so the N=1 line uses the largest
configuration that fits one GPU: configs[4] = cfg5 (2x2x2 unit cubes, p = 3, 64^3 spans per patch,
N = 2,248,091 DoFs, 726.6M nonzeros, 5 levels, hybrid smoother).  The other configs are parity
cases (tests/), selectable here with --config for reference.
A *step* is one full PCG solve (x0 = 0, tol 1e-8, one V(1,1) cycle per
iteration as preconditioner) on the configuration's finest system; the iteration count is
checked against the reference's (EXPECTED_ITS) and the line fails on a mismatch.
  value  = sum over ranks of N_dofs * its / (max over ranks of the mean device time per step),
           inputs resident in HBM (igb_pcg_device), CUDA events on the library stream,
           L2 flushed (256 MiB write) before every step;
  e2e    = same metric through the public host API (Context.pcg: pinned-host b -> device,
           solve, x -> host), wall clock per step;
  roofline = dominant kernel class from a separate profiled pass (CUDA events around every
           launch, same K steps): the class's largest launch (the finest-level kernel,
           igb_profile_top) -> its algorithmic bytes / its mean time vs MEASURED_PEAKS.json, and
           traffic = the DRAM bytes ncu shows for the same launch (profiles/traffic.json);
  roofline_fd = the fast-diagonalisation class's flops / time vs the measured fp64 DGEMM peak
           (profiles/r2_fp64_peak.json; MEASURED_PEAKS.json has no fp64 entry);
  cpu_baseline = oracle/ (reference-faithful NumPy/SciPy restatement) on a bounded sample.
Multi-GPU (torchrun): independent replicas per GPU (the solve does not shard),
weak scaling, NCCL only for the barrier and the max-over-ranks reduction.
--impl reference: the reference-faithful CPU solve (oracle port; the reference itself is pure
Python and does not travel to the GPU box) on rank 0 with all host threads.  On the large
configurations (cfg4, cfg5) one CPU solve takes minutes, so a reference step is a bounded sample:
ONE PCG iteration of the same solve (SpMV A d, the CG vector updates and one V(1,1) hybrid cycle
on the full hierarchy); value = N / (mean seconds per iteration), the same DoF*it/s unit.
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
# reference iteration counts (tests/golden from igamg; cfg4 p=6/8 and cfg5 at full size from the oracle,
# tests/test_fullsize.py) at the default level counts
EXPECTED_ITS = {"cfg1": 8, "cfg2": 6, "cfg3": 12, "cfg4_p2": 5, "cfg4_p4": 7, "cfg4_p6": 9, "cfg4_p8": 11,
                "cfg5": 6}
LARGE = ("cfg4", "cfg5")  # one CPU solve takes minutes: reference steps are single PCG iterations


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--levels", type=int, default=None)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step", default="auto", choices=["auto", "solve", "iteration"])
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


def workload_name(args):
    return f"{args.config}" + (f"_p{args.p}" if args.p else "") + (f"_L{args.levels}" if args.levels else "")


def workload_desc(args, pr, setup, its):
    """The `config` dict -- identical key set and values in both arms."""
    return {"workload": workload_name(args),
            "n_dofs": int(setup.n_dofs), "levels": int(pr.hier.L), "degree": int(pr.hier.p),
            "patches": int(pr.hier.domain.num_patches), "dim": int(pr.hier.dim),
            "mode": pr.hier.mode, "smoother": pr.config.smoother, "tol": pr.config.tol,
            "nnz_finest": int(setup.A[setup.finest].nnz), "iterations": int(its),
            "parallelism": "replicas (one independent solve per GPU)"}


def check_its(args, its):
    """Fail the line when the iteration count differs from the reference's (a smoother defect that
    weakens the preconditioner would raise `its` and with it the DoF*it/s figure)."""
    key = workload_name(args)
    if args.levels is None and key in EXPECTED_ITS and its != EXPECTED_ITS[key]:
        raise SystemExit(f"bench: {key} took {its} PCG iterations, the reference takes {EXPECTED_ITS[key]}")


class OracleCgStepper:
    """One PCG iteration of oracle.solve.cg (reference linsolve.py:83-100) per step: A d, the dots
    and updates, and one cycle as preconditioner on the full hierarchy; restarts from x = 0 when
    the solve converges (the restart is not timed)."""

    def __init__(self, orc, b, tol):
        self.orc, self.b, self.tol = orc, np.asarray(b, dtype=float), tol
        self.A = orc.A[orc.finest]
        self.normb = np.linalg.norm(self.b)
        self.restart()

    def restart(self):
        self.x = np.zeros_like(self.b)
        self.r = self.b.copy()
        self.z = self.orc.cycle(self.orc.finest, self.r)
        self.d = self.z.copy()
        self.rz = self.r @ self.z
        self.done = False

    def step(self):
        if self.done:
            self.restart()
        t = time.perf_counter()
        Ad = self.A @ self.d
        alpha = self.rz / (self.d @ Ad)
        self.x += alpha * self.d
        self.r -= alpha * Ad
        rel = np.linalg.norm(self.r) / self.normb
        self.z = self.orc.cycle(self.orc.finest, self.r)
        rz_new = self.r @ self.z
        beta = rz_new / self.rz
        self.rz = rz_new
        self.d = self.z + beta * self.d
        dt = time.perf_counter() - t
        self.done = rel <= self.tol
        return dt


def ref_mode(args):
    if args.ref_step != "auto":
        return args.ref_step
    return "iteration" if args.config in LARGE and args.levels is None else "solve"


def cpu_rate(setup, f, seconds, threads, mode, warmup=1, steps=None):
    """Reference-faithful CPU solve (oracle port) on `threads` host threads: DoF*it/s.
    mode "solve": whole PCG solves; "iteration": single PCG iterations (OracleCgStepper).
    Runs `steps` timed steps, or until ~`seconds` of timed work."""
    from threadpoolctl import threadpool_limits
    from oracle.solve import OracleSolver
    with threadpool_limits(limits=threads):
        orc = OracleSolver(setup.setup_bundle())
        n = setup.n_dofs
        tol, mi = setup.config.tol, setup.config.max_iters
        if mode == "iteration":
            st = OracleCgStepper(orc, f, tol)
            for _ in range(warmup):
                st.step()
            times = []
            while (steps is None and (sum(times) < seconds or not times)) or (steps is not None and len(times) < steps):
                times.append(st.step())
            return n / float(np.mean(times)), times, 1
        for _ in range(warmup):
            orc.solve(f, tol=tol, max_iters=mi)
        times, its = [], 0
        while (steps is None and (sum(times) < seconds or not times) and len(times) < 50) or \
                (steps is not None and len(times) < steps):
            t = time.perf_counter()
            _, its, _ = orc.solve(f, tol=tol, max_iters=mi)
            times.append(time.perf_counter() - t)
        return n * its / float(np.mean(times)), times, its


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


def fp64_peak_tflops():
    """Measured fp64 DGEMM peak (tools/fp64_peak.py on this pool's B200: profiles/r2_fp64_peak.json)."""
    d, _ = measured_peaks()
    if "fp64_tflops" in d:
        return float(d["fp64_tflops"]), "MEASURED_PEAKS.json"
    try:
        with open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")) as fh:
            return float(json.load(fh)["fp64_tflops"]), "measured (profiles/r2_fp64_peak.json, cuBLAS DGEMM 8192^3)"
    except Exception:
        return 37.0, "fallback (B200 nominal fp64)"


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def run_reference(args, rank, world):
    if rank != 0:
        return
    pr, setup, f, t_setup = build_problem(args)
    cores = len(os.sched_getaffinity(0))
    mode = ref_mode(args)
    value, times, its = cpu_rate(setup, f, 0.0, cores, mode, warmup=args.warmup, steps=args.steps)
    if mode == "iteration":
        its = EXPECTED_ITS.get(workload_name(args))
        if its is None:  # reduced configurations only (full sizes are in EXPECTED_ITS): count once
            from oracle.solve import OracleSolver
            its = OracleSolver(setup.setup_bundle()).solve(f, tol=pr.config.tol, max_iters=pr.config.max_iters)[1]
        sample = (f"{args.steps} single PCG iterations (A d + CG updates + one V(1,1) hybrid cycle on the full "
                  f"{workload_name(args)} hierarchy), oracle/solve.py (reference-faithful SciPy/NumPy restatement; "
                  f"GS sweeps as C substitution where splu(tril) does not fit), {cores} BLAS threads")
    else:
        sample = (f"{args.steps} full PCG solves of {workload_name(args)} (oracle/solve.py, reference-faithful "
                  f"SciPy/NumPy restatement), {cores} BLAS threads")
    ms = 1e3 * float(np.mean(times))
    line = {
        "metric": "MG-PCG DoF*iterations/s", "value": value, "unit": "DoF*it/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic geometry + source, SURVEY 8d)",
        "config": workload_desc(args, pr, setup, its),
        "step": mode, "setup_s": round(t_setup, 2),
        "cpu_baseline": {"value": value, "unit": "DoF*it/s", "cores": cores, "kind": "port", "sample": sample},
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
    check_its(args, its)

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
    # the dominant class's largest launch (the finest level's kernel): the same launch the committed
    # ncu --set full capture shows, so `achieved`, `traffic` and the algorithmic bytes refer to one thing
    T = P["top"]
    mean_launch_s = T["ms"] / 1e3 / max(1, T["launches"])
    bytes_per_launch = T["bytes_per_launch"]
    achieved = bytes_per_launch / mean_launch_s / 1e9 if mean_launch_s > 0 else 0.0
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):  # committed ncu --set full capture of the same workload's dominant kernel
        t = json.load(open(tp)).get(workload_name(args), {}).get(dom)
        if t:
            traffic, traffic_src = t["bytes_per_launch"], t["source"]
    classes = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                   "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else 0.0}
               for k, v in prof.items()}
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "peak_source": peak_kind,
                "launch": f"largest launch of class {dom} (finest level), {T['launches'] / args.steps:.0f} per step, "
                          f"{1e3 * mean_launch_s:.3f} ms each",
                "note": "algorithmic bytes of that launch / its mean CUDA-event time, profiled pass "
                        "(events around every launch, outside the graph); traffic = ncu DRAM bytes of the same launch",
                "classes": classes}
    # fast diagonalisation: fp64 flops / time against the measured DGEMM peak
    fd = prof.get("fd", {})
    fp64_peak, fp64_src = fp64_peak_tflops()
    if fd.get("ms", 0) > 0 and fd.get("flops", 0) > 0:
        tf = fd["flops"] / (fd["ms"] / 1e3) / 1e12
        roofline_fd = {"bound": "fp64", "kernel": "fd", "achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s",
                       "frac": tf / fp64_peak, "flops_per_step": fd["flops"] / args.steps,
                       "ms_per_step": fd["ms"] / args.steps, "peak_source": fp64_src}
    else:
        roofline_fd = None

    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cores = len(os.sched_getaffinity(0))
            mode = ref_mode(args)
            rate, times, cits = cpu_rate(setup, f, args.cpu_sample_seconds, cores, mode, warmup=0)
            what = "single PCG iterations (A d + CG updates + one V(1,1) cycle)" if mode == "iteration" \
                else "full PCG solves"
            cpu = {"value": rate, "unit": "DoF*it/s", "cores": cores, "kind": "port",
                   "sample": f"{len(times)} {what} of {workload_name(args)} ({sum(times):.1f} s), oracle/solve.py, "
                             f"{cores} BLAS threads (SpMV / substitution single-threaded as in SciPy)"}
        out = {
            "metric": "MG-PCG DoF*iterations/s", "value": value, "unit": "DoF*it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic geometry + source, SURVEY 8d)",
            "config": workload_desc(args, pr, setup, its),
            "l2": "inputs (8.7 GB of matrices) exceed L2; also flushed (256 MiB write) before every step",
            "setup_s": round(t_setup, 2), "upload_s": round(solver.setup_timings["upload"], 2),
            "e2e": e2e, "roofline": roofline, "roofline_fd": roofline_fd, "cpu_baseline": cpu,
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
