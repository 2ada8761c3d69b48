#!/usr/bin/env python
"""Benchmark of the iterated stochastic Magnus hot path (arXiv 2207.09776) on B200.

Workload (BASELINE.json configs[1]): constant-coefficient Langevin
SPDE on a 256x256 (x, v) grid, 16384 Brownian paths per GPU, order-3 iterated Magnus
with 100 windows (dt = 0.01, T = 1, dt_leb = 1e-4), expmv tol 1e-10, theta 1.
One "step" = one Magnus window (one subinterval) of every path; the metric is
path*gridpoint*windows/s (BASELINE's "path*gridpoint*steps/s" for Magnus).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Synthetic data: Philox-generated Brownian paths (counter = global path id, Lebesgue step),
Gaussian datum phi.  The per-GPU state (4 x 16384 x 256^2 fp64 = 34 GB) is far larger
than L2, so no explicit L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

A_LANGEVIN = 1.1
SIGMA = 1.0 / np.sqrt(10.0)
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
# Magnus engines (s2b_magnus_stats.engine) -> dominant kernel and its ncu summary in profiles/
ENGINES = {
    3: {"name": "cluster-xmi", "kernel": "cluster_xmi_kernel", "profile": "xmi_kernel_ncu.json",
        "note": "cluster-resident in-place x-march (16-CTA clusters, accumulator in L2): achieved is the "
                "streaming-equivalent rate, traffic the real DRAM bytes; bound by the fp64 pipe; by default "
                "25% of the paths run on the streaming x-march engine (term_xs_kernel) on the idle SMs (S2B_HYBRID)"},
    0: {"name": "stream", "kernel": "term_tma_kernel", "profile": "term_kernel_ncu.json",
        "note": "streaming pass engine: term and accumulator round-trip HBM every Taylor term (constant "
                "Langevin on grids >= 256 columns: the x-march term_xs2_kernel, x-major tiles by TMA, TWO "
                "terms per pass -- 40 B per two terms, so achieved is the 32 B/term streaming-equivalent "
                "rate and traffic the real DRAM bytes)"},
    1: {"name": "cluster-band", "kernel": "cluster_magnus_kernel", "profile": "cluster_kernel_ncu.json",
        "note": "cluster-resident: the path stays in shared memory for the window; achieved is the "
                "streaming-equivalent rate (can exceed HBM peak), traffic the real DRAM bytes"},
    2: {"name": "cluster-xm", "kernel": "cluster_xm_kernel", "profile": "xm_kernel_ncu.json",
        "note": "cluster-resident x-march: the path stays in shared memory for the window; achieved is "
                "the streaming-equivalent rate (can exceed HBM peak), traffic the real DRAM bytes; the "
                "binding limit is the fp64 pipe (compute_roofline); by default 16% of the paths run on "
                "the streaming engine concurrently, on the SMs the 8-CTA clusters leave idle (S2B_HYBRID)"},
}


def stencil_points(order):
    """Union stencil of the constant Langevin family."""
    return {1: 5, 2: 11, 3: 19}[order]


def fp64_peak_tops():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["dmul_dadd_tops"])
    except Exception:
        return None


def kinetic_fields(d):
    """Synthetic x- and v-dependent coefficients of the general kinetic SPDE
    du = (a/2 d_vv + v d_x + b d_v + c) u dt + (sigma d_v + beta) u dW (fields gvv, fv, h, sigv,
    sig; transport fx = -v), sampled at the interior nodes a+(i+1)delta, index j*nx+i."""
    delta = 8.0 / (d + 1)
    x = np.array([-4.0 + (i + 1) * delta for i in range(d)])
    X, V = np.meshgrid(x, x, indexing="xy")
    f = {"h": 0.2 * np.cos(X + 0.3 * V) - 0.1, "fx": -V, "fv": 0.3 * np.sin(X) * np.cos(V),
         "gvv": 1.1 * (1.0 + 1.0 / (X * X + V * V + 1.0)), "sig": 0.1 * np.cos(V + X),
         "sigv": 0.3 * np.sqrt(1.0 + 1.0 / (X * X + 1.0 + 0.1 * V * V))}
    return {k: np.ascontiguousarray(a.reshape(-1)) for k, a in f.items()}


def family_args(args):
    """(family name for the library / oracle, extra keyword arguments)"""
    if args.family == "kinetic-variable":
        return "fields", {"fields": kinetic_fields(args.d)}
    return args.family, {"a": A_LANGEVIN, "sigma": SIGMA}


def workload_name(args):
    fam = {"langevin-constant": "constant-coefficient Langevin",
           "langevin-variable": "variable-coefficient Langevin",
           "kinetic-variable": "general kinetic SPDE, x/v-dependent a,b,c,sigma,beta"}[args.family]
    return f"{args.preset}: {fam}"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--paths", type=int, default=16384, help="paths per GPU")
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--family", default="langevin-constant",
                    choices=["langevin-constant", "langevin-variable", "kinetic-variable"],
                    help="coefficient family (cfg3 = langevin-variable; kinetic-variable = the paper's general "
                         "kinetic SPDE with x- and v-dependent a, b, c, sigma, beta)")
    ap.add_argument("--dt", type=float, default=0.01)
    ap.add_argument("--dt-leb", type=float, default=1e-4)
    ap.add_argument("--T", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-north-star", action="store_true", help="skip the cfg4 (512^2) sub-measurement")
    ap.add_argument("--no-tte", action="store_true", help="skip the time-to-accuracy sub-measurement")
    ap.add_argument("--euler-steps", type=int, default=200, help="E-M steps timed beside Magnus (0 = skip)")
    ap.add_argument("--config", default=None, choices=sorted(PRESETS),
                    help="BASELINE.json workload preset (cfg2 is the default workload); explicit flags win")
    args = ap.parse_args()
    args.preset = args.config or "cfg2"
    if args.config:
        given = {a.split("=")[0].lstrip("-").replace("-", "_") for a in sys.argv[1:] if a.startswith("--")}
        for k, v in PRESETS[args.config].items():
            if k not in given:
                setattr(args, k, v)
    return args


# BASELINE.json configs as bench presets (cfg1: the reference's own CPU-runnable case; cfg4: the
# north-star 512^2 grid, Magnus side of the time-to-accuracy comparison).  cfg5's 128k paths over 8 GPUs are 16384 per GPU, far
# beyond one B200 at 1024^2 (4 state vectors x 8 MB per path): they run as independent waves of
# 4096 resident paths (128 GB of state), and one timed step is one window of one wave — every
# wave is the same work, so the wave's rate is the job's rate.  A full T = 1 is hours at 1024^2
# (SURVEY 8(d)): the preset times a fixed handful of windows (dt = 5e-4, dt_leb = 1e-5).
PRESETS = {
    "cfg1": {"d": 64, "paths": 1000, "dt": 0.1, "dt_leb": 1e-4, "T": 1.0, "order": 2,
             "family": "langevin-constant", "steps": 3, "warmup": 3, "euler_steps": 2000},
    "cfg4": {"d": 512, "paths": 4096, "dt": 0.005, "dt_leb": 1e-4, "T": 1.0, "order": 3,
             "family": "langevin-constant"},
    "cfg2": {"d": 256, "paths": 16384, "dt": 0.01, "dt_leb": 1e-4, "T": 1.0, "order": 3,
             "family": "langevin-constant"},
    "cfg3": {"d": 256, "paths": 16384, "dt": 0.01, "dt_leb": 1e-4, "T": 1.0, "order": 3,
             "family": "langevin-variable"},
    # cfg3 taken literally: the general kinetic SPDE with x/v-dependent a, b, c, sigma, beta
    "cfg3k": {"d": 256, "paths": 16384, "dt": 0.01, "dt_leb": 1e-4, "T": 1.0, "order": 3,
              "family": "kinetic-variable"},
    "cfg5": {"d": 1024, "paths": 4096, "dt": 5e-4, "dt_leb": 1e-5, "T": 0.005, "order": 3,
             "family": "langevin-constant", "steps": 3, "warmup": 3, "euler_steps": 100},
}


# ncu captures in profiles/ per (preset, family, engine): bench.py takes `traffic` from one only
# when its recorded mangled kernel name equals the kernel this run launched
PROFILE_OF = {
    ("cfg2", "langevin-constant", "cluster-xm"): "r02_xm_cfg2_ncu.json",
    ("cfg1", "langevin-constant", "cluster-xm"): "r02_xm_cfg1_ncu.json",
    ("cfg4", "langevin-constant", "cluster-xmi"): "r02_xmi_cfg4_ncu.json",
    ("cfg3", "langevin-variable", "stream"): "r02_term_var_cfg3_ncu.json",
    ("cfg3k", "kinetic-variable", "stream"): "r02_term_varx_cfg3k_ncu.json",
    ("cfg5", "langevin-constant", "stream"): "r02_term_xs2_cfg5_ncu.json",
    ("cfg5", "langevin-variable", "stream"): "r02_term_varx_cfg5var_ncu.json",
    ("hybrid", 256): "r02_term_xs_hybrid256_ncu.json",
    ("hybrid", 512): "r02_term_xs_hybrid512_ncu.json",
}
# E-M captures (scripts/prof_r02.sh em_*): per (preset, kernel) of the bench's E-M leg
EM_PROFILE_OF = {("cfg2", "em_cluster_ip_kernel"): "r02_em_cluster_ip_cfg2_ncu.json",
                 ("cfg5", "em_tb_kernel"): "r02_em_tb_cfg5_ncu.json"}


def peaks():
    try:
        with open(MEASURED) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(gpus):
    """One process per GPU.  `--gpus N` without a launcher re-executes this script under
    torch.distributed.run with N local ranks; a world size that differs from --gpus is an error
    (never a silently mislabelled one-GPU number)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        print(json.dumps({"error": f"--gpus {gpus} but WORLD_SIZE={world}"}), file=sys.stderr, flush=True)
        raise SystemExit(2)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        return rank, local, world, dist
    return 0, 0, 1, None


def self_spawn(args):
    """`python bench.py --gpus N` (N > 1, no WORLD_SIZE): run N ranks on this node."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def max_over_ranks(x, dist, local):
    if dist is None:
        return x
    import torch
    t = torch.tensor([float(x)], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


ENGINE_VAR = {"name": "stream", "kernel": "term_var_kernel", "profile": "term_var_ncu.json",
              "note": "streaming pass engine, x-dependent weights: Y folded per point from the source weights "
                      "(streamed through shared memory by TMA, shared by 4 paths) every term; term and "
                      "accumulator round-trip HBM; bound by the fp64 pipe (fold + apply, compute_roofline)"}


def cpu_reference_leg(args, n_paths, windows, reps=1):
    """The reference C++ (oracle/_ref, OpenMP on every host core) on a bounded sample:
    `n_paths` paths over `windows` Magnus windows of the same workload."""
    from oracle import ref
    fam, kw = family_args(args)
    ops = ref.Ops(fam, args.d, order=args.order, **kw)
    T = windows * args.dt
    vals, _ = ref.simulate_brownian(T, args.dt_leb, n_paths, args.seed)
    threads = ref.max_threads()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ops.solve_magnus(vals, args.dt_leb, T, args.dt, order=args.order, threads=0, seed=args.seed)
        times.append(time.perf_counter() - t0)
    return times, threads


CPU_WINDOWS = 3  # windows per CPU sample: the per-call setup (MagnusLogBuilder, ensembles) is amortised


def cpu_setup_estimate(args, M_cpu):
    """Per-call setup of the reference's solve (MagnusLogBuilder union build, ensemble allocation,
    thread start): t(1 window) - (t(3 windows) - t(1 window)) / 2, best of two each."""
    t1 = min(cpu_reference_leg(args, M_cpu, 1, reps=2)[0])
    t3 = min(cpu_reference_leg(args, M_cpu, 3, reps=2)[0])
    per_window = (t3 - t1) / 2.0
    return max(0.0, t1 - per_window), per_window


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    nproc = os.cpu_count() or 1
    n = args.d * args.d
    M_cpu = max(2, nproc)
    times, threads = cpu_reference_leg(args, M_cpu, CPU_WINDOWS, reps=args.warmup + args.steps)
    timed = times[args.warmup:]
    total = sum(timed)
    value = M_cpu * n * CPU_WINDOWS * len(timed) / total
    setup_s, per_window_s = cpu_setup_estimate(args, M_cpu)
    line = {
        "metric": "magnus path*gridpoint*windows/s", "value": value,
        "unit": "path*gridpoint*windows/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference xoshiro256++ Brownian paths, Gaussian datum)",
        "config": {"workload": f"{args.preset} bounded sample: {M_cpu} paths x {CPU_WINDOWS} windows per step, "
                               f"{args.d}x{args.d}, order {args.order}, dt={args.dt}, dt_leb={args.dt_leb}",
                   "grid": args.d, "paths": M_cpu, "order": args.order, "dt": args.dt,
                   "windows_per_step": CPU_WINDOWS},
        "cpu_baseline": {"value": value, "unit": "path*gridpoint*windows/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{M_cpu} paths x {CPU_WINDOWS} windows per step (OpenMP {threads} threads)",
                         "setup_s_per_call": setup_s, "steady_window_s": per_window_s,
                         "steady_value": M_cpu * n / per_window_s if per_window_s > 0 else None},
        "e2e": {"value": value, "unit": "path*gridpoint*windows/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def sass_sha256(mangled):
    """sha256 of one kernel's SASS instructions in the shipped library (cuobjdump -sass -fun):
    the capture-vs-run check that survives rebuilds (-lineinfo embeds source mtimes, so the
    .so bytes change on every rebuild while the machine code does not)."""
    import hashlib
    import re
    import subprocess
    if not mangled:
        return None
    try:
        out = subprocess.run(["cuobjdump", "-sass", "-fun", mangled,
                              os.path.join(ROOT, "paper_2207_09776_b200", "lib", "libspde2d_b200.so")],
                             capture_output=True, text=True, timeout=120).stdout
    except Exception:
        return None
    ins = [ln.split(";")[0].strip() for ln in out.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln)]
    return hashlib.sha256("\n".join(ins).encode()).hexdigest() if ins else None


def lib_sha256():
    import hashlib
    try:
        with open(os.path.join(ROOT, "paper_2207_09776_b200", "lib", "libspde2d_b200.so"), "rb") as fh:
            return hashlib.sha256(fh.read()).hexdigest()
    except Exception:
        return None


def load_profile(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return {}


def magnus_leg(a, s2b, ctx, torch, stream, dist, local, world, rank, keep_session=False):
    """Time a.steps Magnus windows of every path (after a.warmup) through a resident session.
    Returns the measurement (value, ms, roofline, compute roofline, clocks, launches) and, with
    keep_session, the session and paths for the e2e leg."""
    grid = s2b.GridSpec.square(a.d)
    n = grid.dim()
    M = a.paths
    fam, fkw = family_args(a)
    op = s2b.Operator.from_family(grid, fam, **fkw, order=a.order, ctx=ctx)
    paths = s2b.BrownianPaths.philox(a.T, a.dt_leb, M, seed=a.seed, path_offset=rank * M, ctx=ctx)
    phi = s2b.gaussian_datum(grid)
    sess = s2b.MagnusSession(s2b.MagnusConfig(order=a.order, dt=a.dt), op, phi, paths, a.T)
    nwin = int(round(a.T / a.dt))
    if a.warmup + a.steps > nwin:
        raise SystemExit("warmup + steps exceeds the number of windows; raise T or lower steps")
    for _ in range(a.warmup):
        sess.advance(1)
    st0 = sess.stats()
    l0 = ctx.launches
    sess.set_timing(True)
    clocks = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        sess.advance(1)
    e1.record(stream)
    e1.synchronize()
    ctx.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    sess.set_timing(False)
    ms = e0.elapsed_time(e1)
    st1 = sess.stats()
    launches = ctx.launches - l0
    ms_max = max_over_ranks(ms, dist, local)
    value = world * M * n * a.steps / (ms_max / 1e3)

    # roofline of the dominant kernel: algorithmic bytes per Taylor term (32 B per
    # path*gridpoint*term, 24 B for the k=1 term of a segment), over that kernel's event time
    terms = st1["path_terms"] - st0["path_terms"]
    segs = st1["path_segments"] - st0["path_segments"]
    alg_bytes = n * (32.0 * (terms - segs) + 24.0 * segs)
    tk_ms = st1["term_kernel_ms"] - st0["term_kernel_ms"]
    tk_launches = st1["term_launches"] - st0["term_launches"]
    engine = dict(ENGINES.get(st1.get("engine", 0), ENGINES[0]))
    if engine["name"] == "stream" and a.family != "langevin-constant":
        engine = dict(ENGINE_VAR)
        if a.d > 256 or (a.family == "kinetic-variable" and a.order == 3):
            engine["kernel"] = "term_varx_kernel"  # x-split variant: wide grids, 64 source pairs
    names = ctx.kernel_names()
    launched = names["stream"] if engine["name"] == "stream" else names["cluster"]
    for kname in ("term_varx_kernel", "term_var_kernel", "term_generic_k_kernel", "term2_kernel", "term_xs2_kernel",
                  "term_xs_kernel", "term_tma_kernel"):
        if engine["name"] == "stream" and kname in launched:
            engine["kernel"] = kname  # the name of the kernel that actually ran
            break
    hyb = st1.get("hybrid_paths", 0) or 0
    prof_name = PROFILE_OF.get((a.preset, a.family, engine["name"])) or engine["profile"]
    prof = load_profile(prof_name)
    peak, peak_kind = peaks()
    achieved = alg_bytes / (tk_ms / 1e3) / 1e9 if tk_ms > 0 else 0.0
    # traffic only from a capture of the binary that ran: the profile's mangled kernel name
    # must equal the one this session launched (cudaFuncGetName)
    stale = prof.get("kernel_mangled") != launched
    stream_stale = False
    traffic = None
    if not stale:
        if engine["name"] == "stream" and prof.get("dram_bytes_per_path_term") is not None:
            traffic = prof["dram_bytes_per_path_term"] * terms / max(tk_launches, 1)
        elif prof.get("dram_bytes_per_path_window") is not None:
            slice_bytes = 0.0
            if hyb:
                sp = load_profile(PROFILE_OF.get(("hybrid", a.d)) or "none")
                stream_stale = sp.get("kernel_mangled") != names["stream"]
                slice_bytes = None if stream_stale else sp.get("dram_bytes_per_path_term", 0.0) * terms * hyb / M
            if slice_bytes is not None:
                traffic = (prof["dram_bytes_per_path_window"] * (M - hyb) * a.steps + slice_bytes) / max(tk_launches, 1)
    # the on-chip engines are bound by the fp64 pipe, not HBM: report that ceiling beside it
    # (DMUL + DADD per stencil point, no FMA for bitwise parity; +1 DMUL, +1 DADD per point)
    ops_pt = 2 * stencil_points(a.order) + 2
    # + the per-term fold of Y from the source pairs: a DMUL per pair and a DADD per pair after
    # the first of each stencil entry (the fold starts at its first product; term_var.cu)
    if a.family == "langevin-variable":
        ops_pt += 2 * {1: 7, 2: 15, 3: 39}[a.order] - stencil_points(a.order)
    elif a.family == "kinetic-variable":
        npt = {2: 11, 3: 23}.get(a.order, 5)
        ops_pt = 2 * npt + 2 + 2 * {2: 24, 3: 64}.get(a.order, 7) - npt
    fp64_ops = n * terms * float(ops_pt)
    fp64_peak = fp64_peak_tops()
    compute = {"bound": "fp64", "achieved": fp64_ops / (tk_ms / 1e3) / 1e12 if tk_ms > 0 else 0.0,
               "peak": fp64_peak, "unit": "TFLOP/s (DMUL/DADD, non-FMA)",
               "ops_model": f"{ops_pt} fp64 ops per path*gridpoint*term",
               "ncu_fp64_pipe_pct_of_active": None if stale else prof.get("fp64_pipe_pct_of_active")}
    compute["frac"] = compute["achieved"] / fp64_peak if fp64_peak else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
            "kernel": engine["kernel"], "kernel_mangled": launched, "engine": engine["name"],
            "launches": tk_launches, "kernel_ms": tk_ms,
            "bytes_model": "32 B per path*gridpoint*term (24 B for the k=1 term of a segment)"
                           + ("; term_xs2_kernel moves 40 B per two terms, so this is its streaming-equivalent rate"
                              if engine["kernel"] == "term_xs2_kernel" else ""),
            "traffic_source": f"profiles/{prof_name} (ncu dram__bytes, scaled per launch)"
                              + (" + the streaming-engine capture of the hybrid slice" if hyb else ""),
            "stale_profile": bool(stale or stream_stale),
            "profile_same_binary": (not stale) and prof.get("lib_sha256") == lib_sha256(),
            "profile_same_sass": (not stale) and prof.get("sass_sha256") is not None
                                 and prof.get("sass_sha256") == sass_sha256(launched),
            "hybrid_paths": hyb, "note": engine["note"]}
    if stale:
        roof["profile_kernel"] = prof.get("kernel_mangled") or prof.get("kernel")
    if engine["kernel"] == "term_xs2_kernel":
        # the two-term kernel's own algorithmic bytes: t_{k-1}, s_{k-1} in, t_{k+1}, s_{k+1}, s_k out
        # per two terms (20 B per term); the streaming-equivalent frac above counts 32 B per term
        kb = 20.0 * n * terms
        roof["kernel_bytes_model"] = "40 B per two path*gridpoint*terms (term_xs2_kernel)"
        roof["kernel_bytes_achieved"] = kb / (tk_ms / 1e3) / 1e9 if tk_ms > 0 else 0.0
        roof["kernel_bytes_frac"] = roof["kernel_bytes_achieved"] / peak
    out = {"value": value, "ms_max": ms_max, "terms": terms, "roofline": roof, "compute_roofline": compute,
           "clocks": clk, "launches": launches, "n": n, "M": M, "nwin": nwin, "win": a.warmup + a.steps}
    if keep_session:
        out.update(sess=sess, paths=paths, grid=grid, phi=phi)
    else:
        del sess
    return out


def time_to_error_leg(s2b, ctx, torch, dist, local, rank):
    """north_star's time-to-accuracy claim, measured in every default run (BASELINE configs[3] in
    miniature): one shared Philox batch resolved at dt_leb = 1e-6 (256^2, 64 paths, T = 1), Err
    against the closed form (exact_reference + mean_rel_error, kappa 4), wall time of each
    synchronous solve call.  Magnus reaches the spatial floor at dt = 0.02; E-M at dt = 2e-6 is
    still above it -- so E-M time / Magnus time is a lower bound on the speed-up at matched
    accuracy."""
    d, M, T, dt_leb, a, sigma = 256, 64, 1.0, 1e-6, A_LANGEVIN, SIGMA
    g = s2b.GridSpec.square(d)
    paths = s2b.BrownianPaths.philox(T, dt_leb, M, seed=424242, path_offset=rank * M, ctx=ctx)
    phi = s2b.gaussian_datum(g)
    runs = []

    def timed(fn):
        ctx.synchronize()
        t0 = time.perf_counter()
        ens = fn()
        ctx.synchronize()
        el = max_over_ranks(time.perf_counter() - t0, dist, local)
        e = s2b.exact_errors(ens[-1], a, sigma, paths, 4)
        return el, e["err"]

    for order in (2, 3):
        op = s2b.Operator.from_family(g, "langevin-constant", a=a, sigma=sigma, order=order, ctx=ctx)
        s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=0.02), op, phi, paths, 0.04, g)  # warm-up
        el, err = timed(lambda: s2b.solve_iterated_magnus(s2b.MagnusConfig(order=order, dt=0.02), op, phi, paths,
                                                          T, g))
        runs.append({"method": f"magnus-o{order}", "dt": 0.02, "err": err, "seconds": el})
        del op
    f = s2b.Fields.from_family(g, "langevin-constant", a=a, sigma=sigma, ctx=ctx)
    for dt in (2e-6,):
        el, err = timed(lambda: s2b.solve_euler(s2b.EulerConfig(dt=dt), f, g, phi, paths, T))
        runs.append({"method": "euler", "dt": dt, "err": err, "seconds": el})
    em = runs[-1]
    out = {"config": {"grid": d, "paths_per_gpu": M, "T": T, "dt_leb": dt_leb, "seed": 424242,
                      "error": "mean_rel_error vs exact_reference (closed form), kappa 4",
                      "timing": "wall time of each synchronous solve call (max over ranks)"},
           "runs": runs}
    for r in runs[:2]:
        if em["err"] >= r["err"]:
            out[f"speedup_lower_bound_{r['method']}"] = em["seconds"] / r["seconds"]
    return out


def run_ours(args):
    rank, local, world, dist = dist_setup(args.gpus)
    import paper_2207_09776_b200 as s2b
    import torch

    torch.cuda.set_device(local)
    ctx = s2b.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")
    mg = magnus_leg(args, s2b, ctx, torch, stream, dist, local, world, rank, keep_session=True)
    sess, paths, grid, phi = mg["sess"], mg["paths"], mg["grid"], mg["phi"]
    n, M, nwin, win = mg["n"], mg["M"], mg["nwin"], mg["win"]
    dt_steps = int(round(args.dt / args.dt_leb))
    ms_max, value, terms = mg["ms_max"], mg["value"], mg["terms"]
    roofline, compute, clk, launches = mg["roofline"], mg["compute_roofline"], mg["clocks"], mg["launches"]

    # end-to-end through the C ABI with host buffers: per step the window's Brownian prefix
    # values go H2D from pinned memory, the window runs, the moment statistics come back D2H
    e2e = None
    if not args.no_e2e and win + args.steps <= nwin:
        host_vals = torch.empty((M, paths.steps + 1), dtype=torch.float64).pin_memory()
        hv = host_vals.numpy()
        hv[:] = paths.values()
        mom = torch.empty(2 * n, dtype=torch.float64).pin_memory().numpy()
        h2d = d2h = 0
        if dist is not None:
            dist.barrier()
        ctx.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            k0, k1 = win * dt_steps, (win + 1) * dt_steps
            paths.upload(k0, k1, hv)
            h2d += M * (k1 - k0 + 1) * 8
            sess.advance(1)
            s1, s2, live = sess.moments(mom)
            d2h += 2 * n * 8
            if dist is not None:
                tt = torch.from_numpy(mom).to(f"cuda:{local}")
                dist.all_reduce(tt)
                mom[:] = tt.cpu().numpy()
            win += 1
        ctx.synchronize()
        el = time.perf_counter() - t0
        el = max_over_ranks(el, dist, local)
        e2e = {"value": world * M * n * args.steps / el, "unit": "path*gridpoint*windows/s",
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps}

    # Euler-Maruyama on the same grid/paths (dt = dt_leb), reported beside Magnus; the Magnus
    # session's state is released first (at 1024^2 both would not fit one GPU)
    del sess, mg
    em = None
    if args.euler_steps > 0:
        try:
            em = euler_leg(args, s2b, ctx, grid, phi, paths, stream, torch, dist, local, world, M, n)
        except Exception as ex:  # keep the Magnus line even if the E-M leg fails
            em = {"error": str(ex)[:200]}
    del paths

    # north_star's own target (512^2, >= 60% of the HBM roofline): cfg4 measured in the same
    # run, beside the unchanged cfg2 headline
    ns = None
    if args.preset == "cfg2" and not args.no_north_star:
        try:
            a4 = argparse.Namespace(**vars(args))
            a4.preset = "cfg4"
            for k, v in PRESETS["cfg4"].items():
                setattr(a4, k, v)
            a4.steps, a4.warmup = max(2, min(args.steps, 3)), 3
            a4.T = (a4.warmup + a4.steps) * a4.dt  # the first windows of T = 1: the same per-window work
            r4 = magnus_leg(a4, s2b, ctx, torch, stream, dist, local, world, rank)
            ns = {"metric": "magnus path*gridpoint*windows/s", "value": r4["value"],
                  "ms_per_step": r4["ms_max"] / a4.steps, "steps": a4.steps, "warmup": a4.warmup,
                  "config": {"workload": "cfg4: constant-coefficient Langevin 512x512, 4096 paths/GPU, order-3 "
                                         "iterated Magnus, dt=0.005 (first windows of T=1), dt_leb=1e-4",
                             "grid": 512, "paths_per_gpu": a4.paths, "order": 3, "dt": a4.dt},
                  "path_terms_per_window": r4["terms"] / max(1, a4.paths * a4.steps),
                  "path_gridpoint_terms_per_s": world * r4["n"] * r4["terms"] / (r4["ms_max"] / 1e3),
                  "roofline": r4["roofline"], "compute_roofline": r4["compute_roofline"],
                  "target": "north_star: >= 0.60 of the HBM roofline at 512^2 on 1 B200",
                  "gpu_launches": r4["launches"], "clocks": r4["clocks"]}
        except Exception as ex:
            ns = {"error": str(ex)[:300]}

    tte = None
    if args.preset == "cfg2" and not args.no_tte:
        try:
            tte = time_to_error_leg(s2b, ctx, torch, dist, local, rank)
        except Exception as ex:
            tte = {"error": str(ex)[:300]}

    line = {
        "metric": "magnus path*gridpoint*windows/s", "value": value,
        "unit": "path*gridpoint*windows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Philox Brownian paths, Gaussian datum, Langevin a=1.1 sigma=1/sqrt(10))",
        "config": {"workload": workload_name(args) + f" {args.d}x{args.d}, {M} paths/GPU"
                               + (" (one wave of the 16384 per GPU that 128k paths over 8 GPUs give)"
                                  if args.preset == "cfg5" else "") + ", "
                               f"order-{args.order} iterated Magnus, dt={args.dt} ({nwin} windows), "
                               f"T={args.T}, dt_leb={args.dt_leb}, tol=1e-10, theta=1",
                   "grid": args.d, "family": args.family, "paths_per_gpu": M, "order": args.order, "dt": args.dt,
                   "windows_per_step": 1, "parallelism": f"path-sharded x{world}",
                   "l2": f"inputs larger than L2 ({4 * M * n * 8 / 1e9:.3g} GB resident state per GPU vs 126 MB L2)"},
        "path_terms_per_window": terms / max(1, M * args.steps),
        "path_gridpoint_terms_per_s": world * n * terms / (ms_max / 1e3),
        "roofline": roofline,
        "compute_roofline": compute,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if em is not None:
        line["euler_maruyama"] = em
    if ns is not None:
        line["north_star_512"] = ns
    if tte is not None:
        line["time_to_accuracy"] = tte
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            nproc = os.cpu_count() or 1
            M_cpu = max(2, nproc)
            times, threads = cpu_reference_leg(args, M_cpu, CPU_WINDOWS, reps=1)
            line["cpu_baseline"] = {"value": M_cpu * n * CPU_WINDOWS / times[0], "unit": "path*gridpoint*windows/s",
                                    "cores": threads, "kind": "reference",
                                    "sample": f"{M_cpu} paths x {CPU_WINDOWS} windows of the same workload, "
                                              f"reference C++ (oracle/_ref) with OpenMP"}
        except Exception as ex:
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def euler_leg(args, s2b, ctx, grid, phi, paths, stream, torch, dist, local, world, M, n):
    """E-M at dt = dt_leb on the same paths: path*gridpoint*steps/s (16 B/pt/step roofline)."""
    fam, fkw = family_args(args)
    f = (s2b.Fields.from_arrays(grid, fkw["fields"], ctx=ctx) if "fields" in fkw
         else s2b.Fields.from_family(grid, fam, ctx=ctx, **fkw))
    steps = args.euler_steps
    T = steps * args.dt_leb
    cfg = s2b.EulerConfig(dt=args.dt_leb)
    s2b.solve_euler(cfg, f, grid, phi, paths, 10 * args.dt_leb)  # warm-up
    if dist is not None:
        dist.barrier()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ens = s2b.solve_euler(cfg, f, grid, phi, paths, T)
    e1.record(stream)
    e1.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), dist, local)
    blown = ens[-1].blowup_count()
    del ens
    rate = world * M * n * steps / (ms / 1e3)
    peak, _ = peaks()
    launched = ctx.kernel_names()["em"]  # mangled name of the step kernel that ran
    kname = next((k for k in ("em_cluster_ip_kernel", "em_cluster_kernel", "em_tb_kernel", "em_rows_kernel",
                              "em_step_kernel") if k in launched), launched)
    roof = {"bound": "hbm", "achieved": 16.0 * rate / world / 1e9, "peak": peak,
            "unit": "GB/s", "frac": 16.0 * rate / world / 1e9 / peak, "kernel": kname, "kernel_mangled": launched,
            "note": "whole solve_euler call incl. state init; 16 B/pt/step streaming-equivalent "
                    "(the cluster kernel keeps the state on chip for all steps)"}
    pname = EM_PROFILE_OF.get((args.preset, kname))
    if pname:
        prof = load_profile(pname)
        roof["traffic_source"] = f"profiles/{pname} (ncu dram__bytes per path*step)"
        roof["stale_profile"] = prof.get("kernel_mangled") != launched
        if not roof["stale_profile"]:
            roof["traffic_per_path_step"] = prof.get("dram_bytes_per_path_step")
            roof["traffic_over_algorithmic"] = prof.get("traffic_over_algorithmic")
            roof["ncu_fp64_pipe_pct_of_active"] = prof.get("fp64_pipe_pct_of_active")
            roof["profile_same_binary"] = prof.get("lib_sha256") == lib_sha256()
            roof["profile_same_sass"] = prof.get("sass_sha256") is not None and prof.get("sass_sha256") == sass_sha256(launched)
    return {"metric": "euler path*gridpoint*steps/s", "value": rate, "steps": steps,
            "dt": args.dt_leb, "ms": ms, "blown": blown, "roofline": roof}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_spawn(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
