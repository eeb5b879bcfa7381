#!/usr/bin/env python
"""Benchmark of the pathwise CVA hot path (BASELINE.json metric 1):

  Y x X x step scenarios/s = M * N * n / time of [Y diffusion + MtM cube +
  X over-simulation + labels for every pricing step]

on the paper case C2 (configs/paper_shape.json, 8 clients, 500 swaps,
M = 2^14 Y-paths x N = 2^7 X-replicas, n = 100 quarterly steps, 25 substeps)
per GPU.  A "step" is one in-place re-run of that whole pipeline with fresh
stream keys (hcva_sim_rerun); it writes ~2.5 GB (market block, cube, default
steps, labels of all 101 steps), far beyond the 126 MB L2, so no flush is
needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without torchrun starts N ranks itself (torch.distributed.run on
127.0.0.1, one process per GPU, device = local rank).  Multi-GPU: weak scaling -- rank r simulates its own 2^14 paths
(global path offset r * 2^14); no collective on the data path.  Device time
is the max over ranks.
"""
from __future__ import annotations

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
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "Y×X×step scenarios/s"
UNIT = "scenarios/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--paths", type=int, default=0, help="override M per GPU")
    ap.add_argument("--replicas", type=int, default=0, help="override N")
    ap.add_argument("--cpu-baseline-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-learning", action="store_true", help="skip metric 2 (CVA learning time)")
    ap.add_argument("--learning-steps", type=int, default=0, help="pricing steps for metric 2 (default: all)")
    ap.add_argument("--no-nested", action="store_true", help="skip the nested MC benchmark (C4)")
    ap.add_argument("--nested-step", type=int, default=5)
    ap.add_argument("--nested-inner", type=int, default=128)
    ap.add_argument("--nested-states", type=int, default=0, help="outer states (default: all validation paths)")
    ap.add_argument("--launch-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--learning-timeout", type=float, default=240.0,
                    help="N > 1: if the sharded learning leg (~3 s at C2) exceeds this many seconds, print the "
                         "metric line with the leg marked as timed out and exit")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def workload(args):
    import cases
    import paper_2211_17005_b200 as hcva

    j = cases.case(args.config)
    if args.paths:
        j["simulation"]["paths"] = args.paths
    if args.replicas:
        j["simulation"]["replicas"] = args.replicas
    cfg = hcva.parse_config(json.dumps(j))
    return cfg, j


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------- CPU arm
def run_reference_sample(cfg, seconds_target, probe_paths=64):
    """Time the reference's own CPU pipeline (oracle/_ref, built from
    /root/reference's sources) on a bounded sample of the workload: the same
    config with fewer Y-paths.  Returns (scenarios/s, dict)."""
    import ctypes as C

    import cases
    import oracle_api

    ref = oracle_api.reference()
    kind = "reference"
    if ref is None:
        ref, kind = oracle_api.restatement(), "port"
    threads = cpu_threads()
    os.environ["HIERCVA_THREADS"] = str(threads)
    m = cases.oracle_model(cfg)
    root = ref.key(cfg.seed)
    book = ref.generate_book(m, cfg.book_count, cfg.notional_min, cfg.notional_max, ref.split(root, 0))
    key_sim = ref.split(root, 1)
    mm = ref.model(m)
    bookc = np.ascontiguousarray(book, dtype=oracle_api.SWAP_DTYPE)

    def run(paths):
        sec, chk = C.c_double(), C.c_double()
        rc = ref.lib.or_pipeline_bench(C.byref(mm), bookc.ctypes.data_as(C.c_void_p), len(bookc), paths,
                                       cfg.replicas, C.c_uint64(key_sim), 0, C.byref(sec), C.byref(chk))
        if rc:
            raise RuntimeError(ref.lib.or_last_error().decode())
        return sec.value

    t_probe = run(probe_paths)
    paths = int(max(probe_paths, min(cfg.paths, probe_paths * seconds_target / max(t_probe, 1e-3))))
    paths = max(threads, (paths // threads) * threads)
    t = run(paths)
    value = paths * cfg.replicas * cfg.n_steps / t
    return value, dict(kind=kind, cores=threads if kind == "reference" else 1, paths=paths, seconds=t)


def reference_arm(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    cfg, j = workload(args)
    vals = []
    info = None
    per_step = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    for s in range(args.warmup + args.steps):
        v, info = run_reference_sample(cfg, per_step)
        if s >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    sample = (f"{info['paths']} of {cfg.paths} Y-paths x {cfg.replicas} X-replicas x {cfg.n_steps} steps "
              f"per step ({info['seconds']:.1f} s; simulate_set + defaults_label for i=n..1; features_at is not "
              f"timed on either arm) on {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * info["seconds"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (configs/paper_shape.json model, generated book)",
        "config": config_obj(cfg, args, world=1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_obj(cfg, args, world):
    return {"workload": f"{args.config}: paper CVA case, {cfg.n_clients} clients, {cfg.book_count} swaps, "
                        f"{cfg.n_economies} economies",
            "paths_per_gpu": cfg.paths, "replicas": cfg.replicas, "pricing_steps": cfg.n_steps,
            "substeps": cfg.substeps, "dt_years": cfg.dt, "n_factors": cfg.n_factors,
            "global_paths": cfg.paths * world, "parallelism": f"y-path shards x{world}",
            "l2": "per-step working set ~2.5 GB/GPU >> 126 MB L2 (no flush needed)",
            "step_work": "Y diffusion + MtM cube + X default steps + defaults labels of all n steps (features "
                         "are not materialised on either arm: the regression builds them per batch)",
            "deviations": {
                "mtm_not_fused_with_diffusion": "K1 and K2 are both FP64-issue bound; fusing saves only the "
                                                "0.6 GB market re-read, and labels/features/nested/twin re-read "
                                                "the 106 MB cube (DESIGN.md section 3)",
                "default_steps_not_bitmasks": "X indicators stored as one uint16 default step per (replica, "
                                              "name), which encodes 1{s <= i} for every step i (DESIGN.md "
                                              "section 3)"}}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi can take a second to start on a fresh box: wait for its
            # first sample, then keep only the samples of the timed region
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10.0 and self.proc.poll() is None:
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------- GPU arm
# Algorithmic FP64 work of K1 per path: n*sub*[D*F_N + D(D+1) + 20*D],
# F_N = 120 flop per normal (Acklam + Halley step with erfc/exp, 3 divides).
F_N = 120


def k1_flops_per_path(cfg):
    D = cfg.n_factors
    return cfg.n_steps * cfg.substeps * (D * F_N + D * (D + 1) + 20 * D)


def ours_arm(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2211_17005_b200 as hcva

    cfg, _ = workload(args)
    ctx = hcva.context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    book = hcva.generate_book(cfg)
    M, N, n = cfg.paths, cfg.replicas, cfg.n_steps
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    sim = hcva.simulate_set(cfg, book, M, N, root, path_offset=rank * M, ctx=ctx)
    sim.labels_all("defaults", to_host=False)
    ctx.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for w in range(args.warmup):
        sim.rerun(root.split(1000 + w), "defaults")
    ctx.synchronize()
    barrier()
    launches0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for s in range(args.steps):
            sim.rerun(root.split(2000 + s), "defaults", event_slot=s)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    ties = sim.tie_counts()
    phases = np.array([sim.phase_times(s) for s in range(args.steps)])  # ms [K, 4]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    scen = M * N * n * world
    value = scen / (ms_step * 1e-3)

    # Roofline of the dominant kernel (K1, FP64 pipe): algorithmic flop per
    # launch / mean launch time measured with events on the launch stream.
    fp64_peak = ctypes_peak(ctx)
    k1_ms = float(phases[:, 0].mean())
    k1_flop = k1_flops_per_path(cfg) * M
    achieved = k1_flop / (k1_ms * 1e-3) / 1e12
    phase_ms = {k: float(v) for k, v in zip(["market_K1", "defaults_K3", "cube_K2", "labels_K4"], phases.mean(0))}

    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(hcva, cfg, book, ctx, stream, rank, world, args)
    # The metric line is complete from here on; the secondary legs below add to
    # it, and a failing or stuck secondary leg is reported inside it instead of
    # losing the line (see _secondary / learning_leg's watchdog).
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (configs/paper_shape.json model, generated 500-swap book, quarterly grid)",
        "config": config_obj(cfg, args, world),
        "e2e": e2e,
        "gpu_launches": int(launches),
        "phase_ms": phase_ms,
        "roofline": {"bound": "fp64", "kernel": "k_market (K1 diffusion)", "achieved": achieved,
                     "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                     "peak_source": "measured DFMA microbenchmark on this GPU (hcva_diag_fp64_peak)",
                     "algorithmic_flop_per_launch": k1_flop, "traffic": k1_traffic(),
                     "k1_share_of_step": k1_ms / ms_step},
        "clocks": clocks.summary(),
        "threshold_ties_last_step": {"within_1ulp": int(ties[0]), "within_1e-12": int(ties[1]),
                                     "comparisons": int(M * N * (cfg.n_clients + 1))},
        "cpu_baseline": None,
        "parity": None,
        "cva_learning": None,
        "nested_mc": None,
    }
    _PARTIAL.update(line=line, rank=rank)
    models = None
    if not args.no_learning:
        res = _secondary("cva_learning", lambda: learning_leg(hcva, cfg, book, ctx, args, rank, world))
        if res is not None:
            line["cva_learning"], models = res
    if not args.no_nested:
        del sim
        line["nested_mc"] = _secondary("nested_mc", lambda: nested_leg(hcva, cfg, book, ctx, args, models, rank, world))
    del models
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = run_reference_sample(cfg, args.cpu_baseline_seconds)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
                                "sample": f"{info['paths']} of {M} Y-paths x {N} replicas x {n} steps, "
                                          f"{info['seconds']:.1f} s (simulate_set + defaults_label for i=n..1; "
                                          f"features_at is not timed on either arm) on {cpu_model()}"}
        line["parity"] = _secondary("parity", lambda: parity_leg(hcva, cfg, book, ctx))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


_PARTIAL = {}


def _secondary(key, fn):
    """Run a secondary leg (CVA learning, nested MC); an exception becomes
    {"error": ...} under `key` in the metric line rather than a lost line."""
    try:
        return fn()
    except Exception as exc:  # noqa: BLE001 -- reported in the JSON line
        sys.stderr.write(f"bench: {key} leg failed: {exc!r}\n")
        if key == "cva_learning":
            _PARTIAL["line"][key] = {"error": repr(exc)}
            return None
        return {"error": repr(exc)}


def parity_leg(hcva, cfg, book, ctx):
    """Untimed checker, run with the CPU baseline (rank 0, N=1): the reference's
    own simulate_market + sample_default_block (oracle/_ref, compiled from
    /root/reference's sources, HIERCVA_THREADS = host cores) on the FULL
    workload against the engine's default block for the same stream keys --
    every one of M x N x Cn default steps must be equal (defaults.cpp:20-45);
    threshold ties within 1 ulp / 1e-12 are the engine's counters."""
    import cases
    import oracle_api

    ref = oracle_api.reference()
    kind = "reference"
    if ref is None:
        ref, kind = oracle_api.restatement(), "port"
    os.environ["HIERCVA_THREADS"] = str(cpu_threads())
    M, N = cfg.paths, cfg.replicas
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    sim = hcva.simulate_set(cfg, book, M, N, root, ctx=ctx)
    got = sim.default_steps()
    ties = sim.tie_counts()
    gmk = sim.market_arrays()
    del sim
    m = cases.oracle_model(cfg)
    sk = ref.split(ref.key(cfg.seed), 1)
    c0 = time.perf_counter()
    mk = ref.simulate_market(m, M, ref.split(sk, 0))
    want = ref.sample_defaults(mk["hazard"], N, ref.split(sk, 1))
    sec = time.perf_counter() - c0
    rel = 0.0  # max |engine - reference| over the largest |reference| value, per factor array
    for k in ("rates", "fx", "intens", "lagged", "disc", "hazard"):
        a, b = gmk[k], mk[k]
        if b.size:
            rel = max(rel, float(np.max(np.abs(a - b)) / np.max(np.abs(b))))
    return {"default_mismatches": int((got != want).sum()), "default_steps_compared": int(got.size),
            "ties_1ulp": int(ties[0]), "ties_1e-12": int(ties[1]),
            "defaulted": int((want != 0xFFFF).sum()), "market_max_err_over_scale": rel,
            "against": f"{kind}: simulate_market + sample_default_block on all {M} x {N} x {cfg.n_clients + 1} "
                       f"(path, replica, name) of the bench workload, same stream keys ({sec:.1f} s on "
                       f"{cpu_threads()} host threads)"}


def sgd_roofline(hcva, cfg, sim):
    """Roofline of the regression's dominant kernel chain, the SGD step
    (gradient kernel(s) + optimizer) at the bench network and batch: CUDA
    events on the engine's stream (hcva_diag_sgd_timing) around SGD steps of
    train_base at pricing step n of the learning set; algorithmic tensor flop
    per row = forward 2dU + 2U^2, backward G1 = G2 W1 2U^2, weight gradients
    2U^2 + 2dU (d = 2Cc + 3E - 1 features, U hidden units) -- the 3xTF32
    products issue three MMAs per algorithmic one, so TF32/3 is the attainable
    ceiling."""
    import ctypes as C

    from paper_2211_17005_b200 import _lib
    from paper_2211_17005_b200 import regression as rg

    t = cfg.training
    d = 2 * cfg.n_clients + 3 * cfg.n_economies - 1
    U = t.width
    rows = cfg.paths * cfg.replicas // t.n_batches
    tm = rg.sgd_timing(sim, t, cfg.n_steps, steps=50, label_kind=cfg.label_kind)
    peak = C.c_double()
    _lib.check(_lib.lib().hcva_diag_tc_rate(sim.ctx.handle, 128, 256, 4096, C.byref(peak)))
    flop_row = 4 * d * U + 6 * U * U
    flop = flop_row * rows
    fused = tm.get("fused_step_ms")
    step_ms = fused if fused else tm["step_ms"]  # what backward_learn runs
    achieved = flop / (step_ms * 1e-3) / 1e12
    kern = ("k_sgd_split persistent epoch (gradient + fused optimizer, layer-0 split)" if fused else
            "k_sgd_split (fused gradient, layer-0 split) + k_adam" if tm["split"] else
            "k_sgd_tc + k_wgrad_tc + k_adam")
    return {"bound": "tensor", "kernel": f"SGD step ({kern})", "unit": "TFLOP/s",
            "achieved": achieved, "peak": peak.value, "frac": achieved / peak.value,
            "frac_of_tf32_div3": achieved / (peak.value / 3.0),
            "peak_source": "measured kind::tf32 tcgen05.mma rate, M=128 N=256 chains on every SM "
                           "(hcva_diag_tc_rate)",
            "algorithmic_flop_per_step": flop, "flop_per_row": flop_row, "rows_per_step": rows,
            "d": d, "width": U, "step_ms": step_ms, "per_step_launch_ms": tm["step_ms"],
            "per_step_launch_gradient_ms": tm["gradient_ms"], "per_step_launch_optimizer_ms": tm["optimizer_ms"],
            "traffic": None}


def k1_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch at C2, from
    the committed ncu --set full capture (profiles/r2/ncu_K1_k_market.txt):
    the FP64-bound kernel's only DRAM traffic is its market stores."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2", "ncu_K1_k_market.txt")
    try:
        vals = {}
        for ln in open(path):
            if "dram__bytes_" in ln and "=" in ln:
                k, v = ln.split("=")
                num, unit = v.split()[0], v.split()[1]
                vals[k.strip()] = float(num) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        return {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                "source": "profiles/r2/ncu_K1_k_market.txt (ncu --set full, C2)"}
    except (OSError, KeyError, ValueError, IndexError):
        return None


def ctypes_peak(ctx):
    import ctypes as C

    from paper_2211_17005_b200 import _lib

    v = C.c_double()
    _lib.check(_lib.lib().hcva_diag_fp64_peak(ctx.handle, C.byref(v)))
    return v.value


def e2e_leg(hcva, cfg, book, ctx, stream, rank, world, args):
    """The same metric through the public API with host inputs: per step the
    model/book go host->device inside hcva_simulate_set, the engine simulates
    and labels every step, and the CVA profile (n+1 doubles) comes back."""
    import torch

    M, N, n = cfg.paths, cfg.replicas, cfg.n_steps
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    steps = max(2, min(args.steps, 5))
    for w in range(1):
        sim = hcva.simulate_set(cfg, book, M, N, root.split(3000 + w), path_offset=rank * M, ctx=ctx)
        sim.cva_profile("defaults")
        del sim
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for s in range(steps):
        sim = hcva.simulate_set(cfg, book, M, N, root.split(4000 + s), path_offset=rank * M, ctx=ctx)
        prof = sim.cva_profile("defaults")
        del sim
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        t = torch.tensor([dt], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dt = float(t.item())
    h2d = book.nbytes + cfg.rates.nbytes + cfg.fx.nbytes + cfg.credit.nbytes
    return {"value": M * N * n * world / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(prof.nbytes), "ms_per_step": dt * 1e3,
            "path": "hcva.simulate_set (hcva_simulate_set: stage + K1/K3/K2) + cva_profile (K4 + reduction)",
            "cva0": float(prof[0])}


def learning_leg(hcva, cfg, book, ctx, args, rank=0, world=1):
    """BASELINE metric 2: end-to-end CVA learning time on the same workload --
    host config -> simulate_set -> labels -> backward_learn over every pricing
    step (Alg. 2, E epochs x |B| batches, refit, best tracking) -> the time-0
    CVA estimate back on the host.  One run, wall clock around a synchronised
    device pipeline (the regression is a dependent chain of ~100*(E|B|+E)
    phases, so there is no batch of independent steps to average).  With N
    GPUs (C3) the same global problem is sharded by Y-path (dist.shard_spec,
    strong scaling) and the trainer allgathers FP64 partials over NCCL; the
    time is the max over ranks."""
    import torch

    import copy
    import json as _json

    import cases
    from paper_2211_17005_b200 import dist
    from paper_2211_17005_b200 import regression as rg

    t = cfg.training
    steps = args.learning_steps or cfg.n_steps
    if steps != cfg.n_steps:
        j = cases.case(args.config)
        j["grid"]["pricing_steps"] = steps
        cfg = hcva.parse_config(_json.dumps(j))
        book = hcva.generate_book(cfg)
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    spec = dist.shard_spec(cfg.paths, t.n_batches, world, rank)
    watchdog = None
    if world > 1:  # a stuck collective must not hang the scaling run: fail loudly instead
        def _abort():  # print the metric line with the learning leg marked, then leave
            sys.stderr.write(f"bench: rank {rank}: multi-GPU learning leg exceeded {args.learning_timeout} s\n")
            sys.stderr.flush()
            part = _PARTIAL.get("line")
            if rank == 0 and part is not None:
                part["cva_learning"] = {"error": f"timeout after {args.learning_timeout} s"}
                print(json.dumps(part), flush=True)
            os._exit(0 if part is not None else 3)

        watchdog = threading.Timer(args.learning_timeout, _abort)
        watchdog.daemon = True
        watchdog.start()
    comm = None
    try:
        if world > 1:
            comm = dist.nccl_comm(ctx, world, rank, dist.share_id(dist.nccl_unique_id))
            torch.distributed.barrier()
        # untimed warm-up: the full set and its labels once (the stream-ordered memory
        # pool grown to the run's footprint, which it keeps for the timed run: on a
        # fresh box first-touch allocations cost ~0.3 s), then the same trainer path at
        # full size over two pricing steps (module loading, host-side first calls)
        wsim = hcva.simulate_set(cfg, book, spec["n_paths"], cfg.replicas, root, path_offset=spec["path_offset"],
                                 ctx=ctx, shard=spec["shard"])
        wsim.labels_all(cfg.label_kind, to_host=False)
        del wsim
        wt = copy.copy(t)
        wj = _json.loads(_json.dumps(cases.case(args.config)))
        wj["grid"]["pricing_steps"] = 2
        wcfg = hcva.parse_config(_json.dumps(wj))
        wsim = hcva.simulate_set(wcfg, hcva.generate_book(wcfg), spec["n_paths"], cfg.replicas, root,
                                 path_offset=spec["path_offset"], ctx=ctx, shard=spec["shard"])
        wsim.labels_all(cfg.label_kind, to_host=False)
        rg.backward_learn(wsim, wt, cfg.label_kind, comm=comm)
        del wsim
        if world > 1:
            torch.distributed.barrier()
        ctx.synchronize()
        t0 = time.perf_counter()
        sim = hcva.simulate_set(cfg, book, spec["n_paths"], cfg.replicas, root, path_offset=spec["path_offset"],
                                ctx=ctx, shard=spec["shard"])
        sim.labels_all(cfg.label_kind, to_host=False)
        ctx.synchronize()
        t1 = time.perf_counter()
        models = rg.backward_learn(sim, t, cfg.label_kind, comm=comm)
        p, mean, scale, rep = models.get(1)
        t2 = time.perf_counter()
    finally:
        if watchdog is not None:
            watchdog.cancel()
    total, sim_s, train_s = t2 - t0, t1 - t0, t2 - t1
    if world > 1:  # max over ranks
        tt = torch.tensor([total, sim_s, train_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        total, sim_s, train_s = (float(v) for v in tt)
        comm.close()
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # CPU reference of the regression: the FP64 restatement of regressor.cpp
        # (the reference's own regressor needs Eigen, absent) timed on a bounded
        # sample -- one train_base of step n on the first rows of its data --
        # and extrapolated linearly in rows and steps (train_base is linear in both).
        import oracle_api

        R = oracle_api.restatement()
        rows = min(cfg.paths * cfg.replicas, max(t.n_batches * 64, 4096))
        rows -= rows % t.n_batches
        x = sim.features(cfg.n_steps)[:rows]
        y = sim.labels(cfg.n_steps, cfg.label_kind).reshape(-1)[:rows]
        mean, scale = R.fit_scaler(x, cfg.n_clients)
        init = R.init_network(x.shape[1], t.hidden_layers, t.width, R.key(cfg.seed, 0xBEEF, cfg.n_steps))
        init[-1] = float(np.mean(y))
        c0 = time.perf_counter()
        R.train_base((x - mean) / scale, y, init, t.hidden_layers, t.width, t.n_batches, t.epochs, t.learning_rate)
        sec = time.perf_counter() - c0
        full = sec * (cfg.paths * cfg.replicas / rows) * steps
        cpu = {"value": full, "unit": "s (extrapolated)", "cores": 1, "kind": "port",
               "sample": f"train_base of step {cfg.n_steps} on {rows} rows: {sec:.2f} s, x{cfg.paths * cfg.replicas // rows}"
                         f" rows x {steps} steps (FP64 restatement of regressor.cpp; simulation not included)"}
    out = {"value": total, "unit": "s", "higher_is_better": False, "pricing_steps": steps, "cpu_baseline": cpu,
            "simulate_and_labels_s": sim_s, "backward_learn_s": train_s,
            "sgd_steps": steps * t.epochs * t.n_batches, "rows": cfg.paths * cfg.replicas, "n_gpus": world,
            "scaling": "strong (global C2 problem sharded by Y-path)" if world > 1 else None,
            "net": f"{t.hidden_layers}x{t.width} {t.activation}", "best_loss_step1": rep["best_loss"],
            "path": "hcva_simulate_set + hcva_labels_all + hcva_backward_learn (K1-K5, device resident)"}
    if rank == 0:
        out["roofline"] = _secondary("sgd_roofline", lambda: sgd_roofline(hcva, cfg, sim))
    return out, (models if steps == cfg.n_steps and world == 1 else None)


def nested_leg(hcva, cfg, book, ctx, args, models=None, rank=0, world=1):
    """BASELINE config 4: the nested Monte Carlo CVA benchmark (the accuracy
    oracle, validation.cpp:123-179 as driven by pipeline.cpp:269-292) on the
    paper case -- outer states = the validation set's paths at `step`
    (root.split(2), N=1), `inner` conditional re-simulations per state from
    root.split(2).split(3).split(step).split(s).  The paper quotes >= 32 min on
    a V100 for 16384 states x 128 inner.  Timed: host states -> device ->
    grouped conditional K1 + K2 + payoff/reduction -> values on the host (wall
    clock around the synchronous call; max over ranks).  With N GPUs each rank
    takes a contiguous block of states (no collective; the estimates are
    per-state pure).  When the learning leg trained on one GPU, the nested
    relative RMSE of its predictions (validation.cpp:181-210) is reported."""
    import torch

    step, inner = args.nested_step, args.nested_inner
    vroot = hcva.RandomStream(cfg.seed).split(hcva.K_VALIDATION_SIM)
    n_val = cfg.paths
    val = hcva.simulate_set(cfg, book, n_val, 1, vroot, ctx=ctx)
    states = min(args.nested_states or n_val, n_val)
    lo, hi = rank * states // world, (rank + 1) * states // world
    st, surv = val.states_at(step)
    st = {k: np.ascontiguousarray(v[lo:hi]) for k, v in st.items()}
    surv = np.ascontiguousarray(surv[lo:hi])
    parent = vroot.split(3).split(step)
    # untimed warm-up on one batch worth of states (the engine batches by a
    # 12 GB budget): first-touch of the memory pool and module loading
    warm = max(1, min(hi - lo, int(12e9 / (inner * (cfg.n_steps - step + 1) * (3 * cfg.n_economies + 3 * cfg.n_clients + 2) * 8))))
    hcva.nested_cva(cfg, book, {k: v[:warm] for k, v in st.items()}, surv[:warm], step, inner, parent, ctx=ctx,
                    first_state=lo)
    if world > 1:
        torch.distributed.barrier()
    ctx.synchronize()
    t0 = time.perf_counter()
    value, se = hcva.nested_cva(cfg, book, st, surv, step, inner, parent, ctx=ctx, first_state=lo)
    sec = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([sec], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        sec = float(tt.item())
    h = cfg.n_steps - step
    normals = float(states) * inner * h * cfg.substeps * cfg.n_factors
    out = {"value": sec, "unit": "s", "higher_is_better": False, "states": states, "inner": inner, "step": step,
           "states_per_s": states / sec, "normals_per_s": normals / sec, "n_gpus": world,
           "scaling": "strong (states split across ranks)" if world > 1 else None,
           "mean_nested_cva": float(np.mean(value)), "mean_std_error": float(np.mean(se)),
           "path": "hcva_nested_cva_range (grouped conditional K1 + K2 + k_nested_payoff/k_nested_reduce)",
           "paper_v100": ">= 32 min for 16384 states x 128 inner (PAPER.md:871)"}
    if models is not None and world == 1:
        pred = models.predict(step, val)[:states]
        rm, rse, zero, used = hcva.nested_relative_rmse(pred, value)
        out["relative_rmse"] = {"value": rm, "std_error": rse, "excluded_zero": zero, "used": used,
                                "training": f"M={cfg.paths}, N={cfg.replicas}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = nested_reference_sample(cfg, book, st, surv, step, inner, sec, states)
    return out


def nested_reference_sample(cfg, book, st, surv, step, inner, gpu_sec, states, seconds_target=10.0):
    """The reference's own nested_cva (oracle/_ref, HIERCVA_THREADS = host
    cores, inner paths in its parallel_for) on the first few states of the
    same set, extrapolated linearly to all states."""
    import cases
    import oracle_api

    ref = oracle_api.reference()
    kind = "reference"
    if ref is None:
        ref, kind = oracle_api.restatement(), "port"
    threads = cpu_threads()
    os.environ["HIERCVA_THREADS"] = str(threads)
    m = cases.oracle_model(cfg)
    bk = np.ascontiguousarray(book, dtype=oracle_api.SWAP_DTYPE)
    done, c0 = 0, time.perf_counter()
    while done < states and (time.perf_counter() - c0 < seconds_target or done == 0):
        one = {k: v[done] for k, v in st.items()}
        ref.nested_cva(m, bk, one, surv[done], step, inner, ref.key(cfg.seed, 2, 3, step, done))
        done += 1
    sec = time.perf_counter() - c0
    full = sec * states / done
    return {"value": full, "unit": "s (extrapolated)", "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": f"nested_cva on {done} of {states} states ({sec:.1f} s), x{states / done:.0f}",
            "ratio_vs_gpu": full / gpu_sec}


def self_launch(args):
    """`--gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 with this same command line, and return
    their exit status; None when already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator creation shows nranks
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse_args()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.launch_probe:  # launcher test hook: which rank am I
        rank, world, local = dist_env()
        print(json.dumps({"rank": rank, "world": world, "local_rank": local, "pid": os.getpid()}), flush=True)
        return
    rank, world, _ = dist_env()
    if world != args.gpus and rank == 0:
        sys.stderr.write(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; running {world} rank(s)\n")
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours_arm(args)


if __name__ == "__main__":
    main()
