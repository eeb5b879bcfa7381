"""Small driver for profiling runs: one C2-shaped simulation + R in-place re-runs,
printing the per-phase CUDA-event times (K1 market, K3 defaults, K2 cube, K4 labels).

    python tools/probe.py [--config c2] [--paths M] [--reps R]
    HCVA_K1_MODE=1|2 python tools/probe.py   # K1 with generation / recursion skipped
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import cases  # noqa: E402
import numpy as np  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--paths", type=int, default=0)
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--train", action="store_true", help="time backward_learn on the set")
    ap.add_argument("--steps", type=int, default=0, help="override pricing steps (train probe)")
    args = ap.parse_args()
    if args.train:
        return train_probe(args)
    j = cases.case(args.config)
    if args.paths:
        j["simulation"]["paths"] = args.paths
    if args.replicas:
        j["simulation"]["replicas"] = args.replicas
    cfg = hcva.parse_config(json.dumps(j))
    book = hcva.generate_book(cfg)
    root = hcva.RandomStream(cfg.seed).split(1)
    sim = hcva.simulate_set(cfg, book, cfg.paths, cfg.replicas, root)
    times = []
    for r in range(args.reps):
        sim.rerun(root.split(100 + r), "defaults", event_slot=r)
    sim.ctx.synchronize()
    for r in range(args.reps):
        times.append(sim.phase_times(r))
    t = np.array(times)
    print(json.dumps({"mode": os.environ.get("HCVA_K1_MODE", "0"), "config": args.config,
                      "paths": cfg.paths, "ms": dict(zip(["K1", "K3", "K2", "K4"], t.min(0).round(3).tolist()))}))


def train_probe(args):
    import time

    from paper_2211_17005_b200 import regression as rg

    j = cases.case(args.config)
    if args.paths:
        j["simulation"]["paths"] = args.paths
    if args.replicas:
        j["simulation"]["replicas"] = args.replicas
    if args.steps:
        j["grid"]["pricing_steps"] = args.steps
    cfg = hcva.parse_config(json.dumps(j))
    book = hcva.generate_book(cfg)
    t0 = time.perf_counter()
    sim = hcva.simulate_set(cfg, book, cfg.paths, cfg.replicas, hcva.RandomStream(cfg.seed).split(1))
    sim.labels_all("defaults", to_host=False)
    sim.ctx.synchronize()
    t1 = time.perf_counter()
    models = rg.backward_learn(sim, cfg.training)
    t2 = time.perf_counter()
    p, mean, scale, rep = models.get(1)
    print(json.dumps({"config": args.config, "paths": cfg.paths, "replicas": cfg.replicas, "steps": cfg.n_steps,
                      "simulate_s": round(t1 - t0, 4), "train_s": round(t2 - t1, 4),
                      "best_loss_step1": rep["best_loss"], "best_epoch_step1": rep["best_epoch"],
                      "launches": sim.ctx.launch_count()}))


if __name__ == "__main__":
    main()
