"""Time the nested MC benchmark (BASELINE config 4) alone, a few repetitions:
python tools/nested_probe.py [--states S] [--inner L] [--step i] [--reps R]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import cases  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--states", type=int, default=16384)
    ap.add_argument("--inner", type=int, default=128)
    ap.add_argument("--step", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    cfg = hcva.parse_config(json.dumps(cases.case("c2")))
    book = hcva.generate_book(cfg)
    ctx = hcva.context(0)
    vroot = hcva.RandomStream(cfg.seed).split(hcva.K_VALIDATION_SIM)
    val = hcva.simulate_set(cfg, book, cfg.paths, 1, vroot, ctx=ctx)
    st, surv = val.states_at(args.step)
    st = {k: v[:args.states] for k, v in st.items()}
    surv = surv[:args.states]
    parent = vroot.split(3).split(args.step)
    for r in range(args.reps):
        ctx.synchronize()
        t0 = time.perf_counter()
        v, se = hcva.nested_cva(cfg, book, st, surv, args.step, args.inner, parent, ctx=ctx)
        print(json.dumps({"rep": r, "seconds": round(time.perf_counter() - t0, 4), "mean": float(v.mean())}))


if __name__ == "__main__":
    main()
