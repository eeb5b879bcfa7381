import sys, time, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import cases, paper_2211_17005_b200 as hcva
cfg = hcva.parse_config(json.dumps(cases.case("c2")))
book = hcva.generate_book(cfg)
ctx = hcva.context(0)
root = hcva.RandomStream(cfg.seed).split(1)
M, N = cfg.paths, cfg.replicas
for s in range(6):
    t0 = time.perf_counter()
    sim = hcva.simulate_set(cfg, book, M, N, root.split(4000 + s), ctx=ctx)
    t1 = time.perf_counter()
    ctx.synchronize()
    t2 = time.perf_counter()
    prof = sim.cva_profile("defaults")
    t3 = time.perf_counter()
    del sim
    t4 = time.perf_counter()
    print(f"launch {1e3*(t1-t0):.2f} ms, sim done {1e3*(t2-t0):.2f}, profile {1e3*(t3-t2):.2f}, free {1e3*(t4-t3):.2f}, total {1e3*(t4-t0):.2f}")
