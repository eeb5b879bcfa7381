"""One pricing step of the C5 backward_learn (profiling aid: launch list of the wide-input path)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cases  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402
from paper_2211_17005_b200 import regression as rg  # noqa: E402

j = cases.case("c5")
j["grid"]["pricing_steps"] = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = hcva.parse_config(json.dumps(j))
sim = hcva.simulate_set(cfg, hcva.generate_book(cfg), cfg.paths, cfg.replicas,
                        hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
sim.labels_all("defaults", to_host=False)
hcva.context().synchronize()
t0 = time.perf_counter()
m = rg.backward_learn(sim, cfg.training, "defaults")
m.get(1)
print(json.dumps({"pricing_steps": cfg.n_steps, "backward_learn_s": time.perf_counter() - t0}))
