"""A small backward_learn on the layer-0 split path (C2 model, 64 paths x 128
replicas, 3 pricing steps): the sanitizer target for the split kernels."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cases  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402
from paper_2211_17005_b200 import regression as rg  # noqa: E402

j = cases.case("c2")
j["grid"]["pricing_steps"] = 3
cfg = hcva.parse_config(json.dumps(j))
t = cfg.training
t.epochs, t.n_batches = 2, 4
sim = hcva.simulate_set(cfg, hcva.generate_book(cfg), 64, 128, hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
m = rg.backward_learn(sim, t, "defaults")
print("split_small", rg.sgd_timing(sim, t, 2, steps=2)["split"], m.get(1)[3]["best_loss"])
