"""SGD-step timing at C2 (profiling aid): hcva_diag_sgd_timing on the full
paper-case set for the layer-0 split kernels and the feature-matrix kernels
(HCVA_SPLIT=0 in a second process)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cases  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402
from paper_2211_17005_b200 import regression as rg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
j = cases.case("c2")
j["grid"]["pricing_steps"] = steps
cfg = hcva.parse_config(json.dumps(j))
sim = hcva.simulate_set(cfg, hcva.generate_book(cfg), cfg.paths, cfg.replicas,
                        hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
for rep in range(2):
    print(json.dumps(rg.sgd_timing(sim, cfg.training, 2, steps=100)))
