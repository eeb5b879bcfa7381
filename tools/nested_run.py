"""Nested MC (validation.cpp:123-179) on the C2 validation set at one step
for a block of outer states (profiling aid: ncu of the grouped conditional
K1, K2 and k_nested_payoff)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cases  # noqa: E402
import numpy as np  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402

states = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
inner = int(sys.argv[2]) if len(sys.argv) > 2 else 128
step = 5
cfg = hcva.parse_config(cases.text("c2"))
book = hcva.generate_book(cfg)
vroot = hcva.RandomStream(cfg.seed).split(hcva.K_VALIDATION_SIM)
val = hcva.simulate_set(cfg, book, states, 1, vroot)
st, surv = val.states_at(step)
value, se = hcva.nested_cva(cfg, book, st, surv, step, inner, vroot.split(3).split(step))
print("nested", states, inner, float(np.mean(value)), float(np.mean(se)))
