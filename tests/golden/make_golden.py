"""Generate the golden fixtures in tests/golden/*.npz from the COMPILED REFERENCE.

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
Every array comes from oracle/_ref/libhcva_ref.so, i.e. the reference's own
sources (proj/src/{rng,market,defaults,portfolio,labels,validation}.cpp)
compiled in place.  The fixtures travel with the repo; the reference does not.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import cases  # noqa: E402
import oracle_api  # noqa: E402
from paper_2211_17005_b200.config import parse_config  # noqa: E402

# (case, M, N, label steps, feature step, nested (step, states, inner), twin step)
SPECS = [
    ("minimal", 64, 2, [0, 2, 4], 1, (2, 3, 16), 1),
    ("c1", 48, 16, [0, 10, 25, 49, 50], 25, (5, 2, 32), 10),
    ("desk_corr", 40, 8, [0, 3, 6, 12], 6, (6, 3, 24), 3),
    ("c2", 12, 8, [0, 20, 50, 99, 100], 50, (50, 2, 8), 20),
    ("c5", 8, 4, [0, 50, 100], 50, (50, 2, 4), 20),
]


def make(ref, name, M, N, steps, fstep, nested, tstep):
    cfg = parse_config(cases.text(name))
    m = cases.oracle_model(cfg)
    root = ref.key(cfg.seed)
    book = ref.generate_book(m, cfg.book_count, cfg.notional_min, cfg.notional_max, ref.split(root, 0))
    sk = ref.split(root, 1)
    mk = ref.simulate_market(m, M, ref.split(sk, 0))
    st = ref.sample_defaults(mk["hazard"], N, ref.split(sk, 1))
    cube = ref.build_cube(m, mk, book)
    out = dict(config=np.array(cases.text(name)), M=M, N=N, book=book, steps=st, cube=cube,
               label_steps=np.array(steps), feature_step=fstep, chol=None)
    for k, v in mk.items():
        out["market_" + k] = v
    out["labels_defaults"] = np.stack([ref.defaults_label(i, mk, st, cube, cfg.dt) for i in steps])
    out["labels_intensity"] = np.stack([ref.intensity_label(i, mk, st, cube, cfg.dt) for i in steps])
    out["features"] = ref.features(fstep, mk, st)
    step, states, inner = nested
    vals = []
    for s in range(states):
        state = dict(rates=mk["rates"][s, step], log_fx=np.log(mk["fx"][s, step]),
                     intens=mk["intens"][s, step], lagged=mk["lagged"][s, step])
        surv = (st[s, 0, 1:] > step).astype(np.int32)
        vals.append(ref.nested_cva(m, book, state, surv, step, inner, ref.key(cfg.seed, 2, 3, step, s)))
    out["nested"] = np.array(vals)
    out["nested_spec"] = np.array(nested)
    out["twin1"], out["twin2"], out["twin_stats"] = cases.twin_block(ref, cfg, m, book, mk, st, tstep)
    out["twin_step"] = tstep
    del out["chol"]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: getattr(v, "shape", None) for k, v in out.items()})


def kats(ref):
    """Known-answer draws plus a spread of normals/exponentials."""
    k42 = ref.key(42)
    k7 = ref.key(7, 1, 0, 3)
    out = dict(
        u64_42=ref.u64(k42, 0, 64),
        uniform_42=ref.uniforms(k42, 0, 64),
        normal_42=ref.normals(k42, 0, 4096),
        exp_42=ref.exponentials(k42, 0, 256),
        normal_7_1_0_3=ref.normals(k7, 0, 256),
        keys=np.array([k42, ref.split(k42, 0), ref.split(k42, 1), k7], dtype=np.uint64),
    )
    np.savez_compressed(os.path.join(HERE, "rng_kat.npz"), **out)


if __name__ == "__main__":
    ref = oracle_api.reference()
    if ref is None:
        raise SystemExit("compiled reference unavailable (needs /root/reference)")
    kats(ref)
    only = set(sys.argv[1:])
    for spec in SPECS:
        if not only or spec[0] in only:
            make(ref, *spec)
