"""Multi-rank regression on one B200 (in-process group: one host thread and
context per rank, reductions over UVA copies): the sharded simulation equals
the matching rows of the unsharded one bit for bit, every rank ends with the
same networks, and they match the single-GPU run within the regression
tolerance (per-rank partial sums re-associate FP64 / FP32 rounding)."""
import threading

import numpy as np
import pytest

import cases
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import dist
from paper_2211_17005_b200 import regression as rg

pytestmark = pytest.mark.gpu


def _case(M=64, N=8, width=16, batches=8, epochs=4):
    cfg = hcva.parse_config(cases.text("desk_corr"))
    cfg.training.width, cfg.training.n_batches, cfg.training.epochs = width, batches, epochs
    return cfg, hcva.generate_book(cfg), M, N


def _run_ranks(world, cfg, book, M, N, label_kind="defaults"):
    group = dist.LocalGroup(world)
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    out, errs = [None] * world, []

    def rank(g):
        try:
            ctx = hcva.Context(0)
            spec = dist.shard_spec(M, cfg.training.n_batches, world, g)
            sim = hcva.simulate_set(cfg, book, spec["n_paths"], N, root, path_offset=spec["path_offset"], ctx=ctx,
                                    shard=spec["shard"])
            models = rg.backward_learn(sim, cfg.training, label_kind, comm=group.comm(ctx, g))
            out[g] = (spec, sim, models, ctx)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=rank, args=(g,)) for g in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_training_matches_single_gpu(world):
    cfg, book, M, N = _case()
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    full = hcva.simulate_set(cfg, book, M, N, root)
    single = rg.backward_learn(full, cfg.training, "defaults")
    ranks = _run_ranks(world, cfg, book, M, N)
    mk = full.market_arrays()
    st = full.default_steps()
    cube = full.cube_values()
    for spec, sim, models, _ in ranks:
        ids = dist.shard_paths(spec)
        smk = sim.market_arrays()
        for k in mk:
            assert np.array_equal(smk[k], mk[k][ids]), k
        assert np.array_equal(sim.default_steps(), st[ids])
        assert np.array_equal(sim.cube_values(), cube[ids])
    for i in range(1, cfg.n_steps + 1):
        p0, m0, s0, r0 = ranks[0][2].get(i)
        for _, _, models, _ in ranks[1:]:
            p, m, s, r = models.get(i)
            assert np.array_equal(p, p0) and np.array_equal(m, m0) and np.array_equal(s, s0), i
            assert r["best_loss"] == r0["best_loss"] and r["best_epoch"] == r0["best_epoch"], i
        ps, ms, ss, rs = single.get(i)
        assert np.allclose(m0, ms, rtol=1e-12, atol=1e-15) and np.allclose(s0, ss, rtol=1e-12), i
        assert r0["best_loss"] == pytest.approx(rs["best_loss"], rel=1e-3, abs=1e-12), i
        assert np.max(np.abs(p0 - ps)) <= 1e-3 * max(np.max(np.abs(ps)), 1e-12), i


def test_comm_reports_rank_and_world():
    group = dist.LocalGroup(3)
    ctx = hcva.context()
    c = group.comm(ctx, 2)
    assert c.rank_world == (2, 3)
    with pytest.raises(hcva.ContractError):
        group.comm(ctx, 3)


def test_nccl_transport_single_rank():
    """The NCCL transport (dlopen'ed libnccl, ncclCommInitRank, ncclAllGather on
    the context stream) driving the gather path of the trainer with one rank:
    same networks as the plain single-GPU run within the regression tolerance
    (the gather path reduces losses / scaler moments in a different order)."""
    cfg, book, M, N = _case()
    root = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    ctx = hcva.Context(0)
    sim = hcva.simulate_set(cfg, book, M, N, root, ctx=ctx)
    plain = rg.backward_learn(sim, cfg.training, "defaults")
    comm = dist.nccl_comm(ctx, 1, 0, dist.nccl_unique_id())
    assert comm.rank_world == (0, 1)
    viacomm = rg.backward_learn(sim, cfg.training, "defaults", comm=comm)
    for i in range(1, cfg.n_steps + 1):
        pp, mp, sp, rp = plain.get(i)
        pc, mc, sc, rc = viacomm.get(i)
        assert np.allclose(mc, mp, rtol=1e-12, atol=1e-15) and np.allclose(sc, sp, rtol=1e-12), i
        assert rc["best_loss"] == pytest.approx(rp["best_loss"], rel=1e-3, abs=1e-12), i
        assert np.max(np.abs(pc - pp)) <= 1e-3 * max(np.max(np.abs(pp)), 1e-12), i
    comm.close()
