"""Multi-GPU host logic on CPU: the interleaved Y-path shard
map, and the trainer's cross-rank reduction -- allgather of FP64 partials,
summed in rank order -- exercised with real collectives (gloo, world size 2)
on the FP64 regression restatement."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_api
from paper_2211_17005_b200 import dist


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shards_partition_paths_and_batches(world):
    M, nb = 256, 8
    pb = dist.batch_paths(M, nb)
    seen = []
    for g in range(world):
        spec = dist.shard_spec(M, nb, world, g)
        ids = dist.shard_paths(spec)
        assert spec["n_paths"] == M // world and len(ids) == M // world
        # local batch b (P_B / world consecutive local paths) lies inside global batch b
        loc = ids.reshape(nb, pb // world)
        for b in range(nb):
            assert np.all((loc[b] >= b * pb) & (loc[b] < (b + 1) * pb))
            assert np.array_equal(loc[b], b * pb + g * (pb // world) + np.arange(pb // world))
        seen.append(ids)
    assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(M))


def test_shard_spec_rejects_uneven_layouts():
    with pytest.raises(ValueError):
        dist.shard_spec(100, 8, 1, 0)  # batches must be whole paths
    with pytest.raises(ValueError):
        dist.shard_spec(96, 8, 8, 0)  # 12-path batches do not split over 8 ranks
    with pytest.raises(ValueError):
        dist.shard_spec(64, 8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _adam(p, m, v, g, t, lr=1e-3):
    b1, b2, eps = 0.9, 0.999, 1e-8
    m[:] = b1 * m + (1 - b1) * g
    v[:] = b2 * v + (1 - b2) * g * g
    p -= lr * (m / (1 - b1 ** t)) / (np.sqrt(v / (1 - b2 ** t)) + eps)


def _data(rows=384, d=7, seed=11):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, d))
    y = np.abs(np.sin(x[:, 0]) + 0.3 * x[:, 1] + 0.05 * rng.standard_normal(rows))
    return x, y


def _sgd_epochs(R, x, y, p, n_batches, epochs, part=None, reduce=None):
    """Adam epochs over contiguous batches; with `part` each rank sees its
    interleaved share of every batch and the gradient is reduce(local sum)."""
    m, v = np.zeros_like(p), np.zeros_like(p)
    bs = len(y) // n_batches
    t = 0
    for _ in range(epochs):
        for b in range(n_batches):
            rows = np.arange(b * bs, (b + 1) * bs)
            if part is not None:
                rows = rows[part(bs)]
            _, g = R.loss(p, x[rows], y[rows], 2, 8)
            g = g * (len(rows) / bs)  # this rank's share of the batch mean
            if reduce is not None:
                g = reduce(g)
            t += 1
            _adam(p, m, v, g, t)
    return p


def _rank_main(rank, world, port, out_dir):
    import torch.distributed as tdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. rank-ordered reduction: identical on every rank, equal to the ordered sum
        local = np.array([rank + 0.1, 1e-17 * (rank + 1), -3.0 * rank])
        tot = dist.rank_order_sum(local)
        np.save(os.path.join(out_dir, f"sum{rank}.npy"), tot)
        # 2. id distribution (the NCCL unique id travels the same way)
        uid = dist.share_id(lambda: bytes(range(dist.ID_BYTES)))
        np.save(os.path.join(out_dir, f"uid{rank}.npy"), np.frombuffer(uid, dtype=np.uint8))
        # 3. data-parallel Adam on the FP64 restatement with the trainer's reduction
        R = oracle_api.restatement()
        x, y = _data()
        p0 = R.init_network(x.shape[1], 2, 8, R.key(3))

        def part(bs):
            blk = bs // world
            return np.arange(rank * blk, (rank + 1) * blk)

        p = _sgd_epochs(R, x, y, p0.copy(), 4, 3, part=part, reduce=dist.rank_order_sum)
        np.save(os.path.join(out_dir, f"p{rank}.npy"), p)
    finally:
        tdist.destroy_process_group()


def test_rank_ordered_allgather_training_gloo():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, _free_port(), d), nprocs=world, join=True)
        sums = [np.load(os.path.join(d, f"sum{r}.npy")) for r in range(world)]
        uids = [np.load(os.path.join(d, f"uid{r}.npy")) for r in range(world)]
        ps = [np.load(os.path.join(d, f"p{r}.npy")) for r in range(world)]
    expect = np.zeros(3)
    for r in range(world):
        expect = expect + np.array([r + 0.1, 1e-17 * (r + 1), -3.0 * r])
    for s in sums:
        assert np.array_equal(s, expect)
    for u in uids:
        assert np.array_equal(u, np.arange(dist.ID_BYTES, dtype=np.uint8))
    # every rank applies the same update ...
    assert np.array_equal(ps[0], ps[1])
    # ... equal to the single-process run up to FP64 re-association
    R = oracle_api.restatement()
    x, y = _data()
    p0 = R.init_network(x.shape[1], 2, 8, R.key(3))
    ref = _sgd_epochs(R, x, y, p0.copy(), 4, 3)
    assert np.allclose(ps[0], ref, rtol=1e-10, atol=1e-13)
    assert not np.array_equal(ref, p0)


@pytest.mark.parametrize("n", [2, 4])
def test_bench_self_launch_starts_n_ranks(n):
    """`python bench.py --gpus N` without torchrun starts N rank processes
    (torch.distributed.run on 127.0.0.1) with distinct RANK / LOCAL_RANK and
    WORLD_SIZE = N (the launcher only: --launch-probe prints each rank's
    environment and exits before any device work)."""
    import json
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(oracle_api.ROOT, "bench.py"), "--gpus", str(n),
                          "--launch-probe"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    import re

    ranks = [json.loads(m) for m in re.findall(r'\{"rank"[^{}]*\}', out.stdout)]
    assert sorted(r["rank"] for r in ranks) == list(range(n))
    assert sorted(r["local_rank"] for r in ranks) == list(range(n))
    assert {r["world"] for r in ranks} == {n}
    assert len({r["pid"] for r in ranks}) == n
