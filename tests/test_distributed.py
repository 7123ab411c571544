"""world_size-2 gloo tests of the batch-sharding path on CPU.

The per-rank compute is stood in by the CPU oracle (test infrastructure); the
host logic under test (shard_pairs, gather_terms, sharded_cost_and_grad) is the
product code the GPU ranks run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_08817_b200.distributed import gather_terms, shard_pairs, sharded_cost_and_grad


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_pairs_partitions_exactly():
    for n in (1, 5, 64, 32):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_pairs(n, r, world) for r in range(world)]
            flat = [p for part in parts for p in part]
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_pairs(4, 2, 2)


def _worker(rank, world, port, n_pairs, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import morphreg_oracle as O

    rng = np.random.default_rng(0)
    shape = (12, 10)
    srcs = [np.abs(O.smooth(rng.standard_normal(shape), O.gaussian_weights(1.0))) for _ in range(n_pairs)]
    tgts = [np.abs(O.smooth(rng.standard_normal(shape), O.gaussian_weights(1.0))) for _ in range(n_pairs)]
    zs = [0.2 * O.smooth(rng.standard_normal(shape), O.gaussian_weights(1.0)) for _ in range(n_pairs)]
    w = O.gaussian_weights(1.5)

    def compute(pairs):
        gs, ts = [], []
        for p in pairs:
            gs.append(O.grad(srcs[p], tgts[p], zs[p], 1e-3, 0.5, 3, 0.2, w))
            ts.append(O.cost(srcs[p], tgts[p], zs[p], 1e-3, 0.5, 3, 0.2, w))
        return torch.tensor(np.array(gs)), torch.tensor(np.array(ts), dtype=torch.float64).reshape(-1, 4)

    pairs, g, terms = sharded_cost_and_grad(compute, n_pairs)
    if rank == 0:
        _, ref_terms = compute(list(range(n_pairs)))
        out_q.put((pairs, terms.numpy(), ref_terms.numpy()))
    else:
        out_q.put((pairs, None, None))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_pairs", [5, 4])
def test_two_rank_gloo_sharded_grad_gathers_every_pair(n_pairs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_pairs, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_pairs = sorted(x for r in results for x in r[0])
    assert all_pairs == list(range(n_pairs))
    got = [r for r in results if r[1] is not None][0]
    # the gathered rows equal the single-process rows, in pair order
    assert np.array_equal(got[1], got[2])
