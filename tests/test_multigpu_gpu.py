"""Two-GPU shard equivalence ("batched multi-GPU results must equal
single-GPU per-pair results"): two NCCL ranks, one GPU each, shard a batch of pairs
with distributed.sharded_cost_and_grad over the device path; the gathered cost rows and
each rank's gradients must equal a single-GPU run of the whole batch bit for bit
(deterministic adjoint).  Skipped when fewer than 2 GPUs are visible."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(n_pairs, shape):
    rng = np.random.default_rng(3)
    src = rng.random((n_pairs,) + shape).astype(np.float32)
    tgt = rng.random((n_pairs,) + shape).astype(np.float32)
    z0 = (0.2 * rng.standard_normal((n_pairs,) + shape)).astype(np.float32)
    return src, tgt, z0


def _cfg():
    import paper_2106_08817_b200 as mr

    return mr, mr.ShootingConfig(mr.Scheme.SEMI_LAGRANGIAN, 4, 0.2, mr.GaussianKernel(2.0),
                                 deterministic=True)


def _worker(rank, world, port, n_pairs, shape, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    from paper_2106_08817_b200.distributed import sharded_cost_and_grad

    mr, cfg = _cfg()
    src, tgt, z0 = _inputs(n_pairs, shape)

    def compute(pairs):
        sel = np.asarray(pairs)
        dev = [torch.as_tensor(a[sel]).cuda() for a in (src, tgt, z0)]
        zbar, terms, _ = mr.cost_and_grad_batch(dev[0], dev[1], dev[2], cfg, 1e-3, 0.5)
        return zbar, terms

    pairs, g, terms = sharded_cost_and_grad(compute, n_pairs)
    q.put((rank, pairs, g.cpu().numpy(), terms.cpu().numpy()))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_shards_equal_the_single_gpu_batch():
    import torch.multiprocessing as mp

    n_pairs, shape = 5, (40, 56)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_pairs, shape, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted((q.get(timeout=300) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    mr, cfg = _cfg()
    src, tgt, z0 = _inputs(n_pairs, shape)
    zbar, terms, _ = mr.cost_and_grad_batch(*[torch.as_tensor(a).cuda() for a in (src, tgt, z0)], cfg,
                                            1e-3, 0.5)
    zbar, terms = zbar.cpu().numpy(), terms.cpu().numpy()
    assert sorted(p for r in results for p in r[1]) == list(range(n_pairs))
    for rank, pairs, g, gathered in results:
        assert np.array_equal(gathered, terms)          # every rank holds every pair's rows
        assert np.array_equal(g, zbar[np.asarray(pairs)])  # its own pairs' gradients
