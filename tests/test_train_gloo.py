"""world_size-2 gloo test of the data-parallel gradient exchange of the
training step (paper_2412_16481_b200.train.allreduce_grads):
after the flat-bucket all_reduce(SUM)/world every rank holds the mean of the
ranks' gradients, with shapes and the GRAD_NAMES layout preserved."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_16481_b200.train import GRAD_NAMES, allreduce_grads, flatten_grads, unflatten_grads

D, DH = 12, 48


def _grads(rank):
    g = torch.Generator().manual_seed(100 + rank)
    shapes = {"w_q": (D, D), "w_k": (D, D), "w_v": (D, D), "w_o": (D, D), "w_in": (D, DH),
              "w_out": (DH, D), "b_in": (DH,)}
    return {k: torch.randn(shapes.get(k, (D,)), generator=g) for k in GRAD_NAMES}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = allreduce_grads(_grads(rank))
    q.put((rank, {k: v.clone() for k, v in out.items()}))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_flatten_roundtrip():
    g = _grads(0)
    back = unflatten_grads(flatten_grads(g), g)
    for k in GRAD_NAMES:
        assert torch.equal(back[k], g[k])


def test_allreduce_is_identity_without_group():
    g = _grads(0)
    assert allreduce_grads(g) is g


@pytest.mark.timeout(120)
def test_allreduce_mean_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    want = {k: (_grads(0)[k] + _grads(1)[k]) / 2 for k in GRAD_NAMES}
    for r in (0, 1):
        for k in GRAD_NAMES:
            assert res[r][k].shape == want[k].shape
            torch.testing.assert_close(res[r][k], want[k], rtol=1e-6, atol=1e-6)
