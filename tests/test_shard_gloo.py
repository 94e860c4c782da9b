"""world_size-2 gloo test of the scene-sharded multi-GPU path (CPU): each rank
takes its contiguous block of scenes, runs the per-scene PSH (oracle, since
there is no GPU here — the sharding and collectives are what is under test),
and rank 0 checks the gathered per-scene results equal the 1-rank run and
that the timing reduction is a max."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restated as O
from paper_2412_16481_b200.shard import gather_to_root, max_over_ranks, scenes_for_rank

N_SCENES = 5


def _scene(i):
    c = O.synth_cloud(100 + i, 3000, "uniform-box")
    vox = O.remap_nonnegative(O.voxelize(c, (0, 0, 0), 1 / 32))
    ids, offs, counts, _ = O.psh_assign(vox, None, "zorder-div", 32, 128, 256)
    return i, ids, offs


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = [_scene(i) for i in scenes_for_rank(N_SCENES, world, rank)]
    t = max_over_ranks(1.0 + rank)
    got = gather_to_root(mine, world, rank)
    if rank == 0:
        flat = sorted([s for part in got for s in part], key=lambda s: s[0])
        q.put((t, [(i, ids.tolist(), offs.tolist()) for i, ids, offs in flat]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_covers_all_scenes():
    for n in (1, 5, 16, 64):
        for w in (1, 2, 4, 8):
            parts = [list(scenes_for_rank(n, w, r)) for r in range(w)]
            assert sum(parts, []) == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_sharding_matches_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert t == 2.0                      # max over ranks of (1 + rank)
    single = [_scene(i) for i in range(N_SCENES)]
    assert [r[0] for r in res] == list(range(N_SCENES))
    for (i, ids, offs), (_, sids, soffs) in zip(res, single):
        assert ids == sids.tolist() and offs == soffs.tolist()
