"""World-size-2 gloo test of the sharded path (shard plan, exchange, merge) on CPU.

Local scoring uses the C oracle (the GPU kernels are covered by the -m gpu
tests); what is under test here is that sharding + all-gather + re-rank with
the reference key reproduces the single-process top-k exactly, ties included.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_15748_b200.distributed import all_gather_topk, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(7)
    sizes = rng.integers(1, 40, size=600)
    off = np.concatenate([[0], np.cumsum(sizes)])
    codes = rng.integers(0, 4, size=(int(off[-1]), 16))      # C=2: many ties
    q = rng.integers(0, 4, size=(5, 12, 16))
    ids = rng.permutation(5000)[:600]
    return sizes, off, codes, q, ids


def _rank_oracle(scores, ids, k):
    from oracle import dessert_oracle as O
    return O.rank_topk(scores, ids, k)


def _worker(rank, world, port, k, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle
    from oracle import dessert_oracle as O
    sizes, off, codes, q, ids = _problem()
    s0, s1 = shard_bounds(sizes, world)[rank]
    sub_off = off[s0:s1 + 1] - off[s0]
    sub_codes = codes[off[s0]:off[s1]]
    scores = c_oracle.score(sub_codes, sub_off, q, O.sim_lut(2, 16), threads=1)
    loc_s = np.full((q.shape[0], k), -1.0)
    loc_i = np.full((q.shape[0], k), -1, dtype=np.int64)
    for r in range(q.shape[0]):
        top = _rank_oracle(scores[r], ids[s0:s1], k)
        loc_s[r, :len(top)] = [v for _, v in top]
        loc_i[r, :len(top)] = [d for d, _ in top]
    gs, gi = all_gather_topk(torch.from_numpy(loc_s), torch.from_numpy(loc_i))
    merged = []
    for r in range(q.shape[0]):
        s, i = gs[r].numpy(), gi[r].numpy()
        keep = s >= 0
        merged.append(_rank_oracle(s[keep], i[keep], k))
    if rank == 0:
        out.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_balanced():
    sizes = np.array([5, 5, 5, 100, 5, 5, 5, 5])
    b = shard_bounds(sizes, 2)
    assert b[0][0] == 0 and b[-1][1] == 8 and b[0][1] == b[1][0]
    for w in (1, 2, 3, 8, 16):
        bb = shard_bounds(np.ones(10, int), w)
        assert sum(e - s for s, e in bb) == 10


@pytest.mark.parametrize("k", [7, 50])
def test_gloo_world2_matches_single_process(k):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, k, out)) for r in range(2)]
    for p in procs:
        p.start()
    merged = out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import c_oracle
    from oracle import dessert_oracle as O
    sizes, off, codes, q, ids = _problem()
    scores = c_oracle.score(codes, off, q, O.sim_lut(2, 16), threads=1)
    for r in range(q.shape[0]):
        assert merged[r] == _rank_oracle(scores[r], ids, k)
