"""Multi-GPU sharding of the scoring path.

Sets are independent units (_score_one depends on one sketch, index.py:198),
so the index shards into contiguous set ranges balanced by vector count.
Every rank scores its shard against the same query sets and keeps a local
top-k; the only exchange is one all-gather of (n_qsets x k) scores and doc
ids (NCCL over NVLink on GPUs, gloo in the CPU tests), followed by a re-rank
with the reference key (score desc, doc_id asc).  Because the key is a total
order on (score, doc_id) and every global winner is a local winner of its
shard, the merged list equals the single-GPU result exactly.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(set_sizes, world: int) -> list[tuple[int, int]]:
    """Contiguous set ranges [s0, s1) per rank with ~equal vector counts."""
    sizes = np.asarray(set_sizes, dtype=np.int64)
    n = sizes.shape[0]
    if world < 1:
        raise ValueError(f"invalid parameter: world must be >= 1, got {world}")
    cum = np.concatenate([[0], np.cumsum(sizes)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def all_gather_topk(scores: torch.Tensor, ids: torch.Tensor, group=None):
    """Concatenate every rank's (n_qsets, k) local top-k along dim 1 (rank order)."""
    world = dist.get_world_size(group)
    gs = [torch.empty_like(scores) for _ in range(world)]
    gi = [torch.empty_like(ids) for _ in range(world)]
    dist.all_gather(gs, scores.contiguous(), group=group)
    dist.all_gather(gi, ids.contiguous(), group=group)
    return torch.cat(gs, dim=1).contiguous(), torch.cat(gi, dim=1).contiguous()


def merge_topk_device(scores: torch.Tensor, ids: torch.Tensor, k: int):
    """Device re-rank of gathered candidates with K4 (score desc, doc id asc).  Padding
    entries (score -1.0, id UINT64_MAX) sort after every real score (K4 orders keys by
    IEEE value), so they surface only when fewer than k real candidates exist."""
    from . import engine

    out_s, out_i, _ = engine.topk(scores.contiguous(), min(k, scores.shape[1]), ids=ids.contiguous())
    return out_s, out_i


def sharded_query_batch(index_shard, Qs, top_k: int, group=None):
    """Local top-k on this rank's shard + all-gather + merge -> global top-k (device)."""
    from .index import query_batch

    s, i = query_batch(index_shard, Qs, top_k, return_tensors=True)
    gs, gi = all_gather_topk(s, i, group)
    return merge_topk_device(gs, gi, top_k)
