"""KV-head sharding across GPUs (one process per GPU) with one all-gather of
head outputs per layer.

The reference has no multi-GPU path; its engine is "one instance
per sequence" with independent KV heads, so the
natural B200 partition is by KV head.  Rank r of g owns KV
heads [r*Hkv/g, (r+1)*Hkv/g) and the query heads of those groups
(gqa_map, attn.py:90-96), builds its own Engine over them, and the layer
output is reassembled by ONE ``all_gather_into_tensor`` of the per-rank
head outputs.  Nothing inside attention, selection or append crosses ranks.

Everything here is host plumbing (index arithmetic + the collective call);
the per-shard compute is whatever ``Engine`` the caller runs (the CUDA path
on GPUs; tests drive it over ``gloo`` with the CPU oracle per shard).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .heads import HeadProfile


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_begin: int
    kv_end: int
    q_begin: int
    q_end: int

    @property
    def num_kv_heads(self) -> int:
        return self.kv_end - self.kv_begin

    @property
    def num_heads(self) -> int:
        return self.q_end - self.q_begin


def shard_heads(num_heads: int, num_kv_heads: int, rank: int, world: int) -> HeadShard:
    """KV-head block partition; query heads follow their group (Eq. 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if num_kv_heads < 1 or num_heads % num_kv_heads:
        raise ValueError(f"query head count {num_heads} is not a multiple of KV head count {num_kv_heads}")
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} KV heads do not divide evenly over {world} ranks")
    per = num_kv_heads // world
    group = num_heads // num_kv_heads
    kb, ke = rank * per, (rank + 1) * per
    return HeadShard(rank, world, kb, ke, kb * group, ke * group)


def shard_profiles(profiles: list, shard: HeadShard) -> list:
    """The rank's HeadProfiles, renumbered from 0 (roles and windows kept)."""
    return [HeadProfile(i, p.gate, p.role, p.sink_blocks, p.local_blocks)
            for i, p in enumerate(profiles[shard.q_begin:shard.q_end])]


def shard_prefill_inputs(q, k, v, shard: HeadShard):
    """Slice token-major q [N,H,D], k/v [S,Hkv,D] to the rank's heads."""
    return (q[:, shard.q_begin:shard.q_end], k[:, shard.kv_begin:shard.kv_end],
            v[:, shard.kv_begin:shard.kv_end])


def shard_decode_inputs(q, k, v, shard: HeadShard):
    """Slice decode rows q [H,D], k/v [Hkv,D] to the rank's heads."""
    return q[shard.q_begin:shard.q_end], k[shard.kv_begin:shard.kv_end], v[shard.kv_begin:shard.kv_end]


class HeadGather:
    """Reassembles [rows, H, D] from every rank's [rows, H/g, D] with one
    ``all_gather_into_tensor`` into a head-major [g, rows, H/g, D] buffer
    (each rank's shard is one contiguous block) and one permute.  The buffer
    is reused across layers and steps."""

    def __init__(self, world: int, rows: int, heads_per_rank: int, head_dim: int, dtype, device, group=None):
        self.world = world
        self.group = group
        self.buf = torch.empty((world, rows, heads_per_rank, head_dim), dtype=dtype, device=device)

    def __call__(self, local: torch.Tensor) -> torch.Tensor:
        import torch.distributed as dist

        if local.shape != self.buf.shape[1:]:
            raise ValueError(f"local output {tuple(local.shape)} does not match {tuple(self.buf.shape[1:])}")
        if self.world == 1:
            self.buf[0].copy_(local)
        else:
            w, rows, hp, d = self.buf.shape
            dist.all_gather_into_tensor(self.buf.view(w * rows, hp, d), local.contiguous(), group=self.group)
        w, rows, hp, d = self.buf.shape
        return self.buf.permute(1, 0, 2, 3).reshape(rows, w * hp, d)
