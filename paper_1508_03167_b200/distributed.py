"""Multi-GPU MergeShuffle: contiguous shards by leaf blocks (SURVEY.md §8 e).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  With G
ranks (a power of two dividing q = 2^c), rank r owns leaf blocks
[r*q/G, (r+1)*q/G) = global elements [(n*r*q/G)>>c, (n*(r+1)*q/G)>>c).

* Leaves and merge rounds 1 .. c-log2(G) have all their pairs inside one shard:
  every rank runs them locally with the same substream indices as the
  single-GPU schedule (C ABI sk_merge_shuffle_shard) -- no communication.
* Rounds c-log2(G)+1 .. c merge pairs spanning 2, 4, .., G ranks.  The pair's
  bit stream is regenerated locally (it is a pure function of the seed and the
  substream index r*q+i), the pair's elements are all-gathered inside the
  spanning group, every member runs the merge (sk_merge_range on a fresh
  substream) and keeps its own slice.  This is the NCCL baseline for the
  exchange step; a peer-memory gather of only the positions each rank writes
  (50 / 62.5 / 68.75 % of a shard at spans 2 / 4 / 8) is the planned upgrade.

The result (and the bit count, all-reduced) is identical to the 1-GPU and the
reference output for the same (n, cutoff, seed).

Engines are pluggable so the same driver runs on GPUs (CudaEngine) and in
CPU tests over gloo (the oracle-backed engine in tests/).
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

from . import _lib
from .bitstream import substream_seed
from .shufflers import MERGE_CUTOFF_DEFAULT, merge_plan


class CudaEngine:
    """Local work through the C ABI on the current CUDA device."""

    def __init__(self):
        self.lib = _lib.load()

    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def shard(self, buf: torch.Tensor, n: int, cutoff: int, seed: int, blk0: int, nblk: int, rounds: int) -> int:
        bits = ctypes.c_uint64(0)
        _lib.check(self.lib.sk_merge_shuffle_shard(ctypes.c_void_p(buf.data_ptr()), buf.element_size(), n, cutoff,
                                                   seed & ((1 << 64) - 1), blk0, nblk, rounds, ctypes.byref(bits),
                                                   self._stream()))
        return int(bits.value)

    def merge(self, buf: torch.Tensor, j: int, k: int, l: int, sseed: int) -> int:
        st = _lib.state_array((sseed, 0, 0, 0))
        _lib.check(self.lib.sk_merge_range(ctypes.c_void_p(buf.data_ptr()), buf.element_size(), j, k, l, st,
                                           self._stream()))
        return int(st[3])


def shard_layout(n: int, cutoff: int, world: int):
    """(c, q, bounds, nblk, local_rounds) of a world-way contiguous sharding."""
    c, q, bounds = merge_plan(n, cutoff)
    lg = world.bit_length() - 1
    if world < 1 or (1 << lg) != world:
        raise ValueError("world size must be a power of two")
    if world > q:
        raise ValueError(f"{world} shards need at least {world} leaf blocks (q={q}); lower the cutoff")
    nblk = q // world
    return c, q, bounds, nblk, c - lg


def shard_range(n: int, cutoff: int, world: int, rank: int) -> Tuple[int, int]:
    _, _, bounds, nblk, _ = shard_layout(n, cutoff, world)
    return bounds[rank * nblk], bounds[(rank + 1) * nblk]


class _Groups:
    """Process groups of every span 2, 4, .., world (consecutive ranks)."""

    def __init__(self, world: int, group=None):
        self.g = {}
        span = 2
        while span <= world:
            for g0 in range(0, world, span):
                ranks = list(range(g0, g0 + span))
                if span == world and group is None:
                    self.g[(span, g0)] = dist.group.WORLD
                else:
                    self.g[(span, g0)] = dist.new_group(ranks)
            span *= 2

    def get(self, span: int, g0: int):
        return self.g[(span, g0)]


_GROUPS = {}


def merge_shuffle_sharded(shard: torch.Tensor, n: int, cutoff: Optional[int], seed: int,
                          engine=None) -> int:
    """Shuffle the n-element array whose contiguous shard this rank holds
    (shard_range(n, cutoff, world, rank)); returns the total bit count
    (ShuffleReport.bits of the whole shuffle) on every rank."""
    world, rank = dist.get_world_size(), dist.get_rank()
    cutoff = MERGE_CUTOFF_DEFAULT if cutoff is None else cutoff
    engine = engine or CudaEngine()
    c, q, bounds, nblk, local_rounds = shard_layout(n, cutoff, world)
    blk0 = rank * nblk
    lo, hi = bounds[blk0], bounds[blk0 + nblk]
    if shard.numel() != hi - lo:
        raise ValueError(f"rank {rank} shard has {shard.numel()} elements, expected {hi - lo}")
    bits = engine.shard(shard, n, cutoff, seed, blk0, nblk, local_rounds)
    if world > 1:
        groups = _GROUPS.setdefault(world, _Groups(world))
        sizes = [bounds[(r + 1) * nblk] - bounds[r * nblk] for r in range(world)]
    for r in range(local_rounds + 1, c + 1):
        span = 1 << (r - local_rounds)
        g0 = (rank // span) * span
        p = 1 << (r - 1)
        i = (blk0 // (2 * p)) * (2 * p)  # first block of the spanning pair
        j, k, l = bounds[i], bounds[i + p], bounds[i + 2 * p]
        mx = max(sizes[g0:g0 + span])
        send = torch.empty(mx, dtype=shard.dtype, device=shard.device)
        send[:shard.numel()] = shard
        parts = [torch.empty_like(send) for _ in range(span)]
        dist.all_gather(parts, send, group=groups.get(span, g0))
        pair = torch.cat([parts[m][:sizes[g0 + m]] for m in range(span)])
        pb = engine.merge(pair, 0, k - j, l - j, substream_seed(seed, r * q + i))
        shard.copy_(pair[lo - j:hi - j])
        if rank == g0:
            bits += pb
    if world > 1:
        t = torch.tensor([bits], dtype=torch.float64, device=shard.device)
        # bit counts fit 2^53 exactly for n < 2^47
        dist.all_reduce(t)
        bits = int(t.item())
    return bits


def simulate_sharded(data: torch.Tensor, n: int, cutoff: Optional[int], seed: int, world: int,
                     engine=None) -> int:
    """The sharded schedule of merge_shuffle_sharded executed by ONE process
    over all `world` shards in turn (no collectives): validates the per-shard
    entry point and the cross-round logic on a single device."""
    cutoff = MERGE_CUTOFF_DEFAULT if cutoff is None else cutoff
    engine = engine or CudaEngine()
    c, q, bounds, nblk, local_rounds = shard_layout(n, cutoff, world)
    bits = 0
    for r in range(world):
        lo, hi = bounds[r * nblk], bounds[(r + 1) * nblk]
        shard = data[lo:hi]
        bits += engine.shard(shard, n, cutoff, seed, r * nblk, nblk, local_rounds)
    for rr in range(local_rounds + 1, c + 1):
        p = 1 << (rr - 1)
        for i in range(0, q, 2 * p):
            j, k, l = bounds[i], bounds[i + p], bounds[i + 2 * p]
            pair = data[j:l].clone()
            bits += engine.merge(pair, 0, k - j, l - j, substream_seed(seed, rr * q + i))
            data[j:l].copy_(pair)
    return bits
