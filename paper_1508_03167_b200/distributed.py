"""Multi-GPU MergeShuffle: contiguous shards by leaf blocks (SURVEY.md §8 e).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  With G
ranks (a power of two dividing q = 2^c), rank r owns leaf blocks
[r*q/G, (r+1)*q/G) = global elements [(n*r*q/G)>>c, (n*(r+1)*q/G)>>c).

* Leaves and merge rounds 1 .. c-log2(G) have all their pairs inside one shard:
  every rank runs them locally with the same substream indices as the
  single-GPU schedule (C ABI sk_merge_shuffle_shard) -- no communication.
* Rounds c-log2(G)+1 .. c merge pairs spanning 2, 4, .., G ranks.  The pair's
  bit stream is regenerated locally (it is a pure function of the seed and the
  substream index r*q+i), so no bits travel.  Default exchange ("peer"): every
  rank maps the other ranks' shard buffers (CUDA IPC handles, all-gathered
  once), and the pair is merged by ONE fused kernel per rank over peer memory
  (sk_merge_range_peers phase 1: the rank takes every span-th tile of the
  pair's tree merge, TMA-loading its windows from whichever GPU holds them and
  storing them back there -- the exchange overlaps the merge tile by tile);
  after a barrier of the span the first rank applies the tail insertion
  (phase 2).  Each element crosses NVLink at most once each way.
  The NCCL baseline ("allgather"): the pair's elements all-gathered inside the
  spanning group, every member merges the whole pair, keeps its slice.

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

    # -- peer memory (CUDA IPC over NVLink) --------------------------------
    def peer_handle(self, buf: torch.Tensor) -> bytes:
        h = (ctypes.c_ubyte * 64)()
        off = ctypes.c_uint64(0)
        _lib.check(self.lib.sk_ipc_get_handle(ctypes.c_void_p(buf.data_ptr()), h, ctypes.byref(off)))
        return bytes(h) + int(off.value).to_bytes(8, "little")

    def open_peer(self, handle: bytes) -> int:
        # mappings are cached per process (an allocation is mapped once; the
        # caching allocator keeps shard buffers alive across calls)
        key = bytes(handle[:64])
        base = _PEER_MAPS.get(key)
        if base is None:
            b = ctypes.c_void_p(0)
            h = (ctypes.c_ubyte * 64).from_buffer_copy(key)
            _lib.check(self.lib.sk_ipc_open(h, ctypes.byref(b)))
            base = _PEER_MAPS[key] = int(b.value)
        return base + int.from_bytes(handle[64:72], "little")

    def close_peers(self) -> None:
        pass  # see release_peer_maps()

    def merge_peers(self, bases: List[int], starts: List[int], part: int, elem_bytes: int, n1: int, n2: int,
                    sseed: int, phase: int) -> int:
        n = len(bases)
        pb = (ctypes.c_void_p * n)(*bases)
        ps = (ctypes.c_uint64 * (n + 1))(*starts)
        st = _lib.state_array((sseed, 0, 0, 0))
        bits = ctypes.c_uint64(0)
        _lib.check(self.lib.sk_merge_range_peers(pb, ps, n, part, elem_bytes, n1, n2, st, phase, ctypes.byref(bits),
                                                 self._stream()))
        return int(bits.value)


_PEER_MAPS = {}


def release_peer_maps() -> None:
    """Unmap every peer allocation mapped by this process."""
    lib = _lib.load()
    for base in _PEER_MAPS.values():
        lib.sk_ipc_close(ctypes.c_void_p(base))
    _PEER_MAPS.clear()


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


def _groups(world: int) -> _Groups:
    """The span groups of this world, built once (dist.new_group is a collective)."""
    g = _GROUPS.get(world)
    if g is None:
        g = _GROUPS[world] = _Groups(world)
    return g


def release_groups() -> None:
    """Destroy the span groups (before dist.destroy_process_group)."""
    for g in _GROUPS.values():
        for grp in g.g.values():
            if grp is not dist.group.WORLD:
                dist.destroy_process_group(grp)
    _GROUPS.clear()


def _coll_device(t: torch.Tensor):
    """Where collective buffers live: host tensors for gloo, the shard's device for NCCL."""
    return torch.device("cpu") if dist.get_backend() == "gloo" else t.device


def merge_shuffle_sharded(shard: torch.Tensor, n: int, cutoff: Optional[int], seed: int,
                          engine=None, exchange: str = "peer") -> int:
    """Shuffle the n-element array whose contiguous shard this rank holds
    (shard_range(n, cutoff, world, rank)); returns the total bit count
    (ShuffleReport.bits of the whole shuffle) on every rank.

    exchange = "peer": the spanning rounds run as one fused kernel per rank
    over peer memory (sk_merge_range_peers: each rank merges its share of the
    pair's tiles, reading and writing the other ranks' shards directly over
    NVLink; one rank applies the tail after a barrier).  exchange =
    "allgather": the NCCL baseline (the pair all-gathered, merged redundantly
    by every member, own slice kept)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    cutoff = MERGE_CUTOFF_DEFAULT if cutoff is None else cutoff
    engine = engine or CudaEngine()
    c, q, bounds, nblk, local_rounds = shard_layout(n, cutoff, world)
    blk0 = rank * nblk
    lo, hi = bounds[blk0], bounds[blk0 + nblk]
    if shard.numel() != hi - lo:
        raise ValueError(f"rank {rank} shard has {shard.numel()} elements, expected {hi - lo}")
    bits = engine.shard(shard, n, cutoff, seed, blk0, nblk, local_rounds)
    if world > 1 and exchange == "peer":
        bits += _spanning_rounds_peer(shard, n, seed, engine, c, q, bounds, nblk, local_rounds)
    elif world > 1:
        bits += _spanning_rounds_allgather(shard, seed, engine, c, q, bounds, nblk, local_rounds)
    if world > 1:
        t = torch.tensor([bits], dtype=torch.int64, device=_coll_device(shard))
        dist.all_reduce(t)
        bits = int(t.item())
    return bits


def _spanning_rounds_peer(shard, n, seed, engine, c, q, bounds, nblk, local_rounds) -> int:
    world, rank = dist.get_world_size(), dist.get_rank()
    groups = _groups(world)
    # every rank's shard buffer, mapped into this process (own: its pointer)
    h = torch.tensor(list(engine.peer_handle(shard)), dtype=torch.uint8, device=_coll_device(shard))
    hs = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    ok = torch.ones(1, dtype=torch.int32, device=_coll_device(shard))
    ptr = [0] * world
    err = None
    try:
        for r in range(world):
            ptr[r] = shard.data_ptr() if r == rank else engine.open_peer(bytes(hs[r].cpu().tolist()))
    except Exception as exc:  # noqa: BLE001 - every rank must learn about it before any barrier
        ok.zero_()
        err = exc
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 0:
        raise RuntimeError(f"peer mapping unavailable on at least one rank ({err})")
    eb = shard.element_size()
    bits = 0
    try:
        dist.barrier()  # every rank's local rounds are done before peers are touched
        for r in range(local_rounds + 1, c + 1):
            span = 1 << (r - local_rounds)
            g0 = (rank // span) * span
            p = 1 << (r - 1)
            i = ((rank * nblk) // (2 * p)) * (2 * p)  # first block of the spanning pair
            j, k, l = bounds[i], bounds[i + p], bounds[i + 2 * p]
            starts = [bounds[(g0 + m) * nblk] - j for m in range(span)] + [l - j]
            bases = [ptr[g0 + m] for m in range(span)]
            sseed = substream_seed(seed, r * q + i)
            grp = groups.get(span, g0)
            engine.merge_peers(bases, starts, rank - g0, eb, k - j, l - k, sseed, 1)
            dist.barrier(group=grp)
            if rank == g0:
                bits += engine.merge_peers(bases, starts, 0, eb, k - j, l - k, sseed, 2)
            # the next round's pairs span twice as many ranks: none of them may
            # start touching this pair's buffers before its tail is applied, so
            # the closing barrier is over the NEXT round's group (this one's at
            # the top)
            if r < c:
                nspan = 2 * span
                dist.barrier(group=groups.get(nspan, (rank // nspan) * nspan))
            else:
                dist.barrier(group=grp)
    finally:
        engine.close_peers()
    return bits


def _spanning_rounds_allgather(shard, seed, engine, c, q, bounds, nblk, local_rounds) -> int:
    world, rank = dist.get_world_size(), dist.get_rank()
    blk0 = rank * nblk
    lo, hi = bounds[blk0], bounds[blk0 + nblk]
    bits = 0
    groups = _groups(world)
    sizes = [bounds[(r + 1) * nblk] - bounds[r * nblk] for r in range(world)]
    for r in range(local_rounds + 1, c + 1):
        span = 1 << (r - local_rounds)
        g0 = (rank // span) * span
        p = 1 << (r - 1)
        i = (blk0 // (2 * p)) * (2 * p)  # first block of the spanning pair
        j, k, l = bounds[i], bounds[i + p], bounds[i + 2 * p]
        mx = max(sizes[g0:g0 + span])
        send = torch.empty(mx, dtype=shard.dtype, device=_coll_device(shard))
        send[:shard.numel()] = shard
        parts = [torch.empty_like(send) for _ in range(span)]
        dist.all_gather(parts, send, group=groups.get(span, g0))
        pair = torch.cat([parts[m][:sizes[g0 + m]] for m in range(span)]).to(shard.device)
        pb = engine.merge(pair, 0, k - j, l - j, substream_seed(seed, r * q + i))
        shard.copy_(pair[lo - j:hi - j])
        if rank == g0:
            bits += pb
    return bits


def merge_shuffle_multi(shards: List[torch.Tensor], n: int, cutoff: Optional[int], seed: int) -> int:
    """Single-process multi-GPU form (sk_merge_shuffle_multi): shards[r] is a
    CUDA tensor (any device) holding shard_range(n, cutoff, len(shards), r);
    returns ShuffleReport.bits.  The devices may repeat (e.g. all cuda:0)."""
    cutoff = MERGE_CUTOFF_DEFAULT if cutoff is None else cutoff
    G = len(shards)
    for r, t in enumerate(shards):
        lo, hi = shard_range(n, cutoff, G, r)
        if not t.is_cuda or not t.is_contiguous() or t.numel() != hi - lo:
            raise ValueError(f"shard {r} must be a contiguous CUDA tensor of {hi - lo} elements")
    eb = shards[0].element_size()
    torch.cuda.synchronize()
    ptrs = (ctypes.c_void_p * G)(*[t.data_ptr() for t in shards])
    devs = (ctypes.c_int * G)(*[t.device.index for t in shards])
    bits = ctypes.c_uint64(0)
    _lib.check(_lib.load().sk_merge_shuffle_multi(ptrs, devs, G, eb, n, cutoff, seed & ((1 << 64) - 1),
                                                  ctypes.byref(bits)))
    return int(bits.value)


def simulate_sharded(data: torch.Tensor, n: int, cutoff: Optional[int], seed: int, world: int,
                     engine=None, exchange: str = "allgather") -> int:
    """The sharded schedule of merge_shuffle_sharded executed by ONE process
    over all `world` shards in turn (no collectives): validates the per-shard
    entry point and the cross-round logic on a single device.  exchange =
    "peer" runs the spanning rounds through sk_merge_range_peers with every
    part's phase 1 in turn (the parts are slices of `data`)."""
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
            sseed = substream_seed(seed, rr * q + i)
            if exchange == "peer":
                span = 1 << (rr - local_rounds)
                r0 = i // nblk
                starts = [bounds[(r0 + m) * nblk] - j for m in range(span)] + [l - j]
                eb = data.element_size()
                bases = [data.data_ptr() + eb * bounds[(r0 + m) * nblk] for m in range(span)]
                for m in range(span):
                    engine.merge_peers(bases, starts, m, eb, k - j, l - k, sseed, 1)
                bits += engine.merge_peers(bases, starts, 0, eb, k - j, l - k, sseed, 2)
            else:
                pair = data[j:l].clone()
                bits += engine.merge(pair, 0, k - j, l - j, sseed)
                data[j:l].copy_(pair)
    return bits
