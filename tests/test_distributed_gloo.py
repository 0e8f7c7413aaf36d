"""Multi-rank path of the sharded MergeShuffle (world 2 and 4, gloo on CPU):
contiguous shards, local leaves/rounds, all-gather exchange for the spanning
rounds -- identical permutation and bit count to the 1-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, cutoff, seed, out_dir, exchange="allgather", whole=None):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle_engine import OracleEngine
    from paper_1508_03167_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_range(n, cutoff, world, rank)
    if whole is not None:  # peer exchange: shards are views of one shared-memory array
        shard = whole[lo:hi]
        shard.copy_(torch.arange(lo, hi, dtype=torch.int64))
    else:
        shard = torch.arange(lo, hi, dtype=torch.int64)
    bits = D.merge_shuffle_sharded(shard, n, cutoff, seed, engine=OracleEngine(whole), exchange=exchange)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), shard.numpy())
    np.save(os.path.join(out_dir, f"b{rank}.npy"), np.array([bits], dtype=np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,cutoff,seed", [(2, 5000, 300, 1), (4, 5000, 300, 2), (4, 10_003, 1000, 3),
                                                 (2, 1 << 16, 4096, 4)])
def test_sharded_equals_single(tmp_path, world, n, cutoff, seed):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, cutoff, seed, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)])
    bits = [int(np.load(tmp_path / f"b{r}.npy")[0]) for r in range(world)]
    ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
    assert np.array_equal(got, ref)
    assert all(b == rbits for b in bits)


@pytest.mark.parametrize("world,n,cutoff,seed", [(2, 5000, 300, 5), (4, 10_003, 1000, 6)])
def test_sharded_peer_exchange_orchestration(tmp_path, world, n, cutoff, seed):
    # the peer-exchange driver (handle exchange, phase-1 parts, barrier,
    # phase-2 tail by the span's first rank, bit accounting) over gloo; the
    # "peer memory" is one shared-memory array
    port = _free_port()
    whole = torch.zeros(n, dtype=torch.int64).share_memory_()
    mp.spawn(_worker, args=(world, port, n, cutoff, seed, str(tmp_path), "peer", whole), nprocs=world, join=True)
    bits = [int(np.load(tmp_path / f"b{r}.npy")[0]) for r in range(world)]
    ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
    assert np.array_equal(whole.numpy(), ref)
    assert all(b == rbits for b in bits)


def test_shard_layout_rules():
    from paper_1508_03167_b200 import distributed as D
    with pytest.raises(ValueError):
        D.shard_layout(1000, 10, 3)       # not a power of two
    with pytest.raises(ValueError):
        D.shard_layout(100, 100, 2)       # q = 1 < world
    c, q, bounds, nblk, local = D.shard_layout(1 << 20, 65536, 8)
    assert (c, q, nblk, local) == (4, 16, 2, 1)


def test_simulated_sharding_with_oracle_engine():
    from oracle_engine import OracleEngine
    from paper_1508_03167_b200 import distributed as D
    n, cutoff, seed = 3000, 100, 9
    for world in (1, 2, 4, 8):
        data = torch.arange(n, dtype=torch.int64)
        bits = D.simulate_sharded(data, n, cutoff, seed, world, engine=OracleEngine())
        ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
        assert np.array_equal(data.numpy(), ref) and bits == rbits
