"""The multi-rank path with the REAL CUDA engine: two processes (gloo for the
host collectives, one shard each) on the one GPU of the box.

Each rank runs its leaves and local rounds through sk_merge_shuffle_shard,
exports its shard with sk_ipc_get_handle, maps the other rank's shard with
sk_ipc_open (CUDA IPC works between processes on one device as across
NVLink), and the spanning rounds run as the fused peer-memory tree merge
(sk_merge_range_peers phase 1 on each rank's tiles, host barrier, phase 2 by
the span's first rank) -- distributed.merge_shuffle_sharded(exchange="peer"),
the reference's round barrier (shufflers.py:291-297).  The kernels never wait
on each other (the barriers are host-side), so two ranks on one GPU exercise
the real code without standing in for concurrent multi-GPU timing.  The
result must equal the reference permutation (oracle) and every rank must
report the total bit count."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import oracle as O  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, cutoff, seed, dtype, exchange, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1508_03167_b200 import distributed as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_range(n, cutoff, world, rank)
    shard = torch.arange(lo, hi, dtype=dtype, device="cuda")
    bits = D.merge_shuffle_sharded(shard, n, cutoff, seed, exchange=exchange)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"r{rank}.npy"), shard.cpu().numpy().astype(np.int64))
    np.save(os.path.join(out_dir, f"b{rank}.npy"), np.array([bits], dtype=np.int64))
    dist.barrier()
    D.release_peer_maps()
    D.release_groups()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,cutoff,seed,dtype,exchange", [
    (2, (1 << 20) + 12345, 32768, 41, torch.int32, "peer"),
    (2, 1 << 21, 65536, 42, torch.int64, "peer"),
    (4, 3_000_001, 32768, 43, torch.int32, "peer"),
    (2, (1 << 20) + 7, 32768, 44, torch.int64, "allgather"),
])
def test_ranks_on_one_gpu_real_engine(tmp_path, world, n, cutoff, seed, dtype, exchange):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, cutoff, seed, dtype, exchange, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)])
    bits = [int(np.load(tmp_path / f"b{r}.npy")[0]) for r in range(world)]
    ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
    assert all(b == rbits for b in bits)
    assert np.array_equal(got, ref)
