"""CPU engine for the sharded driver (paper_1508_03167_b200.distributed):
the oracle restatement of the reference tasks, so the multi-rank logic runs
over gloo in CPU tests.  Test infrastructure only."""
import numpy as np

from oracle import oracle as O
from paper_1508_03167_b200.shufflers import merge_plan


class OracleEngine:
    """`whole` (optional): a shared-memory tensor holding every rank's shard
    back to back, so the peer exchange can be emulated across CPU processes:
    phase 1 is a no-op, phase 2 merges the whole pair in place."""

    def __init__(self, whole=None):
        self.whole = whole

    def peer_handle(self, buf):
        off = (buf.data_ptr() - self.whole.data_ptr()) // buf.element_size()
        return bytes(64) + int(off).to_bytes(8, "little")

    def open_peer(self, handle):
        return self.whole.data_ptr() + self.whole.element_size() * int.from_bytes(handle[64:72], "little")

    def close_peers(self):
        pass

    def merge_peers(self, bases, starts, part, elem_bytes, n1, n2, sseed, phase):
        if phase == 1:
            return 0
        off = (bases[0] - self.whole.data_ptr()) // elem_bytes
        st = O.state_vec(sseed, 0, 0, 0)
        O.merge(self.whole.numpy(), off, off + n1, off + n1 + n2, st)
        return int(st[3])

    def shard(self, buf, n, cutoff, seed, blk0, nblk, rounds):
        a = buf.numpy()
        assert a.dtype == np.int64
        c, q, bounds = merge_plan(n, cutoff)
        base = bounds[blk0]
        bits = 0
        for i in range(blk0, blk0 + nblk):
            st = O.state_vec(O.substream_seed(seed, i), 0, 0, 0)
            O.fy_range(a, bounds[i] - base, bounds[i + 1] - base, st)
            bits += int(st[3])
        for r in range(1, rounds + 1):
            p = 1 << (r - 1)
            for i in range(blk0, blk0 + nblk, 2 * p):
                st = O.state_vec(O.substream_seed(seed, r * q + i), 0, 0, 0)
                O.merge(a, bounds[i] - base, bounds[i + p] - base, bounds[i + 2 * p] - base, st)
                bits += int(st[3])
        return bits

    def merge(self, buf, j, k, l, sseed):
        st = O.state_vec(sseed, 0, 0, 0)
        O.merge(buf.numpy(), j, k, l, st)
        return int(st[3])
