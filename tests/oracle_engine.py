"""CPU engine for the sharded driver (paper_1508_03167_b200.distributed):
the oracle restatement of the reference tasks, so the multi-rank logic runs
over gloo in CPU tests.  Test infrastructure only."""
import numpy as np

from decomp_model import stop_point, stream_bits
from oracle import oracle as O
from paper_1508_03167_b200.shufflers import merge_plan


TILE = 64  # window-0 positions per tile of the emulated peer merge


def _phase1_part(a, off, n1, n2, sseed, part, nparts):
    """Phase 1 of the merge of a[off, off+n1+n2) restricted to the tiles of
    `part` (tiles tau = part, part + nparts, ... of window 0), in place: each
    tile follows its windows V_{h+1} = [n1 + rank'(V_h.start), n1 +
    rank'(V_h.end)) (tests/decomp_model.py merge_phase1_model, the split
    csrc/merge.cu merge_tree_peer_kernel uses).  A tile reads and writes only
    its own windows, so the parts can run in any order, in place."""
    N = n1 + n2
    bits = stream_bits(sseed, N + 1)
    t, _ = stop_point(bits, n1, n2)
    ones = np.concatenate([[0], np.cumsum(bits[:t].astype(np.int64))])

    def rankp(p):
        return int(ones[min(p, t)])
    for u0 in range(part * TILE, n1, nparts * TILE):
        s, e = u0, min(u0 + TILE, n1)
        F = a[off + s:off + e].copy()
        writes = []
        while s < e:
            o0, Fn = rankp(s), []
            for p in range(s, e):
                f = F[p - s]
                if p < t and bits[p]:
                    writes.append((p, a[off + n1 + o0 + len(Fn)]))
                    Fn.append(f)
                else:
                    writes.append((p, f))
            s, e = n1 + o0, n1 + o0 + len(Fn)
            F = np.asarray(Fn, dtype=a.dtype)
        for p, v in writes:
            a[off + p] = v
    return t


class OracleEngine:
    """`whole` (optional): a shared-memory tensor holding every rank's shard
    back to back, standing in for peer memory across CPU processes: phase 1
    merges the tiles of this rank's part in place (_phase1_part), phase 2
    applies the tail insertion of the whole pair (_kernels.py:116-121)."""

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
        off = (bases[0] - self.whole.data_ptr()) // elem_bytes
        a = self.whole.numpy()
        if phase == 1:
            _phase1_part(a, off, n1, n2, sseed, part, len(bases))
            return 0
        bits = stream_bits(sseed, n1 + n2 + 1)
        t, _ = stop_point(bits, n1, n2)
        st = O.state_vec(sseed, 0, 0, 0)
        for k in range(0, t + 1, 64):            # phase 1 consumed t+1 bits
            O.take(st, min(64, t + 1 - k))
        for x in range(t, n1 + n2):              # tail insertion, x >= t >= 1
            m = O.fdr(st, x + 1)
            a[off + x], a[off + m] = a[off + m], a[off + x]
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
