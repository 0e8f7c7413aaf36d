"""Experiment (CPU, numba): can a leaf's 65 535 fast-dice-roller draws be decoded
in parallel segments whose start offsets are guessed?  A segment decoded from a
wrong bit offset is usable once its path of (draw index, offset) pairs meets
the true path (after that both consume the same bits).  For each of 8 random
leaves (m = 65536, bounds i+1 for i = m-1..1, the leaf's own splitmix64 word
stream) and start draws i0, start the decode at true_offset(i0) + d for
d in [-300, 300] \\ {0} and count the draws until the paths meet.

    python scripts/exp_decode_resync.py > profiles/r02_decode_resync.txt
"""
import numpy as np
from numba import njit, uint64

GOLDEN = np.uint64(0x9E3779B97F4A7C15)


@njit(cache=True)
def mix64(z):
    z = (z ^ (z >> uint64(30))) * uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> uint64(27))) * uint64(0x94D049BB133111EB)
    return z ^ (z >> uint64(31))


@njit(cache=True)
def words_of(seed, nw):
    w = np.empty(nw, np.uint64)
    for k in range(nw):
        w[k] = mix64(seed + uint64(k + 1) * uint64(0x9E3779B97F4A7C15))
    return w


@njit(cache=True)
def take(words, o, k):  # k <= 32 bits MSB-first at bit offset o
    w = o >> 6
    b = o & 63
    x = words[w] << uint64(b)
    if b:
        x |= words[w + 1] >> uint64(64 - b)
    return x >> uint64(64 - k)


@njit(cache=True)
def consumed(words, o, b):  # bits one FDR(b) draw consumes from offset o (_kernels.py:64-82)
    v = 1
    c = 0
    o0 = o
    while True:
        k = 0
        vv = v
        while vv < b:
            vv *= 2
            k += 1
        c = (c << k) | int(take(words, o, k))
        o += k
        v = vv
        if c < b:
            return o - o0
        c -= b
        v -= b


@njit(cache=True)
def run(words, m, starts, deltas, out):
    offs = np.zeros(m + 1, np.int64)
    o = 0
    for i in range(m - 1, 0, -1):
        offs[i] = o
        o += consumed(words, o, i + 1)
    for a in range(len(starts)):
        i0 = starts[a]
        for di in range(len(deltas)):
            o = offs[i0] + deltas[di]
            if o < 0:
                out[a, di] = -2
                continue
            t = 0
            i = i0
            while i >= 1 and o != offs[i]:
                o += consumed(words, o, i + 1)
                i -= 1
                t += 1
            out[a, di] = t if i >= 1 else -1  # -1: never met before the leaf ended


def main():
    m = 65536
    rng = np.random.default_rng(1)
    starts = np.array([60000, 40000, 20000, 8000, 3000], dtype=np.int64)
    deltas = np.array([d for d in range(-300, 301) if d != 0], dtype=np.int64)
    res = []
    for _ in range(8):
        seed = np.uint64(rng.integers(0, 2**63))
        words = words_of(seed, m * 17 // 64 + 100)
        out = np.zeros((len(starts), len(deltas)), np.int64)
        run(words, m, starts, deltas, out)
        res.append(out)
    R = np.stack(res)
    print("# start draw i0 | share of wrong starts that never meet the true path | "
          "draws to meet (50/90/99 %) among those that do")
    for si, s in enumerate(starts):
        x = R[:, si, :].ravel()
        x = x[x != -2]
        met = x[x >= 0]
        print(f"{s:6d} | never met {np.mean(x < 0):.3f} | "
              + (" / ".join(str(int(v)) for v in np.percentile(met, [50, 90, 99])) if len(met) else "-"))


if __name__ == "__main__":
    main()
