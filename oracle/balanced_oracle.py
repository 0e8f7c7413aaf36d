"""CPU restatement of the reference's BalancedShuffle (SURVEY.md section 8 row
F1) with Python integers.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker for
sk_balanced_shuffle on random sizes and stream states; the product package
never imports it.  Pinned to the reference's own outputs
(tests/golden/balanced.json, balanced_big.json) by tests/test_oracle_balanced.py.

Follows (paths relative to the reference pkg/src/shufflekit/):
  * the bit stream: bitstream.py:134-181 (take: MSB-first, leftover bits of the
    last splitmix64 word kept) -- restated over the 4-word state
    (state, buffered bits, their count, consumed);
  * random_int: bitstream.py:187-210 (fast dice roller, any bound);
  * the schedule: shufflers.py:108-130 (singleton_rounds), pairs with an empty
    side skipped (balanced.py:238-239);
  * per pair: one roll below C(m, n1) (balanced.py:158-164), the recursive
    halving (balanced.py:146-155) with the split point scanned outward from
    the mode (balanced.py:98-143), m <= 32 by the lexicographic walk
    (balanced.py:78-93), the interleave (balanced.py:198-216).
"""
from __future__ import annotations

from math import comb

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class Stream:
    """The reference BitSource's bit order over its 4-word state."""

    def __init__(self, state_tuple):
        self.sm, self.buf, self.nbuf, self.used = (int(v) for v in state_tuple)

    def bits(self, k: int) -> int:
        out, need = 0, k
        while need:
            if self.nbuf == 0:
                self.sm = (self.sm + GOLDEN) & MASK64
                self.buf, self.nbuf = _mix(self.sm), 64
            g = min(need, self.nbuf)
            self.nbuf -= g
            out = (out << g) | (self.buf >> self.nbuf)
            self.buf &= (1 << self.nbuf) - 1
            need -= g
        self.used += k
        return out

    def below(self, bound: int) -> int:
        """Uniform in [0, bound): the batched fast dice roller."""
        if bound < 1:
            raise ValueError("bound must be >= 1")
        v, c = 1, 0
        while bound > 1:
            k = 0
            while (v << k) < bound:
                k += 1
            c = (c << k) | self.bits(k)
            v <<= k
            if c < bound:
                return c
            c, v = c - bound, v - bound
        return 0

    def state(self):
        return (self.sm, self.buf, self.nbuf, self.used)


def _small_word(m: int, zeros: int, r: int):
    w = []
    for pos in range(m):
        if zeros == 0:
            w.append(1)
            continue
        first = comb(m - pos - 1, zeros - 1)  # words with a 0 here come first
        if r < first:
            w.append(0)
            zeros -= 1
        else:
            w.append(1)
            r -= first
    return w


def _split(mL: int, mR: int, zeros: int, r: int):
    """Zero count of the left half and the two sub-ranks: blocks of weight
    C(mL, t) C(mR, zeros - t) in the order t0, t0+1, t0-1, t0+2, ..."""
    lo_t, hi_t = max(0, zeros - mR), min(mL, zeros)
    t0 = min(max((zeros * mL) // (mL + mR), lo_t), hi_t)
    order = [t0]
    up, dn = t0, t0
    while up < hi_t or dn > lo_t:
        if up < hi_t:
            up += 1
            order.append(up)
        if dn > lo_t:
            dn -= 1
            order.append(dn)
    for t in order:
        right = comb(mR, zeros - t)
        weight = comb(mL, t) * right
        if r < weight:
            return t, r // right, r % right
        r -= weight
    raise AssertionError("rank outside the class")


def word(m: int, zeros: int, r: int):
    """The composition word (0 = left element) of rank r among C(m, zeros)."""
    if m <= 32:
        return _small_word(m, zeros, r)
    mL = m >> 1
    t, rl, rr = _split(mL, m - mL, zeros, r)
    return word(mL, t, rl) + word(m - mL, zeros - t, rr)


def pairs(n: int):
    """(j, n1, n2) of singleton_rounds(n) in schedule order, both sides non-empty."""
    c = (n - 1).bit_length() if n > 1 else 0
    q = 1 << c
    p = 1
    while p < q:
        for i in range(0, q, 2 * p):
            j, k, l = (n * i) >> c, (n * (i + p)) >> c, (n * min(i + 2 * p, q)) >> c
            if k > j and l > k:
                yield j, k - j, l - k
        p *= 2


def balanced_shuffle(arr, state_tuple):
    """Permute list arr in place; returns (bits consumed, end state)."""
    s = Stream(state_tuple)
    used0 = s.used
    for j, n1, n2 in pairs(len(arr)):
        m = n1 + n2
        w = word(m, n1, s.below(comb(m, n1)))
        left, right = arr[j:j + n1], arr[j + n1:j + m]
        a = b = 0
        for t in range(m):
            if w[t]:
                arr[j + t] = right[b]
                b += 1
            else:
                arr[j + t] = left[a]
                a += 1
    return s.used - used0, s.state()
