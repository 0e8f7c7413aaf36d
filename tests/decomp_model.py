"""Pure-Python models of the data-parallel decompositions the CUDA kernels use.

Test helper only.  Each model is checked against the serial reference semantics
(oracle) in tests/test_decomp_model.py, so the closed forms the kernels implement
are validated on the CPU before any GPU run:

* leaf_apply_model:  Fisher-Yates given its draws, computed by per-target
  successor chains (kernel: csrc/leaf.cu, leaf_apply_kernel).
* merge_phase1_model: the in-place swap-merge phase 1 computed by the
  segment/window chain (kernel: csrc/merge.cu, merge_level_kernel).
* tail_plan_model:   merge phase-2 insertion as a (dst, src) list over the
  touched set (kernel: csrc/plan.cu, tail_plan_kernel).
* spec_decode_model: the leaf's FDR draws decoded in batches of up to 32 steps
  under start-offset hypotheses (kernel: csrc/leaf.cu, leaf_decode_spec_kernel).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
G = 0x9E3779B97F4A7C15


def mix64(z):
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def stream_bits(sseed: int, nbits: int) -> np.ndarray:
    """Bits of a fresh substream, MSB-first per splitmix64 word."""
    nw = (nbits + 63) // 64
    out = np.empty(nw * 64, dtype=np.uint8)
    for w in range(nw):
        word = mix64(sseed + (w + 1) * G)
        for b in range(64):
            out[w * 64 + b] = (word >> (63 - b)) & 1
    return out[:nbits]


class BitCursor:
    def __init__(self, bits, pos=0):
        self.bits, self.pos = bits, pos

    def take(self, k):
        v = 0
        for _ in range(k):
            v = (v << 1) | int(self.bits[self.pos])
            self.pos += 1
        return v

    def fdr(self, bound):
        if bound <= 1:
            return 0
        v, c = 1, 0
        while True:
            k = ((bound + v - 1) // v - 1).bit_length()
            c = (c << k) | self.take(k)
            v <<= k
            if c < bound:
                return c
            c -= bound
            v -= bound


# ---------------------------------------------------------------- leaf ----

def fy_serial(vals, draws):
    a = list(vals)
    m = len(a)
    for i in range(m - 1, 0, -1):
        j = draws[i]
        a[i], a[j] = a[j], a[i]
    return a


def leaf_apply_model(vals, draws):
    """final[i] = orig[src(i)], src by successor chains over per-target lists.

    N(i) = next larger step with the same target; H(x) = first step > x
    targeting x.  final[i] = orig[W(N(i))] or orig[j_i]; final[0] = orig[W(0)];
    W(x) = W(H(x)) if H(x) exists else x.
    """
    m = len(vals)
    buckets = [[] for _ in range(m)]
    for s in range(1, m):          # ascending => each bucket sorted
        buckets[draws[s]].append(s)
    N = [0] * m
    for p in range(m):
        b = buckets[p]
        for k in range(len(b) - 1):
            N[b[k]] = b[k + 1]
    H = [0] * m
    for x in range(m):
        b = buckets[x]
        if b:
            H[x] = b[0] if b[0] > x else (b[1] if len(b) > 1 else 0)

    def W(x):
        while H[x]:
            x = H[x]
        return x
    out = [None] * m
    for i in range(m):
        if i == 0:
            src = W(0)
        else:
            src = W(N[i]) if N[i] else draws[i]
        out[i] = vals[src]
    return out


# --------------------------------------------------------------- merge ----

def merge_serial(vals, n1, n2, bits):
    """Reference _merge on a list with an explicit bit array; returns
    (out, t, a_exhausted, phase1_out, tail_draws, bits_used)."""
    a = list(vals)
    cur = BitCursor(bits)
    i, mid, n = 0, n1, n1 + n2
    if n1 == 0 or n2 == 0:
        return a, None, None, list(a), [], 0
    while True:
        if cur.take(1) == 0:
            if i == mid:
                aex = True
                break
        else:
            if mid == n:
                aex = False
                break
            a[i], a[mid] = a[mid], a[i]
            mid += 1
        i += 1
    t = i
    p1 = list(a)
    draws = []
    while i < n:
        m = cur.fdr(i + 1)
        draws.append(m)
        a[i], a[m] = a[m], a[i]
        i += 1
    return a, t, aex, p1, draws, cur.pos


def stop_point(bits, n1, n2):
    z = o = 0
    for u in range(len(bits)):
        if bits[u]:
            if o == n2:
                return u, False
            o += 1
        else:
            if z == n1:
                return u, True
            z += 1
    raise ValueError("bit array too short")


def merge_phase1_model(vals, n1, n2, bits, T=16):
    """Window-chain form of phase 1: every A tile [u0,u0+T) walks windows
    V_0=[u0,u1), V_{h+1}=[n1+rank'(start), n1+rank'(end)); zeros emit the
    carried A value, ones emit B[rank'] and carry A to the next window."""
    N = n1 + n2
    t, aex = stop_point(bits, n1, n2)
    ones = np.concatenate([[0], np.cumsum(bits[:t].astype(np.int64))])

    def rankp(p):  # ones in [0, min(p, t))
        return int(ones[min(p, t)])
    out = [None] * N
    for u0 in range(0, n1, T):
        u1 = min(u0 + T, n1)
        F = [vals[u] for u in range(u0, u1)]
        s, e = u0, u1
        while s < e:
            Fn = []
            o0 = rankp(s)
            r = 0
            for p in range(s, e):
                f = F[p - s]
                if p >= t:
                    out[p] = f
                elif bits[p] == 0:
                    out[p] = f
                else:
                    out[p] = vals[n1 + o0 + r]
                    Fn.append(f)
                    r += 1
            s, e = n1 + o0, n1 + o0 + r
            F = Fn
    # segments cover [0, X), X = first fixed point of S -> n1 + rank'(S) from n1;
    # past X the A queue is empty: ones up to t and (A-exhausted) the untouched
    # B suffix, both identity.
    X = n1
    while n1 + rankp(X) != X:
        X = n1 + rankp(X)
    for p in range(X, N):
        assert out[p] is None
        out[p] = vals[p]
    assert all(v is not None for v in out)
    return out, t, aex


# ---------------------------------------------------------------- tail ----

def tail_plan_model(N, t, draws):
    """(dst, src) list: final[dst] = P1[src] for every touched position of the
    ascending insertion steps x=t..N-1, swap(x, m_x), m_x <= x."""
    L = N - t
    recs = [(draws[k], t + k) for k in range(L)]       # (m, x), x ascending
    order = sorted(range(L), key=lambda k: (recs[k][0], k))   # stable by m
    pred = [None] * L
    last_of = {}
    for idx, k in enumerate(order):
        if idx > 0 and recs[order[idx - 1]][0] == recs[k][0]:
            pred[k] = recs[order[idx - 1]][1]
        last_of[recs[k][0]] = recs[k][1]
    plan = []
    keyed = set()
    for q, xl in last_of.items():
        if xl > q:
            plan.append((q, xl))
            keyed.add(q)
    for k in range(L):
        x = t + k
        if x in keyed:
            continue
        r = k
        while True:
            q, xr = recs[r]
            y = pred[r]
            if y is not None and y > q:
                src = y
                break
            if q == xr:
                src = xr
                break
            if q < t:
                src = q
                break
            r = q - t
        plan.append((x, src))
    return plan


def tail_apply(p1, plan):
    out = list(p1)
    for d, s in plan:
        out[d] = p1[s]
    return out


# ------------------------------------------------- speculative leaf decode ----
def _bits_at(bits, p, k):
    v = 0
    for t in range(k):
        v = (v << 1) | int(bits[p + t])
    return v


def _k_of(v, b):
    k = 0
    while (v << k) < b:
        k += 1
    return k


def spec_decode_model(m, bits, H=2, lanes=16):
    """Draws j_i (i = m-1 .. 1, bound i+1) of a leaf from `bits`, decoded as
    leaf_decode_spec_kernel does: a batch = up to `lanes` consecutive steps with
    the same first-iteration width K and the same second-iteration width k1;
    draw l is evaluated at o + l*K + h*k1 for h < H (the kernel: 16 draws x 2
    hypotheses, one per lane); the first rejection
    under hypothesis h hands the later lanes to h+1, a double rejection is
    finished serially and ends the batch.  Returns (draws, bits consumed,
    batches)."""
    draws = [0] * max(m, 1)
    o, i, batches = 0, m - 1, 0
    while i >= 1:
        n = min(lanes, i)
        K = i.bit_length()
        if (i & (i + 1)) == 0:          # bound a power of two: never rejects, alone
            neff, k1 = 1, 1
        else:
            k1 = _k_of((1 << K) - (i + 1), i + 1)
            neff = 0
            while neff < n:
                s = i - neff
                if s.bit_length() != K or (1 << K) == s + 1 or _k_of((1 << K) - (s + 1), s + 1) != k1:
                    break
                neff += 1
        ev = []
        for h in range(H):
            row = []
            for l in range(neff):
                if h * k1 > 64:
                    row.append(None)
                    continue
                b = i - l + 1
                off = o + l * K + h * k1
                c = _bits_at(bits, off, K)
                if c >= b:
                    c2 = ((c - b) << k1) | _bits_at(bits, off + K, k1)
                    row.append((True, c2 >= b, c2))
                else:
                    row.append((False, False, c))
            ev.append(row)
        h, start = 0, 0
        while True:
            if h == H or h * k1 > 64:
                consumed, extra = start, h * k1
                break
            f = next((l for l in range(start, neff) if ev[h][l][0]), None)
            for l in range(start, neff if f is None else f + 1):
                draws[i - l] = ev[h][l][2]
            if f is None:
                consumed, extra = neff, h * k1
                break
            if ev[h][f][1]:               # rejected twice: finish serially, end of batch
                b = i - f + 1
                c, v = ev[h][f][2] - b, (((1 << K) - b) << k1) - b
                p = o + f * K + h * k1 + K + k1
                while True:
                    k = _k_of(v, b)
                    c = (c << k) | _bits_at(bits, p, k)
                    p += k
                    v <<= k
                    if c < b:
                        break
                    c -= b
                    v -= b
                draws[i - f] = c
                consumed, extra = f + 1, p - (o + (f + 1) * K)
                break
            h, start = h + 1, f + 1
            if start == neff:
                consumed, extra = neff, h * k1
                break
        batches += 1
        o += consumed * K + extra
        i -= consumed
    return draws, o, batches
