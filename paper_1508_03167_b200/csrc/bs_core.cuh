// bs_core.cuh -- multi-limb naturals for BalancedShuffle (balanced.cu); host
// and device (the host build is a debugging harness, scripts/bs_host_check.cu,
// never part of the product path).
#pragma once
#include <cstdint>
#include "sk_common.cuh"

#ifndef SK_HD
#define SK_HD __host__ __device__
#endif

namespace sk {

SK_HD inline uint32_t bs_clz(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __clz(x);
#else
  return x ? (uint32_t)__builtin_clz(x) : 32u;
#endif
}
SK_HD inline uint32_t bs_ffs(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __ffs(x);
#else
  return (uint32_t)__builtin_ffs((int)x);
#endif
}
SK_HD inline uint32_t bs_umulhi(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }

namespace bn {

SK_HD inline uint32_t trim(const uint32_t* a, uint32_t n) {
  while (n && a[n - 1] == 0) --n;
  return n;
}
SK_HD inline void copy(uint32_t* r, const uint32_t* a, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) r[i] = a[i];
}
SK_HD int cmp(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  if (na != nb) return na < nb ? -1 : 1;
  for (uint32_t i = na; i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}
SK_HD uint32_t bitlen(const uint32_t* a, uint32_t n) { return n ? 32 * n - bs_clz(a[n - 1]) : 0; }
// r = a + b (r may alias a or b)
SK_HD uint32_t add(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  if (na < nb) {
    const uint32_t* t = a; a = b; b = t;
    uint32_t tn = na; na = nb; nb = tn;
  }
  uint64_t c = 0;
  uint32_t i = 0;
  for (; i < nb; ++i) {
    c += (uint64_t)a[i] + b[i];
    r[i] = (uint32_t)c;
    c >>= 32;
  }
  for (; i < na; ++i) {
    c += a[i];
    r[i] = (uint32_t)c;
    c >>= 32;
  }
  if (c) r[na++] = (uint32_t)c;
  return na;
}
// r = a - b, a >= b (r may alias a)
SK_HD uint32_t sub(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  uint32_t br = 0;
  for (uint32_t i = 0; i < na; ++i) {
    const uint64_t s = (uint64_t)(i < nb ? b[i] : 0u) + br;
    const uint32_t ai = a[i];
    r[i] = ai - (uint32_t)s;
    br = (uint64_t)ai < s ? 1u : 0u;
  }
  return trim(r, na);
}
// a *= m (in place)
SK_HD uint32_t mul_small(uint32_t* a, uint32_t na, uint32_t m) {
  uint64_t c = 0;
  for (uint32_t i = 0; i < na; ++i) {
    c += (uint64_t)a[i] * m;
    a[i] = (uint32_t)c;
    c >>= 32;
  }
  if (c) a[na++] = (uint32_t)c;
  return trim(a, na);
}
// a /= d where d divides a exactly (in place): the power of two by a shift,
// the odd part by multiplying with its inverse mod 2^32 from the low limb up
SK_HD uint32_t divexact_small(uint32_t* a, uint32_t na, uint32_t d) {
  const uint32_t s = bs_ffs(d) - 1;
  d >>= s;
  if (s) {
    for (uint32_t i = 0; i < na; ++i) a[i] = (a[i] >> s) | (i + 1 < na ? a[i + 1] << (32 - s) : 0u);
    na = trim(a, na);
  }
  if (d == 1) return na;
  uint32_t inv = d;  // Newton: 3 -> 6 -> 12 -> 24 -> 48 correct bits
  for (int k = 0; k < 4; ++k) inv *= 2u - d * inv;
  uint32_t borrow = 0;
  for (uint32_t i = 0; i < na; ++i) {
    const uint32_t ai = a[i];
    const uint32_t x = ai - borrow;
    const uint32_t q = x * inv;
    a[i] = q;
    borrow = bs_umulhi(q, d) + (ai < borrow ? 1u : 0u);
  }
  return trim(a, na);
}
// q = a / d (q may alias a), returns the remainder
SK_HD uint32_t divmod_small(uint32_t* q, const uint32_t* a, uint32_t na, uint32_t d, uint32_t& nq) {
  uint64_t r = 0;
  for (uint32_t i = na; i-- > 0;) {
    const uint64_t x = (r << 32) | a[i];
    q[i] = (uint32_t)(x / d);
    r = x - (uint64_t)q[i] * d;
  }
  nq = trim(q, na);
  return (uint32_t)r;
}
// r = a * b (r distinct from a and b)
SK_HD uint32_t mul(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  if (!na || !nb) return 0;
  for (uint32_t i = 0; i < na + nb; ++i) r[i] = 0;
  for (uint32_t i = 0; i < na; ++i) {
    const uint64_t ai = a[i];
    uint64_t c = 0;
    for (uint32_t j = 0; j < nb; ++j) {
      c += ai * b[j] + r[i + j];
      r[i + j] = (uint32_t)c;
      c >>= 32;
    }
    r[i + nb] = (uint32_t)c;
  }
  return trim(r, na + nb);
}
// a <<= k (in place; room for the grown number)
SK_HD uint32_t shl(uint32_t* a, uint32_t na, uint32_t k) {
  if (!na) return 0;
  const uint32_t w = k >> 5, s = k & 31;
  uint32_t n2 = na + w + 1;
  for (uint32_t i = n2; i-- > 0;) {
    const int64_t src = (int64_t)i - w;
    const uint32_t hi = (src >= 0 && src < (int64_t)na) ? a[src] : 0u;
    const uint32_t lo = (s && src - 1 >= 0 && src - 1 < (int64_t)na) ? a[src - 1] : 0u;
    a[i] = s ? (hi << s) | (lo >> (32 - s)) : hi;
  }
  return trim(a, n2);
}
// (v << d) compared with b
SK_HD int cmp_shl(const uint32_t* v, uint32_t nv, uint32_t d, const uint32_t* b, uint32_t nb) {
  const uint32_t w = d >> 5, s = d & 31;
  const uint32_t lv = bitlen(v, nv) + d, lb = bitlen(b, nb);
  if (lv != lb) return lv < lb ? -1 : 1;
  for (uint32_t i = nb; i-- > 0;) {
    const int64_t src = (int64_t)i - w;
    const uint32_t hi = (src >= 0 && src < (int64_t)nv) ? v[src] : 0u;
    const uint32_t lo = (s && src - 1 >= 0 && src - 1 < (int64_t)nv) ? v[src - 1] : 0u;
    const uint32_t x = s ? (hi << s) | (lo >> (32 - s)) : hi;
    if (x != b[i]) return x < b[i] ? -1 : 1;
  }
  return 0;
}
// Schoolbook long division: q = a / b, r = a % b (b has >= 2 limbs, a >= b).
// un: na + 1 limbs of work, vn: nb limbs of work.  q, r distinct from a, b.
SK_HD void divmod(uint32_t* q, uint32_t& nq, uint32_t* r, uint32_t& nr, const uint32_t* a, uint32_t na,
                       const uint32_t* b, uint32_t nb, uint32_t* un, uint32_t* vn) {
  const uint32_t s = bs_clz(b[nb - 1]);
  for (uint32_t i = nb; i-- > 0;) vn[i] = s ? (b[i] << s) | (i ? b[i - 1] >> (32 - s) : 0u) : b[i];
  un[na] = s ? a[na - 1] >> (32 - s) : 0u;
  for (uint32_t i = na; i-- > 0;) un[i] = s ? (a[i] << s) | (i ? a[i - 1] >> (32 - s) : 0u) : a[i];
  const uint64_t vt = vn[nb - 1], vs = vn[nb - 2];
  for (int64_t j = (int64_t)na - nb; j >= 0; --j) {
    const uint64_t top = ((uint64_t)un[j + nb] << 32) | un[j + nb - 1];
    uint64_t qh = top / vt, rh = top - qh * vt;
    while (qh >> 32 || qh * vs > ((rh << 32) | un[j + nb - 2])) {
      --qh;
      rh += vt;
      if (rh >> 32) break;
    }
    // un[j .. j+nb] -= qh * vn
    uint64_t carry = 0;  // product carry
    uint32_t br = 0;     // subtraction borrow
    for (uint32_t i = 0; i < nb; ++i) {
      const uint64_t p = qh * vn[i] + carry;
      carry = p >> 32;
      const uint64_t sub_ = (uint64_t)(uint32_t)p + br;
      const uint32_t u = un[i + j];
      un[i + j] = u - (uint32_t)sub_;
      br = (uint64_t)u < sub_ ? 1u : 0u;
    }
    const uint64_t sub_ = carry + br;
    const uint32_t u = un[j + nb];
    un[j + nb] = u - (uint32_t)sub_;
    const bool neg = (uint64_t)u < sub_;
    if (neg) {  // qh was one too large: add vn back
      --qh;
      uint64_t c = 0;
      for (uint32_t i = 0; i < nb; ++i) {
        c += (uint64_t)un[i + j] + vn[i];
        un[i + j] = (uint32_t)c;
        c >>= 32;
      }
      un[j + nb] += (uint32_t)c;
    }
    q[j] = (uint32_t)qh;
  }
  nq = trim(q, na - nb + 1);
  for (uint32_t i = 0; i < nb; ++i) r[i] = s ? (un[i] >> s) | (un[i + 1] << (32 - s)) : un[i];
  nr = trim(r, nb);
}
// r = C(a, b) as the product of its prime powers (Legendre: the exponent of p
// is the number of borrows when subtracting b from a in base p; every prime
// power dividing C(a, b) is <= a, so it fits a limb).  primes: ascending.
SK_HD uint32_t binom(uint32_t* r, uint32_t a, uint32_t b, const uint32_t* primes, uint32_t np) {
  r[0] = 1;
  uint32_t n = 1;
  if (b > a) { r[0] = 0; return 0; }
  if (b > a - b) b = a - b;
  if (b == 0) return 1;
  uint64_t acc = 1;
  for (uint32_t i = 0; i < np && primes[i] <= a; ++i) {
    const uint32_t p = primes[i];
    uint64_t f = 1;
    for (uint64_t pk = p; pk <= a; pk *= p)
      if (a / pk - b / pk - (a - b) / pk) f *= p;
    if (f == 1) continue;
    if (acc * f >> 32) {
      n = mul_small(r, n, (uint32_t)acc);
      acc = f;
    } else {
      acc *= f;
    }
  }
  if (acc > 1) n = mul_small(r, n, (uint32_t)acc);
  return n;
}

}  // namespace bn

constexpr int kBsSmall = 32;  // balanced.py:40 _SMALL_N

// One pair of the singleton schedule that draws (both sides non-empty).
struct BsPair {
  uint32_t j, n1, n2, level;
  uint32_t bidx;       // its class size in the binomial table (m > 64)
  uint64_t rank_off;   // limbs into the rank pool
  uint64_t word_off;   // bytes into the word buffer (level * n + j)
  uint64_t scr_off;    // limbs into the unrank scratch pool (m > 32)
};

SK_HD inline uint32_t bs_limbs(uint32_t m) { return m / 32 + 4; }
SK_HD inline uint64_t bs_scratch_limbs(uint32_t m) { return 20ull * bs_limbs(m); }

// Word w (MSB = bit 64w) of the stream: the prefix bits of a mid-stream
// state, then the splitmix64 words (sk_common.cuh chunk(), host and device).
SK_HD inline uint64_t bs_word(const StreamDesc& d, uint64_t w) {
  const uint64_t g = mix64(d.state + (w + 1) * GOLDEN);
  if (d.plen == 0) return g;
  const uint64_t prev = (w == 0) ? d.buf : mix64(d.state + w * GOLDEN);
  return (prev << (64 - d.plen)) | (g >> d.plen);
}
// bits [o, o + k) of the stream MSB-first, k <= 32
SK_HD inline uint32_t bs_bits(const StreamDesc& sd, uint64_t o, uint32_t k) {
  if (!k) return 0u;
  const uint64_t w = o >> 6;
  const uint32_t s = (uint32_t)(o & 63);
  uint64_t x = bs_word(sd, w) << s;
  if (s + k > 64) x |= bs_word(sd, w + 1) >> (64 - s);
  return (uint32_t)(x >> (64 - k));
}

// A. the ranks: bitstream.py:187-210 random_int(C(m, n1)) per pair, in
// schedule order on one stream; rank of pair p at pool + rank_off as
// [limb count, limbs].  work: 3 numbers of wl limbs.  Returns the bits used.
SK_HD inline uint64_t bs_ranks(const BsPair* pairs, uint32_t npairs, const StreamDesc& sd, const uint32_t* primes,
                               uint32_t nprimes, uint32_t* pool, uint32_t* work, uint32_t wl) {
  uint32_t* B = work;
  uint32_t* v = work + wl;
  uint32_t* c = work + 2 * wl;
  uint32_t nB = 0, cm = 0, cn1 = 0;
  uint64_t o = 0;  // stream offset
  for (uint32_t p = 0; p < npairs; ++p) {
    const BsPair P = pairs[p];
    const uint32_t m = P.n1 + P.n2;
    if (m != cm || P.n1 != cn1) {  // pairs of a level repeat a handful of sizes
      nB = bn::binom(B, m, P.n1, primes, nprimes);
      cm = m;
      cn1 = P.n1;
    }
    // fast dice roller below B (>= 2): v = 1, c = 0
    v[0] = 1;
    uint32_t nv = 1, nc = 0;
    const uint32_t lb = bn::bitlen(B, nB);
    for (;;) {
      // smallest k with v << k >= B
      uint32_t k = lb - bn::bitlen(v, nv);
      if (bn::cmp_shl(v, nv, k, B, nB) < 0) ++k;
      nc = bn::shl(c, nc, k);
      // or in the next k bits: limb i of them is stream bits
      // [o + k - 32(i+1), o + k - 32 i)
      const uint32_t full = k >> 5, part = k & 31, nk = full + (part ? 1u : 0u);
      for (uint32_t i = nc; i < nk; ++i) c[i] = 0;  // (c << k has zeros below bit k)
      for (uint32_t i = 0; i < full; ++i) c[i] |= bs_bits(sd, o + k - 32 * (i + 1), 32);
      if (part) c[full] |= bs_bits(sd, o, part);
      nc = bn::trim(c, nc > nk ? nc : nk);
      o += k;
      nv = bn::shl(v, nv, k);
      if (bn::cmp(c, nc, B, nB) < 0) break;
      nc = bn::sub(c, c, nc, B, nB);
      nv = bn::sub(v, v, nv, B, nB);
    }
    uint32_t* R = pool + P.rank_off;
    R[0] = nc;  // length, then the limbs
    bn::copy(R + 1, c, nc);
  }
  return o;
}

// _unrank_small (balanced.py:78-93): the word of m <= 32 positions with k
// zeros and lexicographic rank r
SK_HD inline void bs_unrank_small(uint32_t m, uint32_t k, uint64_t r, uint8_t* out, const uint64_t* C) {
  uint32_t kk = k;
  for (uint32_t pos = 0; pos < m; ++pos) {
    if (kk == 0) {
      out[pos] = 1;
      continue;
    }
    const uint32_t rem = m - pos - 1;
    const uint64_t cnt = (kk - 1 <= rem) ? C[rem * (kBsSmall + 1) + kk - 1] : 0ull;
    if (r < cnt) {
      out[pos] = 0;
      --kk;
    } else {
      r -= cnt;
      out[pos] = 1;
    }
  }
}

// B. the word of one pair: _unrank_into (balanced.py:146-155) with the split
// of _locate_split (balanced.py:98-143).  The halves are independent
// sub-problems (disjoint output, their own sub-ranks), kept on an explicit
// stack whose sub-ranks live in a LIFO arena.
struct BsTask {
  uint32_t m, k, off, rlen;
  uint64_t rank;  // arena offset of the sub-rank's limbs
};
constexpr int kBsStack = 64;

// a = a * x * y / (u * v), exact: one limb pass per side when the products
// fit a limb
#pragma nv_exec_check_disable
template <class O>
SK_HD inline uint32_t bs_muldiv(uint32_t* a, uint32_t na, uint32_t x, uint32_t y, uint32_t u, uint32_t v) {
  const uint64_t xy = (uint64_t)x * y, uv = (uint64_t)u * v;
  if (xy >> 32) {
    na = O::mul_small(a, na, x);
    na = O::mul_small(a, na, y);
  } else {
    na = O::mul_small(a, na, (uint32_t)xy);
  }
  if (uv >> 32) {
    na = O::divexact_small(a, na, u);
    na = O::divexact_small(a, na, v);
  } else {
    na = O::divexact_small(a, na, (uint32_t)uv);
  }
  return na;
}

// Working numbers of one split (node of m positions): full-size ones hold up
// to m + 1 bits, half-size ones up to m/2 + 1 bits (plus a limb of growth).
struct BsWork {
  uint32_t *wL, *wR, *wU, *wD, *rU, *rD, *cum, *tmp, *q, *rr, *un, *vn;
  // carve from one region: W limbs per full-size number, H per half-size one
  SK_HD static BsWork carve(uint32_t* p, uint32_t W, uint32_t H) {
    BsWork w;
    w.wU = p; p += W;
    w.wD = p; p += W;
    w.cum = p; p += W;
    w.tmp = p; p += W;
    w.un = p; p += W + 2;
    w.wL = p; p += H;
    w.wR = p; p += H;
    w.rU = p; p += H;
    w.rD = p; p += H;
    w.q = p; p += H;
    w.rr = p; p += H;
    w.vn = p;
    return w;
  }
  SK_HD static uint64_t limbs(uint32_t W, uint32_t H) { return 5ull * W + 2 + 7ull * H; }
};

// One split of _unrank_into (balanced.py:146-155): _locate_split
// (balanced.py:98-143) of the rank rk (nr limbs) of a node of m positions
// with k zeros, then divmod(rank - cum, right factor).  Leaves the left
// half's zero count in t, its sub-rank in w.q (nq limbs) and the right half's
// in w.rr (nrr limbs).  O: the serial (SerialOps) or group-cooperative
// (GroupOps<warp or block>, bs_group.cuh) limb arithmetic.
#pragma nv_exec_check_disable
template <class O>
SK_HD inline void bs_split(uint32_t m, uint32_t k, const uint32_t* rk, uint32_t nr, const BsWork& w,
                           const uint32_t* primes, uint32_t nprimes, uint32_t& t, uint32_t& nq, uint32_t& nrr) {
  uint32_t* wL = w.wL;    // C(mL, t0)
  uint32_t* wR = w.wR;    // C(mR, k - t0)
  uint32_t* wU = w.wU;    // weight of the upward block (first: of the block at t0)
  uint32_t* wD = w.wD;    // weight of the downward block
  uint32_t* rU = w.rU;    // right factor of the upward block
  uint32_t* rD = w.rD;    // right factor of the downward block
  uint32_t* cum = w.cum;
  uint32_t* tmp = w.tmp;
  uint32_t* q = w.q;
  uint32_t* rr = w.rr;
  uint32_t* un = w.un;
  uint32_t* vn = w.vn;
  const uint32_t mL = m >> 1, mR = m - mL;
  // _locate_split(mL, mR, k, rank)
  const uint32_t tmin = k > mR ? k - mR : 0u;
  const uint32_t tmax = mL < k ? mL : k;
  uint32_t t0 = (uint32_t)(((uint64_t)k * mL) / (mL + mR));
  t0 = t0 < tmin ? tmin : (t0 > tmax ? tmax : t0);
  uint32_t nL = O::binom(wL, mL, t0, primes, nprimes);
  uint32_t nR = O::binom(wR, mR, k - t0, primes, nprimes);
  uint32_t nU = O::mul(wU, wL, nL, wR, nR);
  t = t0;
  const uint32_t* rf = wR;  // right factor of the chosen block
  uint32_t nrf = nR;
  const uint32_t* base = nullptr;  // rank - cum of the chosen block
  uint32_t nbase = 0;
  if (O::cmp(rk, nr, wU, nU) < 0) {
    base = rk;
    nbase = nr;
  } else {
    uint32_t nc = nU;
    O::copy(cum, wU, nU);
    uint32_t nD = nU;
    O::copy(wD, wU, nU);
    uint32_t nRU = nR, nRD = nR;
    O::copy(rU, wR, nR);
    O::copy(rD, wR, nR);
    uint32_t ut = t0, dt = t0;
    for (;;) {
      if (ut < tmax) {
        const uint32_t j = k - ut;
        // C(mL, ut+1) C(mR, j-1) = C(mL, ut) C(mR, j) (mL-ut)/(ut+1) j/(mR-j+1)
        nU = bs_muldiv<O>(wU, nU, mL - ut, j, ut + 1, mR - j + 1);
        nRU = O::mul_small(rU, nRU, j);
        nRU = O::divexact_small(rU, nRU, mR - j + 1);
        ++ut;
        const uint32_t nt = O::add(tmp, cum, nc, wU, nU);
        if (O::cmp(rk, nr, tmp, nt) < 0) {
          t = ut;
          rf = rU;
          nrf = nRU;
          break;
        }
        { uint32_t* x = cum; cum = tmp; tmp = x; }  // cum += weight
        nc = nt;
      }
      if (dt > tmin) {
        const uint32_t j = k - dt;
        // C(mL, dt-1) C(mR, j+1) = C(mL, dt) C(mR, j) dt/(mL-dt+1) (mR-j)/(j+1)
        nD = bs_muldiv<O>(wD, nD, dt, mR - j, mL - dt + 1, j + 1);
        nRD = O::mul_small(rD, nRD, mR - j);
        nRD = O::divexact_small(rD, nRD, j + 1);
        --dt;
        const uint32_t nt = O::add(tmp, cum, nc, wD, nD);
        if (O::cmp(rk, nr, tmp, nt) < 0) {
          t = dt;
          rf = rD;
          nrf = nRD;
          break;
        }
        { uint32_t* x = cum; cum = tmp; tmp = x; }
        nc = nt;
      }
    }
    nbase = O::sub(tmp, rk, nr, cum, nc);
    base = tmp;
  }
  // (rank_left, rank_right) = divmod(rank - cum, right factor)
  nq = 0;
  nrr = 0;
  if (O::cmp(base, nbase, rf, nrf) < 0) {
    nq = 0;
    O::copy(rr, base, nbase);
    nrr = nbase;
  } else if (nrf == 1) {
    nrr = O::set1(rr, O::divmod_small(q, base, nbase, rf[0], nq));
  } else {
    O::divmod(q, nq, rr, nrr, base, nbase, rf, nrf, un, vn);
  }
}

struct SerialOps {
  SK_HD static uint32_t binom(uint32_t* r, uint32_t a, uint32_t b, const uint32_t* p, uint32_t np) {
    return bn::binom(r, a, b, p, np);
  }
  SK_HD static uint32_t mul(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return bn::mul(r, a, na, b, nb);
  }
  SK_HD static int cmp(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) { return bn::cmp(a, na, b, nb); }
  SK_HD static void copy(uint32_t* r, const uint32_t* a, uint32_t n) { bn::copy(r, a, n); }
  SK_HD static uint32_t add(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return bn::add(r, a, na, b, nb);
  }
  SK_HD static uint32_t sub(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return bn::sub(r, a, na, b, nb);
  }
  SK_HD static uint32_t mul_small(uint32_t* a, uint32_t na, uint32_t m) { return bn::mul_small(a, na, m); }
  SK_HD static uint32_t divexact_small(uint32_t* a, uint32_t na, uint32_t d) { return bn::divexact_small(a, na, d); }
  SK_HD static uint32_t divmod_small(uint32_t* q, const uint32_t* a, uint32_t na, uint32_t d, uint32_t& nq) {
    return bn::divmod_small(q, a, na, d, nq);
  }
  SK_HD static void divmod(uint32_t* q, uint32_t& nq, uint32_t* r, uint32_t& nr, const uint32_t* a, uint32_t na,
                           const uint32_t* b, uint32_t nb, uint32_t* un, uint32_t* vn) {
    bn::divmod(q, nq, r, nr, a, na, b, nb, un, vn);
  }
  SK_HD static uint32_t set1(uint32_t* r, uint32_t v) {
    r[0] = v;
    return v ? 1u : 0u;
  }
};

// The word of M positions with K zeros and rank R0 ([limb count, limbs]) into
// out, serially (one thread); S: 20 * bs_limbs(M) limbs of scratch when M > 32.
// C: the 33 x 33 table of C(a, b) (0 for b > a).
SK_HD inline void bs_word_task(uint32_t M, uint32_t K, const uint32_t* R0, uint8_t* out, uint32_t* S,
                               const uint32_t* primes, uint32_t nprimes, const uint64_t* C) {
  if (M <= (uint32_t)kBsSmall) {
    const uint64_t r = R0[0] == 0 ? 0ull : (R0[0] == 1 ? (uint64_t)R0[1] : ((uint64_t)R0[2] << 32 | R0[1]));
    bs_unrank_small(M, K, r, out, C);
    return;
  }
  const uint32_t W = bs_limbs(M);
  // arena: [0, 2W) pending sub-ranks (LIFO); [2W, ...) working numbers
  uint32_t* wk = S + 2 * W;
  uint32_t* rk = wk;            // the current task's rank
  const BsWork bw = BsWork::carve(wk + W, W, W / 2 + 3);
  BsTask st[kBsStack];
  int sp = 0;
  uint64_t top = 0;  // arena top (limbs)
  st[sp++] = BsTask{M, K, 0, R0[0], top};
  bn::copy(S, R0 + 1, R0[0]);
  top += R0[0];
  while (sp) {
    const BsTask T = st[--sp];
    uint32_t nr = T.rlen;
    bn::copy(rk, S + T.rank, nr);
    top = T.rank;  // its sub-rank is consumed (LIFO)
    uint32_t m = T.m, k = T.k, off = T.off;
    while (m > (uint32_t)kBsSmall) {
      const uint32_t mL = m >> 1, mR = m - mL;
      uint32_t t, nq, nrr;
      bs_split<SerialOps>(m, k, rk, nr, bw, primes, nprimes, t, nq, nrr);
      const uint32_t* q = bw.q;
      const uint32_t* rr = bw.rr;
      // the left half becomes a pending task (its sub-rank on the arena);
      // this loop continues with the right half (balanced.py:152-154)
      if (sp < kBsStack) st[sp++] = BsTask{mL, t, off, nq, top};  // (depth <= log2(m / 32) + 1)
      bn::copy(S + top, q, nq);
      top += nq;
      bn::copy(rk, rr, nrr);
      nr = nrr;
      off += mL;
      m = mR;
      k -= t;
    }
    const uint64_t r = nr == 0 ? 0ull : (nr == 1 ? (uint64_t)rk[0] : ((uint64_t)rk[1] << 32 | rk[0]));
    bs_unrank_small(m, k, r, out + off, C);
  }
}


SK_HD inline void bs_word_pair(const BsPair& P, const uint32_t* pool, uint32_t* scratch, const uint32_t* primes,
                               uint32_t nprimes, uint8_t* words, const uint64_t* C) {
  bs_word_task(P.n1 + P.n2, P.n1, pool + P.rank_off, words + P.word_off, scratch + P.scr_off, primes, nprimes, C);
}

SK_HD inline void bs_small_table(uint64_t* C, uint32_t i0, uint32_t step) {
  for (uint32_t i = i0; i < (kBsSmall + 1) * (kBsSmall + 1); i += step) {
    const uint32_t a = i / (kBsSmall + 1), b = i % (kBsSmall + 1);
    uint64_t v = 0;
    if (b <= a) {  // C(a, b) by the multiplicative formula (exact at every step)
      v = 1;
      for (uint32_t t = 1; t <= b; ++t) v = v * (a - b + t) / t;
    }
    C[i] = v;
  }
}

}  // namespace sk
