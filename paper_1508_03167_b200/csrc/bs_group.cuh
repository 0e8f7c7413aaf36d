// bs_group.cuh -- group-cooperative multi-limb naturals for the large pairs
// of BalancedShuffle (balanced.cu): a warp (WarpG) or a whole block (BlockG)
// works on one number.  Same number format and semantics as the serial bn::
// functions of bs_core.cuh (little-endian 32-bit limbs, tracked lengths);
// every function is called by all threads of the group with uniform
// arguments and returns uniform results.  Thread t works on the contiguous
// chunk [t*L, (t+1)*L) of the limbs (L = ceil(span / group size)); the carry
// (or borrow) that leaves a chunk is handed to the next thread, which adds
// (subtracts) it at its chunk's bottom, in rounds until none is left (almost
// always one).  A division by a small number runs top-down, each chunk's
// incoming remainder from a suffix scan of the chunks' affine remainder maps
// r -> (r * 2^(32 len) + value) mod d.
#pragma once
#include "bs_core.cuh"

namespace sk {
namespace gp {

constexpr unsigned kFull = 0xffffffffu;

// x / d and x % d for d >= 2 by a reciprocal (minv = floor((2^64 - 1) / d))
struct Div {
  uint64_t d, minv;
  __device__ __forceinline__ explicit Div(uint64_t dd) : d(dd), minv(~0ull / dd) {}
  __device__ __forceinline__ uint64_t qr(uint64_t x, uint64_t& r) const {
    uint64_t q = __umul64hi(x, minv);
    r = x - q * d;
    if (r >= d) { ++q; r -= d; }
    return q;
  }
  __device__ __forceinline__ uint64_t mod(uint64_t x) const {
    uint64_t r;
    qr(x, r);
    return r;
  }
};

// within a warp: the suffix composition C_l = f_l o ... o f_31 of the lanes'
// maps f(r) = r * P + V (mod d); returns C_{l+1}'s (P, V) (identity for lane 31)
__device__ __forceinline__ void warp_suffix_maps(uint64_t& P, uint64_t& V, const Div& D) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t s = 1; s < 32; s <<= 1) {
    const uint64_t P2 = __shfl_down_sync(kFull, P, s), V2 = __shfl_down_sync(kFull, V, s);
    if (lane + s < 32) {  // f_this o f_upper: r -> (r * P2 + V2) * P + V
      V = D.mod(D.mod(V2 * P) + V);
      P = D.mod(P2 * P);
    }
  }
}

// A warp is the group.
struct WarpG {
  __device__ static __forceinline__ uint32_t id() { return threadIdx.x & 31; }
  __device__ static __forceinline__ uint32_t size() { return 32; }
  __device__ static __forceinline__ void sync() { __syncwarp(); }
  __device__ static __forceinline__ uint64_t from_below(uint64_t v) {  // thread id-1's value (0 for thread 0)
    const uint64_t u = __shfl_up_sync(kFull, v, 1);
    return id() == 0 ? 0ull : u;
  }
  __device__ static __forceinline__ uint64_t from(uint64_t v, uint32_t t) { return __shfl_sync(kFull, v, t); }
  __device__ static __forceinline__ bool any(bool p) { return __any_sync(kFull, p); }
  __device__ static __forceinline__ uint32_t max(uint32_t v) { return __reduce_max_sync(kFull, v); }
  __device__ static __forceinline__ int top_nonzero(int s) {  // the highest thread's nonzero value
    const uint32_t m = __ballot_sync(kFull, s != 0);
    return m ? __shfl_sync(kFull, s, 31 - __clz(m)) : 0;
  }
  // remainder entering this thread's chunk (its maps: r -> r * P + V)
  __device__ static __forceinline__ uint64_t suffix_remainder(uint64_t P, uint64_t V, const Div& D) {
    warp_suffix_maps(P, V, D);
    const uint64_t r = __shfl_down_sync(kFull, V, 1);
    return id() == 31 ? 0ull : r;
  }
};

// The whole block is the group (blockDim.x a multiple of 32, <= 1024).
struct BlockG {
  __device__ static __forceinline__ uint32_t id() { return threadIdx.x; }
  __device__ static __forceinline__ uint32_t size() { return blockDim.x; }
  __device__ static __forceinline__ void sync() { __syncthreads(); }
  __device__ static uint64_t* buf() {
    __shared__ uint64_t b[64];
    return b;
  }
  __device__ static uint64_t from_below(uint64_t v) {
    uint64_t* b = buf();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 31) b[w] = v;
    __syncthreads();
    uint64_t u = __shfl_up_sync(kFull, v, 1);
    if (lane == 0) u = w ? b[w - 1] : 0ull;
    __syncthreads();
    return u;
  }
  __device__ static uint64_t from(uint64_t v, uint32_t t) {
    uint64_t* b = buf();
    if (threadIdx.x == t) b[0] = v;
    __syncthreads();
    const uint64_t u = b[0];
    __syncthreads();
    return u;
  }
  __device__ static bool any(bool p) { return __syncthreads_or(p ? 1 : 0) != 0; }
  __device__ static uint32_t max(uint32_t v) {
    uint64_t* b = buf();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t m = __reduce_max_sync(kFull, v);
    if (lane == 0) b[w] = m;
    __syncthreads();
    uint32_t r = 0;
    for (uint32_t k = 0; k < nw; ++k) r = r > (uint32_t)b[k] ? r : (uint32_t)b[k];
    __syncthreads();
    return r;
  }
  __device__ static int top_nonzero(int s) {
    uint64_t* b = buf();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t m = __ballot_sync(kFull, s != 0);
    const int ws = m ? __shfl_sync(kFull, s, 31 - __clz(m)) : 0;
    if (lane == 0) b[w] = (uint64_t)(int64_t)ws;
    __syncthreads();
    int r = 0;
    for (uint32_t k = nw; k-- > 0;)
      if (b[k]) { r = (int)(int64_t)b[k]; break; }
    __syncthreads();
    return r;
  }
  __device__ static uint64_t suffix_remainder(uint64_t P, uint64_t V, const Div& D) {
    uint64_t* b = buf();
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    warp_suffix_maps(P, V, D);  // C_l within the warp
    if (lane == 0) {            // the warp's whole map
      b[2 * w] = P;
      b[2 * w + 1] = V;
    }
    __syncthreads();
    // S = T_{w+1} o ... o T_{nw-1} applied to 0: fold from the top warp down
    uint64_t r0 = 0;
    for (uint32_t k = nw; k-- > w + 1;) r0 = D.mod(D.mod(r0 * b[2 * k]) + b[2 * k + 1]);
    __syncthreads();
    // then the lanes above in this warp: C_{l+1}(r0)
    const uint64_t P1 = __shfl_down_sync(kFull, P, 1), V1 = __shfl_down_sync(kFull, V, 1);
    return lane == 31 ? r0 : D.mod(D.mod(r0 * P1) + V1);
  }
};

// chunk of this thread over [0, S)
template <class G>
__device__ __forceinline__ void chunk_of(uint32_t S, uint32_t& lo, uint32_t& hi) {
  const uint32_t L = (S + G::size() - 1) / G::size();
  lo = min(G::id() * L, S);
  hi = min(lo + L, S);
}

// Carry (borrow) hand-off between chunks: every thread passes what leaves its
// chunk to the thread above, which adds (subtracts) it at its chunk's bottom
// (at limb lo + skip in the first round); what leaves a chunk again goes up
// in the next round -- rounds end when no thread has anything to pass, almost
// always after the first.  Returns what escapes above the last thread.
template <class G>
__device__ uint64_t ripple_add(uint32_t* r, uint32_t lo, uint32_t hi, uint64_t cout, uint32_t skip = 0) {
  uint64_t esc = 0;
  for (;;) {
    const uint64_t cin = G::from_below(cout);
    esc += G::from(cout, G::size() - 1);
    if (!G::any(cin != 0)) break;
    uint64_t c = cin;
    for (uint32_t i = lo + skip; i < hi && c; ++i) {
      const uint64_t sm = (uint64_t)r[i] + (c & 0xffffffffull);
      r[i] = (uint32_t)sm;
      c = (c >> 32) + (sm >> 32);
    }
    skip = 0;
    cout = c;
  }
  G::sync();
  return esc;
}
template <class G>
__device__ uint64_t ripple_sub(uint32_t* r, uint32_t lo, uint32_t hi, uint64_t bout) {
  uint64_t esc = 0;
  for (;;) {
    const uint64_t bin = G::from_below(bout);
    esc += G::from(bout, G::size() - 1);
    if (!G::any(bin != 0)) break;
    uint64_t b = bin;
    for (uint32_t i = lo; i < hi && b; ++i) {
      const uint32_t x = r[i], lv = (uint32_t)b;
      r[i] = x - lv;
      b = (b >> 32) + (x < lv ? 1u : 0u);
    }
    bout = b;
  }
  G::sync();
  return esc;
}

template <class G>
__device__ uint32_t trim(const uint32_t* a, uint32_t n) {
  uint32_t lo, hi;
  chunk_of<G>(n, lo, hi);
  uint32_t top = 0;
  for (uint32_t i = hi; i > lo; --i)
    if (a[i - 1]) { top = i; break; }
  return G::max(top);
}
template <class G>
__device__ void copy(uint32_t* r, const uint32_t* a, uint32_t n) {
  G::sync();
  for (uint32_t i = G::id(); i < n; i += G::size()) r[i] = a[i];
  G::sync();
}
template <class G>
__device__ int cmp(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  if (na != nb) return na < nb ? -1 : 1;
  uint32_t lo, hi;
  chunk_of<G>(na, lo, hi);
  int s = 0;
  for (uint32_t i = hi; i > lo; --i)
    if (a[i - 1] != b[i - 1]) { s = a[i - 1] < b[i - 1] ? -1 : 1; break; }
  return G::top_nonzero(s);
}
template <class G>
__device__ uint32_t bitlen(const uint32_t* a, uint32_t n) { return n ? 32 * n - __clz(a[n - 1]) : 0; }
// r = a + b (r may alias a or b)
template <class G>
__device__ uint32_t add(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  const uint32_t S = max(na, nb) + 1;
  uint32_t lo, hi;
  chunk_of<G>(S, lo, hi);
  uint64_t c = 0;
  for (uint32_t i = lo; i < hi; ++i) {
    c += (uint64_t)(i < na ? a[i] : 0u) + (i < nb ? b[i] : 0u);
    r[i] = (uint32_t)c;
    c >>= 32;
  }
  ripple_add<G>(r, lo, hi, c);
  return trim<G>(r, S);
}
// r = a - b, a >= b (r may alias a)
template <class G>
__device__ uint32_t sub(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  uint32_t lo, hi;
  chunk_of<G>(na, lo, hi);
  uint32_t br = 0;
  for (uint32_t i = lo; i < hi; ++i) {
    const uint64_t s = (uint64_t)(i < nb ? b[i] : 0u) + br;
    const uint32_t ai = a[i];
    r[i] = ai - (uint32_t)s;
    br = (uint64_t)ai < s ? 1u : 0u;
  }
  ripple_sub<G>(r, lo, hi, br);
  return trim<G>(r, na);
}
// a *= m (in place; a has room for one more limb)
template <class G>
__device__ uint32_t mul_small(uint32_t* a, uint32_t na, uint32_t m) {
  const uint32_t S = na + 1;
  uint32_t lo, hi;
  chunk_of<G>(S, lo, hi);
  uint64_t c = 0;
  uint32_t i = lo;
  // (loads batched eight at a time: the walk is a carry chain, the loads are not)
  for (const uint32_t hn = min(hi, na); i + 8 <= hn; i += 8) {
    uint32_t x[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = a[i + e];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      c += (uint64_t)x[e] * m;
      a[i + e] = (uint32_t)c;
      c >>= 32;
    }
  }
  for (; i < hi; ++i) {
    c += (uint64_t)(i < na ? a[i] : 0u) * m;
    a[i] = (uint32_t)c;
    c >>= 32;
  }
  ripple_add<G>(a, lo, hi, c);
  return trim<G>(a, S);
}
// q = a / d (q may alias a), returns the remainder; d >= 2
template <class G>
__device__ uint32_t div_small(uint32_t* q, const uint32_t* a, uint32_t na, uint32_t d, uint32_t& nq) {
  uint32_t lo, hi;
  chunk_of<G>(na, lo, hi);
  const Div D(d);
  // this chunk's value mod d (loads batched) and 2^(32 len) mod d (by squaring)
  uint64_t V = 0, P = 1;
  {
    uint32_t i = hi;
    for (; i >= lo + 8; i -= 8) {
      uint32_t x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = a[i - 1 - e];
#pragma unroll
      for (int e = 0; e < 8; ++e) V = D.mod((V << 32) | x[e]);
    }
    for (; i > lo; --i) V = D.mod((V << 32) | a[i - 1]);
    uint64_t base = D.mod(1ull << 32);
    for (uint32_t e = hi - lo; e; e >>= 1) {
      if (e & 1) P = D.mod(P * base);
      base = D.mod(base * base);
    }
  }
  // the remainder entering this chunk: the maps r -> r * P + V of the
  // chunks above, the top one applied first
  uint64_t r = G::suffix_remainder(P, V, D);
  G::sync();
  {
    uint32_t i = hi;
    for (; i >= lo + 8; i -= 8) {
      uint32_t x[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = a[i - 1 - e];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        uint64_t rr;
        q[i - 1 - e] = (uint32_t)D.qr((r << 32) | x[e], rr);
        r = rr;
      }
    }
    for (; i > lo; --i) {
      uint64_t rr;
      q[i - 1] = (uint32_t)D.qr((r << 32) | a[i - 1], rr);
      r = rr;
    }
  }
  const uint32_t rem = (uint32_t)G::from(r, 0);
  G::sync();
  nq = trim<G>(q, na);
  return rem;
}
// a /= d, d divides a (in place)
template <class G>
__device__ uint32_t divexact_small(uint32_t* a, uint32_t na, uint32_t d) {
  if (d == 1) return na;
  uint32_t nq;
  div_small<G>(a, a, na, d, nq);
  return nq;
}
// r = a << k (r distinct from a; room for na + k/32 + 1 limbs)
template <class G>
__device__ uint32_t shl(uint32_t* r, const uint32_t* a, uint32_t na, uint32_t k) {
  if (!na) return 0;
  const uint32_t w = k >> 5, s = k & 31, S = na + w + 1;
  G::sync();
  for (uint32_t i = G::id(); i < S; i += G::size()) {
    const int64_t src = (int64_t)i - w;
    const uint32_t hi = (src >= 0 && src < (int64_t)na) ? a[src] : 0u;
    const uint32_t lo = (s && src - 1 >= 0 && src - 1 < (int64_t)na) ? a[src - 1] : 0u;
    r[i] = s ? (hi << s) | (lo >> (32 - s)) : hi;
  }
  G::sync();
  return trim<G>(r, S);
}
// (v << d) compared with b
template <class G>
__device__ int cmp_shl(const uint32_t* v, uint32_t nv, uint32_t d, const uint32_t* b, uint32_t nb) {
  const uint32_t lv = bitlen<G>(v, nv) + d, lb = bitlen<G>(b, nb);
  if (lv != lb) return lv < lb ? -1 : 1;
  const uint32_t w = d >> 5, s = d & 31;
  uint32_t lo, hi;
  chunk_of<G>(nb, lo, hi);
  int sg = 0;
  for (uint32_t i = hi; i > lo; --i) {
    const int64_t src = (int64_t)(i - 1) - w;
    const uint32_t h = (src >= 0 && src < (int64_t)nv) ? v[src] : 0u;
    const uint32_t l = (s && src - 1 >= 0 && src - 1 < (int64_t)nv) ? v[src - 1] : 0u;
    const uint32_t x = s ? (h << s) | (l >> (32 - s)) : h;
    if (x != b[i - 1]) { sg = x < b[i - 1] ? -1 : 1; break; }
  }
  return G::top_nonzero(sg);
}
// r = a * b (r distinct): lane l owns the output columns of its chunk (column
// sums with a 96-bit running carry); the carries out of the chunks are then
// added by lane 0
template <class G>
__device__ uint32_t mul(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  if (!na || !nb) return 0;
  const uint32_t S = na + nb;
  if (S < 3 * G::size()) {  // short: one thread (the chunks would be shorter than a carry)
    G::sync();
    if (G::id() == 0) bn::mul(r, a, na, b, nb);
    G::sync();
    return trim<G>(r, S);
  }
  uint32_t lo, hi;
  chunk_of<G>(S, lo, hi);
  uint64_t clo = 0;  // running carry, bits 0..63
  uint32_t chi = 0;  // bits 64..95
  for (uint32_t c = lo; c < hi; ++c) {
    uint64_t slo = clo, shi = chi;
    const uint32_t i0 = c + 1 > nb ? c + 1 - nb : 0u, i1 = min(c + 1, na);
    for (uint32_t i = i0; i < i1; ++i) {
      const uint64_t p = (uint64_t)a[i] * b[c - i];
      slo += p;
      shi += slo < p ? 1u : 0u;
    }
    r[c] = (uint32_t)slo;
    clo = (slo >> 32) | (shi << 32);
    chi = (uint32_t)(shi >> 32);
  }
  ripple_add<G>(r, lo, hi, clo);
  ripple_add<G>(r, lo, hi, chi, 2);  // bits 64..95 of the carries: two limbs up
  return trim<G>(r, S);
}
// Schoolbook long division as bn::divmod (b has >= 2 limbs, a >= b), the
// multiply-subtract of each quotient limb spread over the lanes.
// un: na + 1 limbs of work, vn: nb limbs of work.  q, r distinct from a, b.
template <class G>
__device__ void divmod(uint32_t* q, uint32_t& nq, uint32_t* r, uint32_t& nr, const uint32_t* a, uint32_t na,
                       const uint32_t* b, uint32_t nb, uint32_t* un, uint32_t* vn) {
  const uint32_t s = __clz(b[nb - 1]);
  G::sync();
  for (uint32_t i = G::id(); i < nb; i += G::size()) vn[i] = s ? (b[i] << s) | (i ? b[i - 1] >> (32 - s) : 0u) : b[i];
  for (uint32_t i = G::id(); i <= na; i += G::size()) {
    const uint32_t x = i < na ? a[i] : 0u;
    un[i] = s ? (x << s) | (i ? a[i - 1] >> (32 - s) : 0u) : x;
  }
  G::sync();
  const uint64_t vt = vn[nb - 1], vs = vn[nb - 2];
  const Div DV(vt);
  uint32_t lo, hi;
  chunk_of<G>(nb, lo, hi);
  for (int64_t j = (int64_t)na - nb; j >= 0; --j) {
    const uint64_t top = ((uint64_t)un[j + nb] << 32) | un[j + nb - 1];
    uint64_t rh;
    uint64_t qh = DV.qr(top, rh);
    while (qh >> 32 || qh * vs > ((rh << 32) | un[j + nb - 2])) {
      --qh;
      rh += vt;
      if (rh >> 32) break;
    }
    G::sync();
    // un[j .. j+nb] -= qh * vn: each lane its chunk of vn, the carry of the
    // product and the borrow leaving the chunk as one debt at its top
    uint64_t pc = 0;
    uint32_t br = 0;
    for (uint32_t i = lo; i < hi; ++i) {
      const uint64_t p = qh * vn[i] + pc;
      pc = p >> 32;
      const uint64_t sb = (uint64_t)(uint32_t)p + br;
      const uint32_t u = un[i + j];
      un[i + j] = u - (uint32_t)sb;
      br = (uint64_t)u < sb ? 1u : 0u;
    }
    // the debt leaving the top chunk lands on limb j + nb (chunks cover [0, nb))
    const uint64_t top_debt = ripple_sub<G>(un + j, lo, hi, pc + br);
    uint64_t neg = 0;
    if (G::id() == 0 && top_debt) {
      const uint32_t u2 = un[j + nb];
      un[j + nb] = u2 - (uint32_t)top_debt;
      neg = ((uint64_t)u2 < top_debt) ? 1u : 0u;
    }
    neg = G::from(neg, 0);
    G::sync();
    if (neg) {  // qh was one too large: add vn back (the top wraps to the right value)
      --qh;
      uint64_t c = 0;
      for (uint32_t i = lo; i < hi; ++i) {
        c += (uint64_t)un[i + j] + vn[i];
        un[i + j] = (uint32_t)c;
        c >>= 32;
      }
      const uint64_t top_c = ripple_add<G>(un + j, lo, hi, c);
      if (G::id() == 0) un[j + nb] += (uint32_t)top_c;
      G::sync();
    }
    if (G::id() == 0) q[j] = (uint32_t)qh;
  }
  G::sync();
  nq = trim<G>(q, na - nb + 1);
  for (uint32_t i = G::id(); i < nb; i += G::size()) r[i] = s ? (un[i] >> s) | (un[i + 1] << (32 - s)) : un[i];
  G::sync();
  nr = trim<G>(r, nb);
}
// r = C(a, b) as the product of its prime powers (bn::binom): the factors of
// 32 primes at a time (one per lane), multiplied in as packed limbs
template <class G>
__device__ uint32_t binom(uint32_t* r, uint32_t a, uint32_t b, const uint32_t* primes, uint32_t np) {
  G::sync();
  if (G::id() == 0) r[0] = 1;
  G::sync();
  uint32_t n = 1;
  if (b > a) {
    if (G::id() == 0) r[0] = 0;
    G::sync();
    return 0;
  }
  if (b > a - b) b = a - b;
  if (b == 0) return 1;
  uint64_t acc = 1;
  for (uint32_t base = 0; base < np && primes[base] <= a; base += 32) {
    const uint32_t i = base + (G::id() & 31);
    uint64_t f = 1;
    if (i < np && primes[i] <= a) {
      const uint32_t p = primes[i];
      for (uint64_t pk = p; pk <= a; pk *= p)
        if (a / pk - b / pk - (a - b) / pk) f *= p;
    }
    // every warp of the group computed the same 32 factors: take them in lane order
    uint32_t m = __ballot_sync(kFull, f != 1);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t fl = __shfl_sync(kFull, f, l);
      if ((acc * fl) >> 32) {
        n = mul_small<G>(r, n, (uint32_t)acc);
        acc = fl;
      } else {
        acc *= fl;
      }
    }
  }
  if (acc > 1) n = mul_small<G>(r, n, (uint32_t)acc);
  return n;
}

}  // namespace gp

// bs_split's arithmetic on a group (GroupOps<gp::WarpG>: a warp,
// GroupOps<gp::BlockG>: a block)
template <class G>
struct GroupOps {
  __device__ static uint32_t binom(uint32_t* r, uint32_t a, uint32_t b, const uint32_t* p, uint32_t np) {
    return gp::binom<G>(r, a, b, p, np);
  }
  __device__ static uint32_t mul(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return gp::mul<G>(r, a, na, b, nb);
  }
  __device__ static int cmp(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return gp::cmp<G>(a, na, b, nb);
  }
  __device__ static void copy(uint32_t* r, const uint32_t* a, uint32_t n) { gp::copy<G>(r, a, n); }
  __device__ static uint32_t add(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return gp::add<G>(r, a, na, b, nb);
  }
  __device__ static uint32_t sub(uint32_t* r, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
    return gp::sub<G>(r, a, na, b, nb);
  }
  __device__ static uint32_t mul_small(uint32_t* a, uint32_t na, uint32_t m) { return gp::mul_small<G>(a, na, m); }
  __device__ static uint32_t divexact_small(uint32_t* a, uint32_t na, uint32_t d) {
    return gp::divexact_small<G>(a, na, d);
  }
  __device__ static uint32_t divmod_small(uint32_t* q, const uint32_t* a, uint32_t na, uint32_t d, uint32_t& nq) {
    return gp::div_small<G>(q, a, na, d, nq);
  }
  __device__ static void divmod(uint32_t* q, uint32_t& nq, uint32_t* r, uint32_t& nr, const uint32_t* a,
                                uint32_t na, const uint32_t* b, uint32_t nb, uint32_t* un, uint32_t* vn) {
    gp::divmod<G>(q, nq, r, nr, a, na, b, nb, un, vn);
  }
  __device__ static uint32_t set1(uint32_t* r, uint32_t v) {
    G::sync();
    if (G::id() == 0) r[0] = v;
    G::sync();
    return v ? 1u : 0u;
  }
};
using WarpOps = GroupOps<gp::WarpG>;
using BlockOps = GroupOps<gp::BlockG>;

}  // namespace sk
