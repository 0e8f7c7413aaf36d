// balanced.cu -- BalancedShuffle beyond the machine-word slice (SURVEY.md
// section 8 row F1).  Reference (paths relative to pkg/src/shufflekit/):
//   balanced_shuffle       balanced.py:219-245  (pairs of singleton_rounds,
//                                                shufflers.py:108-114)
//   _sample_bits_into      balanced.py:158-164  (one random_int per pair)
//   BitSource.random_int   bitstream.py:187-210 (fast dice roller, any bound)
//   _unrank_into           balanced.py:146-155  (recursive halving)
//   _locate_split          balanced.py:98-143   (split point, scan from the mode)
//   _unrank_small          balanced.py:78-93    (lexicographic walk, m <= 32)
//   _interleave_bits       balanced.py:198-216
//
// Every pair draws from the caller's ONE stream in schedule order, so the
// stream offset of pair p depends on the consumption of every earlier pair;
// the word of a pair, though, depends only on its rank.  Three stages:
//   A. ranks (one warp, schedule order): per pair the exact class size
//      C(m, n1) and the fast dice roll below it -- machine words for m <= 64
//      (one lane), multi-limb integers on the whole warp above; the rank
//      stored; the stream position at the end gives the bits consumed;
//   B. words: the recursive-halving unranking.  Pairs above kBsTop positions
//      get a warp each for their splits above kBsTop (bs_split on WarpOps);
//      the sub-problems of <= kBsTop positions they leave, and the pairs of <=
//      kBsTop positions, are tasks of one thread each (bs_split on
//      SerialOps, m <= 32 by the lexicographic walk); one byte per position;
//   C. interleave (one launch per level, one thread per pair).
// Big naturals are little-endian 32-bit limbs with tracked lengths.  Exact
// class sizes are products of prime powers (Legendre), divisions in the split
// scan are exact (binomial recurrences) and use the odd-divisor inverse, and
// the remaining division (the sub-ranks) is schoolbook long division.
#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>
#include "sk_kernels.h"
#include "bs_core.cuh"
#include "bs_group.cuh"

namespace sk {
// (the multi-limb naturals and the per-pair stages: bs_core.cuh)


constexpr uint32_t kBsTop = 1024;
constexpr int kBsGroupBlock = 256;  // threads of a block group  // pairs / sub-problems above this many positions: a warp

// A sub-problem of stage B: the word of m positions with k zeros and rank at
// pool + rank_off ([limb count, limbs]), into words + word_off; its serial
// scratch at scratch + scr_off (m > 32).
struct BsJob {
  uint32_t m, k;
  uint64_t word_off, rank_off, scr_off;
};
// device-side bump counters of stage B
struct BsCounters {
  unsigned long long njobs, pool_top, scr_top;
};

// The class sizes C(m, n1) of the pairs above kBsWord positions, one warp
// each (data independent: computed before the sequential rolls need them);
// entry b at table + boff[b] as [limb count, limbs].  One block each.
__global__ void __launch_bounds__(kBsGroupBlock) bs_binoms_kernel(const uint32_t* __restrict__ bm, const uint32_t* __restrict__ bk,
                                                       const uint64_t* __restrict__ boff, uint32_t* table,
                                                       const uint32_t* __restrict__ primes, uint32_t nprimes) {
  extern __shared__ uint32_t num[];
  const uint32_t n = gp::binom<gp::BlockG>(num, bm[blockIdx.x], bk[blockIdx.x], primes, nprimes);
  uint32_t* T = table + boff[blockIdx.x];
  if (threadIdx.x == 0) T[0] = n;
  gp::copy<gp::BlockG>(T + 1, num, n);
}

// A. the rolls, in schedule order on the one stream, as two kernels of one
// warp: A1 the leading pairs of <= kBsWord positions (no class-size table
// needed, so the table kernel runs beside it), A2 the rest.  The machine-word
// rolls of one lane are bitstream.py:187-210 on uint64; the pairs of level 0
// (one element per side: the roll below 2 is exactly one bit, always
// accepted) are read in parallel.
constexpr uint32_t kBsWord = 64;  // C(m, n1) < 2^62 for m <= 64
struct BsSmallTab {
  uint64_t C[(kBsWord + 1) * (kBsWord + 1)];  // C(a, b), a, b <= 64 (Pascal)
  uint8_t lb[(kBsWord + 1) * (kBsWord + 1)];  // bits of C(a, b) - 1
};
__device__ void bs_small_tab(BsSmallTab& T) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t a = 0; a <= kBsWord; ++a) {
    for (uint32_t b = lane; b <= kBsWord; b += 32) {
      const uint64_t v = b > a ? 0ull
                               : (b == 0 || b == a ? 1ull
                                                   : T.C[(a - 1) * (kBsWord + 1) + b - 1] +
                                                         T.C[(a - 1) * (kBsWord + 1) + b]);
      T.C[a * (kBsWord + 1) + b] = v;
      T.lb[a * (kBsWord + 1) + b] = v > 1 ? (uint8_t)(64 - __clzll(v - 1)) : 0;
    }
    __syncwarp();
  }
}
// one machine-word roll below C(m, n1) at stream offset o (one lane), with a
// cache of the stream words cw, cw + 1
__device__ __forceinline__ uint64_t bs_roll_word(const BsSmallTab& T, uint32_t m, uint32_t n1, const StreamDesc& sd,
                                                 uint64_t& o, uint64_t& cw, uint64_t& cw0, uint64_t& cw1) {
  const uint64_t bound = T.C[m * (kBsWord + 1) + n1];
  const uint32_t lb = T.lb[m * (kBsWord + 1) + n1];
  uint64_t vv = 1, cc = 0;
  for (;;) {
    uint32_t k = lb - (64 - __clzll(vv));  // smallest k with vv << k >= bound
    if ((vv << k) < bound) ++k;
    const uint64_t w = o >> 6;
    if (w != cw) {
      if (w == cw + 1) {
        cw0 = cw1;
        cw1 = bs_word(sd, w + 1);
      } else {
        cw0 = bs_word(sd, w);
        cw1 = bs_word(sd, w + 1);
      }
      cw = w;
    }
    const uint32_t sh = (uint32_t)(o & 63);
    const uint64_t x = sh ? (cw0 << sh) | (cw1 >> (64 - sh)) : cw0;
    cc = k ? (cc << k) | (x >> (64 - k)) : cc;
    o += k;
    vv <<= k;
    if (cc < bound) return cc;
    cc -= bound;
    vv -= bound;
  }
}
__device__ __forceinline__ void bs_store_word_rank(uint32_t* R, uint64_t cc) {
  R[0] = cc ? (cc >> 32 ? 2u : 1u) : 0u;
  R[1] = (uint32_t)cc;
  R[2] = (uint32_t)(cc >> 32);
}

// A1: pairs [0, p_end) (level 0 = [0, n0)), all of <= kBsWord positions;
// leaves the stream offset in *o_out
__global__ void __launch_bounds__(32) bs_ranks_small_kernel(const BsPair* __restrict__ pairs, uint32_t n0,
                                                            uint32_t p_end, StreamDesc sd, uint32_t* pool,
                                                            unsigned long long* o_out) {
  __shared__ BsSmallTab T;
  __shared__ uint32_t sm1[32], sm2[32];
  __shared__ uint64_t sro[32];
  const uint32_t lane = threadIdx.x;
  bs_small_tab(T);
  for (uint32_t p = lane; p < n0; p += 32)  // level 0: pair p is bit p
    bs_store_word_rank(pool + pairs[p].rank_off, (bs_word(sd, p >> 6) >> (63 - (p & 63))) & 1u);
  uint64_t o = n0, cw = ~1ull, cw0 = 0, cw1 = 0;
  for (uint32_t p0 = n0; p0 < p_end; p0 += 32) {
    if (p0 + lane < p_end) {
      const BsPair& Q = pairs[p0 + lane];
      sm1[lane] = Q.n1;
      sm2[lane] = Q.n2;
      sro[lane] = Q.rank_off;
    }
    __syncwarp();
    if (lane == 0) {
      const uint32_t cnt = min(32u, p_end - p0);
      for (uint32_t i = 0; i < cnt; ++i)
        bs_store_word_rank(pool + sro[i], bs_roll_word(T, sm1[i] + sm2[i], sm1[i], sd, o, cw, cw0, cw1));
    }
    __syncwarp();
  }
  if (lane == 0) o_out[0] = o;
}

// A2: pairs [p_begin, npairs) from stream offset *bits; the class sizes of
// the pairs above kBsWord from the table; the total bits into *bits
__global__ void __launch_bounds__(32) bs_ranks_kernel(const BsPair* __restrict__ pairs, uint32_t p_begin,
                                                      uint32_t npairs, StreamDesc sd,
                                                      const uint32_t* __restrict__ btab, uint32_t* pool, uint32_t wl,
                                                      unsigned long long* bits, uint32_t* gwork) {
  __shared__ BsSmallTab T;
  extern __shared__ uint32_t swork[];  // B, v, c and a spare: wl limbs each
  uint32_t* work = gwork ? gwork : swork;  // (global when they do not fit)
  const uint32_t lane = threadIdx.x;
  bs_small_tab(T);
  uint32_t* B = work;
  uint32_t* v = work + wl;
  uint32_t* c = work + 2 * wl;
  uint32_t* t = work + 3 * wl;
  uint32_t nB = 0, cb = ~0u;
  uint64_t o = bits[0];  // stream offset (uniform)
  uint64_t cw = ~1ull, cw0 = 0, cw1 = 0;  // lane 0's word cache (no word cached: cw + 1 != 0)
  for (uint32_t p = p_begin; p < npairs; ++p) {
    const BsPair P = pairs[p];
    const uint32_t m = P.n1 + P.n2;
    uint32_t* R = pool + P.rank_off;
    if (m <= kBsWord) {
      if (lane == 0) bs_store_word_rank(R, bs_roll_word(T, m, P.n1, sd, o, cw, cw0, cw1));
      o = __shfl_sync(gp::kFull, o, 0);
      continue;
    }
    if (P.bidx != cb) {  // pairs of a level repeat a handful of sizes
      const uint32_t* TB = btab + P.bidx;
      nB = TB[0];
      gp::copy<gp::WarpG>(B, TB + 1, nB);
      cb = P.bidx;
    }
    // fast dice roller below B (>= 2): v = 1, c = 0
    if (lane == 0) v[0] = 1;
    __syncwarp();
    uint32_t nv = 1, nc = 0;
    const uint32_t lb = gp::bitlen<gp::WarpG>(B, nB);
    for (;;) {
      uint32_t k = lb - gp::bitlen<gp::WarpG>(v, nv);  // smallest k with v << k >= B
      if (gp::cmp_shl<gp::WarpG>(v, nv, k, B, nB) < 0) ++k;
      // c = (c << k) | the next k bits: limb i of them is stream bits
      // [o + k - 32(i+1), o + k - 32 i)
      nc = gp::shl<gp::WarpG>(t, c, nc, k);
      const uint32_t full = k >> 5, part = k & 31, nk = full + (part ? 1u : 0u);
      for (uint32_t i = nc + lane; i < nk; i += 32) t[i] = 0;
      __syncwarp();
      for (uint32_t i = lane; i < full; i += 32) t[i] |= bs_bits(sd, o + k - 32 * (i + 1), 32);
      if (part && lane == 0) t[full] |= bs_bits(sd, o, part);
      __syncwarp();
      nc = gp::trim<gp::WarpG>(t, nc > nk ? nc : nk);
      { uint32_t* x = c; c = t; t = x; }
      o += k;
      nv = gp::shl<gp::WarpG>(t, v, nv, k);
      { uint32_t* x = v; v = t; t = x; }
      if (gp::cmp<gp::WarpG>(c, nc, B, nB) < 0) break;
      nc = gp::sub<gp::WarpG>(c, c, nc, B, nB);
      nv = gp::sub<gp::WarpG>(v, v, nv, B, nB);
    }
    if (lane == 0) R[0] = nc;
    gp::copy<gp::WarpG>(R + 1, c, nc);
  }
  if (lane == 0) bits[0] = o;
}

// B1. the splits above kBsTop, one recursion depth per launch and one warp
// (and block) per node: a node of more than kBsTop positions loads its rank
// into shared memory, splits (bs_split on WarpOps), and hands its halves on --
// as nodes of the next depth when they are still above kBsTop, as B2 jobs
// otherwise; their sub-ranks go to the pool.  The halves of a node are
// independent, so the nodes of one depth run side by side.
struct BsNode {
  uint32_t m, k;
  uint64_t word_off, rank_off;
};
constexpr int kBsMaxDepth = 16;
constexpr uint32_t kBsBlockM = 1u << 15;  // nodes above this split on a block of kBsGroupBlock threads
constexpr uint32_t kBsGlobM = 1u << 16;  // nodes above this may need global slots (the kernel decides exactly)

__host__ __device__ inline uint64_t bs_split_smem_limbs(uint32_t m) {
  const uint32_t W = bs_limbs(m), H = W / 2 + 3;
  return (uint64_t)W + BsWork::limbs(W, H);
}

// a half of a split: a node of the next depth in slot `slot` (when it is
// still above kBsTop) or a B2 job (then the slot holds an empty node)
template <class G>
__device__ void bs_emit(uint32_t m, uint32_t k, uint64_t word_off, const uint32_t* rank, uint32_t nr, BsNode* next,
                        uint64_t slot, uint64_t next_cap, BsJob* jobs, uint32_t* pool, uint64_t pool_cap,
                        uint64_t scr_base, BsCounters* cnt) {
  uint64_t ro = 0;
  if (threadIdx.x == 0) {
    ro = atomicAdd(&cnt->pool_top, (unsigned long long)(nr + 1));
    if (ro + nr + 1 > pool_cap) __trap();  // (the pool is sized for every sub-rank)
    pool[ro] = nr;
    if (m > kBsTop) {
      if (slot >= next_cap) __trap();  // (the slots of a depth cover its nodes)
      next[slot] = BsNode{m, k, word_off, ro};
    } else {
      if (slot < next_cap) next[slot] = BsNode{0, 0, 0, 0};
      const uint64_t j = atomicAdd(&cnt->njobs, 1ull);
      const uint64_t so =
          m > (uint32_t)kBsSmall ? atomicAdd(&cnt->scr_top, (unsigned long long)bs_scratch_limbs(m)) : 0ull;
      jobs[j] = BsJob{m, k, word_off, ro, scr_base + so};
    }
  }
  ro = G::from(ro, 0);
  gp::copy<G>(pool + ro + 1, rank, nr);
}

// Node slots: the roots (pairs above kBsTop) largest first, the children of
// slot i in slots 2i, 2i + 1 of the next depth -- so every depth starts its
// largest splits first; empty slots (m = 0) pass emptiness on.
template <class G, int NT>
__global__ void __launch_bounds__(NT) bs_split_kernel(uint64_t slot0, const BsNode* __restrict__ nodes, BsNode* next,
                                                      uint64_t next_cap, const uint32_t* __restrict__ primes,
                                                      uint32_t nprimes, BsJob* jobs, uint32_t* pool,
                                                      uint64_t pool_cap, uint64_t scr_base, BsCounters* cnt,
                                                      uint32_t smem_max_m, uint32_t* gscr, uint64_t gstride,
                                                      unsigned long long* gslot) {
  extern __shared__ uint32_t smem[];
  const uint64_t slot = slot0 + blockIdx.x;
  const BsNode N = nodes[slot];
  const uint64_t s0 = 2ull * slot;
  if (N.m == 0) {
    if (threadIdx.x == 0)
      for (uint64_t s = s0; s < s0 + 2 && s < next_cap; ++s) next[s] = BsNode{0, 0, 0, 0};
    return;
  }
  // nodes above smem_max_m positions work in a global slot
  uint32_t* sm = smem;
  if (N.m > smem_max_m) {
    uint64_t gs = 0;
    if (threadIdx.x == 0) gs = atomicAdd(gslot, 1ull);
    sm = gscr + G::from(gs, 0) * gstride;
  }
  const uint32_t W = bs_limbs(N.m);
  uint32_t* rk = sm;
  const BsWork bw = BsWork::carve(sm + W, W, W / 2 + 3);
  const uint32_t* R = pool + N.rank_off;
  const uint32_t nr = R[0];
  gp::copy<G>(rk, R + 1, nr);
  uint32_t t, nq, nrr;
  bs_split<GroupOps<G>>(N.m, N.k, rk, nr, bw, primes, nprimes, t, nq, nrr);
  const uint32_t mL = N.m >> 1;
  bs_emit<G>(mL, t, N.word_off, bw.q, nq, next, s0, next_cap, jobs, pool, pool_cap, scr_base, cnt);
  bs_emit<G>(N.m - mL, N.k - t, N.word_off + mL, bw.rr, nrr, next, s0 + 1, next_cap, jobs, pool, pool_cap, scr_base,
          cnt);
}

// B2. one thread per job (pairs of <= kBsTop positions and B1's sub-problems)
__global__ void bs_jobs_kernel(const BsJob* __restrict__ jobs, const BsCounters* __restrict__ cnt, const uint32_t* pool,
                               uint32_t* scratch, const uint32_t* __restrict__ primes, uint32_t nprimes,
                               uint8_t* __restrict__ words) {
  __shared__ uint64_t C[(kBsSmall + 1) * (kBsSmall + 1)];
  bs_small_table(C, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cnt->njobs) return;
  const BsJob J = jobs[j];
  bs_word_task(J.m, J.k, pool + J.rank_off, words + J.word_off, scratch + J.scr_off, primes, nprimes, C);
}

// C. one level's interleaves (balanced.py:198-216): position t takes the next
// left element for a 0 and the next right element for a 1.
template <typename V>
__global__ void bs_interleave_kernel(const BsPair* __restrict__ pairs, uint32_t p0, uint32_t p1, V* a, V* tmp,
                                     const uint8_t* __restrict__ words) {
  const uint32_t p = p0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p1) return;
  const BsPair P = pairs[p];
  const uint32_t m = P.n1 + P.n2;
  const uint8_t* w = words + P.word_off;
  V* x = a + P.j;
  V* s = tmp + P.j;
  for (uint32_t t = 0; t < m; ++t) s[t] = x[t];
  uint32_t ia = 0, ib = P.n1;
  for (uint32_t t = 0; t < m; ++t) x[t] = w[t] ? s[ib++] : s[ia++];
}

// The same for the levels of large pairs: a block per pair; position t takes
// right[#ones before t] or left[#zeros before t], the ones counted by a block
// scan over tiles of 8 positions per thread.
constexpr int kBsIlBlock = 256;
template <typename V>
__global__ void __launch_bounds__(kBsIlBlock) bs_interleave_block_kernel(const BsPair* __restrict__ pairs,
                                                                         uint32_t p0, V* a, V* tmp,
                                                                         const uint8_t* __restrict__ words) {
  __shared__ uint32_t wsum[kBsIlBlock / 32];
  const BsPair P = pairs[p0 + blockIdx.x];
  const uint32_t m = P.n1 + P.n2, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint8_t* w = words + P.word_off;
  V* x = a + P.j;
  V* s = tmp + P.j;
  for (uint32_t t = tid; t < m; t += kBsIlBlock) s[t] = x[t];
  __syncthreads();
  uint32_t ones0 = 0;  // ones before the tile
  for (uint32_t t0 = 0; t0 < m; t0 += 8 * kBsIlBlock) {
    const uint32_t b = t0 + 8 * tid;
    uint32_t bits = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (b + e < m && w[b + e]) bits |= 1u << e;
    const uint32_t c = __popc(bits);
    uint32_t xs = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xs, o);
      if (lane >= (uint32_t)o) xs += y;
    }
    if (lane == 31) wsum[wid] = xs;
    __syncthreads();
    uint32_t before = ones0, tot = 0;
#pragma unroll
    for (int k = 0; k < kBsIlBlock / 32; ++k) {
      before += k < (int)wid ? wsum[k] : 0u;
      tot += wsum[k];
    }
    before += xs - c;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t t = b + e;
      if (t < m) {
        const uint32_t ob = before + __popc(bits & ((1u << e) - 1));  // ones before t
        x[t] = (bits >> e) & 1u ? s[P.n1 + ob] : s[t - ob];
      }
    }
    ones0 += tot;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host
static std::vector<uint32_t> primes_upto(uint32_t n) {
  std::vector<uint8_t> comp(n + 1, 0);
  std::vector<uint32_t> ps;
  for (uint32_t i = 2; i <= n; ++i) {
    if (comp[i]) continue;
    ps.push_back(i);
    for (uint64_t j = (uint64_t)i * i; j <= n; j += i) comp[j] = 1;
  }
  return ps;
}

// The pairs of singleton_rounds(n) (shufflers.py:108-130) that draw, in
// schedule order, with their pools laid out, and stage B's jobs.
struct BsPlan {
  std::vector<BsPair> pairs;
  std::vector<uint32_t> level_start;  // pairs of level L: [level_start[L], level_start[L+1])
  std::vector<BsJob> jobs;            // pairs of <= kBsTop positions
  std::vector<BsNode> roots;          // pairs above kBsTop (B1's depth 0)
  std::vector<uint64_t> node_cap;     // B1 nodes per depth (upper bounds)
  std::vector<uint64_t> block_slots;  // ... the leading ones split by a block (above kBsBlockM)
  std::vector<uint64_t> glob_cap;     // ... of them above kBsGlobM positions
  std::vector<uint32_t> bm, bk;       // distinct class sizes C(bm, bk) of pairs above kBsWord
  std::vector<uint64_t> boff;         // their table offsets
  uint64_t btab_limbs = 0;
  uint64_t rank_limbs = 0, scratch_limbs = 0, word_bytes = 0, job_cap = 0, pool_cap = 0;
  uint32_t max_big = 0;
  uint32_t n_level0 = 0;     // pairs of level 0 (a prefix)
  uint32_t p_small_end = 0;  // the leading pairs of <= kBsWord positions end here
};

static BsPlan bs_plan(uint64_t n) {
  BsPlan pl;
  int c = 0;
  while ((1ull << c) < n) ++c;
  const uint64_t q = 1ull << c;
  auto bnd = [&](uint64_t i) { return (n * i) >> c; };
  uint32_t level = 0;
  uint64_t emit = 0, emit_rank = 0;
  for (uint64_t p = 1; p < q; p += p, ++level) {
    pl.level_start.push_back((uint32_t)pl.pairs.size());
    for (uint64_t i = 0; i < q; i += 2 * p) {
      const uint64_t j = bnd(i), k = bnd(i + p), l = bnd(std::min(i + 2 * p, q));
      if (k == j || l == k) continue;  // balanced.py:238-239
      BsPair P;
      P.j = (uint32_t)j;
      P.n1 = (uint32_t)(k - j);
      P.n2 = (uint32_t)(l - k);
      P.level = level;
      const uint32_t m = P.n1 + P.n2;
      P.bidx = 0;
      if (m > kBsWord) {
        size_t b = 0;
        while (b < pl.bm.size() && !(pl.bm[b] == m && pl.bk[b] == P.n1)) ++b;
        if (b == pl.bm.size()) {
          pl.bm.push_back(m);
          pl.bk.push_back(P.n1);
          pl.boff.push_back(pl.btab_limbs);
          pl.btab_limbs += 1 + bs_limbs(m);
        }
        P.bidx = (uint32_t)pl.boff[b];
      }
      P.rank_off = pl.rank_limbs;
      pl.rank_limbs += 1 + bs_limbs(m);
      P.word_off = (uint64_t)level * n + j;
      P.scr_off = 0;
      if (m > kBsTop) {
        pl.roots.push_back(BsNode{m, P.n1, P.word_off, P.rank_off});
        pl.max_big = std::max(pl.max_big, m);
        // its jobs have > kBsTop / 2 positions each; its nodes at depth d
        // have at most ceil(m / 2^d) positions
        const uint64_t jobs = 2ull * m / kBsTop + 2;
        emit += jobs;
        for (int d = 0; d < kBsMaxDepth && ((m + (1ull << d) - 1) >> d) > kBsTop; ++d) {
          if (pl.glob_cap.size() <= (size_t)d) pl.glob_cap.push_back(0);
          if (((m + (1ull << d) - 1) >> d) > kBsGlobM) pl.glob_cap[d] += 1ull << d;
          emit_rank += m / 32 + 8 + 4 * (2ull << d);
        }
      } else {
        BsJob J;
        J.m = m;
        J.k = P.n1;
        J.word_off = P.word_off;
        J.rank_off = P.rank_off;
        J.scr_off = pl.scratch_limbs;
        if (m > (uint32_t)kBsSmall) pl.scratch_limbs += bs_scratch_limbs(m);
        pl.jobs.push_back(J);
      }
      pl.pairs.push_back(P);
    }
  }
  pl.level_start.push_back((uint32_t)pl.pairs.size());
  pl.word_bytes = (uint64_t)level * n;
  // node slots: roots largest first; depth d has 2^d slots per root that
  // still has nodes there (a prefix of the roots)
  std::stable_sort(pl.roots.begin(), pl.roots.end(), [](const BsNode& x, const BsNode& y) { return x.m > y.m; });
  for (int d = 0; d < kBsMaxDepth; ++d) {
    uint64_t r = 0;
    while (r < pl.roots.size() && ((pl.roots[r].m + (1ull << d) - 1) >> d) > kBsTop) ++r;
    if (!r) break;
    pl.node_cap.push_back(r << d);
    uint64_t rb = 0;
    while (rb < r && ((pl.roots[rb].m + (1ull << d) - 1) >> d) > kBsBlockM) ++rb;
    pl.block_slots.push_back(rb << d);
  }
  pl.n_level0 = pl.level_start.size() > 1 ? pl.level_start[1] : 0;
  while (pl.p_small_end < pl.pairs.size() && pl.pairs[pl.p_small_end].n1 + pl.pairs[pl.p_small_end].n2 <= kBsWord)
    ++pl.p_small_end;
  pl.job_cap = pl.jobs.size() + emit;
  pl.pool_cap = pl.rank_limbs + emit_rank + 16;
  return pl;
}

uint64_t balanced_max_n() { return 1ull << 20; }
constexpr size_t kBsSmemBudget = 200 * 1024;  // dynamic shared memory per CTA we plan with

void run_balanced(int eb, void* data, uint64_t n, StreamDesc sd, unsigned long long* d_bits, cudaStream_t st) {
  if (n < 2) return;
  if (n > balanced_max_n()) throw std::invalid_argument("balanced_shuffle: n above the supported 2^20");
  BsPlan pl = bs_plan(n);
  const uint32_t np = (uint32_t)pl.pairs.size(), nbig = (uint32_t)pl.roots.size();
  const int depths = (int)pl.node_cap.size();
  std::vector<uint64_t> node_off(depths + 2, 0);
  for (int d = 0; d < depths; ++d) node_off[d + 1] = node_off[d] + pl.node_cap[d];
  node_off[depths + 1] = node_off[depths] + 1;  // (the last depth's "next" list stays empty)
  std::vector<uint32_t> primes = primes_upto((uint32_t)n);
  const uint32_t wl = bs_limbs((uint32_t)n) + 8;
  const uint64_t emit_scr = (pl.job_cap - pl.jobs.size()) * bs_scratch_limbs(kBsTop);
  BsCounters hc{};
  hc.njobs = pl.jobs.size();
  hc.pool_top = pl.rank_limbs;
  BsPair* d_pairs = nullptr;
  BsJob* d_jobs = nullptr;
  BsCounters* d_cnt = nullptr;
  BsNode* d_nodes = nullptr;
  uint32_t *d_gwork = nullptr, *d_gscr = nullptr;
  unsigned long long* d_gslot = nullptr;
  uint32_t *d_primes = nullptr, *d_pool = nullptr, *d_scr = nullptr, *d_bm = nullptr,
           *d_bk = nullptr, *d_btab = nullptr;
  uint64_t* d_boff = nullptr;
  uint8_t* d_words = nullptr;
  void* d_tmp = nullptr;
  auto cleanup = [&]() {
    for (void* ptr : {(void*)d_pairs, (void*)d_jobs, (void*)d_cnt, (void*)d_primes, (void*)d_pool, (void*)d_scr,
                      (void*)d_nodes, (void*)d_words, d_tmp, (void*)d_bm, (void*)d_bk, (void*)d_boff,
                      (void*)d_btab, (void*)d_gwork, (void*)d_gscr, (void*)d_gslot})
      if (ptr) cudaFreeAsync(ptr, st);
  };
  auto chk = [](const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
      throw std::runtime_error(std::string("balanced_shuffle: ") + what + ": " + cudaGetErrorString(e));
  };
  try {
    chk("before");
    if (cudaMallocAsync((void**)&d_pairs, np * sizeof(BsPair), st) ||
        cudaMallocAsync((void**)&d_jobs, std::max<uint64_t>(1, pl.job_cap) * sizeof(BsJob), st) ||
        cudaMallocAsync((void**)&d_cnt, sizeof(BsCounters), st) ||
        cudaMallocAsync((void**)&d_primes, std::max<size_t>(1, primes.size()) * 4, st) ||
        cudaMallocAsync((void**)&d_pool, (pl.pool_cap + 1) * 4, st) ||
        cudaMallocAsync((void**)&d_scr, (pl.scratch_limbs + emit_scr + 1) * 4, st) ||
        cudaMallocAsync((void**)&d_nodes, node_off[depths + 1] * sizeof(BsNode), st) ||
        cudaMallocAsync((void**)&d_bm, std::max<size_t>(1, pl.bm.size()) * 4, st) ||
        cudaMallocAsync((void**)&d_bk, std::max<size_t>(1, pl.bm.size()) * 4, st) ||
        cudaMallocAsync((void**)&d_boff, std::max<size_t>(1, pl.bm.size()) * 8, st) ||
        cudaMallocAsync((void**)&d_btab, (pl.btab_limbs + 1) * 4, st) ||
        cudaMallocAsync((void**)&d_words, pl.word_bytes + 1, st) || cudaMallocAsync(&d_tmp, n * eb, st))
      throw std::runtime_error("balanced_shuffle: device allocation failed");
    if (cudaMemcpyAsync(d_pairs, pl.pairs.data(), np * sizeof(BsPair), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(d_jobs, pl.jobs.data(), pl.jobs.size() * sizeof(BsJob), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(d_cnt, &hc, sizeof(hc), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(d_primes, primes.data(), primes.size() * 4, cudaMemcpyHostToDevice, st) ||
        (nbig && cudaMemcpyAsync(d_nodes, pl.roots.data(), nbig * sizeof(BsNode), cudaMemcpyHostToDevice, st)) ||
        (!pl.bm.empty() && (cudaMemcpyAsync(d_bm, pl.bm.data(), pl.bm.size() * 4, cudaMemcpyHostToDevice, st) ||
                            cudaMemcpyAsync(d_bk, pl.bk.data(), pl.bk.size() * 4, cudaMemcpyHostToDevice, st) ||
                            cudaMemcpyAsync(d_boff, pl.boff.data(), pl.boff.size() * 8, cudaMemcpyHostToDevice, st))))
      throw std::runtime_error("balanced_shuffle: upload failed");
    // the host vectors must outlive the (stream-ordered) copies
    if (cudaStreamSynchronize(st)) throw std::runtime_error("balanced_shuffle: upload failed");
    const uint32_t npr = (uint32_t)primes.size();
    // A1 on st while the class sizes are computed on a side stream; A2 after both
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_tab = nullptr;
    const uint32_t nbin = (uint32_t)pl.bm.size();
    if (nbin) {
      if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) || cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) ||
          cudaEventCreateWithFlags(&ev_tab, cudaEventDisableTiming))
        throw std::runtime_error("balanced_shuffle: stream setup failed");
      cudaEventRecord(ev_fork, st);
      cudaStreamWaitEvent(side, ev_fork, 0);
      const size_t smemT = (size_t)(bs_limbs((uint32_t)n) + 2) * 4;
      cudaFuncSetAttribute(bs_binoms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemT);
      bs_binoms_kernel<<<nbin, kBsGroupBlock, smemT, side>>>(d_bm, d_bk, d_boff, d_btab, d_primes, npr);
      count_launch();
      cudaEventRecord(ev_tab, side);
      chk("class sizes");
    }
    bs_ranks_small_kernel<<<1, 32, 0, st>>>(d_pairs, pl.n_level0, pl.p_small_end, sd, d_pool, d_bits);
    count_launch();
    chk("small rolls");
    if (nbin) {
      cudaStreamWaitEvent(st, ev_tab, 0);
      cudaEventDestroy(ev_fork);
      cudaEventDestroy(ev_tab);
      cudaStreamDestroy(side);  // (destroyed once its work completes)
    }
    const size_t smemA = (size_t)4 * wl * 4;
    if (smemA > kBsSmemBudget) {
      if (cudaMallocAsync((void**)&d_gwork, smemA, st)) throw std::runtime_error("balanced_shuffle: allocation failed");
    } else {
      cudaFuncSetAttribute(bs_ranks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemA);
    }
    bs_ranks_kernel<<<1, 32, d_gwork ? 0 : smemA, st>>>(d_pairs, pl.p_small_end, np, sd, d_btab, d_pool, wl, d_bits,
                                                        d_gwork);
    count_launch();
    chk("ranks");
    // nodes up to smem_max_m positions split in shared memory, larger ones
    // (n > 2^17) in global slots
    uint32_t smem_max_m = 1;
    while (bs_split_smem_limbs(2 * smem_max_m + 1) * 4 <= kBsSmemBudget) smem_max_m *= 2;
    if (depths) {
      const size_t smem0 = bs_split_smem_limbs(std::min<uint32_t>(pl.max_big, smem_max_m) + 1) * 4;
      cudaFuncSetAttribute(bs_split_kernel<gp::WarpG, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem0);
      cudaFuncSetAttribute(bs_split_kernel<gp::BlockG, kBsGroupBlock>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem0);
      // global slots: at depth d the nodes above smem_max_m are at most
      // glob_cap[d], each of at most ceil(max_big / 2^d) + 1 positions
      uint64_t gmax = 0;
      for (int d = 0; d < depths; ++d)
        gmax = std::max(gmax, pl.glob_cap[d] * bs_split_smem_limbs((uint32_t)((pl.max_big + (1ull << d) - 1) >> d) + 1));
      if (gmax && (cudaMallocAsync((void**)&d_gscr, gmax * 4, st) ||
                   cudaMallocAsync((void**)&d_gslot, depths * sizeof(unsigned long long), st) ||
                   cudaMemsetAsync(d_gslot, 0, depths * sizeof(unsigned long long), st)))
        throw std::runtime_error("balanced_shuffle: allocation failed");
    }
    for (int d = 0; d < depths; ++d) {  // one recursion depth per launch
      const uint32_t mmax = (uint32_t)((pl.max_big + (1ull << d) - 1) >> d) + 1;
      const uint64_t stride = bs_split_smem_limbs(mmax);
      const uint64_t next_cap = d + 1 < depths ? pl.node_cap[d + 1] : 0;
      const size_t smem = bs_split_smem_limbs(std::min(mmax, smem_max_m + 1)) * 4;
      const uint64_t nblk = pl.block_slots[d];  // the leading slots: nodes above kBsBlockM, a block each
      if (nblk) {
        bs_split_kernel<gp::BlockG, kBsGroupBlock><<<(unsigned)nblk, kBsGroupBlock, smem, st>>>(
            0, d_nodes + node_off[d], d_nodes + node_off[d + 1], next_cap, d_primes, npr, d_jobs, d_pool,
            pl.pool_cap, pl.scratch_limbs, d_cnt, smem_max_m, d_gscr, stride, d_gslot ? d_gslot + d : nullptr);
        count_launch();
      }
      if (pl.node_cap[d] > nblk) {
        bs_split_kernel<gp::WarpG, 32><<<(unsigned)(pl.node_cap[d] - nblk), 32, smem, st>>>(
            nblk, d_nodes + node_off[d], d_nodes + node_off[d + 1], next_cap, d_primes, npr, d_jobs, d_pool,
            pl.pool_cap, pl.scratch_limbs, d_cnt, smem_max_m, d_gscr, stride, d_gslot ? d_gslot + d : nullptr);
        count_launch();
      }
      chk("splits");
    }
    bs_jobs_kernel<<<(unsigned)((pl.job_cap + 63) / 64), 64, 0, st>>>(d_jobs, d_cnt, d_pool, d_scr, d_primes, npr,
                                                                       d_words);
    count_launch();
    chk("jobs");
    for (size_t L = 0; L + 1 < pl.level_start.size(); ++L) {
      const uint32_t p0 = pl.level_start[L], p1 = pl.level_start[L + 1];
      if (p1 == p0) continue;
      const uint32_t mlev = pl.pairs[p0].n1 + pl.pairs[p0].n2;
      if (mlev >= 1024) {  // the top levels: a block per pair
        if (eb == 4)
          bs_interleave_block_kernel<uint32_t><<<p1 - p0, kBsIlBlock, 0, st>>>(d_pairs, p0, (uint32_t*)data,
                                                                               (uint32_t*)d_tmp, d_words);
        else
          bs_interleave_block_kernel<unsigned long long><<<p1 - p0, kBsIlBlock, 0, st>>>(
              d_pairs, p0, (unsigned long long*)data, (unsigned long long*)d_tmp, d_words);
        count_launch();
        continue;
      }
      const unsigned blocks = (p1 - p0 + 127) / 128;
      if (eb == 4)
        bs_interleave_kernel<uint32_t><<<blocks, 128, 0, st>>>(d_pairs, p0, p1, (uint32_t*)data, (uint32_t*)d_tmp,
                                                               d_words);
      else
        bs_interleave_kernel<unsigned long long><<<blocks, 128, 0, st>>>(
            d_pairs, p0, p1, (unsigned long long*)data, (unsigned long long*)d_tmp, d_words);
      count_launch();
    }
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) throw std::runtime_error(std::string("balanced_shuffle: launch failed: ") + cudaGetErrorString(le));
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace sk
