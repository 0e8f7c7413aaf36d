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
//   A. ranks (one thread, schedule order): per pair the exact class size
//      C(m, n1), the fast dice roll below it on multi-limb integers, the rank
//      stored; the stream position at the end gives the bits consumed;
//   B. words (one thread per pair, all pairs at once): the recursive-halving
//      unranking on multi-limb integers, m <= 32 pieces by the lexicographic
//      walk; one byte per position;
//   C. interleave (one launch per level, one thread per pair).
// Big naturals are little-endian 32-bit limbs with tracked lengths.  Exact
// class sizes are products of prime powers (Legendre), divisions in the split
// scan are exact (binomial recurrences) and use the odd-divisor inverse, and
// the remaining division (the sub-ranks) is schoolbook long division.
#include <algorithm>
#include <stdexcept>
#include <vector>
#include "sk_kernels.h"
#include "bs_core.cuh"

namespace sk {
// (the multi-limb naturals and the per-pair stages: bs_core.cuh)

__global__ void bs_ranks_kernel(const BsPair* __restrict__ pairs, uint32_t npairs, StreamDesc sd,
                                const uint32_t* __restrict__ primes, uint32_t nprimes, uint32_t* pool,
                                uint32_t* work, uint32_t wl, unsigned long long* bits) {
  if (blockIdx.x || threadIdx.x) return;
  bits[0] = bs_ranks(pairs, npairs, sd, primes, nprimes, pool, work, wl);
}

__global__ void bs_words_kernel(const BsPair* __restrict__ pairs, uint32_t npairs, const uint32_t* __restrict__ pool,
                                uint32_t* __restrict__ scratch, const uint32_t* __restrict__ primes, uint32_t nprimes,
                                uint8_t* __restrict__ words) {
  __shared__ uint64_t C[(kBsSmall + 1) * (kBsSmall + 1)];
  bs_small_table(C, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < npairs) bs_word_pair(pairs[p], pool, scratch, primes, nprimes, words, C);
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
// schedule order, with their pools laid out.
struct BsPlan {
  std::vector<BsPair> pairs;
  std::vector<uint32_t> level_start;  // pairs of level L: [level_start[L], level_start[L+1])
  uint64_t rank_limbs = 0, scratch_limbs = 0, word_bytes = 0;
};

static BsPlan bs_plan(uint64_t n) {
  BsPlan pl;
  int c = 0;
  while ((1ull << c) < n) ++c;
  const uint64_t q = 1ull << c;
  auto bnd = [&](uint64_t i) { return (n * i) >> c; };
  uint32_t level = 0;
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
      P.rank_off = pl.rank_limbs;
      pl.rank_limbs += 1 + bs_limbs(m);
      P.word_off = (uint64_t)level * n + j;
      P.scr_off = pl.scratch_limbs;
      if (m > (uint32_t)kBsSmall) pl.scratch_limbs += bs_scratch_limbs(m);
      pl.pairs.push_back(P);
    }
  }
  pl.level_start.push_back((uint32_t)pl.pairs.size());
  pl.word_bytes = (uint64_t)level * n;
  return pl;
}

uint64_t balanced_max_n() { return 1ull << 17; }

void run_balanced(int eb, void* data, uint64_t n, StreamDesc sd, unsigned long long* d_bits, cudaStream_t st) {
  if (n < 2) return;
  if (n > balanced_max_n()) throw std::invalid_argument("balanced_shuffle: n above the supported 2^17");
  BsPlan pl = bs_plan(n);
  const uint32_t np = (uint32_t)pl.pairs.size();
  std::vector<uint32_t> primes = primes_upto((uint32_t)n);
  const uint32_t wl = bs_limbs((uint32_t)n) + 8;
  BsPair* d_pairs = nullptr;
  uint32_t *d_primes = nullptr, *d_pool = nullptr, *d_work = nullptr, *d_scr = nullptr;
  uint8_t* d_words = nullptr;
  void* d_tmp = nullptr;
  auto cleanup = [&]() {
    cudaFreeAsync(d_pairs, st);
    cudaFreeAsync(d_primes, st);
    cudaFreeAsync(d_pool, st);
    cudaFreeAsync(d_work, st);
    cudaFreeAsync(d_scr, st);
    cudaFreeAsync(d_words, st);
    cudaFreeAsync(d_tmp, st);
  };
  try {
    if (cudaMallocAsync((void**)&d_pairs, np * sizeof(BsPair), st) ||
        cudaMallocAsync((void**)&d_primes, std::max<size_t>(1, primes.size()) * 4, st) ||
        cudaMallocAsync((void**)&d_pool, (pl.rank_limbs + 1) * 4, st) ||
        cudaMallocAsync((void**)&d_work, (size_t)4 * wl * 4, st) ||
        cudaMallocAsync((void**)&d_scr, (pl.scratch_limbs + 1) * 4, st) ||
        cudaMallocAsync((void**)&d_words, pl.word_bytes + 1, st) || cudaMallocAsync(&d_tmp, n * eb, st))
      throw std::runtime_error("balanced_shuffle: device allocation failed");
    if (cudaMemcpyAsync(d_pairs, pl.pairs.data(), np * sizeof(BsPair), cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(d_primes, primes.data(), primes.size() * 4, cudaMemcpyHostToDevice, st))
      throw std::runtime_error("balanced_shuffle: upload failed");
    // the host vectors must outlive the (stream-ordered) copies
    if (cudaStreamSynchronize(st)) throw std::runtime_error("balanced_shuffle: upload failed");
    bs_ranks_kernel<<<1, 1, 0, st>>>(d_pairs, np, sd, d_primes, (uint32_t)primes.size(), d_pool, d_work, wl,
                                     d_bits);
    count_launch();
    bs_words_kernel<<<(np + 63) / 64, 64, 0, st>>>(d_pairs, np, d_pool, d_scr, d_primes, (uint32_t)primes.size(),
                                                   d_words);
    count_launch();
    for (size_t L = 0; L + 1 < pl.level_start.size(); ++L) {
      const uint32_t p0 = pl.level_start[L], p1 = pl.level_start[L + 1];
      if (p1 == p0) continue;
      const unsigned blocks = (p1 - p0 + 127) / 128;
      if (eb == 4)
        bs_interleave_kernel<uint32_t><<<blocks, 128, 0, st>>>(d_pairs, p0, p1, (uint32_t*)data, (uint32_t*)d_tmp,
                                                               d_words);
      else
        bs_interleave_kernel<unsigned long long><<<blocks, 128, 0, st>>>(
            d_pairs, p0, p1, (unsigned long long*)data, (unsigned long long*)d_tmp, d_words);
      count_launch();
    }
    if (cudaGetLastError() != cudaSuccess) throw std::runtime_error("balanced_shuffle: launch failed");
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace sk
