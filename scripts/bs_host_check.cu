// Debugging harness (not product code): the BalancedShuffle stages of
// csrc/bs_core.cuh run on the HOST for one n and one stream state, printing
// the bits used and the permutation, to compare with oracle/balanced_oracle.py
// (scripts/bs_host_check.py).  Build:
//   nvcc -O2 -std=c++17 -I paper_1508_03167_b200/csrc scripts/bs_host_check.cu -o /tmp/bs_host_check
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <chrono>
#include "bs_core.cuh"

using namespace sk;

int main(int argc, char** argv) {
  const uint64_t n = strtoull(argv[1], 0, 10);
  uint64_t s4[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4 && 2 + i < argc; ++i) s4[i] = strtoull(argv[2 + i], 0, 10);
  StreamDesc sd;
  sd.state = s4[0];
  sd.buf = s4[1];
  sd.plen = (uint32_t)s4[2];
  sd.pad = 0;
  // the plan (as balanced.cu bs_plan)
  std::vector<BsPair> pairs;
  std::vector<uint32_t> lstart;
  uint64_t rank_limbs = 0, scr = 0;
  int c = 0;
  while ((1ull << c) < n) ++c;
  const uint64_t q = 1ull << c;
  uint32_t level = 0;
  for (uint64_t p = 1; p < q; p += p, ++level) {
    lstart.push_back((uint32_t)pairs.size());
    for (uint64_t i = 0; i < q; i += 2 * p) {
      const uint64_t j = (n * i) >> c, k = (n * (i + p)) >> c, l = (n * std::min(i + 2 * p, q)) >> c;
      if (k == j || l == k) continue;
      BsPair P;
      P.j = (uint32_t)j; P.n1 = (uint32_t)(k - j); P.n2 = (uint32_t)(l - k); P.level = level;
      const uint32_t m = P.n1 + P.n2;
      P.rank_off = rank_limbs; rank_limbs += 1 + bs_limbs(m);
      P.word_off = (uint64_t)level * n + j;
      P.scr_off = scr; if (m > 32) scr += bs_scratch_limbs(m);
      pairs.push_back(P);
    }
  }
  lstart.push_back((uint32_t)pairs.size());
  std::vector<uint32_t> primes;
  {
    std::vector<char> comp(n + 1, 0);
    for (uint64_t i = 2; i <= n; ++i) {
      if (comp[i]) continue;
      primes.push_back((uint32_t)i);
      for (uint64_t j = i * i; j <= n; j += i) comp[j] = 1;
    }
  }
  const uint32_t wl = bs_limbs((uint32_t)n) + 8;
  std::vector<uint32_t> pool(rank_limbs + 1), work(4 * wl), sc(scr + 1);
  std::vector<uint8_t> words((uint64_t)level * n + 1);
  auto t0 = std::chrono::steady_clock::now();
  const uint64_t bits = bs_ranks(pairs.data(), (uint32_t)pairs.size(), sd, primes.data(), (uint32_t)primes.size(),
                                 pool.data(), work.data(), wl);
  auto t1 = std::chrono::steady_clock::now();
  uint64_t C[33 * 33];
  bs_small_table(C, 0, 1);
  for (auto& P : pairs) bs_word_pair(P, pool.data(), sc.data(), primes.data(), (uint32_t)primes.size(), words.data(), C);
  auto t2 = std::chrono::steady_clock::now();
  fprintf(stderr, "ranks %.1f ms, words %.1f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count(), std::chrono::duration<double, std::milli>(t2 - t1).count());
  std::vector<uint64_t> a(n), t(n);
  for (uint64_t i = 0; i < n; ++i) a[i] = i;
  for (size_t L = 0; L + 1 < lstart.size(); ++L)
    for (uint32_t p = lstart[L]; p < lstart[L + 1]; ++p) {
      const BsPair& P = pairs[p];
      const uint32_t m = P.n1 + P.n2;
      for (uint32_t x = 0; x < m; ++x) t[x] = a[P.j + x];
      uint32_t ia = 0, ib = P.n1;
      for (uint32_t x = 0; x < m; ++x) a[P.j + x] = words[P.word_off + x] ? t[ib++] : t[ia++];
    }
  printf("%llu\n", (unsigned long long)bits);
  for (uint64_t i = 0; i < n; ++i) printf("%llu ", (unsigned long long)a[i]);
  printf("\n");
  return 0;
}
