// misc.cu -- small-n batched trials (uniformity harness) and the sequential
// single-stream variant.
//
//  * chi_kernel: _kernels.py:211-250 (_chi_trials) + 197-208 (_perm_rank):
//    one thread per trial, trial key mix64(seed + GOLDEN*(t+1)), identity
//    array of n <= 20 elements, rank histogram in shared memory.
//  * bs_small: BalancedShuffle for n <= 32 (_kernels.py:292-341 _bs_small;
//    balanced.py:219-245 takes the same path there: _unrank_small): singleton
//    leaves, per pair one fast dice roll below C(n1+n2, n1) on the ONE
//    stream, the word by the lexicographic walk, the interleave.
//  * seq_kernel: _kernels.py:124-145 (_merge_shuffle, shufflers.py:194-217):
//    every leaf and merge draws from ONE stream in schedule order, so each
//    task's start offset depends on all earlier tasks' variable consumption;
//    it runs as one serial GPU thread (scope note A9 in SURVEY.md §8).
#include "sk_kernels.h"

namespace sk {

__device__ __forceinline__ uint64_t fdr_any(Reader32& rd, uint64_t b, uint64_t& nb) {
  return fdr32(rd, (uint32_t)b, nb);
}
__device__ __forceinline__ uint64_t fdr_any(Reader64& rd, uint64_t b, uint64_t& nb) { return fdr64(rd, b, nb); }

template <typename V, typename RD>
__device__ void fy_serial(V* a, uint64_t lo, uint64_t hi, RD& rd, uint64_t& nb) {
  if (hi - lo < 2) return;
  for (uint64_t i = hi - lo - 1; i >= 1; --i) {
    uint64_t j = fdr_any(rd, i + 1, nb);
    V t = a[lo + i]; a[lo + i] = a[lo + j]; a[lo + j] = t;
  }
}

template <typename V, typename RD>
__device__ void merge_serial(V* a, uint64_t j, uint64_t k, uint64_t l, RD& rd, uint64_t& nb) {
  if (k == j || l == k) return;
  uint64_t i = j, mid = k;
  for (;;) {
    uint32_t b = (uint32_t)rd.take(1);
    ++nb;
    if (b == 0) {
      if (i == mid) break;
    } else {
      if (mid == l) break;
      V t = a[i]; a[i] = a[mid]; a[mid] = t;
      ++mid;
    }
    ++i;
  }
  while (i < l) {
    uint64_t m = j + fdr_any(rd, i - j + 1, nb);
    V t = a[i]; a[i] = a[m]; a[m] = t;
    ++i;
  }
}

__device__ __forceinline__ int plan_c_dev(uint64_t n, uint64_t cutoff) {
  int c = 0;
  while ((n >> c) > cutoff) ++c;
  return c;
}

constexpr int kChiMaxN = 20;
constexpr int kBsMaxN = 32;
constexpr int kBinomW = kBsMaxN + 1;

// C(a, b) for a, b <= 32 (Pascal, _kernels.py:475-482), into shared memory
__device__ void binom_table(uint64_t* C) {
  for (int a = threadIdx.x; a < kBinomW; a += blockDim.x) {
    // row a from the closed product, exact in 64 bits for a <= 32
    uint64_t v = 1;
    for (int b = 0; b < kBinomW; ++b) {
      C[a * kBinomW + b] = b <= a ? v : 0;
      v = v * (uint64_t)(a - b) / (uint64_t)(b + 1);
    }
  }
  __syncthreads();
}

template <typename V, typename RD>
__device__ void bs_small(V* a, int n, RD& rd, uint64_t& nb, const uint64_t* __restrict__ C) {
  int c = 0;
  while ((1 << c) < n) ++c;
  const int q = 1 << c;
  V tmp[kBsMaxN];
  for (int p = 1; p < q; p += p)
    for (int i = 0; i < q; i += 2 * p) {
      const int jb = (n * i) >> c, kb = (n * (i + p)) >> c, lb = (n * min(i + 2 * p, q)) >> c;
      const int n1 = kb - jb, n2 = lb - kb, m = n1 + n2;
      if (n1 <= 0 || n2 <= 0) continue;
      uint64_t r = fdr_any(rd, C[m * kBinomW + n1], nb);  // C(m, n1) >= 2
      for (int t = 0; t < m; ++t) tmp[t] = a[jb + t];
      int kk = n1, ia = 0, ib = n1;
      for (int pos = 0; pos < m; ++pos) {  // word bit 0: next left element
        bool zero = false;
        if (kk > 0) {
          const uint64_t cnt = C[(m - pos - 1) * kBinomW + kk - 1];
          zero = r < cnt;
          if (zero) --kk;
          else r -= cnt;
        }
        a[jb + pos] = zero ? tmp[ia++] : tmp[ib++];
      }
    }
}

__global__ void __launch_bounds__(256) chi_kernel(int algo, int n, uint64_t trials, uint64_t seed, uint64_t cutoff,
                                                  unsigned long long* __restrict__ counts, uint32_t nf,
                                                  int use_smem) {
  extern __shared__ unsigned int hist[];
  __shared__ uint64_t binom[kBinomW * kBinomW];
  if (algo == 3) binom_table(binom);
  if (use_smem) {
    for (uint32_t i = threadIdx.x; i < nf; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  const int c = plan_c_dev((uint64_t)n, cutoff);
  const uint64_t q = 1ULL << c;
  uint8_t a[kChiMaxN];
  for (uint64_t tr = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; tr < trials;
       tr += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t tseed = mix64(seed + GOLDEN * (tr + 1));
    for (int i = 0; i < n; ++i) a[i] = (uint8_t)i;
    uint64_t nb = 0;
    if (algo == 3) {  // balanced (_kernels.py:344-360 _chi_trials_bs)
      Reader64 rd;
      rd.init(fresh_stream(tseed), 0);
      bs_small(a, n, rd, nb, binom);
    } else if (algo == 0 || algo == 1) {
      Reader32 rd;
      rd.init(fresh_stream(tseed), 0);
      if (algo == 0) {
        fy_serial(a, 0, (uint64_t)n, rd, nb);
      } else {
        for (uint64_t i = 0; i < q; ++i) fy_serial(a, bound_at(n, i, c), bound_at(n, i + 1, c), rd, nb);
        for (uint64_t p = 1; p < q; p += p)
          for (uint64_t i = 0; i < q; i += 2 * p)
            merge_serial(a, bound_at(n, i, c), bound_at(n, i + p, c), bound_at(n, i + 2 * p, c), rd, nb);
      }
    } else {  // tasked substreams (_kernels.py:253-289)
      for (uint64_t i = 0; i < q; ++i) {
        Reader32 rd;
        rd.init(fresh_stream(substream_seed(tseed, i)), 0);
        fy_serial(a, bound_at(n, i, c), bound_at(n, i + 1, c), rd, nb);
      }
      uint64_t r = 1;
      for (uint64_t p = 1; p < q; p += p, ++r) {
        for (uint64_t i = 0; i < q; i += 2 * p) {
          Reader32 rd;
          rd.init(fresh_stream(substream_seed(tseed, r * q + i)), 0);
          merge_serial(a, bound_at(n, i, c), bound_at(n, i + p, c), bound_at(n, i + 2 * p, c), rd, nb);
        }
      }
    }
    // little-endian factorial base rank (_kernels.py:197-208)
    uint64_t rank = 0, f = 1;
    for (int k = 1; k < n; ++k) {
      f *= (uint64_t)k;
      uint64_t d = 0;
      for (int j = 0; j < k; ++j) d += a[j] < a[k];
      rank += d * f;
    }
    if (use_smem) atomicAdd(&hist[rank], 1u);
    else atomicAdd(&counts[rank], 1ULL);
  }
  if (use_smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nf; i += blockDim.x)
      if (hist[i]) atomicAdd(&counts[i], (unsigned long long)hist[i]);
  }
}

void launch_chi(int algo, int n, uint64_t trials, uint64_t seed, uint64_t cutoff, unsigned long long* counts,
                cudaStream_t st) {
  uint64_t nf = 1;
  for (int k = 2; k <= n; ++k) nf *= (uint64_t)k;
  int use_smem = nf <= 12288;
  size_t smem = use_smem ? nf * 4 : 0;
  uint64_t want = (trials + 255) / 256;
  unsigned blocks = (unsigned)(want < (uint64_t)num_sms() * 16 ? want : (uint64_t)num_sms() * 16);
  if (!blocks) blocks = 1;
  if (smem > 48 * 1024) cudaFuncSetAttribute(chi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chi_kernel<<<blocks, 256, smem, st>>>(algo, n, trials, seed, cutoff, counts, (uint32_t)nf, use_smem);
  count_launch();
}

template <typename V>
__global__ void bs_kernel(V* a, int n, StreamDesc sd, unsigned long long* bits) {
  __shared__ uint64_t binom[kBinomW * kBinomW];
  binom_table(binom);
  if (threadIdx.x) return;
  Reader64 rd;
  rd.init(sd, 0);
  uint64_t nb = 0;
  bs_small(a, n, rd, nb, binom);
  bits[0] = nb;
}

void launch_bs_small(int eb, void* data, int n, StreamDesc sd, unsigned long long* bits, cudaStream_t st) {
  if (eb == 4) bs_kernel<uint32_t><<<1, 64, 0, st>>>((uint32_t*)data, n, sd, bits);
  else bs_kernel<unsigned long long><<<1, 64, 0, st>>>((unsigned long long*)data, n, sd, bits);
  count_launch();
}

template <typename V>
__global__ void seq_kernel(V* a, uint64_t n, uint64_t cutoff, StreamDesc sd, unsigned long long* bits) {
  if (blockIdx.x || threadIdx.x) return;
  int c = plan_c_dev(n, cutoff);
  uint64_t q = 1ULL << c, nb = 0;
  Reader64 rd;
  rd.init(sd, 0);
  for (uint64_t i = 0; i < q; ++i) fy_serial(a, bound_at(n, i, c), bound_at(n, i + 1, c), rd, nb);
  for (uint64_t p = 1; p < q; p += p)
    for (uint64_t i = 0; i < q; i += 2 * p)
      merge_serial(a, bound_at(n, i, c), bound_at(n, i + p, c), bound_at(n, i + 2 * p, c), rd, nb);
  bits[0] = nb;
}

void launch_seq(int eb, void* data, uint64_t n, uint64_t cutoff, StreamDesc sd, unsigned long long* bits,
                cudaStream_t st) {
  if (eb == 4) seq_kernel<uint32_t><<<1, 1, 0, st>>>((uint32_t*)data, n, cutoff, sd, bits);
  else seq_kernel<unsigned long long><<<1, 1, 0, st>>>((unsigned long long*)data, n, cutoff, sd, bits);
  count_launch();
}

}  // namespace sk
