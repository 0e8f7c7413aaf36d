// leaf.cu -- leaf Fisher-Yates (reference: _kernels.py:85-93 _fy_range,
// shufflers.py:137-155, leaf tasks shufflers.py:268-278).
//
// Two kernels:
//  * leaf_decode_kernel: one thread per leaf decodes the m-1 fast-dice-roller
//    draws j_i (i = m-1 .. 1) of its substream.  This is the only serial part:
//    draws are variable-length so draw k's bit offset depends on draws < k.
//  * leaf_apply_kernel: one CTA per leaf applies the m-1 swaps in parallel via
//    the successor-chain closed form (tests/decomp_model.py leaf_apply_model):
//      N(i) = next larger step with target j_i,  H(x) = first step > x targeting x,
//      final[i] = orig[W(N(i))] (or orig[j_i] if none), final[0] = orig[W(0)],
//      W(x) = W(H(x)) if H(x) exists else x.
//    Steps are bucketed by target with a shared-memory counting sort (16-bit
//    counters, two per 32-bit word, atomics in smem), buckets are tiny so each is
//    insertion-sorted by its owner, then every output gathers through the chain.
#include <algorithm>
#include "sk_kernels.h"

namespace sk {

template <typename DT>
__global__ void __launch_bounds__(128) leaf_decode_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves,
                                                          DT* __restrict__ draws,
                                                          unsigned long long* __restrict__ bits) {
  uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nleaves) return;
  LeafDesc L = leaf_desc(J, E, g);
  uint64_t m = L.hi - L.lo;
  if (m < 2) return;
  Reader32 rd;
  rd.init(L.sd, 0);
  uint64_t nb = 0;
  DT* dr = draws + L.lo;
  for (uint32_t i = (uint32_t)m - 1; i >= 1; --i) dr[i] = (DT)fdr32(rd, i + 1, nb);
  atomicAdd(&bits[L.array], (unsigned long long)nb);
}

// Warp-segmented exclusive scan over `m` 16-bit counters packed in smem.
// Each warp owns [w*S, (w+1)*S); lanes walk it 32 entries per round.
__device__ __forceinline__ void scan_counts16(uint16_t* c16, uint32_t m, uint32_t* warp_tot) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t S = (((m + nw - 1) / nw) + 31) & ~31u;
  const uint32_t b0 = wid * S, b1 = min(m, b0 + S);
  uint32_t sum = 0;
  for (uint32_t base = b0; base < b1; base += 32) {
    uint32_t p = base + lane;
    uint32_t v = (p < b1) ? c16[p] : 0;
    sum += v;
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) warp_tot[wid] = sum;
  __syncthreads();
  uint32_t carry = 0;
  for (uint32_t w = 0; w < wid; ++w) carry += warp_tot[w];
  for (uint32_t base = b0; base < b1; base += 32) {
    uint32_t p = base + lane;
    uint32_t v = (p < b1) ? c16[p] : 0;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (p < b1) c16[p] = (uint16_t)(carry + x - v);
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

template <typename V, int BLOCK>
__global__ void __launch_bounds__(BLOCK) leaf_apply_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves,
                                                           const V* __restrict__ in, V* __restrict__ out,
                                                           const uint16_t* __restrict__ draws,
                                                           uint16_t* __restrict__ scratch, uint32_t mmax) {
  extern __shared__ uint32_t sh[];
  __shared__ uint32_t warp_tot[BLOCK / 32];
  uint16_t* c16 = reinterpret_cast<uint16_t*>(sh);
  uint16_t* bucket = scratch + (uint64_t)blockIdx.x * 2 * mmax;
  uint16_t* Nn = bucket + mmax;
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31, wid = tid >> 5, nw = BLOCK / 32;

  for (uint64_t g = blockIdx.x; g < nleaves; g += gridDim.x) {
    LeafDesc L = leaf_desc(J, E, g);
    const uint32_t m = (uint32_t)(L.hi - L.lo);
    const V* src_in = in + L.lo;
    V* dst = out + L.lo;
    if (m < 2) {
      if (m == 1 && tid == 0) dst[0] = src_in[0];
      continue;
    }
    const uint16_t* dr = draws + L.lo;
    const uint32_t nwords = (m + 1) >> 1;
    for (uint32_t w = tid; w < nwords; w += BLOCK) sh[w] = 0;
    __syncthreads();
    // 1. histogram of targets
    for (uint32_t s = 1 + tid; s < m; s += BLOCK) {
      uint32_t j = dr[s];
      atomicAdd(&sh[j >> 1], 1u << ((j & 1) * 16));
    }
    __syncthreads();
    // 2. bucket starts
    scan_counts16(c16, m, warp_tot);
    __syncthreads();
    // 3. scatter step ids into their target's bucket
    for (uint32_t s = 1 + tid; s < m; s += BLOCK) {
      uint32_t j = dr[s];
      uint32_t sh16 = (j & 1) * 16;
      uint32_t old = atomicAdd(&sh[j >> 1], 1u << sh16);
      bucket[(old >> sh16) & 0xFFFFu] = (uint16_t)s;
    }
    __syncthreads();
    // 4. per target: sort bucket, successor links N, first-step-above H (in place of c16)
    {
      const uint32_t S = (((m + nw - 1) / nw) + 31) & ~31u;
      const uint32_t b0 = wid * S, b1 = min(m, b0 + S);
      uint32_t carry = (b0 > 0 && b0 < m) ? c16[b0 - 1] : 0;  // end of bucket b0-1
      __syncthreads();
      for (uint32_t base = b0; base < b1; base += 32) {
        uint32_t p = base + lane;
        uint32_t en = (p < b1) ? c16[p] : 0;
        uint32_t st = __shfl_up_sync(0xffffffffu, en, 1);
        if (lane == 0) st = carry;
        carry = __shfl_sync(0xffffffffu, en, 31);
        if (p < b1) {
          uint32_t len = en - st;
          uint32_t H = 0;
          if (len) {
            if (len >= 2) {  // insertion sort (buckets hold ~1 entry on average)
              for (uint32_t a = st + 1; a < en; ++a) {
                uint16_t v = bucket[a];
                uint32_t b = a;
                while (b > st && bucket[b - 1] > v) { bucket[b] = bucket[b - 1]; --b; }
                bucket[b] = v;
              }
            }
            uint32_t prev = bucket[st];
            for (uint32_t a = st + 1; a < en; ++a) {
              uint32_t cur = bucket[a];
              Nn[prev] = (uint16_t)cur;
              prev = cur;
            }
            Nn[prev] = 0;
            uint32_t f0 = bucket[st];
            H = (f0 > p) ? f0 : (len >= 2 ? (uint32_t)bucket[st + 1] : 0u);
          }
          c16[p] = (uint16_t)H;
        }
      }
    }
    __syncthreads();
    // 5. chase and gather
    for (uint32_t i = tid; i < m; i += BLOCK) {
      uint32_t x;
      uint32_t src;
      bool done = false;
      if (i == 0) {
        x = 0;
      } else {
        x = Nn[i];
        if (x == 0) { src = dr[i]; done = true; }
      }
      if (!done) {
        uint32_t h;
        while ((h = c16[x]) != 0) x = h;
        src = x;
      }
      dst[i] = src_in[src];
    }
    __syncthreads();
  }
}

// Fallback for leaves larger than 65536 elements (non-default cutoffs and
// fisher_yates on long arrays): one thread per leaf runs the reference loop
// directly on `out` (which already holds a copy of the input).
template <typename V>
__global__ void leaf_serial_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves, V* __restrict__ out,
                                   unsigned long long* __restrict__ bits) {
  uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nleaves) return;
  LeafDesc L = leaf_desc(J, E, g);
  uint64_t m = L.hi - L.lo;
  if (m < 2) return;
  Reader64 rd;
  rd.init(L.sd, 0);
  uint64_t nb = 0;
  V* a = out + L.lo;
  for (uint64_t i = m - 1; i >= 1; --i) {
    uint64_t j = fdr64(rd, i + 1, nb);
    V t = a[i]; a[i] = a[j]; a[j] = t;
  }
  atomicAdd(&bits[L.array], (unsigned long long)nb);
}

// ---------------------------------------------------------------- launchers
void launch_leaf_decode16(const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, uint16_t* draws,
                          unsigned long long* bits, cudaStream_t st) {
  if (!nleaves) return;
  unsigned blocks = (unsigned)((nleaves + 127) / 128);
  leaf_decode_kernel<uint16_t><<<blocks, 128, 0, st>>>(J, E, nleaves, draws, bits);
  count_launch();
}

template <typename V>
static void leaf_apply_t(const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, const void* in, void* out,
                         const uint16_t* draws, uint16_t* scratch, uint32_t mmax, uint32_t grid,
                         cudaStream_t st) {
  size_t smem = (size_t)((mmax + 1) / 2) * 4;
  if (mmax > 8192) {
    auto k = leaf_apply_kernel<V, 1024>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 1024, smem, st>>>(J, E, nleaves, (const V*)in, (V*)out, draws, scratch, mmax);
  } else {
    auto k = leaf_apply_kernel<V, 256>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, st>>>(J, E, nleaves, (const V*)in, (V*)out, draws, scratch, mmax);
  }
  count_launch();
}

uint32_t leaf_apply_grid(uint64_t nleaves, uint32_t mmax, int num_sms) {
  // Persistent CTAs: as many as fit (the per-CTA scratch is reused per leaf and
  // stays L2-resident).
  size_t smem = (size_t)((mmax + 1) / 2) * 4;
  size_t fit = (size_t)(220 * 1024) / (smem + 2048);
  int per_sm = (int)std::max((size_t)1, std::min(fit, (size_t)(mmax > 8192 ? 2 : 8)));
  uint64_t g = (uint64_t)num_sms * per_sm;
  if (g > nleaves) g = nleaves;
  return (uint32_t)(g ? g : 1);
}

void launch_leaf_apply(int eb, const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, const void* in, void* out,
                       const uint16_t* draws, uint16_t* scratch, uint32_t mmax, uint32_t grid, cudaStream_t st) {
  if (!nleaves) return;
  if (eb == 4) leaf_apply_t<uint32_t>(J, E, nleaves, in, out, draws, scratch, mmax, grid, st);
  else leaf_apply_t<unsigned long long>(J, E, nleaves, in, out, draws, scratch, mmax, grid, st);
}

void launch_leaf_serial(int eb, const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, void* out,
                        unsigned long long* bits, cudaStream_t st) {
  if (!nleaves) return;
  unsigned blocks = (unsigned)((nleaves + 63) / 64);
  if (eb == 4) leaf_serial_kernel<uint32_t><<<blocks, 64, 0, st>>>(J, E, nleaves, (uint32_t*)out, bits);
  else leaf_serial_kernel<unsigned long long><<<blocks, 64, 0, st>>>(J, E, nleaves, (unsigned long long*)out, bits);
  count_launch();
}

}  // namespace sk
