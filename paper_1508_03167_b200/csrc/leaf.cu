// leaf.cu -- leaf Fisher-Yates (reference: _kernels.py:85-93 _fy_range,
// shufflers.py:137-155, leaf tasks shufflers.py:268-278).
//
// Two kernels:
//  * leaf_decode16_kernel: one lane per leaf decodes the m-1 fast-dice-roller
//    draws j_i (i = m-1 .. 1) of its substream.  This is the only serial part:
//    draws are variable-length so draw k's bit offset depends on draws < k.
//  * leaf_apply_kernel: one CTA per leaf applies the m-1 swaps in parallel via
//    the successor-chain closed form (tests/decomp_model.py leaf_apply_model):
//      N(i) = next larger step with target j_i,  H(x) = first step > x targeting x,
//      final[i] = orig[W(N(i))] (or orig[j_i] if none), final[0] = orig[W(0)],
//      W(x) = W(H(x)) if H(x) exists else x.
//    Steps are bucketed by target with a shared-memory counting sort (16-bit
//    counters, two per 32-bit word, atomics in smem); each step's bucket
//    successor is found by a min-scan of its (tiny) bucket, then every output
//    gathers through the chain.
#include <algorithm>
#include "sk_kernels.h"

namespace sk {

// One lane per leaf, one fast-dice-roller *iteration* per loop trip (so lanes
// whose draws reject do not stall the others), bits served from a per-lane ring
// of 32-bit half-words in shared memory that the warp tops up in bulk (uniform
// mix64 work, no per-lane divergent word generation).  Bounds <= 65536, so one
// iteration takes k <= 16 bits and TRIPS=16 iterations take at most 9 halves.
constexpr int kDecodeTrips = 16;
__global__ void __launch_bounds__(32) leaf_decode16_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves,
                                                           uint16_t* __restrict__ draws,
                                                           unsigned long long* __restrict__ bits) {
  __shared__ uint32_t ring[16][32];
  const uint32_t lane = threadIdx.x;
  const uint64_t g = (uint64_t)blockIdx.x * 32 + lane;
  LeafDesc L;
  uint32_t m = 0;
  if (g < nleaves) {
    L = leaf_desc(J, E, g);
    m = (uint32_t)(L.hi - L.lo);
  } else {
    L.lo = 0; L.hi = 0; L.array = 0; L.sd = fresh_stream(0);
  }
  uint32_t i = m >= 2 ? m - 1 : 0;
  uint16_t* dr = draws + L.lo;
  uint64_t gw = 0;
  uint32_t wr = 0, rd = 0;
  if (i) {
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      uint64_t x = chunk(L.sd, gw++);
      ring[wr & 15][lane] = (uint32_t)(x >> 32);
      ring[(wr + 1) & 15][lane] = (uint32_t)x;
      wr += 2;
    }
  }
  uint32_t A = ring[0][lane], B = ring[1][lane], C = ring[2][lane];
  rd = 3;
  uint32_t pos = 0;
  uint32_t b = i + 1, bm1 = i, lb = 31 - __clz(i | 1), v = 1, c = 0;
  uint32_t nb = 0;
  while (__any_sync(0xffffffffu, i != 0)) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (i != 0 && wr - rd <= 14) {
        uint64_t x = chunk(L.sd, gw++);
        ring[wr & 15][lane] = (uint32_t)(x >> 32);
        ring[(wr + 1) & 15][lane] = (uint32_t)x;
        wr += 2;
      }
    }
#pragma unroll 4
    for (int tr = 0; tr < kDecodeTrips; ++tr) {
      // branch-free trip: lanes that finished (i == 0) keep their state
      const bool act = i != 0;
      uint32_t lv = 31 - __clz(v);
      uint32_t k = lb - lv;
      k += ((v << k) <= bm1) ? 1u : 0u;
      k = act ? k : 0u;
      uint32_t x = __funnelshift_l(B, A, pos);
      uint32_t r = k ? (x >> (32 - k)) : 0u;
      uint32_t cc = (c << k) | r;
      pos += k;
      nb += k;
      const bool acc = act && cc < b;
      if (acc) dr[i] = (uint16_t)cc;
      const uint32_t i_old = i;
      c = acc ? 0u : cc - b;
      v = acc ? 1u : (v << k) - b;
      i = acc ? i_old - 1 : i_old;          // next step, bound b = i + 1
      b = acc ? i_old : b;
      bm1 = acc ? i_old - 1 : bm1;
      lb = acc ? 31 - __clz((i_old - 1) | 1) : lb;
      const uint32_t nxt = ring[rd & 15][lane];
      const bool cross = pos >= 32;
      pos = cross ? pos - 32 : pos;
      A = cross ? B : A;
      B = cross ? C : B;
      C = cross ? nxt : C;
      rd += cross ? 1u : 0u;
    }
  }
  if (m >= 2) atomicAdd(&bits[L.array], (unsigned long long)nb);
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
  uint16_t* bucket = scratch + (uint64_t)blockIdx.x * 3 * mmax;
  uint16_t* Nn = bucket + mmax;
  uint16_t* Hg = Nn + mmax;
  const uint32_t tid = threadIdx.x;

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
    // 4. successor links without sorting: N(s) = min{s' > s in bucket(j_s)},
    //    H(x) = min{s' > x in bucket(x)}; buckets hold ~1 step on average.
    for (uint32_t s = 1 + tid; s < m; s += BLOCK) {
      uint32_t p = dr[s];
      uint32_t en = c16[p], st = p ? c16[p - 1] : 0u;
      uint32_t best = 0xFFFFFFFFu;
      for (uint32_t a = st; a < en; ++a) {
        uint32_t v = bucket[a];
        if (v > s && v < best) best = v;
      }
      Nn[s] = (uint16_t)(best == 0xFFFFFFFFu ? 0u : best);
    }
    for (uint32_t x = tid; x < m; x += BLOCK) {
      uint32_t en = c16[x], st = x ? c16[x - 1] : 0u;
      uint32_t best = 0xFFFFFFFFu;
      for (uint32_t a = st; a < en; ++a) {
        uint32_t v = bucket[a];
        if (v > x && v < best) best = v;
      }
      Hg[x] = (uint16_t)(best == 0xFFFFFFFFu ? 0u : best);
    }
    __syncthreads();
    for (uint32_t x = tid; x < m; x += BLOCK) c16[x] = Hg[x];
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
  unsigned blocks = (unsigned)((nleaves + 31) / 32);
  leaf_decode16_kernel<<<blocks, 32, 0, st>>>(J, E, nleaves, draws, bits);
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
