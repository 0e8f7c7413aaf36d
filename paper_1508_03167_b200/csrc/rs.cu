// rs.cu -- Rao-Sandelius splitting shuffle (reference: splitshuffle.py,
// _kernels.py:148-194), SURVEY.md §8 row F2.
//
// rs_shuffle_parallel's task tree (splitshuffle.py:92-133): a range larger
// than SPAWN_MIN = 2^14 draws one coin per element from substream
// depth*(n+1)+lo and is stably partitioned (0-group first); smaller ranges
// run the sequential splitting shuffle (rs_range: split until <= cutoff, then
// Fisher-Yates; left range first) on their own substream.
//
// GPU mapping:
//  * big ranges, level by level: chunk zero counts, per-range scan, and a
//    scatter pass (ping-pong buffers); the task tree depends only on bits,
//    so the host reads the zero counts and forms the next level;
//  * small tasks: one lane per task replays the sequential order of bit
//    consumption (splits take `size` bits; leaves take Fisher-Yates draws,
//    decoded into the u16 draws array) and records the split nodes and the
//    leaves; then every split node is applied (CTA per node, level by level)
//    and every leaf through the closed-form leaf kernel (leaf.cu, list mode).
#include <type_traits>
#include "sk_kernels.h"

namespace sk {

constexpr uint32_t kRsChunk = 2048;  // positions per chunk: 256 threads x 8

// ------------------------------------------------------------ big ranges
__device__ __forceinline__ uint32_t rs_range_of_chunk(const RsRange* R, uint32_t nr, uint64_t c) {
  uint32_t lo = 0, hi = nr;  // last range with chunk0 <= c
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (R[mid].chunk0 <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// zeros among the chunk's coin flips (one word per lane of warp 0)
__global__ void rs_chunk_zeros_kernel(const RsRange* __restrict__ R, uint32_t nr, uint64_t* __restrict__ cz,
                                      uint32_t* __restrict__ rmap) {
  const uint64_t c = blockIdx.x;
  const uint32_t r = rs_range_of_chunk(R, nr, c);
  if (threadIdx.x == 0) rmap[c] = r;  // (the split kernel reads it instead of searching again)
  const RsRange rg = R[r];
  const uint64_t size = rg.hi - rg.lo;
  const uint64_t cs = (c - rg.chunk0) * kRsChunk;
  const uint32_t lane = threadIdx.x;
  uint32_t ones = 0, valid = 0;
  const uint64_t p = cs + 64ull * lane;
  if (p < size) {
    const uint64_t nv = min((uint64_t)64, size - p);
    const uint64_t w = chunk(rg.sd, p >> 6);
    ones = __popcll(nv == 64 ? w : (w & ~(~0ull >> nv)));
    valid = (uint32_t)nv;
  }
  uint32_t z = valid - ones;
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) cz[c] = z;
}

// per range: exclusive scan of its chunks' zero counts, and the range's total
__global__ void rs_range_scan_kernel(const RsRange* __restrict__ R, uint64_t* __restrict__ cz,
                                     uint64_t* __restrict__ nz) {
  __shared__ uint32_t wsum[8];
  __shared__ uint64_t carry_s;
  const RsRange rg = R[blockIdx.x];
  const uint64_t nch = (rg.hi - rg.lo + kRsChunk - 1) / kRsChunk;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t b = 0; b < nch; b += 256) {
    const uint64_t c = b + tid;
    const uint32_t v = c < nch ? (uint32_t)cz[rg.chunk0 + c] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int w = 0; w < 8; ++w) {
      before += (w < (int)wid) ? wsum[w] : 0u;
      tot += wsum[w];
    }
    const uint64_t carry = carry_s;
    if (c < nch) cz[rg.chunk0 + c] = carry + before + x - v;  // exclusive
    __syncthreads();
    if (tid == 0) carry_s = carry + tot;
    __syncthreads();
  }
  if (tid == 0) nz[blockIdx.x] = carry_s;
}

// One chunk of a stable partition: positions [cs, cs + len) of a range of the
// given size starting at `lo` in the buffers, coin flips at stream offsets
// off + position; zb = zeros before the chunk, nz = zeros of the range.
template <typename V>
__device__ __forceinline__ uint32_t rs_partition_chunk(const V* __restrict__ in, V* __restrict__ out,
                                                       const StreamDesc& sd, uint64_t off, uint64_t lo,
                                                       uint64_t cs, uint32_t len, uint64_t zb, uint64_t nz,
                                                       uint32_t* wsum) {
  constexpr int CPW = 8;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t wbase = wid * 32 * CPW;
  uint32_t mword = 0, valid = 0;
  if (lane < (uint32_t)CPW) {
    const uint32_t i = wbase + lane * 32;
    if (i < len) {
      valid = min(32u, len - i);
      const uint32_t b = (uint32_t)(bits64_at(sd, off + cs + i) >> 32);
      mword = ~b & (valid == 32 ? 0xffffffffu : ~(0xffffffffu >> valid));  // 1 = zero flip
    }
  }
  const uint32_t cnt = __popc(mword);
  uint32_t x = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  const uint32_t rb = x - cnt;
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint32_t before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    before += (w < (int)wid) ? wsum[w] : 0u;
    total += wsum[w];
  }
  const uint32_t ltmask = ~(0xffffffffu >> lane);
#pragma unroll
  for (int k = 0; k < CPW; ++k) {
    const uint32_t i = wbase + 32 * k + lane;
    const uint32_t m = __shfl_sync(0xffffffffu, mword, k);
    const uint32_t r = __shfl_sync(0xffffffffu, rb, k);
    if (i < len) {
      const uint64_t zeros_before = zb + before + r + __popc(m & ltmask);
      const bool zero = (m >> (31 - lane)) & 1u;
      const uint64_t pos = cs + i;
      const uint64_t dst = zero ? zeros_before : nz + (pos - zeros_before);
      out[lo + dst] = in[lo + pos];
    }
  }
  __syncthreads();  // wsum reuse
  return total;
}

template <typename V>
__global__ void __launch_bounds__(256) rs_split_kernel(const RsRange* __restrict__ R, uint32_t nr,
                                                       const uint64_t* __restrict__ czp,
                                                       const uint64_t* __restrict__ nz, const V* __restrict__ in,
                                                       V* __restrict__ out, const uint32_t* __restrict__ rmap) {
  __shared__ uint32_t wsum[8];
  const uint64_t c = blockIdx.x;
  const uint32_t r = rmap[c];
  const RsRange rg = R[r];
  const uint64_t size = rg.hi - rg.lo;
  const uint64_t cs = (c - rg.chunk0) * kRsChunk;
  const uint32_t len = (uint32_t)min((uint64_t)kRsChunk, size - cs);
  rs_partition_chunk<V>(in, out, rg.sd, 0, rg.lo, cs, len, czp[c], nz[r], wsum);
}

void launch_rs_level(int eb, const RsRange* d_ranges, uint32_t nr, uint64_t nchunks, uint64_t* cz, uint64_t* nz,
                     cudaStream_t st) {
  // (cz holds 2 * nchunks words: the zero counts, then the chunk -> range map)
  rs_chunk_zeros_kernel<<<(unsigned)nchunks, 32, 0, st>>>(d_ranges, nr, cz, reinterpret_cast<uint32_t*>(cz + nchunks));
  rs_range_scan_kernel<<<nr, 256, 0, st>>>(d_ranges, cz, nz);
  count_launch();
  count_launch();
  (void)eb;
}

void launch_rs_split(int eb, const RsRange* d_ranges, uint32_t nr, uint64_t nchunks, const uint64_t* czp,
                     const uint64_t* nz, const void* in, void* out, cudaStream_t st) {
  const uint32_t* rmap = reinterpret_cast<const uint32_t*>(czp + nchunks);
  if (eb == 4)
    rs_split_kernel<uint32_t><<<(unsigned)nchunks, 256, 0, st>>>(d_ranges, nr, czp, nz, (const uint32_t*)in,
                                                                  (uint32_t*)out, rmap);
  else
    rs_split_kernel<unsigned long long><<<(unsigned)nchunks, 256, 0, st>>>(
        d_ranges, nr, czp, nz, (const unsigned long long*)in, (unsigned long long*)out, rmap);
  count_launch();
}

// ------------------------------------------------------------ small tasks
// One lane per task: the sequential order of _kernels.py:148-179 on sizes
// only.  Leaves of at most 65536 elements get their draws in draws[lo + i].
template <bool WIDE>
__global__ void rs_plan_kernel(const RsTask* __restrict__ T, uint32_t ntasks, uint64_t cutoff,
                               uint16_t* __restrict__ draws, RsNode* __restrict__ nodes,
                               unsigned long long* __restrict__ counts, uint64_t node_cap,
                               RsLeaf* __restrict__ leaves, uint64_t leaf_cap,
                               unsigned long long* __restrict__ bits) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntasks) return;
  const RsTask tk = T[t];
  constexpr int kStack = 256;  // as the reference (_kernels.py:455)
  uint64_t slo[kStack], shi[kStack];
  uint32_t sdep[kStack];
  int top = 0;
  slo[0] = tk.lo; shi[0] = tk.hi; sdep[0] = 0; top = 1;
  // 32-bit reader and dice roller when every task is at most 2^31 elements
  // (a split's bits 32 at a time); WIDE: the 64-bit ones
  using Rd = typename std::conditional<WIDE, Reader64, Reader32>::type;
  Rd rd;
  rd.init(tk.sd, 0);
  uint64_t off = 0;
  while (top > 0) {
    --top;
    const uint64_t lo = slo[top], hi = shi[top];
    const uint32_t dep = sdep[top];
    const uint64_t size = hi - lo;
    if (size <= cutoff) {
      const unsigned long long li = atomicAdd(&counts[1], 1ull);
      if (li < leaf_cap) leaves[li] = RsLeaf{lo, hi, off, t, dep};
      for (uint64_t i = size; i >= 2; --i) {  // steps i-1 .. 1, bound i
        uint64_t j;
        if constexpr (WIDE) j = fdr64(rd, i, off);
        else j = fdr32(rd, (uint32_t)i, off);
        if (size <= 65536) draws[lo + i - 1] = (uint16_t)j;
      }
      continue;
    }
    const unsigned long long ni = atomicAdd(&counts[0], 1ull);
    if (ni < node_cap) nodes[ni] = RsNode{lo, hi, off, t, dep};
    uint64_t ones = 0;
    constexpr uint32_t kw = WIDE ? 64u : 32u;
    for (uint64_t k = 0; k < size; k += kw) {
      const uint32_t kk = (uint32_t)min((uint64_t)kw, size - k);
      ones += __popcll((uint64_t)rd.take(kk));
    }
    off += size;
    const uint64_t nz = size - ones;
    if (top + 2 > kStack) {
      atomicOr(&counts[2], 1ull);  // stack overflow (the reference would fail as well)
      break;
    }
    slo[top] = lo + nz; shi[top] = hi; sdep[top] = dep + 1; ++top;
    slo[top] = lo; shi[top] = lo + nz; sdep[top] = dep + 1; ++top;
  }
  atomicAdd(&bits[tk.array], (unsigned long long)off);
}

void launch_rs_plan(const RsTask* T, uint32_t ntasks, uint64_t cutoff, uint16_t* draws, RsNode* nodes,
                    unsigned long long* counts, uint64_t node_cap, RsLeaf* leaves, uint64_t leaf_cap,
                    unsigned long long* bits, cudaStream_t st, bool wide) {
  if (!ntasks) return;
  if (wide)
    rs_plan_kernel<true><<<(ntasks + 63) / 64, 64, 0, st>>>(T, ntasks, cutoff, draws, nodes, counts, node_cap, leaves,
                                                            leaf_cap, bits);
  else
    rs_plan_kernel<false><<<(ntasks + 63) / 64, 64, 0, st>>>(T, ntasks, cutoff, draws, nodes, counts, node_cap,
                                                             leaves, leaf_cap, bits);
  count_launch();
}

// One CTA per split node (all nodes of one level): count the node's zeros,
// then partition it chunk by chunk from buf[par] into buf[par ^ 1].
template <typename V>
__global__ void __launch_bounds__(256) rs_node_kernel(const RsNode* __restrict__ nodes, const RsTask* __restrict__ T,
                                                      V* __restrict__ buf0, V* __restrict__ buf1) {
  __shared__ uint32_t wsum[8];
  __shared__ unsigned long long nz_s;
  const RsNode nd = nodes[blockIdx.x];
  const RsTask tk = T[nd.task];
  const uint32_t par = (tk.parity ^ nd.level) & 1u;
  const V* in = par ? buf1 : buf0;
  V* out = par ? buf0 : buf1;
  const uint64_t size = nd.hi - nd.lo;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) nz_s = 0;
  __syncthreads();
  unsigned long long z = 0;
  for (uint64_t p = 64ull * tid; p < size; p += 64ull * 256) {
    const uint64_t nv = min((uint64_t)64, size - p);
    const uint64_t w = bits64_at(tk.sd, nd.off + p);
    z += nv - __popcll(nv == 64 ? w : (w & ~(~0ull >> nv)));
  }
  atomicAdd(&nz_s, z);
  __syncthreads();
  const uint64_t nz = nz_s;
  uint64_t zb = 0;
  for (uint64_t cs = 0; cs < size; cs += kRsChunk) {
    const uint32_t len = (uint32_t)min((uint64_t)kRsChunk, size - cs);
    zb += rs_partition_chunk<V>(in, out, tk.sd, nd.off, nd.lo, cs, len, zb, nz, wsum);
  }
}

void launch_rs_nodes(int eb, const RsNode* nodes, uint32_t count, const RsTask* T, void* buf0, void* buf1,
                     cudaStream_t st) {
  if (!count) return;
  if (eb == 4)
    rs_node_kernel<uint32_t><<<count, 256, 0, st>>>(nodes, T, (uint32_t*)buf0, (uint32_t*)buf1);
  else
    rs_node_kernel<unsigned long long><<<count, 256, 0, st>>>(nodes, T, (unsigned long long*)buf0,
                                                              (unsigned long long*)buf1);
  count_launch();
}

// Leaves longer than 65536 (only the sequential shuffle with a large cutoff):
// copy, then the reference loop on the copy, re-decoding the draws.
template <typename V>
__global__ void rs_leaf_serial_kernel(const RsLeaf* __restrict__ L, uint32_t count, const RsTask* __restrict__ T,
                                      V* __restrict__ buf0, V* __restrict__ buf1) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= count) return;
  const RsLeaf lf = L[g];
  const RsTask tk = T[lf.task];
  const uint32_t par = (tk.parity ^ lf.depth) & 1u;
  const V* in = par ? buf1 : buf0;
  V* out = par ? buf0 : buf1;
  for (uint64_t i = lf.lo; i < lf.hi; ++i) out[i] = in[i];
  Reader64 rd;
  rd.init(tk.sd, lf.off);
  uint64_t nb = 0;
  V* a = out + lf.lo;
  for (uint64_t i = lf.hi - lf.lo; i >= 2; --i) {
    const uint64_t j = fdr64(rd, i, nb);
    const V tv = a[i - 1]; a[i - 1] = a[j]; a[j] = tv;
  }
}

void launch_rs_leaf_serial(int eb, const RsLeaf* L, uint32_t count, const RsTask* T, void* buf0, void* buf1,
                           cudaStream_t st) {
  if (!count) return;
  if (eb == 4)
    rs_leaf_serial_kernel<uint32_t><<<(count + 31) / 32, 32, 0, st>>>(L, count, T, (uint32_t*)buf0, (uint32_t*)buf1);
  else
    rs_leaf_serial_kernel<unsigned long long><<<(count + 31) / 32, 32, 0, st>>>(L, count, T,
                                                                               (unsigned long long*)buf0,
                                                                               (unsigned long long*)buf1);
  count_launch();
}

// copy [lo, hi) of every listed range from `from` to `to`
template <typename V>
__global__ void rs_copy_ranges_kernel(const uint64_t* __restrict__ list, const V* __restrict__ from,
                                      V* __restrict__ to) {
  const uint64_t lo = list[2 * blockIdx.x], hi = list[2 * blockIdx.x + 1];
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) to[i] = from[i];
}

void launch_rs_copy_ranges(int eb, const uint64_t* list, uint32_t count, const void* from, void* to,
                           cudaStream_t st) {
  if (!count) return;
  if (eb == 4)
    rs_copy_ranges_kernel<uint32_t><<<count, 256, 0, st>>>(list, (const uint32_t*)from, (uint32_t*)to);
  else
    rs_copy_ranges_kernel<unsigned long long><<<count, 256, 0, st>>>(list, (const unsigned long long*)from,
                                                                     (unsigned long long*)to);
  count_launch();
}

}  // namespace sk
