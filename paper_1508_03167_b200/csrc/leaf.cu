// leaf.cu -- leaf Fisher-Yates (reference: _kernels.py:85-93 _fy_range,
// shufflers.py:137-155, leaf tasks shufflers.py:268-278).
//
// Two stages:
//  * decode (leaf_decode_ws_kernel): one lane per leaf decodes the m-1
//    fast-dice-roller draws j_i (i = m-1 .. 1) of its substream, helper warps
//    feed it bits and store its draws.  This is the only serial part: draws
//    are variable-length, so draw k's bit offset depends on the draws before
//    it.
//  * apply: the m-1 swaps in parallel via the successor-chain closed form
//    (tests/decomp_model.py leaf_apply_model):
//      N(i) = next larger step with target j_i,  H(x) = first step > x targeting x,
//      final[i] = orig[W(N(i))] (or orig[j_i] if none), final[0] = orig[W(0)],
//      W(x) = W(H(x)) if H(x) exists else x.
//    leaf_apply_v3_kernel (leaves of 2049..65536) groups the steps by target
//    with byte counters in shared memory; leaf_apply_kernel (leaves of <= 2048
//    and the Rao-Sandelius leaf lists) with 16-bit counters.
#include <stdexcept>
#include <algorithm>
#include "sk_kernels.h"

namespace sk {

// debug: stop the leaf-apply pipeline after phase k (phase timing experiments)
__device__ int g_leaf_stop = 99;

template <bool FRESH>
__device__ __forceinline__ uint64_t leaf_word(const StreamDesc& sd, uint64_t w) {
  if (FRESH) return mix64(sd.state + (w + 1) * GOLDEN);  // fresh substream: no prefix
  return chunk(sd, w);
}

// Blocks of kDecodeBlock leaves: the decode is latency-bound with about one
// chain warp per SM sub-partition, so each block's chain warps must land on
// distinct schedulers.
constexpr int kDecodeBlock = 128;

// Warp-specialised decode: the same one-lane-per-leaf FDR, with everything
// that is not on the draw's dependency chain moved to helper warps.
//  * chain warps (threads kDecodeBlock..2*kDecodeBlock-1, one per leaf; the
//    high warp ids, which the issue arbiter favours): per trip only the FDR
//    iteration, the bit window shift, and one shared-memory store of an
//    accepted draw into the lane's column of `stage`;
//  * helper warps (threads 0..kDecodeBlock-1, helper t serves lane t):
//    generate the lane's stream words into its column of `ring` and move
//    accepted draws from `stage` to global memory as 16-byte chunks.
// Both sides meet at a block barrier every T trips (an epoch): the chain
// lanes publish their ring read position and bound there; between two
// barriers the helpers refill ring slots the chain lanes have already passed
// and flush draws staged before the barrier, while the chain lanes run their
// next epoch.  Ring capacity 2T halves (an epoch reads at most T/2 + 1),
// stage capacity 4T draws (an epoch accepts at most T; at most 7 wait for
// their chunk).  Longer epochs cost fewer barriers but more shared memory:
// T = 64 (128 KB, one block per SM) when the grid fits the SMs, else T = 32
// (64 KB).  Measured alternatives: per-lane flags instead of barriers (two
// CTA fences per epoch cost more than the barrier), precomputing the next
// trip's batch size for both outcomes (no faster: the trip is bound by issue
// and ALU-pipe throughput, not by the v -> k chain).
template <int T>
struct WsGeom {
  static constexpr int kRing = 2 * T;
  static constexpr int kStage = 4 * T;
  static constexpr size_t kSmem = (size_t)kRing * kDecodeBlock * 4 + (size_t)kStage * kDecodeBlock * 2 + 2 * kDecodeBlock * 4;
};

template <bool FRESH, int T>
__global__ void __launch_bounds__(2 * kDecodeBlock) leaf_decode_ws_kernel(ArrayJob J, ExplicitTask E,
                                                                          uint64_t nleaves,
                                                                          uint16_t* __restrict__ draws,
                                                                          unsigned long long* __restrict__ bits) {
  constexpr int kRing = WsGeom<T>::kRing, kStage = WsGeom<T>::kStage;
  extern __shared__ uint4 ws_smem[];
  uint32_t* const ring = reinterpret_cast<uint32_t*>(ws_smem);                        // [kRing][kDecodeBlock]
  uint16_t* const stage = reinterpret_cast<uint16_t*>(ring + kRing * kDecodeBlock);  // [kStage][kDecodeBlock]
  uint32_t* const ctl_rd = reinterpret_cast<uint32_t*>(stage + kStage * kDecodeBlock);
  uint32_t* const ctl_b = ctl_rd + kDecodeBlock;
  const bool chain = threadIdx.x >= kDecodeBlock;
  const uint32_t lane = threadIdx.x & (kDecodeBlock - 1);
  const uint64_t g = (uint64_t)blockIdx.x * kDecodeBlock + lane;
  LeafDesc L;
  uint32_t m = 0;
  if (g < nleaves) {
    L = leaf_desc(J, E, g);
    m = (uint32_t)(L.hi - L.lo);
  } else {
    L.lo = 0; L.hi = 0; L.array = 0; L.sd = fresh_stream(0);
  }
  if (m < 2) m = 1;  // no draws
  uint16_t* const dr = draws + L.lo;

  if (chain) {
    __syncthreads();  // the helpers' first fill
    const uint32_t* const rcol = ring + lane;
    uint32_t A = rcol[0], B = rcol[kDecodeBlock];
    uint32_t rd = 2, pos = 0, v = 1, c = 0;
    uint32_t b = m;  // bound of the current draw i = b - 1
    // byte offset of the next accepted draw's stage slot (row * 256 + lane * 2)
    uint32_t so = lane * 2;
    uint8_t* const sbase = reinterpret_cast<uint8_t*>(stage);
    for (;;) {
#pragma unroll 8
      for (int tr = 0; tr < T; ++tr) {
        const uint32_t nxt = rcol[(rd & (kRing - 1)) * kDecodeBlock];  // next half, used on a crossing
        const bool act = b > 1;
        uint32_t k = __clz(v) - __clz(b);  // smallest k with v << k >= b
        uint32_t vk = v << k;
        const bool up = vk < b;
        k += up ? 1u : 0u;
        vk = up ? vk + vk : vk;
        const uint32_t x = __funnelshift_l(B, A, pos);
        const uint32_t cc = __funnelshift_l(x, c, k);  // (c << k) | top k bits of x
        const bool acc = act && cc < b;
        if (acc) *reinterpret_cast<uint16_t*>(sbase + so) = (uint16_t)cc;
        so = acc ? ((so + 2 * kDecodeBlock) & (kStage * kDecodeBlock * 2 - 1)) : so;
        c = acc ? 0u : cc - b;
        v = acc ? 1u : vk - b;
        b -= acc ? 1u : 0u;
        pos += act ? k : 0u;
        const bool cross = pos >= 32;
        pos = cross ? pos - 32 : pos;
        A = cross ? B : A;
        B = cross ? nxt : B;
        rd += cross ? 1u : 0u;
      }
      ctl_rd[lane] = rd;
      ctl_b[lane] = b;
      if (!__syncthreads_or(b > 1)) break;
    }
    if (m >= 2) atomicAdd(&bits[L.array], 32ull * (rd - 2) + pos);  // bits consumed = halves passed + pos
  } else {
    uint64_t gw = 0;   // next stream word
    uint32_t wr = 0;   // next ring half to fill
    uint32_t fl = 0;   // draws flushed (draw index m-1-fl is the next)
    auto fill = [&](uint32_t upto) {  // halves [wr, upto)
      while (wr + 2 <= upto) {
        const uint64_t w = leaf_word<FRESH>(L.sd, gw++);
        ring[(wr & (kRing - 1)) * kDecodeBlock + lane] = (uint32_t)(w >> 32);
        ring[((wr + 1) & (kRing - 1)) * kDecodeBlock + lane] = (uint32_t)w;
        wr += 2;
      }
    };
    auto flush = [&](uint32_t cnt) {  // draws accepted: t < cnt is draw m-1-t
      while (fl < cnt) {
        const uint32_t itop = m - 1 - fl;
        uint16_t* const p = dr + itop;
        if (((reinterpret_cast<uintptr_t>(p) >> 1) & 7) == 7 && itop >= 8) {
          if (cnt - fl < 8) break;
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t lo16 = stage[((fl + 7 - 2 * q) & (kStage - 1)) * kDecodeBlock + lane];
            const uint32_t hi16 = stage[((fl + 6 - 2 * q) & (kStage - 1)) * kDecodeBlock + lane];
            w[q] = lo16 | (hi16 << 16);
          }
          *reinterpret_cast<uint4*>(p - 7) = make_uint4(w[0], w[1], w[2], w[3]);
          fl += 8;
        } else {
          *p = stage[(fl & (kStage - 1)) * kDecodeBlock + lane];
          fl += 1;
        }
      }
    };
    if (m >= 2) fill(kRing);
    __syncthreads();
    for (;;) {
      // the chain lanes run an epoch; meanwhile flush and top up from the
      // positions published at the previous barrier
      const bool more = __syncthreads_or(0);
      const uint32_t rd = ctl_rd[lane], bb = ctl_b[lane];
      if (m >= 2) {
        flush(m - bb);
        if (more) fill(rd + kRing);
      }
      if (!more) break;
    }
  }
}

template <int T>
static void launch_ws(bool fresh, unsigned blocks, const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves,
                      uint16_t* draws, unsigned long long* bits, cudaStream_t st) {
  constexpr size_t smem = WsGeom<T>::kSmem;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(leaf_decode_ws_kernel<true, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(leaf_decode_ws_kernel<false, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (fresh) leaf_decode_ws_kernel<true, T><<<blocks, 2 * kDecodeBlock, smem, st>>>(J, E, nleaves, draws, bits);
  else leaf_decode_ws_kernel<false, T><<<blocks, 2 * kDecodeBlock, smem, st>>>(J, E, nleaves, draws, bits);
}

// Warp-per-leaf speculative decode, for jobs with few leaves (the
// lane-per-leaf kernel above then leaves the GPU idle for the ~3.8 ms its
// per-lane chain of 65 535 draws takes).  Bit-identical to the serial loop
// (_kernels.py:64-93); what is speculated is only WHERE each draw starts.
//
// A batch is up to 16 consecutive steps s = i - d whose first FDR iteration
// takes the same K bits and whose second iteration (after one rejection:
// v' = 2^K - b, c' = c - b) takes the same k1 bits -- both are functions of
// the bound alone, constant over long runs of steps (the run's lower end in
// closed form: b > 2^(K+k1-1) / (2^(k1-1) + 1)).  Draw d of the batch then
// starts at o + d*K + h*k1 when exactly h earlier draws of the batch were
// rejected once and the rest accepted at once.  Lane 2d + h evaluates draw d
// under hypothesis h in {0, 1}: the first iteration and, on a rejection, the
// second and the third.  Three ballots (rejected once / twice / three times)
// resolve the batch without touching memory: the draws up to the first
// rejection under h = 0 are final; if that draw's second iteration accepts,
// the following draws are read under h = 1 up to the next rejection, which
// ends the batch; a draw rejected twice ends the batch there (its lane knows
// the k2 bits of its third iteration; only after a third rejection does it
// run the serial loop).  About 6 draws per batch at full leaves (model:
// tests/decomp_model.py spec_decode_model, checked against the serial loop).
constexpr int kSpecWarps = 4;
constexpr uint32_t kSpecRing = 128;    // halves: 64 stream words per warp
constexpr uint32_t kSpecAhead = 1536;  // bits kept generated past the batch start
// Jobs with at most this many leaves take the warp-per-leaf decode (measured:
// 2.48 ms per leaf up to ~600 leaves, 2.95 ms at 1024, 4.0 ms at 2048, against
// 3.8 ms at any count for a lane per leaf).
static uint64_t g_spec_decode_max = 1024;

template <bool FRESH>
__global__ void __launch_bounds__(32 * kSpecWarps)
    leaf_decode_spec_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves, uint16_t* __restrict__ draws,
                            unsigned long long* __restrict__ bits) {
  __shared__ uint32_t ring_all[kSpecWarps][kSpecRing];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t g = (uint64_t)blockIdx.x * kSpecWarps + wid;
  if (g >= nleaves) return;  // whole warp
  uint32_t* const ring = ring_all[wid];
  const LeafDesc L = leaf_desc(J, E, g);
  const uint32_t m = (uint32_t)(L.hi - L.lo);
  if (m < 2) return;
  uint16_t* const dr = draws + L.lo;
  uint32_t wgen = 0;  // stream words [wgen - 64, wgen) are in the ring
  auto refill = [&]() {
    const uint64_t x = leaf_word<FRESH>(L.sd, (uint64_t)wgen + lane);
    const uint32_t h = ((wgen + lane) * 2) & (kSpecRing - 1);
    __syncwarp();  // every lane is done reading the slots this overwrites (they lie >= 2048 bits behind o)
    ring[h] = (uint32_t)(x >> 32);
    ring[h + 1] = (uint32_t)x;
    wgen += 32;
    __syncwarp();
  };
  refill();
  refill();
  const uint32_t d = lane >> 1, h = lane & 1;
  const uint32_t lanebit = 1u << lane;
  uint32_t o = 0;       // bit offset of the batch's first draw
  uint32_t i = m - 1;   // the batch's first step (bound i + 1)
  uint32_t run_lo = m;  // steps [run_lo, i] share (K, k1); recomputed when i drops below it
  uint32_t K = 0, k1 = 1;
  bool pow2 = false;  // the run is one step whose bound is a power of two
  while (i >= 1) {
    if (i < run_lo) {  // next run of steps with one (K, k1)
      K = 32 - __clz(i);
      const uint32_t bt = i + 1, vt = (1u << K) - bt;
      pow2 = vt == 0;
      if (pow2) {  // bound a power of two: never rejects, a run of its own
        k1 = 1;
        run_lo = i;
      } else {
        k1 = __clz(vt) - __clz(bt);
        k1 += ((vt << k1) < bt) ? 1u : 0u;
        run_lo = (1u << (K + k1 - 1)) / ((1u << (k1 - 1)) + 1u);  // smallest bound of the run, minus one
      }
    }
    while (o + kSpecAhead > 64 * wgen) refill();
    const uint32_t n = min(16u, i - run_lo + 1);
    const bool live = d < n;
    const uint32_t s = live ? i - d : 1u, b = s + 1;
    const uint32_t lm = 0xffffffffu >> (32 - 2 * n);  // lanes of the batch's draws
    // rejection tests on the left-aligned window: c >= b  <=>  Y >= b << (32 - K), and with
    // Z = Y - (b << (32 - K)) the second iteration's c2 = Z >> (32 - K - k1)
    const uint32_t sh2 = 32 - K - k1;
    const uint32_t bsh = b << (32 - K), bsh2 = b << sh2;
    const uint32_t off = o + d * K + h * k1;
    const uint32_t q = off >> 5;
    const uint32_t w0 = ring[q & (kSpecRing - 1)], w1 = ring[(q + 1) & (kSpecRing - 1)];
    const uint32_t w2 = ring[(q + 2) & (kSpecRing - 1)];
    const uint32_t Y = __funnelshift_l(w1, w0, off);   // stream bits [off, off + 32)
    const uint32_t Y2 = __funnelshift_l(w2, w1, off);  // [off + 32, off + 64)
    // third iteration (after two rejections: v2 = (v' << k1) - b, k2 bits)
    const uint32_t v2 = ((((1u << K) - b)) << k1) - b;
    uint32_t k2 = __clz(v2) - __clz(b);
    k2 += ((v2 << (k2 & 31)) < b) ? 1u : 0u;
    const uint32_t t3 = K + k1;                                     // <= 32
    const uint32_t Y3 = t3 == 32 ? Y2 : __funnelshift_l(Y2, Y, t3);  // [off + K + k1, ... + 32)
    const uint32_t Z = Y - bsh;
    const bool r1 = live && !pow2 && Y >= bsh;  // (b << (32 - K) wraps to 0 for a power of two)
    const bool r2 = r1 && Z >= bsh2;
    const uint32_t c2 = Z >> sh2;
    const uint32_t c3 = ((c2 - b) << (k2 & 31)) | (Y3 >> ((32 - k2) & 31));
    const bool r3 = r2 && c3 >= b;
    uint32_t val = r2 ? c3 : (r1 ? c2 : Y >> (32 - K));
    const uint32_t R = __ballot_sync(0xffffffffu, r1);
    const uint32_t D = __ballot_sync(0xffffffffu, r2);
    const uint32_t T = __ballot_sync(0xffffffffu, r3);
    // h = 0 lanes up to the first rejection f0; then h = 1 lanes up to the next rejection f1
    const uint32_t rm0 = R & 0x55555555u;
    const uint32_t l0 = rm0 & (0u - rm0);   // lane (f0, 0), or 0
    const uint32_t ab0 = 0u - (l0 << 2);    // lanes of the draws after f0 (0 when there is no f0)
    const uint32_t rm1 = R & 0xAAAAAAAAu & ab0;
    const uint32_t l1 = rm1 & (0u - rm1);   // lane (f1, 1), or 0
    const uint32_t ab1 = 0u - (l1 << 1);    // lanes of the draws after f1
    const bool dbl0 = (D & l0) != 0;
    // lanes on the true path
    const uint32_t path0 = 0x55555555u & ~ab0;                      // draws 0..f0 under h = 0 (all when no rejection)
    const uint32_t path1 = dbl0 ? 0u : (0xAAAAAAAAu & ab0 & ~ab1);  // draws f0+1..f1 under h = 1
    const uint32_t path = (path0 | path1) & lm;
    const uint32_t dl = dbl0 ? l0 : (D & l1);  // the lane whose draw was rejected twice (it ends the batch), if any
    const uint32_t consumed = (uint32_t)__popc(path);
    uint32_t extra = (l0 ? k1 : 0u) + ((!dbl0 && l1) ? k1 : 0u);
    if (dl) {
      // bits the batch used beyond K per draw, known to that lane: its own shift, k1 and k2 --
      // or, after a third rejection, whatever the serial loop (_kernels.py:71-82) takes
      uint32_t e = h * k1 + k1 + k2;
      if ((T & dl) && lanebit == dl) {
        uint32_t v = (v2 << k2) - b, cc = c3 - b;
        uint32_t p = off + K + k1 + k2;
        for (;;) {
          uint32_t k = __clz(v) - __clz(b);
          k += ((v << k) < b) ? 1u : 0u;
          uint32_t x;
          if (p + 32 > 64 * wgen) {
            x = (uint32_t)(bits64_at(L.sd, p) >> 32);
          } else {
            const uint32_t qq = p >> 5;
            x = __funnelshift_l(ring[(qq + 1) & (kSpecRing - 1)], ring[qq & (kSpecRing - 1)], p);
          }
          cc = (cc << k) | (x >> (32 - k));
          v <<= k;
          p += k;
          if (cc < b) break;
          cc -= b;
          v -= b;
        }
        val = cc;
        e = p - (o + (d + 1) * K);
      }
      extra = __shfl_sync(0xffffffffu, e, __ffs(dl) - 1);
    }
    if (path & lanebit) dr[s] = (uint16_t)val;
    o += consumed * K + extra;
    i -= consumed;
  }
  if (lane == 0) atomicAdd(&bits[L.array], (unsigned long long)o);
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

// compare-exchange (ascending)
__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
  uint32_t lo = min(a, b), hi = max(a, b);
  a = lo; b = hi;
}

// Leaf apply.  Targets are handled in halves of <= 32768 so that both the
// 16-bit bucket cursors (64 KB) and the bucket array itself (<= 128 KB) live in
// shared memory: histogram, scan, scatter and the per-target bucket sort are
// all shared-memory work.  Successor links N go to global scratch, the H
// table is staged in global and reloaded into shared memory for the chase.
constexpr uint32_t kLeafHalf = 32768;

// list (optional): leaf g = [list[2g], list[2g+1]) instead of the schedule's
// leaf g (the Rao-Sandelius leaves).
template <typename V, int BLOCK>
__global__ void __launch_bounds__(BLOCK) leaf_apply_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves,
                                                           const V* in, V* out,
                                                           const uint16_t* __restrict__ draws,
                                                           uint16_t* __restrict__ scratch, uint32_t mmax,
                                                           const uint64_t* __restrict__ list) {
  extern __shared__ uint32_t sh[];
  __shared__ uint32_t warp_tot[BLOCK / 32];
  const uint32_t half = mmax < kLeafHalf ? mmax : kLeafHalf;
  const uint32_t cw = (half + 1) >> 1;                           // cursor words
  uint16_t* cur = reinterpret_cast<uint16_t*>(sh);               // [half]
  uint16_t* bkt = reinterpret_cast<uint16_t*>(sh + cw);          // [mmax] buckets; later H
  const uint32_t ms = (mmax + 1) & ~1u;
  constexpr bool kStage = BLOCK == 256;
  V* sdata = reinterpret_cast<V*>(sh + ((cw + ((mmax + 1) >> 1) + 1) & ~1u));  // after the buckets, 8-byte aligned
  uint16_t* Nn = scratch + (uint64_t)blockIdx.x * leaf_scratch_stride(mmax);
  uint16_t* Hg = Nn + ms;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr uint32_t NW = BLOCK / 32;

  for (uint64_t g = blockIdx.x; g < nleaves; g += gridDim.x) {
    LeafDesc L;
    if (list) {
      L.lo = list[2 * g];
      L.hi = list[2 * g + 1];
    } else {
      L = leaf_desc(J, E, g);
    }
    const uint32_t m = (uint32_t)(L.hi - L.lo);
    const V* src_in = in + L.lo;
    V* dst = out + L.lo;
    if (m < 2) {
      if (m == 1 && tid == 0) dst[0] = src_in[0];
      continue;
    }
    // small leaves (BLOCK 256 configuration): the data is staged in shared
    // memory, gathered from there, and may be written back in place
    if (kStage) {
      for (uint32_t k = tid; k < m; k += BLOCK) sdata[k] = src_in[k];
    }
    const uint16_t* __restrict__ dr = draws + L.lo;
    if (tid == 0) {  // pull this leaf's data and the next leaf's draws into L2
      if (g == blockIdx.x) l2_prefetch(dr, (size_t)m * 2);
      if (g + gridDim.x < nleaves) {
        uint64_t nlo, nhi;
        if (list) {
          nlo = list[2 * (g + gridDim.x)];
          nhi = list[2 * (g + gridDim.x) + 1];
        } else {
          const LeafDesc Ln = leaf_desc(J, E, g + gridDim.x);
          nlo = Ln.lo;
          nhi = Ln.hi;
        }
        l2_prefetch(draws + nlo, (size_t)(nhi - nlo) * 2);
      }
    }
    for (uint32_t T0 = 0; T0 < m; T0 += kLeafHalf) {
      const uint32_t nt = min(kLeafHalf, m - T0);  // targets [T0, T0+nt)
      // the leaf's data is gathered only at the end: pull it into L2 during
      // the last target half (earlier it would be evicted before use)
      if (tid == 0 && T0 + kLeafHalf >= m) l2_prefetch(src_in, (size_t)m * sizeof(V));
      for (uint32_t w = tid; w < ((nt + 1) >> 1); w += BLOCK) sh[w] = 0;
      __syncthreads();
      // 1. histogram of this half's targets (steps s = 1 .. m-1)
#pragma unroll 4
      for (uint32_t s = 1 + tid; s < m; s += BLOCK) {
        const uint32_t j = (uint32_t)dr[s] - T0;
        if (j < nt) atomicAdd(&sh[j >> 1], 1u << ((j & 1) << 4));
      }
      __syncthreads();
      if (g_leaf_stop <= 1) continue;
      // 2. bucket starts
      scan_counts16(cur, nt, warp_tot);
      __syncthreads();
      if (g_leaf_stop <= 2) continue;
      // 3. scatter step ids into their target's bucket (shared memory)
#pragma unroll 4
      for (uint32_t s = 1 + tid; s < m; s += BLOCK) {
        const uint32_t j = (uint32_t)dr[s] - T0;
        if (j < nt) {
          const uint32_t sh16 = (j & 1) << 4;
          const uint32_t old = atomicAdd(&sh[j >> 1], 1u << sh16);
          bkt[(old >> sh16) & 0xFFFFu] = (uint16_t)s;
        }
      }
      __syncthreads();
      if (g_leaf_stop <= 3) continue;
      // 4. per target (lane-consecutive targets, warps interleaved): sort the
      //    bucket in place (insertion; buckets hold ~1 step, ln(m/p) near 0),
      //    link successors N, H(p) = first step > p targeting p.
      for (uint32_t base = wid * 32; base < nt; base += NW * 32) {
        const uint32_t pl = base + lane;
        if (pl < nt) {
          const uint32_t p = T0 + pl;
          const uint32_t en = cur[pl];
          const uint32_t st = pl ? (uint32_t)cur[pl - 1] : 0u;
          for (uint32_t a = st + 1; a < en; ++a) {
            const uint16_t v = bkt[a];
            uint32_t b = a;
            while (b > st && bkt[b - 1] > v) { bkt[b] = bkt[b - 1]; --b; }
            bkt[b] = v;
          }
          uint32_t H = 0;
          if (en > st) {
            uint32_t prev = bkt[st];
            H = (prev > p) ? prev : 0u;
            for (uint32_t a = st + 1; a < en; ++a) {
              const uint32_t cur_s = bkt[a];
              if (H == 0) H = cur_s;  // first step after a self-step (prev == p)
              Nn[prev] = (uint16_t)cur_s;
              prev = cur_s;
            }
            Nn[prev] = 0;
          }
          Hg[p] = (uint16_t)H;
        }
      }
      __syncthreads();
    }
    if (g_leaf_stop <= 4) continue;
    // H of every target into shared memory (over the bucket area)
    for (uint32_t w = tid; w < ((m + 1) >> 1); w += BLOCK)
      reinterpret_cast<uint32_t*>(bkt)[w] = reinterpret_cast<const uint32_t*>(Hg)[w];
    __syncthreads();
    const uint16_t* Hs = bkt;
    // 5. chase and gather: final[i] = orig[W(N(i))] or orig[j_i]; final[0] = orig[W(0)]
    //    (batches of 8 outputs per thread: the N/draw loads, then the data
    //    gathers, are in flight together)
    for (uint32_t i0 = tid; i0 < m; i0 += 8 * BLOCK) {
      uint32_t x[8], d[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = i0 + k * BLOCK;
        x[k] = (i < m && i != 0) ? (uint32_t)Nn[i] : 0u;
        d[k] = (i < m && i != 0) ? (uint32_t)dr[i] : 0u;
      }
      V v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = i0 + k * BLOCK;
        uint32_t src;
        if (i != 0 && x[k] == 0) {
          src = d[k];
        } else {
          uint32_t y = x[k], h;
          while ((h = Hs[y]) != 0) y = h;
          src = y;
        }
        if (i < m) v[k] = kStage ? sdata[src] : src_in[src];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = i0 + k * BLOCK;
        if (i < m) dst[i] = v[k];
      }
    }
    __syncthreads();
  }
}

// Leaf apply, one pass over all targets (leaves of 8193 .. 65536 elements).
//
// 1024 threads; thread t owns steps s = 8192k + 8t + e (k, e < 8), whose 16-bit
// values (the draw j_s, then its bucket slot, then N(s) or j_s) stay in 32
// registers.  The per-target counters are BYTES (four per word, 64 KB for
// 65536 targets) grouped by 16 targets, with one 16-bit start per group, so
// the counters, the group starts and the whole bucket array (128 KB) fit in
// shared memory together and no target halves are needed:
//  1. histogram: one byte atomic per step;
//  2. per group of 16 targets: its total and the in-group exclusive prefixes
//     (in place, dp4a + a byte-prefix multiply), block scan of the totals.
//     A group total above 255 (never seen: the counts near target 0 are
//     ~ln(m/p), a group of 16 holds ~150 at most) or a lost carry (byte sum
//     != m - 1) sends the leaf to the serial fallback;
//  3. scatter: the byte atomic returns the step's slot in its bucket; the
//     counters end as the bucket ends;
//  4. per target (four per counter word, consecutive targets on consecutive
//     lanes): buckets of <= 2 steps are resolved branch-free in place
//     (slot <- successor N(s), or the target itself when s is the bucket's
//     last step); H(p) = min{b in bucket(p) : b > p} goes to the CTA's
//     scratch; larger buckets are queued;
//  5. queued buckets: <= 8 entries in registers, longer ones through the
//     scratch (O(k^2), k ~ ln(m/p): only the first few hundred targets);
//  6. each owned step picks up its slot's value;
//  7. H into shared memory (over the buckets), then every output gathers
//     orig[W(N(s))] (W: follow H to its root) or orig[j_s]; 16-byte stores.
__device__ int g_leaf_force_fallback = 0;
static int g_leaf_l2pol_host = 1;  // debug knob (host side): 0 = no L2 eviction hints (A/B timing)

__device__ __forceinline__ void cx(uint32_t& a, uint32_t& b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}
// Batcher odd-even merge sorts (19 and 63 compare-exchanges), ascending
__device__ __forceinline__ void sort_net8(uint32_t* k) {
#pragma unroll
  for (int p = 1; p < 8; p <<= 1)
#pragma unroll
    for (int q = p; q >= 1; q >>= 1)
#pragma unroll
      for (int j = q % p; j + q < 8; j += 2 * q)
#pragma unroll
        for (int i = 0; i < q; ++i)
          if ((i + j) / (2 * p) == (i + j + q) / (2 * p) && i + j + q < 8) cx(k[i + j], k[i + j + q]);
}
__device__ __forceinline__ void sort_net16(uint32_t* k) {
#pragma unroll
  for (int p = 1; p < 16; p <<= 1)
#pragma unroll
    for (int q = p; q >= 1; q >>= 1)
#pragma unroll
      for (int j = q % p; j + q < 16; j += 2 * q)
#pragma unroll
        for (int i = 0; i < q; ++i)
          if ((i + j) / (2 * p) == (i + j + q) / (2 * p) && i + j + q < 16) cx(k[i + j], k[i + j + q]);
}

// (BLOCK, NP): 1024 threads x 32 step pairs for leaves of 8193..65536, 256 x
// 16 / 256 x 8 for leaves of <= 8192 / 4096 (several CTAs per SM).  The
// gather stages `chunk` elements per pass; when one chunk holds the whole
// leaf every source is read before any output is written, so in == out is
// allowed (the pure Fisher-Yates jobs run in place).
template <typename V, int BLOCK, int NP, bool POL = true>
__global__ void __launch_bounds__(BLOCK, BLOCK == 256 ? 4 : 1)
    leaf_apply_v3_kernel(ArrayJob J, ExplicitTask E, uint64_t nleaves, const V* __restrict__ in, V* __restrict__ out,
                         const uint16_t* __restrict__ draws, uint16_t* scratch, uint32_t mmax,
                         const uint64_t* __restrict__ list) {
  constexpr uint32_t GPT = NP / 8 > 0 ? NP / 8 : 1;  // groups of 16 targets per thread (phase 2)
  extern __shared__ __align__(16) uint32_t sh[];
  __shared__ uint32_t wsum[BLOCK / 32];
  __shared__ uint32_t s_nlong, s_nhuge, s_bad;
  __shared__ __align__(8) uint64_t s_bar;
  uint32_t s_phase = 0;
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  const uint32_t nwmax = ((mmax + 15) >> 4) << 2;  // counter words, whole groups of 16 targets
  uint32_t* cnt = sh;
  uint16_t* gst = reinterpret_cast<uint16_t*>(sh + nwmax);
  const uint32_t bkt_w = nwmax + (((nwmax >> 2) + 7) >> 3 << 2);
  uint16_t* bkt = reinterpret_cast<uint16_t*>(sh + bkt_w);
  // the gather stages the leaf's data through the whole allocation in chunks
  // (leaves of <= 8192: the allocation holds the whole leaf, see leaf_apply_v3_smem)
  uint32_t chunk = ((bkt_w * 4 + ((mmax + 7) & ~7u) * 2) / (uint32_t)sizeof(V)) & ~3u;
  if (NP <= 16) chunk = max(chunk, (mmax + 3) & ~3u);
  V* sdata = reinterpret_cast<V*>(sh);
  const uint32_t mr = (mmax + 15) & ~15u;
  // the CTA's scratch (H, queue, spill) and the timing knob: loaded from shared
  // memory where used, so the compiler neither keeps them in registers nor
  // rematerialises the address arithmetic (64-register cap)
  __shared__ uint16_t* s_hg;
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    s_hg = reinterpret_cast<uint16_t*>(
        ((uintptr_t)(scratch + (uint64_t)blockIdx.x * leaf_scratch_stride(mmax)) + 15) & ~(uintptr_t)15);
    s_stop = g_leaf_stop;
  }
  __syncthreads();
// L2 policies: scratch and half-written output lines stay (evict_last), the
// leaf's input and its final output lines stream (evict_first); created at the
// use (uniform registers)
#define POL_LAST (POL ? l2_policy_last() : l2_policy_normal())
#define POL_FIRST (POL ? l2_policy_first() : l2_policy_normal())
#define Hg (s_hg)
#define lst (s_hg + mr)
#define tmp (s_hg + 2 * mr)
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  for (uint64_t g = blockIdx.x; g < nleaves; g += gridDim.x) {
    LeafDesc L;
    if (list) {
      L.lo = list[2 * g];
      L.hi = list[2 * g + 1];
    } else {
      L = leaf_desc(J, E, g);
    }
    const uint32_t m = (uint32_t)(L.hi - L.lo);
    const V* src_in = in + L.lo;
    V* dst = out + L.lo;
    if (m < 2) {
      if (m == 1 && tid == 0) dst[0] = src_in[0];
      continue;
    }
    const uint16_t* __restrict__ dr = draws + L.lo;
    if (tid == 0 && g + gridDim.x < nleaves) {  // the next leaf's draws into L2
      uint64_t nlo, nhi;
      if (list) {
        nlo = list[2 * (g + gridDim.x)];
        nhi = list[2 * (g + gridDim.x) + 1];
      } else {
        const LeafDesc Ln = leaf_desc(J, E, g + gridDim.x);
        nlo = Ln.lo;
        nhi = Ln.hi;
      }
      l2_prefetch(draws + nlo, (size_t)(nhi - nlo) * 2);
    }
    const uint32_t nw = ((m + 15) >> 4) << 2;  // this leaf's counter words
    for (uint32_t w = tid; w < (nw >> 2); w += BLOCK) reinterpret_cast<uint4*>(cnt)[w] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
      s_nlong = 0;
      s_nhuge = 0;
      s_bad = g_leaf_force_fallback;
    }
    // r[i]: steps 2P and 2P+1 of pair P = tid + 1024 i (low / high half-word)
    uint32_t r[NP];
    const bool dal = (((uintptr_t)dr) & 3) == 0;
#pragma unroll
    for (int i = 0; i < (int)NP; ++i) {
      const uint32_t s0 = 2 * (tid + BLOCK * i);
      if (dal && s0 + 2 <= m) {
        r[i] = *reinterpret_cast<const uint32_t*>(dr + s0);
      } else {
        const uint32_t lo16 = s0 < m ? (uint32_t)dr[s0] : 0u;
        const uint32_t hi16 = s0 + 1 < m ? (uint32_t)dr[s0 + 1] : 0u;
        r[i] = lo16 | (hi16 << 16);
      }
    }
    __syncthreads();
    // 1. histogram (byte counters)
#pragma unroll
    for (int i = 0; i < (int)NP; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t s = 2 * (tid + BLOCK * i) + h;
        const uint32_t j = (r[i] >> (16 * h)) & 0xFFFFu;
        if (s - 1u < m - 1u) atomicAdd(&cnt[j >> 2], 1u << ((j & 3) << 3));
      }
    __syncthreads();
    if (s_stop <= 1) continue;
    // 2. group totals and in-group prefixes; thread t: groups GPT*t .. GPT*t+GPT-1
    {
      const uint32_t ng = nw >> 2;
      uint32_t tot[GPT], tsum = 0;
      bool bad = false;
#pragma unroll
      for (int q = 0; q < (int)GPT; ++q) {
        const uint32_t G = GPT * tid + q;
        tot[q] = 0;
        if (G < ng) {
          uint4 c4 = reinterpret_cast<uint4*>(cnt)[G];
          const uint32_t s0 = __dp4a(c4.x, 0x01010101u, 0u), s1 = __dp4a(c4.y, 0x01010101u, 0u);
          const uint32_t s2 = __dp4a(c4.z, 0x01010101u, 0u), s3 = __dp4a(c4.w, 0x01010101u, 0u);
          const uint32_t b1 = s0, b2 = s0 + s1, b3 = b2 + s2, T = b3 + s3;
          c4.x = c4.x * 0x01010100u;
          c4.y = c4.y * 0x01010100u + b1 * 0x01010101u;
          c4.z = c4.z * 0x01010100u + b2 * 0x01010101u;
          c4.w = c4.w * 0x01010100u + b3 * 0x01010101u;
          reinterpret_cast<uint4*>(cnt)[G] = c4;
          tot[q] = T;
          bad |= T > 255u;
          tsum += T;
        }
      }
      uint32_t x = tsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (lane == 31) wsum[wid] = x;
      if (bad) s_bad = 1;
      __syncthreads();
      if (wid == 0) {
        const uint32_t v = lane < BLOCK / 32 ? wsum[lane] : 0u;
        uint32_t z = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
          if (lane >= (uint32_t)o) z += y;
        }
        if (lane < BLOCK / 32) wsum[lane] = z - v;
        if (lane == 31 && z != m - 1) s_bad = 1;  // a byte counter wrapped
      }
      __syncthreads();
      uint32_t base = wsum[wid] + x - tsum;
#pragma unroll
      for (int q = 0; q < (int)GPT; ++q) {
        const uint32_t G = GPT * tid + q;
        if (G < ng) gst[G] = (uint16_t)base;
        base += tot[q];
      }
    }
    __syncthreads();
    if (s_bad) {
      // serial fallback (counter overflow: not expected to ever happen)
      for (uint32_t i = tid; i < m; i += BLOCK) dst[i] = src_in[i];
      __syncthreads();
      if (tid == 0)
        for (uint32_t i = m - 1; i >= 1; --i) {
          const uint32_t j = dr[i];
          const V t = dst[i];
          dst[i] = dst[j];
          dst[j] = t;
        }
      __syncthreads();
      continue;
    }
    if (s_stop <= 2) continue;
    // 3. scatter step ids into their buckets; the byte atomic gives the slot
#pragma unroll
    for (int i = 0; i < (int)NP; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t s = 2 * (tid + BLOCK * i) + h;
        const uint32_t j = (r[i] >> (16 * h)) & 0xFFFFu;
        if (s - 1u < m - 1u) {
          const uint32_t sh8 = (j & 3) << 3;
          const uint32_t old = atomicAdd(&cnt[j >> 2], 1u << sh8);
          const uint32_t slot = (uint32_t)gst[j >> 4] + ((old >> sh8) & 0xFFu);
          bkt[slot] = (uint16_t)s;
          r[i] = (r[i] & ~(0xFFFFu << (16 * h))) | (slot << (16 * h));
        }
      }
    __syncthreads();
    if (s_stop <= 3) continue;
    if (tid == 0) l2_prefetch(src_in, (size_t)m * sizeof(V));  // staged in phase 8
    // 4. targets, four per counter word (the counters now hold in-group bucket ends)
    for (uint32_t w = tid; w < nw; w += BLOCK) {
      const uint32_t e4 = cnt[w];
      const uint32_t pe = (w & 3) ? (cnt[w - 1] >> 24) : 0u;
      const uint32_t base = gst[w >> 2];
      uint32_t Hq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t p = 4 * w + q;
        const uint32_t en = (e4 >> (8 * q)) & 0xFFu;
        const uint32_t sn = q ? ((e4 >> (8 * (q - 1))) & 0xFFu) : pe;
        const uint32_t k = p < m ? en - sn : 0u;
        const uint32_t st = base + sn;
        const uint32_t v0 = k >= 1 ? (uint32_t)bkt[st] : 0u;
        const uint32_t v1 = k >= 2 ? (uint32_t)bkt[st + 1] : 0u;
        uint32_t H = 0;
        if (k >= 9) {  // queued from the top of the list area
          st_pol(lst + (mr - 1 - atomicAdd(&s_nhuge, 1u)), (uint16_t)p, POL_LAST);
        } else if (k >= 3) {
          st_pol(lst + atomicAdd(&s_nlong, 1u), (uint16_t)p, POL_LAST);
        } else if (k == 1) {
          bkt[st] = (uint16_t)p;
          H = v0 > p ? v0 : 0u;
        } else if (k == 2) {
          bkt[st] = (uint16_t)(v0 < v1 ? v1 : p);
          bkt[st + 1] = (uint16_t)(v1 < v0 ? v0 : p);
          const uint32_t lo = min(v0, v1), hi = max(v0, v1);
          H = lo > p ? lo : hi;
        }
        Hq[q] = H;
      }
      st_pol2(reinterpret_cast<uint32_t*>(Hg + 4 * w), Hq[0] | (Hq[1] << 16), Hq[2] | (Hq[3] << 16), POL_LAST);
    }
    __syncthreads();
    if (s_stop <= 4) continue;
    // 5. queued buckets of 3..8 steps, one per thread: keys (step << 16 | slot)
    //    through a sorting network; the entry at sorted position a gets the
    //    step at a + 1 (or the target itself at the end)
    for (uint32_t i = tid; i < s_nlong; i += BLOCK) {
      const uint32_t p = ld_pol(lst + i, POL_LAST);
      const uint32_t w = p >> 2, q = p & 3;
      const uint32_t cw = cnt[w];
      const uint32_t en = (cw >> (8 * q)) & 0xFFu;
      const uint32_t sn = q ? ((cw >> (8 * (q - 1))) & 0xFFu) : ((w & 3) ? (cnt[w - 1] >> 24) : 0u);
      const uint32_t k = en - sn, st = (uint32_t)gst[w >> 2] + sn;
      uint32_t key[8];
#pragma unroll
      for (int a = 0; a < 8; ++a)
        key[a] = (uint32_t)a < k ? (((uint32_t)bkt[st + a] << 16) | (st + a)) : 0xFFFFFFFFu;
      sort_net8(key);
#pragma unroll
      for (int a = 0; a < 8; ++a)
        if ((uint32_t)a < k)
          bkt[key[a] & 0xFFFFu] = (uint16_t)((uint32_t)(a + 1) < k ? (key[a < 7 ? a + 1 : 7] >> 16) : p);
      st_pol(Hg + p, (uint16_t)((key[0] >> 16) > p ? (key[0] >> 16) : (key[1] >> 16)), POL_LAST);
    }
    //    buckets of >= 9 steps (the first few hundred targets), one per warp:
    //    a warp bitonic sort of the keys (<= 32 entries)
    for (uint32_t i = wid; i < s_nhuge; i += BLOCK / 32) {
      const uint32_t p = ld_pol(lst + (mr - 1 - i), POL_LAST);
      const uint32_t w = p >> 2, q = p & 3;
      const uint32_t cw = cnt[w];
      const uint32_t en = (cw >> (8 * q)) & 0xFFu;
      const uint32_t sn = q ? ((cw >> (8 * (q - 1))) & 0xFFu) : ((w & 3) ? (cnt[w - 1] >> 24) : 0u);
      const uint32_t k = en - sn, st = (uint32_t)gst[w >> 2] + sn;
      if (k <= 32 && s_stop != 12) {  // (12: timing/test knob, all through the O(k^2) path)
        uint32_t key = lane < k ? (((uint32_t)bkt[st + lane] << 16) | (st + lane)) : 0xFFFFFFFFu;
#pragma unroll
        for (uint32_t kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
          for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, key, jj);
            const bool up = (lane & kk) == 0, low = (lane & jj) == 0;
            key = (low == up) ? min(key, o) : max(key, o);
          }
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, key, 1);
        const uint32_t k1 = __shfl_sync(0xffffffffu, key, 1);
        if (lane < k) bkt[key & 0xFFFFu] = (uint16_t)(lane + 1 < k ? (nxt >> 16) : p);
        if (lane == 0) st_pol(Hg + p, (uint16_t)((key >> 16) > p ? (key >> 16) : (k1 >> 16)), POL_LAST);
      } else if (lane == 0) {  // > 32 steps on one target: O(k^2) through the scratch
        uint32_t H = 0x10000u;
        for (uint32_t a = 0; a < k; ++a) {
          const uint32_t va = bkt[st + a];
          uint32_t best = 0x10000u;
          for (uint32_t b = 0; b < k; ++b) {
            const uint32_t vb = bkt[st + b];
            best = (vb > va && vb < best) ? vb : best;
          }
          tmp[st + a] = (uint16_t)(best < 0x10000u ? best : p);
          H = (va > p && va < H) ? va : H;
        }
        for (uint32_t a = 0; a < k; ++a) bkt[st + a] = tmp[st + a];
        Hg[p] = (uint16_t)(H & 0xFFFFu);
      }
      __syncwarp();
    }
    __syncthreads();
    if (s_stop <= 5) continue;
    // 6. every owned step picks up N(s) (> s) or its target j_s (<= s)
#pragma unroll
    for (int i = 0; i < (int)NP; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t s = 2 * (tid + BLOCK * i) + h;
        if (s - 1u < m - 1u) {
          const uint32_t slot = (r[i] >> (16 * h)) & 0xFFFFu;
          r[i] = (r[i] & ~(0xFFFFu << (16 * h))) | ((uint32_t)bkt[slot] << (16 * h));
        }
      }
    __syncthreads();
    // 7. H into shared memory (over the buckets); every output's source:
    //    W(N(s)) (follow H to its root) or j_s; W(0) for output 0
    for (uint32_t w = tid; w < ((m + 7) >> 3); w += BLOCK)
      reinterpret_cast<uint4*>(bkt)[w] = ld_pol4(Hg + 8 * w, POL_LAST);
    __syncthreads();
    if (s_stop <= 6) continue;
    {
      const uint16_t* Hs = bkt;
#pragma unroll
      for (int i = 0; i < (int)NP; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t s = 2 * (tid + BLOCK * i) + h;
          const uint32_t x = (r[i] >> (16 * h)) & 0xFFFFu;
          if (s < m && (s == 0 || x > s)) {
            uint32_t y = s == 0 ? 0u : x, hh;
            while ((hh = Hs[y]) != 0) y = hh;
            r[i] = (r[i] & ~(0xFFFFu << (16 * h))) | (y << (16 * h));
          }
          if (s >= m) r[i] |= 0xFFFFu << (16 * h);  // no output: a source no chunk holds
        }
    }
    __syncthreads();
    if (s_stop == 7) continue;
    // 8. gather through shared memory: the leaf's data in chunks over the whole
    //    allocation (H is dead); each output is stored in the pass holding its source
    const bool sal = (((uintptr_t)src_in) & 15) == 0;
    for (uint32_t c0 = 0; c0 < m; c0 += chunk) {
      const uint32_t cn = min(chunk, m - c0);
      if (sal && (cn * (uint32_t)sizeof(V)) % 16 == 0) {
        // one TMA bulk copy (the chunk is 16-byte aligned and sized)
        if (tid == 0) {
          fence_proxy_async_smem();  // earlier generic accesses of this smem first
          if (s_stop != 11) {
            mbar_arrive_expect_tx(&s_bar, cn * (uint32_t)sizeof(V));
            for (uint32_t o = 0; o < cn * (uint32_t)sizeof(V); o += 65536u)
              bulk_g2s_pol(reinterpret_cast<char*>(sdata) + o, reinterpret_cast<const char*>(src_in + c0) + o,
                           min(65536u, cn * (uint32_t)sizeof(V) - o), &s_bar, POL_FIRST);
          } else {
            mbar_arrive_expect_tx(&s_bar, 0u);  // timing: no staging
          }
        }
        mbar_wait(&s_bar, s_phase);
        s_phase ^= 1u;
      } else {
        for (uint32_t w = tid; w < cn; w += BLOCK) sdata[w] = src_in[c0 + w];
      }
      __syncthreads();
      // (a per-pass copy of the output pointer keeps the 64 store addresses
      // from being hoisted out of the chunk loop into registers)
      V* dpass;
      asm volatile("mov.b64 %0, %1;" : "=l"(dpass) : "l"(dst + 2 * tid));
      const bool pair8 = ((((uintptr_t)dst) & (2 * sizeof(V) - 1)) == 0) && s_stop < 8;
      // lines completed by a later pass stay in L2 until then
      const bool olast = c0 + cn < m;
      // ... and the per-output source extraction from being hoisted likewise
#pragma unroll
      for (int i = 0; i < (int)NP; ++i) asm volatile("" : "+r"(r[i]));
      // a step pair whose two sources are in this chunk goes out as one
      // 2-element store, otherwise the one present element singly (one copy of
      // the loop per policy: the policy stays a uniform constant)
#define SK_GATHER_PAIRS(PLC)                                                      \
  _Pragma("unroll") for (int i = 0; i < (int)NP; ++i) {                           \
    const uint32_t s0 = (r[i] & 0xFFFFu) - c0, s1 = (r[i] >> 16) - c0;            \
    const bool i0 = s0 < cn, i1 = s1 < cn;                                        \
    if (i0 && i1) {                                                               \
      st_pol2(dpass + 2 * BLOCK * i, sdata[s0], sdata[s1], PLC);                  \
    } else if (i0 || i1) {                                                        \
      st_pol(dpass + 2 * BLOCK * i + (i1 ? 1 : 0), sdata[i1 ? s1 : s0], PLC);     \
    }                                                                             \
  }
      if (pair8 && olast) {
        SK_GATHER_PAIRS(POL_LAST)
      } else if (pair8) {
        SK_GATHER_PAIRS(POL_FIRST)
      } else {
#pragma unroll
      for (int i = 0; i < (int)NP; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t src = ((r[i] >> (16 * h)) & 0xFFFFu) - c0;
          if (src < cn && s_stop != 10) dpass[2 * BLOCK * i + h] = s_stop == 8 ? (V)src : sdata[src];
        }
      }
      __syncthreads();
    }
  }
}
#undef SK_GATHER_PAIRS
#undef POL_LAST
#undef POL_FIRST
#undef Hg
#undef lst
#undef tmp

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
void debug_set_leaf_fallback(int v) { cudaMemcpyToSymbol(g_leaf_force_fallback, &v, sizeof(int)); }
void debug_set_leaf_l2pol(int v) { g_leaf_l2pol_host = v; }
void debug_set_leaf_stop(int v) { cudaMemcpyToSymbol(g_leaf_stop, &v, sizeof(int)); }
void debug_set_spec_decode_max(int v) { g_spec_decode_max = v < 0 ? 0 : (uint64_t)v; }

void launch_leaf_decode16(const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, uint16_t* draws,
                          unsigned long long* bits, cudaStream_t st) {
  if (!nleaves) return;
  const unsigned blocks = (unsigned)((nleaves + kDecodeBlock - 1) / kDecodeBlock);
  const bool fresh = !(E.active && E.sd.plen != 0);
  if (nleaves <= g_spec_decode_max) {
    const unsigned wb = (unsigned)((nleaves + kSpecWarps - 1) / kSpecWarps);
    if (fresh) leaf_decode_spec_kernel<true><<<wb, 32 * kSpecWarps, 0, st>>>(J, E, nleaves, draws, bits);
    else leaf_decode_spec_kernel<false><<<wb, 32 * kSpecWarps, 0, st>>>(J, E, nleaves, draws, bits);
    count_launch();
    return;
  }
  // T = 64 needs one 128 KB block per SM; with more blocks than SMs the
  // 64 KB T = 32 blocks run two or three per SM
  if (blocks <= (unsigned)num_sms()) launch_ws<64>(fresh, blocks, J, E, nleaves, draws, bits, st);
  else launch_ws<32>(fresh, blocks, J, E, nleaves, draws, bits, st);
  count_launch();
}

static size_t leaf_apply_smem(uint32_t mmax, int eb = 0) {
  const uint32_t half = mmax < kLeafHalf ? mmax : kLeafHalf;
  const size_t words = (size_t)((half + 1) / 2) + (size_t)((mmax + 1) / 2);
  if (mmax <= 8192) return ((words + 1) & ~(size_t)1) * 4 + (size_t)mmax * (eb ? eb : 8);  // + staged data
  return words * 4;
}

// v3: byte counters (whole groups of 16 targets), 16-bit group starts,
// buckets; leaves of <= 8192 also room to stage the whole leaf (one chunk)
static size_t leaf_apply_v3_smem(uint32_t mmax, int eb) {
  const size_t nw = ((size_t)(mmax + 15) >> 4) << 2;
  const size_t s = (nw + ((((nw >> 2) + 7) >> 3) << 2)) * 4 + (size_t)((mmax + 7) & ~7u) * 2;
  if (mmax > 8192) return s;
  return std::max(s, (size_t)((mmax + 3) & ~3u) * (size_t)eb);
}

template <typename V>
static void leaf_apply_t(const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, const void* in, void* out,
                         const uint16_t* draws, uint16_t* scratch, uint32_t mmax, uint32_t grid,
                         const uint64_t* list, cudaStream_t st) {
  size_t smem = leaf_apply_smem(mmax, (int)sizeof(V));
  if (mmax > 2048 && (mmax <= 8192 || in != out)) {
    // v3 (leaves > 8192 gather in two or more chunks: distinct buffers only)
    smem = leaf_apply_v3_smem(mmax, (int)sizeof(V));
    if (mmax <= 4096) {
      auto k = leaf_apply_v3_kernel<V, 256, 8>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<<<grid, 256, smem, st>>>(J, E, nleaves, (const V*)in, (V*)out, draws, scratch, mmax, list);
    } else if (mmax <= 8192) {
      auto k = leaf_apply_v3_kernel<V, 256, 16>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<<<grid, 256, smem, st>>>(J, E, nleaves, (const V*)in, (V*)out, draws, scratch, mmax, list);
    } else {
      auto k = g_leaf_l2pol_host ? leaf_apply_v3_kernel<V, 1024, 32, true> : leaf_apply_v3_kernel<V, 1024, 32, false>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<<<grid, 1024, smem, st>>>(J, E, nleaves, (const V*)in, (V*)out, draws, scratch, mmax, list);
    }
  } else if (mmax > 8192) {
    throw std::runtime_error("leaf apply: leaves above 8192 elements need distinct in/out buffers");
  } else {
    auto k = leaf_apply_kernel<V, 256>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, st>>>(J, E, nleaves, (const V*)in, (V*)out, draws, scratch, mmax, list);
  }
  count_launch();
}

uint32_t leaf_apply_grid(uint64_t nleaves, uint32_t mmax, int num_sms, int eb) {
  // Persistent CTAs: as many as fit (the per-CTA scratch is reused per leaf and
  // stays L2-resident).
  size_t smem = leaf_apply_smem(mmax);
  size_t fit = (size_t)(220 * 1024) / (smem + 2048);
  int per_sm = (int)std::max((size_t)1, std::min(fit, (size_t)(mmax > 8192 ? 2 : 8)));
  if (mmax > 8192) per_sm = 1;  // v3: 1024 threads, ~200 KB
  if (mmax > 2048 && mmax <= 8192)  // v3, 256 threads
    per_sm = (int)std::max((size_t)1, std::min((size_t)4, (size_t)(220 * 1024) / (leaf_apply_v3_smem(mmax, eb) + 2048)));
  uint64_t g = (uint64_t)num_sms * per_sm;
  if (g > nleaves) g = nleaves;
  return (uint32_t)(g ? g : 1);
}

void launch_leaf_apply(int eb, const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, const void* in, void* out,
                       const uint16_t* draws, uint16_t* scratch, uint32_t mmax, uint32_t grid, cudaStream_t st,
                       const uint64_t* list) {
  if (!nleaves) return;
  if (eb == 4) leaf_apply_t<uint32_t>(J, E, nleaves, in, out, draws, scratch, mmax, grid, list, st);
  else leaf_apply_t<unsigned long long>(J, E, nleaves, in, out, draws, scratch, mmax, grid, list, st);
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
