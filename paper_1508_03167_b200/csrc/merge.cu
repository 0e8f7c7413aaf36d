// merge.cu -- one merge round of the parallel schedule (reference: _kernels.py:96-121
// _merge, shufflers.py:158-191 merge, rounds shufflers.py:117-130 / 291-297).
//
// Phase 1 (the coin-flip swap merge): the A queue of the in-place merge is the
// stream F with F[u] = A[u] (u < n1) and F[n1 + k] = F[select1(k)].  Segments
// S_0 = [0, n1), S_{h+1} = [n1 + rank'(S_h.start), n1 + rank'(S_h.end))
// (rank' = ones before min(p, t)) partition [0, X); [X, N) is the identity (A
// queue empty).  A tile [a_0, b_0) of S_0 is followed through its windows
// [a_{h+1}, b_{h+1}) = [n1 + rank'(a_h), n1 + rank'(b_h)): the windows of all
// tiles partition [0, X), and a tile's swaps only touch its own windows, so
// one CTA per tile loads them (TMA), swaps them in shared memory window by
// window and stores them back -- one read and one write per element per
// round, in place (merge_tree_kernel).
// (Derivation + CPU check: tests/decomp_model.py merge_phase1_model.)
//
// Phase 2 (tail insertion, x = t..N-1: swap(x, FDR(x+1))) is precomputed as a
// (dst, src) list over the touched set (tests/decomp_model.py tail_plan_model)
// and applied as a gather then a scatter.
//
// Everything except the element movement depends only on (schedule, seed), so
// the rank tables, stop points, window chains, tail draws and tail plans are
// built on a side stream while the leaf stage runs.
#include <algorithm>
#include <stdexcept>
#include "sk_kernels.h"

namespace sk {

// ------------------------------------------------------------- rank tables
__global__ void rank_count_kernel(LevelJob LJ, uint64_t sbs, uint64_t* __restrict__ rank) {
  uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t per = sbs - 1;
  if (idx >= LJ.npairs * per) return;
  uint64_t g = idx / per, k = idx - g * per;
  uint64_t s, n1, n2, arr;
  StreamDesc sd;
  pair_geom(LJ, g, s, n1, n2, sd, arr);
  uint64_t N = n1 + n2;
  uint64_t* R = rank + g * sbs;
  if (k == 0) R[0] = 0;
  uint64_t cnt = 0;
  if (n1 && n2 && (k << 9) < N + 1) {
#pragma unroll
    for (int w = 0; w < 8; ++w) cnt += __popcll(chunk(sd, (k << 3) + w));
  }
  R[k + 1] = cnt;
}

// In-place inclusive scan of every pair's table, chunked so that the few
// huge tables of the top rounds are scanned by many CTAs: (A) chunk sums,
// (B) per-pair exclusive scan of the chunk sums, (C) chunk-local scan + offset.
constexpr uint32_t kScanChunk = 4096;  // entries per CTA (256 threads x 16)

__global__ void __launch_bounds__(256) scan_chunk_sums(const uint64_t* __restrict__ rank, uint64_t sbs, uint32_t cpp,
                                                       uint64_t* __restrict__ csum) {
  __shared__ uint64_t red[8];
  const uint64_t g = blockIdx.x / cpp, ci = blockIdx.x - g * cpp;
  const uint64_t* R = rank + g * sbs;
  const uint64_t b0 = ci * kScanChunk, b1 = min(sbs, b0 + kScanChunk);
  uint64_t v = 0;
  for (uint64_t i = b0 + threadIdx.x; i < b1; i += 256) v += R[i];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    csum[blockIdx.x] = t;
  }
}

__global__ void scan_chunk_offsets(uint64_t* __restrict__ csum, uint32_t cpp) {
  uint64_t* c = csum + (uint64_t)blockIdx.x * cpp;
  const uint32_t lane = threadIdx.x;
  uint64_t carry = 0;
  for (uint32_t base = 0; base < cpp; base += 32) {
    const uint32_t i = base + lane;
    const uint64_t v = (i < cpp) ? c[i] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (i < cpp) c[i] = carry + x - v;  // exclusive
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

__global__ void __launch_bounds__(256) scan_chunk_apply(uint64_t* __restrict__ rank, uint64_t sbs, uint32_t cpp,
                                                        const uint64_t* __restrict__ coff) {
  __shared__ uint64_t wsum[8];
  const uint64_t g = blockIdx.x / cpp, ci = blockIdx.x - g * cpp;
  uint64_t* R = rank + g * sbs;
  const uint64_t b0 = ci * kScanChunk, b1 = min(sbs, b0 + kScanChunk);
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t i0 = b0 + (uint64_t)tid * 16;  // 16 consecutive entries per thread
  uint64_t v[16], sum = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    v[k] = (i0 + k < b1) ? R[i0 + k] : 0;
    sum += v[k];
  }
  uint64_t x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint64_t run = coff[blockIdx.x] + x - sum;
#pragma unroll
  for (int w = 0; w < 8; ++w) run += (w < (int)wid) ? wsum[w] : 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    run += v[k];
    if (i0 + k < b1) R[i0 + k] = run;  // inclusive
  }
}

uint64_t rank_scan_scratch(uint64_t npairs, uint64_t sbs) {
  return npairs * ((sbs + kScanChunk - 1) / kScanChunk);
}

void launch_rank_tables(const LevelJob& LJ, uint64_t sbs, uint64_t* rank, uint64_t* csum, cudaStream_t st) {
  uint64_t total = LJ.npairs * (sbs - 1);
  if (!total) return;
  rank_count_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(LJ, sbs, rank);
  const uint32_t cpp = (uint32_t)((sbs + kScanChunk - 1) / kScanChunk);
  const unsigned nblk = (unsigned)(LJ.npairs * cpp);
  scan_chunk_sums<<<nblk, 256, 0, st>>>(rank, sbs, cpp, csum);
  scan_chunk_offsets<<<(unsigned)LJ.npairs, 32, 0, st>>>(csum, cpp);
  scan_chunk_apply<<<nblk, 256, 0, st>>>(rank, sbs, cpp, csum);
  for (int i = 0; i < 4; ++i) count_launch();
}

// ------------------------------------------------------------ pair plans
// position (from the MSB) of the r-th (0-based) set bit of x; it must exist
__device__ __forceinline__ uint32_t select_msb(uint64_t x, uint32_t r) {
  uint32_t pos = 0, c;
  c = __popcll(x >> 32);            if (r >= c) { r -= c; pos += 32; x <<= 32; }
  c = __popc((uint32_t)(x >> 48));  if (r >= c) { r -= c; pos += 16; x <<= 16; }
  c = __popc((uint32_t)(x >> 56));  if (r >= c) { r -= c; pos += 8;  x <<= 8; }
  c = __popc((uint32_t)(x >> 60));  if (r >= c) { r -= c; pos += 4;  x <<= 4; }
  c = __popc((uint32_t)(x >> 62));  if (r >= c) { r -= c; pos += 2;  x <<= 2; }
  c = (uint32_t)(x >> 63);          if (r >= c) { pos += 1; }
  return pos;
}

// Position of the r-th (0-based) bit equal to `one` in [0, 512*used), or kNone.
__device__ uint64_t select_bit(const StreamDesc& sd, const uint64_t* R, uint64_t used, uint64_t r, bool one) {
  auto before = [&](uint64_t k) -> uint64_t { return one ? R[k] : (k * 512 - R[k]); };
  if (before(used) <= r) return kNone;
  uint64_t lo = 0, hi = used;
  while (hi - lo > 1) {
    uint64_t mid = (lo + hi) >> 1;
    if (before(mid) <= r) lo = mid; else hi = mid;
  }
  uint64_t rem = r - before(lo);
  for (uint64_t w = lo << 3;; ++w) {
    uint64_t x = chunk(sd, w);
    if (!one) x = ~x;
    uint32_t c = __popcll(x);
    if (rem < c) return (w << 6) + select_msb(x, (uint32_t)rem);
    rem -= c;
  }
}

// Stop point (_kernels.py:104-115): t = min(select0(n1), select1(n2)); A is
// exhausted iff the zero comes first.  X = first fixed point of S -> n1 + rank'(S).
__global__ void pair_plan_kernel(LevelJob LJ, uint64_t sbs, const uint64_t* __restrict__ rank,
                                 PairPlan* __restrict__ plans) {
  uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= LJ.npairs) return;
  PairPlan P;
  pair_geom(LJ, g, P.s, P.n1, P.n2, P.sd, P.array);
  P.rank_off = g * sbs;
  P.tail_off = 0;
  P.tail_slow = 0;
  const uint64_t n1 = P.n1, n2 = P.n2, N = n1 + n2;
  if (n1 == 0 || n2 == 0) {  // shufflers.py:169-170: no bits, no change
    P.t = 0; P.X = n1; P.aex = 0; P.degenerate = 1; P.tail_len = 0; P.bits = 0;
    P.nseg = n1 ? 1 : 0;
  } else {
    const uint64_t* R = rank + g * sbs;
    uint64_t used = (N + 1 + 511) >> 9;
    uint64_t z = select_bit(P.sd, R, used, n1, false);
    uint64_t o = select_bit(P.sd, R, used, n2, true);
    uint64_t t = z < o ? z : o;
    P.t = t; P.aex = z < o; P.degenerate = 0;
    // segment chain S_0 = 0, S_{h+1} = n1 + rank'(S_h) up to the fixed point X
    uint64_t S = 0;
    uint32_t h = 0;
    for (;;) {
      uint64_t S2 = n1 + (S ? rank_bits(P.sd, R, S < t ? S : t) : 0);
      if (S2 == S) break;
      ++h;
      S = S2;
    }
    P.nseg = h;
    P.X = S;
    P.tail_len = N - t;
    P.bits = t + 1;
  }
  plans[g] = P;
}

void launch_pair_plan(const LevelJob& LJ, uint64_t sbs, const uint64_t* rank, PairPlan* plans, cudaStream_t st) {
  if (!LJ.npairs) return;
  pair_plan_kernel<<<(unsigned)((LJ.npairs + 127) / 128), 128, 0, st>>>(LJ, sbs, rank, plans);
  count_launch();
}

// ------------------------------------------------------------ tail decode
// One WARP per pair, all rounds in one launch.  Bits continue at offset t+1
// (shufflers.py:188-191): for x = t..N-1, m_x = FDR(x+1).  The draws are
// decoded speculatively 32 at a time: lane l assumes every earlier draw of the
// batch accepted its first FDR iteration (k0 = ceil(log2 bound) bits), so its
// offset is a warp prefix sum of k0; the first lane whose own first iteration
// rejects finishes its draw with the full (serial) FDR and the next batch
// starts after it.  Tail bounds are ~ the pair size, so for power-of-two pairs
// a rejection is rare and 32 draws are decoded per step; the result is
// bit-identical to the serial loop either way.
__global__ void __launch_bounds__(128) tail_decode_kernel(const LevelTail* __restrict__ levels, int nlevels,
                                                          const uint64_t* __restrict__ prefix, uint64_t total,
                                                          unsigned long long* __restrict__ bits) {
  const uint64_t gg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (gg >= total) return;
  int L = 0;
  while (L + 1 < nlevels && prefix[L + 1] <= gg) ++L;
  const uint64_t g = gg - prefix[L];
  const LevelTail lv = levels[L];
  PairPlan* Pp = lv.plans + g;
  if (Pp->degenerate) return;
  const uint64_t t = Pp->t, N = Pp->n1 + Pp->n2, s = Pp->s, off = Pp->tail_off;
  const bool store = !Pp->tail_slow;  // slow pairs: bits only (their tail runs serially)
  const StreamDesc sd = Pp->sd;
  uint64_t o = t + 1;  // bit offset of the next draw
  uint64_t x = t;      // next insertion step
  while (x < N) {
    const uint64_t xl = x + lane;
    const bool valid = xl < N;
    const uint64_t b = xl + 1;
    const uint32_t k0 = valid ? 64u - __clzll(b - 1) : 0u;
    uint32_t ps = k0;  // inclusive warp prefix of k0
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, ps, d);
      if (lane >= (uint32_t)d) ps += y;
    }
    const uint64_t ol = o + (ps - k0);
    uint64_t c = 0;
    bool acc = false;
    if (valid) {
      c = bits64_at(sd, ol) >> (64 - k0);
      acc = c < b;
    }
    const uint32_t fail = __ballot_sync(0xffffffffu, valid && !acc);
    const uint32_t f = fail ? (uint32_t)(__ffs(fail) - 1) : 32u;  // first rejecting lane
    if (store && valid && lane < f) {
      lv.rec_key[off + (xl - t)] = s + c;
      lv.rec_pair[off + (xl - t)] = (uint32_t)g;
    }
    if (f < 32) {
      uint64_t used = 0, m = 0;
      if (lane == f) {  // full fast-dice-roller for this draw (_kernels.py:64-82)
        Reader64 rd;
        rd.init(sd, ol);
        m = fdr64(rd, b, used);
        if (store) {
          lv.rec_key[off + (xl - t)] = s + m;
          lv.rec_pair[off + (xl - t)] = (uint32_t)g;
        }
      }
      used = __shfl_sync(0xffffffffu, used, f);
      const uint64_t of = __shfl_sync(0xffffffffu, ol, f);
      o = of + used;
      x += f + 1;
    } else {
      o += __shfl_sync(0xffffffffu, ps, 31);
      x += 32;
    }
  }
  if (lane == 0) {
    const uint64_t bt = o;  // t+1 phase-1 bits + tail bits
    Pp->bits = bt;
    atomicAdd(&bits[Pp->array], (unsigned long long)bt);
  }
}

void launch_tail_decode(const LevelTail* d_levels, int nlevels, const uint64_t* d_prefix, uint64_t total_pairs,
                        unsigned long long* bits, cudaStream_t st) {
  if (!total_pairs) return;
  tail_decode_kernel<<<(unsigned)((total_pairs * 32 + 127) / 128), 128, 0, st>>>(d_levels, nlevels, d_prefix,
                                                                                  total_pairs, bits);
  count_launch();
}

// ------------------------------------------------------------ merge round
// rank' at an arbitrary position, by the 8 lanes of one warp (one word each).
__device__ __forceinline__ uint64_t warp_rank(const StreamDesc& sd, const uint64_t* R, uint64_t pos, uint32_t lane) {
  const uint64_t sb = pos >> 9, w0 = sb << 3, we = pos >> 6;
  uint32_t c = 0;
  if (lane < 8) {
    const uint64_t w = w0 + lane;
    if (w < we) c = __popcll(chunk(sd, w));
    else if (w == we && (pos & 63)) c = __popcll(chunk(sd, w) >> (64 - (pos & 63)));
  }
  for (int o = 4; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  return R[sb] + __shfl_sync(0xffffffffu, c, 0);
}

// ------------------------------------------------------- merge round (tree)
// One CTA per tile of segment 0 follows the tile through every segment: the
// tile [a_0, b_0) of A positions, then the windows [a_{h+1}, b_{h+1}) =
// [n1 + rank'(a_h), n1 + rank'(b_h)) -- the positions that receive its
// carried A elements, which are also the B slots its ones consume.  The
// windows of all tiles partition [0, X); a CTA reads in[] over its windows
// once, writes out[] over them once, and carries the A elements from one
// window to the next in shared memory: one read and one write per element
// per round (the segment-pass kernel parks them in HBM: 1.5 + 1.5).  The
// window starts a_h are data independent and precomputed per tile
// (tree_chain_kernel, side stream); the CTA works window by window in
// 2048-position chunks while a window has more than 32 positions, then one
// warp finishes the short windows without block barriers.
constexpr int kTreeBlock = 256;
constexpr int kTreeCPW = 8;
constexpr uint32_t kTreeChunk = kTreeBlock * kTreeCPW;
constexpr int kTreeD = 24;  // stored window starts per tile (deeper ones are computed)

uint32_t tree_tiles_per_pair(const LevelJob& LJ, int eb) {
  uint64_t n1max;
  if (LJ.E.active) n1max = LJ.E.n1;
  else n1max = (1ULL << (LJ.r - 1)) * ((LJ.J.len + LJ.J.q - 1) >> LJ.J.c);
  const uint64_t T0 = tree_tile(eb);
  return (uint32_t)std::max<uint64_t>(1, (n1max + T0 - 1) / T0);
}

uint64_t tree_chain_words(uint64_t npairs, uint32_t tpp) { return npairs * (tpp + 1) * kTreeD; }

__global__ void tree_chain_kernel(const PairPlan* __restrict__ plans, uint64_t npairs,
                                  const uint64_t* __restrict__ rank, uint32_t tpp, uint32_t T0,
                                  uint64_t* __restrict__ chains) {
  const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= npairs * (tpp + 1)) return;
  const uint64_t g = idx / (tpp + 1), tau = idx - g * (tpp + 1);
  const PairPlan* Pp = plans + g;
  const uint64_t n1 = Pp->n1, t = Pp->t;
  const StreamDesc sd = Pp->sd;
  const uint64_t* R = rank + Pp->rank_off;
  uint64_t a = min(tau * (uint64_t)T0, n1);
  uint64_t* o = chains + idx * kTreeD;
  for (int h = 0; h < kTreeD; ++h) {
    o[h] = a;
    a = n1 + rank_bits(sd, R, a < t ? a : t);
  }
}

void launch_tree_chains(int eb, const PairPlan* plans, uint64_t npairs, const uint64_t* rank, uint32_t tpp,
                        uint64_t* chains, cudaStream_t st) {
  if (!npairs) return;
  const uint64_t n = npairs * (tpp + 1);
  tree_chain_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(plans, npairs, rank, tpp, tree_tile(eb), chains);
  count_launch();
}

// debug: 1 = every tile takes the direct (window-by-window) path
__device__ int g_tree_force_direct = 0;
void debug_set_tree_force_direct(int v) { cudaMemcpyToSymbol(g_tree_force_direct, &v, sizeof(int)); }

// Element access of one pair for the tree kernels: FlatAcc = the pair in one
// buffer (in/out may differ); PeerAcc = the pair split into up to kMaxParts
// contiguous parts living in different buffers (other GPUs' memory mapped
// into this one: P2P loads/stores over NVLink), always in place.
constexpr int kMaxParts = 8;

template <typename V>
struct FlatAcc {
  const V* in;
  V* out;
  __device__ __forceinline__ V ld(uint64_t p) const { return in[p]; }
  __device__ __forceinline__ void st(uint64_t p, V v) const { out[p] = v; }
  __device__ __forceinline__ const V* src(uint64_t p) const { return in + p; }
  __device__ __forceinline__ V* dst(uint64_t p) const { return out + p; }
  // [x0, x1) as maximal runs inside one buffer: f(run_start, run_end)
  template <class F>
  __device__ __forceinline__ void runs(uint64_t x0, uint64_t x1, F f) const {
    if (x1 > x0) f(x0, x1);
  }
  __device__ __forceinline__ bool same_alignment() const {
    return ((reinterpret_cast<uintptr_t>(out) - reinterpret_cast<uintptr_t>(in)) & 15) == 0;
  }
};

template <typename V>
struct PeerParts {
  V* base[kMaxParts];              // element at pair position start[k]
  uint64_t start[kMaxParts + 1];   // part k = [start[k], start[k+1])
  int n;
  int tma;                         // 1: every part position-aligned mod 16 B and starts multiple of 16 B
};

template <typename V>
struct PeerAcc {
  const PeerParts<V>& P;
  __device__ __forceinline__ int part(uint64_t p) const {
    int k = 0;
    while (k + 1 < P.n && p >= P.start[k + 1]) ++k;
    return k;
  }
  __device__ __forceinline__ V* ptr(uint64_t p) const {
    const int k = part(p);
    return P.base[k] + (p - P.start[k]);
  }
  __device__ __forceinline__ V ld(uint64_t p) const { return *ptr(p); }
  __device__ __forceinline__ void st(uint64_t p, V v) const { *ptr(p) = v; }
  __device__ __forceinline__ const V* src(uint64_t p) const { return ptr(p); }
  __device__ __forceinline__ V* dst(uint64_t p) const { return ptr(p); }
  template <class F>
  __device__ __forceinline__ void runs(uint64_t x0, uint64_t x1, F f) const {
    for (int k = part(x0); k < P.n && x0 < x1; ++k) {
      const uint64_t e = min(x1, P.start[k + 1]);
      if (e > x0) f(x0, e);
      x0 = e;
    }
  }
  __device__ __forceinline__ bool same_alignment() const { return P.tma != 0; }
};

// One chunk of a window: positions [p0, p0 + len), fbase = index of p0 in the
// window (its F slot), bq = position of the chunk's first B element, obase =
// F slot of the chunk's first one in the next window.  Window 0 reads F from
// in[]; deeper windows from shared memory, compacted in place (a barrier
// separates the chunk's loads from its stores).  Returns the chunk's ones.
template <typename V, bool L0, class Acc>
__device__ __forceinline__ uint32_t tree_chunk(const Acc& acc, V* Fs, const StreamDesc& sd, uint64_t t, uint64_t p0,
                                               uint32_t len, uint32_t fbase, uint64_t bq, uint32_t obase,
                                               uint32_t* wsum) {
  constexpr int CPW = kTreeCPW;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t wbase = wid * 32 * CPW;
  uint32_t mword = 0;
  if (lane < (uint32_t)CPW) {
    const uint32_t i = wbase + lane * 32;
    if (i < len) {
      const uint64_t p = p0 + i;
      if (p < t) {
        uint32_t nv = min(32u, len - i);
        const uint64_t nt = t - p;
        if (nt < nv) nv = (uint32_t)nt;
        const uint32_t b = (uint32_t)(bits64_at(sd, p) >> 32);
        mword = (nv == 32) ? b : (b & ~(0xffffffffu >> nv));
      }
    }
  }
  const uint32_t cnt = __popc(mword);
  uint32_t x = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  const uint32_t round_base = x - cnt;
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint32_t before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kTreeBlock / 32; ++w) {
    before += (w < (int)wid) ? wsum[w] : 0u;
    total += wsum[w];
  }
  const uint32_t ltmask = ~(0xffffffffu >> lane);
  V f[CPW], b[CPW];
  uint32_t qo[CPW];
  uint32_t onemask = 0, inmask = 0;
#pragma unroll
  for (int k = 0; k < CPW; ++k) {
    const uint32_t i = wbase + 32 * k + lane;
    const uint32_t m = __shfl_sync(0xffffffffu, mword, k);
    const uint32_t rb = __shfl_sync(0xffffffffu, round_base, k);
    const bool in_t = i < len;
    const bool one = in_t && ((m >> (31 - lane)) & 1u);
    qo[k] = before + rb + __popc(m & ltmask);
    inmask |= (in_t ? 1u : 0u) << k;
    onemask |= (one ? 1u : 0u) << k;
    if (in_t) f[k] = L0 ? acc.ld(p0 + i) : Fs[fbase + i];
    if (one) b[k] = acc.ld(bq + qo[k]);
  }
  __syncthreads();  // loads of F (and of wsum) complete before the in-place stores
#pragma unroll
  for (int k = 0; k < CPW; ++k) {
    const uint64_t p = p0 + wbase + 32 * k + lane;
    if ((onemask >> k) & 1u) {
      acc.st(p, b[k]);
      Fs[obase + qo[k]] = f[k];
    } else if ((inmask >> k) & 1u) {
      acc.st(p, f[k]);
    }
  }
  return total;
}

// Window-by-window fallback (F carried in a T0-element shared buffer): used
// when a tile's windows do not fit the staging buffer or its chain is deeper
// than the stored kTreeD starts.  Never taken for pseudo-random bit streams
// in practice; kept exact for every input.
template <typename V, class Acc>
__device__ void tree_windows_direct(const Acc& acc, V* Fs, const StreamDesc& sd, const uint64_t* R, uint64_t n1,
                                    uint64_t t, const uint64_t* ach, const uint64_t* bch, uint32_t* wsum,
                                    uint64_t* nxt, V* wF) {
  uint64_t a = ach[0], b = bch[0];
  int h = 0;
  while (b - a > 32) {
    uint64_t a1, b1;
    if (h + 1 < kTreeD) {
      a1 = ach[h + 1];
      b1 = bch[h + 1];
    } else {
      if (threadIdx.x < 32) {
        const uint64_t ra = warp_rank(sd, R, a < t ? a : t, threadIdx.x);
        const uint64_t rb = warp_rank(sd, R, b < t ? b : t, threadIdx.x);
        if (threadIdx.x == 0) { nxt[0] = n1 + ra; nxt[1] = n1 + rb; }
      }
      __syncthreads();
      a1 = nxt[0];
      b1 = nxt[1];
    }
    uint32_t done = 0;
    for (uint64_t p0 = a; p0 < b; p0 += kTreeChunk) {
      const uint32_t len = (uint32_t)min((uint64_t)kTreeChunk, b - p0);
      if (h == 0)
        done += tree_chunk<V, true>(acc, Fs, sd, t, p0, len, (uint32_t)(p0 - a), a1 + done, done, wsum);
      else
        done += tree_chunk<V, false>(acc, Fs, sd, t, p0, len, (uint32_t)(p0 - a), a1 + done, done, wsum);
      __syncthreads();  // F slots and wsum settled before the next chunk
    }
    a = a1;
    b = b1;
    ++h;
  }
  if (threadIdx.x >= 32) return;
  // short windows: one warp, F in registers, no block barriers
  const uint32_t lane = threadIdx.x;
  V f{};
  if (lane < b - a) f = (h == 0) ? acc.ld(a + lane) : Fs[lane];
  const uint32_t ltmask = ~(0xffffffffu >> lane);
  while (a < b) {
    uint64_t a1, b1;
    if (h + 1 < kTreeD) {
      a1 = ach[h + 1];
      b1 = bch[h + 1];
    } else {
      a1 = n1 + warp_rank(sd, R, a < t ? a : t, lane);
      b1 = n1 + warp_rank(sd, R, b < t ? b : t, lane);
    }
    const uint32_t L = (uint32_t)(b - a);
    uint32_t w = 0;
    if (a < t) {
      w = (uint32_t)(bits64_at(sd, a) >> 32);
      uint64_t nv = t - a;
      if (nv > L) nv = L;
      if (nv < 32) w &= ~(0xffffffffu >> nv);
    }
    const bool one = (w >> (31 - lane)) & 1u;
    const uint32_t r = __popc(w & ltmask);
    if (one) {
      acc.st(a + lane, acc.ld(a1 + r));
      wF[r] = f;
    } else if (lane < L) {
      acc.st(a + lane, f);
    }
    __syncwarp();
    f = wF[lane];
    __syncwarp();
    a = a1;
    b = b1;
    ++h;
  }
}

template <typename V>
struct TreeCfg {
  static constexpr uint32_t T0 = sizeof(V) == 4 ? 4096u : 2048u;      // positions of window 0 per CTA
  static constexpr uint32_t E = 16 / sizeof(V);                       // elements per 16 bytes
  // windows total ~2*T0 +- O(sqrt(T0)) for a random stream; a tile that does
  // not fit takes the direct path
  static constexpr uint32_t SCAP = T0 * 17 / 8 + 2 * E * kTreeD;       // staged elements (all windows)
  static constexpr uint32_t GCAP = SCAP / 32 + kTreeD;                 // 32-position groups
  static constexpr size_t SMEM = (size_t)SCAP * sizeof(V) + GCAP * 16;  // stage | group descriptors
};

uint32_t tree_tile(int eb) { return eb == 4 ? TreeCfg<uint32_t>::T0 : TreeCfg<unsigned long long>::T0; }

// Staged tree merge.  One CTA per window-0 tile:
//  1. window starts a_h / ends b_h (precomputed chains), staging layout by a
//     warp scan;
//  2. TMA bulk copies of in[a_h, b_h) for every window into shared memory
//     (16-byte aligned interiors; the ragged ends by plain loads);
//  3. the bits of every window as 32-position groups and one block scan for
//     the ones' ranks (a group descriptor: mask, stage index of the group's
//     first position and of its first one's B slot);
//  4. the in-place swap merge itself, window after window: the one at stage
//     position i of window h swaps with slot rank(i) of window h+1 (the
//     reference's swap(a[i], a[mid]) with mid = n1 + rank'(i)); swaps of one
//     window touch distinct slots, so a window is one parallel step;
//  5. TMA bulk stores of every window from shared memory to out[].
// Each element is read once and written once; no global round trip between.
template <typename V, class Acc>
__device__ __forceinline__ void merge_tree_tile(const Acc& acc, const PairPlan* __restrict__ Pp, uint64_t a, uint64_t b,
                                                const uint64_t* __restrict__ rank, const uint64_t* __restrict__ ca) {
  using C = TreeCfg<V>;
  extern __shared__ __align__(128) unsigned char tree_smem[];
  V* stage = reinterpret_cast<V*>(tree_smem);
  // group descriptor: x = ones mask, y = stage index of the group's first
  // position, z = stage index of the B slot of its first one
  uint4* gdesc = reinterpret_cast<uint4*>(stage + C::SCAP);
  __shared__ uint32_t wsum[kTreeBlock / 32];
  __shared__ uint64_t ach[kTreeD], bch[kTreeD], nxt[2];
  __shared__ uint32_t stoff[kTreeD], goff[kTreeD + 1];
  __shared__ uint32_t ilo_s[kTreeD], ihi_s[kTreeD];
  __shared__ int nwin_s;
  __shared__ __align__(8) uint64_t bar;
  __shared__ V wF[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t n1 = Pp->n1;
  const uint64_t t = Pp->t;
  const StreamDesc sd = Pp->sd;
  const uint64_t* R = rank + Pp->rank_off;
  // TMA needs in[] and out[] (every part) equally aligned mod 16 bytes
  const bool tma = acc.same_alignment();
  // 1. windows: lane h owns window h.  Every warp derives the same staging
  //    layout in registers (no block barrier before the bits are ranked);
  //    warp 0 publishes it to shared memory and issues the TMA loads.
  // (a, b): window h's start and end in lane h, loaded by the caller first
  const uint32_t emp = __ballot_sync(0xffffffffu, lane < (uint32_t)kTreeD && a == b);
  const uint32_t nw = emp ? (uint32_t)(__ffs(emp) - 1) : (uint32_t)kTreeD;
  const bool act = lane < nw;
  const uint64_t len = act ? b - a : 0;
  const bool big = len > C::SCAP;
  uint32_t mis = 0, reg = 0, gc = 0, lo = 0, hi = 0, bytes = 0;
  if (act && !big) {
    const uintptr_t A0 = reinterpret_cast<uintptr_t>(acc.src(a));
    const uint32_t l32 = (uint32_t)len;  // (<= SCAP here)
    mis = (uint32_t)((A0 & 15) / sizeof(V));
    reg = (mis + l32 + C::E - 1) & ~(C::E - 1);
    gc = (l32 + 31) >> 5;
    const uint32_t l0 = (C::E - mis) & (C::E - 1);  // first 16-byte aligned offset
    const uint32_t l1 = ((mis + l32) & ~(C::E - 1)) - mis;
    if (tma && l1 > l0 && l1 <= l32) {
      lo = l0;
      hi = l1;
      bytes = (l1 - l0) * (uint32_t)sizeof(V);
    }
  }
  // one scan for three prefixes: staged elements, and packed in 16-bit halves
  // the groups (low) and the ones of the windows before h (high) = the
  // lengths of windows 1..h (|window w+1| = ones of window w below t).  No
  // carry crosses the halves: a tile's group total is < 2^16 (big windows
  // count none), and the high half is used only when the tile is staged
  // (total length <= SCAP < 2^16).
  uint32_t sreg = reg;
  uint32_t spk = gc | ((lane >= 1 ? (uint32_t)min(len, (uint64_t)0xFFFFu) : 0u) << 16);
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y1 = __shfl_up_sync(0xffffffffu, sreg, o);
    const uint32_t y2 = __shfl_up_sync(0xffffffffu, spk, o);
    if (lane >= (uint32_t)o) { sreg += y1; spk += y2; }
  }
  const uint32_t sgc = spk & 0xFFFFu;
  const uint32_t treg = __shfl_sync(0xffffffffu, sreg, 31), tgc = __shfl_sync(0xffffffffu, sgc, 31);
  const uint32_t tby = __reduce_add_sync(0xffffffffu, bytes);  // TMA bytes (only the total is needed)
  const bool ok = nw < (uint32_t)kTreeD && !__any_sync(0xffffffffu, big) && treg <= C::SCAP && tgc <= C::GCAP &&
                  !g_tree_force_direct;
  const uint32_t r_stoff = sreg - reg + mis, r_goff = act ? sgc - gc : tgc;
  const uint32_t r_onesb = spk >> 16;
  const uint32_t r_ilo = hi > lo ? lo : (uint32_t)len, r_ihi = hi > lo ? hi : (uint32_t)len;
  if (wid == 0) {
    if (lane < (uint32_t)kTreeD) {
      ach[lane] = a;
      bch[lane] = b;
    }
    if (act) {
      stoff[lane] = r_stoff;
      goff[lane] = r_goff;
      ilo_s[lane] = r_ilo;
      ihi_s[lane] = r_ihi;
    }
    if (lane == 0) {
      goff[nw] = tgc;
      nwin_s = ok ? (int)nw : -1;
      if (ok) {
        mbar_init(&bar, 1);
        mbar_arrive_expect_tx(&bar, tby);
      }
    }
    __syncwarp();
    if (ok && act && hi > lo) {
      V* st = stage + r_stoff;
      acc.runs(a + lo, a + hi, [&](uint64_t x0, uint64_t x1) {
        bulk_g2s(st + (x0 - a), acc.src(x0), (uint32_t)((x1 - x0) * sizeof(V)), &bar);
      });
    }
  }
  if (!ok) {
    __syncthreads();
    tree_windows_direct<V>(acc, stage, sd, R, n1, t, ach, bch, wsum, nxt, wF);
    return;
  }
  const uint32_t ngroups = tgc;
  // ragged ends (outside the 16-byte aligned interiors) by plain loads, a warp
  // per window.  With TMA they are short (head < 2E-1, tail < E elements):
  // loaded into registers now, stored to shared memory after the bits are
  // ranked, so their latency overlaps that work.
  constexpr int kRagW = (kTreeD + kTreeBlock / 32 - 1) / (kTreeBlock / 32);  // windows per warp
  V rag[kRagW];
  uint32_t ragi[kRagW];
  if (tma) {
#pragma unroll
    for (int k = 0; k < kRagW; ++k) {
      const int h = wid + k * (kTreeBlock / 32);
      ragi[k] = 0xffffffffu;
      if (h < (int)nw) {
        const uint64_t ah = __shfl_sync(0xffffffffu, a, h);
        const uint32_t L = (uint32_t)__shfl_sync(0xffffffffu, len, h);
        const uint32_t wlo = __shfl_sync(0xffffffffu, r_ilo, h), whi = __shfl_sync(0xffffffffu, r_ihi, h);
        const uint32_t so = __shfl_sync(0xffffffffu, r_stoff, h);
        const uint32_t i = lane < 8 ? lane : whi + lane - 8;
        if (lane < 16 && i < (lane < 8 ? wlo : L)) {
          ragi[k] = so + i;
          rag[k] = acc.ld(ah + i);
        }
      }
    }
  } else {
    for (int h = wid; h < (int)nw; h += kTreeBlock / 32) {
      const uint64_t ah = __shfl_sync(0xffffffffu, a, h);
      const uint32_t L = (uint32_t)__shfl_sync(0xffffffffu, len, h);
      const uint32_t wlo = __shfl_sync(0xffffffffu, r_ilo, h), whi = __shfl_sync(0xffffffffu, r_ihi, h);
      V* st = stage + __shfl_sync(0xffffffffu, r_stoff, h);
      for (uint32_t i = lane; i < wlo; i += 32) st[i] = acc.ld(ah + i);
      for (uint32_t i = whi + lane; i < L; i += 32) st[i] = acc.ld(ah + i);
    }
  }
  // 3. group masks (two consecutive groups per thread) and their ones
  uint32_t cnt2[2], mm[2], gy[2], gz[2];
  {
    // window of group 2*tid: the last h < nw with goff[h] <= G (binary search
    // over the lanes); group 2*tid+1 lies in the same window or the next one
    // (windows h < nw are non-empty)
    const uint32_t G0 = 2 * tid;
    uint32_t h0 = 0;
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1) {
      const uint32_t c = h0 + step;
      const uint32_t gc_ = __shfl_sync(0xffffffffu, r_goff, c & 31);
      h0 = (c < nw && gc_ <= G0) ? c : h0;
    }
    const uint32_t gnext = __shfl_sync(0xffffffffu, r_goff, (h0 + 1) & 31);
    const bool step1 = h0 + 1 < nw && gnext <= G0 + 1;
    const uint32_t hh[2] = {h0, step1 ? h0 + 1 : h0};
    uint64_t bits0 = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const uint32_t G = G0 + e, h = hh[e];
      const uint64_t wa = __shfl_sync(0xffffffffu, a, h), wb = __shfl_sync(0xffffffffu, b, h);
      const uint32_t wg = __shfl_sync(0xffffffffu, r_goff, h);
      uint32_t m = 0;
      if (G < ngroups) {
        const uint64_t p = wa + 32ull * (G - wg);
        if (p < t) {
          const uint64_t nv = min(wb - p, t - p);
          // group 2*tid+1 in the same window: the low half of group 2*tid's 64 bits
          if (e == 0) bits0 = bits64_at(sd, p);
          m = (e == 0 || step1) ? (uint32_t)((e == 0 ? bits0 : bits64_at(sd, p)) >> 32) : (uint32_t)bits0;
          if (nv < 32) m &= ~(0xffffffffu >> nv);
        }
      }
      cnt2[e] = __popc(m);
      // descriptor parts known now: stage index of the group's first position,
      // and of its window's B slots minus the ones of the windows before h
      const uint32_t st_h = __shfl_sync(0xffffffffu, r_stoff, h), st_h1 = __shfl_sync(0xffffffffu, r_stoff, (h + 1) & 31);
      const uint32_t ob = __shfl_sync(0xffffffffu, r_onesb, h);
      gy[e] = st_h + 32 * (G - wg);
      gz[e] = st_h1 - ob;
      mm[e] = m;
    }
  }
  const uint32_t c2 = cnt2[0] + cnt2[1];
  uint32_t x = c2;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  if (tma) {
#pragma unroll
    for (int k = 0; k < kRagW; ++k)
      if (ragi[k] != 0xffffffffu) stage[ragi[k]] = rag[k];
  }
  __syncthreads();
  // warp totals' exclusive prefix by a shuffle scan over the first lanes
  uint32_t ws = lane < (uint32_t)(kTreeBlock / 32) ? wsum[lane] : 0u;
#pragma unroll
  for (int o = 1; o < kTreeBlock / 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
    if (lane >= (uint32_t)o) ws += y;
  }
  const uint32_t before = __shfl_sync(0xffffffffu, ws, (wid + 31) & 31) * (wid ? 1u : 0u);
  const uint32_t ex0 = before + x - c2, ex1 = ex0 + cnt2[0];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const uint32_t G = 2 * tid + e;
    // (stage offsets in bytes: the swap loop adds them straight to the shared base)
    if (G < ngroups)
      gdesc[G] = make_uint4(mm[e], gy[e] * (uint32_t)sizeof(V), (gz[e] + (e ? ex1 : ex0)) * (uint32_t)sizeof(V), 0u);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  // 4. the swaps, window by window (the last window has no ones).  Windows
  //    shrink (|window h+1| = ones of window h); from the first window of at
  //    most 64 positions on, warp 0 finishes alone with warp barriers.
  const uint32_t ltmask = ~(0xffffffffu >> lane);
  constexpr uint32_t kSh = sizeof(V) == 4 ? 2u : 3u;
  const uint32_t lb = lane << kSh;
  char* const sb = reinterpret_cast<char*>(stage);
  auto at = [&](uint32_t off) -> V& { return *reinterpret_cast<V*>(sb + off); };
  int h = 0;
  constexpr uint32_t NWp = kTreeBlock / 32;
  // windows of more than two groups (a prefix: window sizes about halve) go
  // to the whole block; their group ranges come from the lanes' registers
  const uint32_t r_gnx = __shfl_down_sync(0xffffffffu, r_goff, 1);  // goff[h + 1] in lane h
  const uint32_t bwin = __ballot_sync(0xffffffffu, lane + 1 < nw && r_gnx - r_goff > 2);
  const int nbw = __ffs(~bwin) - 1;
  for (; h < nbw; ++h) {
    // two groups per trip (independent slots): their smem round trips overlap
    const uint32_t g1 = __shfl_sync(0xffffffffu, r_gnx, h);
    uint32_t G = __shfl_sync(0xffffffffu, r_goff, h) + wid;
    const uint4* dp = gdesc + G;
    for (int trips = G + NWp < g1 ? (int)((g1 - G - NWp - 1) / (2 * NWp)) + 1 : 0; trips > 0; --trips) {
      const uint4 d0 = dp[0], d1 = dp[NWp];
      dp += 2 * NWp;
      G += 2 * NWp;
      const bool on0 = (d0.x << lane) >> 31, on1 = (d1.x << lane) >> 31;
      const uint32_t ia0 = d0.y + lb, ib0 = d0.z + (__popc(d0.x & ltmask) << kSh);
      const uint32_t ia1 = d1.y + lb, ib1 = d1.z + (__popc(d1.x & ltmask) << kSh);
      V va0, vb0, va1, vb1;
      if (on0) { va0 = at(ia0); vb0 = at(ib0); }
      if (on1) { va1 = at(ia1); vb1 = at(ib1); }
      if (on0) { at(ia0) = vb0; at(ib0) = va0; }
      if (on1) { at(ia1) = vb1; at(ib1) = va1; }
    }
    if (G < g1) {
      const uint4 d = gdesc[G];
      if ((d.x << lane) >> 31) {
        const uint32_t ia = d.y + lb, ib = d.z + (__popc(d.x & ltmask) << kSh);
        const V va = at(ia), vb = at(ib);
        at(ia) = vb;
        at(ib) = va;
      }
    }
    __syncthreads();
  }
  // Windows below h are final now (a window is written only by its own swaps
  // and by the previous window's): with TMA their stores start while warp 0
  // finishes the short windows -- warp 1 issues the bulk stores, warps 2..7
  // the ragged ends.
  const int hf = h;
  auto store_ragged = [&](int h0, int h1, uint32_t t0, uint32_t nthr) {
    // a window's head is < 2E-1 and its tail < E elements: 16 slots per window
    for (uint32_t t = t0; t < (uint32_t)(h1 - h0) * 16u; t += nthr) {
      const uint32_t hw = (uint32_t)h0 + (t >> 4), k = t & 15u;
      const uint32_t lo = ilo_s[hw], hi = ihi_s[hw];
      const uint32_t i = k < 8 ? k : hi + (k - 8);
      const uint32_t lim = k < 8 ? lo : (uint32_t)(bch[hw] - ach[hw]);
      if (i < lim) acc.st(ach[hw] + i, stage[stoff[hw] + i]);
    }
  };
  auto store_tma = [&](int h0, int h1) {  // one lane per window
    if (lane >= (uint32_t)h0 && lane < (uint32_t)h1 && ihi_s[lane] > ilo_s[lane]) {
      const uint64_t a = ach[lane];
      const V* st = stage + stoff[lane];
      acc.runs(a + ilo_s[lane], a + ihi_s[lane], [&](uint64_t x0, uint64_t x1) {
        bulk_s2g(acc.dst(x0), st + (x0 - a), (uint32_t)((x1 - x0) * sizeof(V)));
      });
    }
    bulk_commit();
  };
  if (tma) {
    fence_proxy_async_smem();
    __syncthreads();
    if (wid == 1) store_tma(0, hf);
    else if (wid >= 2) store_ragged(0, hf, tid - 64, kTreeBlock - 64);
  }
  if (wid == 0) {
    for (; h + 1 < nw; ++h) {
      for (uint32_t G = goff[h]; G < goff[h + 1]; ++G) {
        const uint4 d = gdesc[G];
        if ((d.x << lane) >> 31) {
          const uint32_t ia = d.y + lb, ib = d.z + (__popc(d.x & ltmask) << kSh);
          const V va = at(ia), vb = at(ib);
          at(ia) = vb;
          at(ib) = va;
        }
      }
      __syncwarp();
    }
    if (tma) fence_proxy_async_smem();
  }
  // 5. the remaining stores
  __syncthreads();
  if (tma) {
    if (wid == 0) store_tma(hf, (int)nw);
    store_ragged(hf, (int)nw, tid, kTreeBlock);
  } else {
    for (int hw = wid; hw < nw; hw += kTreeBlock / 32) {
      const uint32_t L = (uint32_t)(bch[hw] - ach[hw]);
      const uint32_t lo = ilo_s[hw], hi = ihi_s[hw];
      const V* st = stage + stoff[hw];
      for (uint32_t i = lane; i < lo; i += 32) acc.st(ach[hw] + i, st[i]);
      for (uint32_t i = hi + lane; i < L; i += 32) acc.st(ach[hw] + i, st[i]);
    }
  }
  if (tma && wid <= 1) bulk_wait_read0();  // the shared source must outlive the copies
}

// One CTA per (pair, tile) of a round.
template <typename V>
__global__ void __launch_bounds__(kTreeBlock, 5) merge_tree_kernel(const V* __restrict__ in, V* __restrict__ out,
                                                                const PairPlan* __restrict__ plans,
                                                                const uint64_t* __restrict__ rank,
                                                                const uint64_t* __restrict__ chains, uint32_t tpp,
                                                                uint32_t pair_in_y) {
  // 2-D grid (no division): tiles of a pair along x, pairs along y -- or the
  // transpose when there are more than 65535 pairs
  const uint32_t g = pair_in_y ? blockIdx.y : blockIdx.x, tau = pair_in_y ? blockIdx.x : blockIdx.y;
  const PairPlan* Pp = plans + g;
  // the window chain first: its load overlaps the plan's
  const uint64_t* ca = chains + ((uint64_t)g * (tpp + 1) + tau) * kTreeD;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t a = 0, b = 0;
  if (lane < (uint32_t)kTreeD) {
    a = ca[lane];
    b = ca[kTreeD + lane];
  }
  if (tau * (uint64_t)TreeCfg<V>::T0 >= Pp->n1) return;
  const FlatAcc<V> acc{in + Pp->s, out + Pp->s};
  merge_tree_tile<V>(acc, Pp, a, b, rank, chains + ((uint64_t)g * (tpp + 1) + tau) * kTreeD);
}

// One pair split over peer buffers (in place); this launch takes the tiles
// tau = part, part + nparts, ...
template <typename V>
__global__ void __launch_bounds__(kTreeBlock, 5) merge_tree_peer_kernel(const PeerParts<V> parts,
                                                                     const PairPlan* __restrict__ plans,
                                                                     const uint64_t* __restrict__ rank,
                                                                     const uint64_t* __restrict__ chains,
                                                                     uint32_t tpp, uint32_t part, uint32_t nparts) {
  const uint64_t tau = part + (uint64_t)blockIdx.x * nparts;
  if (tau >= tpp || tau * (uint64_t)TreeCfg<V>::T0 >= plans->n1) return;
  const PeerAcc<V> acc{parts};
  const uint64_t* ca = chains + tau * kTreeD;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t a = 0, b = 0;
  if (lane < (uint32_t)kTreeD) {
    a = ca[lane];
    b = ca[kTreeD + lane];
  }
  merge_tree_tile<V>(acc, plans, a, b, rank, ca);
}

template <typename V>
static void merge_tree_peer_t(const PeerSpan& ps, const PairPlan* plans, const uint64_t* rank, const uint64_t* chains,
                              uint32_t tpp, uint32_t part, cudaStream_t st) {
  PeerParts<V> P{};
  P.n = ps.n;
  bool tma = true;
  const uintptr_t ref = reinterpret_cast<uintptr_t>(ps.base[0]) - ps.start[0] * sizeof(V);
  for (int k = 0; k < ps.n; ++k) {
    P.base[k] = reinterpret_cast<V*>(ps.base[k]);
    P.start[k] = ps.start[k];
    const uintptr_t z = reinterpret_cast<uintptr_t>(ps.base[k]) - ps.start[k] * sizeof(V);
    tma = tma && ((z - ref) & 15) == 0 && (ps.start[k] * sizeof(V)) % 16 == 0;
  }
  P.start[ps.n] = ps.start[ps.n];
  P.tma = tma ? 1 : 0;
  // (per device: function attributes belong to the current device's context)
  cudaFuncSetAttribute(merge_tree_peer_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TreeCfg<V>::SMEM);
  const uint32_t nparts = (uint32_t)ps.n;
  const uint32_t grid = (tpp + nparts - 1 - part) / nparts;
  if (!grid) return;
  merge_tree_peer_kernel<V><<<grid, kTreeBlock, TreeCfg<V>::SMEM, st>>>(P, plans, rank, chains, tpp, part, nparts);
  count_launch();
}

void launch_merge_tree_peer(int eb, const PeerSpan& ps, const PairPlan* plans, const uint64_t* rank,
                            const uint64_t* chains, uint32_t tpp, uint32_t part, cudaStream_t st) {
  if (eb == 4) merge_tree_peer_t<uint32_t>(ps, plans, rank, chains, tpp, part, st);
  else merge_tree_peer_t<unsigned long long>(ps, plans, rank, chains, tpp, part, st);
}

template <typename V>
static void merge_tree_t(void* in, void* out, const PairPlan* plans, uint64_t npairs, const uint64_t* rank,
                         const uint64_t* chains, uint32_t tpp, cudaStream_t st) {
  const size_t smem = TreeCfg<V>::SMEM;
  cudaFuncSetAttribute(merge_tree_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const bool piy = npairs <= 65535;
  if (!piy && tpp > 65535) throw std::runtime_error("merge round: too many pairs and tiles for the grid");
  const dim3 grid = piy ? dim3(tpp, (unsigned)npairs) : dim3((unsigned)npairs, tpp);
  merge_tree_kernel<V><<<grid, kTreeBlock, smem, st>>>((const V*)in, (V*)out, plans, rank, chains, tpp, piy ? 1u : 0u);
  count_launch();
}

// Pairs [p0, p1) of a round only (the host entry's chunk-local rounds).
void launch_merge_tree_range(int eb, void* in, void* out, const PairPlan* plans, uint64_t p0, uint64_t p1,
                             const uint64_t* rank, const uint64_t* chains, uint32_t tpp, cudaStream_t st) {
  if (p1 <= p0) return;
  launch_merge_tree(eb, in, out, plans + p0, p1 - p0, rank, chains + p0 * (tpp + 1) * kTreeD, tpp, st);
}

void launch_merge_tree(int eb, void* in, void* out, const PairPlan* plans, uint64_t npairs, const uint64_t* rank,
                       const uint64_t* chains, uint32_t tpp, cudaStream_t st) {
  if (!npairs) return;
  if (eb == 4) merge_tree_t<uint32_t>(in, out, plans, npairs, rank, chains, tpp, st);
  else merge_tree_t<unsigned long long>(in, out, plans, npairs, rank, chains, tpp, st);
}

// [X, N) is untouched by phase 1 (A queue empty past X).
template <typename V>
__global__ void copy_region_kernel(const V* __restrict__ in, V* __restrict__ out, const PairPlan* __restrict__ plans) {
  const PairPlan* P = plans + blockIdx.x;
  uint64_t N = P->n1 + P->n2;
  for (uint64_t i = P->X + threadIdx.x; i < N; i += blockDim.x) out[P->s + i] = in[P->s + i];
}

void launch_copy_tail_region(int eb, const void* in, void* out, const PairPlan* plans, uint64_t npairs,
                             cudaStream_t st) {
  if (!npairs) return;
  if (eb == 4) copy_region_kernel<uint32_t><<<(unsigned)npairs, 256, 0, st>>>((const uint32_t*)in, (uint32_t*)out, plans);
  else copy_region_kernel<unsigned long long><<<(unsigned)npairs, 256, 0, st>>>((const unsigned long long*)in,
                                                                               (unsigned long long*)out, plans);
  count_launch();
}

// -------------------------------------------------------------- tail plan

// Over records sorted by target (stable in x): predecessor in the target's
// group, and for each group's last step x_last > q the output (q <- x_last).
// ------------------------------------------------------------ tail plans
// The records of a round live at [tail_off, tail_off + tail_len) per pair,
// tail_off the exclusive prefix of tail_len over the round's pairs (one CTA
// scans them).  The buffers hold `cap` records (a bound sized on the host
// from the pair geometry, tail_capacity): the pairs from the first one that
// does not fit on are marked tail_slow and keep no records; their tail runs
// serially (tail_slow_apply).  *used = records kept.
__global__ void __launch_bounds__(1024) tail_offsets_kernel(PairPlan* __restrict__ plans, uint64_t npairs,
                                                            uint64_t cap, uint64_t* __restrict__ used) {
  __shared__ uint64_t wsum[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t per = (npairs + 1023) / 1024, g0 = tid * per, g1 = min(npairs, g0 + per);
  uint64_t sum = 0;
  for (uint64_t g = g0; g < g1; ++g) sum += plans[g].tail_len;
  uint64_t x = sum;  // inclusive block scan of the per-thread sums
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  uint64_t before = 0;
  for (uint32_t w = 0; w < wid; ++w) before += wsum[w];
  uint64_t acc = before + x - sum;
  uint64_t first_slow = kNone;
  for (uint64_t g = g0; g < g1; ++g) {
    const uint64_t len = plans[g].tail_len;
    const bool slow = acc + len > cap;
    plans[g].tail_off = slow ? 0 : acc;
    plans[g].tail_slow = slow ? 1u : 0u;
    if (slow && first_slow == kNone) first_slow = acc;
    acc += len;
  }
  // records kept = the prefix at the first slow pair (prefixes grow with g), else the total
  __shared__ unsigned long long s_used;
  if (tid == 0) s_used = ~0ULL;
  __syncthreads();
  if (first_slow != kNone) atomicMin(&s_used, (unsigned long long)first_slow);
  __syncthreads();
  if (tid == 1023) *used = (s_used != ~0ULL) ? s_used : acc;
}

void launch_tail_offsets(PairPlan* plans, uint64_t npairs, uint64_t cap, uint64_t* used, cudaStream_t st) {
  tail_offsets_kernel<<<1, 1024, 0, st>>>(plans, npairs, cap, used);
  count_launch();
}

// Records with the same target (a global position; equal targets lie in one
// pair) are chained through an open-addressing table keyed by the target:
// the slot's head is pushed atomically, so each chain lists every record of
// its target (equal targets are rare: ~L^2/2N per pair).
__device__ __forceinline__ uint32_t tail_hash(uint64_t key, uint32_t mask) {
  return (uint32_t)((key * GOLDEN) >> 32) & mask;
}

__global__ void tail_hash_kernel(const uint64_t* __restrict__ rec_key, const uint64_t* __restrict__ used,
                                 uint64_t* __restrict__ hkey, uint32_t* __restrict__ hhead,
                                 uint32_t* __restrict__ next, uint32_t* __restrict__ slot_of, uint32_t mask) {
  const uint64_t rec = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rec >= *used) return;
  const uint64_t key = rec_key[rec];
  uint32_t h = tail_hash(key, mask);
  for (;;) {
    const unsigned long long prev =
        atomicCAS(reinterpret_cast<unsigned long long*>(hkey + h), ~0ULL, (unsigned long long)key);
    if (prev == ~0ULL || prev == key) break;
    h = (h + 1) & mask;
  }
  slot_of[rec] = h;
  next[rec] = atomicExch(hhead + h, (uint32_t)rec);
}

// Per record x (target q = m_x): predx = the latest earlier step with the same
// target; the LAST step targeting q moves P1[x] into q for good (when x > q)
// -- a (dst, src) pair; a tail position q >= t written that way is "keyed"
// (tests/decomp_model.py tail_plan_model).
__global__ void tail_plan_kernel(const PairPlan* __restrict__ plans, const uint64_t* __restrict__ rec_key,
                                 const uint32_t* __restrict__ rec_pair, const uint64_t* __restrict__ used,
                                 const uint32_t* __restrict__ hhead, const uint32_t* __restrict__ next,
                                 const uint32_t* __restrict__ slot_of, uint64_t* __restrict__ predx,
                                 uint8_t* __restrict__ keyed, uint64_t* __restrict__ dst,
                                 uint64_t* __restrict__ src) {
  const uint64_t rec = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rec >= *used) return;
  const uint64_t key = rec_key[rec];
  const PairPlan* P = plans + rec_pair[rec];
  const uint64_t off = P->tail_off, loc = rec - off, x = P->t + loc;
  // records of one pair are consecutive: step order == record order
  uint64_t pred = kNone;
  bool last = true;
  for (uint32_t r = hhead[slot_of[rec]]; r != 0xffffffffu; r = next[r]) {
    if (r == rec || rec_key[r] != key) continue;
    if (r < rec) pred = (pred == kNone || r > pred) ? r : pred;
    else last = false;
  }
  predx[rec] = pred == kNone ? kNone : P->t + (pred - off);
  if (last) {
    const uint64_t q = key - P->s;
    if (x > q) {
      const uint64_t slot = 2 * off + P->tail_len + loc;
      dst[slot] = key;
      src[slot] = P->s + x;
      if (q >= P->t) keyed[off + (q - P->t)] = 1;
    }
  }
}

void launch_tail_plan(const PairPlan* plans, const uint64_t* rec_key, const uint32_t* rec_pair, const uint64_t* used,
                      uint64_t cap, uint64_t* hkey, uint32_t* hhead, uint32_t* next, uint32_t* slot_of, uint32_t hmask,
                      uint64_t* predx, uint8_t* keyed, uint64_t* dst, uint64_t* src, cudaStream_t st) {
  const unsigned b = (unsigned)((cap + 255) / 256);
  tail_hash_kernel<<<b, 256, 0, st>>>(rec_key, used, hkey, hhead, next, slot_of, hmask);
  tail_plan_kernel<<<b, 256, 0, st>>>(plans, rec_key, rec_pair, used, hhead, next, slot_of, predx, keyed, dst, src);
  count_launch();
  count_launch();
}

// For every insertion position x not overwritten later: chase V(m_x, x).
__global__ void tail_chase_kernel(const PairPlan* __restrict__ plans, const uint64_t* __restrict__ rec_key,
                                  const uint32_t* __restrict__ rec_pair, const uint64_t* __restrict__ predx,
                                  const uint8_t* __restrict__ keyed, const uint64_t* __restrict__ used,
                                  uint64_t* __restrict__ dst, uint64_t* __restrict__ src) {
  uint64_t rec = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rec >= *used) return;
  if (keyed[rec]) return;
  const PairPlan* P = plans + rec_pair[rec];
  const uint64_t t = P->t, s = P->s, off = P->tail_off;
  uint64_t loc = rec - off, x = t + loc;
  uint64_t r = rec, sr;
  for (;;) {
    uint64_t q = rec_key[r] - s;
    uint64_t xr = t + (r - off);
    uint64_t y = predx[r];
    if (y != kNone && y > q) { sr = y; break; }
    if (q == xr) { sr = xr; break; }
    if (q < t) { sr = q; break; }
    r = off + (q - t);
  }
  uint64_t slot = 2 * off + loc;
  dst[slot] = s + x;
  src[slot] = s + sr;
}

void launch_tail_chase(const PairPlan* plans, const uint64_t* rec_key, const uint32_t* rec_pair,
                       const uint64_t* predx, const uint8_t* keyed, const uint64_t* used, uint64_t cap, uint64_t* dst,
                       uint64_t* src, cudaStream_t st) {
  tail_chase_kernel<<<(unsigned)((cap + 255) / 256), 256, 0, st>>>(plans, rec_key, rec_pair, predx, keyed, used, dst,
                                                                   src);
  count_launch();
}

// ------------------------------------------------------------ tail apply
// The (dst, src) slots of a round: gather every source, then scatter (dst =
// kNone: unused slot).  Only slots whose dst lies in [lo, hi) (the host
// entry applies a round chunk by chunk).  The last CTA of the gather also
// runs the tail of every tail_slow pair of the range serially, in place --
// the reference loop itself (shufflers.py:188-191), never taken in practice.
template <typename V, class Acc>
__device__ void tail_serial_pairs(const Acc& acc, const PairPlan* __restrict__ plans, uint64_t npairs, uint64_t lo,
                                  uint64_t hi) {
  for (uint64_t g = threadIdx.x; g < npairs; g += blockDim.x) {
    const PairPlan P = plans[g];
    if (!P.tail_slow || P.s < lo || P.s >= hi) continue;
    Reader64 rd;
    rd.init(P.sd, P.t + 1);
    uint64_t nb = 0;
    for (uint64_t x = P.t; x < P.n1 + P.n2; ++x) {  // x >= t >= 1: bound >= 2
      const uint64_t m = fdr64(rd, x + 1, nb);
      const V a = acc.ld(P.s + x), b = acc.ld(P.s + m);
      acc.st(P.s + x, b);
      acc.st(P.s + m, a);
    }
  }
}

template <typename V>
__global__ void tail_gather_kernel(V* __restrict__ buf, const uint64_t* __restrict__ dst,
                                   const uint64_t* __restrict__ src, V* __restrict__ tmp, uint64_t n, uint64_t lo,
                                   uint64_t hi, const PairPlan* __restrict__ plans, uint64_t npairs) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    const uint64_t d = dst[k];
    if (d != kNone && d >= lo && d < hi) tmp[k] = buf[src[k]];
  }
  if (blockIdx.x == gridDim.x - 1) tail_serial_pairs<V>(FlatAcc<V>{buf, buf}, plans, npairs, lo, hi);
}
template <typename V>
__global__ void tail_scatter_kernel(V* __restrict__ buf, const uint64_t* __restrict__ dst,
                                    const V* __restrict__ tmp, uint64_t n, uint64_t lo, uint64_t hi) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    const uint64_t d = dst[k];
    if (d != kNone && d >= lo && d < hi) buf[d] = tmp[k];
  }
}

// Tail insertion over a pair split across peer buffers (positions are pair
// relative: the (dst, src) plan of an explicit pair with lo = 0).
template <typename V>
__global__ void tail_gather_peer_kernel(const PeerParts<V> P, const uint64_t* __restrict__ dst,
                                        const uint64_t* __restrict__ src, V* __restrict__ tmp, uint64_t n,
                                        const PairPlan* __restrict__ plans) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const PeerAcc<V> acc{P};
  if (k < n && dst[k] != kNone) tmp[k] = acc.ld(src[k]);
  if (blockIdx.x == gridDim.x - 1) tail_serial_pairs<V>(acc, plans, 1, 0, ~0ULL);
}
template <typename V>
__global__ void tail_scatter_peer_kernel(const PeerParts<V> P, const uint64_t* __restrict__ dst,
                                         const V* __restrict__ tmp, uint64_t n) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const PeerAcc<V> acc{P};
  if (k < n && dst[k] != kNone) acc.st(dst[k], tmp[k]);
}

template <typename V>
static void tail_apply_peer_t(const PeerSpan& ps, const uint64_t* dst, const uint64_t* src, void* tmp,
                              uint64_t nslots, const PairPlan* plans, cudaStream_t st) {
  PeerParts<V> P{};
  P.n = ps.n;
  for (int k = 0; k < ps.n; ++k) {
    P.base[k] = reinterpret_cast<V*>(ps.base[k]);
    P.start[k] = ps.start[k];
  }
  P.start[ps.n] = ps.start[ps.n];
  unsigned b = (unsigned)((nslots + 255) / 256);
  tail_gather_peer_kernel<V><<<b, 256, 0, st>>>(P, dst, src, (V*)tmp, nslots, plans);
  tail_scatter_peer_kernel<V><<<b, 256, 0, st>>>(P, dst, (const V*)tmp, nslots);
  count_launch();
  count_launch();
}

void launch_tail_apply_peer(int eb, const PeerSpan& ps, const uint64_t* dst, const uint64_t* src, void* tmp,
                            uint64_t nslots, const PairPlan* plans, cudaStream_t st) {
  if (!nslots) return;
  if (eb == 4) tail_apply_peer_t<uint32_t>(ps, dst, src, tmp, nslots, plans, st);
  else tail_apply_peer_t<unsigned long long>(ps, dst, src, tmp, nslots, plans, st);
}

template <typename V>
static void tail_apply_t(void* buf, const uint64_t* dst, const uint64_t* src, void* tmp, uint64_t nslots,
                         const PairPlan* plans, uint64_t npairs, uint64_t lo, uint64_t hi, cudaStream_t st) {
  const unsigned b = (unsigned)((nslots + 255) / 256);
  tail_gather_kernel<V><<<b, 256, 0, st>>>((V*)buf, dst, src, (V*)tmp, nslots, lo, hi, plans, npairs);
  tail_scatter_kernel<V><<<b, 256, 0, st>>>((V*)buf, dst, (const V*)tmp, nslots, lo, hi);
  count_launch();
  count_launch();
}

void launch_tail_apply(int eb, void* buf, const uint64_t* dst, const uint64_t* src, void* tmp, uint64_t nslots,
                       const PairPlan* plans, uint64_t npairs, uint64_t lo, uint64_t hi, cudaStream_t st) {
  if (!nslots) return;
  if (eb == 4) tail_apply_t<uint32_t>(buf, dst, src, tmp, nslots, plans, npairs, lo, hi, st);
  else tail_apply_t<unsigned long long>(buf, dst, src, tmp, nslots, plans, npairs, lo, hi, st);
}

}  // namespace sk
