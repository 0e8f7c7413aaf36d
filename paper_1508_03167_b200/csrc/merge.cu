// merge.cu -- one merge round of the parallel schedule (reference: _kernels.py:96-121
// _merge, shufflers.py:158-191 merge, rounds shufflers.py:117-130 / 291-297).
//
// Phase 1 (the coin-flip swap merge) is rewritten as a gather over "windows":
// the A queue of the in-place merge is the stream F with F[u] = A[u] (u < n1)
// and F[n1 + k] = F[select1(k)], so a tile of A elements [u0, u1) travels through
// contiguous windows V_0 = [u0, u1), V_{h+1} = [n1 + rank'(start V_h),
// n1 + rank'(end V_h)) (rank' = ones before min(p, t)).  In a window, a zero at p
// emits the carried A element, a one emits B[rank'(p)] and carries the A element
// on to the next window.  Windows of all tiles partition [0, X); [X, N) is the
// identity (A queue empty).  Every element is read once and written once.
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

// In-place inclusive scan of each pair's table (one CTA per pair).
__global__ void __launch_bounds__(1024) seg_scan_kernel(uint64_t* __restrict__ rank, uint64_t sbs) {
  uint64_t* R = rank + (uint64_t)blockIdx.x * sbs;
  __shared__ uint64_t wsum[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint64_t carry = 0;
  for (uint64_t base = 0; base < sbs; base += 1024) {
    uint64_t i = base + tid;
    uint64_t x = (i < sbs) ? R[i] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint64_t w = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= (uint32_t)o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    uint64_t add = carry + (wid ? wsum[wid - 1] : 0);
    if (i < sbs) R[i] = x + add;
    carry += wsum[31];
    __syncthreads();
  }
}

void launch_rank_tables(const LevelJob& LJ, uint64_t sbs, uint64_t* rank, cudaStream_t st) {
  uint64_t total = LJ.npairs * (sbs - 1);
  if (!total) return;
  rank_count_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(LJ, sbs, rank);
  count_launch();
  seg_scan_kernel<<<(unsigned)LJ.npairs, 1024, 0, st>>>(rank, sbs);
  count_launch();
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
  const uint64_t n1 = P.n1, n2 = P.n2, N = n1 + n2;
  if (n1 == 0 || n2 == 0) {  // shufflers.py:169-170: no bits, no change
    P.t = 0; P.X = n1; P.aex = 0; P.degenerate = 1; P.tail_len = 0; P.bits = 0;
  } else {
    const uint64_t* R = rank + g * sbs;
    uint64_t used = (N + 1 + 511) >> 9;
    uint64_t z = select_bit(P.sd, R, used, n1, false);
    uint64_t o = select_bit(P.sd, R, used, n2, true);
    uint64_t t = z < o ? z : o;
    P.t = t; P.aex = z < o; P.degenerate = 0;
    uint64_t S = n1;
    for (;;) {
      uint64_t S2 = n1 + rank_bits(P.sd, R, S < t ? S : t);
      if (S2 == S) break;
      S = S2;
    }
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
// One thread per pair, all rounds in one launch so the long top-round tails
// decode concurrently with the short ones.  Bits continue at offset t+1
// (shufflers.py:188-191): for x = t..N-1, m_x = FDR(x+1).
__global__ void tail_decode_kernel(const LevelTail* __restrict__ levels, int nlevels,
                                   const uint64_t* __restrict__ prefix, uint64_t total,
                                   unsigned long long* __restrict__ bits) {
  uint64_t gg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gg >= total) return;
  int L = 0;
  while (L + 1 < nlevels && prefix[L + 1] <= gg) ++L;
  uint64_t g = gg - prefix[L];
  LevelTail lv = levels[L];
  PairPlan* Pp = lv.plans + g;
  if (Pp->degenerate) return;
  const uint64_t t = Pp->t, N = Pp->n1 + Pp->n2, s = Pp->s, off = Pp->tail_off;
  uint64_t nb = 0;
  if (t < N) {
    Reader64 rd;
    rd.init(Pp->sd, t + 1);
    for (uint64_t x = t; x < N; ++x) {
      uint64_t m = fdr64(rd, x + 1, nb);
      lv.rec_key[off + (x - t)] = s + m;
      lv.rec_pair[off + (x - t)] = (uint32_t)g;
    }
  }
  uint64_t b = t + 1 + nb;
  Pp->bits = b;
  atomicAdd(&bits[Pp->array], (unsigned long long)b);
}

void launch_tail_decode(const LevelTail* d_levels, int nlevels, const uint64_t* d_prefix, uint64_t total_pairs,
                        unsigned long long* bits, cudaStream_t st) {
  if (!total_pairs) return;
  tail_decode_kernel<<<(unsigned)((total_pairs + 63) / 64), 64, 0, st>>>(d_levels, nlevels, d_prefix, total_pairs,
                                                                         bits);
  count_launch();
}

// ---------------------------------------------------------- window chains
// Window chain of every tile.  nwin = number of windows (the chain ends with an
// empty window), or kHMax+1+stored when the chain is longer than kHMax or the
// tile's carried elements exceed the parallel kernel's buffer (cap): such tiles
// take the sequential-window kernel.
__global__ void windows_kernel(const PairPlan* __restrict__ plans, uint64_t npairs, uint32_t tpp, uint32_t T,
                               const uint64_t* __restrict__ rank, WinRec* __restrict__ wins,
                               uint32_t* __restrict__ nwin, uint64_t cap, uint32_t* __restrict__ flag_list,
                               uint32_t* __restrict__ flag_count) {
  uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= npairs * tpp) return;
  uint64_t g = idx / tpp, tau = idx - g * tpp;
  const PairPlan& P = plans[g];
  uint64_t u0 = tau * (uint64_t)T;
  uint32_t h = 0;
  if (u0 < P.n1) {
    const uint64_t* R = rank + P.rank_off;
    const uint64_t t = P.t, n1 = P.n1;
    uint64_t S = u0, len = min((uint64_t)T, n1 - u0), carried = 0;
    while (len > 0 && h < (uint32_t)kHMax) {
      wins[idx * kHMax + h] = WinRec{S, len};
      if (h) carried += len;
      ++h;
      uint64_t os = rank_bits(P.sd, R, S < t ? S : t);
      uint64_t e = S + len;
      uint64_t oe = rank_bits(P.sd, R, e < t ? e : t);
      S = n1 + os;
      len = oe - os;
    }
    if (len > 0 || carried > cap) {  // flagged; stored count kept
      h += kHMax + 1;
      flag_list[atomicAdd(flag_count, 1u)] = (uint32_t)idx;
    }
  }
  nwin[idx] = h;
}

void launch_windows(const PairPlan* plans, uint64_t npairs, uint32_t tpp, uint32_t tile, const uint64_t* rank,
                    WinRec* wins, uint32_t* nwin, uint32_t* flag_list, uint32_t* flag_count, cudaStream_t st) {
  uint64_t total = npairs * tpp;
  if (!total) return;
  windows_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(plans, npairs, tpp, tile, rank, wins, nwin,
                                                                  merge_carry_cap(tile), flag_list, flag_count);
  count_launch();
}

// ------------------------------------------------------------ merge round
// One-bit masks of a warp's rounds: lane l < E covers window positions
// [seg0 + 32l, seg0 + 32l + 32); only positions < len and < t count.
template <int E>
__device__ __forceinline__ uint32_t round_mask(const StreamDesc& sd, uint64_t P0, uint32_t seg0, uint32_t len,
                                               uint64_t t, uint32_t lane) {
  uint32_t mword = 0;
  if (lane < (uint32_t)E) {
    uint32_t i = seg0 + lane * 32;
    if (i < len) {
      uint64_t p = P0 + i;
      if (p < t) {
        uint32_t nv = min(32u, len - i);
        uint64_t nt = t - p;
        if (nt < nv) nv = (uint32_t)nt;
        uint32_t b = (uint32_t)(bits64_at(sd, p) >> 32);
        mword = (nv == 32) ? b : (b & ~(0xffffffffu >> nv));
      }
    }
  }
  return mword;
}

// Phase B for one warp: ones take B[rank'] (from bbuf), their A element moves
// to the next window's buffer.  Lane-consecutive positions: conflict-free smem.
template <typename V, int E>
__device__ __forceinline__ void move_ones(V* Fc, V* Fn, const V* bbuf, uint32_t mword, uint32_t round_base,
                                          uint32_t before, uint32_t seg0, uint32_t len, uint32_t lane) {
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if (seg0 + 32 * k >= len) break;
    uint32_t m = __shfl_sync(0xffffffffu, mword, k);
    uint32_t rb = __shfl_sync(0xffffffffu, round_base, k);
    if ((m >> (31 - lane)) & 1u) {
      uint32_t i = seg0 + 32 * k + lane;
      uint32_t r = before + rb + __popc(m & ~(0xffffffffu >> lane));
      Fn[r] = Fc[i];
      Fc[i] = bbuf[r];
    }
  }
}

// Split a run of `cnt` elements at global address `src` into an unaligned
// head, a 16-byte aligned body (TMA bulk copy) and a tail; `off` is chosen so
// the body lands 16-byte aligned in shared memory.
template <typename V>
struct RunSplit {
  uint32_t head, body, tail;  // elements
};
template <typename V>
__device__ __forceinline__ RunSplit<V> split_run(const V* src, uint32_t cnt) {
  constexpr uint32_t VPA = 16 / sizeof(V);
  uint32_t mis = (uint32_t)((uintptr_t)src & 15);
  uint32_t head = ((16 - mis) & 15) / sizeof(V);
  RunSplit<V> r;
  if (head >= cnt) { r.head = cnt; r.body = 0; r.tail = 0; return r; }
  r.head = head;
  r.body = ((cnt - head) / VPA) * VPA;
  r.tail = cnt - head - r.body;
  return r;
}

// Sequential-window fallback (tiles flagged by windows_kernel): windows are
// walked one after the other, B runs of the stored windows prefetched by TMA.
template <typename V, int BLOCK, int E, int BCAP>
__device__ __noinline__ void merge_seq_tile(const uint64_t tile, const V* __restrict__ in, V* __restrict__ out,
                                            const PairPlan* __restrict__ plans, uint32_t tpp,
                                            const uint64_t* __restrict__ rank, const WinRec* __restrict__ wins,
                                            const uint32_t* __restrict__ nwin, unsigned char* smem_raw) {
  constexpr int T = BLOCK * E;
  constexpr uint32_t VPA = 16 / sizeof(V);
  constexpr uint32_t WSPAN = 32 * E;  // positions per warp
  constexpr uint32_t NOPF = 0xFFFFFFFFu;
  static_assert(E <= 32, "E bits are taken from one 64-bit window");
  V* bufA = reinterpret_cast<V*>(smem_raw);   // T + VPA (tile, misaligned start)
  V* bufB = bufA + T + VPA;                   // T
  V* bbuf = bufB + T;                         // BCAP: every window's B run
  __shared__ __align__(8) uint64_t mbar;
  __shared__ WinRec sw[kHMax];
  __shared__ uint32_t boff[kHMax];
  __shared__ uint32_t wsum[BLOCK / 32];
  __shared__ uint32_t a_off_s;
  __shared__ uint64_t o0_s;

  const uint32_t nw = nwin[tile] - (kHMax + 1);  // stored windows; later ones computed here
  const uint64_t g = tile / tpp;
  const PairPlan* Pp = plans + g;
  const uint64_t s = Pp->s, n1 = Pp->n1, t = Pp->t;
  const StreamDesc sd = Pp->sd;
  const uint64_t* R = rank + Pp->rank_off;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const V* pin = in + s;
  V* pout = out + s;

  // ---- prefetch: A tile + the B run of every stored window, one TMA batch
  if (tid < nw) sw[tid] = wins[tile * kHMax + tid];
  if (tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  const uint64_t u0 = sw[0].start;
  uint32_t len = (uint32_t)sw[0].len;
  if (tid == 0) {
    RunSplit<V> ra = split_run<V>(pin + u0, len);
    uint32_t aoff = (VPA - (ra.head % VPA)) % VPA;
    a_off_s = aoff;
    uint32_t tx = ra.body * sizeof(V);
    uint32_t cur = 0;
    for (uint32_t h = 0; h + 1 < nw; ++h) {
      uint32_t cnt = (uint32_t)sw[h + 1].len;
      RunSplit<V> rb = split_run<V>(pin + sw[h + 1].start, cnt);
      uint32_t off = ((cur + rb.head + VPA - 1) / VPA) * VPA - rb.head;
      if (off + cnt <= (uint32_t)BCAP) {
        boff[h] = off;
        cur = off + cnt;
        tx += rb.body * sizeof(V);
      } else {
        boff[h] = NOPF;
      }
    }
    mbar_arrive_expect_tx(&mbar, tx);
    if (ra.body) bulk_g2s(bufA + aoff + ra.head, pin + u0 + ra.head, ra.body * sizeof(V), &mbar);
    for (uint32_t h = 0; h + 1 < nw; ++h) {
      if (boff[h] == NOPF) continue;
      uint32_t cnt = (uint32_t)sw[h + 1].len;
      RunSplit<V> rb = split_run<V>(pin + sw[h + 1].start, cnt);
      if (rb.body)
        bulk_g2s(bbuf + boff[h] + rb.head, pin + sw[h + 1].start + rb.head, rb.body * sizeof(V), &mbar);
    }
  }
  __syncthreads();
  if (wid == 1) {  // unaligned heads/tails with plain loads
    for (uint32_t h = lane; h < nw; h += 32) {
      const V* src;
      V* dst;
      uint32_t cnt;
      if (h == 0) {
        src = pin + u0; dst = bufA + a_off_s; cnt = len;
      } else {
        if (boff[h - 1] == NOPF) continue;
        src = pin + sw[h].start; dst = bbuf + boff[h - 1]; cnt = (uint32_t)sw[h].len;
      }
      RunSplit<V> r = split_run<V>(src, cnt);
      for (uint32_t k = 0; k < r.head; ++k) dst[k] = src[k];
      for (uint32_t k = r.head + r.body; k < cnt; ++k) dst[k] = src[k];
    }
  }
  __syncthreads();
  mbar_wait(&mbar, 0);

  V* Fc = bufA + a_off_s;
  V* Fn = bufB;
  uint64_t P0 = u0;
  uint32_t h = 0;
  bool done = false;
  // ---- block mode: windows wider than one warp's span
  while (len > WSPAN) {
    const uint32_t seg0 = wid * WSPAN;
    uint32_t mword = round_mask<E>(sd, P0, seg0, len, t, lane);
    const uint32_t cnt = __popc(mword);
    uint32_t x = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    const uint32_t round_base = x - cnt;
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    uint32_t total = 0, before = 0;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) {
      uint32_t v = wsum[w];
      before += (w < (int)wid) ? v : 0u;
      total += v;
    }
    if (total == 0) {
      for (uint32_t i = tid; i < len; i += BLOCK) pout[P0 + i] = Fc[i];
      done = true;
      break;
    }
    uint64_t o0;
    const V* bsrc;
    if (h + 1 < nw) {
      o0 = sw[h + 1].start - n1;
      bsrc = (boff[h] != NOPF) ? (const V*)(bbuf + boff[h]) : pin + n1 + o0;
    } else {  // chain longer than kHMax: rank' computed here, B read from global
      if (tid == 0) o0_s = rank_bits(sd, R, P0 < t ? P0 : t);
      __syncthreads();
      o0 = o0_s;
      bsrc = pin + n1 + o0;
    }
    if (seg0 < len) move_ones<V, E>(Fc, Fn, bsrc, mword, round_base, before, seg0, len, lane);
    __syncthreads();
    for (uint32_t i = tid; i < len; i += BLOCK) pout[P0 + i] = Fc[i];
    P0 = n1 + o0;
    len = total;
    // the next window's first barrier orders these reads of Fc before the
    // next phase B rewrites it as Fn
    V* tmp = Fc; Fc = Fn; Fn = tmp;
    ++h;
  }
  if (done) return;
  __syncthreads();
  if (wid != 0) return;
  // ---- warp mode: the remaining (geometrically shrinking) windows, warp 0 only
  for (;;) {
    uint32_t mword = round_mask<E>(sd, P0, 0, len, t, lane);
    const uint32_t cnt = __popc(mword);
    uint32_t x = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    const uint32_t round_base = x - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
    if (total == 0) {
      for (uint32_t i = lane; i < len; i += 32) pout[P0 + i] = Fc[i];
      return;
    }
    uint64_t o0;
    const V* bsrc;
    if (h + 1 < nw) {
      o0 = sw[h + 1].start - n1;
      bsrc = (boff[h] != NOPF) ? (const V*)(bbuf + boff[h]) : pin + n1 + o0;
    } else {
      o0 = rank_bits(sd, R, P0 < t ? P0 : t);
      bsrc = pin + n1 + o0;
    }
    move_ones<V, E>(Fc, Fn, bsrc, mword, round_base, 0, 0, len, lane);
    __syncwarp();
    for (uint32_t i = lane; i < len; i += 32) pout[P0 + i] = Fc[i];
    P0 = n1 + o0;
    len = total;
    V* tmp = Fc; Fc = Fn; Fn = tmp;
    ++h;
    __syncwarp();
  }
}

template <typename V, int BLOCK, int E, int BCAP>
__global__ void __launch_bounds__(BLOCK) merge_level_seq_kernel(const V* __restrict__ in, V* __restrict__ out,
                                                                const PairPlan* __restrict__ plans, uint32_t tpp,
                                                                const uint64_t* __restrict__ rank,
                                                                const WinRec* __restrict__ wins,
                                                                const uint32_t* __restrict__ nwin,
                                                                const uint32_t* __restrict__ flag_list,
                                                                const uint32_t* __restrict__ flag_count) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const uint32_t nf = *flag_count;
  for (uint32_t k = blockIdx.x; k < nf; k += gridDim.x) {
    merge_seq_tile<V, BLOCK, E, BCAP>(flag_list[k], in, out, plans, tpp, rank, wins, nwin, smem_raw);
    __syncthreads();
  }
}

// All windows of a tile at once.  The plan fixes every window's position range,
// so every window's bits are known up front: window h's k-th one-bit carries
// the element at sel_h[k] (its position in window h) into window h+1, position
// k.  A zero at position i of window h therefore outputs
// A[sel_0[sel_1[... sel_{h-1}[i]]]] (mean chain length 0.5), a one outputs
// window h's k-th B element.  Phases (each over all windows, block-parallel):
// TMA prefetch -> bit masks + segmented rank scan -> sel scatter -> outputs.
template <typename V, int BLOCK, int T, int BCAP>
__global__ void __launch_bounds__(BLOCK) merge_level_kernel(const V* __restrict__ in, V* __restrict__ out,
                                                            const PairPlan* __restrict__ plans, uint32_t tpp,
                                                            const WinRec* __restrict__ wins,
                                                            const uint32_t* __restrict__ nwin) {
  constexpr uint32_t VPA = 16 / sizeof(V);
  constexpr uint32_t NOPF = 0xFFFFFFFFu;
  constexpr int MAXCH = (T + BCAP) / 32 + kHMax;  // 32-position chunks over all windows
  constexpr int CPT = (MAXCH + BLOCK - 1) / BLOCK;
  constexpr int BBUF = BCAP + 2 * VPA * kHMax;      // B runs incl. alignment padding
  extern __shared__ __align__(128) unsigned char smem_raw[];
  V* bufA = reinterpret_cast<V*>(smem_raw);    // T + VPA: the A tile
  V* bbuf = bufA + T + VPA;                    // BBUF: B run of every window
  uint16_t* sel = reinterpret_cast<uint16_t*>(bbuf + BBUF);  // BCAP
  uint32_t* cmask = reinterpret_cast<uint32_t*>(sel + BCAP);  // MAXCH one-bit masks
  uint32_t* cinfo = cmask + MAXCH;                            // MAXCH (window << 16 | chunk in window)
  uint32_t* crank = cinfo + MAXCH;                            // MAXCH window rank of first one
  __shared__ __align__(8) uint64_t mbar;
  __shared__ WinRec sw[kHMax];
  __shared__ uint32_t boff[kHMax];
  __shared__ uint32_t cbase[kHMax + 1];   // first chunk of window h
  __shared__ uint32_t sbase[kHMax + 1];   // first sel slot of window h
  __shared__ uint32_t wsum[BLOCK / 32];
  __shared__ uint32_t a_off_s;

  const uint64_t tile = blockIdx.x;
  const uint32_t nw = nwin[tile];
  if (nw == 0 || nw > (uint32_t)kHMax) return;
  const PairPlan* Pp = plans + tile / tpp;
  const uint64_t s = Pp->s, t = Pp->t;
  const StreamDesc sd = Pp->sd;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const V* pin = in + s;
  V* pout = out + s;

  if (tid < nw) sw[tid] = wins[tile * kHMax + tid];
  if (tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (wid == 0) {
    // warp 0 lays out the runs (lane owns windows lane and lane+32): chunk
    // bases, sel bases and padded B-run slots by warp scans, then every lane
    // issues its own TMA bulk copies and plain head/tail loads.
    uint32_t carry_c = 0, carry_s = 0, carry_b = 0, tx = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t h = lane + 32 * q;
      const bool valid = h < nw;
      const uint32_t lh = valid ? (uint32_t)sw[h].len : 0u;
      const uint32_t nchh = (lh + 31) / 32;
      const uint32_t cnt = (valid && h + 1 < nw) ? (uint32_t)sw[h + 1].len : 0u;
      RunSplit<V> rb = split_run<V>(pin + (cnt ? sw[h + 1].start : 0), cnt);
      const uint32_t slot = cnt ? ((cnt + 2 * VPA - 1) / VPA) * VPA : 0u;
      uint32_t xc = nchh, xs = cnt, xb = slot;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t yc = __shfl_up_sync(0xffffffffu, xc, o);
        uint32_t ys = __shfl_up_sync(0xffffffffu, xs, o);
        uint32_t yb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= (uint32_t)o) { xc += yc; xs += ys; xb += yb; }
      }
      const uint32_t cb = carry_c + xc - nchh, sb = carry_s + xs - cnt, bs = carry_b + xb - slot;
      if (valid) {
        cbase[h] = cb;
        sbase[h] = sb;
        uint32_t off = NOPF;
        if (cnt && bs + slot <= (uint32_t)BBUF) {
          off = bs + (VPA - (rb.head % VPA)) % VPA;
          tx += rb.body * sizeof(V);
        }
        boff[h] = off;
        if (h == nw - 1) { cbase[nw] = cb + nchh; sbase[nw] = sb + cnt; }
      }
      carry_c += __shfl_sync(0xffffffffu, xc, 31);
      carry_s += __shfl_sync(0xffffffffu, xs, 31);
      carry_b += __shfl_sync(0xffffffffu, xb, 31);
    }
    const uint32_t len0 = (uint32_t)sw[0].len;
    RunSplit<V> ra = split_run<V>(pin + sw[0].start, len0);
    const uint32_t aoff = (VPA - (ra.head % VPA)) % VPA;
    if (lane == 0) tx += ra.body * sizeof(V);
    for (int o = 16; o; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
    if (lane == 0) {
      a_off_s = aoff;
      mbar_arrive_expect_tx(&mbar, tx);
      if (ra.body) bulk_g2s(bufA + aoff + ra.head, pin + sw[0].start + ra.head, ra.body * sizeof(V), &mbar);
    }
    __syncwarp();
    if (lane < ra.head) bufA[aoff + lane] = pin[sw[0].start + lane];
    for (uint32_t k = ra.head + ra.body + lane; k < len0; k += 32) bufA[aoff + k] = pin[sw[0].start + k];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t h = lane + 32 * q;
      if (h + 1 < nw && boff[h] != NOPF) {
        const uint32_t cnt = (uint32_t)sw[h + 1].len;
        const V* src = pin + sw[h + 1].start;
        V* dst = bbuf + boff[h];
        RunSplit<V> rb = split_run<V>(src, cnt);
        if (rb.body) bulk_g2s(dst + rb.head, src + rb.head, rb.body * sizeof(V), &mbar);
        for (uint32_t k = 0; k < rb.head; ++k) dst[k] = src[k];
        for (uint32_t k = rb.head + rb.body; k < cnt; ++k) dst[k] = src[k];
      }
    }
  }
  __syncthreads();
  const uint32_t nch = cbase[nw];
  // ---- bit masks of every chunk (positions >= t count as zeros) + rank scan.
  // Thread tid owns chunks [tid*CPT, tid*CPT+CPT) (contiguous, so the window
  // index only moves forward).
  uint32_t csum[CPT];
  uint32_t tsum = 0;
  uint32_t h = 0;
  {
    const uint32_t c0 = tid * CPT;
    uint32_t lo = 0, hi = nw;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (cbase[mid] <= c0) lo = mid; else hi = mid;
    }
    h = lo;
  }
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const uint32_t c = tid * CPT + q;
    uint32_t m = 0;
    if (c < nch) {
      while (cbase[h + 1] <= c) ++h;
      const uint32_t i0 = (c - cbase[h]) * 32;
      const uint64_t p = sw[h].start + i0;
      if (p < t) {
        uint32_t nv = min(32u, (uint32_t)sw[h].len - i0);
        uint64_t nt = t - p;
        if (nt < nv) nv = (uint32_t)nt;
        uint32_t b = (uint32_t)(bits64_at(sd, p) >> 32);
        m = (nv == 32) ? b : (b & ~(0xffffffffu >> nv));
      }
      cmask[c] = m;
    }
    csum[q] = __popc(m);
    tsum += csum[q];
  }
  uint32_t x = tsum;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  {
    uint32_t run = x - tsum;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) run += (w < (int)wid) ? wsum[w] : 0u;
    // per chunk: (window, chunk-in-window) and the window rank of its first one
    // (ones before window h == sbase[h], fixed by the plan)
    uint32_t hh;
    const uint32_t c0 = tid * CPT;
    uint32_t lo = 0, hi = nw;
    while (hi - lo > 1) {
      uint32_t mid = (lo + hi) >> 1;
      if (cbase[mid] <= c0) lo = mid; else hi = mid;
    }
    hh = lo;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const uint32_t c = c0 + q;
      if (c < nch) {
        while (cbase[hh + 1] <= c) ++hh;
        cinfo[c] = (hh << 16) | (c - cbase[hh]);
        crank[c] = run - sbase[hh];
      }
      run += csum[q];
    }
  }
  __syncthreads();
  // ---- sel scatter: window h's r-th one sits at position i of window h
  const uint32_t ltmask = ~(0xffffffffu >> lane);  // lanes before this one (MSB-first)
  for (uint32_t c = wid; c < nch; c += BLOCK / 32) {
    const uint32_t m = cmask[c];
    if ((m >> (31 - lane)) & 1u) {
      const uint32_t info = cinfo[c];
      const uint32_t r = crank[c] + __popc(m & ltmask);
      sel[sbase[info >> 16] + r] = (uint16_t)(((info & 0xFFFFu) << 5) + lane);
    }
  }
  __syncthreads();
  mbar_wait(&mbar, 0);
  // ---- outputs: one warp per chunk (window uniform across the warp), both the
  // one-path (B element) and the zero-path (A element through the sel chain)
  // evaluated branch-free, one coalesced store per lane.
  const V* Fa = bufA + a_off_s;
  for (uint32_t c = wid; c < nch; c += BLOCK / 32) {
    const uint32_t info = cinfo[c];
    const uint32_t hw = info >> 16;
    const uint32_t i = ((info & 0xFFFFu) << 5) + lane;
    const uint32_t lh = (uint32_t)sw[hw].len;
    const uint32_t m = cmask[c];
    const bool inb = i < lh;
    const bool one = (m >> (31 - lane)) & 1u;
    uint32_t r = inb ? i : lh - 1;
    for (int k = (int)hw - 1; k >= 0; --k) r = sel[sbase[k] + r];
    const V vz = Fa[r];
    const uint32_t ro = crank[c] + __popc(m & ltmask);
    const uint32_t bo = boff[hw];
    V vo = vz;
    if (bo != NOPF) vo = bbuf[bo + ro];
    else if (one && inb) vo = pin[sw[hw + 1].start + ro];
    if (inb) pout[sw[hw].start + i] = one ? vo : vz;
  }
}

constexpr int kMergeBlock = 256;
constexpr int kE32 = 16;  // 4096-element tiles for 4-byte payloads
constexpr int kE64 = 8;   // 2048-element tiles for 8-byte payloads

uint32_t merge_tile(int eb) { return kMergeBlock * (eb == 4 ? kE32 : kE64); }

uint64_t merge_carry_cap(uint32_t tile) { return tile + tile / 4; }

template <typename V, int E>
static void merge_level_t(const void* in, void* out, const PairPlan* plans, uint64_t npairs, uint32_t tpp,
                          const uint64_t* rank, const WinRec* wins, const uint32_t* nwin, const uint32_t* flag_list,
                          const uint32_t* flag_count, cudaStream_t st) {
  uint64_t tiles = npairs * tpp;
  if (!tiles) return;
  constexpr int T = kMergeBlock * E;
  constexpr int BCAP = T + T / 4;  // == merge_carry_cap(T)
  constexpr int MAXCH = (T + BCAP) / 32 + kHMax;
  {
    constexpr int BBUF = BCAP + 2 * (16 / sizeof(V)) * kHMax;
    size_t smem = (size_t)(T + 16 / sizeof(V) + BBUF) * sizeof(V) + (size_t)BCAP * 2 + (size_t)MAXCH * 12;
    auto k = merge_level_kernel<V, kMergeBlock, T, BCAP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<(unsigned)tiles, kMergeBlock, smem, st>>>((const V*)in, (V*)out, plans, tpp, wins, nwin);
    count_launch();
  }
  {
    size_t smem = (size_t)(T + 16 / sizeof(V) + T + BCAP) * sizeof(V);
    auto k = merge_level_seq_kernel<V, kMergeBlock, E, BCAP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned g = (unsigned)std::min<uint64_t>(tiles, (uint64_t)num_sms() * 2);
    k<<<g, kMergeBlock, smem, st>>>((const V*)in, (V*)out, plans, tpp, rank, wins, nwin, flag_list, flag_count);
    count_launch();
  }
}

void launch_merge_level(int eb, const void* in, void* out, const PairPlan* plans, uint64_t npairs, uint32_t tpp,
                        const uint64_t* rank, const WinRec* wins, const uint32_t* nwin, const uint32_t* flag_list,
                        const uint32_t* flag_count, cudaStream_t st) {
  if (eb == 4) merge_level_t<uint32_t, kE32>(in, out, plans, npairs, tpp, rank, wins, nwin, flag_list, flag_count, st);
  else merge_level_t<unsigned long long, kE64>(in, out, plans, npairs, tpp, rank, wins, nwin, flag_list, flag_count,
                                               st);
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
__global__ void iota32_kernel(uint32_t* v, uint64_t n) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}
void launch_iota32(uint32_t* v, uint64_t n, cudaStream_t st) {
  if (!n) return;
  iota32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v, n);
  count_launch();
}

// Over records sorted by target (stable in x): predecessor in the target's
// group, and for each group's last step x_last > q the output (q <- x_last).
__global__ void tail_plan_kernel(const PairPlan* __restrict__ plans, const uint64_t* __restrict__ rec_key,
                                 const uint32_t* __restrict__ rec_pair, const uint64_t* __restrict__ skey,
                                 const uint32_t* __restrict__ sval, uint64_t total, uint64_t* __restrict__ predx,
                                 uint8_t* __restrict__ keyed, uint64_t* __restrict__ dst, uint64_t* __restrict__ src) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= total) return;
  uint32_t rec = sval[k];
  uint64_t key = skey[k];
  const PairPlan* P = plans + rec_pair[rec];
  uint64_t loc = rec - P->tail_off, x = P->t + loc;
  predx[rec] = (k > 0 && skey[k - 1] == key) ? (P->t + (sval[k - 1] - P->tail_off)) : kNone;
  bool last = (k + 1 == total) || skey[k + 1] != key;
  if (last) {
    uint64_t q = key - P->s;
    if (x > q) {
      uint64_t slot = 2 * P->tail_off + P->tail_len + loc;
      dst[slot] = key;
      src[slot] = P->s + x;
      if (q >= P->t) keyed[P->tail_off + (q - P->t)] = 1;
    }
  }
  (void)rec_key;
}

// For every insertion position x not overwritten later: chase V(m_x, x).
__global__ void tail_chase_kernel(const PairPlan* __restrict__ plans, const uint64_t* __restrict__ rec_key,
                                  const uint32_t* __restrict__ rec_pair, const uint64_t* __restrict__ predx,
                                  const uint8_t* __restrict__ keyed, uint64_t total, uint64_t* __restrict__ dst,
                                  uint64_t* __restrict__ src) {
  uint64_t rec = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rec >= total) return;
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

void launch_tail_plan(const PairPlan* plans, const uint64_t* rec_key, const uint32_t* rec_pair,
                      const uint64_t* skey, const uint32_t* sval, uint64_t total, uint64_t* predx,
                      uint8_t* keyed, uint64_t* dst, uint64_t* src, cudaStream_t st) {
  if (!total) return;
  tail_plan_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(plans, rec_key, rec_pair, skey, sval, total,
                                                                    predx, keyed, dst, src);
  count_launch();
}

void launch_tail_chase(const PairPlan* plans, const uint64_t* rec_key, const uint32_t* rec_pair,
                       const uint64_t* predx, const uint8_t* keyed, uint64_t total, uint64_t* dst, uint64_t* src,
                       cudaStream_t st) {
  if (!total) return;
  tail_chase_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(plans, rec_key, rec_pair, predx, keyed, total,
                                                                     dst, src);
  count_launch();
}

// ------------------------------------------------------------ tail apply
template <typename V>
__global__ void tail_gather_kernel(const V* __restrict__ buf, const uint64_t* __restrict__ dst,
                                   const uint64_t* __restrict__ src, V* __restrict__ tmp, uint64_t n) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && dst[k] != kNone) tmp[k] = buf[src[k]];
}
template <typename V>
__global__ void tail_scatter_kernel(V* __restrict__ buf, const uint64_t* __restrict__ dst,
                                    const V* __restrict__ tmp, uint64_t n) {
  uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && dst[k] != kNone) buf[dst[k]] = tmp[k];
}

void launch_tail_apply(int eb, void* buf, const uint64_t* dst, const uint64_t* src, void* tmp, uint64_t nslots,
                       cudaStream_t st) {
  if (!nslots) return;
  unsigned b = (unsigned)((nslots + 255) / 256);
  if (eb == 4) {
    tail_gather_kernel<uint32_t><<<b, 256, 0, st>>>((const uint32_t*)buf, dst, src, (uint32_t*)tmp, nslots);
    tail_scatter_kernel<uint32_t><<<b, 256, 0, st>>>((uint32_t*)buf, dst, (const uint32_t*)tmp, nslots);
  } else {
    tail_gather_kernel<unsigned long long><<<b, 256, 0, st>>>((const unsigned long long*)buf, dst, src,
                                                              (unsigned long long*)tmp, nslots);
    tail_scatter_kernel<unsigned long long><<<b, 256, 0, st>>>((unsigned long long*)buf, dst,
                                                               (const unsigned long long*)tmp, nslots);
  }
  count_launch();
  count_launch();
}

}  // namespace sk
