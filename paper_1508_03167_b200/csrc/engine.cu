// engine.cu -- orchestration of the B200 MergeShuffle pipeline and the C ABI.
//
// Data path (caller stream):   leaf decode -> leaf apply -> round 1 .. round c
//   (round = window gather kernel, identity region, tail gather/scatter),
//   ping-ponging between the caller's buffer and one O(n) scratch buffer.
// Plan path (side stream, data independent, overlaps the leaf stage):
//   per round: superblock rank tables -> stop points / X -> window chains;
//   then one launch decodes every pair's tail draws (all rounds at once),
//   then per round: radix sort of tail targets -> (dst, src) tail plan.
// Reference driver: shufflers.py:251-299 / _kernels.py:253-289.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cmath>

#include "../../include/shufflekit_b200.h"
#include "sk_kernels.h"

namespace sk {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local std::string g_err;
static void set_err(const std::string& s) { g_err = s; }

int num_sms() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

struct CudaError {
  int code;
};

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      set_err(std::string(#expr) + ": " + cudaGetErrorString(e_));                            \
      throw CudaError{e_ == cudaErrorMemoryAllocation ? SK_ENOMEM : SK_ECUDA};                \
    }                                                                                         \
  } while (0)

// ------------------------------------------------------------------ profiling
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static constexpr int kStages = 5;
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof;
static uint64_t g_prof_launch[kStages];

struct StageTimer {
  int stage;
  cudaStream_t st;
  cudaEvent_t a{}, b{};
  uint64_t l0;
  bool on;
  StageTimer(int s, cudaStream_t stream) : stage(s), st(stream), l0(g_launches.load()), on(g_prof_on) {
    if (on) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~StageTimer() {
    if (on) {
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_prof_mu);
      g_prof.push_back({stage, a, b});
      g_prof_launch[stage] += g_launches.load() - l0;
    }
  }
};

// ------------------------------------------------------------ device memory
// Keep freed stream-ordered memory in the current device's pool (repeated
// calls reuse it instead of returning it to the driver); once per device.
static void setup_pool_once() {
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && (done >> dev & 1)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (dev < 64) done |= 1ull << dev;
}

// All allocations of one call; freed stream-ordered on the data stream.
struct Arena {
  std::vector<void*> ptrs;
  template <typename T>
  T* alloc(size_t count, cudaStream_t st) {
    if (count == 0) count = 1;
    void* p = nullptr;
    CK(cudaMallocAsync(&p, count * sizeof(T), st));
    ptrs.push_back(p);
    return (T*)p;
  }
  void release(cudaStream_t st) {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    ptrs.clear();
  }
};

static int plan_c(uint64_t n, uint64_t cutoff) {
  int c = 0;
  while ((n >> c) > cutoff) ++c;
  return c;
}

struct LevelBufs {
  LevelJob LJ;
  uint64_t sbs = 0, npairs = 0;
  uint64_t* rank = nullptr;
  PairPlan* plans = nullptr;
  uint64_t* chains = nullptr;               // per tile: window starts of the tree merge
  uint32_t tpp = 1;                          // tree tiles per pair
  // tails: `cap` record slots (host bound), *used of them filled (device)
  uint64_t cap = 0;
  uint64_t* used = nullptr;
  uint64_t* rec_key = nullptr;
  uint32_t* rec_pair = nullptr;
  uint64_t* predx = nullptr;
  uint8_t* keyed = nullptr;
  uint64_t* hkey = nullptr;                  // target -> chain of its records
  uint32_t* hhead = nullptr;
  uint32_t* next = nullptr;
  uint32_t* slot_of = nullptr;
  uint32_t hmask = 0;
  uint64_t* dst = nullptr;                   // 2 * cap (dst, src) slots
  uint64_t* src = nullptr;
  void* tmp = nullptr;
  cudaEvent_t ev_chain{};                    // plans + window chains of this round done (plan stream)
  cudaEvent_t ev_tail{};                     // tail (dst, src) done
};

// Record capacity of a round's tail buffers, from the pair geometry alone (no
// device data, no host synchronization): the tail of a pair of N elements has
// L = N - t insertions with mean 0.80 sqrt(N) and variance 0.37 N (|random
// walk| at the stop point; measured: tests/test_host_logic.py).  Mean + 9
// standard deviations of the round's sum, + 4096: a pair beyond it (never
// seen) falls back to the serial tail (PairPlan.tail_slow), still exact.
static uint64_t tail_capacity(const LevelJob& LJ) {
  double mean = 0, var = 0;
  for (uint64_t g = 0; g < LJ.npairs; ++g) {
    uint64_t s, n1, n2, array;
    StreamDesc sd;
    pair_geom(LJ, g, s, n1, n2, sd, array);
    if (!n1 || !n2) continue;
    const double N = (double)(n1 + n2);
    mean += 0.80 * std::sqrt(N);
    var += 0.37 * N;
  }
  return (uint64_t)(mean + 9.0 * std::sqrt(var)) + 4096;
}

// Small host->device uploads as kernel parameters (no copy engine).
struct PokeBuf {
  unsigned char b[2048];
};
__global__ void poke_kernel(unsigned char* dst, PokeBuf p, uint32_t n) {
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = p.b[i];
}
static void poke(void* dst, const void* src, size_t n, cudaStream_t st) {
  for (size_t o = 0; o < n; o += sizeof(PokeBuf)) {
    PokeBuf p;
    const size_t k = std::min(sizeof(PokeBuf), n - o);
    memcpy(p.b, (const unsigned char*)src + o, k);
    poke_kernel<<<1, 256, 0, st>>>((unsigned char*)dst + o, p, (uint32_t)k);
    count_launch();
  }
}

// Order `ps` after everything queued on `st` so far (allocations, bit counters).
static void fork_side(cudaStream_t st, cudaStream_t ps) {
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventRecord(ev, st));
  CK(cudaStreamWaitEvent(ps, ev, 0));
  cudaEventDestroy(ev);
}

// Build every round's plan on `ps`, all on the device (no host
// synchronization, no host->device copies: on the host entry those would queue
// behind the big H2D transfer): per round the rank tables, stop points and
// window chains (then lv[r].ev_chain), the tail offsets; one launch decodes
// every pair's tail draws; per round the (dst, src) tail plan (then
// lv[r].ev_tail).
static cudaStream_t side_stream2();
static int g_plan_streams = 2;  // 1: every round's plan on one side stream (debug knob)

static void build_plans(std::vector<LevelBufs>& lv, int eb, unsigned long long* d_bits, Arena& A, cudaStream_t ps) {
  const int nl = (int)lv.size();
  // The rounds' plans are independent of one another until the tail draws, and
  // their kernels are small: odd rounds go to a second side stream (forked
  // from `ps` after the allocations, joined before the tail decode and again
  // at the end), so the two streams fill each other's launch gaps and tails
  // while the leaf decode holds its one warp per scheduler.
  cudaStream_t ps2 = g_plan_streams > 1 && nl > 1 ? side_stream2() : ps;
  std::vector<uint64_t*> csum(nl);
  for (int i = 0; i < nl; ++i) {
    auto& L = lv[i];
    L.rank = A.alloc<uint64_t>(L.npairs * L.sbs, ps);
    L.plans = A.alloc<PairPlan>(L.npairs, ps);
    L.chains = A.alloc<uint64_t>(tree_chain_words(L.npairs, L.tpp), ps);
    L.used = A.alloc<uint64_t>(1, ps);
    csum[i] = A.alloc<uint64_t>(rank_scan_scratch(L.npairs, L.sbs), ps);
    CK(cudaEventCreateWithFlags(&L.ev_chain, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&L.ev_tail, cudaEventDisableTiming));
  }
  if (ps2 != ps) fork_side(ps, ps2);
  for (int i = 0; i < nl; ++i) {
    auto& L = lv[i];
    cudaStream_t s = (i & 1) ? ps2 : ps;
    launch_rank_tables(L.LJ, L.sbs, L.rank, csum[i], s);
    launch_pair_plan(L.LJ, L.sbs, L.rank, L.plans, s);
    launch_tree_chains(eb, L.plans, L.npairs, L.rank, L.tpp, L.chains, s);
    CK(cudaEventRecord(L.ev_chain, s));
  }
  if (ps2 != ps) fork_side(ps2, ps);  // the tail decode reads every round's plans
  uint64_t tot_pairs = 0;
  std::vector<uint64_t> pprefix(nl + 1, 0);
  std::vector<LevelTail> ht(nl);
  for (int i = 0; i < nl; ++i) {
    auto& L = lv[i];
    pprefix[i] = tot_pairs;
    tot_pairs += L.npairs;
    L.cap = tail_capacity(L.LJ);
    launch_tail_offsets(L.plans, L.npairs, L.cap, L.used, ps);
    L.rec_key = A.alloc<uint64_t>(L.cap, ps);
    L.rec_pair = A.alloc<uint32_t>(L.cap, ps);
    ht[i] = LevelTail{L.plans, L.npairs, L.rec_key, L.rec_pair};
  }
  pprefix[nl] = tot_pairs;
  LevelTail* d_lt = A.alloc<LevelTail>(nl, ps);
  uint64_t* d_pp = A.alloc<uint64_t>(nl + 1, ps);
  poke(d_lt, ht.data(), nl * sizeof(LevelTail), ps);
  poke(d_pp, pprefix.data(), (nl + 1) * 8, ps);
  launch_tail_decode(d_lt, nl, d_pp, tot_pairs, d_bits, ps);
  for (auto& L : lv) {  // (allocations first: they are ordered on `ps`)
    uint32_t hb = 1;
    while ((1ull << hb) < 2 * L.cap) ++hb;
    L.hmask = (uint32_t)((1ull << hb) - 1);
    L.hkey = A.alloc<uint64_t>(1ull << hb, ps);
    L.hhead = A.alloc<uint32_t>(1ull << hb, ps);
    L.next = A.alloc<uint32_t>(L.cap, ps);
    L.slot_of = A.alloc<uint32_t>(L.cap, ps);
    L.predx = A.alloc<uint64_t>(L.cap, ps);
    L.keyed = A.alloc<uint8_t>(L.cap, ps);
    L.dst = A.alloc<uint64_t>(2 * L.cap, ps);
    L.src = A.alloc<uint64_t>(2 * L.cap, ps);
    L.tmp = A.alloc<uint64_t>(2 * L.cap, ps);
  }
  if (ps2 != ps) fork_side(ps, ps2);
  for (int i = 0; i < nl; ++i) {
    auto& L = lv[i];
    cudaStream_t s = (i & 1) ? ps2 : ps;
    const uint64_t hsz = (uint64_t)L.hmask + 1;
    CK(cudaMemsetAsync(L.hkey, 0xFF, 8 * hsz, s));
    CK(cudaMemsetAsync(L.hhead, 0xFF, 4 * hsz, s));
    CK(cudaMemsetAsync(L.keyed, 0, L.cap, s));
    CK(cudaMemsetAsync(L.dst, 0xFF, 2 * L.cap * 8, s));
    launch_tail_plan(L.plans, L.rec_key, L.rec_pair, L.used, L.cap, L.hkey, L.hhead, L.next, L.slot_of, L.hmask,
                     L.predx, L.keyed, L.dst, L.src, s);
    launch_tail_chase(L.plans, L.rec_key, L.rec_pair, L.predx, L.keyed, L.used, L.cap, L.dst, L.src, s);
    CK(cudaEventRecord(L.ev_tail, s));
  }
  if (ps2 != ps) fork_side(ps2, ps);  // callers wait for `ps` before releasing the arena
  CK(cudaGetLastError());
}

static void destroy_events(std::vector<LevelBufs>& lv) {
  for (auto& L : lv) {
    if (L.ev_chain) cudaEventDestroy(L.ev_chain);
    if (L.ev_tail) cudaEventDestroy(L.ev_tail);
    L.ev_chain = L.ev_tail = nullptr;
  }
}

// Helper streams of the calling thread on the CURRENT device (a thread may
// drive several devices in turn): plan, round and copy streams, created on
// first use per device.
enum HelperStream { kPlanStream = 0, kRoundStream = 1, kCopyStream = 2, kPlanStream2 = 3 };
constexpr int kMaxDevices = 64;
struct HelperStreams {
  cudaStream_t s[4][kMaxDevices] = {};
  ~HelperStreams() {
    for (auto& row : s)
      for (cudaStream_t x : row)
        if (x) cudaStreamDestroy(x);
  }
};

static cudaStream_t helper_stream(HelperStream which) {
  static thread_local HelperStreams hs;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw std::runtime_error("device ordinal out of range");
  cudaStream_t& s = hs.s[which][dev];
  if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

static cudaStream_t side_stream() { return helper_stream(kPlanStream); }
static cudaStream_t side_stream2() { return helper_stream(kPlanStream2); }

// Run rounds 1..c over `cur` (data currently there); the result lands in
// `other`.  The tree merge reads every window of a CTA before writing it back
// (and CTAs own disjoint windows), so rounds 1..c-1 run in place on `cur`
// and only the last round writes `other` (plus the untouched [X, N) regions).
// The segment-pass debug kernels park elements in their input and need the
// ping-pong.  Returns the buffer holding the result.
// Pairs [p0, p1) of one round, in place (tree merge), with their tail insertions.
// (positions [lo, hi) = the pairs' elements: the tail slots are filtered by it)
static void run_round_range(LevelBufs& L, int eb, void* buf, uint64_t p0, uint64_t p1, uint64_t lo, uint64_t hi,
                            cudaStream_t st) {
  {
    StageTimer tm(2, st);
    CK(cudaStreamWaitEvent(st, L.ev_chain, 0));
    launch_merge_tree_range(eb, buf, buf, L.plans, p0, p1, L.rank, L.chains, L.tpp, st);
  }
  StageTimer tm(3, st);
  CK(cudaStreamWaitEvent(st, L.ev_tail, 0));
  launch_tail_apply(eb, buf, L.dst, L.src, L.tmp, 2 * L.cap, L.plans, L.npairs, lo, hi, st);
}

static void* run_rounds(std::vector<LevelBufs>& lv, int eb, void* cur, void* other, cudaStream_t st,
                        size_t first = 0) {
  for (size_t r = first; r < lv.size(); ++r) {
    auto& L = lv[r];
    void* out = r + 1 == lv.size() ? other : cur;
    {
      StageTimer tm(2, st);
      CK(cudaStreamWaitEvent(st, L.ev_chain, 0));
      launch_merge_tree(eb, cur, out, L.plans, L.npairs, L.rank, L.chains, L.tpp, st);
    }
    {
      StageTimer tm(3, st);
      if (out != cur) launch_copy_tail_region(eb, cur, out, L.plans, L.npairs, st);
      CK(cudaStreamWaitEvent(st, L.ev_tail, 0));
      launch_tail_apply(eb, out, L.dst, L.src, L.tmp, 2 * L.cap, L.plans, L.npairs, 0, ~0ull, st);
    }
    if (out != cur) std::swap(cur, other);
  }
  CK(cudaGetLastError());
  return cur;
}

static std::vector<LevelBufs> make_levels(const ArrayJob& J, int eb) {
  std::vector<LevelBufs> lv;
  for (int r = 1; r <= J.rmax; ++r) {
    LevelBufs L;
    L.LJ.J = J;
    L.LJ.E = ExplicitTask{};
    L.LJ.r = r;
    L.npairs = J.batch << (J.lognblk - r);
    L.LJ.npairs = L.npairs;
    L.tpp = tree_tiles_per_pair(L.LJ, eb);
    uint64_t Nmax = (J.len >> (J.c - r)) + 2;
    L.sbs = (Nmax + 1 + 511) / 512 + 1;
    lv.push_back(L);
  }
  return lv;
}

// The whole tasked schedule for a batch of arrays (batch = 1: one array).
static void run_job(int eb, void* data, const ArrayJob& J, unsigned long long* d_bits, cudaStream_t st) {
  const uint64_t ntot = (J.lognblk == J.c && J.blk0 == 0)
                            ? J.batch * J.len
                            : bound_at(J.len, J.blk0 + (1ULL << J.lognblk), J.c) - bound_at(J.len, J.blk0, J.c);
  if (ntot == 0) return;
  setup_pool_once();
  Arena A;
  cudaStream_t ps = side_stream();
  std::vector<LevelBufs> lv = make_levels(J, eb);
  void* scratch = A.alloc<unsigned char>(ntot * eb, st);
  const uint64_t nleaves = J.batch << J.lognblk;
  const uint64_t mmax = (J.len + J.q - 1) >> J.c;  // largest leaf: ceil(len / q)
  ExplicitTask E0{};
  try {
    uint16_t* draws = nullptr;
    uint16_t* lscr = nullptr;
    uint32_t grid = 0;
    bool fast_leaf = mmax <= 65536;
    if (fast_leaf) {
      draws = A.alloc<uint16_t>(ntot, st);
      grid = leaf_apply_grid(nleaves, (uint32_t)mmax, num_sms(), eb);
      lscr = A.alloc<uint16_t>((uint64_t)grid * leaf_scratch_stride(mmax) + 8, st);
    }
    fork_side(st, ps);
    {
      StageTimer tm(0, st);
      if (fast_leaf) launch_leaf_decode16(J, E0, nleaves, draws, d_bits, st);
    }
    void* cur = nullptr;
    {
      StageTimer tm(1, st);
      if (fast_leaf && lv.empty() && mmax <= 8192) {
        // no merge rounds and small leaves: staged in shared memory, in place
        launch_leaf_apply(eb, J, E0, nleaves, data, data, draws, lscr, (uint32_t)mmax, grid, st);
        cur = data;
      } else if (fast_leaf) {
        launch_leaf_apply(eb, J, E0, nleaves, data, scratch, draws, lscr, (uint32_t)mmax, grid, st);
      } else {
        CK(cudaMemcpyAsync(scratch, data, ntot * eb, cudaMemcpyDeviceToDevice, st));
        launch_leaf_serial(eb, J, E0, nleaves, scratch, d_bits, st);
      }
      if (cur != data) cur = scratch;
    }
    CK(cudaGetLastError());
    // plans run on the side stream while the leaf stage runs
    if (!lv.empty()) build_plans(lv, eb, d_bits, A, ps);
    void* res = run_rounds(lv, eb, cur, data, st);
    if (res != data) {
      StageTimer tm(4, st);
      CK(cudaMemcpyAsync(data, res, ntot * eb, cudaMemcpyDeviceToDevice, st));
    }
  } catch (...) {
    cudaStreamSynchronize(ps);
    cudaStreamSynchronize(st);
    destroy_events(lv);
    A.release(st);
    throw;
  }
  cudaEvent_t done;
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventRecord(done, ps));
  CK(cudaStreamWaitEvent(st, done, 0));
  cudaEventDestroy(done);
  destroy_events(lv);
  A.release(st);
}

static cudaStream_t round_stream() { return helper_stream(kRoundStream); }
static cudaStream_t copy_stream() { return helper_stream(kCopyStream); }

// The host entry for big arrays: the H2D copy runs in 2^k chunks on a copy
// stream; the leaf draws (no data needed) and the merge plans are prepared
// meanwhile, chunk j's leaves are applied as soon as chunk j has landed, and
// its local rounds (1 .. c-k: pairs inside the chunk) follow on a round
// stream, so everything but the top k rounds hides under the transfer.  Then
// the top rounds, then the D2H copy.  Same result as copy +
// sk_merge_shuffle_parallel + copy.  (build_plans makes no host->device
// copies: on this path they would queue behind the big H2D on the copy engine.)
static void run_job_host(int eb, void* host, const ArrayJob& J, int k, unsigned long long* d_bits, cudaStream_t st) {
  const uint64_t n = J.len;
  const int c = J.c;
  setup_pool_once();
  Arena A;
  cudaStream_t ps = side_stream(), cs = copy_stream();
  std::vector<LevelBufs> lv = make_levels(J, eb);
  unsigned char* dev = A.alloc<unsigned char>(n * eb, st);
  unsigned char* scr = A.alloc<unsigned char>(n * eb, st);
  uint16_t* draws = A.alloc<uint16_t>(n, st);
  const uint64_t nleaves = J.q, K = 1ull << k, B = nleaves >> k;
  const uint32_t mmax = (uint32_t)((n + J.q - 1) >> c);
  const uint32_t grid = leaf_apply_grid(B, mmax, num_sms(), eb);
  uint16_t* lscr = A.alloc<uint16_t>((uint64_t)grid * leaf_scratch_stride(mmax) + 8, st);
  std::vector<cudaEvent_t> ev(K + 1, nullptr);
  ExplicitTask E0{};
  try {
    fork_side(st, ps);
    fork_side(st, cs);
    for (uint64_t j = 0; j < K; ++j) {
      const uint64_t lo = bound_at(n, j * B, c), hi = bound_at(n, (j + 1) * B, c);
      CK(cudaMemcpyAsync(dev + lo * eb, (unsigned char*)host + lo * eb, (hi - lo) * eb, cudaMemcpyHostToDevice, cs));
      CK(cudaEventCreateWithFlags(&ev[j], cudaEventDisableTiming));
      CK(cudaEventRecord(ev[j], cs));
    }
    {
      StageTimer tm(0, st);
      launch_leaf_decode16(J, E0, nleaves, draws, d_bits, st);  // needs no data
    }
    // leaves per chunk as it lands (on st), then the plans (host-blocking on
    // the side stream), then each chunk's local rounds -- rounds 1 .. c-k
    // merge pairs inside one chunk -- on the round stream, in place on the
    // scratch, after that chunk's leaves (the tree merge runs in place; the
    // debug segment-pass kernels do not)
    std::vector<cudaEvent_t> evl(K, nullptr);
    for (uint64_t j = 0; j < K; ++j) {
      const uint64_t lo = bound_at(n, j * B, c);
      CK(cudaStreamWaitEvent(st, ev[j], 0));
      ArrayJob Jj = J;
      Jj.blk0 = j * B;
      Jj.lognblk = c - k;
      Jj.elem0 = lo;
      {
        StageTimer tm(1, st);
        launch_leaf_apply(eb, Jj, E0, B, dev + lo * eb, scr + lo * eb, draws + lo, lscr, mmax, grid, st);
      }
      CK(cudaEventCreateWithFlags(&evl[j], cudaEventDisableTiming));
      CK(cudaEventRecord(evl[j], st));
    }
    build_plans(lv, eb, d_bits, A, ps);
    const size_t nloc = (size_t)std::max(0, std::min((int)lv.size() - 1, c - k));
    cudaStream_t rs = round_stream();  // ordered after st by the per-chunk events only
    for (uint64_t j = 0; j < K; ++j) {
      CK(cudaStreamWaitEvent(rs, evl[j], 0));
      for (size_t r = 0; r < nloc; ++r) {
        const uint64_t pp = B >> (r + 1);  // pairs of round r+1 per chunk
        run_round_range(lv[r], eb, scr, j * pp, (j + 1) * pp, bound_at(n, j * B, c), bound_at(n, (j + 1) * B, c), rs);
      }
    }
    for (auto e : evl) cudaEventDestroy(e);
    fork_side(rs, st);  // st after the local rounds
    void* res = run_rounds(lv, eb, scr, dev, st, nloc);
    if (res != dev) CK(cudaMemcpyAsync(dev, res, n * eb, cudaMemcpyDeviceToDevice, st));
    CK(cudaEventCreateWithFlags(&ev[K], cudaEventDisableTiming));
    CK(cudaEventRecord(ev[K], st));
    CK(cudaStreamWaitEvent(cs, ev[K], 0));
    CK(cudaMemcpyAsync(host, dev, n * eb, cudaMemcpyDeviceToHost, cs));
    CK(cudaEventRecord(ev[K], cs));
    CK(cudaStreamWaitEvent(st, ev[K], 0));
    CK(cudaGetLastError());
  } catch (...) {
    cudaStreamSynchronize(ps);
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(st);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    destroy_events(lv);
    A.release(st);
    throw;
  }
  cudaEvent_t done;
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventRecord(done, ps));
  CK(cudaStreamWaitEvent(st, done, 0));
  cudaEventDestroy(done);
  for (auto e : ev)
    if (e) cudaEventDestroy(e);
  destroy_events(lv);
  A.release(st);
}

// ---------------------------------------------------- bit-source state maths
// State after consuming T more bits (SURVEY A2 closed form of bitstream.py:152-176).
static void advance_state(uint64_t s[4], uint64_t T) {
  uint64_t state = s[0], buf = s[1], buflen = s[2], consumed = s[3];
  if (T <= buflen) {
    buflen -= T;
    buf = buflen ? (buf & ((1ULL << buflen) - 1)) : 0;
  } else {
    uint64_t need = T - buflen;
    uint64_t w = (need + 63) / 64;
    state += w * GOLDEN;
    uint64_t rem = 64 * w - need;
    buf = rem ? (mix64(state) & ((1ULL << rem) - 1)) : 0;
    buflen = rem;
  }
  s[0] = state; s[1] = buf; s[2] = buflen; s[3] = consumed + T;
}

static StreamDesc desc_from_state(const uint64_t s[4]) {
  StreamDesc d;
  d.state = s[0];
  d.plen = (uint32_t)s[2];
  d.buf = d.plen ? (s[1] & ((1ULL << d.plen) - 1)) : 0;
  d.pad = 0;
  return d;
}

static void run_single_pair(int eb, void* data, uint64_t j, uint64_t k, uint64_t l, const StreamDesc& sd,
                            unsigned long long* d_bits, cudaStream_t st) {
  setup_pool_once();
  Arena A;
  cudaStream_t ps = side_stream();
  std::vector<LevelBufs> lv(1);
  LevelBufs& L = lv[0];
  uint64_t N = l - j;
  L.LJ.J = make_job(1, N, 0, 0, 0);
  L.LJ.E = ExplicitTask{1, j, k - j, l - k, sd};
  L.LJ.r = 1;
  L.LJ.npairs = 1;
  L.npairs = 1;
  L.sbs = (N + 1 + 511) / 512 + 1;
  L.tpp = tree_tiles_per_pair(L.LJ, eb);
  try {
    fork_side(st, ps);
    build_plans(lv, eb, d_bits, A, ps);
    CK(cudaStreamWaitEvent(st, L.ev_chain, 0));
    launch_merge_tree(eb, data, data, L.plans, 1, L.rank, L.chains, L.tpp, st);  // in place
    CK(cudaStreamWaitEvent(st, L.ev_tail, 0));
    launch_tail_apply(eb, data, L.dst, L.src, L.tmp, 2 * L.cap, L.plans, 1, 0, ~0ull, st);
    CK(cudaGetLastError());
  } catch (...) {
    cudaStreamSynchronize(ps);
    cudaStreamSynchronize(st);
    destroy_events(lv);
    A.release(st);
    throw;
  }
  cudaEvent_t done;
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventRecord(done, ps));
  CK(cudaStreamWaitEvent(st, done, 0));
  cudaEventDestroy(done);
  destroy_events(lv);
  A.release(st);
}

// One pair [0, n1+n2) split over peer buffers (PeerSpan, pair-relative
// positions).  phase 1: the phase-1 tiles of `part` (in place); phase 2 (one
// part, after every part's phase 1 has completed): the tail insertion.  Both
// phases derive the same data-independent plan from the stream.
static void run_pair_peers(int eb, const PeerSpan& span, uint64_t n1, uint64_t n2, const StreamDesc& sd, int part,
                           int phase, unsigned long long* d_bits, cudaStream_t st) {
  setup_pool_once();
  Arena A;
  cudaStream_t ps = side_stream();
  std::vector<LevelBufs> lv(1);
  LevelBufs& L = lv[0];
  const uint64_t N = n1 + n2;
  L.LJ.J = make_job(1, N, 0, 0, 0);
  L.LJ.E = ExplicitTask{1, 0, n1, n2, sd};
  L.LJ.r = 1;
  L.LJ.npairs = 1;
  L.npairs = 1;
  L.sbs = (N + 1 + 511) / 512 + 1;
  L.tpp = tree_tiles_per_pair(L.LJ, eb);
  try {
    fork_side(st, ps);
    build_plans(lv, eb, d_bits, A, ps);
    if (phase == 1) {
      CK(cudaStreamWaitEvent(st, L.ev_chain, 0));
      launch_merge_tree_peer(eb, span, L.plans, L.rank, L.chains, L.tpp, (uint32_t)part, st);
    } else {
      CK(cudaStreamWaitEvent(st, L.ev_tail, 0));
      launch_tail_apply_peer(eb, span, L.dst, L.src, L.tmp, 2 * L.cap, L.plans, st);
    }
    CK(cudaGetLastError());
  } catch (...) {
    cudaStreamSynchronize(ps);
    cudaStreamSynchronize(st);
    destroy_events(lv);
    A.release(st);
    throw;
  }
  cudaEvent_t done;
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventRecord(done, ps));
  CK(cudaStreamWaitEvent(st, done, 0));
  cudaEventDestroy(done);
  destroy_events(lv);
  A.release(st);
}

// ---------------------------------------------------------------- Rao-Sandelius
// Small tasks of the splitting shuffle (rs.cu): plan on the device (one lane
// per task), then the split nodes level by level, then the Fisher-Yates
// leaves; every leaf's result is left in buf0 (the caller's buffer).
// buf0/buf1/draws are indexed by global position.  Returns the tasks' bits.
static uint64_t run_rs_tasks(int eb, void* buf0, void* buf1, const std::vector<RsTask>& tasks, uint64_t span_lo,
                             uint64_t span_hi, uint64_t cutoff, Arena& A, cudaStream_t st) {
  if (tasks.empty()) return 0;
  const uint32_t nt = (uint32_t)tasks.size();
  const uint64_t span = span_hi - span_lo;
  RsTask* dT = A.alloc<RsTask>(nt, st);
  CK(cudaMemcpyAsync(dT, tasks.data(), nt * sizeof(RsTask), cudaMemcpyHostToDevice, st));
  uint16_t* draws = A.alloc<uint16_t>(span, st) - span_lo;
  unsigned long long* counts = A.alloc<unsigned long long>(3, st);
  unsigned long long* tbits = A.alloc<unsigned long long>(nt, st);
  uint64_t cap = std::min<uint64_t>(span + 1, 4 * span / std::max<uint64_t>(cutoff, 1) + 4ull * nt + 1024);
  uint64_t ncap = cap, lcap = cap;
  std::vector<RsNode> nodes;
  std::vector<RsLeaf> leaves;
  for (int attempt = 0; attempt < 2; ++attempt) {
    RsNode* dN = A.alloc<RsNode>(ncap, st);
    RsLeaf* dL = A.alloc<RsLeaf>(lcap, st);
    CK(cudaMemsetAsync(counts, 0, 3 * 8, st));
    CK(cudaMemsetAsync(tbits, 0, nt * 8, st));
    // per-task bit counts: RsTask.array indexes tbits
    uint64_t maxsz = 0;
    for (const auto& tk : tasks) maxsz = std::max<uint64_t>(maxsz, tk.hi - tk.lo);
    launch_rs_plan(dT, nt, cutoff, draws, dN, counts, ncap, dL, lcap, tbits, st, maxsz > (1ull << 31));
    unsigned long long hc[3];
    CK(cudaMemcpyAsync(hc, counts, 24, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hc[2]) throw std::runtime_error("splitting-shuffle stack overflow (more than 256 pending ranges)");
    if (hc[0] > ncap || hc[1] > lcap) {
      ncap = hc[0];
      lcap = hc[1];
      continue;
    }
    nodes.resize(hc[0]);
    leaves.resize(hc[1]);
    if (hc[0]) CK(cudaMemcpyAsync(nodes.data(), dN, hc[0] * sizeof(RsNode), cudaMemcpyDeviceToHost, st));
    if (hc[1]) CK(cudaMemcpyAsync(leaves.data(), dL, hc[1] * sizeof(RsLeaf), cudaMemcpyDeviceToHost, st));
    break;
  }
  std::vector<unsigned long long> hb(nt);
  CK(cudaMemcpyAsync(hb.data(), tbits, nt * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  uint64_t bits = 0;
  for (auto b : hb) bits += b;
  // split nodes, level by level (a node's input is its parent's output)
  std::stable_sort(nodes.begin(), nodes.end(), [](const RsNode& a, const RsNode& b) { return a.level < b.level; });
  if (!nodes.empty()) {
    RsNode* dN = A.alloc<RsNode>(nodes.size(), st);
    CK(cudaMemcpyAsync(dN, nodes.data(), nodes.size() * sizeof(RsNode), cudaMemcpyHostToDevice, st));
    size_t i = 0;
    while (i < nodes.size()) {
      size_t j = i;
      while (j < nodes.size() && nodes[j].level == nodes[i].level) ++j;
      launch_rs_nodes(eb, dN + i, (uint32_t)(j - i), dT, buf0, buf1, st);
      i = j;
    }
  }
  // leaves: their data is in buf[parity ^ depth]
  std::vector<uint64_t> lst[2], back, serial_back;
  std::vector<RsLeaf> serial;
  uint32_t mmax[2] = {0, 0};
  for (const RsLeaf& lf : leaves) {
    const uint32_t par = (tasks[lf.task].parity ^ lf.depth) & 1u;
    const uint64_t m = lf.hi - lf.lo;
    if (m <= 1) {
      if (m == 1 && par == 1) { back.push_back(lf.lo); back.push_back(lf.hi); }
      continue;
    }
    if (m > 65536) {
      serial.push_back(lf);
      if (par == 0) { back.push_back(lf.lo); back.push_back(lf.hi); }
      continue;
    }
    lst[par].push_back(lf.lo);
    lst[par].push_back(lf.hi);
    mmax[par] = std::max(mmax[par], (uint32_t)m);
    if (par == 0) { back.push_back(lf.lo); back.push_back(lf.hi); }  // the result lands in buf1
  }
  ArrayJob J0 = make_job(1, 1, 0, 0, 0);
  ExplicitTask E0{};
  for (int par = 0; par < 2; ++par) {
    const uint64_t cnt = lst[par].size() / 2;
    if (!cnt) continue;
    uint64_t* dl = A.alloc<uint64_t>(lst[par].size(), st);
    CK(cudaMemcpyAsync(dl, lst[par].data(), lst[par].size() * 8, cudaMemcpyHostToDevice, st));
    const uint32_t grid = leaf_apply_grid(cnt, mmax[par], num_sms(), eb);
    uint16_t* lscr = A.alloc<uint16_t>((uint64_t)grid * leaf_scratch_stride(mmax[par]) + 8, st);
    launch_leaf_apply(eb, J0, E0, cnt, par ? buf1 : buf0, par ? buf0 : buf1, draws, lscr, mmax[par], grid, st, dl);
  }
  if (!serial.empty()) {
    RsLeaf* dS = A.alloc<RsLeaf>(serial.size(), st);
    CK(cudaMemcpyAsync(dS, serial.data(), serial.size() * sizeof(RsLeaf), cudaMemcpyHostToDevice, st));
    launch_rs_leaf_serial(eb, dS, (uint32_t)serial.size(), dT, buf0, buf1, st);
  }
  if (!back.empty()) {
    uint64_t* db = A.alloc<uint64_t>(back.size(), st);
    CK(cudaMemcpyAsync(db, back.data(), back.size() * 8, cudaMemcpyHostToDevice, st));
    launch_rs_copy_ranges(eb, db, (uint32_t)(back.size() / 2), buf1, buf0, st);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));  // host vectors above are the copies' sources
  return bits;
}

// rs_shuffle_parallel (splitshuffle.py:92-133): big ranges level by level,
// then the small tasks.  Returns ShuffleReport.bits.
static uint64_t run_rs_parallel(int eb, void* data, uint64_t n, uint64_t cutoff, uint64_t seed, cudaStream_t st) {
  setup_pool_once();
  Arena A;
  uint64_t bits = 0;
  try {
    void* scratch = A.alloc<unsigned char>(n * eb, st);
    void* buf[2] = {data, scratch};
    struct F { uint64_t lo, hi, depth; };
    std::vector<F> frontier{{0, n, 0}};
    std::vector<RsTask> tasks;
    const uint64_t kSpawnMin = 1ull << 14;  // shufflers.py:32
    while (!frontier.empty()) {
      std::vector<RsRange> big;
      uint64_t nch = 0, depth = frontier[0].depth;
      for (const F& f : frontier) {
        const uint64_t size = f.hi - f.lo;
        const StreamDesc sd = fresh_stream(substream_seed(seed, f.depth * (n + 1) + f.lo));
        if (size > kSpawnMin) {
          big.push_back(RsRange{f.lo, f.hi, sd, nch});
          nch += (size + 2047) / 2048;
        } else {
          tasks.push_back(RsTask{f.lo, f.hi, sd, (uint32_t)(f.depth & 1), (uint32_t)tasks.size()});
        }
      }
      if (big.empty()) break;
      const uint32_t nr = (uint32_t)big.size();
      RsRange* dR = A.alloc<RsRange>(nr, st);
      CK(cudaMemcpyAsync(dR, big.data(), nr * sizeof(RsRange), cudaMemcpyHostToDevice, st));
      uint64_t* cz = A.alloc<uint64_t>(2 * nch, st);  // zero counts, then the chunk -> range map
      uint64_t* dnz = A.alloc<uint64_t>(nr, st);
      launch_rs_level(eb, dR, nr, nch, cz, dnz, st);
      const uint32_t par = (uint32_t)(depth & 1);
      launch_rs_split(eb, dR, nr, nch, cz, dnz, buf[par], buf[par ^ 1], st);
      std::vector<uint64_t> hnz(nr);
      CK(cudaMemcpyAsync(hnz.data(), dnz, nr * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<F> next;
      for (uint32_t r = 0; r < nr; ++r) {
        const uint64_t lo = big[r].lo, hi = big[r].hi, nz = hnz[r];
        bits += hi - lo;
        if (nz) next.push_back(F{lo, lo + nz, depth + 1});
        if (hi - lo - nz) next.push_back(F{lo + nz, hi, depth + 1});
      }
      frontier.swap(next);
    }
    bits += run_rs_tasks(eb, buf[0], buf[1], tasks, 0, n, cutoff, A, st);
  } catch (...) {
    cudaStreamSynchronize(st);
    A.release(st);
    throw;
  }
  A.release(st);
  return bits;
}

// rs_range_inplace (_kernels.py:449-457): the sequential splitting shuffle of
// [lo, hi) from a mid-stream state.  Returns the bits consumed.
static uint64_t run_rs_range(int eb, void* data, uint64_t lo, uint64_t hi, uint64_t cutoff, const StreamDesc& sd,
                             cudaStream_t st) {
  setup_pool_once();
  Arena A;
  uint64_t bits = 0;
  try {
    unsigned char* scratch = A.alloc<unsigned char>((hi - lo) * eb, st);
    std::vector<RsTask> tasks{RsTask{lo, hi, sd, 0u, 0u}};
    bits = run_rs_tasks(eb, data, (void*)(scratch - lo * eb), tasks, lo, hi, cutoff, A, st);
  } catch (...) {
    cudaStreamSynchronize(st);
    A.release(st);
    throw;
  }
  A.release(st);
  return bits;
}

static void run_single_leaf(int eb, void* data, uint64_t lo, uint64_t hi, const StreamDesc& sd,
                            unsigned long long* d_bits, cudaStream_t st) {
  setup_pool_once();
  Arena A;
  uint64_t m = hi - lo;
  ArrayJob J = make_job(1, m, 0, 0, 0);
  ExplicitTask E{1, lo, m, 0, sd};
  try {
    if (m <= 65536) {
      uint16_t* draws = A.alloc<uint16_t>(m, st);
      unsigned char* scratch = A.alloc<unsigned char>(m * eb, st);
      uint16_t* lscr = A.alloc<uint16_t>(leaf_scratch_stride(m) + 8, st);
      // absolute-index kernels: shift bases so index lo lands on element 0
      launch_leaf_decode16(J, E, 1, draws - lo, d_bits, st);
      launch_leaf_apply(eb, J, E, 1, data, (void*)(scratch - lo * eb), draws - lo, lscr, (uint32_t)m, 1, st);
      CK(cudaMemcpyAsync((unsigned char*)data + lo * eb, scratch, m * eb, cudaMemcpyDeviceToDevice, st));
    } else {
      launch_leaf_serial(eb, J, E, 1, data, d_bits, st);
    }
    CK(cudaGetLastError());
  } catch (...) {
    cudaStreamSynchronize(st);
    A.release(st);
    throw;
  }
  A.release(st);
}

}  // namespace sk

// ===================================================================== C ABI
using namespace sk;

#define SK_TRY try {
#define SK_CATCH                                   \
  }                                                \
  catch (const CudaError& e) {                     \
    return e.code;                                 \
  }                                                \
  catch (const std::exception& e) {                \
    set_err(e.what());                             \
    return SK_ECUDA;                               \
  }                                                \
  return SK_OK;

static int check_eb(int eb) {
  if (eb != 4 && eb != 8) {
    set_err("elem_bytes must be 4 or 8");
    return SK_EINVAL;
  }
  return SK_OK;
}

static int fetch_bits(unsigned long long* d_bits, uint64_t* out, uint64_t count, cudaStream_t st) {
  if (out) {
    CK(cudaMemcpyAsync(out, d_bits, count * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return SK_OK;
}

extern "C" {

int sk_version(void) { return 1; }

// Internal knobs for performance experiments and tests (not part of the public
// header): 1 = cut the leaf apply after phase k / test paths, 4 = tree merge
// direct path, 6 = force the leaf apply's serial fallback, 7 = leaf-apply L2
// eviction hints on/off, 8 = largest leaf count that takes the warp-per-leaf
// speculative decode (0: always a lane per leaf), 10 = side streams for the
// rounds' plans (1 or 2).
int sk_debug_set(int key, int value) {
  if (key == 1) { debug_set_leaf_stop(value); return 0; }
  if (key == 4) { debug_set_tree_force_direct(value); return 0; }
  if (key == 6) { debug_set_leaf_fallback(value); return 0; }
  if (key == 7) { debug_set_leaf_l2pol(value); return 0; }
  if (key == 8) { debug_set_spec_decode_max(value); return 0; }
  if (key == 10) { g_plan_streams = value; return 0; }
  return -1;
}
const char* sk_last_error(void) { return g_err.c_str(); }
uint64_t sk_launch_count(void) { return g_launches.load(); }

void sk_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  memset(g_prof_launch, 0, sizeof(g_prof_launch));
  g_prof_on = on != 0;
}

int sk_profile_read(double* ms_out, uint64_t* launches_out, int max_stages) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int ns = std::min(max_stages, kStages);
  std::vector<double> acc(kStages, 0.0);
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    acc[r.stage] += ms;
  }
  for (int i = 0; i < ns; ++i) {
    if (ms_out) ms_out[i] = acc[i];
    if (launches_out) launches_out[i] = g_prof_launch[i];
  }
  return ns;
}

int sk_merge_shuffle_parallel(void* data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t seed,
                              uint64_t* bits_out, void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (n && !data) { set_err("null data"); return SK_EINVAL; }
  if (cutoff == 0) cutoff = 65536;
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  int c = plan_c(n, cutoff);
  ArrayJob J = make_job(1, n, c, 0, seed);
  try {
    run_job(elem_bytes, data, J, d_bits, st);
    fetch_bits(d_bits, bits_out, 1, st);
  } catch (...) {
    cudaFreeAsync(d_bits, st);
    throw;
  }
  CK(cudaFreeAsync(d_bits, st));
  SK_CATCH
}

int sk_merge_shuffle_parallel_host(void* host_data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t seed,
                                   uint64_t* bits_out, void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (n && !host_data) { set_err("null data"); return SK_EINVAL; }
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  {
    const uint64_t cut = cutoff ? cutoff : 65536;
    const int c = plan_c(n, cut);
    if (n >= (1ull << 24) && c >= 3 && ((n + (1ull << c) - 1) >> c) <= 65536) {
      unsigned long long* d_bits;
      CK(cudaMallocAsync((void**)&d_bits, 8, st));
      CK(cudaMemsetAsync(d_bits, 0, 8, st));
      uint64_t bits = 0;
      try {
        run_job_host(elem_bytes, host_data, make_job(1, n, c, 0, seed), 3, d_bits, st);
        fetch_bits(d_bits, &bits, 1, st);
      } catch (...) {
        cudaFreeAsync(d_bits, st);
        throw;
      }
      CK(cudaFreeAsync(d_bits, st));
      CK(cudaStreamSynchronize(st));
      if (bits_out) *bits_out = bits;
      return SK_OK;
    }
  }
  void* d = nullptr;
  CK(cudaMallocAsync(&d, n ? n * elem_bytes : 1, st));
  CK(cudaMemcpyAsync(d, host_data, n * elem_bytes, cudaMemcpyHostToDevice, st));
  uint64_t bits = 0;
  int rc = sk_merge_shuffle_parallel(d, elem_bytes, n, cutoff, seed, &bits, stream);
  if (rc == SK_OK) {
    CK(cudaMemcpyAsync(host_data, d, n * elem_bytes, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaFreeAsync(d, st));
  CK(cudaStreamSynchronize(st));
  if (rc) return rc;
  if (bits_out) *bits_out = bits;
  SK_CATCH
}

// Single-process multi-GPU merge_shuffle_parallel (SURVEY.md §8 b/e): shard r
// (elements [(n*r*q/G)>>c, (n*(r+1)*q/G)>>c)) lives on devices[r]; a host
// thread per shard runs its leaves and local rounds, then every spanning round
// runs as the fused peer-memory merge (phase 1 on every part's device in
// parallel, phase 2 once per pair).  Devices may repeat.
int sk_merge_shuffle_multi(void* const* shards, const int* devices, int ngpu, int elem_bytes, uint64_t n,
                           uint64_t cutoff, uint64_t seed, uint64_t* bits_out) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!shards || !devices || ngpu < 1 || ngpu > 8 || (ngpu & (ngpu - 1))) {
    set_err("multi: 1..8 shards, a power of two");
    return SK_EINVAL;
  }
  if (cutoff == 0) cutoff = 65536;
  const int c = plan_c(n, cutoff);
  const uint64_t q = 1ull << c;
  int lg = 0;
  while ((1 << lg) < ngpu) ++lg;
  if ((uint64_t)ngpu > q) {
    set_err("multi: more shards than leaf blocks (lower the cutoff)");
    return SK_EINVAL;
  }
  const uint64_t nblk = q >> lg;
  const int local = c - lg;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  // peer access between distinct devices
  for (int a = 0; a < ngpu; ++a)
    for (int b = 0; b < ngpu; ++b) {
      if (devices[a] == devices[b]) continue;
      cudaSetDevice(devices[a]);
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        cudaSetDevice(cur_dev);
        set_err(std::string("peer access: ") + cudaGetErrorString(e));
        return SK_ECUDA;
      }
      cudaGetLastError();
    }
  cudaSetDevice(cur_dev);
  std::vector<std::string> errs;
  std::mutex emu;
  auto run_all = [&](int count, const std::function<int(int)>& fn) {
    std::vector<std::thread> th;
    for (int w = 0; w < count; ++w)
      th.emplace_back([&, w] {
        if (fn(w) != SK_OK) {
          std::lock_guard<std::mutex> lk(emu);
          errs.push_back(sk_last_error());
        }
      });
    for (auto& t : th) t.join();
    return errs.empty();
  };
  auto on_device = [&](int dev, const std::function<int(cudaStream_t)>& fn) -> int {
    cudaSetDevice(dev);
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      set_err("stream creation failed");
      return SK_ECUDA;
    }
    int rc = fn(s);
    if (rc == SK_OK && cudaStreamSynchronize(s) != cudaSuccess) {
      set_err("stream synchronize failed");
      rc = SK_ECUDA;
    }
    cudaStreamDestroy(s);
    return rc;
  };
  std::vector<uint64_t> b(ngpu, 0);
  std::mutex bmu;
  uint64_t total = 0;
  bool ok = run_all(ngpu, [&](int r) {
    return on_device(devices[r], [&](cudaStream_t s) {
      return sk_merge_shuffle_shard(shards[r], elem_bytes, n, cutoff, seed, r * nblk, nblk, local, &b[r], s);
    });
  });
  for (int r = 0; r < ngpu; ++r) total += b[r];
  auto bound = [&](uint64_t i) { return bound_at(n, i, c); };
  for (int rr = local + 1; ok && rr <= c; ++rr) {
    const int span = 1 << (rr - local);
    const int groups = ngpu / span;
    const uint64_t p = 1ull << (rr - 1);
    auto pair_args = [&](int gi, std::vector<void*>& bases, std::vector<uint64_t>& starts, uint64_t& n1,
                         uint64_t& n2, uint64_t st[4]) {
      const int g0 = gi * span;
      const uint64_t i = (uint64_t)g0 * nblk;
      const uint64_t j = bound(i), k = bound(i + p), l = bound(i + 2 * p);
      bases.resize(span);
      starts.resize(span + 1);
      for (int m = 0; m < span; ++m) {
        bases[m] = shards[g0 + m];
        starts[m] = bound((uint64_t)(g0 + m) * nblk) - j;
      }
      starts[span] = l - j;
      n1 = k - j;
      n2 = l - k;
      st[0] = substream_seed(seed, (uint64_t)rr * q + i);
      st[1] = st[2] = st[3] = 0;
    };
    ok = run_all(ngpu, [&](int w) {  // phase 1: every part of every spanning pair
      const int gi = w / span, m = w % span;
      std::vector<void*> bases;
      std::vector<uint64_t> starts;
      uint64_t n1, n2, st[4];
      pair_args(gi, bases, starts, n1, n2, st);
      return on_device(devices[w], [&](cudaStream_t s) {
        return sk_merge_range_peers(bases.data(), starts.data(), span, m, elem_bytes, n1, n2, st, 1, nullptr, s);
      });
    });
    if (!ok) break;
    ok = run_all(groups, [&](int gi) {  // phase 2: the tail, once per pair
      std::vector<void*> bases;
      std::vector<uint64_t> starts;
      uint64_t n1, n2, st[4], pb = 0;
      pair_args(gi, bases, starts, n1, n2, st);
      const int rc = on_device(devices[gi * span], [&](cudaStream_t s) {
        return sk_merge_range_peers(bases.data(), starts.data(), span, 0, elem_bytes, n1, n2, st, 2, &pb, s);
      });
      std::lock_guard<std::mutex> lk(bmu);
      total += pb;
      return rc;
    });
  }
  cudaSetDevice(cur_dev);
  if (!ok) {
    set_err(errs.empty() ? std::string("multi: failed") : errs[0]);
    return SK_ECUDA;
  }
  if (bits_out) *bits_out = total;
  return SK_OK;
}

int sk_merge_shuffle_shard(void* data, int elem_bytes, uint64_t n_total, uint64_t cutoff, uint64_t seed,
                           uint64_t blk0, uint64_t nblk, int rounds, uint64_t* bits_out, void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (cutoff == 0) cutoff = 65536;
  const int c = plan_c(n_total, cutoff);
  int lg = 0;
  while ((1ULL << lg) < nblk) ++lg;
  if (nblk == 0 || (1ULL << lg) != nblk || blk0 % nblk || blk0 + nblk > (1ULL << c) || rounds < 0 || rounds > lg) {
    set_err("shard: nblk must be a power of two dividing blk0, within 2^c blocks; rounds <= log2(nblk)");
    return SK_EINVAL;
  }
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  ArrayJob J = make_job(1, n_total, c, 0, seed);
  J.blk0 = blk0; J.lognblk = lg; J.rmax = rounds; J.elem0 = bound_at(n_total, blk0, c);
  try {
    run_job(elem_bytes, data, J, d_bits, st);
    fetch_bits(d_bits, bits_out, 1, st);
  } catch (...) {
    cudaFreeAsync(d_bits, st);
    throw;
  }
  CK(cudaFreeAsync(d_bits, st));
  SK_CATCH
}

int sk_batched_shuffle(void* data, int elem_bytes, uint64_t batch, uint64_t len, uint64_t cutoff, uint64_t seed,
                       uint64_t* bits_out, void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (batch && len && !data) { set_err("null data"); return SK_EINVAL; }
  if (cutoff == 0) cutoff = 65536;
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, (batch ? batch : 1) * 8, st));
  CK(cudaMemsetAsync(d_bits, 0, (batch ? batch : 1) * 8, st));
  int c = plan_c(len, cutoff);
  ArrayJob J = make_job(batch, len, c, 1, seed);
  try {
    run_job(elem_bytes, data, J, d_bits, st);
    fetch_bits(d_bits, bits_out, batch, st);
  } catch (...) {
    cudaFreeAsync(d_bits, st);
    throw;
  }
  CK(cudaFreeAsync(d_bits, st));
  SK_CATCH
}

int sk_fy_range(void* data, int elem_bytes, uint64_t lo, uint64_t hi, uint64_t state_io[4], void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!state_io || hi < lo) { set_err("bad range or state"); return SK_EINVAL; }
  if (state_io[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  if (hi - lo >= 2) {
    unsigned long long* d_bits;
    CK(cudaMallocAsync((void**)&d_bits, 8, st));
    CK(cudaMemsetAsync(d_bits, 0, 8, st));
    uint64_t bits = 0;
    try {
      run_single_leaf(elem_bytes, data, lo, hi, desc_from_state(state_io), d_bits, st);
      fetch_bits(d_bits, &bits, 1, st);
    } catch (...) {
      cudaFreeAsync(d_bits, st);
      throw;
    }
    CK(cudaFreeAsync(d_bits, st));
    advance_state(state_io, bits);
  }
  SK_CATCH
}

int sk_merge_range(void* data, int elem_bytes, uint64_t j, uint64_t k, uint64_t l, uint64_t state_io[4],
                   void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!state_io || k < j || l < k) { set_err("bad merge range or state"); return SK_EINVAL; }
  if (state_io[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  if (k == j || l == k) return SK_OK;  // _kernels.py:99-100
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  uint64_t bits = 0;
  try {
    run_single_pair(elem_bytes, data, j, k, l, desc_from_state(state_io), d_bits, st);
    fetch_bits(d_bits, &bits, 1, st);
  } catch (...) {
    cudaFreeAsync(d_bits, st);
    throw;
  }
  CK(cudaFreeAsync(d_bits, st));
  advance_state(state_io, bits);
  SK_CATCH
}

int sk_merge_range_peers(void* const* part_bases, const uint64_t* part_starts, int nparts, int part, int elem_bytes,
                         uint64_t n1, uint64_t n2, const uint64_t state[4], int phase, uint64_t* bits_out,
                         void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!part_bases || !part_starts || !state || nparts < 1 || nparts > 8 || part < 0 || part >= nparts ||
      (phase != 1 && phase != 2)) {
    set_err("bad peer span arguments");
    return SK_EINVAL;
  }
  if (part_starts[0] != 0 || part_starts[nparts] != n1 + n2) {
    set_err("parts must cover [0, n1+n2)");
    return SK_EINVAL;
  }
  for (int k = 0; k < nparts; ++k)
    if (part_starts[k + 1] < part_starts[k] || !part_bases[k]) {
      set_err("parts must be ordered and non-null");
      return SK_EINVAL;
    }
  if (state[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  if (bits_out) *bits_out = 0;
  if (n1 == 0 || n2 == 0) return SK_OK;  // _kernels.py:99-100
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  PeerSpan span{};
  span.n = nparts;
  for (int k = 0; k < nparts; ++k) {
    span.base[k] = part_bases[k];
    span.start[k] = part_starts[k];
  }
  span.start[nparts] = part_starts[nparts];
  uint64_t sv[4] = {state[0], state[1], state[2], state[3]};
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  uint64_t bits = 0;
  try {
    run_pair_peers(elem_bytes, span, n1, n2, desc_from_state(sv), part, phase, d_bits, st);
    fetch_bits(d_bits, &bits, 1, st);
  } catch (...) {
    cudaFreeAsync(d_bits, st);
    throw;
  }
  CK(cudaFreeAsync(d_bits, st));
  if (bits_out && phase == 2) *bits_out = bits;
  SK_CATCH
}

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda link)
typedef int (*sk_get_range_fn)(unsigned long long*, size_t*, unsigned long long);
static sk_get_range_fn get_range_fn() {
  static sk_get_range_fn f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = (sk_get_range_fn)p;
  }
  return f;
}

int sk_ipc_get_handle(const void* ptr, void* handle_out, uint64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) { set_err("null argument"); return SK_EINVAL; }
  SK_TRY
  sk_get_range_fn f = get_range_fn();
  if (!f) { set_err("cuMemGetAddressRange unavailable"); return SK_ECUDA; }
  unsigned long long base = 0;
  size_t size = 0;
  if (f(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) { set_err("cuMemGetAddressRange failed"); return SK_ECUDA; }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((uintptr_t)ptr - (uintptr_t)base);
  SK_CATCH
}

int sk_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) { set_err("null argument"); return SK_EINVAL; }
  SK_TRY
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CK(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  SK_CATCH
}

int sk_ipc_close(void* base) {
  SK_TRY
  CK(cudaIpcCloseMemHandle(base));
  SK_CATCH
}

int sk_rs_shuffle_parallel(void* data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t seed, uint64_t* bits_out,
                           void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (cutoff == 0) cutoff = 1ull << 12;  // RS_CUTOFF_DEFAULT (splitshuffle.py:27)
  if (bits_out) *bits_out = 0;
  if (n < 2) return SK_OK;
  SK_TRY
  const uint64_t bits = run_rs_parallel(elem_bytes, data, n, cutoff, seed, (cudaStream_t)stream);
  if (bits_out) *bits_out = bits;
  SK_CATCH
}

int sk_rs_range(void* data, int elem_bytes, uint64_t lo, uint64_t hi, uint64_t cutoff, uint64_t state_io[4],
                void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!state_io || hi < lo) { set_err("bad range or state"); return SK_EINVAL; }
  if (state_io[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  if (cutoff == 0) cutoff = 1ull << 12;
  SK_TRY
  const uint64_t bits = run_rs_range(elem_bytes, data, lo, hi, cutoff, desc_from_state(state_io), (cudaStream_t)stream);
  advance_state(state_io, bits);
  SK_CATCH
}

int sk_merge_shuffle_seq(void* data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t state_io[4],
                         void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!state_io) { set_err("null state"); return SK_EINVAL; }
  if (state_io[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  if (cutoff == 0) cutoff = 65536;
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  uint64_t bits = 0;
  if (n) launch_seq(elem_bytes, data, n, cutoff, desc_from_state(state_io), d_bits, st);
  CK(cudaGetLastError());
  fetch_bits(d_bits, &bits, 1, st);
  CK(cudaFreeAsync(d_bits, st));
  advance_state(state_io, bits);
  SK_CATCH
}

int sk_balanced_small(void* data, int elem_bytes, uint64_t n, uint64_t state_io[4], void* stream) {
  if (int e = check_eb(elem_bytes)) return e;
  if (!state_io || n > 32 || (n && !data)) { set_err("balanced_small: n <= 32 and a state"); return SK_EINVAL; }
  if (state_io[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  if (n < 2) return SK_OK;
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  uint64_t bits = 0;
  launch_bs_small(elem_bytes, data, (int)n, desc_from_state(state_io), d_bits, st);
  CK(cudaGetLastError());
  fetch_bits(d_bits, &bits, 1, st);
  CK(cudaFreeAsync(d_bits, st));
  advance_state(state_io, bits);
  SK_CATCH
}

int sk_balanced_shuffle(void* data, int elem_bytes, uint64_t n, uint64_t state_io[4], void* stream) {
  if (n <= 32) return sk_balanced_small(data, elem_bytes, n, state_io, stream);
  if (int e = check_eb(elem_bytes)) return e;
  if (!state_io || !data) { set_err("balanced_shuffle: data and a state"); return SK_EINVAL; }
  if (state_io[2] > 63) { set_err("buffered_bits must be < 64"); return SK_EINVAL; }
  if (n > balanced_max_n()) { set_err("balanced_shuffle: n above the supported 2^20"); return SK_EINVAL; }
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  unsigned long long* d_bits;
  CK(cudaMallocAsync((void**)&d_bits, 8, st));
  CK(cudaMemsetAsync(d_bits, 0, 8, st));
  uint64_t bits = 0;
  try {
    run_balanced(elem_bytes, data, n, desc_from_state(state_io), d_bits, st);
    fetch_bits(d_bits, &bits, 1, st);
  } catch (...) {
    cudaFreeAsync(d_bits, st);
    throw;
  }
  CK(cudaFreeAsync(d_bits, st));
  advance_state(state_io, bits);
  SK_CATCH
}

int sk_chi_counts(int algo, int n, uint64_t trials, uint64_t seed, uint64_t cutoff, int64_t* counts_out,
                  void* stream) {
  if (algo < 0 || algo > 3 || n < 1 || n > 20 || !counts_out) {
    set_err("chi_counts: algo in {0,1,2,3}, 1 <= n <= 20");
    return SK_EINVAL;
  }
  if (cutoff == 0) cutoff = 65536;
  SK_TRY
  cudaStream_t st = (cudaStream_t)stream;
  setup_pool_once();
  uint64_t nf = 1;
  for (int i = 2; i <= n; ++i) nf *= (uint64_t)i;
  unsigned long long* d;
  CK(cudaMallocAsync((void**)&d, nf * 8, st));
  CK(cudaMemsetAsync(d, 0, nf * 8, st));
  if (trials) launch_chi(algo, n, trials, seed, cutoff, d, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(counts_out, d, nf * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(d, st));
  CK(cudaStreamSynchronize(st));
  SK_CATCH
}

}  // extern "C"
