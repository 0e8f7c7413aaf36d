// sk_types.h -- job/plan descriptors shared by host orchestration and kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "sk_common.cuh"

namespace sk {

// A batch of `batch` equal-length arrays laid out back to back.  Array a is
// shuffled with the frozen substream schedule of merge_shuffle_parallel
// (shufflers.py:224-240, 251-299) keyed by key(a):
//   keymode 0: key = seed                       (merge_shuffle_parallel)
//   keymode 1: key = substream_seed(seed, a)    (per-trial key, _kernels.py:219-220)
struct ArrayJob {
  uint64_t batch;
  uint64_t len;
  uint64_t q;      // 2^c blocks per array
  int c;           // merge rounds
  int keymode;
  uint64_t seed;
  // shard of the schedule (multi-GPU): blocks [blk0, blk0 + 2^lognblk) of each
  // array, rounds 1..rmax; element 0 of the buffer is global element elem0.
  // A whole job has blk0 = 0, lognblk = c, rmax = c, elem0 = 0.
  uint64_t blk0;
  int lognblk;
  int rmax;
  uint64_t elem0;
};

__host__ __device__ __forceinline__ ArrayJob make_job(uint64_t batch, uint64_t len, int c, int keymode,
                                                       uint64_t seed) {
  ArrayJob J;
  J.batch = batch; J.len = len; J.q = 1ULL << c; J.c = c; J.keymode = keymode; J.seed = seed;
  J.blk0 = 0; J.lognblk = c; J.rmax = c; J.elem0 = 0;
  return J;
}

__host__ __device__ __forceinline__ uint64_t array_key(const ArrayJob& J, uint64_t a) {
  return J.keymode ? substream_seed(J.seed, a) : J.seed;
}

// Single explicit task (fisher_yates / merge on a mid-stream BitSource).
struct ExplicitTask {
  int active;
  uint64_t lo, n1, n2;  // leaf: [lo, lo+n1); merge: [lo, lo+n1) + [lo+n1, lo+n1+n2)
  StreamDesc sd;
};

// Per-pair plan of one merge round (data independent: depends only on the
// schedule and the pair's bit stream).
struct PairPlan {
  uint64_t s, n1, n2;   // pair = [s, s+n1) ++ [s+n1, s+n1+n2), global element offsets
  StreamDesc sd;        // the pair's bit stream
  uint64_t t;           // phase-1 stop position (pair relative); bits = t+1
  uint64_t X;           // end of the window segments; [X, N) is identity
  uint64_t rank_off;    // entry 0 of this pair's superblock table
  uint64_t tail_off;    // first tail record
  uint64_t tail_len;    // N - t tail insertions
  uint64_t bits;        // t+1 + tail bits (0 for degenerate pairs)
  uint64_t array;       // owning array (bit accounting)
  uint32_t aex;         // 1: A exhausted (zero stop), 0: B exhausted
  uint32_t degenerate;  // n1 == 0 || n2 == 0: no bits, identity
  uint32_t nseg;        // segments [S_h, S_{h+1}) of the A queue, h < nseg; X = S_nseg
  uint32_t tail_slow;   // 1: the tail records did not fit the round's capacity -> serial tail
};



constexpr uint64_t kNone = ~0ULL;

// Leaf descriptor computed on device from an ArrayJob (or the explicit task).
struct LeafDesc {
  uint64_t lo, hi, array;
  StreamDesc sd;
};

__host__ __device__ __forceinline__ LeafDesc leaf_desc(const ArrayJob& J, const ExplicitTask& E, uint64_t g) {
  LeafDesc L;
  if (E.active) {
    L.lo = E.lo; L.hi = E.lo + E.n1; L.array = 0; L.sd = E.sd;
    return L;
  }
  uint64_t a = g >> J.lognblk, i = J.blk0 + (g & ((1ULL << J.lognblk) - 1));
  uint64_t base = a * J.len - J.elem0;
  L.lo = base + bound_at(J.len, i, J.c);
  L.hi = base + bound_at(J.len, i + 1, J.c);
  L.array = a;
  L.sd = fresh_stream(substream_seed(array_key(J, a), i));  // leaf i -> index i
  return L;
}

// One merge round over all arrays of a job (round r, 1-based), or the single
// explicit pair of the merge() entry point.
struct LevelJob {
  ArrayJob J;
  ExplicitTask E;
  int r;
  uint64_t npairs;
};

// Pair geometry of round r (shufflers.py:117-130, substream index r*q+i from
// shufflers.py:230-240 / _kernels.py:274-276).
__host__ __device__ __forceinline__ void pair_geom(const LevelJob& LJ, uint64_t g, uint64_t& s, uint64_t& n1,
                                                   uint64_t& n2, StreamDesc& sd, uint64_t& array) {
  if (LJ.E.active) {
    s = LJ.E.lo; n1 = LJ.E.n1; n2 = LJ.E.n2; sd = LJ.E.sd; array = 0;
    return;
  }
  const ArrayJob& J = LJ.J;
  int sh = J.lognblk - LJ.r;  // pairs per array (shard) = 2^sh
  uint64_t a = g >> sh, k = g & ((1ULL << sh) - 1);
  uint64_t i = J.blk0 + (k << LJ.r), p = 1ULL << (LJ.r - 1);
  uint64_t base = a * J.len - J.elem0;
  uint64_t j = bound_at(J.len, i, J.c), kk = bound_at(J.len, i + p, J.c), l = bound_at(J.len, i + 2 * p, J.c);
  s = base + j; n1 = kk - j; n2 = l - kk;
  sd = fresh_stream(substream_seed(array_key(J, a), (uint64_t)LJ.r * J.q + i));
  array = a;
}

}  // namespace sk
