// sk_kernels.h -- host-side launchers for the engine's kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "sk_types.h"

namespace sk {

void count_launch();          // engine-wide launch counter (bench "gpu_launches")
int num_sms();

// leaf.cu
// draws[lo + i] = j_i (uint16) for every leaf [lo, lo + m) with m <= 65536
void launch_leaf_decode16(const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, uint16_t* draws,
                          unsigned long long* bits, cudaStream_t st);
uint32_t leaf_apply_grid(uint64_t nleaves, uint32_t mmax, int num_sms, int eb = 8);
// per-CTA leaf-apply scratch (uint16 elements)
__host__ __device__ inline uint64_t leaf_scratch_stride(uint64_t mmax) { return 3 * ((mmax + 15) & ~15ULL) + 16; }
void launch_leaf_apply(int eb, const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, const void* in, void* out,
                       const uint16_t* draws, uint16_t* scratch, uint32_t mmax, uint32_t grid, cudaStream_t st,
                       const uint64_t* list = nullptr);
void launch_leaf_serial(int eb, const ArrayJob& J, const ExplicitTask& E, uint64_t nleaves, void* out,
                        unsigned long long* bits, cudaStream_t st);

void debug_set_leaf_stop(int v);
void debug_set_spec_decode_max(int v);
void debug_set_leaf_fallback(int v);
void debug_set_leaf_l2pol(int v);
void debug_set_tree_force_direct(int v);

// merge.cu
struct PeerSpan {             // a pair split into contiguous parts in different (peer) buffers
  void* base[8];              // element at pair position start[k] of part k
  uint64_t start[9];
  int n;
};
struct LevelTail {            // device-side view used by the all-levels tail decoder
  PairPlan* plans;
  uint64_t npairs;
  uint64_t* rec_key;          // s + m_x (global position of the insertion target)
  uint32_t* rec_pair;
};
void launch_rank_tables(const LevelJob& LJ, uint64_t sbs, uint64_t* rank, uint64_t* csum, cudaStream_t st);
uint64_t rank_scan_scratch(uint64_t npairs, uint64_t sbs);
void launch_pair_plan(const LevelJob& LJ, uint64_t sbs, const uint64_t* rank, PairPlan* plans, cudaStream_t st);
void launch_tail_decode(const LevelTail* d_levels, int nlevels, const uint64_t* d_pair_prefix, uint64_t total_pairs,
                        unsigned long long* bits, cudaStream_t st);

uint32_t tree_tile(int eb);
uint32_t tree_tiles_per_pair(const LevelJob& LJ, int eb);
uint64_t tree_chain_words(uint64_t npairs, uint32_t tpp);
void launch_tree_chains(int eb, const PairPlan* plans, uint64_t npairs, const uint64_t* rank, uint32_t tpp,
                        uint64_t* chains, cudaStream_t st);
void launch_merge_tree_range(int eb, void* in, void* out, const PairPlan* plans, uint64_t p0, uint64_t p1,
                             const uint64_t* rank, const uint64_t* chains, uint32_t tpp, cudaStream_t st);
void launch_merge_tree(int eb, void* in, void* out, const PairPlan* plans, uint64_t npairs, const uint64_t* rank,
                       const uint64_t* chains, uint32_t tpp, cudaStream_t st);
void launch_copy_tail_region(int eb, const void* in, void* out, const PairPlan* plans, uint64_t npairs,
                             cudaStream_t st);
void launch_tail_offsets(PairPlan* plans, uint64_t npairs, uint64_t cap, uint64_t* used, cudaStream_t st);
void launch_tail_plan(const PairPlan* plans, const uint64_t* rec_key, const uint32_t* rec_pair, const uint64_t* used,
                      uint64_t cap, uint64_t* hkey, uint32_t* hhead, uint32_t* next, uint32_t* slot_of, uint32_t hmask,
                      uint64_t* predx, uint8_t* keyed, uint64_t* dst, uint64_t* src, cudaStream_t st);
void launch_tail_chase(const PairPlan* plans, const uint64_t* rec_key, const uint32_t* rec_pair,
                       const uint64_t* predx, const uint8_t* keyed, const uint64_t* used, uint64_t cap, uint64_t* dst,
                       uint64_t* src, cudaStream_t st);
void launch_merge_tree_peer(int eb, const PeerSpan& ps, const PairPlan* plans, const uint64_t* rank,
                            const uint64_t* chains, uint32_t tpp, uint32_t part, cudaStream_t st);
void launch_tail_apply_peer(int eb, const PeerSpan& ps, const uint64_t* dst, const uint64_t* src, void* tmp,
                            uint64_t nslots, const PairPlan* plans, cudaStream_t st);
void launch_tail_apply(int eb, void* buf, const uint64_t* dst, const uint64_t* src, void* tmp, uint64_t nslots,
                       const PairPlan* plans, uint64_t npairs, uint64_t lo, uint64_t hi, cudaStream_t st);

// rs.cu (Rao-Sandelius, §8 row F2)
struct RsRange {              // a big range of one frontier level
  uint64_t lo, hi;
  StreamDesc sd;              // its substream (flip i <-> element lo + i)
  uint64_t chunk0;            // its first 2048-position chunk in the level's chunk list
};
struct RsTask {               // a small task: the sequential splitting shuffle of [lo, hi)
  uint64_t lo, hi;
  StreamDesc sd;
  uint32_t parity;            // its data is in buf[parity] (0: the caller's buffer)
  uint32_t array;
};
struct RsNode { uint64_t lo, hi, off; uint32_t task, level; };   // a split of a task at stream offset off
struct RsLeaf { uint64_t lo, hi, off; uint32_t task, depth; };   // a Fisher-Yates leaf of a task
void launch_rs_level(int eb, const RsRange* d_ranges, uint32_t nr, uint64_t nchunks, uint64_t* cz, uint64_t* nz,
                     cudaStream_t st);
void launch_rs_split(int eb, const RsRange* d_ranges, uint32_t nr, uint64_t nchunks, const uint64_t* czp,
                     const uint64_t* nz, const void* in, void* out, cudaStream_t st);
void launch_rs_plan(const RsTask* T, uint32_t ntasks, uint64_t cutoff, uint16_t* draws, RsNode* nodes,
                    unsigned long long* counts, uint64_t node_cap, RsLeaf* leaves, uint64_t leaf_cap,
                    unsigned long long* bits, cudaStream_t st, bool wide);
void launch_rs_nodes(int eb, const RsNode* nodes, uint32_t count, const RsTask* T, void* buf0, void* buf1,
                     cudaStream_t st);
void launch_rs_leaf_serial(int eb, const RsLeaf* L, uint32_t count, const RsTask* T, void* buf0, void* buf1,
                           cudaStream_t st);
void launch_rs_copy_ranges(int eb, const uint64_t* list, uint32_t count, const void* from, void* to,
                           cudaStream_t st);

// balanced.cu (BalancedShuffle beyond n <= 32, §8 row F1)
uint64_t balanced_max_n();
void run_balanced(int eb, void* data, uint64_t n, StreamDesc sd, unsigned long long* d_bits, cudaStream_t st);

// misc.cu
void launch_chi(int algo, int n, uint64_t trials, uint64_t seed, uint64_t cutoff, unsigned long long* counts,
                cudaStream_t st);
void launch_bs_small(int eb, void* data, int n, StreamDesc sd, unsigned long long* bits, cudaStream_t st);
void launch_seq(int eb, void* data, uint64_t n, uint64_t cutoff, StreamDesc sd, unsigned long long* bits,
                cudaStream_t st);

}  // namespace sk
