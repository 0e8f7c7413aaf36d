/*
 * shufflekit_b200.h -- C ABI of the B200-native MergeShuffle engine.
 *
 * Drop-in boundary for the reference's operator layer (shufflekit._kernels,
 * the numba engine behind shufflekit.shufflers; paths relative to the
 * reference's pkg/src/shufflekit/).  Every entry point is stream-ordered on the
 * caller's CUDA stream (`stream` = cudaStream_t, NULL = legacy default),
 * works on caller-owned DEVICE memory (except the *_host variants), permutes in
 * place, and treats elements as opaque 4- or 8-byte words (elem_bytes in {4,8}).
 * The result is bit-identical to the reference for the same seed / BitSource
 * state, for any element type of that width.
 *
 * Return value: 0 on success, a negative SK_E* code on failure; sk_last_error()
 * describes the last failure of the calling thread.  Internal scratch (O(n)
 * ping-pong buffer, per-round plans) comes from the device's stream-ordered
 * memory pool and is released before the call returns.
 *
 * Bit-source state vectors are the reference's 4-word state
 * [sm64_state, bit_buffer, buffered_bits, bits_consumed]
 * (_kernels.py:5-7, bitstream.py:125-130); *_io variants read the state before
 * the call and write back the state after it, exactly as the reference's
 * _state_vec/_sync round-trip does (_kernels.py:408-414).
 */
#ifndef SHUFFLEKIT_B200_H
#define SHUFFLEKIT_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_OK 0
#define SK_EINVAL (-1)   /* bad argument (reference raises ValueError) */
#define SK_ECUDA (-2)    /* CUDA runtime error */
#define SK_ENOMEM (-3)   /* device allocation failed */

/* Replaces shufflers.merge_shuffle_parallel (shufflers.py:251-299) /
 * _kernels.merge_shuffle_tasked (_kernels.py:540-543): the frozen substream
 * schedule, leaf i keyed substream_seed(seed, i), round-r merge at block i keyed
 * substream_seed(seed, r*q + i).  cutoff = 0 selects MERGE_CUTOFF_DEFAULT
 * (65536, shufflers.py:29).  *bits_out (host, may be NULL) = ShuffleReport.bits;
 * when non-NULL the call synchronizes the stream before returning. */
int sk_merge_shuffle_parallel(void *data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t seed,
                              uint64_t *bits_out, void *stream);

/* Same, on HOST memory: copies in, shuffles, copies out, synchronizes
 * (the end-to-end path; pinned host memory gives full PCIe bandwidth). */
int sk_merge_shuffle_parallel_host(void *host_data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t seed,
                                   uint64_t *bits_out, void *stream);

/* One GPU's share of merge_shuffle_parallel on an n_total-element array that is
 * sharded contiguously by leaf blocks (multi-GPU, SURVEY.md §8 e): `data` holds
 * global elements [(n*blk0)>>c, (n*(blk0+nblk))>>c); runs the leaves blk0 ..
 * blk0+nblk-1 and merge rounds 1..`rounds` whose pairs lie inside the shard
 * (same substream indices as the whole-array schedule).  nblk is a power of
 * two dividing blk0; rounds <= log2(nblk).  *bits_out = bits of those tasks.
 * The remaining (cross-shard) rounds are driven by
 * paper_1508_03167_b200.distributed with sk_merge_range. */
int sk_merge_shuffle_shard(void *data, int elem_bytes, uint64_t n_total, uint64_t cutoff, uint64_t seed,
                           uint64_t blk0, uint64_t nblk, int rounds, uint64_t *bits_out, void *stream);

/* `batch` independent arrays of `len` elements, back to back; array t is
 * shuffled as merge_shuffle_parallel with BitSource(substream_seed(seed, t))
 * (the per-trial key of _kernels.py:219-220 and cli.py:136).
 * bits_out: host array of `batch` counts (may be NULL). */
int sk_batched_shuffle(void *data, int elem_bytes, uint64_t batch, uint64_t len, uint64_t cutoff, uint64_t seed,
                       uint64_t *bits_out, void *stream);

/* Replaces _kernels.fy_range_inplace (_kernels.py:423-427) / fisher_yates
 * (shufflers.py:145-155): Fisher-Yates on [lo, hi) from a mid-stream state. */
int sk_fy_range(void *data, int elem_bytes, uint64_t lo, uint64_t hi, uint64_t state_io[4], void *stream);

/* Replaces _kernels.merge_inplace (_kernels.py:430-434) / merge
 * (shufflers.py:158-191): shuffled merge of [j,k) and [k,l). */
int sk_merge_range(void *data, int elem_bytes, uint64_t j, uint64_t k, uint64_t l, uint64_t state_io[4],
                   void *stream);

/* Rao-Sandelius splitting shuffle (the paper's baseline).
 * Replaces splitshuffle.rs_shuffle_parallel (splitshuffle.py:92-133): ranges
 * larger than 2^14 flip one coin per element from substream depth*(n+1)+lo and
 * are stably partitioned, smaller ones run the sequential splitting shuffle
 * (Fisher-Yates at <= cutoff) on their own substream.  cutoff = 0 selects
 * RS_CUTOFF_DEFAULT (4096, splitshuffle.py:27).  *bits_out = ShuffleReport.bits
 * (synchronizes). */
int sk_rs_shuffle_parallel(void *data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t seed,
                           uint64_t *bits_out, void *stream);

/* Replaces _kernels.rs_range_inplace (_kernels.py:449-457) / rs_shuffle
 * (splitshuffle.py:66-79): the sequential splitting shuffle of [lo, hi) from a
 * mid-stream state (cutoff 0 = 4096). */
int sk_rs_range(void *data, int elem_bytes, uint64_t lo, uint64_t hi, uint64_t cutoff, uint64_t state_io[4],
                void *stream);

/* Multi-GPU exchange step (SURVEY.md §8 e): the merge of one pair [0, n1+n2)
 * whose elements are split into `nparts` contiguous parts held by different
 * GPUs; part k = positions [part_starts[k], part_starts[k+1]) at device
 * address part_bases[k] (this GPU's own buffer or a peer buffer mapped with
 * sk_ipc_open; P2P over NVLink).  `state` is the pair's bit-source state at
 * the merge start (a fresh substream_seed(seed, r*q+i) in the parallel
 * schedule).  phase 1: this GPU merges the tiles of part `part` in place,
 * reading and writing peers directly (one fused kernel, no staging copy);
 * phase 2: after every part's phase 1 has completed (a barrier of the
 * caller), ONE part applies the tail insertion (shufflers.py:188-191) and
 * returns the pair's bit count in *bits_out.  Result identical to
 * sk_merge_range on the whole pair. */
int sk_merge_range_peers(void *const *part_bases, const uint64_t *part_starts, int nparts, int part, int elem_bytes,
                         uint64_t n1, uint64_t n2, const uint64_t state[4], int phase, uint64_t *bits_out,
                         void *stream);

/* Single-process multi-GPU merge_shuffle_parallel: shards[r] (device pointer on
 * devices[r]) holds elements [(n*r*q/G)>>c, (n*(r+1)*q/G)>>c) of the array,
 * G = ngpu (a power of two <= 8 and <= q = 2^c).  Leaves and local rounds run
 * per shard (a host thread per device), the spanning rounds as the fused
 * peer-memory merge (peer access is enabled between the devices).  Devices may
 * repeat.  *bits_out = ShuffleReport.bits.  Synchronizes. */
int sk_merge_shuffle_multi(void *const *shards, const int *devices, int ngpu, int elem_bytes, uint64_t n,
                           uint64_t cutoff, uint64_t seed, uint64_t *bits_out);

/* CUDA IPC plumbing for sk_merge_range_peers: the 64-byte handle and byte
 * offset of the allocation holding `ptr`; map a peer's allocation (returns its
 * base; add the offset); unmap. */
int sk_ipc_get_handle(const void *ptr, void *handle_out, uint64_t *offset_out);
int sk_ipc_open(const void *handle, void **base_out);
int sk_ipc_close(void *base);

/* Replaces _kernels.merge_shuffle_inplace (_kernels.py:437-441) /
 * merge_shuffle (shufflers.py:194-217): the sequential single-stream variant.
 * Inherently serial (every task's start offset depends on all earlier tasks);
 * runs as one GPU thread. */
int sk_merge_shuffle_seq(void *data, int elem_bytes, uint64_t n, uint64_t cutoff, uint64_t state_io[4],
                         void *stream);

/* Replaces _kernels.balanced_small_inplace (_kernels.py:546-553) and
 * balanced.balanced_shuffle (balanced.py:219-245) for n <= 32 (SURVEY.md §8
 * row F1): singleton leaves merged bottom-up, each pair interleaved along a
 * word drawn as ONE fast dice roll below C(n1+n2, n1) from the source's
 * stream and unranked lexicographically.  state_io as sk_fy_range. */
int sk_balanced_small(void *data, int elem_bytes, uint64_t n, uint64_t state_io[4], void *stream);

/* Replaces balanced.balanced_shuffle (balanced.py:219-245) for any n up to
 * 2^20: the same singleton schedule and ONE stream;
 * each pair's class size C(n1+n2, n1) exact in multi-limb integers, the fast
 * dice roll below it (bitstream.py:187-210 random_int), the word by the
 * recursive-halving unranking (balanced.py:98-155 _locate_split /
 * _unrank_into), the interleave (balanced.py:198-216).  n <= 32 takes the
 * machine-word kernel of sk_balanced_small.  state_io as sk_fy_range.
 * SK_EINVAL above 2^20. */
int sk_balanced_shuffle(void *data, int elem_bytes, uint64_t n, uint64_t state_io[4], void *stream);

/* Replaces _kernels.chi_counts (_kernels.py:489-526) for algo "fy" (0),
 * "merge" (1), "merge_parallel" (2) and "balanced" (3); 2 <= n <= 20 ...
 * counts_out: host array of n! int64 bins.  Synchronizes. */
int sk_chi_counts(int algo, int n, uint64_t trials, uint64_t seed, uint64_t cutoff, int64_t *counts_out,
                  void *stream);

/* Diagnostics. */
const char *sk_last_error(void);
int sk_version(void);
uint64_t sk_launch_count(void);       /* kernels launched by this library so far */
void sk_profile_enable(int on);       /* record CUDA events around the data-path stages */
/* stage times (ms, summed) and launch counts since enable: stage 0 leaf decode,
 * 1 leaf apply, 2 merge rounds (segment-pass kernels), 3 identity region + tail
 * apply, 4 final copy; returns number of stages written.  Synchronizes. */
int sk_profile_read(double *ms_out, uint64_t *launches_out, int max_stages);

#ifdef __cplusplus
}
#endif
#endif
