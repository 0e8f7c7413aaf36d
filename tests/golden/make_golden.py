"""Generate golden fixtures by running the UNMODIFIED reference (shufflekit).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (committed, small):
  tests/golden/golden.json   -- scalars, hashes, bit counts, small permutations
  tests/golden/chi_n6.npz    -- 720-bin chi-square histograms (chi_counts)

Every case is produced through the reference's own public API
(shufflekit.merge_shuffle_parallel / fisher_yates / merge / merge_shuffle /
BitSource / _kernels.chi_counts), never through this repo's code.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import shufflekit as sk
from shufflekit import _kernels
from shufflekit.shufflers import MergeRange, ShuffleConfig

OUT = os.path.dirname(os.path.abspath(__file__))
THREADS = os.cpu_count() or 1


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def perm_case(n, cutoff, seed, keep_full):
    idx = np.arange(n, dtype=np.int64)
    cfg = ShuffleConfig(cutoff=cutoff, threads=THREADS)
    rep = sk.merge_shuffle_parallel(idx, cfg, sk.BitSource(seed))
    case = {
        "n": n, "cutoff": cutoff, "seed": seed, "bits": int(rep.bits),
        "head": idx[:8].tolist(), "tail": idx[-2:].tolist() if n >= 2 else idx.tolist(),
        "sha_u32": sha(idx.astype("<u4")) if n <= (1 << 32) else None,
        "sha_u64": sha(idx.astype("<u8")),
    }
    if keep_full:
        case["perm"] = idx.tolist()
    return case


def main():
    g = {"threads_used": THREADS}
    # --- bitstream known answers (pkg/tests/test_bitstream.py:75-82 plus more) ---
    words = {}
    for seed in (0, 1, 42, 12345, (1 << 64) - 1):
        for idx in (0, 1, 2, 7, 1000, 123456789):
            words[f"{seed}:{idx}"] = sk.BitSource(seed).split_substream(idx).take(256)
    g["substream_take256"] = {k: hex(v) for k, v in words.items()}
    g["substream_seed"] = {f"{s}:{i}": sk.substream_seed(s, i)
                           for s in (0, 42, 2**63 + 5) for i in (0, 1, 65535, 2**40)}
    # take(k) sequences across word boundaries (test_bitstream.py:94-104 shape)
    seqs = []
    for seed in (0, 1, 12345):
        src = sk.BitSource(seed)
        ks = [1, 3, 64, 65, 7, 200, 1, 31, 33, 63]
        vals = [src.take(k) for k in ks]
        seqs.append({"seed": seed, "ks": ks, "vals": [hex(v) for v in vals],
                     "state": [int(x) for x in src.state_tuple()]})
    g["take_sequences"] = seqs
    # FDR draws: one source, many bounds (incl. powers of two and 2^k+1)
    rng = np.random.default_rng(7)
    bounds = [2, 3, 4, 5, 7, 8, 9, 17, 1000, 65535, 65536, 65537, 2**31 - 1, 2**31,
              2**32 + 1, 2**40 + 3, 2**61 + 1] + [int(b) for b in rng.integers(2, 2**34, 40)]
    fdr = []
    for seed in (3, 99):
        src = sk.BitSource(seed)
        draws = [src.random_int(b) for b in bounds]
        fdr.append({"seed": seed, "bounds": bounds, "draws": draws,
                    "bits": src.bits_consumed, "state": [int(x) for x in src.state_tuple()]})
    g["fdr"] = fdr

    # --- merge_shuffle_parallel permutations (the parity target) ---
    perms = []
    small = [(0, None), (1, None), (2, 1), (3, 1), (5, 1), (6, 1), (6, 2), (7, 1), (16, 1),
             (17, 2), (100, 1), (100, 7), (1000, 3), (4096, None), (5000, 64),
             (65536, None), (65537, None), (65536, 1000), (100_000, None), (100_000, 100)]
    for n, cut in small:
        for seed in (0, 5):
            perms.append(perm_case(n, cut, seed, keep_full=n <= 5000))
    big = [(1 << 20, None, 0), (1 << 20, None, 1), (1_000_000, None, 0),
           (3 * (1 << 20) + 5, None, 0), (1 << 22, 4096, 0), (1 << 22, 1 << 20, 3),
           (1 << 24, None, 0), (1 << 26, None, 0), (1 << 26, None, 9)]
    for n, cut, seed in big:
        perms.append(perm_case(n, cut, seed, keep_full=False))
        print("perm", n, cut, seed, file=sys.stderr)
    g["merge_shuffle_parallel"] = perms

    # --- mid-stream fisher_yates / merge with state write-back ---
    mids = []
    for seed, pre, n in ((11, 0, 1), (11, 5, 2), (12, 13, 100), (13, 64, 1000),
                         (14, 77, 4097), (15, 3, 65536), (16, 100, 70000)):
        src = sk.BitSource(seed)
        src.take(pre) if pre else None
        st0 = [int(x) for x in src.state_tuple()]
        a = np.arange(n, dtype=np.int64)
        sk.fisher_yates(a, src)
        mids.append({"op": "fy", "n": n, "state_in": st0,
                     "state_out": [int(x) for x in src.state_tuple()], "sha_u64": sha(a.astype("<u8")),
                     "perm": a.tolist() if n <= 5000 else None})
    for seed, pre, s, n1, n2, tot in ((21, 0, 0, 3, 4, 7), (22, 9, 2, 50, 50, 110),
                                      (23, 70, 10, 1000, 1, 1020), (24, 1, 0, 1, 1000, 1001),
                                      (25, 33, 5, 2000, 3000, 5005), (26, 63, 0, 0, 10, 10),
                                      (27, 0, 0, 40000, 25536, 65536), (28, 2, 0, 131072, 131072, 262144)):
        src = sk.BitSource(seed)
        src.take(pre) if pre else None
        st0 = [int(x) for x in src.state_tuple()]
        a = np.arange(tot, dtype=np.int64)
        sk.merge(a, MergeRange(s, n1, n2), src)
        mids.append({"op": "merge", "s": s, "n1": n1, "n2": n2, "total": tot, "state_in": st0,
                     "state_out": [int(x) for x in src.state_tuple()], "sha_u64": sha(a.astype("<u8")),
                     "perm": a.tolist() if tot <= 5000 else None})
    g["mid_stream"] = mids

    # --- sequential single-stream merge_shuffle (A9) ---
    seqs = []
    for n, cut, seed in ((6, 1, 0), (1000, 10, 1), (100_000, None, 2), (1 << 20, None, 0)):
        a = np.arange(n, dtype=np.int64)
        rep = sk.merge_shuffle(a, ShuffleConfig(cutoff=cut), sk.BitSource(seed))
        seqs.append({"n": n, "cutoff": cut, "seed": seed, "bits": int(rep.bits),
                     "head": a[:8].tolist(), "sha_u64": sha(a.astype("<u8"))})
    g["merge_shuffle_seq"] = seqs

    # --- batched (config 5): 65536 x 4096, key substream_seed(seed, t) per array ---
    # reference per-array call: merge_shuffle_parallel(arange(4096), cfg, BitSource(key_t))
    bat = []
    for B, L, cut, seed in ((65536, 4096, None, 0), (64, 1000, 50, 3)):
        rows = np.tile(np.arange(L, dtype=np.int64), (B, 1))
        bits = np.zeros(B, dtype=np.uint64)
        for t in range(B):
            r = sk.merge_shuffle_parallel(rows[t], ShuffleConfig(cutoff=cut),
                                          sk.BitSource(sk.substream_seed(seed, t)))
            bits[t] = r.bits
        bat.append({"batch": B, "len": L, "cutoff": cut, "seed": seed,
                    "row0": rows[0, :8].tolist(), "row_last": rows[-1, :8].tolist(),
                    "bits0": int(bits[0]), "bits_last": int(bits[-1]), "bits_sum": int(bits.sum()),
                    "sha_u32": sha(rows.astype("<u4")), "sha_bits": sha(bits.astype("<u8"))})
        print("batched", B, L, file=sys.stderr)
    g["batched"] = bat

    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(g, fh, indent=1)

    # --- chi-square histograms (config 2 uniformity harness), _kernels.chi_counts ---
    chi = {}
    for cut in (65536, 1, 2):
        chi[f"merge_parallel_c{cut}_t10000000_s0"] = _kernels.chi_counts(
            "merge_parallel", 6, 10_000_000, 0, cut, threads=THREADS)
        print("chi", cut, file=sys.stderr)
    chi["merge_parallel_c1_t100000_s7"] = _kernels.chi_counts("merge_parallel", 6, 100_000, 7, 1, threads=THREADS)
    chi["merge_parallel_n5_c1_t100000_s3"] = _kernels.chi_counts("merge_parallel", 5, 100_000, 3, 1, threads=THREADS)
    chi["merge_parallel_n7_c2_t200000_s4"] = _kernels.chi_counts("merge_parallel", 7, 200_000, 4, 2, threads=THREADS)
    chi["fy_t100000_s1"] = _kernels.chi_counts("fy", 6, 100_000, 1, 1, threads=THREADS)
    chi["merge_c1_t100000_s2"] = _kernels.chi_counts("merge", 6, 100_000, 2, 1, threads=THREADS)
    stats = {}
    from shufflekit.verify import chi_square_uniformity
    for cut in (65536, 1):
        r = chi_square_uniformity("merge_parallel", 6, 10_000_000, 0, cutoff=cut, threads=THREADS)
        stats[str(cut)] = {"statistic": r.statistic, "threshold": r.threshold, "passed": r.passed}
    np.savez_compressed(os.path.join(OUT, "chi_n6.npz"), **chi)
    with open(os.path.join(OUT, "chi_stats.json"), "w") as fh:
        json.dump(stats, fh, indent=1)


if __name__ == "__main__":
    main()
