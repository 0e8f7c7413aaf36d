"""Benchmark: MergeShuffle of n = 2^30 uint32 uniform-random payload (BASELINE
config 3 at 1 GPU), metric Gelem/s permuted.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full merge_shuffle_parallel (leaf Fisher-Yates + 14 merge rounds,
bit-exact with the reference: the checked step's bit count must equal the
reference's 31908987766) of the resident 4 GiB array.  Timing: CUDA events on
the launching stream, barrier + synchronize on both sides, max over ranks, no
per-stage instrumentation inside the timed region.  The array (4 GiB) is 32x
the L2, so no flush is needed between steps.

Extra keys: roofline (dominant kernel = one merge round: merge_tree_kernel,
its average duration from a second, profiled pass of the same steps),
cpu_baseline (the C oracle port on all host cores, one run of the FULL n),
e2e (through the C ABI host entry with pinned host buffers, H2D+D2H inside
the timed region), gpu_launches, clocks.

--impl reference: the reference's CPU path at the same n (not a sample):
the unmodified reference package from baseline/_ref (numba, all host
threads) when it imports, with the oracle port timed beside it; one warm-up
and at most 3 timed full-size runs (the line reports the counts it ran).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gelem/s permuted (uint32, n=2^30) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gelem/s"
LOG2N = 30


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--log2n", type=int, default=LOG2N)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_init(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# Reference bit counts (tests/golden/big.json, from the unmodified reference at seed 0)
REF_BITS = {30: 31908987766, 31: 65963304485}
REF_RUNS_MAX = 3     # timed reference runs (median), after one warm-up


def _payload(n):
    import numpy as np
    return np.random.default_rng(0).integers(0, 2 ** 32, n, dtype=np.uint32)


def _time_runs(fn, runs, warm):
    for _ in range(warm):
        fn()
    times = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return times


def time_port(log2n, runs, warm=0):
    """The oracle port (C restatement of _kernels.py:253-289, oracle/) on all host
    threads at the FULL size: merge_shuffle_tasked on 2^log2n int64 indices, then
    the uint32 payload gather payload[idx] -- the same work as one GPU step."""
    import numpy as np
    from oracle import oracle as O
    O.build()
    cores, n = cpu_cores(), 1 << log2n
    payload = _payload(n)
    idx = np.empty(n, dtype=np.int64)
    bits = [0]

    def one():
        idx[:] = np.arange(n, dtype=np.int64)
        bits[0] = O.merge_shuffle_tasked(idx, 65536, 0, cores)
        payload[idx]
    times = _time_runs(one, runs, warm)
    if log2n in REF_BITS and bits[0] != REF_BITS[log2n]:
        raise RuntimeError(f"oracle port bits {bits[0]} != reference {REF_BITS[log2n]}")
    med = statistics.median(times)
    return {"value": round(n / med / 1e9, 6), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"oracle port merge_shuffle_tasked, n=2^{log2n} int64 indices + uint32 payload gather "
                      f"(the full workload), {warm} warm-up + {runs} timed run(s), median {med:.2f}s, "
                      f"{cores} threads ({cpu_model()})",
            "seconds": [round(t, 3) for t in times]}


def reference_package():
    """The unmodified reference installed in baseline/_ref (pip --target), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "shufflekit")):
        return None
    sys.path.insert(0, path)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(path, ".numba_cache"))
    try:
        import shufflekit
    except Exception:  # noqa: BLE001 - its dependencies (numba) missing on this host
        return None
    return shufflekit if os.path.abspath(shufflekit.__file__).startswith(path) else None


def time_reference(sk_ref, log2n, runs, warm=1):
    """The reference's own public API and stock code path: merge_shuffle_parallel
    (shufflers.py:251-299) on int64 indices (its fast numba path) with all host
    threads, then the uint32 payload gather.  The first run JIT-compiles."""
    import numpy as np
    cores, n = cpu_cores(), 1 << log2n
    payload = _payload(n)
    idx = np.empty(n, dtype=np.int64)
    bits = [0]

    def one():
        idx[:] = np.arange(n, dtype=np.int64)
        rep = sk_ref.merge_shuffle_parallel(idx, sk_ref.ShuffleConfig(threads=cores), sk_ref.BitSource(0))
        bits[0] = rep.bits
        payload[idx]
    times = _time_runs(one, runs, warm)
    if log2n in REF_BITS and bits[0] != REF_BITS[log2n]:
        raise RuntimeError(f"reference bits {bits[0]} != {REF_BITS[log2n]}")
    med = statistics.median(times)
    return {"value": round(n / med / 1e9, 6), "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"unmodified reference (baseline/_ref, numba) merge_shuffle_parallel, n=2^{log2n} int64 "
                      f"indices + uint32 payload gather (the full workload), threads={cores}, {warm} warm-up + "
                      f"{runs} timed run(s), median {med:.2f}s ({cpu_model()})",
            "seconds": [round(t, 3) for t in times]}


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def pcie_roofline(host, dev, step_s, reps=3):
    """The e2e step's transfer floor: the pinned host<->device copy rates of
    this box measured here (the step's own buffers, one direction at a time,
    CUDA events, best of `reps`), the floor = H2D bytes / H2D rate + D2H
    bytes / D2H rate (the shuffle needs all its input before its last round
    and produces its output only after it, so the two transfers cannot
    overlap each other), and the fraction floor / measured e2e step time."""
    import torch
    nbytes = host.numel() * host.element_size()
    st = torch.cuda.current_stream()
    rates = {}
    for name, fn in (("h2d", lambda: dev.copy_(host, non_blocking=True)),
                     ("d2h", lambda: host.copy_(dev, non_blocking=True))):
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        rates[name] = nbytes / (best * 1e-3) / 1e9
    floor_s = nbytes / (rates["h2d"] * 1e9) + nbytes / (rates["d2h"] * 1e9)
    return {"bound": "pcie", "h2d_gbs": round(rates["h2d"], 2), "d2h_gbs": round(rates["d2h"], 2),
            "floor_ms": round(floor_s * 1e3, 2), "step_ms": round(step_s * 1e3, 2),
            "frac": round(floor_s / step_s, 4)}


def traffic_from_profile():
    p = os.path.join(ROOT, "profiles", "merge_kernel_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path at the
    bench's own configuration (n = 2^log2n, not a sample), rank 0 only.  The
    unmodified reference from baseline/_ref when it imports here, else the
    oracle port; the port is timed beside it either way.  Each timed step is
    one full shuffle of 2^log2n elements; at most REF_RUNS_MAX steps are timed
    (and one warmed), and the line reports the counts actually run."""
    if rank != 0:
        return
    runs, warm = max(1, min(args.steps, REF_RUNS_MAX)), min(args.warmup, 1)
    port = time_port(args.log2n, runs, warm=0)
    ref_pkg = reference_package()
    primary = time_reference(ref_pkg, args.log2n, runs, warm) if ref_pkg is not None else port
    if primary is port:
        warm = 0
    v = primary["value"]
    n = 1 << args.log2n
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": runs,
            "warmup": warm, "ms_per_step": round(statistics.median(primary["seconds"]) * 1e3, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"merge_shuffle_parallel n=2^{args.log2n} uint32 uniform payload, cutoff 65536",
                       "n": n, "elem_bytes": 4, "cutoff": 65536, "seed": 0, "parallelism": "host threads",
                       "requested_steps": args.steps, "requested_warmup": args.warmup},
            "cpu_baseline": primary, "port": port if primary is not port else None,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1508_03167_b200 as sk
    from paper_1508_03167_b200 import _lib
    from paper_1508_03167_b200 import distributed as D
    lib = _lib.load()
    # BASELINE config 3: ONE n = 2^30 array sharded contiguously over the
    # ranks (strong scaling); each rank holds n_total / world elements
    n_total = 1 << args.log2n
    n = n_total // world
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    bits = ctypes.c_uint64(0)

    # N > 1: contiguous shards of one n_total array; the spanning rounds run as
    # the fused peer-memory merge (CUDA IPC over NVLink).  If the peer mapping
    # fails on this box, every rank falls back to the NCCL all-gather exchange.
    exchange = os.environ.get("SK_EXCHANGE", "peer")
    if world > 1 and exchange == "peer":
        ok = torch.tensor([1], device="cuda")
        try:
            D.merge_shuffle_sharded(x, n_total, 65536, 0, exchange="peer")
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] peer exchange unavailable on rank {rank}: {exc}", file=sys.stderr)
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            exchange = "allgather"
        x.copy_(torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g))

    def step():
        if world == 1:
            _lib.check(lib.sk_merge_shuffle_parallel(ctypes.c_void_p(x.data_ptr()), 4, n, 65536, 0, None, sp))
        else:
            D.merge_shuffle_sharded(x, n_total, 65536, 0, exchange=exchange)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # one checked step: bits equal the reference's for this n (seed 0)
    if world == 1:
        _lib.check(lib.sk_merge_shuffle_parallel(ctypes.c_void_p(x.data_ptr()), 4, n, 65536, 0, ctypes.byref(bits),
                                                 sp))
    else:
        bits.value = D.merge_shuffle_sharded(x, n_total, 65536, 0, exchange=exchange)
    if args.log2n in REF_BITS and bits.value != REF_BITS[args.log2n]:
        raise SystemExit(f"bits {bits.value} != reference {REF_BITS[args.log2n]}: not the reference's shuffle")

    def timed(nsteps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(nsteps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        el = ev0.elapsed_time(ev1)
        if dist:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return el

    # the timed region: clean steps (no per-stage events)
    l0 = lib.sk_launch_count()
    with ClockSampler(local) as clk:
        ms = timed(args.steps)
    launches = lib.sk_launch_count() - l0
    # a second, profiled pass of the same steps: per-stage CUDA events on the
    # launching stream give the merge round's average duration (roofline)
    lib.sk_profile_enable(1)
    ms_prof = timed(args.steps)
    stage_ms = (ctypes.c_double * 5)()
    stage_l = (ctypes.c_uint64 * 5)()
    lib.sk_profile_read(stage_ms, stage_l, 5)
    lib.sk_profile_enable(0)
    ms_per_step = ms / args.steps
    value = n_total / (ms_per_step * 1e-3) / 1e9

    # roofline: the dominant kernel is the merge round (merge_tree_kernel, one
    # launch per round, stage 2); algorithmic bytes per round = one read + one
    # write of the shard (2 * 4 B * n).
    from paper_1508_03167_b200.shufflers import merge_plan
    c_tot = merge_plan(n_total, 65536)[0]
    local_rounds = c_tot - (world.bit_length() - 1)
    merge_ms = stage_ms[2]
    rounds = max(1, local_rounds * args.steps)
    per_round_ms = merge_ms / rounds
    alg_bytes = 2 * 4 * n
    achieved = alg_bytes / (per_round_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    tr = traffic_from_profile()
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": tr.get("bytes_per_round") if tr else None,
            "peak_source": peak_kind,
            "kernel": "one merge round (merge_tree_kernel, one launch)",
            "algorithmic_bytes_per_round": alg_bytes, "avg_round_ms": round(per_round_ms, 4),
            "launches_per_round": round(stage_l[2] / rounds, 2),
            "stage_ms_per_step": {k: round(stage_ms[i] / args.steps, 4) for i, k in
                                  enumerate(["leaf_decode", "leaf_apply", "merge_rounds", "identity+tail",
                                             "final_copy"])},
            # the whole step: c+1 passes over the shard (leaves + local rounds)
            "step_passes": local_rounds + 1,
            "profiled_pass_ms_per_step": round(ms_prof / args.steps, 3),
            "step_frac_of_roofline": round((local_rounds + 1) * alg_bytes / (peak * 1e9) * 1e3 / ms_per_step, 4),
            # achieved GB/s of the whole step = P * 2 * sizeof(T) * n / t, against the
            # measured copy peak, the nominal 8 TB/s, and the one-pass floor (8 B/elem)
            "step_achieved_gbs": round((local_rounds + 1) * alg_bytes / (ms_per_step * 1e-3) / 1e9, 1),
            "step_frac_of_nominal_8tbs": round((local_rounds + 1) * alg_bytes / 8e12 * 1e3 / ms_per_step, 4),
            "step_frac_of_one_pass_floor": round(alg_bytes / (peak * 1e9) * 1e3 / ms_per_step, 4)}

    # e2e through the public API with host buffers (pinned), H2D + D2H inside
    e2e = None
    if args.e2e_steps > 0:
        host = torch.empty(n, dtype=torch.int32, pin_memory=True)
        host.copy_(x.cpu())
        hp = ctypes.c_void_p(host.data_ptr())

        def e2e_step():
            if world == 1:  # C ABI host entry: copy in, shuffle, copy out, sync
                _lib.check(lib.sk_merge_shuffle_parallel_host(hp, 4, n, 65536, 0, ctypes.byref(bits), sp))
            else:
                x.copy_(host, non_blocking=True)
                bits.value = D.merge_shuffle_sharded(x, n_total, 65536, 0, exchange=exchange)
                host.copy_(x, non_blocking=True)
                torch.cuda.current_stream().synchronize()

        e2e_step()  # warm
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": round(n_total * args.e2e_steps / el / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": 4 * n_total, "d2h_bytes_per_step": 4 * n_total + 8 * world,
               "path": ("sk_merge_shuffle_parallel_host (C ABI), pinned host buffer" if world == 1 else
                        "per rank: pinned host shard -> device, merge_shuffle_sharded, device -> host")}
        e2e["roofline"] = pcie_roofline(host, x, el / args.e2e_steps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = time_port(args.log2n, 1)   # one full-size run of the oracle port (~20-30 s)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic: uniform-random 32-bit payload (torch.Generator seed 1234+rank)",
                "config": {"workload": f"merge_shuffle_parallel n=2^{args.log2n} uint32 uniform payload over {world} GPU(s), "
                                       f"cutoff 65536 ({1 << c_tot} leaves, {c_tot} merge rounds), seed 0",
                           "n_per_gpu": n, "elem_bytes": 4, "cutoff": 65536, "seed": 0,
                           "n_total": n_total,
                           "parallelism": (f"{world} contiguous shards; top {world.bit_length() - 1} rounds "
                                           + ("fused peer-memory merge over NVLink (CUDA IPC)" if exchange == "peer"
                                              else "exchange over NCCL all-gather")) if world > 1 else "1 GPU",
                           "l2": f"input {4 * n >> 20} MiB per GPU >> 126 MB L2; no flush needed",
                           "bits_per_shuffle": int(bits.value)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
