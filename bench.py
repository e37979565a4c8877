#!/usr/bin/env python
"""Benchmark driver (one JSON line on rank 0).

Headline (default): PageRank, 20 fixed fp64 iterations, damping 0.85, on
the BASELINE R-MAT graph (a=.57 b=c=.19, edge factor 16, seed 1) at scale
24 -- configs[1]'s algorithm at the scale where BASELINE.json's north_star
states the HBM-roofline target (the s20 graph of configs[1] is ~L2-sized
and is reported in ``workloads.pr_s20``).  One step = one full
``pagerank`` call (20 pull iterations) on a device-resident CSR; value =
GTEPS = 20*m / t.

The same line carries ``workloads`` with every other BASELINE config
(configs[0] BFS s16, configs[1] PR s20, configs[2] DO-BFS + CC s24,
configs[3] TC s20, configs[4] batch updates on the blocked container at
s22, three reps per size), each with the reference CPU path timed on this
host beside it (``cpu_baseline``); ``roofline`` for the PageRank pull
kernel, ``roofline_bfs`` and ``roofline_updates``; ``e2e`` through the C
ABI with host buffers.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` runs the UNMODIFIED reference library (oracle/_ref,
compiled from /root/reference's sources) and nothing of this package: the
scale-24 graph comes from the host-side OpenMP generator in oracle/
(identical to gb::generate_rmat), goes through a GBCSR1 file and
gb::load_binary_csr (io.cpp:87-110), and each step is one stock
gb::pagerank(view, 0.85, 20, DBL_MIN) call (algorithms.cpp:508-555), W
warm-up calls then K timed ones (bench.cpp:85-103).

Multi-GPU: one process per GPU (torchrun); the path does not shard in this
tier, so every rank runs an independent replica (weak scaling), timed as
the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

RMAT = (0.57, 0.19, 0.19)
TINY = float(np.finfo(np.float64).tiny)
METRIC = "PageRank GTEPS (20 fixed fp64 iterations, 20*m/t)"
UNIT = "GTEPS"
L2_BYTES = 126 * 2**20
_T0 = time.perf_counter()


def log(msg):
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


# ---------------------------------------------------------------- plumbing
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if os.environ.get("GBG_BENCH_BACKEND", "nccl") == "nccl" else "gloo"
        dist.init_process_group(backend=backend)
    return rank, local, world


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class Clocks:
    """nvidia-smi clock / throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def events_time(torch, stream_ptr: int, fn, steps: int) -> float:
    """Seconds for `steps` calls of fn, CUDA events on the library's stream."""
    s = torch.cuda.ExternalStream(stream_ptr)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    e1.synchronize()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def pr_bytes(n: int, m: int, w: int = 8) -> int:
    """B_PR = W(n+1) + 4m + 16n per iteration (offsets, ids,
    one fp64 read + one fp64 write per vertex)."""
    return w * (n + 1) + 4 * m + 16 * n


def bfs_model_bytes(n, modes, sizes, degsums, examined, w=8):
    """SURVEY §8(d) BFS byte model over the levels actually run: a sparse
    level moves 4|F| + 2W|F| + 4 sum deg(F) + 8|N| + bm, a dense one
    W(n+1) + 3 bm + 4 E_scan + 4|N| with E_scan the arcs inspected (the
    library reports them per level, equal to the reference's)."""
    bm = (n + 7) // 8
    total = 0
    for i, md in enumerate(modes):
        f = sizes[i]
        nxt = sizes[i + 1] if i + 1 < len(sizes) else 0
        if md == 0:
            total += 4 * f + 2 * w * f + 4 * degsums[i] + 8 * nxt + bm
        else:
            total += w * (n + 1) + 3 * bm + 4 * examined[i] + 4 * nxt
    return total


# ---------------------------------------------------------------- workloads
def run_pagerank(torch, gbg, g, steps, warmup, iters=20, prepare=True):
    """prepare=True: the tiled index (gbg_pagerank_prepare, cached in the
    container); False: the one-shot row path (its cheap layout is built by
    the first, untimed warm-up call)."""
    n, m = g.num_vertices(), g.num_edges()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    if prepare:
        prep_ms = gbg.pagerank_prepare(g)
        log(f"pagerank index build: {prep_ms:.1f} ms")
    step = lambda: gbg.pagerank_device(g, out.data_ptr(), 0.85, iters, TINY)  # noqa: E731
    for _ in range(warmup):
        step()
    l0 = g.launch_count()
    t = events_time(torch, g.stream(), step, steps)
    launches = g.launch_count() - l0
    return t / steps, launches, out


def host_time(fn, steps, warmup):
    """Wall time of a synchronous host-API call (it ends with a stream sync)."""
    for _ in range(warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(steps):
        out = fn()
    return (time.perf_counter() - t0) / steps, out


def run_bfs(torch, gbg, g, src, steps, warmup):
    """Timed steps: gbg_bfs_device with NULL statistics (depths stay on the
    device, nothing returns to the host, calls queue on the handle's
    stream).  `ms_with_stats`: the same call with statistics (one readback
    and a host sync per call)."""
    depth = torch.empty(g.num_vertices(), dtype=torch.int32, device="cuda")
    stats = {}

    def step_stats():
        stats.update(gbg.bfs_device(g, src, depth.data_ptr()))

    for _ in range(warmup):
        step_stats()
    t = events_time(torch, g.stream(), lambda: gbg.bfs_device(g, src, depth.data_ptr(), stats=False), steps)
    ts = events_time(torch, g.stream(), step_stats, steps)
    # per-level device timestamps from one extra, untimed call (the timed
    # path carries no instrumentation)
    os.environ["GBG_BFS_LEVEL_TIMES"] = "1"
    step_stats()
    os.environ.pop("GBG_BFS_LEVEL_TIMES")
    stats["ms_with_stats"] = ts / steps * 1e3
    return t / steps, stats, depth


def update_bytes(size, passes, old_touched, new_touched):
    """SURVEY §8(d) batch-insert byte model: radix passes x 2 x 8 B x raw
    arcs (sort), 8 B x raw arcs (read the raw pairs), and per touched
    source its old list read and its new list written (4 B per id)."""
    raw = 2 * size
    return passes * 2 * 8 * raw + 8 * raw + 4 * old_touched + 4 * new_touched


def run_updates(torch, gbg, S, warmup, sizes, reps=3, cpu=None):
    """configs[4] with the reference protocol (bench.cpp:150-187): per size
    and rep r = 0..2 a batch drawn with seed hash_combine(hash_combine(2,
    size), r), filtered to arcs absent from the base (untimed,
    bench.cpp:150-169), inserted (timed: device prepare = sort + dedup, then
    the merge), BFS from the max-degree vertex, deleted (timed).
    Throughput = sampled batch size / seconds (bench.hpp:72-74); batches are
    device-resident before timing.  With `cpu`, the reference chunked_set
    container replays the same filtered batches (prepare + apply timed in
    the reference library, bench.cpp:171-186)."""
    g = gbg.generate_rmat(S, 16 << S, 1, *RMAT, kind=gbg.KIND_BLOCKED)
    n = g.num_vertices()
    deg0 = g.degrees().astype(np.int64)
    src = int(np.argmax(deg0))
    depth = torch.empty(n, dtype=torch.int32, device="cuda")
    ref_c = None
    if cpu is not None:
        off, nbr = g.to_csr()
        pairs = np.stack([np.repeat(np.arange(n, dtype=np.uint32), np.diff(off.astype(np.int64))), nbr], 1)
        t0 = time.perf_counter()
        ref_c = cpu.ref.chunked(n, pairs)
        log(f"cpu: chunked_set s{S} built in {time.perf_counter() - t0:.1f} s")
        del off, nbr, pairs
    res = {}
    for size in sizes:
        batches = []
        for rep in range(reps):
            buf = torch.empty(4 * size, dtype=torch.int32, device="cuda")
            seed = _hash_combine(_hash_combine(2, size), rep)
            gbg.generate_update_batch_device(S, size, seed, buf.data_ptr(), *RMAT)
            present = torch.empty(2 * size, dtype=torch.uint8, device="cuda")
            g.contains_device(buf.data_ptr(), 2 * size, present.data_ptr())
            batches.append(buf.view(-1, 2)[present == 0].contiguous())
        box = {}
        ins_t, del_t, bfs_t, applied = [], [], [], []
        # untimed warm-up passes on rep 0, then every rep once, timed
        order = [0] * warmup + list(range(reps))
        for k, rep in enumerate(order):
            dev = batches[rep]
            cnt = dev.shape[0]
            ti = events_time(torch, g.stream(), lambda: box.__setitem__("a", g.insert_batch_device(dev.data_ptr(), cnt)), 1)
            tb = events_time(torch, g.stream(), lambda: gbg.bfs_device(g, src, depth.data_ptr()), 1)
            td = events_time(torch, g.stream(), lambda: box.__setitem__("d", g.delete_batch_device(dev.data_ptr(), cnt)), 1)
            if k >= warmup:
                ins_t.append(ti)
                del_t.append(td)
                bfs_t.append(tb)
                applied.append(box["a"])
                assert box["d"] == box["a"], "delete did not restore the base"
        ti, td = statistics.mean(ins_t), statistics.mean(del_t)
        # byte model (§8(d)) for the rep-0 batch: touched sources' lists
        b0 = np.unique(batches[0].cpu().numpy().view(np.uint64))  # unique (src, dst) arcs
        b0 = b0.view(np.uint32).reshape(-1, 2)
        touched = np.unique(b0[:, 0])
        new_deg = np.bincount(b0[:, 0], minlength=n)[touched]
        old_t = int(deg0[touched].sum())
        passes = -(-2 * max(1, (n - 1).bit_length()) // 8)
        ub = update_bytes(size, passes, old_t, old_t + int(new_deg.sum()))
        row = {"insert_edges_per_s": size / ti, "delete_edges_per_s": size / td,
               "insert_ms": ti * 1e3, "delete_ms": td * 1e3, "bfs_after_insert_ms": statistics.mean(bfs_t) * 1e3,
               "insert_ms_per_rep": [x * 1e3 for x in ins_t], "delete_ms_per_rep": [x * 1e3 for x in del_t],
               "raw_arcs": 2 * size, "fresh_arcs_per_rep": [int(b.shape[0]) for b in batches],
               "applied_arcs_per_rep": applied, "applied_arcs_per_s": statistics.mean(applied) / ti,
               "model_bytes": ub, "model_gbs": ub / ti / 1e9, "radix_passes": passes,
               "seeds": "hash_combine(hash_combine(2,size),rep), rep 0..2 (bench.cpp:159-161)"}
        if ref_c is not None:
            ci, cd, cb = [], [], []
            for rep in range(reps):
                hb = batches[rep].cpu().numpy().view(np.uint32)
                a1, t1 = ref_c.apply_timed(hb, True)
                tb1, _ = ref_c.time_bfs(src)
                a2, t2 = ref_c.apply_timed(hb, False)
                assert a1 == applied[rep] == a2, "reference applied count differs"
                ci.append(t1)
                cd.append(t2)
                cb.append(tb1)
            cti, ctd = statistics.mean(ci), statistics.mean(cd)
            row["cpu_baseline"] = {"kind": "reference", "cores": cpu.threads, "unit": "edges/s",
                                   "insert_edges_per_s": size / cti, "delete_edges_per_s": size / ctd,
                                   "insert_ms": cti * 1e3, "delete_ms": ctd * 1e3,
                                   "bfs_after_insert_ms": statistics.mean(cb) * 1e3,
                                   "sample": "reference chunked_set, prepare(GlobalSort)+apply_insert / "
                                             "apply_delete on the same filtered batches, reps 0..2, mean; "
                                             "gb::bfs on the container after each insert"}
        res[str(size)] = row
        log(f"updates s{S} {size}: insert {ti * 1e3:.3f} ms, delete {td * 1e3:.3f} ms")
        if size == 10**6:
            # PageRank right after an update: the batch drops both derived
            # PageRank layouts; the row path rebuilds its cheap layout inside
            # the first call, the tiled index is rebuilt by prepare
            dev = batches[0]
            g.insert_batch_device(dev.data_ptr(), dev.shape[0])
            out = torch.empty(n, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, TINY)
            torch.cuda.synchronize()
            rows_first = time.perf_counter() - t0
            t_rows = events_time(torch, g.stream(), lambda: gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, TINY), 3) / 3
            rows_bytes = gbg.pagerank_index_bytes(g)[1]
            index_ms = gbg.pagerank_prepare(g)
            tiled_bytes = gbg.pagerank_index_bytes(g)[0]
            t_tiled = events_time(torch, g.stream(), lambda: gbg.pagerank_device(g, out.data_ptr(), 0.85, 20, TINY), 3) / 3
            g.delete_batch_device(dev.data_ptr(), dev.shape[0])
            res["pagerank_after_insert_1e6"] = {
                "rows_first_call_ms": rows_first * 1e3, "rows_call_ms": t_rows * 1e3,
                "tiled_index_build_ms": index_ms, "tiled_call_ms": t_tiled * 1e3,
                "rows_layout_bytes": rows_bytes, "tiled_index_bytes": tiled_bytes,
                "container_bytes": g.memory_bytes(),
                "note": "s22 blocked container after the 10^6 rep-0 insert; 20 iterations"}
    return res, g


def _mix64(x):
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def _hash_combine(a, b):
    M = (1 << 64) - 1
    return _mix64(a ^ ((b + 0x9E3779B97F4A7C15 + (a << 6) + (a >> 2)) & M))


# ---------------------------------------------------------------- CPU (reference library)
class Cpu:
    """The UNMODIFIED reference library (oracle/_ref/libgbref.so, compiled
    from /root/reference's sources) with every host thread, plus the C
    restatement for TC (the reference has none).  Trials follow
    bench.cpp:85-103: untimed warm-up, then timed calls (steady_clock
    inside the shim, around the gb:: call alone)."""

    def __init__(self):
        from oracle.bindings import Oracle, Ref

        self.ref = Ref()
        self.orc = Oracle()
        self.threads = os.cpu_count() or 1
        self.ref.set_threads(self.threads)
        self.threads = self.ref.num_threads()

    def csr(self, n, off, nbr):
        t0 = time.perf_counter()
        g = self.ref.csr(n, off, nbr)
        log(f"cpu: reference CsrGraph n={n} built in {time.perf_counter() - t0:.1f} s")
        return g

    def trials(self, fn, warmup, trials):
        for _ in range(warmup):
            fn()
        return [fn() for _ in range(trials)]

    def entry(self, kind, value, unit, sample, **extra):
        return {"value": value, "unit": unit, "cores": self.threads if kind == "reference" else 1, "kind": kind,
                "sample": sample, **extra}


def cpu_pagerank(cpu, rg, m, warmup=1, trials=3, iters=20):
    ts = cpu.trials(lambda: rg.time_pagerank(0.85, iters, TINY)[0], warmup, trials)
    t = statistics.mean(ts)
    return cpu.entry("reference", iters * m / t / 1e9, UNIT,
                     f"gb::pagerank(view, 0.85, {iters}, DBL_MIN), {warmup} warm-up + {trials} timed call(s), mean",
                     seconds=t)


def cpu_bfs(cpu, rg, src, g500_edges, warmup=1, trials=3):
    ts = cpu.trials(lambda: rg.time_bfs(src)[0], warmup, trials)
    t = statistics.mean(ts)
    return cpu.entry("reference", g500_edges / t / 1e9, "GTEPS (Graph500)",
                     f"gb::bfs from {src}, {warmup} warm-up + {trials} timed, mean", ms=t * 1e3)


def cpu_cc(cpu, rg, m, warmup=1, trials=3):
    ts = cpu.trials(lambda: rg.time_cc()[0], warmup, trials)
    t = statistics.mean(ts)
    return cpu.entry("reference", m / t, "arcs/s", f"gb::cc, {warmup} warm-up + {trials} timed, mean", ms=t * 1e3)


def cpu_tc(cpu, n, off, nbr):
    t0 = time.perf_counter()
    tri = cpu.orc.tc(n, off, nbr)
    t = time.perf_counter() - t0
    return cpu.entry("port", 1.0 / t, "calls/s",
                     "oracle/gbo.c gbo_tc restatement (derive_filter orientation + merge intersection; the "
                     "reference has no TC), serial, one call", ms=t * 1e3, triangles=int(tri))


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_for(S, world):
    return {"workload": f"pagerank_rmat_s{S}", "graph": f"R-MAT scale {S}, edge factor 16, a=.57 b=c=.19, seed 1, "
            "symmetrized, self-loops/duplicates removed (bit-exact with gb::generate_rmat)",
            "iterations": 20, "damping": 0.85, "container": "csr (uint64 offsets, uint32 ids)",
            "l2_policy": "inputs larger than L2 (2.2 GB CSR vs 126 MB L2); no flush",
            "parallelism": f"replicas x{world}"}


# ---------------------------------------------------------------- reference arm
def reference_arm(args):
    """The reference's own CPU path, nothing of this package: the graph from
    the host-side generator (oracle/gbo_omp.c, identical to
    gb::generate_rmat, whose serial sort takes ~400 s here), written as
    GBCSR1 and loaded by gb::load_binary_csr (io.cpp:87-110); each step one
    stock gb::pagerank(view, 0.85, 20, DBL_MIN) (algorithms.cpp:508-555)."""
    import tempfile

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if int(os.environ.get("RANK", "0")) != 0:
        return  # rank 0 alone runs the reference arm
    S = args.scale
    cpu = Cpu()
    t0 = time.perf_counter()
    off, nbr = cpu.orc.rmat_csr(S, 16 << S, 1, *RMAT)
    n = off.size - 1
    gen_s = time.perf_counter() - t0
    log(f"reference arm: host R-MAT s{S} generated in {gen_s:.1f} s (m={int(off[n])})")
    with tempfile.TemporaryDirectory(prefix="gbref_") as d:
        path = os.path.join(d, f"rmat_s{S}.gbcsr1")
        cpu.orc.save_gbcsr1(path, n, off, nbr)
        del off, nbr
        t0 = time.perf_counter()
        rg = cpu.ref.load_binary_graph(path)
        load_s = time.perf_counter() - t0
    m = rg.m
    log(f"reference arm: gb::load_binary_csr {load_s:.1f} s; timing {args.warmup} + {args.steps} calls")
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for _ in range(args.warmup):
            rg.time_pagerank(0.85, 20, TINY)
        ts, sums = [], []
        for _ in range(args.steps):
            t, tot = rg.time_pagerank(0.85, 20, TINY)
            ts.append(t)
            sums.append(tot)
    t = sum(ts) / len(ts)
    value = 20 * m / t / 1e9
    sample = (f"full workload per step: stock gb::pagerank(view, 0.85, 20, DBL_MIN) over the whole scale-{S} "
              f"graph (m={m}) loaded with gb::load_binary_csr, {args.warmup} warm-up + {args.steps} timed calls, "
              f"OMP threads={cpu.threads}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_for(S, world), container="reference gb::CsrGraph (GBCSR1 via load_binary_csr)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu.threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0, "clocks": clk.summary(), "host_cpu": cpu_model(),
            "step_seconds": ts, "rank_sum": sums[-1], "generate_s": gen_s, "load_binary_s": load_s,
            "graph": {"n": n, "m": m}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
        return
    rank, local, world = dist_setup()

    import torch

    torch.cuda.set_device(local)
    import paper_2405_11671_b200.graph as gbg

    gbg.set_device(local)
    S = args.scale
    config = config_for(S, world)
    cpu = Cpu() if rank == 0 and world == 1 and not args.no_cpu else None

    # ---- headline: PageRank on the device CSR
    g = gbg.generate_rmat(S, 16 << S, 1, *RMAT)
    n, m = g.num_vertices(), g.num_edges()
    layout_ms = gbg.pagerank_prepare(g)  # tiled index: container-side, cached, dropped by updates
    layout_bytes = gbg.pagerank_index_bytes(g)[0]
    log(f"pagerank index build: {layout_ms:.1f} ms, {layout_bytes / 1e9:.2f} GB")
    barrier(world)
    with Clocks(local) as clk:
        t_step, launches, pr_out = run_pagerank(torch, gbg, g, args.steps, args.warmup)
    t_max = max_over_ranks(t_step, world, device="cuda")
    log(f"pagerank s{S}: {t_step * 1e3:.2f} ms/step")
    value = world * 20 * m / t_max / 1e9
    peaks, peak_src = measured_peaks()
    # the iteration kernel's own average: the 20-iteration call minus a
    # 1-iteration call (same init / unpermute), timed the same way, over 19
    out1 = torch.empty(n, dtype=torch.float64, device="cuda")
    one = lambda: gbg.pagerank_device(g, out1.data_ptr(), 0.85, 1, TINY)  # noqa: E731
    one()
    t_one = events_time(torch, g.stream(), one, args.steps) / args.steps
    del out1
    it_s = (t_step - t_one) / 19
    t_fixed = t_one - it_s
    achieved = pr_bytes(n, m) / it_s / 1e9
    kname = gbg.pagerank_kernel_name()
    traffic = ncu_traffic(kname)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "kernel": f"{kname} (one fused pull iteration)",
                "algorithmic_bytes_per_launch": pr_bytes(n, m),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                "launch_seconds": it_s, "call_fixed_seconds": t_fixed,
                "note": "launch time = (20-iteration call - 1-iteration call) / 19, CUDA events on the library "
                        "stream; algorithmic bytes = SURVEY 8(d) B_PR = 8(n+1) + 4m + 16n"}

    # ---- e2e through the C ABI with host buffers: pinned CSR upload,
    # 20 iterations, ranks read back to host, every step
    off, nbr = g.to_csr()
    off_p = torch.from_numpy(off.view(np.int64)).pin_memory()
    nbr_p = torch.from_numpy(nbr.view(np.int32)).pin_memory()
    off_h = off_p.numpy().view(np.uint64)
    nbr_h = nbr_p.numpy().view(np.uint32)
    ranks_h = torch.empty(n, dtype=torch.float64).pin_memory().numpy()

    def e2e_step():
        # pinned CSR upload, pipelined with validation and the PageRank
        # layout build (gbg_csr_create_ex), then 20 iterations, ranks to host
        h = gbg.CsrGraph.from_csr(off_h, nbr_h, prepare_pagerank=True)
        gbg.pagerank(h, 0.85, 20, TINY, out=ranks_h)
        del h

    e2e_step()
    barrier(world)
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = max_over_ranks((time.perf_counter() - t0) / e2e_steps, world, device="cuda")
    e2e = {"value": world * 20 * m / t_e2e / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": int(off.nbytes + nbr.nbytes), "d2h_bytes_per_step": 8 * n,
           "ms_per_step": t_e2e * 1e3,
           "path": "gbg_csr_create_ex (pinned host CSR -> device in chunks, validated, PageRank index built as "
                   "chunks land) + gbg_pagerank (ranks -> host)"}
    log(f"e2e: {t_e2e * 1e3:.1f} ms/step")

    # the one-shot row path on a second copy of the graph (no tiled index):
    # its layout build and its 20 iterations, for value_incl_layout's
    # comparison and the e2e path's kernel
    g_rows = gbg.generate_rmat(S, 16 << S, 1, *RMAT)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gbg.pagerank(g_rows, 0.85, 1, TINY)  # builds the row layout (plus one iteration)
    rows_first_s = time.perf_counter() - t0
    t_rows, _, _ = run_pagerank(torch, gbg, g_rows, args.steps, args.warmup, prepare=False)
    rows_path = {"ms": t_rows * 1e3, "gteps": 20 * m / t_rows / 1e9, "first_call_incl_layout_ms": rows_first_s * 1e3,
                 "kernel": "pr_iter_k (row path: one-shot calls; r01 kernel)"}
    del g_rows
    log(f"row path s{S}: {t_rows * 1e3:.2f} ms/step")

    cpu_line = None
    rg24 = None
    if cpu is not None:
        rg24 = cpu.csr(n, off, nbr)
        # the headline's CPU beside it: one full 20-iteration call after a
        # 1-iteration warm-up (the whole call is ~14 s on 16 threads)
        rg24.time_pagerank(0.85, 1, TINY)
        t_cpu, _ = rg24.time_pagerank(0.85, 20, TINY)
        cpu_line = cpu.entry("reference", 20 * m / t_cpu / 1e9, UNIT,
                             f"full workload: one stock gb::pagerank(view, 0.85, 20, DBL_MIN) call over the "
                             f"scale-{S} graph (reference CsrGraph), after a 1-iteration warm-up; "
                             f"OMP threads={cpu.threads}", seconds=t_cpu)
        log(f"cpu baseline: PR s{S} {t_cpu:.2f} s")

    workloads = {}
    roofline_bfs = roofline_upd = None
    if rank == 0 and not args.no_secondary:
        # configs[2]: DO-BFS + CC on the same scale-24 graph
        deg = np.diff(off.astype(np.int64))
        src = int(np.argmax(deg))
        tb, st, depth = run_bfs(torch, gbg, g, src, args.steps, args.warmup)
        d = depth.cpu().numpy()
        g500 = int(deg[d >= 0].sum() // 2)
        mb = bfs_model_bytes(n, st["modes"], st["frontier_sizes"], st["degree_sums"], st["examined"])
        workloads[f"bfs_s{S}"] = {"ms": tb * 1e3, "gteps_graph500": g500 / tb / 1e9, "arcs_per_s": m / tb,
                                  "modes": st["modes"], "frontier_sizes": st["frontier_sizes"],
                                  "level_ms": st["level_ms"], "reached": st["reached"], "source": src,
                                  "ms_with_stats": st["ms_with_stats"],
                                  "call": "gbg_bfs_device(stats=NULL): asynchronous, depths device-resident; ms_with_stats = the call with per-level statistics (readback + host sync)",
                                  "examined_arcs": st["examined"], "model_bytes": mb, "model_gbs": mb / tb / 1e9,
                                  "model_frac_of_hbm": mb / tb / 1e9 / peaks["hbm_gbs"]}
        roofline_bfs = {"bound": "hbm", "achieved": mb / tb / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": mb / tb / 1e9 / peaks["hbm_gbs"], "traffic": ncu_traffic("bfs_coop_k"),
                        "kernel": "bfs_coop_k (whole direction-optimising BFS, one cooperative launch)",
                        "algorithmic_bytes_per_launch": mb,
                        "note": "SURVEY 8(d) BFS byte model over the levels actually run (W=8); one launch per BFS"}
        lab = torch.empty(n, dtype=torch.int32, device="cuda")
        for _ in range(args.warmup):
            gbg.cc_device(g, lab.data_ptr())
        tc_ = events_time(torch, g.stream(), lambda: gbg.cc_device(g, lab.data_ptr()), args.steps) / args.steps
        workloads[f"cc_s{S}"] = {"ms": tc_ * 1e3, "arcs_per_s": m / tc_,
                                 "components": int(np.unique(lab.cpu().numpy()).size)}
        if rg24 is not None:
            workloads[f"bfs_s{S}"]["cpu_baseline"] = cpu_bfs(cpu, rg24, src, g500)
            workloads[f"cc_s{S}"]["cpu_baseline"] = cpu_cc(cpu, rg24, m)
            log("cpu baseline: BFS/CC s24 done")
        # §8(f) row 3 on the same graph, through the host API (result copied
        # back to host memory inside the timed call)
        for name, fn, summary in (("kcore", lambda: gbg.kcore(g), lambda o: {"max_core": int(o.max())}),
                                  ("coloring", lambda: gbg.coloring(g), lambda o: {"colors": int(o.max()) + 1}),
                                  ("mis", lambda: gbg.mis(g, 1), lambda o: {"size": int(o.sum())}),
                                  ("ldd", lambda: gbg.ldd(g, 0.2, 1),
                                   lambda o: {"clusters": int((o[0] == np.arange(o[0].size)).sum()),
                                              "rounds": int(o[2].max()) + 1})):
            t_alg, out = host_time(fn, max(1, min(args.steps, 3)), 1)
            workloads[f"{name}_s{S}"] = {"ms": t_alg * 1e3, "arcs_per_s": m / t_alg, **summary(out)}
            log(f"{name}_s{S}: {t_alg * 1e3:.1f} ms")
    del pr_out, rg24
    if rank == 0 and not args.no_secondary:
        # configs[1] exactly: PR s20; configs[3]: TC s20; configs[0]: BFS s16
        g20 = gbg.generate_rmat(20, 16 << 20, 1, *RMAT)
        m20 = g20.num_edges()
        t20r, _, _ = run_pagerank(torch, gbg, g20, args.steps, args.warmup, prepare=False)
        lay20 = gbg.pagerank_prepare(g20)
        t20, _, _ = run_pagerank(torch, gbg, g20, args.steps, args.warmup, prepare=False)
        workloads["pr_s20"] = {"gteps": 20 * m20 / t20 / 1e9, "ms": t20 * 1e3, "layout_build_ms": lay20,
                               "rows_path_ms": t20r * 1e3,
                               "gteps_incl_layout": 20 * m20 / (t20 + lay20 / 1e3) / 1e9,
                               "note": "~L2-resident graph (134 MB CSR vs 126 MB L2)"}
        gbg.triangle_count(g20)
        t0 = time.perf_counter()
        tri = gbg.triangle_count(g20)
        ttc = time.perf_counter() - t0
        workloads["tc_s20"] = {"ms": ttc * 1e3, "triangles": tri}
        if cpu is not None:
            o20, n20 = g20.to_csr()
            rg20 = cpu.csr(g20.num_vertices(), o20, n20)
            workloads["pr_s20"]["cpu_baseline"] = cpu_pagerank(cpu, rg20, m20)
            del rg20
            workloads["tc_s20"]["cpu_baseline"] = cpu_tc(cpu, g20.num_vertices(), o20, n20)
            log("cpu baseline: PR/TC s20 done")
            del o20, n20
        del g20
        g16 = gbg.generate_rmat(16, 16 << 16, 1, *RMAT)
        o16, nb16 = g16.to_csr()
        s16 = int(np.argmax(np.diff(o16.astype(np.int64))))
        t16, st16, d16 = run_bfs(torch, gbg, g16, s16, args.steps * 4, args.warmup)
        dd = d16.cpu().numpy()
        e16 = int(np.diff(o16.astype(np.int64))[dd >= 0].sum() // 2)
        workloads["bfs_s16"] = {"ms": t16 * 1e3, "gteps_graph500": e16 / t16 / 1e9, "modes": st16["modes"],
                                "ms_with_stats": st16["ms_with_stats"]}
        if cpu is not None:
            workloads["bfs_s16"]["cpu_baseline"] = cpu_bfs(cpu, cpu.csr(g16.num_vertices(), o16, nb16), s16, e16,
                                                           warmup=1, trials=10)
        del g16
        # configs[4]: updates on the blocked container at s22, reps 0..2
        upd, _gb = run_updates(torch, gbg, 22, 1, [10**4, 10**5, 10**6, 10**7], cpu=cpu)
        workloads["updates_s22"] = upd
        del _gb
        u7 = upd[str(10**7)]
        roofline_upd = {"bound": "hbm", "achieved": u7["model_gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": u7["model_gbs"] / peaks["hbm_gbs"], "traffic": None,
                        "kernel": "10^7-edge batch insert (device prepare + merge, whole call)",
                        "algorithmic_bytes_per_launch": u7["model_bytes"],
                        "note": "SURVEY 8(d) batch-insert byte model with the radix passes the sort runs; the "
                                "call is ~25 launches, so the fraction is per batch, not per kernel"}
        # capacity: the same PageRank at scale 26 (67M vertices, 2.1G arcs)
        t0 = time.perf_counter()
        g26 = gbg.generate_rmat(26, 16 << 26, 1, *RMAT)
        gen26 = time.perf_counter() - t0
        m26 = g26.num_edges()
        t26, _, _ = run_pagerank(torch, gbg, g26, max(1, min(args.steps, 2)), 1)
        workloads["pr_s26"] = {"gteps": 20 * m26 / t26 / 1e9, "ms": t26 * 1e3, "m": m26,
                               "generate_s": gen26, "note": "capacity run, not a BASELINE config"}
        del g26
        log("secondary workloads done")

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (device R-MAT, bit-exact with the reference generator)",
                "config": config, "gpu_launches": launches, "clocks": clk.summary(), "roofline": roofline,
                "roofline_bfs": roofline_bfs, "roofline_updates": roofline_upd,
                "value_incl_layout": world * 20 * m / (t_max + layout_ms / 1e3) / 1e9,
                "layout_build_ms": layout_ms,
                "layout_bytes": layout_bytes, "container_bytes": g.memory_bytes(),
                "layout_note": "value = calls on the prepared tiled index (built once per graph version, "
                               "layout_build_ms); value_incl_layout charges one index build to one call; "
                               "one-shot calls use the row path (pagerank_rows), which e2e measures",
                "pagerank_rows": rows_path,
                "e2e": e2e, "cpu_baseline": cpu_line, "workloads": workloads, "host_cpu": cpu_model(),
                "graph": {"n": n, "m": m}}
        print(json.dumps(line), flush=True)
    barrier(world)


if __name__ == "__main__":
    main()
