"""Benchmark of the B200 distance threshold search (driver contract in DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config random-1m] [--d 50]
    python bench.py --impl reference ...      # the CPU oracle arm (rank 0 only)

One step = one pass of the whole hot path over the workload, device-resident
inputs: tds_build_index (validate, t_start radix sort, bins, subbin arrays,
FSG) + for each index variant (GPUTemporal, GPUSpatioTemporal, GPUSpatial)
tds_search + tds_fetch_results into device buffers.  ``value`` counts query
segments answered per second over all ranks (3 x |Q| per step per rank: each
query is answered once per variant).  Multi-GPU: one process per GPU, every
rank holds D and answers its own query trajectories (weak scaling; results
stay sharded, no data-path collective); timing is max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "query segments/s & segment-pair tests/s vs HBM roofline at 1/2/4/8 B200"
VARIANTS = ("temporal", "spatiotemporal", "spatial")
# algorithmic work of one pair test: the certified fp32 filter of DESIGN.md
# ("Pair test numerics"): 43 FP32 instructions, 16 of them FFMA -> 59 flops
FLOPS_PER_PAIR = 59
BYTES_PER_SPATIAL_PAIR = 36          # GPUSpatial: 32-B record + 4-B id streamed per pair test
L2_FLUSH_BYTES = 256 << 20


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(args, kname, variant):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    ncu --set full capture of the same configuration (profiles/ncu_traffic.json,
    written by tools/ncu_traffic.py), else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        key = f"{args.config}|{args.d if args.d is not None else 'default'}|{kname}|{variant}"
        return t[key]["dram_bytes"]
    except Exception:
        return None


def fp32_peak_tflops(peaks, n_sms=148):
    # 128 FP32 lanes per SM, FFMA = 2 flops, at the maximum SM clock
    mhz = peaks.get("sm_max_mhz", 1965.0)
    return n_sms * 128 * 2 * mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled in the background."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def mark(self, which):
        if which == 0:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        inside = [r for t, r in self.rows if self.t0 - 0.06 <= t <= self.t1 + 0.06] or \
                 [r for t, r in self.rows if t >= self.t0 - 0.5][:3]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in inside:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except Exception:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = os.environ.get("TDS_DIST_BACKEND", "nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            # one process per GPU; TDS_DIST_BACKEND=gloo allows several ranks on one GPU (tests)
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def max_over_ranks(dist, x, dev):
    """Max of a host float over ranks (NCCL needs a CUDA tensor, gloo a CPU one)."""
    import torch
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, x, dev):
    import torch
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_workload(args, rank):
    import synth
    kw = {}
    if args.config in ("random-1m", "random-dense", "random-dense-1m", "merger"):
        kw["offset"] = rank                       # weak scaling: each rank its own query set
    elif args.config == "scale-out":
        kw["shard"] = (rank, int(os.environ.get("WORLD_SIZE", "1")))   # strong: one query set, sharded
    w = synth.make_workload(args.config, **kw)
    if args.d is not None:
        w.d = args.d
    if args.m is not None:
        w.m_bins = args.m
    if args.v is not None:
        w.v_subbins = args.v
    if args.grid is not None:
        w.grid = (args.grid,) * 3
    return w


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (all-pairs, fp64)
# ---------------------------------------------------------------------------
def host_cores():
    """The box's host cores available to this process (torchrun sets
    OMP_NUM_THREADS=1 per rank; the oracle is given the cores explicitly)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_rate(w, seconds, seed=0, max_q=None):
    """Time the oracle as it stands on a bounded query sample of the workload."""
    import oracle
    rng = np.random.default_rng(seed)
    nq = w.Q.shape[0]
    cores = host_cores()
    cal = np.sort(rng.choice(nq, min(8, nq), replace=False))
    t = time.perf_counter()
    oracle.search(w.D, w.Q, w.d, qsel=cal, nthreads=cores)
    dt = max(time.perf_counter() - t, 1e-6)
    n = int(min(nq, max(8, seconds * len(cal) / dt)))
    if max_q:
        n = min(n, max_q)
    sel = np.sort(rng.choice(nq, n, replace=False))
    t = time.perf_counter()
    r = oracle.search(w.D, w.Q, w.d, qsel=sel, nthreads=cores)
    dt = time.perf_counter() - t
    return n, dt, int(r["hit"].sum()), cores


def run_reference(args, ws, rank):
    if rank != 0:
        return
    w = make_workload(args, 0)
    # each step: a bounded query sample (~step_seconds of CPU work)
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    import oracle
    oracle.build()
    n, dt, hits, cores = oracle_rate(w, per_step)
    rng = np.random.default_rng(1)
    times = []
    for k in range(args.warmup + args.steps):
        sel = np.sort(rng.choice(w.Q.shape[0], n, replace=False))
        t = time.perf_counter()
        oracle.search(w.D, w.Q, w.d, qsel=sel, nthreads=cores)
        el = time.perf_counter() - t
        if k >= args.warmup:
            times.append(el)
    tot = sum(times)
    value = n * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "query segments/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, w, ws),
        "cpu_baseline": {"value": value, "unit": "query segments/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} random queries of {w.Q.shape[0]} per step, all-pairs fp64 against "
                                   f"all {w.D.shape[0]} entries"},
        "e2e": {"value": value, "unit": "query segments/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pair_tests_per_s": n * w.D.shape[0] * len(times) / tot,
    }
    print(json.dumps(line), flush=True)


def config_dict(args, w, ws):
    return {"workload": f"{w.name}-shaped", "n_entries": int(w.D.shape[0]), "n_queries_per_rank": int(w.Q.shape[0]),
            "d": w.d, "m_bins": w.m_bins, "v_subbins": w.v_subbins, "grid": list(w.grid),
            "variants": list(args.variants), "parallelism": f"query-sharded x{ws}, index replicated",
            "variant_streams": 1 if (args.serial and not args.batched) else len(args.variants),
            "search_api": "tds_search_many" if args.batched else "tds_search",
            "l2": "flushed between steps (256 MiB write); timed steps bracketed by barrier + synchronize",
            "note": w.note}


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
def run_tds(args, ws, rank, local):
    import torch
    import paper_1410_2698_b200 as tds
    tds.load_library()
    dev = torch.device("cuda", local)
    w = make_workload(args, rank)
    Dh = torch.from_numpy(w.D).pin_memory()
    Qh = torch.from_numpy(w.Q).pin_memory()
    D = Dh.to(dev)
    Q = Qh.to(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    dist = None
    if ws > 1:
        import torch.distributed as dist

    def barrier():
        if dist is not None:
            dist.barrier()

    # the three variants are independent searches of one index; --concurrent runs
    # them one host thread + CUDA stream each (the C-ABI releases the GIL and
    # supports concurrent searches on different streams).  Default: serial (faster
    # on Random-1M: 1.86 vs 2.05 ms per step, thread/join overheads dominate)
    side = [torch.cuda.Stream(dev) for _ in args.variants]
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=len(args.variants))

    def one_variant(j, kind, idx, host):
        st_ = side[j] if not args.serial else stream
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        with torch.cuda.stream(st_):
            e[0].record(st_)
            r = idx.search(Qh if host else Q, w.d, kind=kind, capacity=args.capacity, stream=st_.cuda_stream)
            e[1].record(st_)
            r.fetch(device=not host, stream=st_.cuda_stream)
            e[2].record(st_)
            stt = r.stats()
            n = r.count
            r.close()
        return e, stt, 16 * n

    def step(collect=None, host=False):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        idx = tds.Index(Dh if host else D, kinds=tds.ALL, m=w.m_bins, v=w.v_subbins, grid=w.grid,
                        stream=stream.cuda_stream)
        ev[1].record(stream)                    # build_index synchronises: the index is ready
        if args.batched:
            # one tds_search_many call: the variants run concurrently on side streams
            # (overlapping their host synchronisations), then each fetches on its stream
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in args.variants]
            for j in range(len(args.variants)):
                side[j].wait_stream(stream)
                evs[j][0].record(side[j])
            rs = idx.search_many([{"queries": Qh if host else Q, "d": w.d, "kind": k, "capacity": args.capacity,
                                   "stream": side[j].cuda_stream} for j, k in enumerate(args.variants)])
            outs = []
            for j, r in enumerate(rs):
                with torch.cuda.stream(side[j]):
                    evs[j][1].record(side[j])
                    r.fetch(device=not host, stream=side[j].cuda_stream)
                    evs[j][2].record(side[j])
                    stt = r.stats()
                    n = r.count
                    r.close()
                outs.append((evs[j], stt, 16 * n))
            for sj in side:
                stream.wait_stream(sj)
        elif args.serial:
            outs = [one_variant(j, k, idx, host) for j, k in enumerate(args.variants)]
        else:
            futs = [pool.submit(one_variant, j, k, idx, host) for j, k in enumerate(args.variants)]
            outs = [f.result() for f in futs]
            for sj in side:
                stream.wait_stream(sj)
        end = torch.cuda.Event(enable_timing=True)
        end.record(stream)
        idx.close()
        per = {k: o[1] for k, o in zip(args.variants, outs)}
        d2h = sum(o[2] for o in outs)
        if collect is not None:
            collect.append((ev + [end], per, d2h, [o[0] for o in outs]))
        return per

    # warm-up.  The first warm-up step runs the variants one after another and
    # measures them: tds_search_many overlaps the searches' host synchronisations
    # and launch chains, which pays only when the searches are short (each under
    # 1 ms of device time, e.g. Random-1M); long pair kernels just compete for the
    # SMs (Random-dense d = 0.01: 26 vs 21 ms per step), and it holds every
    # variant's result at once (Random-dense d = 0.09: 40 GB each), so those stay serial.
    want_batched = args.batched
    args.batched = False
    step()                                   # cold (first-touch, pool growth): not measured
    per0 = step()
    out_bytes = 16 * sum(int(v["n_results"]) for v in per0.values())
    short = all(float(v["ms_total"]) < 1.0 for v in per0.values())
    args.batched = (want_batched and short
                    and out_bytes < 0.1 * torch.cuda.get_device_properties(dev).total_memory)
    for _ in range(args.warmup - 2):
        step()
    torch.cuda.synchronize(dev)

    # timed region: K steps, L2 flushed before each (outside the events)
    launches0 = tds.kernel_launches()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    recs = []
    step_ms = []
    sampler.mark(0)
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(recs)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        if os.environ.get("TDS_BENCH_STEPS") == "1":
            free_b, _ = torch.cuda.mem_get_info(dev)
            print(f"[bench] step {len(step_ms) - 1}: {step_ms[-1]:.3f} ms; torch reserved "
                  f"{torch.cuda.memory_reserved(dev) / 1e9:.1f} GB, device free {free_b / 1e9:.1f} GB",
                  file=sys.stderr, flush=True)
    sampler.mark(1)
    clocks = sampler.stop()
    launches = tds.kernel_launches() - launches0
    total_ms = sum(step_ms)
    if dist is not None:
        total_ms = max_over_ranks(dist, total_ms, dev)

    nq = w.Q.shape[0]
    nvar = len(args.variants)
    nq_all = nq if dist is None else int(round(sum_over_ranks(dist, float(nq), dev)))
    value = nvar * nq_all * args.steps / (total_ms / 1e3)
    # per-phase breakdown (medians over the timed steps)
    build_ms = statistics.median(r[0][0].elapsed_time(r[0][1]) for r in recs)
    per_kind = {}
    for j, kind in enumerate(args.variants):
        pt = [r[1][kind]["pair_tests"] for r in recs]
        pm = [r[1][kind]["ms_pairs"] for r in recs]
        first = recs[0][1][kind]
        per_kind[kind] = {
            "search_ms": statistics.median(r[3][j][0].elapsed_time(r[3][j][1]) for r in recs),
            "fetch_ms": statistics.median(r[3][j][1].elapsed_time(r[3][j][2]) for r in recs),
            "pair_kernel_ms": statistics.median(pm),
            "pair_tests": int(pt[0]),
            "pairs_executed": int(first["pairs_executed"]),
            "refined_pairs": int(first["refined_pairs"]),
            "results": int(first["n_results"]),
            "passes": int(first["passes"]),
            "fallback_queries": int(first["fallback_queries"]),
            "pair_tests_per_s": pt[0] / (statistics.median(pm) / 1e3) if statistics.median(pm) > 0 else None,
        }
    searches_ms = statistics.median(r[0][1].elapsed_time(r[0][2]) for r in recs)
    pair_tests_step = sum(v["pair_tests"] for v in per_kind.values())
    # the paper's response time excludes the index build: search + fetch only
    search_ms = searches_ms
    pt_all = pair_tests_step if dist is None else sum_over_ranks(dist, float(pair_tests_step), dev)
    peaks = load_peaks()
    # roofline of the dominant kernel: the pair kernel with the largest share.
    # GPUSpatial streams one record + id per pair test (FSG slices are per (query,
    # cell)) and is bound by HBM (36 B per pair test).  The range
    # kernels (GPUTemporal / GPUSpatioTemporal) reuse each loaded record for up to
    # 32 queries: their roof is the larger of the FP32 time (59 flops per scheduled
    # pair test) and the HBM time of their algorithmic bytes (SURVEY 8(d):
    # 36 B per entry of D + 48 B per query + 16 B per result record written), i.e.
    # FP32 on sparse outputs and HBM on output-bound searches (Random-dense d=0.09).
    dom = max(per_kind, key=lambda k: per_kind[k]["pair_kernel_ms"])
    dk = per_kind[dom]
    kname = "k_pair_spatial" if dom == "spatial" else "k_pair_range"
    secs = dk["pair_kernel_ms"] / 1e3
    hbm_peak = float(peaks.get("hbm_gbs", 6537.0))
    alu_peak = fp32_peak_tflops(peaks, torch.cuda.get_device_properties(dev).multi_processor_count)
    if dom == "spatial":
        achieved = BYTES_PER_SPATIAL_PAIR * dk["pair_tests"] / secs / 1e9
        peak = hbm_peak
        roof = {"bound": "hbm", "kernel": f"{kname} ({dom})", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy); algorithmic 36 B (record + id) per pair test"}
    else:
        flops = FLOPS_PER_PAIR * dk["pair_tests"]
        nbytes = 36 * w.D.shape[0] + 48 * w.Q.shape[0] + 16 * dk["results"]
        if nbytes / (hbm_peak * 1e9) > flops / (alu_peak * 1e12):
            achieved = nbytes / secs / 1e9
            peak = hbm_peak
            roof = {"bound": "hbm", "kernel": f"{kname} ({dom})", "achieved": achieved, "peak": peak,
                    "unit": "GB/s",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy); algorithmic bytes 36 B x |D| + 48 B x |Q| "
                                   "+ 16 B x results (output-bound: the HBM time exceeds the FP32 time)"}
        else:
            achieved = flops / secs / 1e12
            peak = alu_peak
            roof = {"bound": "alu", "kernel": f"{kname} ({dom})", "achieved": achieved, "peak": peak,
                    "unit": "TFLOP/s",
                    "peak_source": "148 SMs x 128 FP32 lanes x 2 x sm_max_mhz (MEASURED_PEAKS.json); "
                                   "algorithmic 59 flops per scheduled pair test"}
    roof["frac"] = achieved / peak
    roof["traffic"] = ncu_traffic(args, kname, dom)
    roof["share_of_step"] = dk["pair_kernel_ms"] / statistics.median(step_ms)

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        for _ in range(max(1, args.warmup // 2)):
            step(host=True)
        torch.cuda.synchronize(dev)
        er = []
        e2e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            step(er, host=True)
            torch.cuda.synchronize(dev)
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
            barrier()
        tot = sum(e2e_ms)
        if dist is not None:
            tot = max_over_ranks(dist, tot, dev)
        e2e = {"value": nvar * nq_all * args.steps / (tot / 1e3), "unit": "query segments/s",
               "h2d_bytes_per_step": int(w.D.nbytes + nvar * w.Q.nbytes),
               "d2h_bytes_per_step": int(statistics.median(x[2] for x in er)),
               "timing": "host wall clock around each step, synchronize on both sides, max over ranks"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        n, dt, hits, cores = oracle_rate(w, args.cpu_seconds)
        cpu = {"value": n / dt, "unit": "query segments/s", "cores": cores, "kind": "oracle",
               "sample": f"{n} random queries of {nq}, all-pairs fp64 vs all {w.D.shape[0]} entries, "
                         f"one answer per query ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "query segments/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.config == "scale-out" else "weak", "vs_baseline": None,
            "dtype": "f32+f64", "data": "synthetic",
            "config": config_dict(args, w, ws),
            "pair_tests_per_s": pt_all * args.steps / (total_ms / 1e3),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks,
            "breakdown": {"build_index_ms": build_ms, "variants": per_kind,
                          "step_ms_median": statistics.median(step_ms),
                          "step_ms_min": min(step_ms), "step_ms_max": max(step_ms)},
            "search_only": {"value": ws * nvar * nq / (search_ms / 1e3), "unit": "query segments/s",
                            "ranks": "rank 0's time, scaled by the rank count",
                            "note": "per-step median of the three variants' tds_search + tds_fetch_results "
                                    "(index build excluded, as in the paper's response time, P:1301-1304); rank 0"},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="tds", choices=["tds", "reference"])
    ap.add_argument("--config", default="random-1m")
    ap.add_argument("--d", type=float, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--v", type=int, default=None)
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--variants", default="all")
    ap.add_argument("--capacity", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--concurrent", action="store_true",
                    help="run the variants concurrently from Python threads (one stream each)")
    ap.add_argument("--serial-search", action="store_true",
                    help="one tds_search call per variant, one after another (default: one "
                         "tds_search_many call running the variants concurrently on side streams)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.variants = VARIANTS if args.variants == "all" else tuple(args.variants.split(","))
    args.serial = not args.concurrent
    args.batched = not args.concurrent and not args.serial_search
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    run_tds(args, ws, rank, local)


if __name__ == "__main__":
    main()
