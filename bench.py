"""Benchmark of the B200 distance threshold search (driver contract in DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config random-dense] [--d 0.03]
                    [--variants spatiotemporal,temporal]
    python bench.py --impl reference ...      # the CPU oracle arm (rank 0 only)

The workload is the one BASELINE.json's metric and north-star target are
quoted on: Random-dense-shaped, 65,536 x 192 = 12,582,912 segments, the S3
query set of 50,880 segments (Table 1),
GPUSpatioTemporal (m = 1,000, v = 2) at d = 0.03 kpc, with GPUTemporal
beside it.  The index is built once, before the timed region: the paper's
response time excludes the index build and the upload of D.

One step = tds_search of the full query set with each listed variant (the
first is the headline), inputs resident in HBM; the results stay
device-resident (T_search, T_fetch and T_gather are reported
separately).  ``value`` = #Q / T_search of the headline variant, query
segments per second over all ranks.  N GPUs (one process each): every rank
holds D and its index and the full query set and runs its work-balanced part
of each search (tds_search_part: equal shares of the exact pair tests); the
union of the parts is the answer, left sharded (strong scaling); T_search is
the max over ranks.  T_gather (the records to rank 0 over NCCL) is measured
after the timed region and reported separately.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "query segments/s & segment-pair tests/s vs HBM roofline at 1/2/4/8 B200"
DEFAULT_D = {"random-dense": 0.03, "random-dense-1m": 0.03, "merger": 1.0, "random-1m": 50.0,
             "scale-out": 50.0, "tiny": 2.0}
DEFAULT_VARIANTS = {"merger": "spatiotemporal,temporal,spatial", "random-1m": "temporal,spatiotemporal,spatial",
                    "tiny": "spatiotemporal,temporal,spatial"}
# SURVEY §8(d) algorithmic work: 42 FP32 operations per pair test, 25 more per
# hit; bytes: 36 per entry of D touched (32-B record + 4-B id), 48 per query
# (32-B record + 16-B schedule entry), 16 per result record, + 4 per entry
# id read from X/Y/Z (GPUSpatioTemporal)
OPS_PER_PAIR, OPS_PER_HIT = 42, 25
L2_FLUSH_BYTES = 256 << 20


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(config, d, kname, variant):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    ncu capture of the same configuration (profiles/ncu_traffic.json), else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return t[f"{config}|{d:g}|{kname}|{variant}"]
    except Exception:
        return None


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


def dist_setup():
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


def reduce_over_ranks(dist, x, dev, op):
    """Max / sum of a host float over ranks (NCCL needs a CUDA tensor, gloo a CPU one)."""
    import torch
    if dist is None:
        return x
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def make_workload(args):
    import synth
    w = synth.make_workload(args.config)
    w.d = args.d
    if args.m is not None:
        w.m_bins = args.m
    if args.v is not None:
        w.v_subbins = args.v
    if args.grid is not None:
        w.grid = (args.grid,) * 3
    return w


def config_dict(args, w, ws):
    return {"workload": f"{w.name}-shaped", "n_entries": int(w.D.shape[0]), "n_queries": int(w.Q.shape[0]),
            "d": w.d, "m_bins": w.m_bins, "v_subbins": w.v_subbins, "grid": list(w.grid),
            "variants": list(args.variants), "headline_variant": args.variants[0],
            "parallelism": (f"query-sharded x{ws}: work-balanced parts of the sorted schedule "
                            f"(tds_search_part), D + index replicated") if ws > 1 else "1 GPU",
            "index": "built once before the timed region (excluded, P:1301-1304)",
            "l2": "inputs (D 403 MB at Random-dense) exceed L2, and L2 is flushed (256 MiB write) before "
                  "every timed search, outside its events",
            "note": w.note}


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


def oracle_sample_size(w, seconds, cores, seed=0):
    """Queries of the workload the oracle answers in about ``seconds``."""
    import oracle
    rng = np.random.default_rng(seed)
    nq = w.Q.shape[0]
    cal = np.sort(rng.choice(nq, min(max(cores, 8), nq), replace=False))
    t = time.perf_counter()
    oracle.search(w.D, w.Q, w.d, qsel=cal, nthreads=cores)
    dt = max(time.perf_counter() - t, 1e-6)
    return int(min(nq, max(8, seconds * len(cal) / dt)))


def oracle_time(w, n, cores, seed):
    import oracle
    rng = np.random.default_rng(seed)
    sel = np.sort(rng.choice(w.Q.shape[0], n, replace=False))
    t = time.perf_counter()
    oracle.search(w.D, w.Q, w.d, qsel=sel, nthreads=cores)
    return time.perf_counter() - t


def run_reference(args, ws, rank):
    if rank != 0:
        return
    import oracle
    oracle.build()
    w = make_workload(args)
    cores = host_cores()
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    n = oracle_sample_size(w, per_step, cores)
    times = []
    for k in range(args.warmup + args.steps):
        el = oracle_time(w, n, cores, seed=1 + k)
        if k >= args.warmup:
            times.append(el)
    tot = sum(times)
    value = n * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "query segments/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, w, 1),
        "cpu_baseline": {"value": value, "unit": "query segments/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} random queries of {w.Q.shape[0]} per step, all-pairs fp64 against "
                                   f"all {w.D.shape[0]} entries"},
        "e2e": {"value": value, "unit": "query segments/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "pair_tests_per_s": n * w.D.shape[0] * len(times) / tot,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
def roofline(dk, nD, nQ, kind, peaks, n_sms, traffic, nA=0):
    """SURVEY §8(d) roofline of one pair-kernel launch: T_roof = max(B_alg / HBM,
    ops / FP32) against the measured kernel time; bound = the larger term."""
    secs = dk["pair_kernel_ms"] / 1e3
    hits = dk["results"]
    ops = OPS_PER_PAIR * dk["pair_tests"] + OPS_PER_HIT * hits
    nbytes = 36 * nD + 48 * nQ + 16 * hits + (4 * nD if kind == "spatiotemporal" else 0)
    if kind == "spatial":       # the cell-ordered copy: 32-B record + 4-B entry row + 4-B min cell per A entry
        nbytes = 40 * nA + 48 * nQ + 16 * hits
    hbm = float(peaks.get("hbm_gbs", 6548.8))                      # GB/s, measured copy
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu = n_sms * 128 * mhz * 1e6                                  # FP32 lane-ops/s (B200_PROFILING unit counts)
    t_hbm, t_alu = nbytes / (hbm * 1e9), ops / alu
    out = {"kernel": f"k_pair_range ({kind})",
           "alu": {"achieved": ops / secs / 1e12, "peak": alu / 1e12, "unit": "Tops/s (FP32 lane ops)",
                   "frac": t_alu / secs, "ops": ops,
                   "work": f"{OPS_PER_PAIR} x {dk['pair_tests']} pair tests + {OPS_PER_HIT} x {hits} hits"},
           "hbm": {"achieved": nbytes / secs / 1e9, "peak": hbm, "unit": "GB/s", "frac": t_hbm / secs,
                   "bytes": nbytes},
           "kernel_ms": dk["pair_kernel_ms"]}
    if t_hbm >= t_alu:
        out.update(bound="hbm", achieved=out["hbm"]["achieved"], peak=hbm, unit="GB/s", frac=t_hbm / secs,
                   peak_source="MEASURED_PEAKS.json hbm_gbs (copy, burst)")
    else:
        out.update(bound="alu", achieved=out["alu"]["achieved"], peak=alu / 1e12, unit="Tops/s",
                   frac=t_alu / secs,
                   peak_source=f"{n_sms} SMs x 128 FP32 lanes x sm_max_mhz {mhz:g} (MEASURED_PEAKS.json)")
    out["traffic"] = traffic["dram_bytes"] if traffic else None
    if traffic:
        out["traffic_source"] = traffic.get("source")
    return out


def run_tds(args, ws, rank, local):
    import torch
    import paper_1410_2698_b200 as tds
    tds.load_library()
    dev = torch.device("cuda", local)
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    w = make_workload(args)
    Dh = torch.from_numpy(w.D).pin_memory()
    Qh = torch.from_numpy(w.Q).pin_memory()
    D = Dh.to(dev)
    Q = Qh.to(dev)
    nQ, nD = int(w.Q.shape[0]), int(w.D.shape[0])
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    dist = None
    if ws > 1:
        import torch.distributed as dist

    def barrier():
        if dist is not None:
            dist.barrier()

    kinds = 0
    for v in args.variants:
        kinds |= tds.KINDS[v]
    e_b = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e_b[0].record(stream)
    idx = tds.Index(D, kinds=kinds, m=w.m_bins, v=w.v_subbins, grid=w.grid, stream=stream.cuda_stream)
    e_b[1].record(stream)
    torch.cuda.synchronize(dev)
    build_ms = e_b[0].elapsed_time(e_b[1])

    def search(kind, host=False):
        return idx.search(Qh if host else Q, w.d, kind=kind, capacity=args.capacity, stream=stream.cuda_stream,
                          part=rank, nparts=ws)

    def step(collect=None):
        rec = {}
        for kind in args.variants:
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = search(kind)
            e1.record(stream)
            st = r.stats()
            r.close()
            rec[kind] = (e0, e1, st)
        if collect is not None:
            collect.append(rec)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, barrier + synchronize on both sides of each
    launches0 = tds.kernel_launches()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    recs = []
    sampler.mark(0)
    for _ in range(args.steps):
        barrier()
        torch.cuda.synchronize(dev)
        step(recs)
        torch.cuda.synchronize(dev)
        barrier()
    sampler.mark(1)
    clocks = sampler.stop()
    launches = tds.kernel_launches() - launches0

    per_kind = {}
    for kind in args.variants:
        ms = [r[kind][0].elapsed_time(r[kind][1]) for r in recs]
        tot = reduce_over_ranks(dist, sum(ms), dev, "max")
        st = recs[0][kind][2]
        pt = [r[kind][2]["pair_tests"] for r in recs]
        pk = statistics.median(r[kind][2]["ms_pairs"] for r in recs)
        pt_all = reduce_over_ranks(dist, float(pt[0]), dev, "sum")
        res_all = reduce_over_ranks(dist, float(st["n_results"]), dev, "sum")
        per_kind[kind] = {
            "t_search_ms": tot / args.steps, "t_search_ms_rank0_median": statistics.median(ms),
            "t_search_ms_rank0_min": min(ms), "t_search_ms_rank0_max": max(ms),
            "query_segments_per_s": nQ * args.steps / (tot / 1e3),
            "pair_tests_per_s": pt_all * args.steps / (tot / 1e3),
            "pair_tests": int(pt_all), "results": int(res_all),
            "pair_kernel_ms": pk, "pair_tests_rank0": int(pt[0]), "results_rank0": int(st["n_results"]),
            "pairs_executed": int(st["pairs_executed"]), "refined_pairs_fp64": int(st["refined_pairs"]),
            "refined_pairs_fp32": int(st["refined32"]), "direct_records": int(st["direct_records"]),
            "passes": int(st["passes"]), "fallback_queries": int(st["fallback_queries"]),
            "ms_schedule": statistics.median(r[kind][2]["ms_schedule"] for r in recs),
            "pair_kernel_share_of_search": pk / statistics.median(ms),
        }
    head = args.variants[0]
    total_ms = per_kind[head]["t_search_ms"] * args.steps
    value = nQ * args.steps / (total_ms / 1e3)
    peaks = load_peaks()
    # dominant kernel: the headline search's pair kernel (rank 0's launch: its own part)
    dk = dict(per_kind[head])
    dk["pair_tests"], dk["results"] = dk["pair_tests_rank0"], dk["results_rank0"]
    kname = "k_pair_range"
    nA = idx.export_nbytes("fsg_A") // 4 if idx.kinds & tds.SPATIAL else 0
    roof = roofline(dk, nD, nQ / ws, head, peaks, n_sms,
                    ncu_traffic(args.config, w.d, kname, head) if ws == 1 else None, nA)
    for kind in args.variants[1:]:
        dk2 = dict(per_kind[kind])
        dk2["pair_tests"], dk2["results"] = dk2["pair_tests_rank0"], dk2["results_rank0"]
        r2 = roofline(dk2, nD, nQ / ws, kind, peaks, n_sms, None, nA)
        per_kind[kind]["roofline"] = {"bound": r2["bound"], "frac": r2["frac"], "alu_frac": r2["alu"]["frac"],
                                      "hbm_frac": r2["hbm"]["frac"]}

    # ---- fetch (A11) and gather, timed after the region (reported separately)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r = search(head)
    e0.record(stream)
    cols = r.fetch(device=True, stream=stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t_fetch = e0.elapsed_time(e1)
    t_gather = None
    if dist is not None:
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        tds_dist = __import__("paper_1410_2698_b200.dist", fromlist=["gather_results"])
        g = tds_dist.gather_results(*cols, dst=0)
        torch.cuda.synchronize(dev)
        t_gather = reduce_over_ranks(dist, 1e3 * (time.perf_counter() - t0), dev, "max")
        del g
    r.close()
    del cols

    # ---- e2e through the public API with host buffers: tds_search_stream takes the
    # queries from pinned host memory (copied in chunk by chunk inside the call) and
    # leaves the records in pinned host memory (copied out while the next chunk is
    # searched); the step ends when this rank's records are readable on the host
    e2e = None
    if not args.no_e2e:
        chunk = max(1, -(-nQ // 4))
        e2e_ms, d2h = [], []
        for k in range(args.steps + 1):
            flush.zero_()
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            r = idx.search_stream(Qh, w.d, kind=head, chunk=chunk, stream=stream.cuda_stream, part=rank, nparts=ws)
            blocks = r.host_records()                           # host-resident records (zero-copy)
            n = sum(len(b) for b in blocks)
            el = 1e3 * (time.perf_counter() - t0)
            r.close()
            barrier()
            if k:                                   # the first is a warm-up
                e2e_ms.append(el)
                d2h.append(16 * n)
        tot = reduce_over_ranks(dist, sum(e2e_ms), dev, "max")
        e2e = {"value": nQ * len(e2e_ms) / (tot / 1e3), "unit": "query segments/s",
               "h2d_bytes_per_step": int(w.Q.nbytes), "d2h_bytes_per_step": int(statistics.median(d2h)),
               "variant": head, "api": f"tds_search_stream (chunks of {chunk} queries, copies overlapped)",
               "timing": "host wall clock around tds_search_stream (queries from pinned host memory, records "
                         "into pinned host memory), synchronize on both sides, max over ranks; index resident"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        cores = host_cores()
        n = oracle_sample_size(w, args.cpu_seconds, cores)
        dt = oracle_time(w, n, cores, seed=7)
        cpu = {"value": n / dt, "unit": "query segments/s", "cores": cores, "kind": "oracle",
               "sample": f"{n} random queries of {nQ}, all-pairs fp64 vs all {nD} entries ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "query segments/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": config_dict(args, w, ws),
            "pair_tests_per_s": per_kind[head]["pair_tests_per_s"],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks,
            "breakdown": {"build_index_ms_untimed": build_ms, "t_fetch_ms": t_fetch, "t_gather_ms": t_gather,
                          "variants": per_kind},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="tds", choices=["tds", "reference"])
    ap.add_argument("--config", default="random-dense")
    ap.add_argument("--d", type=float, default=None)
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--v", type=int, default=None)
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--variants", default=None, help="comma list; the first is the headline")
    ap.add_argument("--capacity", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.d is None:
        args.d = DEFAULT_D.get(args.config, 1.0)
    v = args.variants or DEFAULT_VARIANTS.get(args.config, "spatiotemporal,temporal")
    args.variants = ("spatiotemporal", "temporal", "spatial") if v == "all" else tuple(v.split(","))
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    run_tds(args, ws, rank, local)


if __name__ == "__main__":
    main()
