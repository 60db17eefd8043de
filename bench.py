"""bench.py — time-to-R / join rows per second of the Figaro two-table path on B200.

Workload (BASELINE.json configs[3], the north-star config): uniform Cartesian
join of A (1e8 x 64) and B (1e8 x 64) fp64, i.e. 1e16 join rows, 128 columns;
synthetic SplitMix64 data generated on the device (no datasets).  A "step" is
one figaro_r (grouping-free for a Cartesian product): head/tail prefix pass over
B, fused Claim-1 assembly + TSQR leaves, TSQR tree, canonical R.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

N > 1 is launched by torchrun, one rank per GPU (NCCL): each rank generates its
row shard of A and B in place, exchanges the B column sums (carry all-gather),
computes its local R and all-gathers the R factors, then every rank runs the
same TSQR tree (`jq_tsqr_stack`).  Strong scaling: the join is fixed.

Timing: W >= 3 untimed steps, then K steps on the device stream with CUDA
events, barrier + synchronize on both sides, max over ranks.  Inputs (102.4 GB)
exceed the 126 MB L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.13   # measured DMMA (mma.sync f64) peak on this pool, profiles/r01_fp64_peak.txt
CONFIGS = {
    1: dict(m=1000, n=4, keys=None, name="C1 cartesian 1000x4 |x| 1000x4"),
    2: dict(m=1_000_000, n=16, keys="groups", key_groups=10_000, name="C2 natural join 10k keys x 100 rows/side, 16+16"),
    3: dict(m=10_000_000, n=32, keys="zipf", name="C3 Zipf(1.1) keys, 1e7 rows/side, 32+32"),
    4: dict(m=100_000_000, n=64, keys=None, name="C4 uniform cartesian 1e8 x 64 |x| 1e8 x 64"),
    5: dict(m=1_000_000, n=128, keys=None, want_v=True, name="C5 full SVD cartesian 1e6 x 128 |x| 1e6 x 128"),
}
METRIC = "join rows/sec (m1*m2/t), time-to-R"
# dram__bytes_read.sum + dram__bytes_write.sum per leaf-kernel launch (ncu --set full)
NCU_TRAFFIC = {(4, "footnote"): {"bytes": 53.184211e9 + 381.695744e6,
                                 "note": "first tsqr_ws2_kernel<CfgS<64,16,12,1,24,direct>> launch (side A, carry-free "
                                         "leaves; profiles/r02_ncu_ws64d_c4.md / _raw.csv, 63.63 ms under ncu): its own "
                                         "1e8 x 64 f64 rows = 51.2e9 algorithmic bytes (+3.9 %: the direct loads "
                                         "re-fetch a little of what the L2 prefetch brought in; writes: R and spills)"},
               (5, "footnote"): {"bytes": 1.061011e9 + 10.555904e6,
                                 "note": "first tsqr_ws2_kernel<CfgS<128,12,9,1,16,direct>> launch (side A, carry-free "
                                         "leaves; profiles/r02_ncu_ws128_c5.md, r02_ncu_ws128w12_c5_raw.csv, 2.474 ms "
                                         "under ncu): its own 1e6 x 128 f64 rows = 1.024e9 algorithmic bytes (+3.6 %)"}}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg_id: int):
    """The reference's CPU path: the oracle port of SPEC.md (numpy / LAPACK, all host
    threads) on a bounded sample of the same workload, extrapolated linearly in
    m1 + m2 (the Figaro CPU cost is O((m1+m2) N^2))."""
    import oracle as O
    cfg = CONFIGS[cfg_id]
    m_full = cfg["m"]
    m_s = min(m_full, args.ref_rows)
    a, b = O.config_tables(cfg_id, rows=m_s)
    join_full = float(m_full) * float(m_full) if cfg["keys"] is None else None
    if join_full is None:
        ag, bg = O.config_tables(cfg_id)
        _, _, ac, _, bc, _ = O.group_keys(ag.keys, bg.keys)
        join_full = float(np.sum(ac.astype(np.float64) * bc))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if cfg.get("want_v"):
            O.figaro_svd(a, b, want_vectors=True, lapack=True)
        else:
            O.figaro_r(a, b, lapack=True)
        t = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(t)
    t_sample = float(np.mean(times))
    t_full = t_sample * (2.0 * m_full) / (2.0 * m_s)
    value = join_full / t_full
    cores = len(os.sched_getaffinity(0))
    return {"value": value, "unit": "join rows/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(), "extrapolated": m_s < m_full, "sample_rows_per_side": m_s,
            "sample_join_rows": (float(m_s) ** 2 if cfg["keys"] is None else None),
            "sample": f"{cfg['name']} with m1=m2={m_s} rows (same SplitMix64 recipe), full SPEC "
                      f"pipeline reduce->LAPACK Householder QR->canonicalize, mean of {args.steps} after "
                      f"{args.warmup} warm-up = {t_sample:.3f} s, extrapolated x{m_full / m_s:.0f} linearly "
                      f"in m1+m2 to {t_full:.1f} s for the full config",
            "ms_per_step_sample": t_sample * 1e3, "ms_per_step_full_extrapolated": t_full * 1e3}


# ---------------------------------------------------------------- our arm
def make_inputs(cfg_id, rank, world, device):
    import torch
    from paper_2503_23385_b200 import datagen
    cfg = CONFIGS[cfg_id]
    m, n = cfg["m"], cfg["n"]
    a0, a1 = m * rank // world, m * (rank + 1) // world
    A = torch.empty((a1 - a0, n), dtype=torch.float64, device=device)
    B = torch.empty((a1 - a0, n), dtype=torch.float64, device=device)
    datagen.uniform(1000 * cfg_id + 1, a1 - a0, n, row0=a0, out=A)
    datagen.uniform(1000 * cfg_id + 2, a1 - a0, n, row0=a0, out=B)
    ka = kb = None
    if cfg["keys"] == "groups":
        ka = torch.from_numpy(datagen.near_equal_keys(m, cfg["key_groups"])).to(device)
        kb = ka.clone()
    elif cfg["keys"] == "zipf":
        # SURVEY.md §8d C3 recipe: per-row keys, then the stable (key, row) sort permutes
        # the data rows (GPU radix sort + gather; input preparation, outside the step)
        del A, B
        ta = datagen.zipf_table(1000 * cfg_id + 3, 1000 * cfg_id + 1, m, n, device=device)
        tb = datagen.zipf_table(1000 * cfg_id + 4, 1000 * cfg_id + 2, m, n, device=device)
        A, ka, B, kb = ta.data, ta.keys, tb.data, tb.keys
    torch.cuda.synchronize()
    return A, B, ka, kb, a0


def time_radix_sort(cfg_id, device):
    """Device time of the opt-in key sort of one unsorted C3 table (radix sort of the
    keys + gather of the data rows), CUDA events, mean of 3."""
    import torch
    from paper_2503_23385_b200 import datagen, argsort_keys, gather_rows
    cfg = CONFIGS[cfg_id]
    m, n = cfg["m"], cfg["n"]
    ku = datagen.zipf_keys(1000 * cfg_id + 3, m, out=torch.empty(m, dtype=torch.int64, device=device))
    x = datagen.uniform(1000 * cfg_id + 1, m, n, out=torch.empty((m, n), dtype=torch.float64, device=device))
    _, p0 = argsort_keys(ku)
    gather_rows(x, p0)          # warm-up of both kernels (module loading)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    s = torch.cuda.current_stream()
    t_sort = t_gather = 0.0
    for _ in range(3):
        e[0].record(s)
        _, perm = argsort_keys(ku)
        e[1].record(s)
        gather_rows(x, perm)
        e[2].record(s)
        torch.cuda.synchronize()
        t_sort += e[0].elapsed_time(e[1]) / 3
        t_gather += e[1].elapsed_time(e[2]) / 3
    return {"keys": m, "sort_ms": t_sort, "gather_ms": t_gather, "keys_per_s": m / (t_sort / 1e3),
            "gather_gbs": 2 * 8 * m * n / (t_gather / 1e3) / 1e9,
            "note": "stable LSD radix sort (jq_sort.cu, digit passes whose digit is constant skipped) of one "
                    "side's unsorted Zipf keys + row gather; input preparation, not in the timed step"}


def tsqr_flops(variant, cfg, m, n, st):
    """Algorithmic TSQR flops of one step (2*rows*N^2 - 2/3 N^3 per Householder QR)."""
    nn = 2 * n
    if cfg["keys"] is None:
        rows_a = rows_b = m - 1   # tails of each side (one group); dense: m1 + m2 - 1 rows
    else:
        rows_a = rows_b = None
    if variant == "dense":
        mr = (2 * m - 1) if cfg["keys"] is None else float(st["reduced_rows"])
        return 2.0 * mr * nn * nn - 2.0 / 3.0 * nn ** 3, f"2*M*N^2 - 2/3*N^3, M={int(mr)}, N={nn}"
    if rows_a is None:
        rows_a = rows_b = float(st["reduced_rows"]) / 2
    f = 2.0 * rows_a * n * n - 2.0 / 3.0 * n ** 3 + 2.0 * rows_b * n * n - 2.0 / 3.0 * n ** 3
    return f, f"footnote: 2*(m1-G)*n1^2 + 2*(m2-G)*n2^2 (-2/3 n^3 each), n1=n2={n}"


def join_rows(cfg_id, ka, kb):
    cfg = CONFIGS[cfg_id]
    if ka is None:
        return float(cfg["m"]) ** 2
    from paper_2503_23385_b200 import group_keys
    g = group_keys(ka, kb)
    return float(np.sum(g[2].astype(np.float64) * g[4]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=1_000_000)
    ap.add_argument("--variant", default="auto", choices=["auto", "footnote", "dense"],
                    help="figaro reduction timed as the headline (the other one is timed too and "
                         "reported under 'variants'); auto = what the library's default picks for "
                         "this shape (footnote from (m1 + m2)(n1 + n2) > 1e8 reduced elements)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pageable", action="store_true", help="skip the pageable-memory e2e step")
    ap.add_argument("--force-sharded", action="store_true",
                    help="(testing) run the multi-GPU code path even with one rank (torchrun, 1 process)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.variant == "auto":  # the library's "auto" rule (jq_api.cu use_footnote)
        c = CONFIGS[args.config]
        args.variant = "footnote" if 2.0 * c["m"] * 2 * c["n"] > 1e8 else "dense"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    sharded_path = world > 1 or args.force_sharded
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]


    if args.impl == "reference":
        if rank != 0:
            return
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))
        cb = run_reference(args, args.config)
        line = {"metric": METRIC, "value": cb["value"], "unit": cb["unit"], "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": cb["ms_per_step_full_extrapolated"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference",
                "config": {"workload": cfg["name"], "sample_rows_per_side": min(cfg["m"], args.ref_rows)},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                    "extrapolated", "ms_per_step_sample")},
                "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2503_23385_b200 import _native as N
    import paper_2503_23385_b200 as P

    torch.cuda.set_device(local)
    N.set_device(local)
    device = torch.device("cuda", local)
    if sharded_path:
        dist.init_process_group("nccl", device_id=device)

    keyed_sharded = sharded_path and cfg["keys"] is not None
    plan = None
    if keyed_sharded:
        # natural join over ranks: every rank builds the full key-sorted tables, the
        # key-range co-partition (sharded.co_partition, giant keys split by rows) picks
        # its rows, the rest is freed (input preparation, outside the timed step)
        from paper_2503_23385_b200 import sharded
        A, B, ka, kb, _ = make_inputs(args.config, 0, 1, device)
        jrows = join_rows(args.config, ka, kb)
        plan = sharded.co_partition(ka.cpu().numpy(), kb.cpu().numpy(), world)
        (x0, x1), (y0, y1) = plan.a_ranges[rank], plan.b_ranges[rank]
        A, ka = A[x0:x1].clone(), ka[x0:x1].clone()
        B, kb = B[y0:y1].clone(), kb[y0:y1].clone()
        a0 = x0
        torch.cuda.empty_cache()
    else:
        A, B, ka, kb, a0 = make_inputs(args.config, rank, world, device)
        jrows = join_rows(args.config, ka, kb) if world == 1 else float(cfg["m"]) ** 2
    m, n = cfg["m"], cfg["n"]
    nn = 2 * n
    lib, ctx = N.lib(), N.ctx()
    stream = torch.cuda.current_stream()

    def step():
        N.use_torch_stream(A)
        if not sharded_path:
            if cfg.get("want_v"):
                return P.figaro_svd(P.Table(A, ka), P.Table(B, kb), want_vectors=True).values
            return P.figaro_r(P.Table(A, ka), P.Table(B, kb))
        from paper_2503_23385_b200 import sharded
        if keyed_sharded:   # one all-gather (interior R, split-part R's and sums) over NCCL
            r = sharded.figaro_r_sharded_join(A, ka, B, kb, plan)
        elif N.get_variant() == "footnote":
            r = sharded.figaro_r_sharded_local(A, B, m, m, a0, a0)  # one all-gather (R + sums) over NCCL
        else:
            r = sharded.figaro_r_sharded(A, B, m, m, a0, a0)   # carry + R all-gathers over NCCL
        if cfg.get("want_v"):   # sigma and V of the (replicated) R on every rank, inside the step
            return P.svd_of_r(r, want_vectors=True).values
        return r

    def timed(variant, steps):
        N.set_variant(variant)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = Clocks(local)
        clocks.start()
        launches0 = N.kernel_launches()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        stage = []
        torch.cuda.synchronize()
        for i in range(steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            if world == 1:
                stage.append(N.last_timing())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = N.kernel_launches() - launches0
        clk = clocks.stop()
        step_ms = [s_.elapsed_time(e_) for s_, e_ in ev]
        ms = float(np.mean(step_ms))
        if world > 1:
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, step_ms, stage, launches, clk

    other = "dense" if args.variant == "footnote" else "footnote"
    ms_o, _, stage_o, _, _ = timed(other, max(1, min(args.steps, 3)))
    ms, step_ms, stage, launches, clk = timed(args.variant, args.steps)
    value = jrows / (ms / 1e3)

    # time-to-sigma (north star: R *and* singular values): figaro_svd without V on the
    # same inputs (for C5 the headline step already includes V)
    sigma_ms = None
    if not sharded_path and not cfg.get("want_v"):
        N.set_variant(args.variant)
        for _ in range(2):
            P.figaro_svd(P.Table(A, ka), P.Table(B, kb), want_vectors=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, min(args.steps, 3))
        e0.record(stream)
        for _ in range(reps):
            P.figaro_svd(P.Table(A, ka), P.Table(B, kb), want_vectors=False)
        e1.record(stream)
        torch.cuda.synchronize()
        sigma_ms = e0.elapsed_time(e1) / reps

    # ---- roofline of the dominant kernel (TSQR leaves, FP64 tensor pipe)
    roof, roof_hbm, stage_avg = None, None, None
    if stage:
        stage_avg = {k: float(np.mean([s[k] for s in stage])) for k in ("group_ms", "scan_ms", "tsqr_ms", "tree_ms", "svd_ms", "total_ms")}
        flops, alg = tsqr_flops(args.variant, cfg, m, n, stage[0])
        achieved = flops / (stage_avg["tsqr_ms"] / 1e3) / 1e12
        # DRAM traffic of one leaf launch from the ncu --set full capture of this config
        # (profiles/r01_ncu_ws2_c4.md): footnote C4, one side = 1e8 x 64 f64 rows
        traffic = NCU_TRAFFIC.get((args.config, args.variant))
        leaf_n = n if args.variant == "footnote" else 2 * n  # columns of one leaf
        if leaf_n <= 32:
            kname = ("tsqr_ws2_kernel (warp-specialised TSQR leaf: loader warps build the Claim-1 / tail rows, "
                     "chain warp runs the Cholesky panel factorisation, 12 data warps do the DMMA updates)")
        elif leaf_n <= 64:
            kname = ("tsqr_ws2_kernel<CfgS<64,16,12,1,24,direct>> (warp-specialised TSQR leaf: 12 data warps load "
                     "their 24 rows straight into the DMMA layout and run the tail transform there, chain warp "
                     "alone on SM sub-partition 0 runs the Cholesky panel factorisation)")
        elif leaf_n <= 128:
            kname = ("tsqr_ws2_kernel<CfgS<128,12,9,1,16,direct>> (warp-specialised TSQR leaf: 9 data warps load "
                     "their 16 rows straight into the DMMA layout and run the tail transform there, chain warp "
                     "alone on SM sub-partition 0)")
        else:
            kname = "tsqr_kernel (CTA-wide TSQR leaf, Cholesky / Gram panel chain + explicit fallback, DMMA updates)"
        roof = {"kernel": kname,
                "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS,
                "traffic": traffic["bytes"] if traffic else None,
                "traffic_note": traffic["note"] if traffic else "no ncu capture for this config",
                "peak_source": "measured FP64 DMMA peak (profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no FP64 figure",
                "algorithmic": alg, "share_of_step": stage_avg["tsqr_ms"] / ms}
        pk = peaks()
        # one side in the scan interval: dense scans B only (Claim 1); footnote scans A there
        # and runs B's tile pass inside A's TSQR interval (spare warps of the leaf)
        sides = 1
        gbs = (8.0 * m * n * sides) / (stage_avg["scan_ms"] / 1e3) / 1e9 if stage_avg["scan_ms"] > 0.05 else None
        # the tile-pass kernel(s) alone: CUDA events around each launch on its stream
        tile_ms = float(np.mean([s.get("scan_tile_ms", 0.0) for s in stage]))
        tile_bytes = float(np.mean([s.get("scan_tile_bytes", 0.0) for s in stage]))
        gbs_kernel = tile_bytes / (tile_ms / 1e3) / 1e9 if tile_ms > 0.05 and tile_bytes > 0 else None
        if gbs is None:
            # Cartesian footnote default: carry-free leaves, no prefix-scan pass in the step
            roof_hbm = {"kernel": None, "bound": "hbm", "achieved": None, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "note": "no HBM-bound pass in this step: the carry-free TSQR leaves transform their own "
                                "row blocks inside the leaf (N <= 64: the loader warp, from a TMA copy; N = 128: the data "
                                "warps, from their direct loads; every input byte read once); the head/tail "
                                "kernels' own roofline (reduced-matrix API, keyed configs) is in "
                                "profiles/r01_ncu_headtail.md and the C3 line"}
        if gbs and gbs_kernel:
            roof_hbm = {"kernel": "segscan_tile_kernel (head/tail tile pass: segmented column sums, one warp per "
                                  "1024-row tile)", "bound": "hbm",
                        "achieved": gbs_kernel, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": gbs_kernel / pk["hbm_gbs"], "frac_datasheet": gbs_kernel / 8000.0,
                        "kernel_ms": tile_ms, "bytes": tile_bytes,
                        "algorithmic": "8*rows*cols + 4*rows (segment ids) per launch, summed over the step's launches",
                        "stage": {"scan_ms": stage_avg["scan_ms"], "achieved_over_stage": gbs,
                                  "note": "the scan stage also holds the carry scan, the group fix-up and "
                                          "the head rows (latency-bound small kernels)"},
                        "peak_note": "MEASURED_PEAKS hbm_gbs is a copy (read+write) figure; this pass only reads"}
        elif gbs:
            roof_hbm = {"kernel": "segscan (head/tail prefix pass, tile sums + carry scan)", "bound": "hbm",
                        "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
                        "peak_note": "MEASURED_PEAKS hbm_gbs is a copy (read+write) figure; this pass only reads, "
                                     "so it can exceed it; vs the 8000 GB/s datasheet: frac_datasheet",
                        "frac_datasheet": gbs / 8000.0,
                        "algorithmic": f"8*m*n per scanned side x {sides} = {8 * m * n * sides} bytes read"}

    # ---- end-to-end through the public API with host buffers (N=1)
    e2e = None
    if sharded_path and not args.no_e2e and not keyed_sharded:
        e2e = run_e2e_sharded(args, A, B, m, a0, jrows, world, device)
    elif world == 1 and not args.no_e2e:
        N.set_variant(args.variant)
        r_ref = np.asarray(P.figaro_r(P.Table(A, ka), P.Table(B, kb)).cpu())
        host = to_host(A, B, ka, kb)
        del A, B
        A = B = None
        torch.cuda.empty_cache()
        e2e = run_e2e(args, host, jrows, r_ref)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        A = B = None
        torch.cuda.empty_cache()
        try:
            ra = argparse.Namespace(**vars(args))
            ra.steps, ra.warmup = 2, 1
            cb = run_reference(ra, args.config)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "extrapolated",
                                      "ms_per_step_sample")}
            # the measured same-config pair: our GPU path on the CPU sample's exact inputs
            cpu["gpu_same_sample"] = gpu_on_sample(args, cb["sample_rows_per_side"])
            cpu["gpu_same_sample"]["ratio_vs_cpu_sample"] = (cb["ms_per_step_sample"] /
                                                             cpu["gpu_same_sample"]["ms_per_step"])
        except Exception as exc:  # reported, never fatal for the GPU line
            cpu = {"value": None, "unit": "join rows/s", "cores": None, "kind": "port", "sample": f"failed: {exc}"}

    sort_info = None
    if world == 1 and cfg["keys"] == "zipf":
        A = B = None
        torch.cuda.empty_cache()
        sort_info = time_radix_sort(args.config, device)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "join rows/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "time_to_r_ms": ms, "time_to_sigma_ms": sigma_ms if sigma_ms is not None else ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (SplitMix64 uniform(0,1), generated on device)",
                "config": {"workload": cfg["name"], "m1": m, "m2": m, "n1": n, "n2": n,
                           "join_rows": jrows, "parallelism": (f"keyrange{world}" if keyed_sharded else f"rows{world}"),
                           "l2": "inputs 16*m*n bytes >> 126 MB L2 (no flush needed)" if m * n * 16 > 2**28 else "small config: L2-resident"},
                "gpu_launches": launches, "clocks": clk, "roofline": roof, "roofline_hbm": roof_hbm,
                "stages_ms": stage_avg, "step_ms_all": step_ms, "e2e": e2e, "cpu_baseline": cpu,
                "variant": args.variant, "radix_sort": sort_info,
                "variants": {args.variant: {"ms_per_step": ms, "value": value},
                             other: ({"ms_per_step": ms_o, "value": jrows / (ms_o / 1e3)} if ms_o else None)}}
        print(json.dumps(line), flush=True)
    if sharded_path:
        dist.destroy_process_group()


def gpu_on_sample(args, rows):
    """Device time of our path on the CPU baseline's sample (identical inputs: the same
    recipe and seeds at `rows` rows per side), so one GPU/CPU ratio is measured on the
    same config rather than extrapolated."""
    import torch
    import oracle as O      # the sample's generator (cpu_baseline leg only)
    import paper_2503_23385_b200 as P
    from paper_2503_23385_b200 import _native as N
    cfg = CONFIGS[args.config]
    a, b = O.config_tables(args.config, rows=rows)
    dev = lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ta, tb = P.Table(dev(a.data), dev(a.keys)), P.Table(dev(b.data), dev(b.keys))
    N.set_variant(args.variant)

    def run():
        if cfg.get("want_v"):
            return P.figaro_svd(ta, tb, want_vectors=True).values
        return P.figaro_r(ta, tb)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    e0.record(stream)
    for _ in range(reps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"ms_per_step": ms, "rows_per_side": rows, "variant": args.variant,
            "note": "device-resident inputs, CUDA events, mean of 10 after 3 warm-up"}


def rel_err_abs(r, r_ref) -> float:
    r, r_ref = np.abs(np.asarray(r)), np.abs(np.asarray(r_ref))
    return float(np.linalg.norm(r - r_ref) / max(np.linalg.norm(r_ref), 1e-300))


def to_host(A, B, ka, kb):
    """Copy the device tables into page-locked host memory (outside any timing)."""
    import torch
    cudart = torch.cuda.cudart()
    host = {}
    for name, t in (("A", A), ("B", B)):
        h = np.empty(tuple(t.shape), dtype=np.float64)
        rc = cudart.cudaHostRegister(h.ctypes.data, h.nbytes, 0)
        pinned = (int(rc) if not hasattr(rc, "value") else rc.value) == 0
        torch.cuda.synchronize()
        torch.from_numpy(h).copy_(t)
        host[name] = (h, pinned)
    host["ka"] = ka.cpu().numpy() if ka is not None else None
    host["kb"] = kb.cpu().numpy() if kb is not None else None
    return host


def run_e2e(args, host, jrows, r_ref):
    """figaro_r(Table(host), Table(host)) through the public API: the H2D copy of both
    tables (page-locked host memory) and the D2H of R are inside the timed region.
    Every timed R is compared with the device-resident path's R on the same inputs
    (`parity`: max relative Frobenius error of |R|, bar 1e-12).  A pageable-memory step
    (the plain-numpy drop-in caller) is timed after the pinned ones."""
    import torch
    import paper_2503_23385_b200 as P
    cudart = torch.cuda.cudart()
    try:
        ta = P.Table(host["A"][0], host["ka"])
        tb = P.Table(host["B"][0], host["kb"])
        nsteps = max(1, min(args.steps, 3))
        P.figaro_r(ta, tb)                     # warm-up (workspace sizing)
        times, errs = [], []
        for _ in range(nsteps):
            t0 = time.perf_counter()
            r = P.figaro_r(ta, tb)              # returns after the D2H of R
            times.append(time.perf_counter() - t0)
            errs.append(rel_err_abs(r, r_ref))
        t = float(np.mean(times))
        pageable = None
        if all(host[k][1] for k in ("A", "B")) and not args.no_pageable:
            for key in ("A", "B"):
                cudart.cudaHostUnregister(host[key][0].ctypes.data)
                host[key] = (host[key][0], False)
            P.figaro_r(ta, tb)            # warm-up: the context allocates its pinned staging ring once
            t0 = time.perf_counter()
            rp = P.figaro_r(ta, tb)
            tp = time.perf_counter() - t0
            pageable = {"value": jrows / tp, "ms_per_step": tp * 1e3, "steps": 1,
                        "parity": rel_err_abs(rp, r_ref),
                        "note": "plain numpy inputs: host threads copy them through a pinned staging ring "
                                "(allocated once per context, in the warm-up call)"}
        h2d = host["A"][0].nbytes + host["B"][0].nbytes
        if host["ka"] is not None:
            h2d += host["ka"].nbytes + host["kb"].nbytes
        return {"value": jrows / t, "unit": "join rows/s", "ms_per_step": t * 1e3, "steps": nsteps,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(r.nbytes),
                "pinned": True if pageable else bool(host["A"][1] and host["B"][1]),
                "parity": {"max_rel_err_vs_device_path": max(errs), "bar": 1e-12, "ok": max(errs) <= 1e-12},
                "pageable": pageable,
                "api": "paper_2503_23385_b200.figaro_r(Table(numpy), Table(numpy)) -> jq_figaro_r"}
    finally:
        for key in ("A", "B"):
            h, pinned = host[key]
            if pinned:
                cudart.cudaHostUnregister(h.ctypes.data)


def run_e2e_sharded(args, A, B, m, a0, jrows, world, device):
    """Multi-GPU end to end through the public sharded API (paper_2503_23385_b200.sharded):
    every rank copies its own row shards of A and B from page-locked host memory into
    HBM, runs figaro_r_sharded_local (local carry-free leaves, one NCCL all-gather, the
    fixed tree) and reads R back to the host -- all inside the timed region.  Timed with
    CUDA events on the launching stream around the whole step (the D2H of R synchronises),
    max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2503_23385_b200 import sharded, svd
    from paper_2503_23385_b200 import _native as N
    want_v = bool(CONFIGS[args.config].get("want_v"))
    N.use_torch_stream(A)
    if N.get_variant() == "footnote":
        r_ref = sharded.figaro_r_sharded_local(A, B, m, m, a0, a0).cpu().numpy()
    else:
        r_ref = sharded.figaro_r_sharded(A, B, m, m, a0, a0).cpu().numpy()
    host = to_host(A, B, None, None)
    cudart = torch.cuda.cudart()
    try:
        ha, hb = torch.from_numpy(host["A"][0]), torch.from_numpy(host["B"][0])
        stream = torch.cuda.current_stream()

        def step():
            A.copy_(ha, non_blocking=True)
            B.copy_(hb, non_blocking=True)
            N.use_torch_stream(A)
            if N.get_variant() == "footnote":
                r = sharded.figaro_r_sharded_local(A, B, m, m, a0, a0)
            else:
                r = sharded.figaro_r_sharded(A, B, m, m, a0, a0)
            if want_v:   # sigma and V of the replicated R, inside the step (read back with R)
                sv = svd.svd_of_r(r, want_vectors=True)
                sv.values.cpu(), sv.right_vectors.cpu()
            return r.cpu()

        step()                                   # warm-up
        torch.cuda.synchronize()
        dist.barrier()
        nsteps = max(1, min(args.steps, 3))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rs = []
        for _ in range(nsteps):
            r = step()
            rs.append(r)
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        err = max(rel_err_abs(x.numpy(), r_ref) for x in rs)
        t = torch.tensor([e0.elapsed_time(e1) / nsteps], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        return {"value": jrows / (ms / 1e3), "unit": "join rows/s", "ms_per_step": ms, "steps": nsteps,
                "h2d_bytes_per_step": int(host["A"][0].nbytes + host["B"][0].nbytes),
                "d2h_bytes_per_step": int(r.numpy().nbytes) + (8 * (r.shape[0] + r.shape[0] ** 2) if want_v else 0),
                "per_rank": True, "pinned": bool(host["A"][1] and host["B"][1]),
                "parity": {"max_rel_err_vs_device_path": err, "bar": 1e-12, "ok": err <= 1e-12,
                           "rank": int(os.environ.get("RANK", "0"))},
                "note": "per rank: its own shards' H2D and R's D2H (bytes above are one rank's); "
                        "time = max over ranks; H2D not overlapped with the leaves on this path",
                "api": "paper_2503_23385_b200.sharded.figaro_r_sharded_local (torch.distributed NCCL)"}
    finally:
        for key in ("A", "B"):
            h, pinned = host[key]
            if pinned:
                cudart.cudaHostUnregister(h.ctypes.data)


if __name__ == "__main__":
    main()
