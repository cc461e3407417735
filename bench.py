#!/usr/bin/env python
"""Benchmark of the B200 embedding-lookup path (BASELINE.json metric:
pooled lookups/sec and achieved HBM GB/s vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload = the largest single-GPU configuration of BASELINE.json,
configs[2]: 32 tables x 10M rows x dim 128 fp32
(163.84 GB in HBM), batch 4096, pooling 20, Zipf alpha 1.0, hot-row cache of
2% of all rows with the reference semantics (threshold None, sketch
admission, 64 staged admissions per batch, adaptive maintenance with the
memory model pinned). A step = one batch through the whole Ranker pipeline
(Ranker.execute_csr): validation, dedup, cache probe, plan, the fused
gather+pool (K4), ordered offers and maintenance (`run_ranker`).
`--config cfg2` (configs[1], Criteo-Kaggle-shaped, K4 alone) and the cold
control are extra lines. N>1 (torchrun, one rank per GPU) defaults to cfg4r
(100 tables x 1M rows, table-wise) sharded across the GPUs with the fused
NVLink exchange (see run_sharded), weak scaling, max-over-ranks device
time.

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def algorithmic_bytes(hb, dim, idx_bytes=4):
    nnz = int(hb.offsets[-1])
    n_bags = hb.offsets.size - 1
    return nnz * dim * 4 + nnz * idx_bytes + n_bags * 8 + n_bags * dim * 4


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.f = None

    def start(self):
        if os.environ.get("FX_NO_CLOCKS") == "1":  # A/B of the sampler's own cost
            self.proc = None
            return
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            # nvidia-smi start-up is slow when several ranks launch it at once:
            # wait for its first sample so a short timed region is still covered
            t_end = time.time() + 5.0
            while time.time() < t_end and os.path.getsize(self.f.name) == 0:
                time.sleep(0.05)
            time.sleep(0.1)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = [l.strip().split(", ") for l in open(self.f.name) if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 10:
                continue
            try:
                sm.append(float(r[2]))
                mx = float(r[3])
            except ValueError:
                continue
            for n, v in zip(names, r[6:10]):
                if v.strip() == "Active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "samples": len(sm), "reasons": sorted(reasons)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(config_name):
    """dram bytes per launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(config_name)
    return None


def build_cfg(cfg_key, rank, n_batches, alpha=None, table_rows=None):
    from flexemb_workload import CONFIGS, DlrmBatchGen
    cfg = dict(CONFIGS[cfg_key])
    if table_rows is not None:
        cfg["table_rows"] = (table_rows,) * len(cfg["table_rows"])
        cfg["name"] = cfg["name"] + f"-rows{table_rows}"
    if alpha is not None:
        cfg["alpha"] = alpha
        cfg["name"] = cfg["name"] + f"-alpha{alpha:g}"
    # cfg5 (row-wise fan-out) uses a fixed bijective row permutation so hot rows
    # do not all land on shard 0 (SURVEY §7 hard part 4)
    gen = DlrmBatchGen(cfg["table_rows"], cfg["alpha"], cfg["batch"], cfg["pooling"], seed=1000 * rank,
                       permute=cfg.get("permute", False))
    return cfg, [gen.next() for _ in range(n_batches)]


def cpu_baseline_port(hb, cfg, seconds_target=10.0):
    """The oracle's port of the reference pipeline on ONE host core over a
    bounded sample (a slice of one batch, row-reduced replica)."""
    from oracle.cpu_pipeline import RefPipelinePort
    port = RefPipelinePort(0, cfg["table_rows"], cfg["dim"], row_cap=20_000)
    samples, bags, t0 = 0, 0, time.perf_counter()
    F = len(hb.feature_tables)
    while time.perf_counter() - t0 < seconds_target and samples < hb.batch_size:
        port.run(hb, range(samples, min(samples + 16, hb.batch_size)))
        samples = min(samples + 16, hb.batch_size)
    dt = time.perf_counter() - t0
    bags = samples * F
    return {"value": bags / dt, "unit": "pooled lookups/s", "cores": 1, "kind": "port",
            "sample": f"{samples} samples x {F} features of one cfg2 batch ({bags} bags, {dt:.1f}s), "
                      "reference Ranker pipeline restated in oracle/cpu_pipeline.py (threshold 2, cache off), "
                      "tables row-reduced to 20K rows (per-row cost is table-size independent)"}


def ranker_config(cfg, cache_frac, extra=None):
    """The `config` dict both arms print for the Ranker (cfg3) workload."""
    d = {"workload": cfg["name"] + f"-cache{cache_frac * 100:g}pct", "global_batch": cfg["batch"],
         "per_gpu_batch": cfg["batch"], "pooling": cfg["pooling"] if not isinstance(cfg["pooling"], tuple)
         else list(cfg["pooling"]), "alpha": cfg["alpha"], "dim": cfg["dim"], "tables": len(cfg["table_rows"]),
         "rows_per_table": cfg["table_rows"][0], "cache_rows_frac": cache_frac, "pushdown_threshold": None,
         "admission": "sketch", "admit_per_batch": 64, "pipeline": "Ranker.execute_csr (validate, dedup, probe, "
         "plan, gather+pool, offers, maintenance)"}
    if extra:
        d.update(extra)
    return d


def sharded_config(cfg, args, world):
    """The `config` dict both arms print for the N>1 sharded workload (derived
    from the configuration and the flags only, so the reference arm prints the
    identical dict)."""
    rows, B, F, mode = cfg["table_rows"], cfg["batch"], len(cfg["table_rows"]), args.mode
    repl = ([t for t, n in enumerate(rows) if n <= args.replicate_rows]
            if mode == "tablewise" and args.exchange == "p2p" else [])
    if len(repl) == F:
        repl = repl[:-1]
    return {"workload": cfg["name"] + f"-{mode}", "global_batch": B * world, "per_gpu_batch": B,
            "pooling": list(cfg["pooling"]) if isinstance(cfg["pooling"], tuple) else cfg["pooling"],
            "alpha": cfg["alpha"], "dim": cfg["dim"], "tables": F, "rows_per_table": rows[0],
            "cache_rows_frac": 0.0,
            "parallelism": f"{mode}-sharded x{world} ({args.exchange} exchange)"
                           + (f", {len(repl)} small tables replicated" if repl else "")
                           + (f", {args.partial} partials" if mode == "rowwise" else "")
                           + (f", pushdown threshold {args.threshold} (raw fetch over NVLink below)"
                              if mode == "rowwise" and args.threshold else "")
                           + (", pipelined (depth 2)" if args.exchange == "p2p" and not args.sync else ""),
            "l2": f"inputs larger than L2: a distinct batch per rank and step over "
                  f"{sum(rows) * cfg['dim'] * 4 / 1e9:.1f} GB of tables"}


def cfg3_config(cfg, args):
    """The `config` dict both arms print for the N=1 cfg3 Ranker workload."""
    N, T, D = cfg["table_rows"][0], len(cfg["table_rows"]), cfg["dim"]
    budget = int(T * N * args.cache) * D * 4
    return ranker_config(cfg, args.cache, {
        "parallelism": "single" + (", whole Ranker batch replayed as one CUDA graph" if args.graph_step else ""),
        "l2": f"inputs larger than L2: distinct batches (up to 40, cycled) over {N * T * D * 4 / 1e9:.1f} GB of "
              f"tables + {budget / 1e9:.2f} GB of cached rows"})


REF_ROWS = 20_000  # row-reduced replica for the reference's host tables


def ref_baseline(cfg, cache_frac, procs, samples_per_step, steps, warmup):
    """The unmodified reference (oracle/_ref/embserve) over `procs` forked
    host processes; returns (bags/s, per-step wall ms, cores, sample text)."""
    from oracle import ref_arm
    if not ref_arm.available():
        return None
    B, L = cfg["batch"], cfg["pooling"] if not isinstance(cfg["pooling"], tuple) else cfg["pooling"][0]
    T = len(cfg["table_rows"])
    t0 = time.perf_counter()
    res = ref_arm.run_parallel(procs, T, REF_ROWS, cfg["dim"], B, L, cfg["alpha"], cache_frac, samples_per_step,
                               steps, warmup)
    wall = time.perf_counter() - t0
    bags = sum(b for r, _ in res for b, _ in r)
    busy = max(sum(t for _, t in r) for r, _ in res)
    step_ms = [1000 * max(r[i][1] for r, _ in res) for i in range(steps)]
    sample = (f"{procs} forked process(es) x {steps} timed steps (after {warmup} warm-up steps) of a "
              f"{samples_per_step}-lookup batch ({samples_per_step * T} bags) each, through the unmodified "
              f"reference (oracle/_ref copy of embserve: Ranker.run_trace with VirtualTransport, "
              f"AdaptiveCache {cache_frac * 100:g}% of rows, threshold None, sketch admission, admit 64); "
              f"tables row-reduced to {REF_ROWS} rows per table (indices mod rows; steady-state reference "
              f"rate measured within 10% at 20K vs 200K rows, profiles/r2_reference_rows.json); "
              f"{wall:.0f}s wall")
    return bags / busy, statistics.median(step_ms), procs, sample


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (the unmodified embserve Ranker, copied into oracle/_ref by build()) on
    all host cores, rank 0 only; this process never imports the product
    package (libflexemb.so stays unloaded)."""
    if rank != 0:
        return
    cfg_key = args.config or "cfg3"
    cfg, _ = build_cfg(cfg_key, 0, 0, args.alpha)
    procs = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    # N>1: the GPU arm's sharded lookup has no cache, so neither has the reference's Ranker here
    cache_frac = 0.0 if world > 1 else args.cache
    r = ref_baseline(cfg, cache_frac, procs, samples_per_step=32, steps=args.steps, warmup=args.warmup)
    assert not any(k.startswith("paper_2410_12794_b200") for k in sys.modules), "reference arm loaded the product"
    if r is None:
        emit({"impl": "reference", "unavailable": "oracle/_ref/embserve missing (run __graft_entry__.build())"}, args)
        return
    value, step_ms, cores, sample = r
    line = {
        "impl": "reference", "metric": "pooled lookups/s (bags/s)", "value": value, "unit": "pooled lookups/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 rows, f64 accumulate",
        "data": "synthetic",
        "config": sharded_config(cfg, args, world) if world > 1 else (cfg3_config(cfg, args) if cfg_key == "cfg3"
                                                                     else ranker_config(cfg, args.cache)),
        "cpu_baseline": {"value": value, "unit": "pooled lookups/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "pooled lookups/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line, args)


def emit(line: dict, args) -> None:
    """Print the bench JSON line; with --report DIR also write it as a
    summary in the reference's MetricsReport schema (bench/report.py)."""
    print(json.dumps(line), flush=True)
    if getattr(args, "report", None):
        from paper_2410_12794_b200.report import from_bench_line
        from_bench_line(line).write(args.report)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    help="workload: cfg3 (N=1 default: full Ranker pipeline with the cache), cfg2 / cfg1 (K4 "
                         "alone), cfg4r (N>1 default), cfg4, cfg5")
    ap.add_argument("--cache", type=float, default=0.02, help="cfg3: cache budget as a fraction of all rows")
    ap.add_argument("--graph-step", type=int, default=1,
                    help="cfg3: replay the whole Ranker batch as one CUDA graph (Ranker.capture_csr); 0 = eager "
                         "execute_csr(sync=False) per batch")
    ap.add_argument("--batches", type=int, default=4, help="distinct batches cycled through")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--alpha", type=float, default=None, help="override Zipf alpha (0 = uniform cold control)")
    ap.add_argument("--table-rows", type=int, default=None, help="override every table's row count (cold control)")
    ap.add_argument("--mode", default="tablewise", choices=["tablewise", "rowwise"], help="N>1 sharding")
    ap.add_argument("--sync", action="store_true",
                    help="N>1 fused exchange: synchronous steps (2 barriers each) instead of the pipelined stream "
                         "(push of step k+1 overlapping the gather of step k, one barrier per step)")
    ap.add_argument("--partial", default="f32", choices=["f64", "f32"],
                    help="N>1 row-wise partial format: f32 (default) = the reference's PartialResult / "
                         "combine_partials semantics, bit-identical to its hierarchical result and half the "
                         "NVLink bytes; f64 = bit-identical to the flat f64 pool instead")
    ap.add_argument("--graph", type=int, default=0,
                    help="N=1: capture this many batch launches per CUDA graph and time graph replays")
    ap.add_argument("--replicate-rows", type=int, default=None,
                    help="N>1 table-wise: replicate tables with <= this many rows on every rank (hybrid "
                         "placement: small tables data-parallel, big tables table-sharded); 0 = pure table-wise")
    ap.add_argument("--threshold", type=int, default=0,
                    help="N>1 row-wise fused exchange: the reference's pushdown threshold (groups below it are "
                         "raw-fetched over NVLink by the requester); 0 = push every group down")
    ap.add_argument("--report", default=None,
                    help="also write the line as a MetricsReport-schema summary (+ text report) into this dir")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 pooled-result exchange: fused NVLink peer stores (p2p) or NCCL all-to-all")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    if args.config is None:
        args.config = "cfg3" if world == 1 else "cfg4r"
    if args.replicate_rows is None:
        args.replicate_rows = 1_000_000 if args.config == "cfg2" else 0
    if args.impl == "reference":
        return run_reference(args, rank, world)

    # NCCL's own log lines (e.g. "NCCL version ..." under NCCL_DEBUG=WARN)
    # default to stdout; keep stdout to the one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2410_12794_b200 as P
    from paper_2410_12794_b200.engine import CsrBatch, HostLookup, LookupEngine
    if world > 1:
        return run_sharded(args, rank, world, local)
    if args.config == "cfg3":
        return run_ranker(args, rank, world, local)

    cfg, host_batches = build_cfg(args.config, rank, args.batches, args.alpha, args.table_rows)
    dim = cfg["dim"]
    metas = [P.TableMeta(t, n, dim) for t, n in enumerate(cfg["table_rows"])]
    placement = [P.ShardSpec(t, 0, n, rank) for t, n in enumerate(cfg["table_rows"])]
    t0 = time.perf_counter()
    dep = P.init_store(metas, placement, seed=0)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    eng = LookupEngine(dep)
    dev = eng.device
    batches = [CsrBatch(torch.from_numpy(hb.indices).to(dev), torch.from_numpy(hb.offsets).to(dev),
                        hb.feature_tables, hb.feature_ops, hb.batch_size) for hb in host_batches]
    B = cfg["batch"]
    outs = [torch.empty((B, len(cfg["table_rows"]) * dim), dtype=torch.float32, device=dev) for _ in range(2)]
    bytes_per = [algorithmic_bytes(hb, dim) for hb in host_batches]
    bags_per = B * len(cfg["table_rows"])
    stream = torch.cuda.current_stream()

    # correctness gate before timing (the pooled output is checked against the oracle in tests)
    eng.pool(batches[0], out=outs[0], check=True)
    for i in range(args.warmup):
        eng.pool(batches[i % len(batches)], out=outs[i % 2], check=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = 0
    tot_bytes = 0
    if args.graph > 0:
        gb = [batches[i % len(batches)] for i in range(args.graph)]
        gouts = [outs[i % 2] for i in range(args.graph)]
        graph = eng.capture(gb, gouts)
        graph.replay()
        torch.cuda.synchronize()
        reps = max(1, args.steps // args.graph)
        args.steps = reps * args.graph
        ev0.record(stream)
        for _ in range(reps):
            graph.replay()
        launches = args.steps
        tot_bytes = sum(bytes_per[i % len(batches)] for i in range(args.graph)) * reps
    else:
        ev0.record(stream)
        for i in range(args.steps):
            eng.pool(batches[i % len(batches)], out=outs[i % 2], check=False)
            launches += 1
            tot_bytes += bytes_per[i % len(batches)]
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    eng.raise_if_bad(batches[0])
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = bags_per * args.steps * world / (ms_max / 1e3)
    kernel_ms = ms / launches
    achieved = (tot_bytes / launches) / (kernel_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()

    # e2e: host pinned CSR in -> host pooled out through the public host API
    # (HostLookup.stream: H2D / K4 / D2H of consecutive batches overlapped)
    e2e = None
    if not args.no_e2e:
        hl = HostLookup(eng)
        pinned = [CsrBatch(torch.from_numpy(hb.indices).pin_memory(), torch.from_numpy(hb.offsets).pin_memory(),
                           hb.feature_tables, hb.feature_ops, hb.batch_size) for hb in host_batches]
        for _ in hl.stream([pinned[i % len(pinned)] for i in range(4)]):
            pass
        torch.cuda.synchronize()
        ksteps = max(3, min(args.steps, 100))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d = d2h = 0
        e0.record(stream)
        for i, out_h in enumerate(hl.stream([pinned[i % len(pinned)] for i in range(ksteps)])):
            pb = pinned[i % len(pinned)]
            h2d += pb.indices.numel() * pb.indices.element_size() + pb.offsets.numel() * 8
            d2h += out_h.numel() * 4
        e1.record(stream)
        e1.synchronize()
        ems = e0.elapsed_time(e1)
        # synchronous single-batch API for reference
        for i in range(3):
            hl.lookup(pinned[i % len(pinned)])
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(20):
            hl.lookup(pinned[i % len(pinned)])
        s1.record(stream)
        s1.synchronize()
        sync_val = bags_per * 20 / (s0.elapsed_time(s1) / 1e3)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": bags_per * ksteps * world / (ems / 1e3), "unit": "pooled lookups/s",
               "h2d_bytes_per_step": h2d // ksteps, "d2h_bytes_per_step": d2h // ksteps,
               "steps": ksteps, "api": "engine.HostLookup.stream (pinned host CSR -> pinned host pooled, "
                                       "3-stream pipelined, depth 3)",
               "sync_api_value": sync_val}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_port(host_batches[0], cfg)

    if rank == 0:
        tr = committed_traffic(cfg["name"])
        line = {
            "metric": "pooled lookups/s (bags/s)", "value": value, "unit": "pooled lookups/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 rows, f64 accumulate", "data": "synthetic",
            "config": {"workload": cfg["name"], "global_batch": B * world, "per_gpu_batch": B,
                       "pooling": list(cfg["pooling"]) if isinstance(cfg["pooling"], tuple) else cfg["pooling"],
                       "alpha": cfg["alpha"], "dim": dim, "tables": len(cfg["table_rows"]),
                       "parallelism": ("single" if world == 1 else f"replicas{world}")
                                      + (f", CUDA graph of {args.graph} launches" if args.graph else ""),
                       "l2": f"inputs larger than L2: {len(batches)} distinct batches cycled, "
                             f"{bytes_per[0] / 1e9:.2f} GB algorithmic bytes/batch over "
                             f"{sum(cfg['table_rows']) * dim * 4 / 1e9:.1f} GB of tables",
                       "init_store_s": round(init_s, 2)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": tr, "peak_source": peak_src,
                         "kernel": (f"fx::k_pool_bulk<G=32,CR=12> (TMA bulk-copy staged gather+pool, "
                                    f"D={dim})" if os.environ.get("FX_POOL_VARIANT", "2") == "2" and dim == 128
                                    else f"fx::k_pool_async<G={min(32, dim // 4)},CR={12 if dim == 64 else 16}> "
                                         f"(cp.async-staged gather+pool, D={dim})"),
                         "bytes_per_launch": tot_bytes / launches, "launch_ms": kernel_ms,
                         "note": ("L2-assisted: Zipf hot rows and the small tables are served from the 126 MB "
                                  "L2, so DRAM traffic (ncu, `traffic`) is well below the algorithmic bytes and "
                                  "frac can exceed 1; the DRAM-bound cold control (bench.py --alpha 0 "
                                  "--table-rows 4000000) measures 0.86-0.88 of the copy peak "
                                  "(profiles/r1_summary.md)")
                         if (tr and tr < 0.9 * tot_bytes / launches) else None},
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        emit(line, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_ranker(args, rank, world, local):
    """N=1 headline: cfg3 through the whole Ranker pipeline. `value` times K
    consecutive distinct batches already in HBM through Ranker.execute_csr
    (sync=False: the fused cache step + K4 on a side stream, no host sync);
    `e2e` runs Ranker.stream_host (pinned host CSR in, pinned host pooled out,
    H2D / step / D2H overlapped on three streams)."""
    import torch
    import paper_2410_12794_b200 as P
    from paper_2410_12794_b200 import cache as C
    from paper_2410_12794_b200.ranker import Ranker, RankerParams

    n_timed = min(args.steps, 40)       # distinct timed batches (cycled beyond 40 steps)
    n_dev = args.warmup + n_timed
    cfg, host_batches = build_cfg(args.config, rank, n_dev + max(3, min(args.steps, 40)) + 3, args.alpha,
                                  args.table_rows)
    T, D, B = len(cfg["table_rows"]), cfg["dim"], cfg["batch"]
    N = cfg["table_rows"][0]
    metas = [P.TableMeta(t, n, D) for t, n in enumerate(cfg["table_rows"])]
    placement = [P.ShardSpec(t, 0, n, 0) for t, n in enumerate(cfg["table_rows"])]
    t0 = time.perf_counter()
    dep = P.init_store(metas, placement, seed=0)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    rows_c = int(sum(cfg["table_rows"]) * args.cache)
    budget = rows_c * D * 4
    cache = C.AdaptiveCache(budget, admission="sketch", max_dim=D, slot_capacity=rows_c + 1,
                            sketch_capacity=8_000_000)
    rk = Ranker(dep, P.build_routing(metas, placement), None,
                RankerParams(pushdown_threshold=None, admit_per_batch=64),
                cache=cache, policy=C.CachePolicy(C.MemoryModel(budget + 1_000 + B, 1_000, 1)),
                tracker=C.LoadTracker(16, 10 ** 9, 0))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    dbs = [(torch.from_numpy(hb.indices).to(dev), torch.from_numpy(hb.offsets).to(dev))
           for hb in host_batches[:n_dev]]
    ft, fo = host_batches[0].feature_tables, host_batches[0].feature_ops
    # warm-up: fills the cache to its steady state (first batches insert everything)
    for i in range(args.warmup):
        rk.execute_csr(*dbs[i], ft, fo, B, batch_id=i, sync=False)
    rk.sync()   # resolves metrics; may grow the sketch table / rebuild the step outside the timed region
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    graph = None
    if args.graph_step:
        # static input buffers: each timed step copies its batch in (D2D, inside
        # the timed region), then replays the captured batch
        sidx, soffs = dbs[0][0].clone(), dbs[0][1].clone()
        lc0 = rk._step.launches()
        graph = rk.capture_csr(sidx, soffs, ft, fo, B)
        n_graph_launches = rk._step.launches() - lc0  # step kernels recorded into the graph (+ K4)
        torch.cuda.synchronize()
        for i in range(2):  # graph warm-up replays on warm-up batches (cache state keeps evolving)
            sidx.copy_(dbs[i][0])
            soffs.copy_(dbs[i][1])
            graph.replay(batch_id=-1 - i)
        rk.sync()
    # K4 alone, timed on its own stream over the timed batches (events inside
    # a replayed graph are not available): the roofline kernel's launch time,
    # at full occupancy (inside the step it shares the SMs: FX_OUT_SHARE)
    k4_ev = []
    pst = rk._pool_stream
    for i in range(min(args.steps, n_timed)):
        idx_, offs_ = dbs[args.warmup + i]
        from paper_2410_12794_b200.dedup import sample_major_starts  # noqa: F401
        out_ = torch.empty((B, T * D), dtype=torch.float32, device=dev)
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pst.wait_stream(stream)
        with torch.cuda.stream(pst):
            e_a.record(pst)
            from paper_2410_12794_b200.ranker import CsrLayout
            rk._pool_sample_major(CsrLayout(idx_, offs_, None, None, None, [], None, None, None, B), out_, ft, fo, B,
                                  share=False)
            e_b.record(pst)
        k4_ev.append((e_a, e_b))
    torch.cuda.synchronize()
    k4_ms = [a.elapsed_time(b) for a, b in k4_ev]
    l0 = rk._step.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    th0 = time.perf_counter()
    if graph is not None:
        for i in range(args.steps):
            j = args.warmup + i % n_timed
            sidx.copy_(dbs[j][0])
            soffs.copy_(dbs[j][1])
            graph.replay(batch_id=args.warmup + i)
    else:
        for i in range(args.steps):
            rk.execute_csr(*dbs[args.warmup + i % n_timed], ft, fo, B, batch_id=args.warmup + i, sync=False)
    host_ms = (time.perf_counter() - th0) * 1e3 / args.steps
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = ((n_graph_launches + 1) * args.steps if graph is not None
                else rk._step.launches() - l0 + args.steps)
    ms = ev0.elapsed_time(ev1)
    rk.sync()
    mets = rk.batch_metrics[args.warmup:]
    hit = sum(m.cache_hits for m in mets) / max(1, sum(m.cache_hits + m.cache_misses for m in mets))
    lat = sorted(m.latency * 1e3 for m in mets)
    bags = B * T
    value = bags * args.steps / (ms / 1e3)
    tot_bytes = sum(algorithmic_bytes(host_batches[args.warmup + i % n_timed], D) for i in range(args.steps))
    k4_mean = sum(k4_ms) / len(k4_ms)
    k4_achieved = tot_bytes / args.steps / (k4_mean / 1e3) / 1e9
    pipe_achieved = tot_bytes / (ms / 1e3) / 1e9
    peak, peak_src = measured_peak()

    e2e = None
    if not args.no_e2e:
        ksteps = max(3, min(args.steps, 40))
        hbs = host_batches[n_dev:n_dev + ksteps + 3]
        pinned = [(torch.from_numpy(hb.indices).pin_memory(), torch.from_numpy(hb.offsets).pin_memory())
                  for hb in hbs]
        for _ in rk.stream_host(pinned[:3], ft, fo, B, first_batch_id=10_000):
            pass
        torch.cuda.synchronize()
        h2d = sum(ih.numel() * ih.element_size() + oh.numel() * 8 for ih, oh in pinned[3:])
        d2h = 0
        t0 = time.perf_counter()
        for out_h in rk.stream_host(pinned[3:], ft, fo, B, first_batch_id=20_000):
            d2h += out_h.numel() * 4
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        e2e = {"value": bags * ksteps / e2e_s, "unit": "pooled lookups/s", "h2d_bytes_per_step": h2d // ksteps,
               "d2h_bytes_per_step": d2h // ksteps, "steps": ksteps,
               "api": "Ranker.stream_host (pinned host CSR -> pinned host pooled [B, F*D]; H2D, the whole Ranker "
                      "batch (two captured graphs, ping-pong buffers) and D2H on three streams; wall clock)"}

    cpu = None
    if not args.no_cpu:
        r = ref_baseline(cfg, args.cache, 1, samples_per_step=32, steps=8, warmup=8)
        if r is not None:
            cpu = {"value": r[0], "unit": "pooled lookups/s", "cores": 1, "kind": "reference", "sample": r[3]}

    prof = os.path.join(ROOT, "profiles", "r2_cfg3_kernels.json")
    shares = json.load(open(prof)) if os.path.exists(prof) else None
    tr3 = committed_traffic(cfg["name"])  # ncu DRAM bytes per K4 launch (profiles/traffic.json)
    line = {
        "metric": "pooled lookups/s (bags/s)", "value": value, "unit": "pooled lookups/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 rows, f64 accumulate", "data": "synthetic",
        "config": cfg3_config(cfg, args), "init_store_s": round(init_s, 2),
        "hit_rate": hit, "latency_ms": {"p50": lat[len(lat) // 2], "max": lat[-1]},
        "host_enqueue_ms_per_step": host_ms,
        "roofline": {"bound": "hbm", "achieved": k4_achieved, "peak": peak, "unit": "GB/s",
                     "frac": k4_achieved / peak, "traffic": tr3, "peak_source": peak_src,
                     "dram_gbs": (tr3 / (k4_mean * 1e6)) if tr3 and k4_mean else None,
                     "kernel": "fx::k_pool_bulk (fused gather+pool K4 of the Ranker step, timed alone on its stream "
                               "over the timed batches)",
                     "bytes_per_launch": tot_bytes / args.steps, "launch_ms": k4_mean,
                     "pipeline": {"achieved": pipe_achieved, "frac": pipe_achieved / peak,
                                  "note": "algorithmic bytes of the batch over the whole Ranker step (cache "
                                          "bookkeeping is latency-bound hash / LRU work, not credited)"},
                     "kernel_shares": shares},
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    emit(line, args)


def run_sharded(args, rank, world, local):
    """N>1: the cfg2 tables sharded across the ranks, every rank a requester
    with its own 4096-sample batch stream (weak scaling). Default placement is
    hybrid table-wise: tables <= 1M rows replicated on every rank and pooled
    locally, the big tables table-sharded (SURVEY §8(e) cfg4 pattern); use
    --replicate-rows 0 for pure table-wise, --mode rowwise for the cfg5
    pattern. Default exchange is fused over NVLink (--exchange p2p): a step =
    validate + push index slices into the owners' staging (P2P stores) ->
    barrier -> one owner gather+pool (K4) launch storing pooled rows into the
    requesters' buffers -> barrier (-> K5 combine, row-wise). --exchange nccl
    runs the all-to-all baseline (K1 route/bucket -> C1 -> K4 -> C2)."""
    import torch
    import torch.distributed as dist
    from paper_2410_12794_b200.sharded import P2PShardedLookup, ShardedLookup, rowwise_placement, tablewise_placement
    from paper_2410_12794_b200.store import TableMeta
    cfg, host_batches = build_cfg(args.config, rank, args.batches, args.alpha, args.table_rows)
    rows, dim, B = cfg["table_rows"], cfg["dim"], cfg["batch"]
    F = len(rows)
    mode = args.mode
    repl = ([t for t, n in enumerate(rows) if n <= args.replicate_rows]
            if mode == "tablewise" and args.exchange == "p2p" else [])
    if len(repl) == F:  # everything would be replicated: keep at least the largest table sharded
        repl.remove(max(range(F), key=lambda t: rows[t]))
    big = [t for t in range(F) if t not in repl]
    if mode == "tablewise":
        sub = tablewise_placement([rows[t] for t in big], world)
        from paper_2410_12794_b200.store import ShardSpec
        placement = [ShardSpec(big[s.table_id], s.start, s.end, s.server_id) for s in sub]
    else:
        placement = rowwise_placement(rows, world)
    metas = [TableMeta(t, n, dim) for t, n in enumerate(rows)]
    dev = torch.device("cuda", local)
    t0 = time.perf_counter()
    if args.exchange == "p2p":
        max_nnz = int(max(int(hb.offsets[-1]) for hb in host_batches) * 1.05) + 1024
        sl = P2PShardedLookup(metas, placement, 0, tuple(range(F)), ("sum",) * F, B, rank, world, dev, mode=mode,
                              replicated_tables=repl, max_nnz=max_nnz, partial_dtype=args.partial,
                              pushdown_threshold=(args.threshold or None) if mode == "rowwise" else None)
    else:
        if repl:
            raise SystemExit("--replicate-rows needs --exchange p2p")
        sl = ShardedLookup(metas, placement, 0, tuple(range(F)), ("sum",) * F, B, rank, world, dev, mode=mode)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    batches = [(torch.from_numpy(hb.indices).to(dev), torch.from_numpy(hb.offsets).to(dev)) for hb in host_batches]
    out = torch.empty((B, F * dim), dtype=torch.float32, device=dev) if args.exchange == "nccl" else None
    sl.lookup(*batches[0], out=out, check=True)
    for i in range(args.warmup):
        sl.lookup(*batches[i % len(batches)], out=out, check=False)
    torch.cuda.synchronize()
    dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.exchange == "nccl":
        sl.stats.c1_bytes_sent = sl.stats.c2_bytes_sent = 0
    l0 = getattr(sl, "launches", None)
    torch.cuda.synchronize()
    dist.barrier()
    pipelined = args.exchange == "p2p" and not args.sync

    def run_steps(n):
        if pipelined:
            for _ in sl.stream((batches[i % len(batches)] for i in range(n)), check=False):
                pass
        else:
            for i in range(n):
                sl.lookup(*batches[i % len(batches)], out=out, check=False)

    ev0.record(stream)
    run_steps(args.steps)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    clocks_ranks = [None] * world  # every rank's own GPU clocks during the timed region
    dist.all_gather_object(clocks_ranks, clocks)
    ms = ev0.elapsed_time(ev1)
    l1 = getattr(sl, "launches", None)
    # a peer that stopped participating makes the spin barrier give up after
    # ~10 s and set a flag: the timed steps are then void — raise
    if hasattr(sl, "_check"):
        sl._check()
    # per-phase device times from a separate profiled pass (events on every
    # phase would perturb the timed region)
    prof_steps = min(args.steps, 50)
    if args.exchange == "nccl":
        sl.stats.c1_bytes_sent = sl.stats.c2_bytes_sent = 0
    sl.profile = True
    run_steps(prof_steps)
    torch.cuda.synchronize()
    phases = {k: v * args.steps / prof_steps for k, v in sl.phase_ms().items()}
    sl.profile = False
    dist.barrier()
    sl.ops.check()
    # owner-pool algorithmic bytes: every rank pools, for each requester, the
    # rows routed to it; measured on this rank over the timed steps
    t = torch.tensor([ms, phases.get("pool", 0.0), phases.get("a2a", 0.0)], device=dev, dtype=torch.float64)
    allpool = [torch.zeros(1, device=dev, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allpool, t[1:2].clone())
    pool_ms_ranks = [round(float(x.item()) / args.steps, 4) for x in allpool]
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax[0].item())
    value = world * B * F * args.steps / (ms_max / 1e3)
    # algorithmic bytes pooled on this rank per step: all ranks' bags of the tables it owns.
    # With identical batch statistics per rank, the rank's share is rows_owned / total.
    if args.exchange == "nccl":
        a2a_bytes = (sl.stats.c1_bytes_sent + sl.stats.c2_bytes_sent) / prof_steps
    else:
        # bytes crossing NVLink per step from this rank as owner: pooled rows (+ indices read) to the
        # other ranks; table-wise f32 rows, row-wise f64 partials
        per_row = dim * (4 if mode == "tablewise" or args.partial == "f32" else 8)
        if mode == "tablewise" and hasattr(sl, "execu"):
            # (requester, feature) pairs this rank pools for OTHER requesters
            rows_out = B * sum(1 for q in range(world) if q != rank for f in range(F) if sl.execu[q][f] == rank)
        else:
            rows_out = (world - 1) * (B * sum(1 for s in placement if s.server_id == rank) if mode == "tablewise"
                                      else B * F)
        a2a_bytes = rows_out * per_row
    sl.ops.check() if hasattr(sl, "ops") else None
    total_alg = sum(algorithmic_bytes(hb, dim) for hb in host_batches) / len(host_batches)
    if mode == "tablewise" and hasattr(sl, "execu"):
        share = sum(1 for q in range(world) for f in range(F) if sl.execu[q][f] == rank) / (F * world)
    elif mode == "tablewise":
        owned = sum(1 for s in placement if s.server_id == rank)
        share = (owned * world + len(repl)) / (F * world)
    else:
        share = 1.0 / world
    pool_bytes_step = total_alg * world * share
    pool_ms = float(t[1].item()) / args.steps
    achieved = pool_bytes_step / (pool_ms / 1e3) / 1e9 if pool_ms > 0 else None
    peak, peak_src = measured_peak()
    a2a_ms = float(t[2].item()) / args.steps if args.exchange == "nccl" else float(t[1].item()) / args.steps
    step_ms = ms_max / args.steps
    # fused compute+collective roofline (B200_PROFILING.md): the step cannot
    # beat max(HBM bytes / HBM peak, NVLink bytes / measured 770 GB/s peer copy)
    nvl_peak = 770.0
    t_hbm = pool_bytes_step / (peak * 1e9) * 1e3
    t_nvl = a2a_bytes / (nvl_peak * 1e9) * 1e3
    fused_roof = {"hbm_bytes_per_step": pool_bytes_step, "nvlink_bytes_per_step": a2a_bytes,
                  "target_ms": max(t_hbm, t_nvl), "bound": "hbm" if t_hbm >= t_nvl else "nvlink",
                  "frac": max(t_hbm, t_nvl) / step_ms, "nvlink_peak_gbs": nvl_peak,
                  "nvlink_gbs_over_step": a2a_bytes / (step_ms / 1e3) / 1e9}
    # e2e: pinned host CSR -> device -> sharded lookup -> pinned host out
    e2e = None
    if not args.no_e2e:
        # pinned staging next to this rank's GPU (multi-socket boxes)
        from paper_2410_12794_b200.numa import bind_to_device
        bind_to_device(local)
        pinned = [(torch.from_numpy(hb.indices).pin_memory(), torch.from_numpy(hb.offsets).pin_memory())
                  for hb in host_batches]
        out_h = torch.empty((B, F * dim), dtype=torch.float32, pin_memory=True)
        ksteps = max(3, min(args.steps, 60))
        piped = args.exchange == "p2p" and not args.sync
        if piped:  # warm the pipelined host path (slots, pinned buffers, events)
            for _ in sl.stream_host([pinned[i % len(pinned)] for i in range(4)], check=False):
                pass
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h2d = 0
        if piped:
            for i, oh_ in enumerate(sl.stream_host([pinned[i % len(pinned)] for i in range(ksteps)], check=False)):
                ih, oh = pinned[i % len(pinned)]
                h2d += ih.numel() * ih.element_size() + oh.numel() * 8
            api = ("sharded.P2PShardedLookup.stream_host per rank (pinned host CSR -> pinned host pooled; H2D, "
                   "fused exchange and D2H pipelined)")
        else:
            for i in range(ksteps):
                ih, oh = pinned[i % len(pinned)]
                o = sl.lookup(ih.to(dev, non_blocking=True), oh.to(dev, non_blocking=True), out=out, check=False)
                out_h.copy_(o, non_blocking=True)
                stream.synchronize()
                h2d += ih.numel() * ih.element_size() + oh.numel() * 8
            api = f"sharded.{type(sl).__name__}.lookup per rank (pinned host CSR -> pinned host pooled, sync)"
        e1.record(stream)
        e1.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * B * F * ksteps / (float(te.item()) / 1e3), "unit": "pooled lookups/s",
               "h2d_bytes_per_step": h2d // ksteps, "d2h_bytes_per_step": out_h.numel() * 4, "steps": ksteps,
               "api": api}
    if rank == 0:
        line = {
            "metric": "pooled lookups/s (bags/s)", "value": value, "unit": "pooled lookups/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 rows, f64 accumulate", "data": "synthetic",
            "config": sharded_config(cfg, args, world), "init_store_s": round(init_s, 2),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": None,
                         "peak_source": peak_src, "kernel": "owner gather+pool (K4) launches, rank 0",
                         "bytes_per_step": pool_bytes_step, "pool_ms_per_step": pool_ms,
                         "pool_ms_per_step_all_ranks": pool_ms_ranks},
            "fused_roofline": fused_roof,
            "a2a": {"bytes_sent_per_step_rank0": a2a_bytes, "ms_per_step_rank0": a2a_ms,
                    "gbs": (a2a_bytes / (a2a_ms / 1e3) / 1e9) if a2a_ms > 0 else None,
                    "peak_gbs": 900.0, "phases_ms_total": {k: round(v, 3) for k, v in phases.items()},
                    "note": ("NCCL all_to_all_single; includes the self-slice" if args.exchange == "nccl" else
                             "fused: pooled rows stored to peers inside K4; ms = the fused kernel's time")},
            "gpu_launches": (l1 - l0) if l0 is not None else None,
            "e2e": e2e, "cpu_baseline": None, "clocks": clocks, "clocks_ranks": clocks_ranks,
        }
        emit(line, args)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
