#!/usr/bin/env python
"""bench.py — VQhull hot path on B200 (driver contract).

Workload (BASELINE.json configs[1]): N = 1e8 float64 points uniform in the
square [-1, 1]^2, seed 2; one "step" = one full hull (extremes, fused
partition + arg-max levels, recursion, clockwise first-occurrence index
list) over one batch.  With --gpus N (torchrun, one process per GPU) every
rank hulls its own 1e8-point contiguous shard of the global seed-2 stream
(weak scaling) and the ranks merge through one NCCL all-gather of the
candidate vertices (paper_2510_09417_b200/distributed.py).

  value : whole-job points/s with inputs resident in HBM (device-timed, CUDA
          events, max over ranks; inputs 1.6 GB/GPU >> 126 MB L2, so no flush)
  e2e   : points/s through the public API with HOST buffers (pinned), i.e.
          vqhull_compute's H2D of the coordinates and D2H of the index list
          inside the timed region
  roofline : the dominant kernel's algorithmic bytes / its CUDA-event time
  cpu_baseline : the reference library (oracle/_ref, compiled from the
          reference sources) on this host's cores, same workload

`--impl reference` times the reference's own CPU implementation of the path
(convex_hull, all host threads) on the same config and prints the same line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: ("disk", 10**6, 1),
    2: ("square", 10**8, 2),
    3: ("circle", 10**7, 3),
    4: ("kuzmin", 10**9, 4),
    5: ("disk", 4 * 10**9, 5),
}
L2_BYTES = 126 * 2**20
METRIC = "points/sec per hull (f64 2D) and achieved HBM GB/s vs peak"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    p.add_argument("--n", type=int, default=0, help="override points per rank")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--profile", action="store_true", help="minimal run for ncu (no extras)")
    p.add_argument("--csv", default="", help="also write one row per timed step in the reference's "
                   "CSV schema (bench.cpp:156-160) to this path (rank 0)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        mx = max((float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 5 + k and s[5 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_reference_baseline(kind, n, seed, offset_ranks=1, budget_s=20.0, reps=None):
    """The reference library (oracle/_ref) on this host: convex_hull with all
    host threads, run_bench_points semantics (fresh copy per rep, hull timed)."""
    import numpy as np

    import paper_2510_09417_b200 as vq
    from oracle import Oracle, Reference

    threads = os.cpu_count() or 1
    total = n * offset_ranks
    m = min(total, 4 * 10**8)  # bounded sample (config 5: 4e9 points would need 128 GB host RAM)
    xs, ys = vq.generate(kind, m, seed, threads=threads)
    if Reference.available():
        R = Reference()
        secs, h = R.bench_hull(xs, ys, threads, 1)  # first rep calibrates
        t = float(secs[0])
        k = reps or max(1, min(5, int(budget_s / max(t, 1e-3))))
        secs2, h = R.bench_hull(xs, ys, threads, k)
        allsecs = np.concatenate([secs, secs2])
        what = "full workload" if m == total else f"first {m} of {total} points"
        return {"kind": "reference", "cores": threads, "seconds": allsecs.tolist(),
                "value": m / float(np.mean(secs2)), "hull": int(h),
                "sample": f"{what}: {kind} n={m} seed={seed}, "
                          f"{len(secs2)} timed reps after 1 untimed, convex_hull workers={threads}"}
    # oracle port (single thread): bounded sample
    O = Oracle()
    m = min(m, 10**7)
    t0 = time.perf_counter()
    O.convex_hull(xs[:m], ys[:m])
    dt = time.perf_counter() - t0
    return {"kind": "port", "cores": 1, "value": m / dt, "seconds": [dt],
            "sample": f"first {m} points of {kind} seed={seed}, oracle convex_hull, 1 thread"}


def emit(obj):
    print(json.dumps(obj), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    kind, n, seed = CONFIGS[args.config]
    if args.n:
        n = args.n
    import numpy as np

    import paper_2510_09417_b200 as vq
    from oracle import Oracle, Reference

    threads = os.cpu_count() or 1
    strong = args.config == 5 and not args.n
    total = n if strong else n * world
    xs, ys = vq.generate(kind, total, seed, threads=threads)
    if Reference.available():
        R = Reference()
        R.bench_hull(xs, ys, threads, max(args.warmup, 0)) if args.warmup else None
        secs, h = R.bench_hull(xs, ys, threads, args.steps)
        kind_s, cores = "reference", threads
        sample = (f"{kind} n={total} seed={seed}: {args.steps} timed convex_hull reps "
                  f"(fresh copy each, hull timed), workers={threads}")
    else:
        O = Oracle()
        secs = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            O.convex_hull(xs, ys)
            secs.append(time.perf_counter() - t0)
        secs = np.array(secs)
        kind_s, cores = "port", 1
        sample = f"{kind} n={total} seed={seed}: oracle port, 1 thread"
    mean = float(np.mean(secs))
    value = total / mean
    emit({
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference RNG, seeded)", "impl": "reference",
        "config": {"workload": (f"config{args.config}: {kind} n={total} total, sharded, seed={seed}" if strong
                                else f"config{args.config}: {kind} n={n} per GPU seed={seed}"),
                   "points_total": total, "parallelism": f"host threads={cores}"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": kind_s,
                         "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    })
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_09417_b200 as vq
    from paper_2510_09417_b200.distributed import sharded_hull

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kind, n, seed = CONFIGS[args.config]
    if args.n:
        n = args.n
    # configs 1-4: weak scaling, each rank owns n points of the global stream;
    # config 5 (BASELINE: 4e9 points sharded evenly over 1/2/4/8 GPUs): strong
    strong = args.config == 5 and not args.n
    if strong:
        total = n
        n = total // world + (1 if rank < total % world else 0)
        offset = rank * (total // world) + min(rank, total % world)
    else:
        offset = rank * n

    # host generation (libm, same bytes as the reference generators) into pinned memory
    Xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    Yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    vq.generate(kind, n, seed, first=offset, out=(Xh, Yh))
    X = Xh.cuda(non_blocking=False)
    Y = Yh.cuda(non_blocking=False)
    out_u32 = torch.empty(n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        if world == 1:
            return vq.hull_device(X, Y, stream=stream, out=out_u32, u32=True)
        return sharded_hull(X, Y, offset)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res = None
    for _ in range(max(args.warmup, 0)):
        res = step()
    if res is None:  # --warmup 0: one untimed call still gives h and the launch count
        res = step()
    barrier()
    h = int(res.numel())
    launches_per_step = int(vq.stats()["launches"]) * (2 if world > 1 else 1)

    # ---- timed region: device resident inputs
    # inputs (16 B/pt) that fit in L2 twice over are timed step by step with
    # an L2 flush (a 512 MB write) between steps, outside the events
    flush = None
    if 16 * n < 2 * L2_BYTES:
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        if flush is None:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            barrier()
            ms = ev0.elapsed_time(ev1)
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                step()
                b.record(stream)
            barrier()
            ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    points_total = total if strong else world * n
    value = points_total / (ms_step / 1e3)
    clocks = clk.summary()

    result = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference RNG streams, seeded; generated on host with libm)",
        "config": {"workload": (f"config{args.config}: {kind} n={points_total} total, sharded, seed={seed}"
                                if strong else f"config{args.config}: {kind} n={n} per GPU seed={seed}")
                               + (" (BASELINE configs[1])" if args.config == 2 else ""),
                   "points_per_gpu": n, "points_total": points_total, "hull_vertices": h,
                   "parallelism": f"shard{world}" if world > 1 else "single GPU",
                   "l2": ("inputs 16 B/pt x n >> 126 MB L2 (no flush needed)" if flush is None else
                          "L2 flushed (512 MB write) before every timed step; per-step CUDA events summed")},
        "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
    }
    if args.profile:
        if rank == 0:
            emit(result)
        return 0

    # ---- roofline: per-kernel CUDA-event times inside the library (same stream)
    vq.set_timing(True)
    fam = {"extremes": [0.0, 0], "bootstrap": [0.0, 0], "root_partition": [0.0, 0],
           "levels": [0.0, 0], "finisher": [0.0, 0]}
    st = {}
    rep_rows = []  # (seconds, bytes_moved) per step, for --csv
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        step()
        st = vq.stats()
        rep_rows.append((st["ms_total"] / 1e3, int(st["bytes_moved"])))
        for k in fam:
            fam[k][0] += st[f"ms_{k}"]
            fam[k][1] += st[f"bytes_{k}"]
    vq.set_timing(False)
    barrier()
    dom = max(fam, key=lambda k: fam[k][0])
    peak, peak_src = peaks()
    achieved = (fam[dom][1] / 1e9) / (fam[dom][0] / 1e3) if fam[dom][0] > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"config{args.config}", {}).get(dom)
    except Exception:
        pass
    kname = {"root_partition": ("root_filter_tma (split root pass 1: octagon filter over every point)"
                                if st.get("root_filtered") == 2 else "root pass"),
             "levels": "tail_kernel (persistent recursion)" if st.get("root_filtered") == 2 else "level kernels",
             "extremes": "poly_sample_kernel" if st.get("root_filtered") == 2 else "extremes"}.get(dom, dom)
    result["roofline"] = {
        "bound": "hbm", "kernel": kname, "family": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "peak_source": peak_src, "traffic": traffic,
        "bytes_per_launch": fam[dom][1] / args.steps,
        "ms_per_launch": fam[dom][0] / args.steps,
        "families_ms_per_step": {k: v[0] / args.steps for k, v in fam.items()},
        "families_gbs": {k: (v[1] / 1e9) / (v[0] / 1e3) if v[0] else None for k, v in fam.items()},
        "hull_ms_events": st.get("ms_total"), "bytes_moved_per_step": st.get("bytes_moved"),
        "lower_bound_16n_frac": (16 * n / 1e9) / (ms_step / 1e3) / peak,
    }

    # ---- e2e: public API with HOST buffers (H2D + D2H inside the timed region)
    if not args.no_e2e:
        xs_np, ys_np = Xh.numpy(), Yh.numpy()
        if world == 1:  # the C ABI makes its own device copy: release ours first
            del X, Y, out_u32
            torch.cuda.empty_cache()
        else:
            Xd = torch.empty_like(X)
            Yd = torch.empty_like(Y)

        def e2e_step():
            if world == 1:
                rc, idx = vq.vqhull_compute(xs_np, ys_np)
                assert rc == 0
                return idx.size
            Xd.copy_(Xh, non_blocking=True)
            Yd.copy_(Yh, non_blocking=True)
            g = sharded_hull(Xd, Yd, offset)
            return g.cpu().numel()

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hh = e2e_step()
        barrier()
        dt = (time.perf_counter() - t0) / args.steps
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        result["e2e"] = {"value": points_total / dt, "unit": "points/s",
                         "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": (4 if world == 1 else 8) * hh,
                         "ms_per_step": dt * 1e3,
                         "api": "vqhull_compute (C ABI, pinned host arrays)" if world == 1
                         else "H2D + sharded_hull + D2H"}

    # ---- CPU baseline (rank 0, N=1 only)
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cb = cpu_reference_baseline(kind, n, seed)
            result["cpu_baseline"] = {"value": cb["value"], "unit": "points/s", "cores": cb["cores"],
                                      "kind": cb["kind"], "sample": cb["sample"]}
        except Exception as e:  # never lose the GPU line over the baseline
            result["cpu_baseline"] = {"value": None, "unit": "points/s", "cores": None,
                                      "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0 and args.csv:
        write_csv(args.csv, kind, points_total, seed, world, rep_rows, h, peak)
    if rank == 0:
        emit(result)
    if world > 1:
        dist.destroy_process_group()
    return 0


CSV_HEADER = ("kind,n,seed,workers,block_size,lanes,simd,write_combining,reps,"
              "rep,seconds,mean_seconds,stddev_seconds,model_bytes,"
              "bandwidth_gbps,baseline_gbps,hull_vertices,joules")


def write_csv(path, kind, n, seed, workers, rep_rows, h, peak_gbs):
    """The reference's bench CSV (header: bench.cpp:156-160, rows: :162-199),
    one row per timed step.  Column meaning on the GPU: workers = GPUs,
    block_size = points per tile, lanes = threads per warp, simd = sm_100a,
    seconds = the hull's device time (CUDA events in the library),
    model_bytes = the device byte model (vqhull_stats.bytes_moved, DESIGN.md
    §9 — the algorithmic bytes of OUR kernels, not the reference's traced
    extraction bytes), baseline_gbps = the measured HBM copy peak standing in
    for the STREAM Scale baseline, joules left empty as in the reference."""
    import statistics
    secs = [r[0] for r in rep_rows]
    mean = statistics.fmean(secs) if secs else 0.0
    # shortest round-trip numbers, as append_number's std::to_chars (bench.cpp:91-95);
    # the reference's stddev_of is the sample deviation (n - 1), 0 for one rep
    sd = statistics.stdev(secs) if len(secs) > 1 else 0.0
    mb = rep_rows[-1][1] if rep_rows else 0
    bw = mb / mean / 1e9 if mean > 0 else 0.0
    with open(path, "w") as f:
        f.write(CSV_HEADER + "\n")
        for i, (sec, _) in enumerate(rep_rows):
            f.write(f"{kind},{n},{seed},{workers},1024,32,sm_100a,0,{len(rep_rows)},{i + 1},"
                    f"{sec!r},{mean!r},{sd!r},{mb},{bw!r},{float(peak_gbs)!r},{h},\n")


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
