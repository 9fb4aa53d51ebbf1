#!/usr/bin/env python
"""bench.py — VQhull hot path on B200 (driver contract).

One "step" = one full hull (sample polygon, filter pass, fused partition +
arg-max levels, recursion, clockwise first-occurrence index list) over one
batch of the workload.  Workloads (BASELINE.json configs):

  --gpus 1 (default)  config 2: 1e8 f64 points uniform in [-1, 1]^2, seed 2
                      (BASELINE configs[1], "single B200").
  --gpus N > 1        config 5: 4e9 f64 points uniform in the unit disk,
                      seed 5, sharded evenly over the N GPUs (strong
                      scaling): per rank the local hull and its certified
                      candidates, one NCCL all-gather, the merge hull
                      (paper_2510_09417_b200/distributed.py).
  --config K          any BASELINE config (1-4 weak-scaled per GPU at N > 1).

With --gpus N > 1 and no torchrun environment, bench.py relaunches itself
through torch.distributed.run (one process per GPU, 127.0.0.1); it refuses to
run when fewer than N GPUs are visible.

  value    : whole-job points/s, inputs resident in HBM (CUDA events on the
             launching stream, max over ranks)
  e2e      : points/s through the public API with HOST buffers: the C ABI
             vqhull_compute at N = 1 (pinned arrays; the pageable case is
             reported beside it), per-rank H2D + sharded hull + D2H at N > 1
  roofline : the dominant kernel's algorithmic bytes / its CUDA-event time
  cpu_baseline : the reference library (oracle/_ref, compiled from the
             reference sources) on this host's cores, bounded sample of the
             same workload, workers = 1 and workers = nproc, plus the
             reference's Scale baseline

`--impl reference` times the reference's own CPU implementation of the path
(convex_hull, all host threads) on the same workload and prints the same
line; it generates its inputs with the reference's own generators and never
loads this repository's library.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import socket
import subprocess
import sys
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
# the reference arm's bounded sample (host RAM and minutes): the first
# REF_SAMPLE points of the workload's stream
REF_SAMPLE = 4 * 10**8


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=0, choices=[0, *sorted(CONFIGS)],
                   help="BASELINE config (default: 2 on one GPU, 5 sharded on N > 1)")
    p.add_argument("--points", "--n", dest="n", type=int, default=0, help="override the workload's point count")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--profile", action="store_true", help="minimal run for ncu (no extras)")
    p.add_argument("--csv", default="", help="also write one row per timed step in the reference's "
                   "CSV schema (bench.cpp:156-160) to this path (rank 0)")
    return p.parse_args(argv)


class Workload:
    """The one description both arms print (identical `config` objects)."""

    def __init__(self, args, world: int):
        cfg = args.config or (5 if world > 1 else 2)
        kind, n, seed = CONFIGS[cfg]
        if args.n:
            n = args.n
        self.cfg, self.kind, self.seed, self.world = cfg, kind, seed, world
        # config 5 is defined sharded (strong scaling); configs 1-4 are
        # single-GPU workloads, weak-scaled (n per GPU) when N > 1
        self.strong = cfg == 5
        self.total = n if self.strong else n * world
        self.n_arg = n

    def shard(self, rank: int):
        """(offset, count) of this rank's contiguous shard."""
        if self.strong:
            base, rem = divmod(self.total, self.world)
            return rank * base + min(rank, rem), base + (1 if rank < rem else 0)
        return rank * self.n_arg, self.n_arg

    @property
    def name(self) -> str:
        w = f"config{self.cfg}: {self.kind} seed={self.seed}, "
        if self.strong:
            w += f"n={self.total} total, sharded evenly over {self.world} GPU(s)"
        elif self.world > 1:
            w += f"n={self.n_arg} per GPU x {self.world} GPUs (contiguous ranges of one stream)"
        else:
            w += f"n={self.n_arg}"
        if self.cfg == 2 and self.world == 1 and not self.strong:
            w += " (BASELINE configs[1])"
        return w

    def config(self) -> dict:
        return {"workload": self.name, "points_total": self.total, "n_gpus": self.world,
                "parallelism": f"shard{self.world}" if self.world > 1 else "single GPU"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class Clocks:
    """Clocks and throttle reasons DURING the timed region: one
    `nvidia-smi ... -lms 200` process started before the region and stopped
    after it (B200_PROFILING.md's clocks line) — no process is spawned while
    the timed kernels run."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.25)  # its first sample precedes the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.21)  # at least one sample after the region
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=10)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in (out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.samples.append(f)

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


def emit(obj):
    print(json.dumps(obj), flush=True)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: check the GPUs, then one process per GPU."""
    import torch

    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < args.gpus:
        print(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible; refusing to run "
              f"(a {args.gpus}-GPU line measured on {have} GPU(s) would be wrong)", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__),
           # (torchrun's own parser reads "--n" as an ambiguous abbreviation)
           *[re.sub(r"^--n(?==|$)", "--points", a) for a in sys.argv[1:]]]
    return subprocess.run(cmd).returncode


# ---------------------------------------------------------------------------
# reference arm and CPU baseline: the reference library only (oracle/_ref)
# ---------------------------------------------------------------------------
def _ref_inputs(R, wl: Workload, m: int, threads: int):
    """The first m points of the workload's stream, from the reference's own
    generators (dataset.cpp:58-75; square: its rng::uniform01)."""
    if wl.kind == "square":
        return R.generate_square(m, wl.seed, 0, threads)
    return R.generate(wl.kind, m, wl.seed, threads)


def reference_runs(wl: Workload, steps: int, warmup: int, workers: int, R=None, m=None):
    import numpy as np

    from oracle import Reference

    R = R or Reference()
    threads = os.cpu_count() or 1
    m = min(wl.total, REF_SAMPLE) if m is None else m
    xs, ys = _ref_inputs(R, wl, m, threads)
    if warmup:
        R.bench_hull(xs, ys, workers, warmup)
    secs, h = R.bench_hull(xs, ys, workers, steps)
    what = "the full workload" if m == wl.total else f"the first {m} of {wl.total} points"
    return np.asarray(secs), int(h), m, what


def run_reference(args) -> int:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    wl = Workload(args, world)
    from oracle import Reference

    if not Reference.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libvqhull_ref.so was not built"})
        return 0
    threads = os.cpu_count() or 1
    secs, h, m, what = reference_runs(wl, args.steps, max(args.warmup, 0), threads)
    mean = float(secs.mean())
    value = m / mean
    emit({
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "strong" if wl.strong else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generators, seeded)", "impl": "reference",
        "config": wl.config(),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"{what} ({wl.kind}, seed {wl.seed}): {args.steps} timed "
                                   f"convex_hull reps after {args.warmup} untimed, fresh copy each, "
                                   f"hull timed (run_bench_points), workers={threads}",
                         "seconds": secs.tolist(), "hull_vertices_of_sample": h},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    return 0


def cpu_reference_baseline(wl: Workload, budget_s: float = 20.0) -> dict:
    """BASELINE.md §3 on this host: convex_hull at workers = nproc and
    workers = 1 on a bounded sample of the workload, plus the Scale baseline."""
    import numpy as np

    from oracle import Oracle, Reference

    threads = os.cpu_count() or 1
    if not Reference.available():  # the oracle port, one thread, bounded sample
        import paper_2510_09417_b200 as vq

        m = min(wl.total, 10**7)
        xs, ys = vq.generate(wl.kind, m, wl.seed)
        t0 = time.perf_counter()
        Oracle().convex_hull(xs, ys)
        dt = time.perf_counter() - t0
        return {"kind": "port", "cores": 1, "value": m / dt, "unit": "points/s",
                "cpu_model": cpu_model(),
                "sample": f"first {m} points of {wl.kind} seed {wl.seed}, oracle convex_hull, 1 thread"}
    R = Reference()
    m = min(wl.total, REF_SAMPLE)
    xs, ys = _ref_inputs(R, wl, m, threads)
    out = {"kind": "reference", "cores": threads, "unit": "points/s", "cpu_model": cpu_model()}
    for workers, key in ((threads, "nproc"), (1, "one")):
        s0, _ = R.bench_hull(xs, ys, workers, 1)  # calibration rep (untimed)
        k = max(1, min(10, int(budget_s / 2 / max(float(s0[0]), 1e-3))))
        secs, h = R.bench_hull(xs, ys, workers, k)
        out[f"workers_{key}"] = {"workers": workers, "reps": k, "mean_s": float(np.mean(secs)),
                                 "stddev_s": float(np.std(secs, ddof=1)) if k > 1 else 0.0,
                                 "best_s": float(np.min(secs)), "points_per_s": m / float(np.mean(secs))}
    out["value"] = out["workers_nproc"]["points_per_s"]
    out["scale_baseline_gbps"] = R.scale_baseline(threads, 5)
    what = "the full workload" if m == wl.total else f"the first {m} of {wl.total} points"
    out["sample"] = (f"{what} ({wl.kind}, seed {wl.seed}), reference generators; convex_hull "
                     f"(run_bench_points: fresh copy per rep, hull timed) at workers={threads} "
                     f"and workers=1; Scale baseline (bench.cpp:33-74) at workers={threads}")
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args) -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_09417_b200 as vq
    from paper_2510_09417_b200.distributed import sharded_hull

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if not torch.cuda.is_available():
        print("bench.py: no CUDA device visible", file=sys.stderr)
        return 2
    # test hook (tests/test_sharded_gpu.py): every rank on cuda:0 over gloo, so
    # the N > 1 code path runs on a one-GPU box; never used for a bench line
    share = os.environ.get("VQHULL_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = Workload(args, world)
    offset, n = wl.shard(rank)

    # host generation (libm, the reference generators' bytes) into pinned memory
    Xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    Yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    vq.generate(wl.kind, n, wl.seed, first=offset, out=(Xh, Yh))
    X = Xh.cuda(non_blocking=False)
    Y = Yh.cuda(non_blocking=False)
    out_u32 = torch.empty(n, dtype=torch.int32, device="cuda") if world == 1 else None
    stream = torch.cuda.current_stream()

    def step():
        if world == 1:
            return vq.hull_device(X, Y, stream=stream, out=out_u32, u32=True)
        return sharded_hull(X, Y, offset)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device-resident inputs.  Inputs (16 B/pt) that fit in
    # L2 twice over are timed step by step with an L2 flush (a 512 MB write)
    # between steps, outside the events.  The clock sampler is started BEFORE
    # the warm-up steps (its start-up sleep would otherwise leave the GPU idle
    # for a quarter of a second right in front of the timed steps, and the
    # first of them would pay for the wake-up).
    flush = None
    if 16 * n < 2 * L2_BYTES:
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        res = None
        for _ in range(max(args.warmup, 0)):
            res = step()
        if res is None:  # --warmup 0: one untimed call still gives h and the launch count
            res = step()
        barrier()
        h = int(res.numel())
        from paper_2510_09417_b200 import distributed as D
        launches_per_step = int(vq.stats()["launches"]) if world == 1 else D.last_launches()
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
    value = wl.total / (ms_step / 1e3)
    clocks = clk.summary()

    result = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if wl.strong else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (reference RNG streams, seeded; generated on host with libm)",
        "config": wl.config(),
        "details": {"points_per_gpu": n, "hull_vertices": h,
                    "l2": ("inputs 16 B/pt x n >> 126 MB L2 (no flush needed)" if flush is None else
                           "L2 flushed (512 MB write) before every timed step; per-step CUDA events summed")},
        "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
    }
    if world > 1:
        result["details"]["merge"] = D.last_info()
    if args.profile:
        if rank == 0:
            emit(result)
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline: per-kernel CUDA-event times inside the library (same
    # stream) for this rank's hull (at N > 1: the local hull of its shard)
    vq.set_timing(True)
    fam = {"extremes": [0.0, 0], "bootstrap": [0.0, 0], "root_partition": [0.0, 0],
           "levels": [0.0, 0], "finisher": [0.0, 0]}
    st = {}
    rep_rows = []  # (seconds, bytes_moved) per step, for --csv
    tmp_out = out_u32 if out_u32 is not None else torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        vq.hull_device(X, Y, stream=stream, out=tmp_out, u32=True)
        st = vq.stats()
        rep_rows.append((st["ms_total"] / 1e3, int(st["bytes_moved"])))
        for k in fam:
            fam[k][0] += st[f"ms_{k}"]
            fam[k][1] += st[f"bytes_{k}"]
    vq.set_timing(False)
    del tmp_out
    barrier()
    dom = max(fam, key=lambda k: fam[k][0])
    peak, peak_src = peaks()
    achieved = (fam[dom][1] / 1e9) / (fam[dom][0] / 1e3) if fam[dom][0] > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"config{wl.cfg}", {}).get(dom)
    except Exception:
        pass
    kname = {"root_partition": ("root_filter_tma (split root pass 1: polygon filter over every point)"
                                if st.get("root_filtered") == 2 else "root pass"),
             "levels": "cluster_tail_kernel / tail_kernel / level kernels (recursion)",
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
        "scope": "rank 0's local hull of its shard" if world > 1 else "the whole hull",
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

        def e2e_step(pinned=True):
            if world == 1:
                a, b = (xs_np, ys_np) if pinned else (xs_pg, ys_pg)
                rc, idx = vq.vqhull_compute(a, b)
                assert rc == 0
                return idx.size
            Xd.copy_(Xh, non_blocking=True)
            Yd.copy_(Yh, non_blocking=True)
            g = sharded_hull(Xd, Yd, offset)
            return g.cpu().numel()

        def timed(fn, steps):
            fn()
            barrier()
            t0 = time.perf_counter()
            for _ in range(steps):
                hh = fn()
            barrier()
            dt = (time.perf_counter() - t0) / steps
            tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item()), hh

        dt, hh = timed(e2e_step, args.steps)
        result["e2e"] = {"value": wl.total / dt, "unit": "points/s",
                         "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": (8 if world > 1 else 8) * hh,
                         "ms_per_step": dt * 1e3,
                         "api": "vqhull_compute (C ABI, pinned host arrays)" if world == 1
                         else "per rank: H2D of its shard + sharded_hull + D2H of the index list"}
        if world == 1:  # a drop-in C caller passes pageable memory: measured beside it
            xs_pg, ys_pg = np.array(xs_np), np.array(ys_np)
            dtp, _ = timed(lambda: e2e_step(False), max(1, min(args.steps, 5)))
            result["e2e"]["pageable"] = {"value": wl.total / dtp, "unit": "points/s",
                                         "ms_per_step": dtp * 1e3}
            del xs_pg, ys_pg

    # ---- CPU baseline (rank 0, N=1 only)
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            result["cpu_baseline"] = cpu_reference_baseline(wl)
        except Exception as e:  # never lose the GPU line over the baseline
            result["cpu_baseline"] = {"value": None, "unit": "points/s", "cores": None,
                                      "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0 and args.csv:
        write_csv(args.csv, wl.kind, wl.total, wl.seed, world, rep_rows, h, peak)
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
    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
