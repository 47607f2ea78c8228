#!/usr/bin/env python
"""CPRAND iters/sec on B200 (BASELINE.json metric), one JSON line.

Workload (default `c4` = configs[3]): 1000^3 fp64 tensor (8 GB) from rank-50
factors with congruence 0.9 and 1% noise, generated in HBM; CPRAND R=50,
S=2000; bench mode = exactly K outer iterations with no fit checks
(`cprand bench-iter`, tools/cprand_main.cpp:179-206). A step = one outer
iteration (3 mode updates). The tensor (8 GB) is ~64x the 126 MB L2 and each
iteration gathers fresh uniform samples, so no L2 flush is needed between
steps ("inputs larger than L2").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port)

Multi-GPU (N > 1, torchrun): one process per GPU; the tensor is slab-sharded
along its last mode (NCCL allreduce of the R x I_n right-hand sides, allgather
of the last factor), one global problem ("strong" scaling).

Beside the bench-mode headline the line carries the two other parts of the
BASELINE.json metric: `full_loop` (iters/s with the sampled fit estimator and
the stop rule every iteration) and `time_to_fit` (wall time from solver entry,
tensor resident in HBM, to the estimated fit reaching 0.99 and 1 - 1.2 eta).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: dims, R, S, P_hat, congruence, eta, method, transform
    "c1": dict(dims=(100, 100, 100), r=5, s=100, phat=4096, c=0.0, eta=0.01, method="rand", transform=None),
    "c2": dict(dims=(300, 300, 300), r=10, s=300, phat=1 << 14, c=0.5, eta=0.01, method="rand", transform=None),
    "c3": dict(dims=(80, 80, 80, 80), r=10, s=300, phat=1 << 14, c=0.9, eta=0.01, method="mix", transform="dct"),
    "c4": dict(dims=(1000, 1000, 1000), r=50, s=2000, phat=1 << 16, c=0.9, eta=0.01, method="rand", transform=None),
    "c5": dict(dims=(320, 320, 320, 320), r=20, s=1200, phat=1 << 18, c=0.5, eta=0.001, method="mix", transform="dct"),
}
METRIC = "CPRAND iters/sec"
SEED = 1
DFMA_PEAK_TF = 33.5  # FP64 FMA throughput measured on this pool's B200 (tests/micro/probe.cu)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append((time.perf_counter(), parts))

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter() + 0.05

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        during = [r for (ts, r) in self.rows if t0 <= ts <= t1]
        window = "timed region"
        if not during:  # region shorter than the sampling period: nearest samples
            during = [r for (ts, r) in sorted(self.rows, key=lambda q: abs(q[0] - t0))[:3]]
            window = "nearest samples to a timed region shorter than the 20 ms sampling period"
        if not during:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        rows = during
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows),
                "window": window}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def dist_init(ws):
    if ws <= 1:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    return dist


def allreduce_max(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def config_of(name: str, cfg, ws: int) -> dict:
    """The workload description, identical in both arms (the driver compares them)."""
    nbytes = 8 * int(np.prod(cfg["dims"]))
    return {"workload": name, "dims": list(cfg["dims"]), "R": cfg["r"], "S": cfg["s"], "P_hat": cfg["phat"],
            "method": cfg["method"], "transform": cfg["transform"], "bench_mode": True,
            "parallelism": f"slab{ws} (last mode)" if ws > 1 else "single",
            "l2": (f"inputs larger than L2 ({nbytes / 1e9:.2f} GB tensor, fresh random samples every step)"
                   if nbytes > 126e6 else
                   f"tensor ({nbytes / 1e6:.0f} MB) fits in L2; no flush: fresh random samples every step")}


def launches_per_iter(cfg, fused: bool) -> int:
    if fused:
        return 1  # one persistent kernel per outer iteration
    n = len(cfg["dims"])
    # z, gram, gram_inverse (+ fallback check), rhs_gemm, mode_apply; the gather
    # kernel only for modes without in-place reads
    per_mode = 6 + (3 if cfg["method"] == "mix" and cfg["transform"] == "dct" else 0)
    return n * per_mode


def cpu_oracle_rate(x_host: np.ndarray, cfg, budget_s: float = 15.0, max_iters: int = 40):
    """Reference CPU path (oracle port) in bench mode on the same tensor:
    (total - setup) / iters, as bench-iter reports. Bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    os.environ.setdefault("CPRAND_THREADS", str(os.cpu_count() or 1))
    kw = dict(rng_seed=SEED, bench_mode=True, transform=cfg["transform"])
    probe = orc.solve(cfg["method"], x_host, cfg["r"], cfg["s"], orc.SolveOptions(max_iters=1, **kw))
    per = max(probe.total_seconds - probe.setup_seconds, 1e-6)
    n = int(max(1, min(max_iters, budget_s / per)))
    res = orc.solve(cfg["method"], x_host, cfg["r"], cfg["s"], orc.SolveOptions(max_iters=n, **kw))
    t = max(res.total_seconds - res.setup_seconds, 1e-9)
    return n / t, n, t


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc
    cores = os.cpu_count() or 1
    os.environ.setdefault("CPRAND_THREADS", str(cores))
    x, _ = orc.gen_baseline(cfg["dims"], cfg["r"], cfg["c"], cfg["eta"], SEED)
    kw = dict(rng_seed=SEED, bench_mode=True, transform=cfg["transform"])
    # warm-up steps (one outer iteration each), then K timed steps; the
    # reference's own bench-iter timing excludes its setup
    if args.warmup > 0:
        orc.solve(cfg["method"], x, cfg["r"], cfg["s"], orc.SolveOptions(max_iters=args.warmup, **kw))
    res = orc.solve(cfg["method"], x, cfg["r"], cfg["s"], orc.SolveOptions(max_iters=args.steps, **kw))
    t = max(res.total_seconds - res.setup_seconds, 1e-9)
    value = args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json generator in HBM, seed 1)",
        "config": config_of(args.config, cfg, ws),
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} bench-mode outer iterations of {args.config} "
                                   f"(oracle restatement of the C++ reference; gather on "
                                   f"{cores} threads, LS single-threaded as the reference)"},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def fit_runs(pb, t, cfg, dev, comm, steps, fresh, big):
    """full_loop: `steps` iterations with the estimator + should_stop every
    iteration (stall limit out of reach, so none stops early), device loop
    time. time_to_fit: SolveOptions(fit_threshold=thr), reference defaults
    otherwise (max_iters 200, stall limit 10), timed by wall clock from
    solver entry (session setup: sample tables, estimator, replicas, MIX pass)
    to the stop; counts only if the stop reason is fit_threshold."""
    common = dict(rng_seed=SEED, fit_sample_count=cfg["phat"], transform=cfg["transform"],
                  x_mutable=big, device=dev, comm=comm,
                  shard_total=cfg["dims"][-1] if comm is not None else 0)
    fresh()
    s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"],
                   pb.SolveOptions(max_iters=steps + 3, stall_limit=1 << 30, **common))
    s.run(3)
    s.sync()
    t0 = time.perf_counter()
    ran = s.run(steps)
    wall = time.perf_counter() - t0
    res = s.result()
    s.close()
    loop_dev = res.loop_seconds_device
    full = {"value": ran / wall, "unit": "iters/s", "iterations": ran, "wall_seconds": wall,
            "device_loop_seconds_incl_warmup": loop_dev, "fit_sample_count": cfg["phat"],
            "final_fit_estimate": res.trace[-1][2] if res.trace else None,
            "note": "Session.run: estimate_fit + should_stop on device every iteration, host polls the stop flag"}
    # the exact fit of the same final model (solver.hpp:161-181, device MTTKRP),
    # the check the sampled estimate replaces (bench-fitcheck)
    if comm is None and not big:
        t.exact_fit(res.lam, res.factors)  # warm
        t0 = time.perf_counter()
        ef = t.exact_fit(res.lam, res.factors)
        full["exact_fit"] = {"value": ef, "seconds": time.perf_counter() - t0,
                             "estimate_minus_exact": (res.trace[-1][2] - ef) if res.trace else None}
    ttf = []
    for thr in (0.99, round(1.0 - 1.2 * cfg["eta"], 6)):
        fresh()
        t0 = time.perf_counter()
        s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"], pb.SolveOptions(fit_threshold=thr, **common))
        s.run(200)
        s.sync()
        wall = time.perf_counter() - t0
        res = s.result()
        s.close()
        reached = res.reason == "fit_threshold"
        ttf.append({"threshold": thr, "reached": reached, "seconds": wall if reached else None,
                    "wall_seconds": wall, "setup_seconds": res.setup_seconds, "iterations": res.iterations,
                    "reason": res.reason, "final_fit_estimate": res.trace[-1][2] if res.trace else None,
                    "best_fit": res.trace[-1][4] if res.trace else None, "stall_limit": 10})
        if not reached and res.reason == "best_fit_stall":
            # the same run with the best-fit stall stop out of reach
            # (stall_limit = max_iters): how long the threshold takes when
            # the solver is allowed to continue
            fresh()
            t0 = time.perf_counter()
            s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"],
                           pb.SolveOptions(fit_threshold=thr, stall_limit=200, **common))
            s.run(200)
            s.sync()
            wall = time.perf_counter() - t0
            res = s.result()
            s.close()
            reached = res.reason == "fit_threshold"
            ttf.append({"threshold": thr, "reached": reached, "seconds": wall if reached else None,
                        "wall_seconds": wall, "setup_seconds": res.setup_seconds, "iterations": res.iterations,
                        "reason": res.reason, "final_fit_estimate": res.trace[-1][2] if res.trace else None,
                        "best_fit": res.trace[-1][4] if res.trace else None, "stall_limit": 200})
    return full, ttf


def c5_record(pb, dev, hbm_peak, steps, warmup, cpu: bool):
    """The largest single-GPU configuration (C5: 320^4 = 84 GB, R = 20,
    S = 1200, DCT CPRAND-MIX) measured beside the C4 headline: the mixing
    pass per mode, the bench-mode rate of the persistent CPRAND-MIX kernel
    on the session-mixed tensor, and the CPU reference path's bench-iter rate
    on the same (device-mixed) tensor."""
    cfg = CONFIGS["c5"]
    p = int(np.prod(cfg["dims"]))
    t = pb.DeviceTensor(cfg["dims"], device=dev)
    t.synth(cfg["r"], cfg["c"], cfg["eta"], SEED)
    ms_modes = t.mix("dct", SEED)
    gbs = [16.0 * p / (m * 1e-3) / 1e9 for m in ms_modes]
    out = {"config": config_of("c5", cfg, 1),
           "mix_pass": {"ms_per_mode": [round(m, 3) for m in ms_modes], "gbs_per_mode": [round(g, 1) for g in gbs],
                        "frac_per_mode": [round(g / hbm_peak, 3) for g in gbs],
                        "bytes_model": "16 B per element per mode (read + write)"}}
    t.synth(cfg["r"], cfg["c"], cfg["eta"], SEED)
    s = pb.Session("mix", t, cfg["r"], cfg["s"],
                   pb.SolveOptions(rng_seed=SEED, max_iters=warmup + steps + 2, bench_mode=True, transform="dct",
                                   x_mutable=True, device=dev))
    s.run(warmup)
    ms = s.timed_enqueue(steps)
    out.update({"value": steps / (ms * 1e-3), "unit": "iters/s", "ms_per_step": ms / steps, "steps": steps,
                "kernel": "fused_iteration_kernel<32, MIX> (persistent)" if s.fused else "multi-kernel chain"})
    s.close()
    if cpu:
        try:
            buf = pb.PinnedBuffer(p)
        except Exception as exc:  # host RAM too small for the 84 GB copy
            out["cpu_baseline"] = {"value": None, "note": f"no host copy of the 84 GB mixed tensor: {exc}"}
        else:
            t.download_into(buf.array)  # the session mixed t in place: X_hat
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as orc
            os.environ.setdefault("CPRAND_THREADS", str(os.cpu_count() or 1))
            per = orc.bench_mix_premixed(buf.array, cfg["dims"], cfg["r"], cfg["s"], "dct", SEED, 1)
            n = int(max(1, min(40, 15.0 / max(per, 1e-6))))
            secs = orc.bench_mix_premixed(buf.array, cfg["dims"], cfg["r"], cfg["s"], "dct", SEED, n)
            out["cpu_baseline"] = {
                "value": n / secs, "unit": "iters/s", "cores": os.cpu_count() or 1, "kind": "port",
                "sample": f"{n} bench-mode CPRAND-MIX iterations (the reference's loop body, mixing.hpp:283-298) "
                          f"on the device-mixed C5 tensor ({secs:.1f} s); bench-iter excludes setup "
                          f"(tools/cprand_main.cpp:195-198), so the host mixing pass (hours) is not run"}
            buf.close()
    t.close()
    return out


def small_records(pb, dev, hbm_peak, steps, warmup, cpu: bool):
    """C1-C3 beside the C4 headline, so every BASELINE.json configuration has a
    driver-run number: bench-mode rate of the persistent kernel, the full loop
    (estimator + stop rule every iteration) with its final fit estimate, the
    one-shot call from a host tensor (e2e), C3's mixing pass, and the CPU
    reference path on the same tensor (bounded sample)."""
    out = {}
    for name in ("c1", "c2", "c3"):
        cfg = CONFIGS[name]
        p = int(np.prod(cfg["dims"]))
        t = pb.DeviceTensor(cfg["dims"], device=dev)
        t.synth(cfg["r"], cfg["c"], cfg["eta"], SEED)
        buf = pb.PinnedBuffer(p)
        t.download_into(buf.array)
        xh = buf.array.reshape(cfg["dims"], order="F")
        rec = {"config": config_of(name, cfg, 1)}
        kw = dict(rng_seed=SEED, transform=cfg["transform"], device=dev)
        s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"],
                       pb.SolveOptions(max_iters=warmup + steps + 2, bench_mode=True, **kw))
        s.run(warmup)
        ms = s.timed_enqueue(steps)
        rec.update({"value": steps / (ms * 1e-3), "unit": "iters/s", "ms_per_step": ms / steps, "steps": steps,
                    "kernel": "persistent kernel" if s.fused else "multi-kernel chain"})
        s.close()
        s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"],
                       pb.SolveOptions(max_iters=steps + 3, fit_sample_count=cfg["phat"], stall_limit=1 << 30, **kw))
        s.run(3)
        s.sync()
        t0 = time.perf_counter()
        n = s.run(steps)
        dt = time.perf_counter() - t0
        rec["full_loop"] = {"value": n / dt, "unit": "iters/s", "iterations": n,
                            "final_fit_estimate": s.result().trace[-1][2]}
        s.close()
        eo = pb.SolveOptions(max_iters=100, bench_mode=True, **kw)
        pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo)  # warm
        t0 = time.perf_counter()
        for _ in range(3):
            res = pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo)
            _ = float(res.lam[0])
        dt = (time.perf_counter() - t0) / 3
        rec["e2e"] = {"value": 100 / dt, "unit": "iters/s", "iters_per_step": 100, "seconds_per_step": dt,
                      "h2d_bytes_per_step": p * 8, "note": "cprand_solve(host tensor), 100 bench-mode iterations"}
        if cfg["method"] == "mix":
            ms_modes = t.mix("dct", SEED)
            gbs = [16.0 * p / (m * 1e-3) / 1e9 for m in ms_modes]
            rec["mix_pass"] = {"ms_per_mode": [round(m, 4) for m in ms_modes], "gbs_per_mode": [round(g, 1) for g in gbs],
                               "frac_per_mode": [round(g / hbm_peak, 3) for g in gbs],
                               "bytes_model": "16 B per element per mode (read + write)"}
        if cpu and cfg["method"] == "mix":
            # bench-iter semantics (setup excluded, tools/cprand_main.cpp:195-198): the reference's loop
            # body on the device-mixed tensor, so the single-threaded host mixing pass is not run
            t.download_into(buf.array)
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as orc
            os.environ.setdefault("CPRAND_THREADS", str(os.cpu_count() or 1))
            per = orc.bench_mix_premixed(buf.array, cfg["dims"], cfg["r"], cfg["s"], "dct", SEED, 1)
            n_it = int(max(1, min(200, 3.0 / max(per, 1e-6))))
            secs = orc.bench_mix_premixed(buf.array, cfg["dims"], cfg["r"], cfg["s"], "dct", SEED, n_it)
            rec["cpu_baseline"] = {"value": n_it / secs, "unit": "iters/s", "cores": os.cpu_count() or 1, "kind": "port",
                                   "sample": f"{n_it} bench-mode CPRAND-MIX iterations on the device-mixed tensor ({secs:.1f} s)"}
        elif cpu:
            rate, n_it, secs = cpu_oracle_rate(xh, cfg, budget_s=3.0, max_iters=200)
            rec["cpu_baseline"] = {"value": rate, "unit": "iters/s", "cores": os.cpu_count() or 1, "kind": "port",
                                   "sample": f"{n_it} bench-mode outer iterations ({secs:.1f} s)"}
        buf.close()
        t.close()
        out[name] = rec
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-iters", type=int, default=100, help="iterations per e2e solve call")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 record of the default (c4) run")
    ap.add_argument("--atomic-gram", action="store_true",
                    help="time the loop with SolveOptions(atomic_gram=True) (not bitwise reproducible)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import paper_1701_06600_b200 as pb
    ws, rank, local = dist_env()
    dist = dist_init(ws)
    dev = local
    hbm_peak, peak_src = peaks()

    # ---- inputs resident in HBM: the whole tensor, or (N > 1) this rank's
    # slab of the last mode (BASELINE.json: slab-sharded with NCCL)
    comm = None
    dims = list(cfg["dims"])
    if ws > 1:
        # the communicator's topology / NVLS choice in the log (to stderr-bound
        # NCCL INFO lines; the JSON line stays the last stdout line)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        from paper_1701_06600_b200 import shard
        uid = [pb.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = pb.Comm(uid[0], rank, ws, dev)
        dims[-1] = shard.slab(cfg["dims"][-1], ws, rank)[1]
    t = pb.DeviceTensor(dims, device=dev)
    if comm is None:
        t.synth(cfg["r"], cfg["c"], cfg["eta"], SEED)
    else:
        t.synth_slab(cfg["r"], cfg["c"], cfg["eta"], SEED, cfg["dims"][-1], comm)
    # MIX on a tensor too large for a private mixed copy beside the replicas
    # (C5, 84 GB): sessions mix `t` in place and `t` is regenerated before
    # each new session, so every session starts from the same tensor
    big = cfg["method"] in ("mix", "premix") and 8 * int(np.prod(dims)) > 40e9

    def fresh():
        if big:
            if comm is None:
                t.synth(cfg["r"], cfg["c"], cfg["eta"], SEED)
            else:
                t.synth_slab(cfg["r"], cfg["c"], cfg["eta"], SEED, cfg["dims"][-1], comm)

    timing_iters = max(args.steps, 10)
    total_iters = args.warmup + args.steps + timing_iters + 2
    opts = pb.SolveOptions(rng_seed=SEED, max_iters=total_iters, bench_mode=True,
                           transform=cfg["transform"], x_mutable=big, device=dev,
                           comm=comm, shard_total=cfg["dims"][-1] if comm is not None else 0,
                           atomic_gram=args.atomic_gram)
    s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"], opts)
    peer_fallback = None
    if ws > 1:
        # the peer kernel's first multi-GPU launches: if any rank's run fails
        # (a peer mapping or a peer wait that timed out raises), every rank
        # agrees and re-runs on the multi-kernel chain with NCCL
        failed = 0.0
        try:
            s.run(args.warmup)
        except Exception as exc:  # noqa: BLE001 - reported in the JSON line
            failed, peer_fallback = 1.0, f"peer kernel failed on rank {rank}: {exc}"
        if allreduce_max(dist, failed) > 0:
            try:
                s.close()
            except Exception:  # noqa: BLE001
                pass
            opts.fused = 0
            s = pb.Session(cfg["method"], t, cfg["r"], cfg["s"], opts)
            peer_fallback = peer_fallback or "peer kernel failed on another rank"
    clk = ClockSampler(dev).__enter__()
    s.run(args.warmup)
    time.sleep(0.3)  # sampler live before the timed region

    # ---- timed region: K steps between CUDA events on the solver stream
    barrier(dist)
    s.sync()
    clk.mark_start()
    ms = s.timed_enqueue(args.steps)
    clk.mark_end()
    clk.__exit__(None, None, None)
    ms = allreduce_max(dist, ms)
    barrier(dist)
    # one global problem: iterations of the whole (sharded) decomposition per second
    value = args.steps / (ms * 1e-3)

    # ---- roofline: per-launch CUDA events on each kernel's own stream
    s.set_kernel_timing(True)
    s.enqueue(timing_iters)
    s.sync()
    n_modes = len(cfg["dims"])
    phases = s.phase_us()
    kinds = ["gather", "rhs_gemm", "z", "gram", "gram_inverse", "apply", "mix_factor", "fused_iteration"]
    stats = {k: [s.kernel_stats(m, i) for m in range(n_modes)] for i, k in enumerate(kinds)}
    breakdown = {k: [round(x[1] / x[0] * 1e3, 2) if x[0] else None for x in st]
                 for k, st in stats.items() if sum(x[0] for x in st)}
    elems = [cfg["s"] * d for d in cfg["dims"]]
    gather = stats["gather"]
    gemm = stats["rhs_gemm"]
    gemm_ms = sum(g[1] for g in gemm)
    gemm_tflops = sum(g[2] for g in gemm) / (gemm_ms * 1e-3) / 1e12 if gemm_ms else 0.0
    fused = stats["fused_iteration"][0]
    if fused[0]:
        # one persistent kernel per outer iteration: its algorithmic bytes are
        # every mode's sampled fibers (8 B/elem, read in place) + Z_S
        kname = ("fused_rand_kernel (CPRAND: all modes of an outer iteration, persistent, flag hand-offs)"
                 if cfg["method"] == "rand" else
                 "fused_iteration_kernel (CPRAND-MIX: all modes of an outer iteration, persistent)")
        launches, kms = fused[0], fused[1]
        kbytes = launches * sum(e * 8 + cfg["s"] * cfg["r"] * 8 for e in elems)
        per_mode = None
        bytes_model = "fibers 8 B/elem (in place) + Z_S 8 B/entry, all modes"
        gemm_tflops = launches * sum(2.0 * e * cfg["r"] for e in elems) / (kms * 1e-3) / 1e12
    elif sum(g[0] for g in gather):
        # sampled-fiber gather kernel: B_min bytes (8 B/elem mode 1, 32 B/elem strided)
        kname = "gather_rows_kernel (sampled-fiber gather)"
        launches = sum(g[0] for g in gather)
        kms = sum(g[1] for g in gather)
        kbytes = sum(g[2] for g in gather)
        per_mode = [g[2] / (g[1] * 1e-3) / 1e9 if g[0] else None for g in gather]
        bytes_model = "B_min: 8 B/elem mode 1, 32 B/elem strided modes"
    else:
        # every mode reads its sampled fibers in place (mode 1 / mode-major
        # replicas): the dominant kernel is the RHS GEMM, whose algorithmic
        # bytes are the sampled fibers (8 B/elem, contiguous rows) + Z_S
        kname = "rhs_gemm_kernel (in-place fiber reads + Z_S^T X_S^T)"
        launches = sum(g[0] for g in gemm)
        kms = gemm_ms
        kbytes = sum((e * 8 + cfg["s"] * cfg["r"] * 8) * g[0] for e, g in zip(elems, gemm))
        per_mode = [(e * 8 + cfg["s"] * cfg["r"] * 8) / (g[1] / g[0] * 1e-3) / 1e9 for e, g in zip(elems, gemm)]
        bytes_model = "fibers 8 B/elem (contiguous rows) + Z_S 8 B/entry"
    achieved = (kbytes / launches) / (kms / launches * 1e-3) / 1e9
    share = (kms / timing_iters) / (ms / args.steps)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("traffic_bytes_per_launch")
    fallbacks = s.gram_fallbacks()
    used_fused = bool(fused[0])
    # ---- the metric's "sampled-gather HBM GB/s vs peak": gather_fibers of
    # 10 iterations' sample tables (every mode) into scratch, batched (the
    # samples are data independent), from the mode-major replicas and from
    # the tensor's own layout (B_min = 8 B / element for
    # contiguous rows, 32 B for strided modes)
    gather = None
    if comm is None:
        gi = min(10, total_iters)
        ms_r, bu_r, bm_r = s.gather_bench(gi, True)
        ms_x, bu_x, bm_x = s.gather_bench(gi, False)
        gather = {"iterations": gi, "kernel": "gather_rows_kernel",
                  "replicas": {"ms": round(ms_r, 4), "useful_gbs": round(bu_r / (ms_r * 1e-3) / 1e9, 1),
                               "frac_useful": round(bu_r / (ms_r * 1e-3) / 1e9 / hbm_peak, 3),
                               "read_write_gbs": round(2 * bu_r / (ms_r * 1e-3) / 1e9, 1),
                               "frac_read_write": round(2 * bu_r / (ms_r * 1e-3) / 1e9 / hbm_peak, 3)},
                  "tensor_layout": {"ms": round(ms_x, 4), "useful_gbs": round(bu_x / (ms_x * 1e-3) / 1e9, 1),
                                    "b_min_gbs": round(bm_x / (ms_x * 1e-3) / 1e9, 1),
                                    "frac_b_min": round(bm_x / (ms_x * 1e-3) / 1e9 / hbm_peak, 3)},
                  "note": "one launch per mode over all iterations' fibers (strided modes processed in "
                          "base-offset order); useful / B_min count the reads, read_write adds the X_S write "
                          "(8 B / element); the solver itself reads the fibers in place inside the persistent "
                          "kernel. ncu (profiles/r02_gather_c4.txt): a strided 8 B element moves 127 B of "
                          "DRAM (the L2 fetches whole 128 B lines; cudaLimitMaxL2FetchGranularity 32 is "
                          "accepted but not applied), so the strided pass runs at ~86 % of HBM by DRAM bytes",
                  "dram_bytes_per_strided_element_ncu": 127.4}
    s.close()

    # ---- full loop (sampled fit estimate + stop rule every iteration) and
    # time to fit, both from the same resident tensor
    full, ttf = fit_runs(pb, t, cfg, dev, comm, args.steps, fresh, big)

    # ---- the same timed loop with the Gram summed by L2 fp64 atomics
    # (SolveOptions.atomic_gram: one round trip fewer per mode, not bitwise
    # reproducible; reported beside the default, reproducible, value)
    atomic = None
    if cfg["method"] == "rand" and not args.atomic_gram:
        import dataclasses
        s2 = pb.Session(cfg["method"], t, cfg["r"], cfg["s"], dataclasses.replace(opts, atomic_gram=True))
        s2.run(args.warmup)
        barrier(dist)
        s2.sync()
        ms2 = allreduce_max(dist, s2.timed_enqueue(args.steps))
        s2.close()
        atomic = {"value": args.steps / (ms2 * 1e-3), "unit": "iters/s", "ms_per_step": ms2 / args.steps,
                  "option": "SolveOptions(atomic_gram=True)"}

    # ---- host copy of the tensor for e2e / cpu_baseline, taken before the
    # mixing-pass measurement below mixes `t` in place
    fresh()
    want_host = (rank == 0 or comm is not None) and (args.e2e_steps > 0 or (not args.no_cpu and ws == 1))
    buf = None
    p = int(np.prod(dims))
    if want_host:
        try:
            buf = pb.PinnedBuffer(p)
            t.download_into(buf.array)
        except Exception as exc:  # host RAM too small for a pinned copy
            buf, host_skip = None, f"no pinned host copy of the {8 * p / 1e9:.1f} GB tensor: {exc}"
    # ---- CPRAND-MIX preprocessing pass (mix_tensor, in place) on the same tensor
    mix_pass = None
    if rank == 0 and comm is None:
        ms_modes = t.mix("dct", SEED)
        pbytes = 16.0 * float(p)
        gbs = [pbytes / (m * 1e-3) / 1e9 for m in ms_modes]
        mix_pass = {"kernel": ("mixing pass v4 (mixreg.cu, whole-tensor sign + DCT-II per fiber, in place): "
                               "mix_reg3c_kernel on mode 1, mix_reg3_kernel on the strided modes" if cfg["dims"][0] == 1000
                               else "mixing pass (whole-tensor sign + DCT-II per fiber, in place)"),
                    "bytes_model": "16 B per element per mode (read + write)",
                    "ms_per_mode": [round(m, 3) for m in ms_modes],
                    "gbs_per_mode": [round(g, 1) for g in gbs],
                    "frac_per_mode": [round(g / hbm_peak, 3) for g in gbs]}
    t.close()  # e2e allocates its own device copy

    # ---- e2e through the public one-shot call with host buffers
    e2e, cpu = None, None
    if buf is not None:
        xh = buf.array.reshape(dims, order="F")
        eo = pb.SolveOptions(rng_seed=SEED, max_iters=args.e2e_iters, bench_mode=True,
                             transform=cfg["transform"], device=dev, comm=comm,
                             shard_total=cfg["dims"][-1] if comm is not None else 0)
        if args.e2e_steps > 0:
            pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo)  # warm
            t0 = time.perf_counter()
            calls = []
            for _ in range(args.e2e_steps):
                tc = time.perf_counter()
                res = pb.solve(cfg["method"], xh, cfg["r"], cfg["s"], eo)
                _ = float(res.lam[0])  # result on the host
                calls.append({"wall": round(time.perf_counter() - tc, 4), "setup": round(res.setup_seconds, 4),
                              "loop_device": round(res.loop_seconds_device, 4)})
            dt = (time.perf_counter() - t0) / args.e2e_steps
            table_bytes = args.e2e_iters * n_modes * cfg["s"] * ((n_modes - 1) * 4 + 8)
            e2e = {"value": args.e2e_iters / dt, "unit": "iters/s",
                   "h2d_bytes_per_step": p * 8 + table_bytes,
                   "d2h_bytes_per_step": 8 * cfg["r"] * (sum(cfg["dims"]) + 1),
                   "iters_per_step": args.e2e_iters, "seconds_per_step": dt, "calls": calls,
                   "note": "cprand_solve(host pinned tensor): H2D + setup + bench-mode loop + D2H"}
        if not args.no_cpu and ws == 1:
            if cfg["method"] == "mix" and p > (1 << 31):
                cpu = {"value": None, "unit": "iters/s", "cores": os.cpu_count() or 1, "kind": "port",
                       "sample": "not run: the CPU path's setup mixes the whole tensor with a single-threaded "
                                 "Bluestein DCT per fiber (hours at this size), SURVEY.md 8(d)"}
            else:
                rate, n_it, secs = cpu_oracle_rate(xh, cfg)
                cpu = {"value": rate, "unit": "iters/s", "cores": os.cpu_count() or 1, "kind": "port",
                       "sample": f"{n_it} bench-mode outer iterations of {args.config} on the same "
                                 f"tensor ({secs:.1f} s); gather on all host threads, LS single-threaded"}
        buf.close()
    elif want_host:
        e2e = {"value": None, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": host_skip}

    c5 = None
    if args.config == "c4" and ws == 1 and not args.no_c5:
        pb.lib().cprand_device_cache_release()
        c5 = c5_record(pb, dev, hbm_peak, args.steps, args.warmup, not args.no_cpu)
        pb.lib().cprand_device_cache_release()

    small = None
    if args.config == "c4" and ws == 1 and not args.no_c5:
        small = small_records(pb, dev, hbm_peak, args.steps, args.warmup, not args.no_cpu)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE.json generator in HBM, seed 1)",
            "config": config_of(args.config, cfg, ws),
            "gram_sum": "L2 fp64 atomics (atomic_gram)" if args.atomic_gram else
                        "fixed-order split partials (bitwise reproducible)",
            "comm": (("peer kernel: RHS rows / last-mode slabs stored into every rank's buffers "
                      "(CUDA IPC mappings over NVLink, sys-scope flags); NCCL for setup")
                     if used_fused else "NCCL allreduce / allgather / send-recv") if ws > 1 else None,
            "peer_fallback": peer_fallback,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "kernel": kname,
                         "bytes_model": bytes_model, "per_mode_gbs": per_mode,
                         "share_of_step": share, "peak_source": peak_src,
                         "rhs_gemm_fp64_tflops": gemm_tflops,  # fused: RHS flops over the whole kernel
                         "rhs_gemm_fp64_frac_of_dfma": gemm_tflops / DFMA_PEAK_TF,
                         "per_kernel_us_by_mode": breakdown,
                         "fused_phase_us_per_mode": dict(zip(
                             (["z", "z_barrier", "phaseB_cta0", "B_barrier", "apply", "apply_barrier",
                               "inverse_done_after_z_barrier"] if cfg["method"] == "mix" else
                              ["z_tile", "gram_blocks", "rhs_tiles", "apply_share", "ssq", "release",
                               "inverse_done_after_mode_start", "gram_ready_after_mode_start",
                               "z_share_done_after_mode_start", "z_split_ready_after_mode_start",
                               "inverse_prologue", "inverse_steps", "norms_done_after_mode_start",
                               "gram_reduce"]),
                             [round(x, 2) for x in phases])) if phases else None,
                         "gram_fallbacks": fallbacks, "mix_pass": mix_pass},
            "atomic_gram": atomic, "full_loop": full, "time_to_fit": ttf, "sampled_gather": gather,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "c5": c5, "c1_c3": small,
            "gpu_launches": launches_per_iter(cfg, used_fused) * args.steps,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
