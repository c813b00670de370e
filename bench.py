#!/usr/bin/env python
"""VDAMP image-iterations/s on B200 (BASELINE.json metric), one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--precision fp32|fp64]
                    [--impl ours|reference] [--no-extras] [--with-trace]

A step = one VDAMP reconstruction (setup scatter, 30 iterations, finalize)
of one batch of synthetic slices of ``--config`` (default cfg1: 64 x 256^2
complex64, Haar s=4, R=4, 40 dB).  Each rank reconstructs its own batch of
distinct slices (weak scaling, no collective in the data path).

value        device-resident: inputs already in HBM, CUDA events per step, L2
             flushed (256 MiB write) between steps, max over ranks.
e2e          the public StreamingReconstructor with pinned host inputs; H2D of
             y / indices / density and D2H of x_hat inside the timed region.
fixed_batch  BASELINE's "64 slices sharded across 1/2/4/8 GPUs": the config's
             batch split over the ranks, dist.gather of x_hat to rank 0 timed.
configs      (1 GPU) the other BASELINE configs and the fp64 parity mode, each
             device-resident with its own B_iter roofline.
roofline     dominant kernel class: algorithmic bytes / its
             CUDA-event time inside the timed region, vs MEASURED_PEAKS hbm_gbs.
cpu_baseline the numpy oracle port (oracle/vdamp_oracle.py) on a bounded
             sample of the same slices, all host cores and one core.
--impl reference  times that oracle port alone on the same slices (rank 0;
             other ranks exit 0).
"""

from __future__ import annotations

import os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1911_01234_b200 import workload  # noqa: E402

METRIC = "VDAMP image-iterations/s"
UNIT = "img-iter/s"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------- CPU leg --
_W = None


def _oracle_slice(b):
    from oracle import vdamp_oracle as O
    w = _W
    O.run(w.ys[b].astype(np.complex128), w.masks[b].indices, w.pmap.probs, float(w.noise_vars[b]),
          w.config.scales, w.config.n_iters)
    return b


def cpu_oracle_rate(w, n_images, procs, repeats=1):
    """img-iter/s of the oracle on the first n_images slices of w, `procs` processes (fork)."""
    import multiprocessing as mp
    global _W
    _W = w
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_oracle_slice, [0])                        # warm the workers' imports
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            pool.map(_oracle_slice, [i % len(w.masks) for i in range(n_images)], chunksize=1)
            times.append(time.perf_counter() - t0)
    return n_images * w.config.n_iters / float(np.mean(times)), times


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled in a thread during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock"}

    def __init__(self, index, period=0.02):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self.period = period
        self.samples = []
        self.reasons = 0
        self._stop = threading.Event()

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.samples)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def class_bytes(cfg, N, n_mean, images, iters, b_c):
    """Algorithmic bytes per kernel class over `iters` iterations of `images` images."""
    f = b_c / 8.0
    it = images * iters
    return {
        "synth_rowfft": 16 * N * f * it,                         # read r, write T1
        "col_residual": (16 * N + 12 * n_mean) * f * it + N / 8 * it,   # T1, y, 1/p, mask -> T2
        "rowifft_analysis": 24 * N * f * it,                     # T2, r -> r
        "sure_select": 8 * N * f * it,                           # read r
        "finalize": (48 * N + 8 * n_mean) * f * images,          # once per run
    }


def traffic_from_profiles(kernel_class):
    """(dram bytes per launch, source note) from the committed ncu summary (profiles/), if present."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel_class), d.get("_note")
    except Exception:
        return None, None


# ------------------------------------------------------- per-config lines --
EXTRAS = [("cfg1", "fp64"), ("cfg0", "fp32"), ("cfg2", "fp32"), ("cfg2", "fp64"), ("cfg3", "fp32"),
          ("cfg3", "fp64"), ("cfg4_r2", "fp32"), ("cfg4_r2", "fp64"), ("cfg4_r4", "fp32"),
          ("cfg4_r8", "fp32"), ("cfg4_r8", "fp64"), ("cfg4_r16", "fp32"), ("cfg4_r16", "fp64")]


def measure_config(name, precision, steps, warmup, local, procs, peak, trace=False):
    """Device-resident img-iter/s of one BASELINE config on this GPU (same timing rules as
    the headline: CUDA events per step, L2 flushed between steps, all images of the config).
    trace: with ground truth, i.e. per-iteration NMSE and trace records as the reference CLI
    asks for (src/cli.py:51-55)."""
    import torch
    from paper_1911_01234_b200 import vdamp
    from paper_1911_01234_b200.plan import clear_plans
    cfg = workload.CONFIGS[name]
    w = workload.make_workload(cfg, procs=procs)
    inp = vdamp.prepare_batch(w.ys, w.masks, w.pmap, w.noise_vars)
    dev = torch.device("cuda", local)
    rec = vdamp.BatchReconstructor(cfg.size, cfg.size, cfg.scales, cfg.batch, precision=precision, device=local)
    cd = rec.plan.cdtype
    y = torch.from_numpy(inp.y).to(dev, cd)
    idx = torch.from_numpy(inp.indices).to(dev)
    probs = torch.from_numpy(inp.probs).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    step = lambda: rec(y, idx, inp.counts, probs, inp.noise_var, cfg.n_iters, shared_probs=True, sync=False)
    if trace:
        plan = rec.plan
        plan.set_measurements(y, idx, inp.counts, probs, inp.noise_var, True)
        plan.set_ground_truth(torch.from_numpy(w.x0).to(dev, cd))
        trace_buf = plan.new_trace(cfg.n_iters)
        nmse_buf = torch.zeros((cfg.n_iters, cfg.batch, 2), dtype=torch.float64, device=dev)

        def step():
            plan.set_measurements(y, idx, inp.counts, probs, inp.noise_var, True, sync_validation=False)
            return plan.run(cfg.n_iters, x_hat=rec._x, trace=trace_buf, nmse=nmse_buf)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    rec.plan.measurement_status(wait=True)
    ms = [a.elapsed_time(b) for a, b in evs]
    value = cfg.batch * cfg.n_iters * steps / (sum(ms) / 1e3)
    n_mean = float(np.mean(inp.counts))
    b_c = 8 if precision == "fp32" else 16
    b_iter = workload.algorithmic_bytes_per_image_iter(cfg.size * cfg.size, n_mean, b_c)
    out = {"value": value, "unit": UNIT, "precision": precision, "images": cfg.batch, "n_iters": cfg.n_iters,
           "steps": steps, "ms_per_step": float(np.mean(ms)),
           "trace": "ground truth + per-iteration NMSE/trace records" if trace else "off",
           "workload": f"{cfg.batch} x {cfg.size}^2, Haar s={cfg.scales}, R={cfg.undersampling:g}, "
                       f"{cfg.snr_db:g} dB, {cfg.n_iters} iterations",
           "iteration_roofline": {"B_iter_bytes": b_iter, "achieved_GBps": value * b_iter / 1e9,
                                  "frac": value * b_iter / 1e9 / peak}}
    del rec, y, idx, probs, flush
    clear_plans()
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--batch", type=int, default=None, help="images per rank (default: config batch)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-depth", type=int, default=1, help="batches reconstructing side by side in the e2e leg")
    ap.add_argument("--quick", action="store_true", help="print a short human summary instead of JSON")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the per-config lines (cfg0/2/3/4 and fp64) of a 1-GPU run")
    ap.add_argument("--extras-steps", type=int, default=5)
    ap.add_argument("--with-trace", action="store_true",
                    help="time the production trace path: ground truth set, per-iteration NMSE + trace records")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    cfg = workload.CONFIGS[args.config]
    B = args.batch or cfg.batch
    cores = host_cores()

    if args.impl == "reference":
        if rank != 0:
            return
        ns = min(B, 64)                                  # the same slices as our arm (cfg1: all 64)
        w = workload.make_workload(cfg, batch=ns, procs=cores)
        rates = []
        t_all = []
        rate, _ = cpu_oracle_rate(w, ns, cores, repeats=args.warmup)    # warm-up steps
        for _ in range(args.steps):
            r, t = cpu_oracle_rate(w, ns, cores, repeats=1)
            rates.append(r)
            t_all += t
        value = ns * cfg.n_iters * args.steps / float(np.sum(t_all))
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(t_all)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded BASELINE workload generator)",
            "config": {"workload": f"{cfg.name}: {cfg.size}^2 complex, Haar s={cfg.scales}, R={cfg.undersampling:g}, "
                                   f"{cfg.snr_db:g} dB, {cfg.n_iters} iterations", "images_per_step": ns},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                             "sample": f"{ns} slices x {cfg.n_iters} iterations per step (the first {ns} slices of "
                                       f"our arm's batch), one slice per process "
                                       f"(oracle/vdamp_oracle.py, numpy float64)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    # ---- our arm ------------------------------------------------------
    w = workload.make_workload(cfg, batch=B, first=rank * B)
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ns = max(8, min(2 * cores, B))                     # ~0.55 s of CPU per slice: 10-30 s of work
        rate, ts = cpu_oracle_rate(w, ns, cores, repeats=1)
        n1 = 2
        rate1, ts1 = cpu_oracle_rate(w, n1, 1, repeats=1)
        cpu_base = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                    "sample": f"{ns} of the {B} slices x {cfg.n_iters} iterations, one slice per process, "
                              f"{cores} processes (oracle/vdamp_oracle.py, numpy float64), {ts[0]:.1f} s wall",
                    "one_core": {"value": rate1, "unit": UNIT, "cores": 1,
                                 "sample": f"{n1} slices x {cfg.n_iters} iterations in one process, {ts1[0]:.1f} s"}}

    import torch
    import torch.distributed as dist
    from paper_1911_01234_b200 import vdamp
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    inp = vdamp.prepare_batch(w.ys, w.masks, w.pmap, w.noise_vars)
    rec = vdamp.BatchReconstructor(cfg.size, cfg.size, cfg.scales, B, precision=args.precision, device=local)
    plan = rec.plan
    cd = plan.cdtype
    dev_in = dict(y=torch.from_numpy(inp.y).to(dev, cd), indices=torch.from_numpy(inp.indices).to(dev),
                  counts=inp.counts, probs=torch.from_numpy(inp.probs).to(dev), noise_var=inp.noise_var)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    trace_buf = nmse_buf = None
    if args.with_trace:
        plan.set_measurements(dev_in["y"], dev_in["indices"], dev_in["counts"], dev_in["probs"], dev_in["noise_var"], True)
        plan.set_ground_truth(torch.from_numpy(w.x0).to(dev, cd))
        trace_buf = plan.new_trace(cfg.n_iters)
        nmse_buf = torch.zeros((cfg.n_iters, B, 2), dtype=torch.float64, device=dev)

    def step():
        if args.with_trace:
            plan.set_measurements(dev_in["y"], dev_in["indices"], dev_in["counts"], dev_in["probs"],
                                  dev_in["noise_var"], True, sync_validation=False)
            return plan.run(cfg.n_iters, x_hat=rec._x, trace=trace_buf, nmse=nmse_buf)
        return rec(dev_in["y"], dev_in["indices"], dev_in["counts"], dev_in["probs"], dev_in["noise_var"],
                   cfg.n_iters, shared_probs=True, sync=False)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- device-resident timed region (no per-kernel events inside) ---
    plan.launch_count(reset=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))                       # evict L2 between steps (untimed)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    launches = plan.launch_count()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    # per-kernel-class breakdown (roofline): the same steps again with CUDA
    # events around every launch, on the launching stream; not used for value.
    # One lane, so each event pair brackets its own kernel only.
    plan.set_lanes(1)
    plan.set_timing(True)
    for i in range(args.steps):
        flush.fill_(float(i))
        step()
    torch.cuda.synchronize(dev)
    ktimes = plan.kernel_times()
    plan.set_timing(False)
    plan.set_lanes(0)                       # back to the default lanes (the e2e arms share this plan)
    total_s = max_over_ranks(float(np.sum(step_ms)) / 1e3)
    images_all = B * world
    value = images_all * cfg.n_iters * args.steps / total_s
    ms_per_step = 1e3 * total_s / args.steps

    # ---- end to end through the public call, pinned host buffers -----
    e2e = None
    if not args.no_e2e:
        host = rec.upload(inp, pin=True)
        out = torch.empty((B, cfg.size, cfg.size), dtype=cd).pin_memory()
        h2d = (host["y"].numel() * host["y"].element_size() + host["indices"].numel() * 8
               + host["probs"].numel() * 8 + B * 8)
        d2h = out.numel() * out.element_size()
        # (a) one synchronous call per batch (copy in, reconstruct, copy out, wait)
        for _ in range(args.warmup):
            rec(host["y"], host["indices"], host["counts"], host["probs"], host["noise_var"], cfg.n_iters, out=out)
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rec(host["y"], host["indices"], host["counts"], host["probs"], host["noise_var"], cfg.n_iters, out=out)
        t_sync = max_over_ranks(time.perf_counter() - t0)
        barrier()
        # (b) the streaming API: batch k+1's H2D and batch k-1's D2H overlap batch k; at the
        # default depth 2 the reconstructions of two consecutive batches also run side by side
        # (own plans and streams); depth 1 (one reconstruction at a time) is reported beside it
        def stream_run(depth):
            srec = vdamp.StreamingReconstructor(cfg.size, cfg.size, cfg.scales, B, precision=args.precision,
                                                device=local, depth=depth)
            outs = [torch.empty_like(out).pin_memory() for _ in range(depth + 1)]
            for i in range(max(args.warmup, depth + 1)):
                srec.submit(host, cfg.n_iters, outs[i % len(outs)])
            srec.wait()
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for i in range(args.steps):
                srec.submit(host, cfg.n_iters, outs[i % len(outs)])
            srec.wait()
            t = max_over_ranks(time.perf_counter() - t0)
            barrier()
            assert torch.equal(outs[0], out), "streaming result differs from the synchronous call"
            return t
        t_e2e = stream_run(args.e2e_depth)
        e2e = {"value": images_all * cfg.n_iters * args.steps / t_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": 1e3 * t_e2e / args.steps,
               "api": "StreamingReconstructor.submit: H2D of batch k+1 and D2H of batch k-1 overlap the reconstruction "
                      "of batch k; x_hat checked bitwise against the synchronous call",
               "depth": args.e2e_depth,
               "sync_call_value": images_all * cfg.n_iters * args.steps / t_sync}

    # ---- fixed batch sharded across the ranks (BASELINE cfg1/cfg4 wording) ----
    # the config's batch (cfg1: 64 slices) split into contiguous slices, one per rank;
    # each timed step reconstructs the rank's slice and gathers x_hat to rank 0
    # (dist.gather over NCCL, the only collective) inside the timed region
    fixed = None
    if not args.with_trace:
        from paper_1911_01234_b200.dist import gather_images, shard_range
        Bf = cfg.batch
        if world == 1 and B == Bf:
            fixed = {"value": value, "ms_per_step": ms_per_step, "images": Bf,
                     "note": "N=1: the headline steps themselves (no gather)"}
        else:
            lo, hi = shard_range(Bf, rank, world)
            if hi > lo:
                wf = workload.make_workload(cfg, batch=hi - lo, first=lo)
                inf = vdamp.prepare_batch(wf.ys, wf.masks, wf.pmap, wf.noise_vars)
                recf = vdamp.BatchReconstructor(cfg.size, cfg.size, cfg.scales, hi - lo, precision=args.precision,
                                                device=local)
                fin = dict(y=torch.from_numpy(inf.y).to(dev, cd), indices=torch.from_numpy(inf.indices).to(dev),
                           probs=torch.from_numpy(inf.probs).to(dev))
                fstep = lambda: recf(fin["y"], fin["indices"], inf.counts, fin["probs"], inf.noise_var, cfg.n_iters,
                                     shared_probs=True, sync=False)
            else:
                fstep = lambda: torch.empty((0, cfg.size, cfg.size), dtype=cd, device=dev)

            def fstep_gather():
                x = fstep()
                return gather_images(x, Bf) if world > 1 else x
            for _ in range(args.warmup):
                fstep_gather()
            torch.cuda.synchronize(dev)
            fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            barrier()
            for i in range(args.steps):
                flush.fill_(float(i))
                fev[i][0].record(stream)
                fstep_gather()
                fev[i][1].record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            tf = max_over_ranks(sum(a.elapsed_time(b) for a, b in fev) / 1e3)
            fixed = {"value": Bf * cfg.n_iters * args.steps / tf, "ms_per_step": 1e3 * tf / args.steps, "images": Bf,
                     "gather": "dist.gather of x_hat to rank 0 inside the timed region" if world > 1 else "none (N=1)"}
        fixed.update(unit=UNIT, scaling="strong",
                     workload=f"{cfg.name}: {Bf} x {cfg.size}^2 slices in total, contiguous slice per rank")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- the other BASELINE configs and the fp64 parity mode (1 GPU) ----
    peak, peak_src = measured_peak()
    extras = None
    if world == 1 and not args.no_extras and not args.with_trace and args.config == "cfg1" and args.batch is None:
        extras = {}
        for name, prec in EXTRAS:
            if name == cfg.name and prec == args.precision:
                continue
            try:
                extras[f"{name}_{prec}"] = measure_config(name, prec, args.extras_steps, 3, local, cores, peak)
            except Exception as e:          # report, never hide a failure
                extras[f"{name}_{prec}"] = {"error": f"{type(e).__name__}: {e}"}
        try:                                # the production path: ground truth given, trace recorded
            extras[f"{cfg.name}_{args.precision}_trace"] = measure_config(cfg.name, args.precision, args.extras_steps, 3,
                                                                          local, cores, peak, trace=True)
        except Exception as e:
            extras[f"{cfg.name}_{args.precision}_trace"] = {"error": f"{type(e).__name__}: {e}"}

    # ---- roofline of the dominant kernel class -----------------------
    N = cfg.size * cfg.size
    n_mean = float(np.mean(inp.counts))
    b_c = 8 if args.precision == "fp32" else 16
    cb = class_bytes(cfg, N, n_mean, B, cfg.n_iters * args.steps, b_c)
    cb["finalize"] *= args.steps
    dom = max((k for k in cb), key=lambda k: ktimes[k][0])
    kms, kl = ktimes[dom]
    achieved = cb[dom] / (kms / 1e3) / 1e9
    traffic, traffic_src = traffic_from_profiles(dom)
    kernels = {k: {"ms_per_step": ktimes[k][0] / args.steps, "launches_per_step": ktimes[k][1] / args.steps,
                   "GBps": (cb[k] / (ktimes[k][0] / 1e3) / 1e9) if ktimes[k][0] > 0 and k in cb else None}
               for k in ktimes}
    b_iter = workload.algorithmic_bytes_per_image_iter(N, n_mean, b_c)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c64" if args.precision == "fp32" else "c128",
        "data": "synthetic (seeded BASELINE workload generator: random ellipses x smooth phase, offset-law masks)",
        "config": {"workload": f"{cfg.name}: {B} x {cfg.size}^2 complex slices per GPU, Haar s={cfg.scales}, "
                               f"R={cfg.undersampling:g}, {cfg.snr_db:g} dB, {cfg.n_iters} iterations",
                   "images_per_gpu": B, "n_iters": cfg.n_iters, "precision": args.precision,
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "trace": "ground truth + per-iteration NMSE/trace records" if args.with_trace else "off (as the CPU timing)",
                   "parallelism": f"images sharded, {world} process(es), 1 GPU each, no collective"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": cb[dom] / max(kl, 1),
                     "avg_launch_ms": kms / max(kl, 1)},
        "iteration_roofline": {"B_iter_bytes": b_iter, "achieved_GBps": value / world * b_iter / 1e9,
                               "frac": value / world * b_iter / 1e9 / peak},
        "kernels": kernels,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if e2e is not None:
        line["e2e"] = e2e
    if fixed is not None:
        line["fixed_batch"] = fixed
    if extras is not None:
        line["configs"] = extras
    if cpu_base is not None:
        line["cpu_baseline"] = cpu_base
    if args.quick:
        print(f"value={value:.0f} ms/step={ms_per_step:.3f} clocks={line['clocks']}")
        for k, v in kernels.items():
            print(f"  {k:18s} {v['ms_per_step']:.3f} ms/step  {v['GBps'] or 0:.0f} GB/s")
    else:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
