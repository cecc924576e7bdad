#!/usr/bin/env python
"""BaB-ND hot-path benchmark on B200 (BASELINE.json metric: subdomains bounded/s
and sample*steps/s).

A step is one steady-state BaB iteration of the C2 workload (BASELINE.json
configs[1]: MLP [12,128,128,128,10], H=20, M=1024 samples per CEM iteration,
10 CEM iterations, D=512 children = 2 x batch 256): pick_out, split, device
search (Philox sampling -> fused rollout + extrema -> incumbent / top-K / CEM
refit), device early-stop CROWN bound, merge, prune.  Timed with CUDA events on
the launching stream, L2 flushed between steps, max over ranks.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): one planner sharded over the ranks -- every iteration's
children go round-robin to the GPUs and their reports are allgathered over
NCCL (paper_2412_09584_b200.parallel); the batch grows with the GPU count so
each GPU keeps D=512 children per step (weak scaling).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


TF32_DENSE_TFLOPS = 1100.0  # /opt/skills/guides/B200_PROFILING.md, dense (non-sparse) TF32


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_children_per_s(wl, n_children: int, steps: int = 1, warmup: int = 0):
    """The oracle (FP64 CPU restatement of the reference path) on n_children boxes:
    batch_search + CrownBounder::lower, all host threads (parallel_chunks over boxes)."""
    from oracle import oracle as orc
    from paper_2412_09584_b200 import workloads

    ob = orc.Objective(wl.spec)
    los, his = workloads.presplit_boxes(wl.spec, n_children)
    cfg = wl.planner_config()
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        reps = ob.batch_search(los, his, None, cfg, seed=1000 + i)
        reps.bound_all()
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return n_children / (sum(times) / len(times)), times, orc.thread_count()


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc

    n = max(8, orc.thread_count())
    rate, times, cores = cpu_children_per_s(wl, n, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": "subdomains_bounded_per_s", "value": rate, "unit": "subdomains/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the same workload as this repo's arm (its config keys); each timed step is a bounded sample of it
        "config": {"workload": f"{wl.name} (BASELINE.json configs[1])", "widths": wl.spec.widths, "H": wl.spec.horizon,
                   "M": wl.samples_per_iter, "D_per_step": n, "cem_iterations": wl.planner_config()["search"]["iterations"],
                   "batch": wl.planner_config()["batch"], "parallelism": "host threads",
                   "sample": f"{n} pre-split boxes per step (the GPU arm bounds {2 * wl.planner_config()['batch']} per step)"},
        "cpu_baseline": {"value": rate, "unit": "subdomains/s", "cores": cores, "kind": "port",
                         "sample": f"{n} pre-split C2 boxes per step: batch_search (CEM, M=1024, 10 iters) + "
                                   "early-stop-empirical CROWN, FP64 oracle restatement (reference does not build "
                                   "here: Eigen/vendor headers absent)"},
        "e2e": {"value": rate, "unit": "subdomains/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_2412_09584_b200 import workloads

    wl = workloads.ALL[args.config]()
    if args.impl == "reference":
        run_reference(args, wl)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2412_09584_b200 as bp

    peak_fp32 = peak_tf32 = None
    if rank == 0:
        import ctypes as C
        from paper_2412_09584_b200 import _capi
        t, ms = C.c_double(), C.c_double()
        _capi.check(_capi.load().bp_measure_fp32_peak(local, C.byref(t), C.byref(ms)))
        peak_fp32 = t.value
        _capi.check(_capi.load().bp_measure_tf32_peak(local, C.byref(t), C.byref(ms)))
        peak_tf32 = t.value

    from paper_2412_09584_b200 import parallel

    dev = bp.Device(local).load(wl.spec)
    path = dev.rollout_path()  # "tcgen05" (3xTF32 tensor cores) or "simt" (FP32 FFMA)
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    parallel.attach(dev)
    cfg = wl.planner_config()
    cfg["batch"] = cfg["batch"] * world
    cfg["termination"]["max_iterations"] = 10**6
    planner = dev.planner(cfg)
    batch = cfg["batch"]
    setup = 0
    while True:  # grow the pool to the steady-state batch (2*batch children per step)
        ok, ch, pool = planner.step()
        setup += 1
        if pool >= batch or setup >= 16:
            break
    for _ in range(args.warmup):
        planner.step()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    dev.timing()
    bp.Device.io_bytes()
    step_ms, children = [], 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (outside the timed interval)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            ok, ch, pool = planner.step()
            ev1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            children += ch
    tm = dev.timing()
    total_ms = sum(step_ms)
    stats = torch.tensor([total_ms, float(children), tm["rollout_ms"], float(tm["launches"])], device="cuda",
                         dtype=torch.float64)
    if world > 1:
        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        total_ms_max = mx[0].item()
    else:
        total_ms_max = total_ms
    children_all = float(children)  # the planner's global child count (identical on every rank)
    rows = wl.rows_per_search_iter
    H = wl.spec.horizon
    iters = cfg["search"]["iterations"]
    value = children_all / (total_ms_max / 1e3)
    sample_steps = children_all * rows * iters * H / (total_ms_max / 1e3)
    # roofline of the dominant kernel (rollout): algorithmic FLOPs / device time of its launches
    flop = children / world * rows * iters * H * wl.flops_per_sample_step  # this rank's share
    achieved = flop / (tm["rollout_ms"] / 1e3) / 1e12 if tm["rollout_ms"] > 0 else None
    traffic = None
    kern = dev.rollout_kernel()  # "tc1" (rollout_tc.cu), "tc2" (rollout_tc2.cu) or "simt" (rollout.cu)
    info = dev.rollout_info()
    # DRAM bytes per launch from the committed ncu --set full capture of this kernel on this workload
    tp = os.path.join(ROOT, "profiles", {"tc1": "rollout_tc_ncu_summary.json", "simt": "rollout_ncu_summary.json",
                                         "tc2": f"rollout_tc2_{args.config}_ncu_summary.json"}[kern])
    if os.path.exists(tp) and (kern == "tc2" or args.config == "c2"):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    kname = {"tc1": "rollout_tc_kernel (K1 v1, rollout_tc.cu: tcgen05 kind::tf32, 3xTF32, one 128-row tile per CTA)",
             "tc2": f"rollout_tc2_kernel<{info['tiles_per_cta']},{256 if info['tiles_per_cta'] == 1 and max(wl.spec.widths) > 128 else 128}> "
                    "(K1 v2, rollout_tc2.cu: tcgen05 kind::tf32, 3xTF32, in-place TMEM regions)",
             "simt": "rollout_kernel (K1, rollout.cu: SIMT FFMA)"}[kern]
    if path == "tcgen05":
        # 3xTF32: three dense kind::tf32 MMAs per FP32 product, so the ceiling for the
        # algorithmic (FP32) FLOP rate is the TF32 tensor peak / 3.
        roof = {"bound": "tensor", "achieved": achieved, "peak": TF32_DENSE_TFLOPS / 3.0, "unit": "TFLOP/s",
                "kernel": kname,
                "peak_source": "B200_PROFILING.md fallback: dense TF32 1100 TFLOP/s (MEASURED_PEAKS.json has no TF32 "
                               "entry) / 3 MMAs per FP32 product",
                "peak_measured_live": (peak_tf32 / 3.0) if peak_tf32 else None,
                "tensor_tflops_executed": 3.0 * achieved if achieved else None}
    else:
        roof = {"bound": "fp32", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
                "kernel": kname,
                "peak_source": "bp_measure_fp32_peak: FFMA microbenchmark run live in this process "
                               "(MEASURED_PEAKS.json has no FP32 SIMT entry)"}
    roof["frac"] = (roof["achieved"] / roof["peak"]) if (roof["achieved"] and roof["peak"]) else None
    roof["traffic"] = traffic
    roof.update({"flop_per_sample_step": wl.flops_per_sample_step, "rollout_ms": tm["rollout_ms"],
                 "rollout_launches": tm["rollout_launches"]})

    e2e = None
    if not args.no_e2e:
        # end to end through the public API: objective upload, plan() from the root for the same number
        # of iterations, host buffers in and the result dict out, wall clock around the whole call.
        dev2 = bp.Device(local)
        parallel.attach(dev2)
        cfg2 = wl.planner_config()
        cfg2["batch"] = cfg2["batch"] * world
        n_it = setup + args.warmup + args.steps
        cfg2["termination"]["max_iterations"] = n_it
        bp.Device.io_bytes()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev2.load(wl.spec)
        res = dev2.plan(cfg2)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        h2d, d2h = bp.Device.io_bytes()
        # every searched box (root and children) evaluates rows x iters samples
        bounded = res["samples"] / (rows * iters)
        e2e = {"value": bounded / wall, "unit": "subdomains/s", "h2d_bytes_per_step": int(h2d / max(1, n_it)),
               "d2h_bytes_per_step": int(d2h / max(1, n_it)), "iterations": n_it,
               "note": "plan() from the root incl. ramp-up iterations with fewer children; objective upload inside"}
        dev2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as orc
            n = max(8, orc.thread_count())
            rate, times, cores = cpu_children_per_s(wl, n, steps=1)
            cpu = {"value": rate, "unit": "subdomains/s", "cores": cores, "kind": "port",
                   "sample": f"{n} pre-split {wl.name} boxes: batch_search (CEM M={wl.samples_per_iter}, "
                             f"{iters} iters) + early-stop-empirical CROWN in the FP64 oracle, {times[0]:.1f} s"}
        except Exception as e:  # the checker is optional on the box
            cpu = {"value": None, "unit": "subdomains/s", "cores": None, "kind": "port", "sample": f"unavailable: {e}"}

    if rank == 0:
        clk = clocks.summary()
        line = {
            "metric": "subdomains_bounded_per_s", "value": value, "unit": "subdomains/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32" if path == "simt" else "tf32x3",
            "data": "synthetic (seeded He-init weights, x0/goal/obstacles from the reference Rng)",
            "config": {"workload": f"{wl.name} (BASELINE.json configs[1])", "widths": wl.spec.widths,
                       "H": H, "M": wl.samples_per_iter, "D_per_step": children / args.steps, "D_per_gpu": children / args.steps / world,
                       "cem_iterations": iters, "batch": batch, "setup_iterations": setup,
                       "l2": "flushed (256 MB write) between timed steps", "parallelism": f"subdomain-sharded x{world}" if world > 1 else "1 GPU"},
            "sample_steps_per_s": sample_steps,
            "roofline": roof,
            "e2e": e2e, "gpu_launches": int(tm["launches"]), "clocks": clk, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
