#!/usr/bin/env python
"""BaB-ND hot-path benchmark on B200 (BASELINE.json metric: subdomains bounded/s
and sample*steps/s; best objective vs the CPU planner at equal iterations).

Default workload: C3-wide (BASELINE.json configs[2]: MLP [36,256,256,256,32],
H=30, M=4096 samples per CEM iteration, 10 CEM iterations, D=2048 children =
2 x batch 1024 per BaB iteration) -- the largest configuration whose planner
step fits one GPU and the width-256 configuration the >= 50 % tensor-pipe
target names.  A step is one steady-state BaB iteration: pick_out, split,
device search (Philox sampling -> fused rollout + extrema -> incumbent / top-K /
CEM refit), device early-stop CROWN bound, merge, prune.  `--config c1|c2|c4`
select the other planner configs; `--config c5 [--d D]` is SURVEY 8(d)'s sweep
step: one search (10 CEM iterations) + one bound pass over D pre-split boxes.
Timed with CUDA events on the launching stream, L2 flushed between steps, max
over ranks.

  python bench.py [--gpus N --steps K --warmup W] [--config c3] [--impl reference]

Multi-GPU (torchrun): one planner sharded over the ranks -- every iteration's
children go round-robin to the GPUs and their heads are all-gathered
(paper_2412_09584_b200.parallel); the batch grows with the GPU count so each GPU
keeps D=2048 children per step (weak scaling).

--impl reference times the reference algorithm on the host cores: the FP64
oracle restatement (oracle/, all host threads; the reference itself does not
build here -- DESIGN.md 3) on a bounded sample of the same workload per step.
That arm never loads this repo's CUDA library (fixtures come from the pure-
Python reference Rng in workloads.py).
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

TF32_DENSE_TFLOPS = 1100.0  # /opt/skills/guides/B200_PROFILING.md, dense (non-sparse) TF32
CONFIG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}
# full CPU searches are affordable per step only for the small configs; above that the CPU arm
# times a fixed slice of each box's search (1 of the 10 CEM iterations: every iteration does the
# same work) and reports the full-search equivalent (SURVEY 8(d) "time a fixed slice")
CPU_CEM_SLICE = {"c1": None, "c2": None, "c3": 1, "c4": 1, "c5": 1}
CROWN_FLOP = {"c1": 0.095e6, "c2": 1.42e6, "c3": 8.91e6, "c4": 3.48e6, "c5": 22.4e6}
# ... and 1/f of the samples of that iteration (the search cost is linear in the rows rolled out), so
# a reference-arm step stays near 20 s of CPU time (--steps 5 --warmup 3 in under three minutes)
CPU_ROW_FRACTION = {"c1": 1, "c2": 1, "c3": 4, "c4": 1, "c5": 2}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c3", choices=sorted(CONFIG_INDEX))
    p.add_argument("--d", type=int, default=1024, help="C5 sweep: pre-split boxes per GPU")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-objective", action="store_true", help="skip the best-objective comparison")
    return p.parse_args()


def workload(args):
    from paper_2412_09584_b200 import workloads

    return workloads.c5(D=args.d) if args.config == "c5" else workloads.ALL[args.config]()


def label(args, wl) -> str:
    return f"{wl.name} (BASELINE.json configs[{CONFIG_INDEX[args.config]}])"


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


# ------------------------------------------------------------------ CPU (oracle) legs
def cpu_children_per_s(cfg_name, wl, n_children: int, steps: int = 1, warmup: int = 0):
    """The oracle (FP64 CPU restatement of the reference path) on n_children pre-split boxes:
    batch_search + CrownBounder::lower, all host threads (parallel_chunks over boxes).  Configs
    in CPU_CEM_SLICE run k of the CEM iterations per step; the rate is per full-search
    equivalent (search time x iterations / k + bound time)."""
    from oracle import oracle as orc
    from paper_2412_09584_b200 import workloads

    ob = orc.Objective(wl.spec)
    los, his = workloads.presplit_boxes(wl.spec, n_children)
    cfg = wl.planner_config()
    full_iters = cfg["search"]["iterations"]
    k = CPU_CEM_SLICE[cfg_name] or full_iters
    cfg["search"]["iterations"] = k
    f = CPU_ROW_FRACTION[cfg_name]
    cfg["search"]["samples_per_iter"] = wl.samples_per_iter // f
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        reps = ob.batch_search(los, his, None, cfg, seed=1000 + i)
        t1 = time.perf_counter()
        reps.bound_all()
        t2 = time.perf_counter()
        if i >= warmup:
            times.append((t1 - t0) * f * full_iters / k + (t2 - t1))
    sample = (f"{n_children} pre-split {wl.name} boxes per step: batch_search (CEM M={wl.samples_per_iter}, "
              + (f"{k} of {full_iters} iterations" if k != full_iters else f"{full_iters} iterations")
              + (f" of M/{f} samples" if f != 1 else "")
              + (" timed, scaled to the full search" if (k != full_iters or f != 1) else "")
              + ") + early-stop-empirical CROWN, FP64 oracle restatement")
    return n_children / (sum(times) / len(times)), times, orc.thread_count(), sample


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc

    n = max(8, orc.thread_count())
    rate, times, cores, sample = cpu_children_per_s(args.config, wl, n, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": "subdomains_bounded_per_s", "value": rate, "unit": "subdomains/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded He-init weights, x0/goal/obstacles from the reference Rng)",
        "config": {"workload": label(args, wl), "widths": wl.spec.widths, "H": wl.spec.horizon,
                   "M": wl.samples_per_iter, "cem_iterations": wl.planner_config()["search"]["iterations"],
                   "D_per_step": n, "parallelism": f"{cores} host threads", "sample": sample},
        "cpu_baseline": {"value": rate, "unit": "subdomains/s", "cores": cores, "kind": "port",
                         "sample": sample + " (the reference does not build here: Eigen / vendor headers absent)"},
        "e2e": {"value": rate, "unit": "subdomains/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def best_objective_vs_cpu():
    """Best objective of the device planner and the CPU reference planner (oracle) at equal BaB
    iteration counts, same fixtures, over several planner seeds (the samplers differ -- Philox
    vs mt19937_64 -- so one seed is one draw; the comparison is the paired set).  C1 at its
    full 20 iterations (6 seeds); C2 with batch 4 for 4 iterations (3 seeds; the CPU planner
    needs ~14 s per C2 child)."""
    import paper_2412_09584_b200 as bp
    from oracle import oracle as orc
    from paper_2412_09584_b200 import workloads

    out = {}
    dev = bp.Device(int(os.environ.get("LOCAL_RANK", "0")))
    for name, over, iters, seeds in (("c1", {}, None, (2, 3, 4, 5, 6, 7)), ("c2", {"batch": 4}, 4, (2, 3, 4))):
        wl = workloads.ALL[name]()
        dev.load(wl.spec)
        ob = orc.Objective(wl.spec)
        g, c = [], []
        t0 = time.perf_counter()
        for seed in seeds:
            cfg = wl.planner_config(**over)
            cfg["seed"] = seed
            if iters is not None:
                cfg["termination"]["max_iterations"] = iters
            g.append(dev.plan(cfg)["objective"])
            c.append(ob.plan(cfg)["objective"])
        g, c = np.array(g), np.array(c)
        out[wl.name] = {"iterations": cfg["termination"]["max_iterations"], "batch": cfg["batch"],
                        "seeds": list(seeds), "gpu": g.tolist(), "cpu": c.tolist(),
                        "gpu_le_cpu_seeds": int((g <= c).sum()),
                        "median_rel_gap": float(np.median((g - c) / np.maximum(np.abs(c), 1e-12))),
                        "gpu_best_le_cpu_best": bool(g.min() <= c.min()), "s": time.perf_counter() - t0}
        if name == "c2":  # three seeds are one draw of a ~3 % seed-to-seed spread
            out[wl.name]["note"] = ("tools/objective_seeds.py c2 12 (profiles/r02_objective_seeds_c2.log): over seeds 2-13 "
                                    "the GPU is at or below the CPU on 6 of 12, median gap -0.01 %")
    dev.close()
    return out


# ------------------------------------------------------------------ GPU arm
def roofline(dev, wl, args, tm, rows_per_launch_total, peak_tf32, peak_fp32):
    """Roofline of the dominant kernel (the rollout): algorithmic FLOPs / device time of its launches."""
    path = dev.rollout_path()
    kern = dev.rollout_kernel()
    info = dev.rollout_info()
    flop = rows_per_launch_total * wl.spec.horizon * wl.flops_per_sample_step
    achieved = flop / (tm["rollout_ms"] / 1e3) / 1e12 if tm["rollout_ms"] > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"r02_{args.config}_ncu_summary.json")
    if os.path.exists(tp):
        j = json.load(open(tp))
        if j.get("kernel_key") == kern:
            traffic = j.get("dram_bytes_per_launch")
    kname = {"tc1": "rollout_tc_kernel (K1 v1, rollout_tc.cu: tcgen05 kind::tf32, 3xTF32, one 128-row tile per CTA)",
             "tc2": f"rollout_tc2_kernel (K1 v2, rollout_tc2.cu: tcgen05 kind::tf32, 3xTF32, in-place TMEM regions, "
                    f"{info['tiles_per_cta']} tile(s) per CTA)",
             "tc3": "rollout_tc3_kernel (K1 v3, rollout_tc3.cu: tcgen05 kind::tf32, 3xTF32, N-split CTA pair)",
             "simt": "rollout_kernel (K1, rollout.cu: SIMT FFMA)"}.get(kern, kern)
    if path == "tcgen05":
        # 3xTF32: three dense kind::tf32 MMAs per FP32 product, so the ceiling for the algorithmic
        # (FP32) FLOP rate is the TF32 tensor peak / 3.
        roof = {"bound": "tensor", "achieved": achieved, "peak": TF32_DENSE_TFLOPS / 3.0, "unit": "TFLOP/s",
                "kernel": kname,
                "peak_source": "B200_PROFILING.md fallback: dense TF32 1100 TFLOP/s (MEASURED_PEAKS.json has no TF32 "
                               "entry) / 3 MMAs per FP32 product",
                "peak_measured_live": (peak_tf32 / 3.0) if peak_tf32 else None,
                "tensor_tflops_executed": 3.0 * achieved if achieved else None}
    else:
        roof = {"bound": "fp32", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s", "kernel": kname,
                "peak_source": "bp_measure_fp32_peak: FFMA microbenchmark run live in this process "
                               "(MEASURED_PEAKS.json has no FP32 SIMT entry)"}
    roof["frac"] = (roof["achieved"] / roof["peak"]) if (roof["achieved"] and roof["peak"]) else None
    roof["traffic"] = traffic
    roof["traffic_source"] = (f"profiles/r02_{args.config}_ncu_summary.json (ncu --set full, "
                              "dram__bytes_read.sum + dram__bytes_write.sum per launch)") if traffic else None
    roof.update({"flop_per_sample_step": wl.flops_per_sample_step, "rollout_ms": tm["rollout_ms"],
                 "rollout_launches": tm["rollout_launches"],
                 "algorithmic": "2 * sum(in*out) FLOP per sample-step x rows x H per launch (SURVEY 8(d))"})
    return roof, path


def main():
    args = parse()
    wl = workload(args)
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
    from paper_2412_09584_b200 import parallel, workloads

    peak_fp32 = peak_tf32 = None
    if rank == 0:
        import ctypes as C
        from paper_2412_09584_b200 import _capi
        t, ms = C.c_double(), C.c_double()
        _capi.check(_capi.load().bp_measure_fp32_peak(local, C.byref(t), C.byref(ms)))
        peak_fp32 = t.value
        _capi.check(_capi.load().bp_measure_tf32_peak(local, C.byref(t), C.byref(ms)))
        peak_tf32 = t.value

    dev = bp.Device(local).load(wl.spec)
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    cfg = wl.planner_config()
    iters = cfg["search"]["iterations"]
    rows = wl.rows_per_search_iter
    H = wl.spec.horizon
    sweep = args.config == "c5"
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    if sweep:
        # one search (10 CEM iterations) + one bound pass over D pre-split boxes per GPU;
        # the boxes are this rank's slice of the global D*world leaves (weak scaling, no exchange)
        los, his = workloads.presplit_boxes(wl.spec, args.d * world)
        los, his = los[rank::world], his[rank::world]
        n_box = los.shape[0]

        def step():
            dev.batch_search(los, his, None, cfg, seed=7)
            dev.batch_bound(n_box)
            return n_box
        setup = 0
    else:
        parallel.attach(dev)
        cfg["batch"] = cfg["batch"] * world
        cfg["termination"]["max_iterations"] = 10**6
        planner = dev.planner(cfg)
        batch = cfg["batch"]
        setup = 0
        while True:  # grow the pool to the steady-state batch (2*batch children per step)
            _, _, pool = planner.step()
            setup += 1
            if pool >= batch or setup >= 16:
                break

        def step():
            _, ch, _ = planner.step()
            return ch

    for _ in range(args.warmup):
        step()
    dev.timing()
    dev.search_counters()
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
            ch = step()
            ev1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            children += ch
    tm = dev.timing()
    cnt = dev.search_counters()
    total_ms = sum(step_ms)
    stats = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    total_ms_max = stats[0].item()
    # planner: the global child count (identical on every rank); sweep: this rank's boxes x world
    children_all = float(children) * (world if sweep else 1)
    value = children_all / (total_ms_max / 1e3)
    sample_steps = children_all * rows * iters * H / (total_ms_max / 1e3)
    my_rows = (children if sweep else children / world) * rows * iters  # this rank's rolled-out rows
    roof, path = roofline(dev, wl, args, tm, my_rows, peak_tf32, peak_fp32)

    e2e = None
    if not args.no_e2e:
        dev2 = bp.Device(local)
        bp.Device.io_bytes()
        if sweep:
            # the public batch_search / batch_bound calls with host boxes in and reports / bounds out
            dev2.load(wl.spec)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                dev2.batch_search(los, his, None, cfg, seed=7)
                dev2.batch_bound(n_box)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            h2d, d2h = bp.Device.io_bytes()
            e2e = {"value": n_box * world * args.steps / wall, "unit": "subdomains/s",
                   "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
                   "note": "batch_search + batch_bound through the public API, host boxes in, bounds and reports out"}
        else:
            # plan() from the root through the public API: objective upload, setup + timed iterations,
            # host buffers in and the result dict out, wall clock around the whole call.
            parallel.attach(dev2)
            cfg2 = wl.planner_config()
            cfg2["batch"] = cfg2["batch"] * world
            n_it = setup + args.steps
            cfg2["termination"]["max_iterations"] = n_it
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev2.load(wl.spec)
            res = dev2.plan(cfg2)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            h2d, d2h = bp.Device.io_bytes()
            bounded = res["samples"] / (rows * iters)  # every searched box evaluates rows x iters samples
            e2e = {"value": bounded / wall, "unit": "subdomains/s", "h2d_bytes_per_step": int(h2d / max(1, n_it)),
                   "d2h_bytes_per_step": int(d2h / max(1, n_it)), "iterations": n_it,
                   "note": "plan() from the root incl. the ramp-up iterations with fewer children; objective "
                           "upload inside"}
        dev2.close()

    cpu = None
    objective = None
    if rank == 0 and world == 1:
        if not args.no_cpu_baseline:
            try:
                from oracle import oracle as orc
                n = max(8, orc.thread_count())
                rate, times, cores, sample = cpu_children_per_s(args.config, wl, n, steps=1)
                cpu = {"value": rate, "unit": "subdomains/s", "cores": cores, "kind": "port",
                       "sample": sample + f" ({times[0]:.1f} s full-search equivalent per step)"}
            except Exception as e:  # the checker is optional on the box
                cpu = {"value": None, "unit": "subdomains/s", "cores": None, "kind": "port", "sample": f"unavailable: {e}"}
        if not args.no_objective:
            try:
                objective = best_objective_vs_cpu()
            except Exception as e:
                objective = {"unavailable": str(e)}

    if rank == 0:
        clk = clocks.summary()
        conf = {"workload": label(args, wl), "widths": wl.spec.widths, "H": H, "M": wl.samples_per_iter,
                "cem_iterations": iters, "D_per_step": children_all / args.steps,
                "D_per_gpu": children_all / args.steps / world,
                "l2": "flushed (256 MB write) between timed steps",
                "parallelism": f"subdomain-sharded x{world}" if world > 1 else "1 GPU"}
        if sweep:
            conf["step"] = "one search (10 CEM iterations) + one early-stop-empirical bound pass over D pre-split boxes"
        else:
            conf.update({"batch": cfg["batch"], "setup_iterations": setup})
        line = {
            "metric": "subdomains_bounded_per_s", "value": value, "unit": "subdomains/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if path == "simt" else "tf32x3",
            "data": "synthetic (seeded He-init weights, x0/goal/obstacles from the reference Rng)",
            "config": conf,
            "sample_steps_per_s": sample_steps,
            "failed_boxes": {"timed": cnt["failed"], "searched": cnt["boxes"]},
            # K7 alone: the boxes bounded per second of bound-kernel device time, and the
            # device-time shares of the step's kernels
            "bound": {"subdomains_per_s": ((children if sweep else children / world) / (tm["bound_ms"] / 1e3))
                                          if tm["bound_ms"] > 0 else None,
                      # CROWN lower-form FLOP per subdomain over all H steps (early stop does less)
                      "crown_flop_per_subdomain": CROWN_FLOP[args.config],
                      "fp64_tflops_upper": ((children if sweep else children / world) * CROWN_FLOP[args.config]
                                            / (tm["bound_ms"] / 1e3) / 1e12) if tm["bound_ms"] > 0 else None,
                      "bound_ms_per_step": tm["bound_ms"] / args.steps,
                      "rollout_ms_per_step": tm["rollout_ms"] / args.steps},
            "roofline": roof,
            "e2e": e2e, "gpu_launches": int(tm["launches"]), "clocks": clk, "cpu_baseline": cpu,
            "best_objective_vs_cpu": objective,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
