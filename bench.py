#!/usr/bin/env python
"""Benchmark of the B200 Stripe block executor (BASELINE.json contract).

Default workload (N=1): BASELINE config 5 -- the ResNet-50-shaped Stripe program
(paper_1903_06498_b200.workloads.resnet50: 53 convs, max-pool, residuals, global sum, fc) at
its named global batch of 1024 images, i8 x i8 -> i32 with i8 activations (the reference's
integer semantics; bit-exact vs its interpreter).  With N GPUs the batch index is sharded
1024/N images per rank (strong scaling, no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c2|c3|c4a|c4b|c1|c1_i32]
    python bench.py --impl reference ...   (the reference interpreter on the host cores)

--gpus N starts N ranks itself (torch.distributed.run, NCCL only for the barrier and the
max-over-ranks time) unless it already runs under a launcher (WORLD_SIZE set).

A step = prepare_outputs + execute of the config's program over one batch.
value  : useful GFLOP/s (2 x constraint-satisfying MAC points, tile.cpp:338-370) or, for the
         memory-bound configs C4a/C4b, algorithmic GB/s; inputs resident in HBM, K steps
         replayed as one CUDA graph, CUDA events on the launching stream, max over ranks.
e2e    : the same metric through the public API from HOST buffers, host<->device copies
         inside the timed region: `value` = sb_execute_async with native-width pinned buffers
         (two contexts ping-ponging), `dropin` = sb_execute with int64 carriers (the
         stripe::b200::execute boundary, synchronous, int64<->native conversion included).
roofline: the dominant kernel family, from a per-step CUDA-event pass (sb_context_set_profile)
         after the timed region; `network` = whole step against the same peak.
cpu_baseline: the unmodified reference interpreter (oracle/_ref) on 1 and P host threads over
         a bounded sample of the same workload (rank 0, N=1 only).
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Stripe-kernel GFLOP/s & GB/s vs B200 roofline at 1/2/4/8 GPU; x vs CPU ref"
L2_BYTES = 126 * 1024 * 1024
ISZ = {8: 1, 16: 2, 32: 4, 0x20F: 4}


# ------------------------------------------------------------------------------------------
def peaks():
    """HBM and dense tensor peaks: MEASURED_PEAKS.json (driver) + profiles/r02_peaks.json
    (int8 / tf32 dense measured on this pool's B200 by tools/measure_peaks.py)."""
    out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "kind": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        out.update(hbm_gbs=float(p["hbm_gbs"]), bf16_tflops=float(p["bf16_tflops"]), kind="measured")
    except Exception:
        pass
    out["int8_tops"], out["int8_kind"] = 2 * out["bf16_tflops"], "derived: 2 x bf16"
    try:
        with open(os.path.join(ROOT, "profiles", "r02_peaks.json")) as f:
            q = json.load(f)
        out["int8_tops"], out["int8_kind"] = float(q["int8_tops"]), f"measured ({q['int8_how']})"
    except Exception:
        pass
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def wait_first_sample(self, timeout=3.0):
        t0 = time.time()
        while self.proc and time.time() - t0 < timeout:
            if os.path.getsize(self.path) > 0:
                return
            time.sleep(0.02)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    sm.append(float(f[1]))
                    smax.append(float(f[2]))
                except ValueError:
                    continue
                for n, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            os.unlink(self.path)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ------------------------------------------------------------------------------------------
# Config specs.  Everything a rank needs: its program text, useful work, algorithmic bytes,
# which roofline bounds it, and the CPU-reference sample.
def spec(cfg, world, rank, args):
    from paper_1903_06498_b200 import workloads as Wk
    s = {"cfg": cfg, "scaling": "weak"}
    if cfg == "c5":
        total = args.batch or 1024
        lo, hi = Wk.shard_range(total, world, rank)
        n = hi - lo
        text, info = Wk.resnet50(n)
        conv_flops = 2.0 * sum(c["macs"] for c in info["convs"])
        s.update(text=text, flops=float(info["flops"]), unit="GFLOP/s", bound="tensor", scaling="strong",
                 global_batch=total, images=n, dominant=("conv_igemm_tc", "conv_i8_tc", "gemm_i8_tc"),
                 dominant_flops=float(info["flops"]), conv_flops=conv_flops, nsets=2,
                 workload=f"BASELINE config 5: ResNet-50 Stripe program (53 convs, max-pool, residuals, global sum, fc), "
                          f"global batch {total} sharded on n ({n} images on this rank)",
                 cpu=dict(text=Wk.resnet50(1, image=32)[0], work=float(Wk.resnet50(1, image=32)[1]["flops"]),
                          what="ResNet-50 program at 32x32, batch 1 per thread (same layer mix, 1/49 of the "
                               "spatial work): rate EXTRAPOLATED to the 224x224 config", seed=1005))
    elif cfg == "c2":
        n = args.batch or 32
        text = Wk.conv2d(n, 56, 56, 64, 64)
        s.update(text=text, flops=2.0 * Wk.conv_useful_macs(n, 56, 56, 64, 64), unit="GFLOP/s", bound="hbm",
                 global_batch=n * world, images=n, dominant=("conv_i8_tc", "conv_igemm_tc"),
                 workload=f"BASELINE config 2: conv2d 3x3 NHWC 56x56x64->64, batch {n} per GPU, padding "
                          f"constraints, one Stripe block (i8 x i8 -> i32)",
                 cpu=dict(text=Wk.conv2d(1, 56, 56, 64, 64), work=2.0 * Wk.conv_useful_macs(1, 56, 56, 64, 64),
                          what="one image of config 2 per thread (a batch shard)", seed=1001))
    elif cfg == "c3":
        n = args.batch or 128
        # the program the reference's own passes produce (tests/golden/make_pipeline_programs.py)
        piped = os.path.join(ROOT, "configs", f"c3_pipeline_b{n}.stripe")
        text = open(piped).read() if os.path.exists(piped) else Wk.conv_bias_relu(n, 56, 56, 64, 64)
        s.update(text=text, flops=2.0 * Wk.conv_useful_macs(n, 56, 56, 64, 64),
                 unit="GFLOP/s", bound="hbm", global_batch=n * world, images=n, dominant=("conv_i8_tc", "conv_igemm_tc"),
                 workload=f"BASELINE config 3: fused conv3x3+bias+ReLU produced by the reference's "
                          f"tile_rewrite/fuse/localize/scalarize passes ({os.path.basename(piped) if os.path.exists(piped) else 'hand-built equivalent'}), "
                          f"56x56x64->64, batch {n} per GPU",
                 cpu=dict(text=Wk.conv_bias_relu(1, 56, 56, 64, 64),
                          work=2.0 * Wk.conv_useful_macs(1, 56, 56, 64, 64),
                          what="one image of config 3 per thread (a batch shard)", seed=1003))
    elif cfg == "c4a":
        n = args.batch or 128
        s.update(text=Wk.maxpool2x2(n, 112, 112, 64), flops=0.0, unit="GB/s", bound="hbm", global_batch=n * world,
                 images=n, dominant=("reduce", "pool"),
                 workload=f"BASELINE config 4a: 2x2 max-pool 112x112x64 i32, batch {n} per GPU",
                 cpu=dict(text=Wk.maxpool2x2(8, 112, 112, 64), work=8 * (112 * 112 * 64 + 56 * 56 * 64) * 4.0,
                          what="8 images of config 4a per thread (a batch shard)", seed=1004))
    elif cfg == "c4b":
        n = args.batch or 1024
        s.update(text=Wk.global_sum(n, 7, 7, 2048), flops=0.0, unit="GB/s", bound="hbm", global_batch=n * world,
                 images=n, dominant=("reduce",),
                 workload=f"BASELINE config 4b: global sum 7x7x2048 i32, batch {n} per GPU",
                 cpu=dict(text=Wk.global_sum(64, 7, 7, 2048), work=64 * (49 * 2048 + 2048) * 4.0,
                          what="64 images of config 4b per thread (a batch shard)", seed=1004))
    elif cfg in ("c1", "c1_i32"):
        dt = "i8" if cfg == "c1" else "i32"
        M = 1024
        lo, hi = Wk.shard_range(M, world, rank)
        m = hi - lo
        if world == 1:
            # "as one autotiled Stripe block": the reference's tile_rewrite of the shape the device
            # autotile search chose (configs/c1_autotile.json, tests/golden/make_pipeline_programs.py)
            with open(os.path.join(ROOT, "configs", f"c1_autotiled_{dt}.stripe")) as f:
                text = f.read()
            with open(os.path.join(ROOT, "configs", "c1_autotile.json")) as f:
                shape = json.load(f)[dt]["chosen"]
            what = f"one block autotiled on the B200 to {shape} (1331 candidates), rewritten by the reference's tile_rewrite"
        else:
            text = Wk.matmul(m, 1024, 1024, in_dtype=dt, out_dtype="i32")
            what = f"rows sharded ({m} on this rank)"
        s.update(text=text, flops=2.0 * m * 1024 * 1024,
                 unit="GFLOP/s", bound="tensor", scaling="strong", global_batch=M, images=m,
                 dominant=("gemm_i8_tc",),
                 workload=f"BASELINE config 1: matmul C[i,j] += A[i,k]*B[k,j] 1024^3 ({dt} x {dt} -> i32, exact), "
                          f"{what}",
                 cpu=dict(text=Wk.matmul(64, 1024, 1024, in_dtype=dt, out_dtype="i32"), work=2.0 * 64 * 1024 * 1024,
                          what="64 rows of config 1 per thread (a row shard; 16 threads = the whole matmul)",
                          seed=1001))
    else:
        raise SystemExit(f"unknown config {cfg}")
    return s


def alg_bytes_of(prog):
    """Algorithmic bytes: every root buffer once at native width (inputs read, outputs written)."""
    return sum(d.elements * ISZ[d.dtype] for d in prog.buffers.values())


# ------------------------------------------------------------------------------------------
def cpu_reference(sp, threads_list, steps=1):
    """The unmodified reference interpreter (oracle/_ref: stripe::execute) on host threads.
    Returns [{threads, rate, seconds}] -- each thread runs its own Program/BufferStore on one
    unit of the config's work (a batch or row shard), all threads at once."""
    import numpy as np

    from oracle import Ref, random_inputs
    L = Ref.lib()
    c = sp["cpu"]
    prog = Ref.parse(c["text"])
    bufs = prog.buffers()
    inputs = random_inputs(bufs, c["seed"])
    res = []
    for threads in threads_list:
        times = []
        for _ in range(steps):
            progs = (ctypes.c_void_p * threads)(*([prog.h] * threads))
            stores = []
            for t in range(threads):
                s = L.sr_store_new()
                for n, bits, el, d in bufs:
                    arr = inputs[n] if n in inputs else np.zeros(el, np.int64)
                    L.sr_store_set(s, n.encode(), bits, arr.ctypes.data, arr.size)
                stores.append(s)
            st = (ctypes.c_void_p * threads)(*stores)
            t0 = time.perf_counter()
            bad = L.sr_execute_many(progs, st, threads, threads)
            dt = time.perf_counter() - t0
            for s in stores:
                L.sr_store_free(s)
            if bad:
                raise RuntimeError("reference execute failed")
            times.append(dt)
        sec = statistics.mean(times)
        res.append({"threads": threads, "rate": c["work"] * threads / sec / 1e9, "seconds": round(sec, 3)})
    return res


def host_cpu():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


def cpu_baseline_obj(sp, steps=1):
    from oracle import Ref
    if not Ref.available():
        return None
    model, ncpu = host_cpu()
    r = cpu_reference(sp, [1, ncpu], steps)
    one, many = r[0], r[-1]
    return {"value": round(many["rate"], 4), "unit": sp["unit"], "cores": ncpu, "kind": "reference",
            "sample": f"{sp['cpu']['what']}; unmodified stripe::execute from oracle/_ref (-O2), one "
                      f"Program/BufferStore per thread; {ncpu} threads {many['seconds']} s",
            "one_thread": round(one["rate"], 5), "one_thread_seconds": one["seconds"],
            "threads": ncpu, "cpu_model": model}


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import Ref
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libstripe_ref.so not built"}))
        return
    sp = spec(args.config, 1, 0, args)
    model, ncpu = host_cpu()
    t0 = time.perf_counter()
    r = cpu_reference(sp, [ncpu], steps=args.steps if args.steps <= 3 else 3)[0]
    wall = time.perf_counter() - t0
    v = round(r["rate"], 4)
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": sp["unit"], "impl": "reference", "n_gpus": args.gpus,
        "steps": min(args.steps, 3), "warmup": 0, "ms_per_step": round(1000 * r["seconds"], 3),
        "higher_is_better": True, "scaling": sp["scaling"], "vs_baseline": None,
        "dtype": "int64 carriers (i8/i32 program dtypes)", "data": f"synthetic (splitmix64 random_inputs, seed "
                                                                  f"{sp['cpu']['seed']})",
        "config": {"workload": sp["workload"], "sample": sp["cpu"]["what"]},
        "cpu_baseline": {"value": v, "unit": sp["unit"], "cores": ncpu, "kind": "reference",
                         "sample": f"{sp['cpu']['what']}; {ncpu} host threads, one stripe::execute each",
                         "cpu_model": model, "wall_s": round(wall, 2)},
        "e2e": {"value": v, "unit": sp["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1903_06498_b200 as sb

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    sp = spec(args.config, world, rank, args)
    prog = sb.parse_program(sp["text"])
    ctx = sb.Context(local)
    ctx.set_stream(stream.cuda_stream)
    pk = peaks()
    alg_bytes = alg_bytes_of(prog)
    in_names = [n for n, d in prog.buffers.items() if int(d.dir) == 0]
    out_names = [n for n in prog.buffers if n not in in_names]
    nbytes = {n: d.elements * ISZ[d.dtype] for n, d in prog.buffers.items()}
    # rotate through enough input/output sets that the working set exceeds L2 (C5: each step's
    # > 1 GB of activations flushes L2 anyway)
    nsets = sp.get("nsets") or max(2, int(3 * L2_BYTES // max(alg_bytes, 1)) + 1)
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    sets = []
    for _ in range(nsets):
        bufs, keep = {}, []
        for n, d in prog.buffers.items():
            t = torch.randint(-128, 128, (nbytes[n],), dtype=torch.int8, device=dev, generator=g)
            keep.append(t)
            bufs[n] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
        sets.append((bufs, keep))
    bound = [ctx.bind_device(prog, b) for b, _ in sets]

    def step(i):
        bound[i % nsets]()

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        clk = ClockSampler(local).__enter__()
        clk.wait_first_sample()
        for i in range(args.warmup):
            step(i)
        # keep the GPU busy ~1 s before the timed region so the sampled clocks reflect load
        settle, t_settle = 0, time.perf_counter()
        while time.perf_counter() - t_settle < 1.0:
            for _ in range(max(1, 2000 // max(1, int(sp["flops"] / 1e9) + 1))):
                step(args.warmup + settle)
                settle += 1
            torch.cuda.synchronize(dev)
        ctx.sync()
        # the timed region: exactly K steps captured once as a CUDA graph (sb_graph_*) so host
        # launch latency is off the device timeline
        graph = sb.Graph(ctx, lambda: [step(args.warmup + i) for i in range(args.steps)])
        graph.launch()  # warm the graph itself (untimed)
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        launches0 = ctx.launch_count
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        graph.launch()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        clk.__exit__(None, None, None)
        ctx.sync()
        barrier()
        torch.cuda.synchronize(dev)
        launches = ctx.launch_count - launches0
        elapsed_ms = t_start.elapsed_time(t_end)

        # isolated launches: one step at a time, synchronized on both sides (no overlap with a
        # neighbouring step), median of 10
        iso = []
        for i in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            a.record(stream)
            step(i)
            b.record(stream)
            torch.cuda.synchronize(dev)
            iso.append(a.elapsed_time(b))
        iso_ms = statistics.median(iso)
        # per-step device times (serial, CUDA events around every launch) for the roofline
        ctx.set_profile(True)
        prof = []
        for i in range(3):
            step(i)
            ctx.sync()
            prof.append(ctx.read_profile())
        ctx.set_profile(False)

    t = torch.tensor([elapsed_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    work = sp["flops"] if sp["unit"] == "GFLOP/s" else float(alg_bytes)
    value = work * world * args.steps / (elapsed_ms / 1e3) / 1e9 if sp["scaling"] == "weak" else \
        sum_over_ranks(dist, world, dev, work) * args.steps / (elapsed_ms / 1e3) / 1e9

    # ---- roofline of the dominant kernel family (median over the profiled executes) ----
    fam = {}
    for rec in prof:
        per = {}
        for (_, ms, kern, _, _) in rec:
            per[kern] = per.get(kern, 0.0) + ms
        for k, v in per.items():
            fam.setdefault(k, []).append(v)
    fam_ms = {k: statistics.median(v) for k, v in fam.items()}
    prof_total = sum(fam_ms.values())
    dom = [k for k in sp["dominant"] if k in fam_ms]
    dom_ms = sum(fam_ms[k] for k in dom)
    dom_launches = sum(1 for (_, _, kern, _, _) in prof[-1] if kern in dom)
    if sp["bound"] == "tensor":
        dflops = sp.get("dominant_flops", sp["flops"])
        ach = dflops / (dom_ms / 1e3) / 1e12 if dom_ms else None
        roof = {"bound": "tensor", "achieved": round(ach, 2) if ach else None, "peak": round(pk["int8_tops"], 1),
                "unit": "TFLOP/s", "frac": round(ach / pk["int8_tops"], 4) if ach else None,
                "traffic": c5_traffic() if sp["cfg"] == "c5" else traffic_of(sp["cfg"]), "peak_kind": pk["int8_kind"],
                "kernel": "+".join(dom),
                "kernel_ms_per_step": round(dom_ms, 5), "launches_per_step": dom_launches,
                "algorithmic_ops_per_step": dflops,
                "network": {"achieved": round(work / (ms_per_step / 1e3) / 1e12, 2),
                            "frac": round(work / (ms_per_step / 1e3) / 1e12 / pk["int8_tops"], 4),
                            "note": "whole step (all launches, lanes overlapped, graph replay) / int8 peak"}}
    else:
        # HBM-bound: algorithmic bytes of the step / the dominant kernel's time.  The step of
        # C2/C3/C4 is ONE launch, so the graph-timed step is that kernel's launch duration.
        kms = ms_per_step if dom_launches == 1 and len(prof[-1]) == 1 else dom_ms
        ach = alg_bytes / (kms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / pk["hbm_gbs"], 4), "traffic": traffic_of(sp["cfg"]), "peak_kind": pk["kind"],
                "kernel": "+".join(dom), "kernel_ms": round(kms, 5), "algorithmic_bytes_per_launch": alg_bytes,
                "isolated": {"kernel_ms": round(iso_ms, 5),
                             "frac": round(alg_bytes / (iso_ms / 1e3) / 1e9 / pk["hbm_gbs"], 4),
                             "note": "one step alone, synchronized before and after (no PDL overlap)"}}
        if sp["flops"]:
            roof["tensor"] = {"achieved_tops": round(sp["flops"] / (kms / 1e3) / 1e12, 2),
                              "int8_peak_tops": round(pk["int8_tops"], 1), "peak_kind": pk["int8_kind"],
                              "frac": round(sp["flops"] / (kms / 1e3) / 1e12 / pk["int8_tops"], 4)}
    breakdown = {k: {"ms": round(v, 5), "share": round(v / prof_total, 4)} for k, v in
                 sorted(fam_ms.items(), key=lambda kv: -kv[1])} if prof_total else {}

    # ---- end to end through the public API (host buffers, copies inside the timed region) ----
    e2e = e2e_native(args, sb, np, torch, dist, world, ctx, prog, nbytes, in_names, out_names, work, sp['unit'],
                     dev, local)
    dropin = e2e_dropin(args, sb, np, torch, dist, world, ctx, prog, in_names, out_names, work, sp['unit'], dev)
    e2e["dropin"] = dropin

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline_obj(sp)
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "unit": sp["unit"], "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        cfgj = {"workload": sp["workload"], "global_batch": sp["global_batch"],
                "parallelism": f"batch-sharded x{world} (no collective)" if sp["cfg"] not in ("c1", "c1_i32")
                else f"row-sharded x{world} (no collective)",
                "l2": f"{nsets} rotating input/output sets ({nsets * alg_bytes / 2**20:.0f} MiB)"
                      + (" + >1 GB activation arena per step" if sp["cfg"] == "c5" else "")}
        if sp["cfg"] == "c5":
            cfgj["images_per_s"] = round(sp["global_batch"] / (ms_per_step / 1e3), 1)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": sp["unit"], "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": sp["scaling"], "vs_baseline": None, "dtype": "i8xi8->i32" if sp["flops"] else "i32",
            "data": "synthetic (uniform random bytes in HBM; i8 images/weights, i32 biases)",
            "config": cfgj, "roofline": roof, "kernel_breakdown": breakdown, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "launches_per_step": int(launches) // args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def sum_over_ranks(dist, world, dev, work):
    import torch
    t = torch.tensor([work], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t)
    return float(t.item())


def c5_traffic():
    """DRAM bytes per step of C5's conv family from the committed ncu capture of one b1024 step
    (profiles/r02_c5_traffic.json: 26.8 GB against 28.0 GB algorithmic), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_c5_traffic.json")) as f:
            return json.load(f)["c5"]["dram_bytes_per_step"]
    except Exception:
        return None


def traffic_of(cfg):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed ncu
    capture: the steady-state one (profiles/r02_traffic_warm.json, `--cache-control none` on
    launches after the set rotation, so earlier launches' dirty outputs are written back inside
    the profiled ones; profiles/capture_r02_warm.sh), else the cold-cache one
    (profiles/r02_traffic.json), else None."""
    for name in ("r02_traffic_warm.json", "r02_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)[cfg]["dram_bytes_per_launch"]
        except Exception:
            continue
    return None


def e2e_native(args, sb, np, torch, dist, world, ctx, prog, nbytes, in_names, out_names, work, unit, dev, local):
    """sb_execute_async on two contexts ping-ponging steps: every step copies its inputs in
    from pinned host memory and its outputs out; step i's D2H overlaps step i+1's H2D."""
    ctx.set_stream(None)
    ctxs = [ctx, sb.Context(local)]
    ordered = not os.environ.get("SB_E2E_UNORDERED")
    for c_ in ctxs:  # one step's kernels at a time; copies overlap the other step's kernels
        c_.set_kernel_order(ordered)
    pins, hosts = [], []
    for _ in ctxs:
        host = {}
        for n, d in prog.buffers.items():
            p = ctypes.c_void_p()
            sb._check(sb.lib().sb_host_alloc_pinned(nbytes[n], ctypes.byref(p)))
            pins.append(p)
            ct = {8: ctypes.c_int8, 16: ctypes.c_int16, 32: ctypes.c_int32}[d.dtype]
            host[n] = np.ctypeslib.as_array((ct * d.elements).from_address(p.value))
        hosts.append(host)
    rng = np.random.default_rng(11)
    for n in in_names:
        vals = rng.integers(-128, 128, hosts[0][n].size).astype(hosts[0][n].dtype)
        for h in hosts:
            h[n][:] = vals
    outs = tuple(out_names)
    for i in range(2):
        ctxs[i % 2].execute_native_async(prog, hosts[i % 2], prepare=outs)
    for c_ in ctxs:
        c_.sync()
    if world > 1:
        dist.barrier()
    steps = max(4, min(args.steps, 10))
    t0 = time.perf_counter()
    for i in range(steps):
        ctxs[i % 2].execute_native_async(prog, hosts[i % 2], prepare=outs)
    for c_ in ctxs:
        c_.sync()
    te = torch.tensor([time.perf_counter() - t0], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    tot = sum_over_ranks(dist, world, dev, work)
    for p in pins:
        sb.lib().sb_host_free_pinned(p)
    return {"value": round(tot * steps / float(te.item()) / 1e9, 3), "unit": unit, "h2d_bytes_per_step": int(sum(nbytes[n] for n in in_names)),
            "d2h_bytes_per_step": int(sum(nbytes[n] for n in out_names)), "steps": steps,
            "api": "sb_execute_async, native-width pinned host buffers",
            "timer": "host wall clock from the first sb_execute_async to the last context sync (2 contexts)",
            "kernel_order": ordered}


def e2e_dropin(args, sb, np, torch, dist, world, ctx, prog, in_names, out_names, work, unit, dev):
    """The stripe::b200::execute boundary: sb_execute with int64 carriers (interp.h:14-17), one
    synchronous call per step -- int64 -> native conversion, H2D, execute, D2H, native -> int64."""
    rng = np.random.default_rng(12)
    store = {}
    for n in in_names:
        store[n] = sb.Buffer(prog.buffers[n].dtype, rng.integers(-128, 128, prog.buffers[n].elements,
                                                                   dtype=np.int64))
    c2 = sb.Context(ctx.device)
    st = dict(store)
    sb.prepare_outputs(prog, st)
    c2.execute(prog, st)  # warm (plan, device buffers, pinned staging)
    if world > 1:
        dist.barrier()
    steps = 2 if work > 1e12 else max(3, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(steps):
        st = dict(store)
        sb.prepare_outputs(prog, st)
        c2.execute(prog, st)
    te = torch.tensor([time.perf_counter() - t0], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    tot = sum_over_ranks(dist, world, dev, work)
    return {"value": round(tot * steps / float(te.item()) / 1e9, 3), "unit": unit,
            "h2d_bytes_per_step": int(sum(prog.buffers[n].elements * 8 for n in in_names)),
            "d2h_bytes_per_step": int(sum(prog.buffers[n].elements * 8 for n in out_names)), "steps": steps,
            "api": "sb_execute with int64 carriers (the stripe::b200::execute drop-in boundary), synchronous",
            "note": "bytes counted at the int64 carrier width the caller hands over"}


def dry_run(args):
    """What run_ours does across ranks, without a GPU: gloo process group, each rank's shard of
    the config, the barrier and the max-over-ranks reduction of a (fake) device time."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    sp = spec(args.config, world, rank, args)
    t = torch.tensor([1.0 + rank])
    imgs = torch.tensor([float(sp["images"])])
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(imgs)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_elapsed": float(t.item()),
                          "images_total": int(imgs.item()), "global_batch": sp["global_batch"],
                          "scaling": sp["scaling"], "pid": os.getpid()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------
def launch_ranks(args):
    """`--gpus N` outside a launcher: start N ranks with torch.distributed.run (127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c5", choices=["c5", "c2", "c3", "c4a", "c4b", "c1", "c1_i32"])
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch (C5: global batch)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check on CPU: gloo ranks report their shard and the max-over-ranks time")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
