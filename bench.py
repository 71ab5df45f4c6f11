#!/usr/bin/env python
"""Benchmark of the B200 Stripe block executor (BASELINE.json contract).

Workload (N=1): BASELINE config 2 — a 3x3 conv2d NHWC 56x56x64->64, batch 32,
with padding constraints, as ONE Stripe block (paper_1903_06498_b200.workloads.conv2d),
i8 x i8 -> i32 (the reference's integer semantics; bit-exact vs its interpreter).
A step = prepare_outputs + execute of that program over one batch (the identity
fill of the output is fused into the conv epilogue).  Multi-GPU: weak scaling,
each rank runs its own batch-32 shard (the batch index partitions with no
data-path collective).

value  : useful GFLOP/s (2 x constraint-satisfying MAC points, tile.cpp:338-370),
         inputs resident in HBM, max-over-ranks device time.
e2e    : same metric through the public API (sb_execute) from pinned host
         buffers: H2D of I and F and D2H of O inside the timed region.
--impl reference: the reference interpreter (oracle/_ref, stripe::execute) on
         the host cores over a bounded sample of the same workload.

--config c5: BASELINE config 5 instead -- the ResNet-50-shaped Stripe program
         (workloads.resnet50), 128 images per GPU (batch 1024 over 8 GPUs, sharded on
         the batch index, no collective).  value = useful GFLOP/s of the whole network.
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
N_IMG, H, W, C, K = 32, 56, 56, 64, 64
L2_BYTES = 126 * 1024 * 1024


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


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


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------------------
def cpu_reference(samples_rows=8, threads=None, steps=1, warmup=0):
    """Reference interpreter (unmodified stripe::execute from oracle/_ref) on host cores.
    One step = `threads` concurrent executions (one per host thread, execute is reentrant,
    SPEC.md:263) of a row-band sample of config 2: 1 image x `samples_rows` output rows."""
    import numpy as np

    from oracle import Ref, random_inputs
    from paper_1903_06498_b200 import workloads as Wk
    threads = threads or os.cpu_count() or 1
    text = Wk.conv2d(1, samples_rows, W, C, K)
    macs = Wk.conv_useful_macs(1, samples_rows, W, C, K)
    L = Ref.lib()
    prog = Ref.parse(text)
    bufs = prog.buffers()
    inputs = random_inputs(bufs, 1001)
    times = []
    for it in range(warmup + steps):
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
        if it >= warmup:
            times.append(dt)
    gflops = 2.0 * macs * threads / (sum(times) / len(times)) / 1e9
    sample = (f"{threads} concurrent stripe::execute runs (one per host thread) of config 2 restricted to "
              f"1 image x {samples_rows} output rows ({macs} useful MACs each), reference built -O2 from "
              f"/root/reference/proj/src")
    return gflops, threads, sample, times


def cpu_reference_resnet(threads=None, steps=1, warmup=0):
    """Reference interpreter on a bounded sample of config 5: concurrent executions (one per
    host thread) of the full-width ResNet-50 program on one 32x32 image (1.4e8 useful MACs
    after the stem), i.e. the same layer mix at 1/49 of the spatial work."""
    import numpy as np

    from oracle import Ref, random_inputs
    from paper_1903_06498_b200 import workloads as Wk
    threads = threads or os.cpu_count() or 1
    text, info = Wk.resnet50(1, image=32)
    L = Ref.lib()
    prog = Ref.parse(text)
    bufs = prog.buffers()
    inputs = random_inputs(bufs, 1005)
    times = []
    for it in range(warmup + steps):
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
        if it >= warmup:
            times.append(dt)
    gflops = info["flops"] * threads / (sum(times) / len(times)) / 1e9
    sample = (f"{threads} concurrent stripe::execute runs (one per host thread) of the config-5 ResNet-50 program "
              f"at 32x32 image, batch 1 ({info['macs']} useful MACs each)")
    return gflops, threads, sample, times


def run_reference_arm(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    if args.config == "c5":
        from oracle import Ref
        if not Ref.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libstripe_ref.so not built"}))
            return
        gflops, cores, sample, times = cpu_reference_resnet(steps=args.steps, warmup=min(args.warmup, 1))
        print(json.dumps({
            "metric": METRIC, "value": round(gflops, 4), "unit": "GFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * sum(times) / len(times), 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "i8xi8->i32 (int64 carriers)", "data": "synthetic (random_inputs, seed 1005)",
            "config": {"workload": "BASELINE config 5: ResNet-50 Stripe program", "sample": "32x32 image"},
            "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return
    from oracle import Ref
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libstripe_ref.so not built"}))
        return
    gflops, cores, sample, times = cpu_reference(samples_rows=8, steps=args.steps, warmup=args.warmup)
    print(json.dumps({
        "metric": METRIC, "value": round(gflops, 4), "unit": "GFLOP/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * sum(times) / len(times), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "i8xi8->i32 (int64 carriers)",
        "data": "synthetic (splitmix64 random_inputs, seed 1001)",
        "config": {"workload": "BASELINE config 2: conv2d 3x3 NHWC 56x56x64->64 batch 32, padding constraints",
                   "sample": "row band"},
        "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as Wk

    world, rank, local = dist_setup()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)

    text = Wk.conv2d(N_IMG, H, W, C, K)
    prog = sb.parse_program(text)
    plan = prog.describe_plan(fresh_outputs=True)
    assert "conv_i8_tc" in plan, plan
    ctx = sb.Context(local)
    ctx.set_stream(stream.cuda_stream)

    macs = Wk.conv_useful_macs(N_IMG, H, W, C, K)
    flops_step = 2.0 * macs
    in_bytes = N_IMG * H * W * C + 3 * 3 * K * C
    out_bytes = N_IMG * H * W * K * 4
    alg_bytes = in_bytes + out_bytes

    # rotate through enough input/output sets that the working set exceeds L2
    nsets = max(4, int(3 * L2_BYTES // alg_bytes) + 1)
    g = torch.Generator(device=dev).manual_seed(1001 + rank)
    sets = []
    for _ in range(nsets):
        I = torch.randint(-128, 128, (N_IMG, H, W, C), dtype=torch.int8, device=dev, generator=g)
        F = torch.randint(-128, 128, (3, 3, K, C), dtype=torch.int8, device=dev, generator=g)
        O = torch.empty((N_IMG, H, W, K), dtype=torch.int32, device=dev)
        sets.append({"I": (I.data_ptr(), I.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                     "O": (O.data_ptr(), O.numel(), sb.SB_BUF_PREPARE), "_keep": (I, F, O)})

    bound = [ctx.bind_device(prog, {k: v for k, v in s.items() if not k.startswith("_")}) for s in sets]

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
        settle = 0
        t_settle = time.perf_counter()
        while time.perf_counter() - t_settle < 1.0:
            for _ in range(20):
                step(args.warmup + settle)
                settle += 1
            torch.cuda.synchronize(dev)
        ctx.sync()
        barrier()
        torch.cuda.synchronize(dev)
        # eager (one host call per step) timing, for reference only
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        eager_ms = e0.elapsed_time(e1) / args.steps
        # the timed region: exactly K steps, captured once as a CUDA graph (sb_graph_*) so
        # host launch latency is off the device timeline
        graph = sb.Graph(ctx, lambda: [step(args.warmup + i) for i in range(args.steps)])
        graph.launch()  # warm the graph itself (untimed)
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        launches0 = ctx.launch_count
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
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
        kernel_ms = [elapsed_ms / args.steps]  # one conv launch per step, back to back

    t = torch.tensor([elapsed_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = flops_step * world * args.steps / (elapsed_ms / 1e3) / 1e9

    # ---- end-to-end through the public API (host buffers, H2D + D2H inside the region) ----
    # sb_execute_async on two contexts ping-ponging steps: step i's device-to-host copy of O
    # overlaps step i+1's host-to-device copy of I and F (the two copy directions run
    # concurrently over PCIe); every step still copies its inputs in and its result out.
    ctx.set_stream(None)
    e2e_steps = max(4, min(args.steps, 20))
    ctxs = [ctx, sb.Context(local)]
    pins = []

    def pinned(n, ct):
        p = ctypes.c_void_p()  # pinned host memory from the library's own allocator
        sb._check(sb.lib().sb_host_alloc_pinned(n * ctypes.sizeof(ct), ctypes.byref(p)))
        pins.append(p)
        return np.ctypeslib.as_array((ct * n).from_address(p.value))

    hI = pinned(N_IMG * H * W * C, ctypes.c_int8)
    hF = pinned(3 * 3 * K * C, ctypes.c_int8)
    hO = [pinned(N_IMG * H * W * K, ctypes.c_int32) for _ in ctxs]
    rng = np.random.default_rng(7 + rank)
    hI[:] = rng.integers(-128, 128, hI.size, dtype=np.int8)
    hF[:] = rng.integers(-128, 128, hF.size, dtype=np.int8)
    for i in range(4):
        ctxs[i % 2].execute_native_async(prog, {"I": hI, "F": hF, "O": hO[i % 2]}, prepare=("O",))
    for c_ in ctxs:
        c_.sync()
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        ctxs[i % 2].execute_native_async(prog, {"I": hI, "F": hF, "O": hO[i % 2]}, prepare=("O",))
    for c_ in ctxs:
        c_.sync()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": round(flops_step * world * e2e_steps / float(te.item()) / 1e9, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(hI.nbytes + hF.nbytes), "d2h_bytes_per_step": int(hO[0].nbytes),
           "steps": e2e_steps,
           "timer": "host wall clock from the first sb_execute_async to the last context sync (2 contexts)"}
    for p in pins:
        sb.lib().sb_host_free_pinned(p)

    hbm_peak, bf16_peak, peak_kind = peaks()
    avg_kernel_ms = statistics.mean(kernel_ms)
    achieved_gbs = alg_bytes / (avg_kernel_ms / 1e3) / 1e9
    tensor_tops = flops_step / (avg_kernel_ms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "conv_tc_traffic.json")) as f:
            traffic = json.load(f).get("bytes_per_launch")
    except Exception:
        pass

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            from oracle import Ref
            if Ref.available():
                gf, cores, sample, _ = cpu_reference(samples_rows=8, steps=1, warmup=0)
                cpu = {"value": round(gf, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                       "sample": sample}
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "i8xi8->i32",
            "data": "synthetic (uniform random int8 inputs in HBM)",
            "config": {"workload": "BASELINE config 2: conv2d 3x3 NHWC 56x56x64->64, batch 32 per GPU, "
                                   "padding constraints, one Stripe block",
                       "global_batch": N_IMG * world, "parallelism": f"batch-sharded x{world} (no collective)",
                       "l2": f"{nsets} rotating input/output sets ({nsets * alg_bytes / 2**20:.0f} MiB > L2)"},
            "roofline": {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved_gbs / hbm_peak, 4), "traffic": traffic,
                         "peak_kind": peak_kind, "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel_ms": round(avg_kernel_ms, 5),
                         "tensor": {"achieved_tops": round(tensor_tops, 2),
                                    "int8_peak_tops_derived": round(2 * bf16_peak, 1),
                                    "frac": round(tensor_tops / (2 * bf16_peak), 4)}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "eager_ms_per_step": round(eager_ms, 5),
            "clock_settle_steps": settle,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_ours_resnet(args):
    """Config 5: ResNet-50 program, 128 images per GPU, weak scaling over batch shards."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as Wk

    world, rank, local = dist_setup()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    per_gpu = args.batch_per_gpu
    text, info = Wk.resnet50(per_gpu)
    prog = sb.parse_program(text)
    ctx = sb.Context(local)
    ctx.set_stream(stream.cuda_stream)
    flops_step = float(info["flops"])
    nbytes = {n: d.elements * {8: 1, 16: 2, 32: 4}[d.dtype] for n, d in prog.buffers.items()}
    in_names = [n for n, d in prog.buffers.items() if int(d.dir) == 0]
    alg_bytes = sum(nbytes.values())
    # two input/output sets: each step's activations (> 1 GB of scratch) flush L2 anyway
    g = torch.Generator(device=dev).manual_seed(1005 + rank)
    sets = []
    for _ in range(2):
        bufs, keep = {}, []
        for n, d in prog.buffers.items():
            t = torch.randint(-128, 128, (nbytes[n],), dtype=torch.int8, device=dev, generator=g)
            keep.append(t)
            bufs[n] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
        sets.append((bufs, keep))
    bound = [ctx.bind_device(prog, b) for b, _ in sets]

    def step(i):
        bound[i % 2]()

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        clk = ClockSampler(local).__enter__()
        clk.wait_first_sample()
        for i in range(args.warmup):
            step(i)
        t_settle = time.perf_counter()
        settle = 0
        while time.perf_counter() - t_settle < 1.0:
            step(settle)
            settle += 1
            torch.cuda.synchronize(dev)
        ctx.sync()
        graph = sb.Graph(ctx, lambda: [step(i) for i in range(args.steps)])
        graph.launch()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        launches0 = ctx.launch_count
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
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
    t = torch.tensor([elapsed_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = flops_step * world * args.steps / (elapsed_ms / 1e3) / 1e9

    # end to end through the public API from pinned host buffers (every program input copied
    # in, the logits copied out, each step): sb_execute_async on two contexts ping-ponging
    # steps, so step i+1's host-to-device copies overlap step i's compute
    ctx.set_stream(None)
    ctxs = [ctx, sb.Context(local)]
    pins = []
    hosts = []
    for _ in ctxs:
        host = {}
        for n, d in prog.buffers.items():
            p = ctypes.c_void_p()
            sb._check(sb.lib().sb_host_alloc_pinned(nbytes[n], ctypes.byref(p)))
            pins.append(p)
            ct = {8: ctypes.c_int8, 16: ctypes.c_int16, 32: ctypes.c_int32}[d.dtype]
            host[n] = np.ctypeslib.as_array((ct * d.elements).from_address(p.value))
        hosts.append(host)
    rng = np.random.default_rng(11 + rank)
    for n in in_names:
        vals = rng.integers(-128, 128, hosts[0][n].size).astype(hosts[0][n].dtype)
        for h in hosts:
            h[n][:] = vals
    outs = tuple(n for n in prog.buffers if n not in in_names)
    for i in range(2):
        ctxs[i % 2].execute_native_async(prog, hosts[i % 2], prepare=outs)
    for c_ in ctxs:
        c_.sync()
    barrier()
    e2e_steps = max(4, min(args.steps, 10))
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        ctxs[i % 2].execute_native_async(prog, hosts[i % 2], prepare=outs)
    for c_ in ctxs:
        c_.sync()
    te = torch.tensor([time.perf_counter() - t0], device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": round(flops_step * world * e2e_steps / float(te.item()) / 1e9, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(sum(nbytes[n] for n in in_names)),
           "d2h_bytes_per_step": int(sum(nbytes[n] for n in outs)), "steps": e2e_steps,
           "timer": "host wall clock from the first sb_execute_async to the last context sync (2 contexts)"}
    for p in pins:
        sb.lib().sb_host_free_pinned(p)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            from oracle import Ref
            if Ref.available():
                gf, cores, sample, _ = cpu_reference_resnet(steps=1, warmup=0)
                cpu = {"value": round(gf, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                       "sample": sample}
        except Exception as e:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    if rank == 0:
        hbm_peak, bf16_peak, peak_kind = peaks()
        tops = flops_step / (ms_per_step / 1e3) / 1e12
        i8_peak = 2 * bf16_peak
        print(json.dumps({
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "i8xi8->i32",
            "data": "synthetic (uniform random int8 image, weights, i32 biases in HBM)",
            "config": {"workload": f"BASELINE config 5: ResNet-50 Stripe program (53 convs, max-pool, residuals, "
                                   f"global sum, fc), {per_gpu} images per GPU",
                       "global_batch": per_gpu * world, "parallelism": f"batch-sharded x{world} (no collective)",
                       "images_per_s": round(per_gpu * world / (ms_per_step / 1e3), 1),
                       "l2": "activations > 1 GB per step (scratch arena) flush L2"},
            "roofline": {"bound": "tensor", "achieved": round(tops, 2), "peak": round(i8_peak, 1), "unit": "TFLOP/s",
                         "frac": round(tops / i8_peak, 4), "traffic": None,
                         "peak_kind": f"dense int8 = 2 x {peak_kind} bf16 ({bf16_peak})",
                         "note": "whole-network useful ops / step time (all 59 launches)"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        }))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c2", choices=["c2", "c5"])
    ap.add_argument("--batch-per-gpu", type=int, default=128, help="config 5 images per GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.config == "c5":
        run_ours_resnet(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
