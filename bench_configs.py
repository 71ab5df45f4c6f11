#!/usr/bin/env python
"""Per-config device throughput of the executor on every BASELINE.json configuration
(the headline bench line is bench.py = config 2).  HBM-resident buffers, CUDA-graph
replay of K steps, CUDA-event timing; one JSON line per config.

    python bench_configs.py [--configs c1,c2,c3,c4a,c4b] [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"])
    except Exception:
        return 6650.0, 1590.0


def configs(want=None):
    from paper_1903_06498_b200 import workloads as W
    out = {}
    # C1: matmul 1024^3 (integer modes; the reference has no f32)
    M = N = Kd = 1024
    for dt, od in (("i8", "i32"), ("i32", "i32"), ("f32", "f32")):
        out[f"c1_matmul_{dt}"] = dict(text=W.matmul(M, N, Kd, in_dtype=dt, out_dtype=od),
                                      flops=2.0 * M * N * Kd,
                                      bytes=(M * Kd + Kd * N) * (1 if dt == "i8" else 4) + M * N * 4)
    # (f32 inputs: torch.randint bytes reinterpreted as floats; finite values are not needed for timing)
    out["c1_matmul_f32_tf32x3"] = dict(text=W.matmul(M, N, Kd, in_dtype="f32", out_dtype="f32"),
                                       flops=2.0 * M * N * Kd, bytes=(M * Kd + Kd * N) * 4 + M * N * 4,
                                       opts=dict(fp32_mode=1))
    out["c2_conv"] = dict(text=W.conv2d(32, 56, 56, 64, 64), flops=2.0 * W.conv_useful_macs(32, 56, 56, 64, 64),
                          bytes=32 * 56 * 56 * 64 + 9 * 64 * 64 + 32 * 56 * 56 * 64 * 4)
    out["c3_conv_bias_relu"] = dict(text=W.conv_bias_relu(128, 56, 56, 64, 64),
                                    flops=2.0 * W.conv_useful_macs(128, 56, 56, 64, 64),
                                    bytes=128 * 56 * 56 * 64 + 9 * 64 * 64 + 64 * 4 + 128 * 56 * 56 * 64 * 4)
    out["c4a_maxpool"] = dict(text=W.maxpool2x2(128, 112, 112, 64), flops=0.0,
                              bytes=128 * 112 * 112 * 64 * 4 + 128 * 56 * 56 * 64 * 4)
    out["c4b_global_sum"] = dict(text=W.global_sum(1024, 7, 7, 2048), flops=0.0,
                                 bytes=1024 * 49 * 2048 * 4 + 1024 * 2048 * 4)
    # C5: ResNet-50 program; batch 1024 sharded 8 ways -> 128 images per GPU
    if want and not any(w.startswith("c5") for w in want):
        return out
    b5 = int(os.environ.get("SB_C5_BATCH", "128"))
    text, info = W.resnet50(b5)
    out["c5_resnet50"] = dict(text=text, flops=float(info["flops"]), bytes=b5 * 224 * 224 * 3 + b5 * 1000 * 4,
                              images=b5)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--generic", action="store_true", help="disable specialised kernels")
    args = ap.parse_args()
    import torch

    import paper_1903_06498_b200 as sb
    hbm, bf16 = peaks()
    ctx = sb.Context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    want = set(args.configs.split(",")) if args.configs else None
    for name, cfg in configs(want).items():
        if want and not any(name.startswith(w) for w in want):
            continue
        prog = sb.parse_program(cfg["text"])
        bufs, keep = {}, []
        for bn, d in prog.buffers.items():
            nbytes = d.elements * {8: 1, 16: 2, 32: 4, 0x20F: 4}[d.dtype]
            t = torch.randint(-128, 128, (nbytes,), dtype=torch.int8, device="cuda")
            keep.append(t)
            bufs[bn] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
        opts = sb.ExecOptions(disable_tensor_cores=args.generic, **cfg.get("opts", {}))
        run = ctx.bind_device(prog, bufs, opts)
        with torch.cuda.stream(stream):
            run()
            ctx.sync()
            launches0 = ctx.launch_count
            g = sb.Graph(ctx, lambda: [run() for _ in range(args.steps)])
            g.launch()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.launch()
            e1.record(stream)
            torch.cuda.synchronize()
            ctx.sync()
        ms = e0.elapsed_time(e1) / args.steps
        line = {"config": name, "ms_per_step": round(ms, 5),
                "launches_per_step": (ctx.launch_count - launches0) // (2 * args.steps),
                "GB/s": round(cfg["bytes"] / ms / 1e6, 1), "hbm_frac": round(cfg["bytes"] / ms / 1e6 / hbm, 4),
                "plan": [l.split(" mode")[0] for l in
                         prog.describe_plan(True, not args.generic, cfg.get("opts", {}).get("fp32_mode", 0)).splitlines()]}
        if cfg["flops"]:
            line["GOP/s"] = round(cfg["flops"] / ms / 1e6, 1)
        if "images" in cfg:
            line["images_per_s"] = round(cfg["images"] / ms * 1e3, 1)
            line["plan"] = [p for p in line["plan"] if not p.startswith("(elided)") and not p.startswith("note")]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
