#!/usr/bin/env python
"""Per-layer roofline table of the config-5 ResNet-50 program.

Runs resnet50(B) on cuda:0 with per-step CUDA-event timing (sb_context_set_profile: steps
serial, no lane overlap), maps each conv step to its layer, and compares the time with the
layer's floor max(HBM bytes / HBM peak, 2*MACs / int8 peak) -- peaks from MEASURED_PEAKS.json
and profiles/r02_peaks.json.  HBM bytes = i8 input + weights + i32 bias + i8 output (+ i8
residual), each once.

    python tools/c5_layers.py [--batch 128] [--reps 3] > profiles/r02_c5_layers.txt
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    import bench
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    pk = bench.peaks()
    hbm, i8 = pk["hbm_gbs"] * 1e9, pk["int8_tops"] * 1e12
    text, info = W.resnet50(a.batch)
    prog = sb.parse_program(text)
    ctx = sb.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    bufs, keep = {}, []
    for n, d in prog.buffers.items():
        t = torch.randint(-128, 128, (d.elements * bench.ISZ[d.dtype],), dtype=torch.int8, device="cuda")
        keep.append(t)
        bufs[n] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
    run = ctx.bind_device(prog, bufs)
    with torch.cuda.stream(s):
        run()
        ctx.sync()
        ctx.set_profile(True)
        recs = []
        for _ in range(a.reps):
            run()
            ctx.sync()
            recs.append(ctx.read_profile())
        ctx.set_profile(False)
    ms = {}
    for rec in recs:
        for (step, t, kern, path, pts) in rec:
            ms.setdefault((step, kern, path), []).append(t)
    rows = []
    N = a.batch
    for (step, kern, path), ts in sorted(ms.items()):
        t = statistics.median(ts) / 1e3
        parts = path.split(".")
        stmt = int(parts[1]) if len(parts) > 1 and parts[1].isdigit() else -1
        layer = 0 if stmt == 0 else stmt - 1 if 2 <= stmt <= 53 else None
        if kern.startswith("conv") and layer is not None:
            c = info["convs"][layer]
            by = N * c["H"] * c["W"] * c["C"] + c["R"] * c["S"] * c["K"] * c["C"] + 4 * c["K"] + \
                N * c["P"] * c["Q"] * c["K"] * (2 if c["residual"] else 1)
            fl = 2.0 * c["macs"]
            name = f"L{layer:02d} {c['R']}x{c['S']}/{c['stride']} {c['H']}x{c['W']}x{c['C']}->{c['K']}" + \
                (" +res" if c["residual"] else "")
        elif kern == "gemm_i8_tc" or stmt == 55:
            C, K = 2048, 1000
            by, fl, name = N * C + K * C + 4 * K + 4 * N * K, 2.0 * N * C * K, "fc 2048->1000"
        elif kern == "pool":
            by, fl, name = N * 112 * 112 * 64 + N * 56 * 56 * 64, 0.0, "maxpool 3x3/2"
        elif kern == "reduce":
            by, fl, name = N * 7 * 7 * 2048 + N * 2048, 0.0, "global sum 7x7"
        else:
            by, fl, name = 0, 0.0, f"{kern} {path}"
        floor = max(by / hbm, fl / i8)
        rows.append((name, kern, t, by, fl, floor))
    tot = sum(r[2] for r in rows)
    tfloor = sum(r[5] for r in rows)
    print(f"# tools/c5_layers.py --batch {N}: per-step CUDA events (serial), median of {a.reps}; "
          f"peaks HBM {pk['hbm_gbs']} GB/s ({pk['kind']}), int8 {pk['int8_tops']:.1f} TOPS ({pk['int8_kind']})")
    print(f"{'layer':34s} {'kernel':14s} {'us':>8s} {'MB':>8s} {'GOP':>8s} {'floor_us':>8s} {'bound':>6s} "
          f"{'frac':>6s} {'share':>6s}")
    for name, kern, t, by, fl, floor in rows:
        bound = "tensor" if fl / i8 > by / hbm else "hbm"
        print(f"{name:34s} {kern:14s} {t * 1e6:8.1f} {by / 1e6:8.2f} {fl / 1e9:8.2f} {floor * 1e6:8.1f} {bound:>6s} "
              f"{floor / t if t else 0:6.3f} {t / tot:6.3f}")
    print(f"TOTAL {tot * 1e6:.1f} us, floor {tfloor * 1e6:.1f} us, frac of per-layer roofline {tfloor / tot:.3f}; "
          f"useful {info['flops'] / tot / 1e12:.1f} TOPS = {info['flops'] / tot / i8:.3f} of int8 peak")


if __name__ == "__main__":
    main()
