#!/usr/bin/env python
"""Runs one BASELINE config's program for a few eager steps (rotating input/output sets whose
working set exceeds L2) -- the command the ncu captures in profiles/capture_r02.sh profile.

    python tools/run_config.py --config c2 [--steps 6] [--profile]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--profile", action="store_true", help="print per-step device times")
    args = ap.parse_args()
    import torch

    import bench
    import paper_1903_06498_b200 as sb
    sp = bench.spec(args.config, 1, 0, args)
    prog = sb.parse_program(sp["text"])
    ctx = sb.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    alg = bench.alg_bytes_of(prog)
    nsets = sp.get("nsets") or max(2, int(3 * bench.L2_BYTES // max(alg, 1)) + 1)
    keep, runs = [], []
    for _ in range(nsets):
        bufs = {}
        for n, d in prog.buffers.items():
            t = torch.randint(-128, 128, (d.elements * bench.ISZ[d.dtype],), dtype=torch.int8, device="cuda")
            keep.append(t)
            bufs[n] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
        runs.append(ctx.bind_device(prog, bufs))
    if args.profile:
        ctx.set_profile(True)
    with torch.cuda.stream(s):
        for i in range(args.steps):
            runs[i % nsets]()
            ctx.sync()
    if args.profile:
        for rec in ctx.read_profile():
            print(*rec)
    print("plan:", prog.describe_plan(True).splitlines()[0][:200])


if __name__ == "__main__":
    main()
