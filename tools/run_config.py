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


N_, H_, C_ = 128, 56, 64
S_ = (H_ * H_ * C_, H_ * C_, C_, 1)
# config 3's epilogue block alone (an element-wise Stripe block -> the map kernel)
MAP_TEXT = f"""block []:1 (
	in T[0, 0, 0, 0] i32({N_}, {H_}, {H_}, {C_}):{S_}
	in Bias[0] i32({C_}):(1)
	out O[0, 0, 0, 0]:assign i32({N_}, {H_}, {H_}, {C_}):{S_}
) {{
	0:
	block [n:{N_}, x:{H_}, y:{H_}, k:{C_}]:{N_ * H_ * H_ * C_} (
		in T[n, x, y, k] i32(1, 1, 1, 1):{S_}
		in Bias[k] i32(1):(1)
		out O[n, x, y, k]:assign i32(1, 1, 1, 1):{S_}
	) {{
		0: $t = load(T)
		1: $b = load(Bias)
		2: $s = add($t, $b)
		3: $z = constant(0)
		4: $r = max($s, $z)
		5: O = store($r)
	}}
}}
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--profile", action="store_true", help="print per-step device times")
    ap.add_argument("--program", default="", help="instead of a config: map (config 3's bias+ReLU "
                    "epilogue alone, element-wise kernel) | pool (the ResNet stem max-pool)")
    args = ap.parse_args()
    import torch

    import bench
    import paper_1903_06498_b200 as sb
    if args.program == "map":
        text = MAP_TEXT
    elif args.program == "pool":
        from paper_1903_06498_b200 import workloads as W
        text = W.pool2d(args.batch or 128, 112, 112, 64)
    else:
        text = bench.spec(args.config, 1, 0, args)["text"]
    sp = {"text": text}
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
