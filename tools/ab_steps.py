#!/usr/bin/env python
"""In-process A/B of environment switches read at launch time: per-step device times of one
program (sb_context_set_profile), variants interleaved so box and clock drift hit all alike.

    python tools/ab_steps.py PROG BATCH REPS VAR[=VAL][+VAR..] ...    ('-' = no switch)
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1903_06498_b200 as sb
    args = sys.argv[1:]
    prog_name, batch, reps, variants = args[0], int(args[1]), int(args[2]), args[3:]
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import profile_steps
    text = profile_steps.program_text(prog_name, batch)
    prog = sb.parse_program(text)
    ctx = sb.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    bufs, keep = {}, []
    for bn, d in prog.buffers.items():
        nbytes = d.elements * {8: 1, 16: 2, 32: 4}[d.dtype]
        t = torch.randint(-128, 128, (nbytes,), dtype=torch.int8, device="cuda")
        keep.append(t)
        bufs[bn] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
    run = ctx.bind_device(prog, bufs)

    def setv(v, on):
        # one variant = "-" (no switch) or VAR[=VAL] switches joined by "+"
        if v == "-":
            return
        for one in v.split("+"):
            k, _, val = one.partition("=")
            if on:
                os.environ[k] = val or "1"
            else:
                os.environ.pop(k, None)

    res = {v: {} for v in variants}
    with torch.cuda.stream(s):
        run()
        ctx.sync()
        ctx.set_profile(True)
        for _ in range(reps):
            for v in variants:
                setv(v, True)
                run()
                ctx.sync()
                for (step, t, kern, path, pts) in ctx.read_profile():
                    res[v].setdefault((step, kern), []).append(t * 1e3)
                setv(v, False)
    for v in variants:
        tot = sum(statistics.median(ts) for ts in res[v].values())
        per = " ".join(f"{k[1]}:{statistics.median(ts):.1f}" for k, ts in sorted(res[v].items()))
        print(f"{prog_name} b{batch} {v:24s} total {tot:9.1f} us | {per}", flush=True)


if __name__ == "__main__":
    main()
