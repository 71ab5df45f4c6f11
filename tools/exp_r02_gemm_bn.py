#!/usr/bin/env python
"""i8 GEMM throughput at a large square size through sb_execute_device (CUDA events, best of
reps x 10 back-to-back calls): `python tools/exp_r02_gemm_bn.py N` (SB_GEMM_BN=128|256 forces
the tile width)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    prog = sb.parse_program(W.matmul(n, n, n, in_dtype="i8", out_dtype="i32"))
    ctx = sb.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    a = torch.randint(-128, 128, (n * n,), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 128, (n * n,), dtype=torch.int8, device="cuda")
    c = torch.empty(n * n, dtype=torch.int32, device="cuda")
    run = ctx.bind_device(prog, {"A": (a.data_ptr(), n * n, 0), "B": (b.data_ptr(), n * n, 0),
                                 "C": (c.data_ptr(), n * n, sb.SB_BUF_PREPARE)})
    best = 1e30
    with torch.cuda.stream(s):
        run()
        ctx.sync()
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                run()
            e1.record(s)
            ctx.sync()
            best = min(best, e0.elapsed_time(e1) / 10)
    ref = (a.view(n, n)[:256].cpu().to(torch.int64) @ b.view(n, n)[:, :256].cpu().to(torch.int64)).to(torch.int32)
    ok = torch.equal(c.view(n, n)[:256, :256].cpu(), ref)
    print(f"n={n} bn={os.environ.get('SB_GEMM_BN', 'auto')} {best * 1e3:.1f} us {2 * n ** 3 / best / 1e9:.1f} TOPS exact={ok}")


if __name__ == "__main__":
    main()
