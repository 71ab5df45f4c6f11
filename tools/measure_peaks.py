#!/usr/bin/env python
"""Dense tensor-core peaks on this B200 (the roofline denominators MEASURED_PEAKS.json lacks).

int8 (i8 x i8 -> i32): the best of cuBLASLt (torch._int_mm) and this repo's own tcgen05
gemm_i8_tc (an 8192^3 matmul Stripe program through sb_execute_device), 2*M*N*K ops per call,
best of 10 back-to-back calls timed with CUDA events.  tf32: torch.matmul fp32 with TF32
enabled (cuBLAS), same method.  fp32 SIMT and int32 IMAD are bounded analytically in
DESIGN.md.  Writes profiles/r02_peaks.json (committed; bench.py reads it).

    python tools/measure_peaks.py [--out profiles/r02_peaks.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def best_of(fn, iters=10, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / iters)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_peaks.json"))
    ap.add_argument("--n", type=int, default=8192)
    args = ap.parse_args()
    import torch

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    n = args.n
    ops = 2.0 * n * n * n
    res = {"gpu": torch.cuda.get_device_name(0), "n": n, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    A = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    B = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
    try:
        ms = best_of(lambda: torch._int_mm(A, B))
        res["int8_cublaslt_tops"] = round(ops / ms / 1e9, 1)
    except Exception as e:
        res["int8_cublaslt_tops"] = None
        res["int8_cublaslt_error"] = str(e)[:200]
    prog = sb.parse_program(W.matmul(n, n, n, in_dtype="i8", out_dtype="i32"))
    ctx = sb.Context(0)
    s = torch.cuda.Stream()  # a real stream: the events below are recorded on it too
    ctx.set_stream(s.cuda_stream)
    C = torch.empty((n, n), dtype=torch.int32, device="cuda")
    run = ctx.bind_device(prog, {"A": (A.data_ptr(), A.numel(), 0), "B": (B.data_ptr(), B.numel(), 0),
                                 "C": (C.data_ptr(), C.numel(), sb.SB_BUF_PREPARE)})
    with torch.cuda.stream(s):
        ms = best_of(run)
    res["int8_gemm_i8_tc_tops"] = round(ops / ms / 1e9, 1)
    res["int8_gemm_i8_tc_plan"] = prog.describe_plan(True).splitlines()[0]
    cands = [v for v in (res.get("int8_cublaslt_tops"), res["int8_gemm_i8_tc_tops"]) if v]
    res["int8_tops"] = max(cands)
    res["int8_how"] = (f"best of cuBLASLt torch._int_mm and gemm_i8_tc, {n}^3, best of 10 back-to-back "
                       f"calls, CUDA events, {res['when']}")
    Af = torch.randn(n, n, device="cuda")
    Bf = torch.randn(n, n, device="cuda")
    torch.backends.cuda.matmul.allow_tf32 = True
    ms = best_of(lambda: torch.matmul(Af, Bf))
    res["tf32_tflops"] = round(ops / ms / 1e9, 1)
    torch.backends.cuda.matmul.allow_tf32 = False
    ms = best_of(lambda: torch.matmul(Af, Bf), iters=3, reps=2)
    res["fp32_cublas_tflops"] = round(ops / ms / 1e9, 1)
    Ah = Af.to(torch.bfloat16)
    Bh = Bf.to(torch.bfloat16)
    ms = best_of(lambda: torch.matmul(Ah, Bh))
    res["bf16_tflops_check"] = round(ops / ms / 1e9, 1)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
