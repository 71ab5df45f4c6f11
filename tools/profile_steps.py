#!/usr/bin/env python
"""Per-plan-step device times of one program (SB_PROFILE_STEPS tracing aid).

    SB_PROFILE_STEPS=1 python tools/profile_steps.py c5 [batch]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def program_text(which, batch):
    from paper_1903_06498_b200 import workloads as W
    if which == "c5":
        text, _ = W.resnet50(batch)
    elif which == "stem":
        text = W.conv_fused(batch, 224, 224, 3, 64, 7, 7, 2, 3)
    elif which == "l3x3":
        text = W.conv_fused(batch, 56, 56, 64, 64, 3, 3, 1, 1)
    elif which == "s3_3x3":
        text = W.conv_fused(batch, 14, 14, 256, 256, 3, 3, 1, 1)
    elif which == "s3_1024":
        text = W.conv_fused(batch, 14, 14, 1024, 256, 1, 1, 1, 0)
    elif which == "l44":
        text = W.conv_fused(batch, 14, 14, 1024, 512, 1, 1, 1, 0)
    elif which == "l43":
        text = W.conv_fused(batch, 14, 14, 1024, 2048, 1, 1, 2, 0, relu=False)
    elif which == "l47":
        text = W.conv_fused(batch, 7, 7, 2048, 512, 1, 1, 1, 0)
    elif which == "s4_3x3":
        text = W.conv_fused(batch, 7, 7, 512, 512, 3, 3, 1, 1)
    elif which == "s4_1x1":
        text = W.conv_fused(batch, 7, 7, 512, 2048, 1, 1, 1, 0, residual=True)
    elif which == "s3_1x1":
        text = W.conv_fused(batch, 14, 14, 256, 1024, 1, 1, 1, 0, residual=True)
    elif which == "s2_3x3":
        text = W.conv_fused(batch, 28, 28, 128, 128, 3, 3, 1, 1)
    elif which == "l24":
        text = W.conv_fused(batch, 28, 28, 512, 1024, 1, 1, 2, 0, relu=False)
    elif which == "l25":
        text = W.conv_fused(batch, 28, 28, 512, 256, 1, 1, 1, 0)
    elif which == "l11":
        text = W.conv_fused(batch, 56, 56, 256, 512, 1, 1, 2, 0, relu=False)
    elif which == "s2_1x1":
        text = W.conv_fused(batch, 28, 28, 128, 512, 1, 1, 1, 0, residual=True)
    elif which == "l1x1r":
        text = W.conv_fused(batch, 56, 56, 64, 256, 1, 1, 1, 0, residual=True)
    elif which == "l1x1p":
        text = W.conv_fused(batch, 56, 56, 64, 256, 1, 1, 1, 0, relu=False)
    elif which == "pool":
        text = W.pool2d(batch, 112, 112, 64)
    elif which == "l1x1":
        text = W.conv_fused(batch, 56, 56, 64, 64, 1, 1, 1, 0)
    elif which == "c4a":
        text = W.maxpool2x2(batch, 112, 112, 64)
    elif which == "c4b":
        text = W.global_sum(batch, 7, 7, 2048)
    elif which == "gsum_i8":  # C5's global sum (7x7, 2048 channels, i8)
        text = W.global_sum(batch, 7, 7, 2048, in_dtype="i8", out_dtype="i8")
    elif which == "c2":
        text = W.conv2d(32, 56, 56, 64, 64)
    else:
        raise SystemExit("unknown program " + which)
    return text


def main():
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    which = sys.argv[1] if len(sys.argv) > 1 else "c5"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    text = program_text(which, batch)
    prog = sb.parse_program(text)
    ctx = sb.Context(0)
    bufs, keep = {}, []
    for bn, d in prog.buffers.items():
        nbytes = d.elements * {8: 1, 16: 2, 32: 4}[d.dtype]
        t = torch.randint(-128, 128, (nbytes,), dtype=torch.int8, device="cuda")
        keep.append(t)
        bufs[bn] = (t.data_ptr(), d.elements, sb.SB_BUF_PREPARE if int(d.dir) != 0 else 0)
    run = ctx.bind_device(prog, bufs)
    for _ in range(3):
        print("---- run", flush=True)
        sys.stderr.flush()
        run()
        ctx.sync()


if __name__ == "__main__":
    main()
