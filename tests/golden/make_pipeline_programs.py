"""Config programs as the reference's own passes produce them.

configs/c3_pipeline_b{N}.stripe -- config 3:

Runs the UNMODIFIED reference passes (oracle/_ref) on the config-3 program before fusion
(workloads.conv_relu_prefuse: conv_relu.stripe's structure at batch 128, 56x56x64->64, i8 in,
i32 accumulator, a bias in the ReLU block), following test_passes.cpp:357-379:
tile both kernels per (image, 2-row band) with tile_rewrite (the pinned-tile form of
`pass autotile tiles=...`, tile.cpp:477-483 -- the autotile search itself evaluates
count_valid_points per candidate and does not finish at this size), then
`fuse block=0 i=0 j=1`, `localize`, `scalarize` through apply_pipeline.  The resulting
program text is committed (c3_pipeline_b{N}.stripe) because /root/reference is not on the
GPU box.

configs/c2_partition_n8.stripe -- config 2 after `pass partition block=0 index=n n=8`
(tile.cpp:644-691): the batch index split into 8 disjoint banks (Location.bank = n), the
reference's own work-splitting construct and the multi-GPU shard carrier.

configs/c1_autotiled_{i8,i32}.stripe -- config 1 "as one autotiled Stripe block": the 1024^3
matmul block tiled by the reference's tile_rewrite with the shape the DEVICE autotile search
chose (configs/c1_autotile.json, written on a B200 by tools/c1_autotile.py: sb_autotile over
all 1331 divisor candidates under configs/b200_matmul.hwcfg's SMEM model, 128-element lines,
cap 232448 elements; the reference's own search does not finish at this size).

    python tests/golden/make_pipeline_programs.py [N ...]
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref  # noqa: E402
from paper_1903_06498_b200 import workloads as W  # noqa: E402

PASSES = """mem SRAM cap=1048576 line=64 banks=1
pass fuse block=0 i=0 j=1
pass localize
pass scalarize
"""


def make(N, H=56, C=64, K=64):
    t = W.conv_relu_prefuse(N, H, H, C, K)
    t = Ref.tile_rewrite(t, "0.0", "n:1,x:2")
    t = Ref.tile_rewrite(t, "0.1", "n:1,x:2")
    return Ref.pipeline(t, PASSES)


CONFIGS = os.path.join(os.path.dirname(os.path.dirname(HERE)), "configs")

PARTITION = """mem HBM cap=1073741824 line=128 banks=8
pass partition block=0 index=n n=8 unit=HBM
"""


if __name__ == "__main__":
    for n in [int(a) for a in sys.argv[1:]] or [128, 2]:
        with open(os.path.join(CONFIGS, f"c3_pipeline_b{n}.stripe"), "w") as f:
            f.write(make(n))
        print("wrote c3", n)
    with open(os.path.join(CONFIGS, "c1_autotile.json")) as f:
        chosen = json.load(f)
    for dt in ("i8", "i32"):
        text = Ref.tile_rewrite(W.matmul(1024, 1024, 1024, in_dtype=dt, out_dtype="i32"), "0", chosen[dt]["chosen"])
        with open(os.path.join(CONFIGS, f"c1_autotiled_{dt}.stripe"), "w") as f:
            f.write(text)
        print("wrote c1 autotiled", dt, chosen[dt]["chosen"])
    for n in (32, 8):
        with open(os.path.join(CONFIGS, f"c2_partition_n8_b{n}.stripe"), "w") as f:
            f.write(Ref.pipeline(W.conv2d(n, 56, 56, 64, 64), PARTITION))
        print("wrote c2 partition", n)
