#!/usr/bin/env python
"""Config 1 "as one autotiled Stripe block" (BASELINE config 1): the device
autotile search (sb_autotile: tile.cpp:475-535 with every candidate's lines on the B200) over
the 1024^3 matmul block under the B200 SMEM model of configs/b200_matmul.hwcfg (128-element
lines, cap 232448 elements).  Writes the chosen shape and the search statistics as JSON; the
reference's own tile_rewrite then turns it into configs/c1_autotiled_*.stripe
(tests/golden/make_pipeline_programs.py)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    out = {}
    for dt in ("i8", "i32"):
        prog = sb.parse_program(W.matmul(1024, 1024, 1024, in_dtype=dt, out_dtype="i32"))
        t0 = time.perf_counter()
        r = prog.autotile("0", 128, 232448)
        dt_s = time.perf_counter() - t0
        out[dt] = {"chosen": r.chosen, "lines_total": r.report.lines_total, "useful_ops": r.report.useful_ops,
                   "tile_elements": r.report.tile_elements, "candidates": r.candidates, "excluded": r.excluded,
                   "seconds": round(dt_s, 3), "line": 128, "mem_cap": 232448}
        print(dt, out[dt], flush=True)
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "c1_autotile.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
