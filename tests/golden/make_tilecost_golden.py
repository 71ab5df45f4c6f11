"""Generates tests/golden/tilecost.json from the UNMODIFIED reference's tile_cost and
autotile (tile.cpp:380-535, through oracle/_ref).

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_tilecost_golden.py
Cases: seeded random tile shapes (in range and out of range, interleaved or not, several cache
lines and memory caps) on every corpus block the reference can count, the reference's own
known-answer cases (test_tile.cpp:165-260: fig6a_fixed, copy16, gen_conv 6x6x2x2) and exhaustive
autotile searches.  Each stores the program text, the block path, the arguments and the
reference's report, or its error code.  The GPU box has no /root/reference; these pin
sb_tile_cost / sb_autotile there.
"""
import json
import os
import random
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from harness import corpus  # noqa: E402
from oracle import OracleError, Ref  # noqa: E402
from paper_1903_06498_b200 import workloads as W  # noqa: E402


def ranged(text, path):
    hdrs = re.findall(r"block \[([^\]]*)\]", text)
    depth = path.count(".") + 1
    if len(hdrs) <= depth:
        return []
    return [(a.split(":")[0].strip(), int(a.split(":")[1])) for a in hdrs[depth].split(",") if ":" in a and "=" not in a]


def err_code(e):
    return str(e).split(":", 1)[0]


def tile_case(text, path, tiles, line, cap, il):
    try:
        lines, ops, elems, excl = Ref.tile_cost(text, path, tiles, line, cap, interleaved=il)
        exp = {"lines_total": lines, "useful_ops": ops, "tile_elements": elems, "excluded": excl}
    except OracleError as e:
        exp = {"error": err_code(e)}
    return {"kind": "tile_cost", "path": path, "tiles": tiles, "line": line, "mem_cap": cap, "interleaved": il,
            "expect": exp}


def auto_case(text, path, line, cap, p2):
    try:
        chosen, rep, cands, excl = Ref.autotile(text, path, line, cap, power_of_two=p2)
        exp = {"chosen": chosen, "lines_total": rep[0], "useful_ops": rep[1], "tile_elements": rep[2],
               "candidates": cands, "excluded": excl}
    except OracleError as e:
        exp = {"error": err_code(e)}
    return {"kind": "autotile", "path": path, "line": line, "mem_cap": cap, "power_of_two": p2, "expect": exp}


def main():
    rng = random.Random(1903)
    programs = {c.name: c.text for c in corpus() if "block [" in c.text}
    programs["conv_pad"] = W.conv2d(2, 9, 7, 4, 4)
    programs["conv_s2"] = W.conv2d(1, 11, 10, 4, 4, R=5, S=3, pad=2, stride=2)
    programs["pool"] = W.pool2d(2, 9, 9, 4)
    programs["mm"] = W.matmul(12, 16, 10)
    programs["conv_med"] = W.conv2d(2, 16, 16, 8, 8)
    programs["mm64"] = W.matmul(64, 64, 64)
    programs["pool_med"] = W.pool2d(2, 16, 16, 16)
    out = {"programs": programs, "cases": {}}
    for name, text in programs.items():
        cases = []
        for path in ("0", "0.0"):
            rg = ranged(text, path)
            try:
                Ref.tile_cost(text, path, "", 1, 1 << 40)
            except OracleError as e:
                if err_code(e) == "Exception":  # the shim's "bad block path": no block there
                    continue
            if not rg:
                continue
            big = name in ("conv_med", "mm64", "pool_med")
            for _ in range(0 if big else 8):
                tiles = ",".join(f"{k}:{rng.randint(1, r)}" for k, r in rg if rng.random() < 0.7)
                if rng.random() < 0.05:
                    tiles += ",zz:2"
                if rng.random() < 0.05 and rg:
                    tiles = f"{rg[0][0]}:{rg[0][1] + 1}"
                cases.append(tile_case(text, path, tiles, rng.choice([1, 2, 4, 8, 16, 32]),
                                       rng.choice([1 << 40, 50, 200, 1000]), rng.random() < 0.3))
            if big:
                cases.append(auto_case(text, path, 16, 4096, True))
                cases.append(auto_case(text, path, 32, 8192, False))
            else:
                cases.append(auto_case(text, path, rng.choice([4, 8, 16]), rng.choice([1 << 40, 100, 300]),
                                       rng.random() < 0.5))
        if cases:
            out["cases"][name] = cases
    # the reference's known answers (test_tile.cpp:165-260)
    fig = programs["fx_fig6a_fixed"]
    kat = [tile_case(fig, "0", "x:3,y:4", 8, 512, False),         # 432 elements, 200192 ops
           tile_case(fig, "0", "x:12,y:16", 8, 512, False),       # MemCap, 4608 elements
           tile_case(fig, "0", "x:12,y:16,i:3,j:3,c:8,k:16", 8, 1 << 20, False),
           auto_case(fig, "0", 8, 512, True),                      # 1600 power-of-two candidates
           auto_case(fig, "0", 8, 512, False)]                     # acceptance crit5 argmin
    copy = programs["fx_copy16"]
    kat += [auto_case(copy, "0", 8, 8, False), auto_case(copy, "0", 8, 1, False),
            tile_case(copy, "0", "i:17", 8, 8, False), tile_case(copy, "0", "q:2", 8, 8, False)]
    conv = Ref.gen("conv", 6, 6, 2, 2, 32)
    out["programs"]["gen_conv_6x6x2x2"] = conv
    kat += [auto_case(conv, "0", 8, 1 << 20, False)]
    out["cases"]["kat_fig6a_fixed"] = kat[:5]
    out["cases"]["kat_copy16"] = kat[5:9]
    out["cases"]["kat_gen_conv_6x6x2x2"] = kat[9:]
    for k in ("kat_fig6a_fixed", "kat_copy16", "kat_gen_conv_6x6x2x2"):
        for c in out["cases"][k]:
            c["program"] = {"kat_fig6a_fixed": "fx_fig6a_fixed", "kat_copy16": "fx_copy16"}.get(k, "gen_conv_6x6x2x2")
    with open(os.path.join(HERE, "tilecost.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    n = sum(len(v) for v in out["cases"].values())
    print("wrote", n, "cases")


if __name__ == "__main__":
    main()
