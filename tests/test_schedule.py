"""Statement-DAG lanes (csrc/schedule.cpp) and the scratch arena, checked from the plan
description (host only): independent statements go to different lanes, dependent ones
stay ordered, arena reuse follows live intervals."""
import re

import paper_1903_06498_b200 as sb


def two_independent(n=4096):
    return f"""block []:1 (
\tin A[0] i32({n}):(1)
\tout X[0]:assign i32({n}):(1)
\tout Y[0]:assign i32({n}):(1)
) {{
\t0:
\tblock [i:{n}]:{n} (
\t\tin A[i] i32(1):(1)
\t\tout X[i]:assign i32(1):(1)
\t) {{
\t\t0: $a = load(A)
\t\t1: X = store($a)
\t}}
\t1:
\tblock [i:{n}]:{n} (
\t\tin A[i] i32(1):(1)
\t\tout Y[i]:assign i32(1):(1)
\t) {{
\t\t0: $a = load(A)
\t\t1: $b = add($a, 1)
\t\t2: Y = store($b)
\t}}
}}
"""


def lanes_of(plan):
    m = re.search(r"^lanes (\d+):(.*)$", plan, re.M)
    return (int(m.group(1)), [int(x) for x in m.group(2).split()]) if m else (1, [])


def test_independent_statements_get_two_lanes():
    n, lanes = lanes_of(sb.parse_program(two_independent()).describe_plan())
    assert n == 2 and sorted(set(lanes)) == [0, 1]


def test_chain_keeps_one_lane():
    text = two_independent().replace("in A[i] i32(1):(1)\n\t\tout Y[i]", "in X[i] i32(1):(1)\n\t\tout Y[i]").replace(
        "\t\t0: $a = load(A)\n\t\t1: $b = add", "\t\t0: $a = load(X)\n\t\t1: $b = add").replace(
        "\tout Y[0]:assign i32(4096):(1)", "\tout Y[0]:assign i32(4096):(1)")
    # statement 1 reads X written by statement 0 (the root keeps X as an out buffer)
    text = text.replace("\t1:\n\tblock [i:4096]:4096 (\n\t\tin A[i]", "\t1:\n\tblock [i:4096]:4096 (\n\t\tin X[i]")
    n, _ = lanes_of(sb.parse_program(text).describe_plan())
    assert n == 1


def test_resnet_arena_reuse():
    from paper_1903_06498_b200 import workloads as W
    text, info = W.resnet50(4)
    plan = sb.parse_program(text).describe_plan()
    arena = int(re.search(r"^arena (\d+) bytes", plan, re.M).group(1))
    # every activation materialised separately would need sum of all locals; reuse keeps a
    # small multiple of the largest layer
    largest = 4 * 112 * 112 * 64  # stem output, i8
    assert 0 < arena < 12 * largest, arena
