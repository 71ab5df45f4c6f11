"""tile_cost / autotile (tile.cpp:380-535) with every candidate's line
counts on the device (sb_tile_cost / sb_autotile), against the reference.

Fixtures: tests/golden/tilecost.json, made by the UNMODIFIED reference
(tests/golden/make_tilecost_golden.py): seeded random tile shapes over the golden corpus,
the reference's own known answers (test_tile.cpp:165-260, acceptance.cpp:318-400) and
exhaustive searches.  Bit-exact: line totals, useful ops, footprints, exclusions, the chosen
shape, candidate/excluded counts and error codes."""
import json
import os
import time

import pytest

from harness import gpu_available
from oracle import Ref

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "tilecost.json")) as _f:
    GOLD = json.load(_f)


def _cases(kind=None):
    for group, cases in sorted(GOLD["cases"].items()):
        for i, c in enumerate(cases):
            if kind is None or c["kind"] == kind:
                yield group, i, c


def _program(group, c):
    return GOLD["programs"][c.get("program", group)]


# ---- CPU: the fixtures themselves ------------------------------------------------------------

def test_known_answers_from_reference_tests():
    """test_tile.cpp:165-260 as literal values."""
    kat = GOLD["cases"]["kat_fig6a_fixed"]
    assert kat[0]["expect"]["tile_elements"] == 432 and not kat[0]["expect"]["excluded"]
    assert kat[0]["expect"]["useful_ops"] == 200192
    assert kat[1]["expect"]["excluded"] and kat[1]["expect"]["tile_elements"] == 4608
    assert kat[3]["expect"]["candidates"] == 4 * 5 * 2 * 2 * 4 * 5
    assert all((int(t.split(":")[1]) & (int(t.split(":")[1]) - 1)) == 0
               for t in kat[3]["expect"]["chosen"].split(","))
    copy = GOLD["cases"]["kat_copy16"]
    assert copy[0]["expect"]["chosen"] in ("i:4", "i:8")
    assert copy[1]["expect"]["chosen"] is None and copy[1]["expect"]["excluded"] == 5
    assert copy[2]["expect"]["error"] == copy[3]["expect"]["error"] == "InvalidTile"
    conv = GOLD["cases"]["kat_gen_conv_6x6x2x2"][0]["expect"]
    assert conv["chosen"] == "c:2,i:3,j:3,k:2,x:6,y:6"  # identity-shaped tiling wins


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_fixtures_pinned_against_reference():
    """Re-derive every cheap fixture from the reference (the generator's output is what the
    unmodified reference says today)."""
    checked = 0
    for group, i, c in _cases("tile_cost"):
        if group in ("conv_med", "mm64", "pool_med"):
            continue
        text = _program(group, c)
        try:
            got = Ref.tile_cost(text, c["path"], c["tiles"], c["line"], c["mem_cap"], interleaved=c["interleaved"])
            got = {"lines_total": got[0], "useful_ops": got[1], "tile_elements": got[2], "excluded": got[3]}
        except Exception as e:  # noqa: BLE001
            got = {"error": str(e).split(":", 1)[0]}
        assert got == c["expect"], (group, i)
        checked += 1
    assert checked > 500


# ---- B200 ----------------------------------------------------------------------------------

def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def _device_tile_cost(sb, text, c):
    prog = sb.parse_program(text)
    try:
        r = prog.tile_cost(c["path"], c["tiles"], c["line"], c["mem_cap"], interleaved=c["interleaved"])
        return {"lines_total": r.lines_total, "useful_ops": r.useful_ops, "tile_elements": r.tile_elements,
                "excluded": r.excluded is not None}
    except sb.ExecError as e:
        return {"error": e.code}


def _device_autotile(sb, text, c):
    prog = sb.parse_program(text)
    try:
        r = prog.autotile(c["path"], c["line"], c["mem_cap"], power_of_two=c["power_of_two"])
        return {"chosen": r.chosen, "lines_total": r.report.lines_total, "useful_ops": r.report.useful_ops,
                "tile_elements": r.report.tile_elements, "candidates": r.candidates, "excluded": r.excluded}
    except sb.ExecError as e:
        return {"error": e.code}


@pytest.mark.gpu
def test_tile_cost_matches_reference_fixtures():
    _need_gpu()
    import paper_1903_06498_b200 as sb
    n = 0
    for group, i, c in _cases("tile_cost"):
        assert _device_tile_cost(sb, _program(group, c), c) == c["expect"], (group, i, c)
        n += 1
    assert n > 600


@pytest.mark.gpu
def test_autotile_matches_reference_fixtures():
    _need_gpu()
    import paper_1903_06498_b200 as sb
    n = 0
    for group, i, c in _cases("autotile"):
        assert _device_autotile(sb, _program(group, c), c) == c["expect"], (group, i, c)
        n += 1
    assert n > 80


@pytest.mark.gpu
def test_wide_tiles_take_the_global_scratch_path():
    """Tiles spanning more than the shared-memory q slots (12288 lines) count in global
    scratch: a 1-element cache line over a 128x128 matmul tile of a 1024-wide B."""
    _need_gpu()
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.matmul(256, 1024, 128)
    ops = 256 * 1024 * 128
    for tiles, line in (("m:128,n:1024,k:128", 1), ("m:64,n:512,k:128", 2), ("m:256,n:1024,k:64", 3)):
        exp = Ref.tile_cost(text, "0", tiles, line, 1 << 40, hint=ops) if Ref.available() else None
        r = sb.parse_program(text).tile_cost("0", tiles, line, 1 << 40)
        if exp is not None:
            assert r.as_tuple() == exp, tiles


@pytest.mark.gpu
def test_autotile_config2_scale():
    """The C2 conv block (32x56x56, 3x3, 64->64; 7 indexes) searched over every
    power-of-two candidate, which the reference cannot do (§0.7): the device finishes it, and
    the chosen shape's report equals the reference's tile_cost for that shape."""
    _need_gpu()
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.conv2d(32, 56, 56, 64, 64)
    prog = sb.parse_program(text)
    t0 = time.perf_counter()
    res = prog.autotile("0", 16, 1 << 16, power_of_two=True)
    dt = time.perf_counter() - t0
    print(f"C2 autotile: {res.candidates} candidates ({res.excluded} over the cap) in {dt:.2f} s, "
          f"chose {res.chosen}, lines {res.report.lines_total}")
    assert res.candidates == 6 * 6 * 6 * 2 * 2 * 7 * 7
    assert res.chosen is not None and res.report.useful_ops == W.conv_useful_macs(32, 56, 56, 64, 64)
    if Ref.available():
        exp = Ref.tile_cost(text, "0", res.chosen, 16, 1 << 16, hint=res.report.useful_ops)
        assert res.report.as_tuple() == exp
