"""Generates tests/golden/*.npz from the UNMODIFIED reference interpreter.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
Each case stores the canonical program text (the reference's print_program),
the input store (reference random_inputs / test_interp.cpp KAT inputs) and the
reference's outputs after execute(), or the reference's error code.  The GPU
box has no /root/reference; these fixtures pin the oracle and the executor
there.
"""
import glob
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import OracleError, Ref  # noqa: E402

TESTDATA = "/root/reference/proj/testdata"

CONV_RELU_HWCFG = """mem SRAM cap=2048 line=8 banks=1
pass autotile unit=SRAM tiles=x:3,y:4 block=0.0
pass autotile unit=SRAM tiles=x:3,y:4 block=0.1
pass fuse block=0 i=0 j=1
pass localize
pass scalarize
pass schedule unit=SRAM
"""


def save(name, text, store, note=""):
    prog = Ref.parse(text)
    bufs = prog.buffers()
    arrays = {}
    for n, (bits, arr) in store.items():
        arrays[f"in_{n}"] = arr
        arrays[f"bits_{n}"] = np.array(bits)
    try:
        out = Ref.execute(prog, store)
        err = ""
        for n, (bits, arr) in out.items():
            arrays[f"out_{n}"] = arr
    except OracleError as e:
        err = str(e)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), text=np.array(prog.text()), error=np.array(err),
                        note=np.array(note), order=np.array([b[0] for b in bufs]), **arrays)
    return err


SCATTER = """block []:1 (
	in SRC[0, 0] {dt}(12, 4):(4, 1)
	in IDX[0, 0] i32(12, 4):(4, 1)
	out DST[0, 0]:assign {dt}(8, 4):(4, 1)
) {{
	0:
	block []:1 (
		in SRC[0, 0] {dt}(12, 4):(4, 1)
		in IDX[0, 0] i32(12, 4):(4, 1)
		out DST[0, 0]:{agg} {dt}(8, 4):(4, 1)
	) {{
		0: special scatter(DST, SRC, IDX)
	}}
}}
"""

LOCAL_GATHER = """block []:1 (
	in SRC[0, 0] i32(8, 4):(4, 1)
	in IDX[0, 0] i32(6, 4):(4, 1)
	out DST[0, 0]:assign i32(6, 4):(4, 1)
) {
	0:
	block [i:6]:6 (
		in SRC[0, 0] i32(8, 4):(4, 1)
		in IDX[i, 0] i32(1, 4):(4, 1)
		inout T[0, 0]:assign i32(1, 4):(4, 1)
		out DST[i, 0]:assign i32(1, 4):(4, 1)
	) {
		0: special gather(T, SRC, IDX)
		1: $t = load(T)
		2: DST = store($t)
	}
}
"""

LOCAL_SCATTER = """block []:1 (
	in A[0, 0] i32(6, 4):(4, 1)
	in IDX[0, 0] i32(6, 4):(4, 1)
	out DST[0, 0]:assign i32(8, 4):(4, 1)
) {
	0:
	block [i:6]:6 (
		in A[i, 0] i32(1, 4):(4, 1)
		in IDX[i, 0] i32(1, 4):(4, 1)
		inout T[0, 0]:assign i32(1, 4):(4, 1)
		out DST[0, 0]:add i32(8, 4):(4, 1)
	) {
		0: $a = load(A)
		1: $b = mul($a, 3)
		2: T = store($b)
		3: special scatter(DST, T, IDX)
	}
}
"""


def special_cases():
    """gather/scatter specials the reference runs (interp.cpp:540-600): scatter with add /
    assign (last writer in lexicographic order) / max aggregation, with index collisions, an
    i8 scatter-add that wraps (ir.cpp:79-97), an out-of-range index (OutOfBoundsAccess), and
    specials whose operand is a block-local allocation (interp.cpp:433-447)."""
    from oracle import Rng, wrap
    rng = Rng(4242)
    idx = (rng.bulk(48) % np.uint64(8)).astype(np.int64)  # 12 x 4 indexes into 8 rows: collisions
    for agg, dt, bits in [("add", "i32", 32), ("assign", "i32", 32), ("max", "i32", 32), ("add", "i8", 8),
                          ("min", "i16", 16)]:
        text = SCATTER.format(dt=dt, agg=agg)
        src = wrap(bits, rng.bulk(48))
        dst = wrap(bits, rng.bulk(32))
        save(f"kat_scatter_{agg}_{dt}", text, {"SRC": (bits, src), "IDX": (32, idx), "DST": (bits, dst)},
             f"scatter {agg} {dt} with index collisions (interp.cpp:578-590)")
    bad = idx.copy()
    bad[13] = 8
    save("kat_scatter_oob", SCATTER.format(dt="i32", agg="add"),
         {"SRC": (32, wrap(32, rng.bulk(48))), "IDX": (32, bad), "DST": (32, np.zeros(32, np.int64))},
         "scatter index outside [0, 8) -> OutOfBoundsAccess (interp.cpp:578-582)")
    save("kat_gather_local", LOCAL_GATHER, {"SRC": (32, 100 + np.arange(32, dtype=np.int64)),
                                            "IDX": (32, (rng.bulk(24) % np.uint64(8)).astype(np.int64)),
                                            "DST": (32, wrap(32, rng.bulk(24)))},
         "gather into a per-point local allocation")
    save("kat_scatter_local", LOCAL_SCATTER, {"A": (32, wrap(32, rng.bulk(24))),
                                              "IDX": (32, (rng.bulk(24) % np.uint64(8)).astype(np.int64)),
                                              "DST": (32, wrap(32, rng.bulk(32)))},
         "scatter-add from a per-point local allocation")


def main():
    if "--only-specials" in sys.argv:
        special_cases()
        return
    for f in glob.glob(os.path.join(HERE, "*.npz")):
        os.remove(f)
    n = 0
    # 1. every reference fixture with seeded random inputs (support.h:55-70)
    for f in sorted(glob.glob(os.path.join(TESTDATA, "*.stripe"))):
        base = os.path.basename(f)[:-7]
        prog = Ref.parse(open(f).read())
        save(f"fx_{base}", prog.text(), Ref.random_inputs(prog, 7), f"fixture {base}, seed 7")
        n += 1
    # 2. test_interp.cpp known-answer cases
    t = Ref.parse(open(os.path.join(TESTDATA, "fig6a_fixed_i32.stripe")).read()).text()
    save("kat_ones_conv", t, {"I": (32, np.ones(12 * 16 * 8, np.int64)), "F": (32, np.ones(3 * 3 * 16 * 8, np.int64)),
                              "O": (32, np.zeros(12 * 16 * 16, np.int64))}, "test_interp.cpp:88-102")
    empty = ("block []:1 (\n\tout B[0]:assign i32(4):(1)\n) {\n\tblock [i:4] (\n\t\t-1 >= 0\n"
             "\t\tout B[i]:assign i32(1):(1)\n\t) {\n\t\t$c = constant(9)\n\t\tB = store($c)\n\t}\n}\n")
    save("kat_empty_space", empty, {"B": (32, np.array([1, 2, 3, 4], np.int64))}, "test_interp.cpp:104-121")
    oob = ("block []:1 (\n\tin A[0] i32(4):(1)\n\tout B[0]:assign i32(4):(1)\n) {\n\tblock [i:4] (\n"
           "\t\tin A[i + 1] i32(1):(1)\n\t\tout B[i]:assign i32(1):(1)\n\t) {\n\t\t$a = load(A)\n"
           "\t\tB = store($a)\n\t}\n}\n")
    save("kat_oob", oob, {"A": (32, np.array([1, 2, 3, 4], np.int64)), "B": (32, np.zeros(4, np.int64))},
         "test_interp.cpp:217-236")
    bad = "block [] ( in A[0] i32(1):(1) out B[0]:assign i32(1):(1) ) { $a = frobnicate() }"
    save("kat_unknown_intrinsic", bad, {"A": (32, np.array([1], np.int64)), "B": (32, np.array([0], np.int64))},
         "test_interp.cpp:208-214")
    g = Ref.parse(open(os.path.join(TESTDATA, "gather.stripe")).read()).text()
    idx = np.array([[7 - r] * 4 for r in range(8)], np.int64).ravel()
    save("kat_gather", g, {"SRC": (32, 100 + np.arange(32, dtype=np.int64)), "IDX": (32, idx),
                           "DST": (32, np.zeros(32, np.int64))}, "test_interp.cpp:179-198")
    idx_bad = idx.copy()
    idx_bad[0] = 8
    save("kat_gather_oob", g, {"SRC": (32, 100 + np.arange(32, dtype=np.int64)), "IDX": (32, idx_bad),
                               "DST": (32, np.zeros(32, np.int64))}, "test_interp.cpp:195-197")
    # 3. generator oracle-equivalence cases (test_interp.cpp:123-133, seed 31)
    from oracle import Rng  # noqa
    for name, args, bits in [("matmul", (9, 7, 5, 0), 32), ("conv", (8, 6, 3, 4), 32), ("maxpool", (8, 6, 3, 0), 32),
                             ("matmul", (6, 6, 6, 0), 8), ("conv", (10, 12, 16, 32), 8), ("matmul", (33, 17, 40, 0), 16)]:
        text = Ref.gen(name, *args, bits=bits)
        prog = Ref.parse(text)
        save(f"gen_{name}_{'x'.join(map(str, args))}_i{bits}", text, Ref.random_inputs(prog, 31), "generator")
    # 4. random programs (acceptance.cpp:293-315 generator; seeds from 1002)
    state = 1002
    for i in range(24):
        text, state = Ref.gen_random(state, text_variant=False)
        save(f"rnd_prog_{i:02d}", text, Ref.random_inputs(Ref.parse(text), 1000 + i), "gen_random_program")
    state = 2024
    for i in range(24):
        text, state = Ref.gen_random(state, text_variant=True)
        save(f"rnd_text_{i:02d}", text, Ref.random_inputs(Ref.parse(text), 3000 + i), "gen_random_text_program")
    # 5. pass-pipeline shapes (tile_rewrite, fuse/localize/scalarize)
    mm = Ref.gen("matmul", 32, 24, 20, bits=32)
    for tiles in ["m:8,n:8,k:4", "m:5,n:7,k:3", "k:20"]:
        tt = Ref.tile_rewrite(mm, "0", tiles)
        save("tile_matmul_" + tiles.replace(":", "").replace(",", "_"), tt, Ref.random_inputs(Ref.parse(tt), 5), tiles)
    cv = Ref.gen("conv", 12, 10, 4, 6, bits=8)
    tt = Ref.tile_rewrite(cv, "0", "x:3,y:4")
    save("tile_conv_x3y4", tt, Ref.random_inputs(Ref.parse(tt), 6), "conv tiled x:3,y:4")
    cr = open(os.path.join(TESTDATA, "conv_relu.stripe")).read()
    fused = Ref.pipeline(cr, CONV_RELU_HWCFG)
    save("pipe_conv_relu_fused", fused, Ref.random_inputs(Ref.parse(fused), 32), "test_passes.cpp:357-379")
    special_cases()
    print("wrote", len(glob.glob(os.path.join(HERE, "*.npz"))), "cases")


if __name__ == "__main__":
    main()
