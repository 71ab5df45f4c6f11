"""The oracle pinned against the reference: golden vectors (tests/golden, made
by the unmodified reference) and, where oracle/_ref is built, live differential
runs over the reference's own generators."""
import numpy as np
import pytest

from harness import corpus
from oracle import OracleError, Port, Ref, Rng, random_inputs, wrap

CASES = corpus()


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
def test_port_matches_golden(case):
    store = {n: arr for n, (bits, arr) in case.inputs.items()}
    if case.error:
        with pytest.raises(OracleError) as e:
            Port.execute(case.text, store)
        assert e.value.code == case.error.split(":")[0]
        return
    out = Port.execute(case.text, store)
    for n, exp in case.expected.items():
        np.testing.assert_array_equal(out[n], exp, err_msg=f"{case.name}:{n}")


def test_golden_kats():
    """Frozen values of test_interp.cpp:88-102 / 104-121 / 179-198 / test_ir.cpp:19-28."""
    c = {x.name: x for x in CASES}
    o = c["kat_ones_conv"].expected["O"]
    assert o[5 * 16 * 16 + 7 * 16 + 3] == 72 and o[0] == 32 and o[7 * 16] == 48
    assert list(c["kat_empty_space"].expected["B"]) == [1, 2, 3, 4]
    dst = c["kat_gather"].expected["DST"].reshape(8, 4)
    for r in range(8):
        for col in range(4):
            assert dst[r, col] == 100 + (7 - r) * 4 + col
    assert c["kat_gather_oob"].error.startswith("OutOfBoundsAccess")
    assert c["kat_oob"].error.startswith("OutOfBoundsAccess")
    assert c["kat_unknown_intrinsic"].error.startswith("UnknownIntrinsic")
    # wrap / aggregation KATs (ir.cpp:39-97; test_ir.cpp:11-28)
    assert list(wrap(8, np.array([127, 128, 256], dtype=np.int64))) == [127, -128, 0]
    assert wrap(16, np.array([-32769]))[0] == 32767


def test_numpy_rng_matches_splitmix():
    r = Rng(1234)
    scalar = [r.next() for _ in range(50)]
    r2 = Rng(1234)
    assert [int(x) for x in r2.bulk(50)] == scalar


ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built (needs /root/reference)")


@ref
def test_random_inputs_matches_reference():
    for name, args, bits in [("matmul", (5, 6, 7), 8), ("conv", (6, 5, 3, 2), 16), ("maxpool", (8, 6, 3), 32)]:
        prog = Ref.parse(Ref.gen(name, *args, bits=bits))
        ref_store = Ref.random_inputs(prog, 99)
        mine = random_inputs(prog.buffers(), 99)
        for n, arr in mine.items():
            np.testing.assert_array_equal(arr, ref_store[n][1])


@ref
def test_port_matches_reference_random_programs():
    """acceptance.cpp:293-315 style: random generated programs, port == reference."""
    state = 77
    for i in range(60):
        text, state = Ref.gen_random(state, text_variant=bool(i % 2))
        prog = Ref.parse(text)
        st = Ref.random_inputs(prog, i)
        exp = Ref.execute(prog, st)
        got = Port.execute(text, {n: a for n, (b, a) in st.items()})
        for n in exp:
            np.testing.assert_array_equal(got[n], exp[n][1])


@ref
def test_port_reversed_order_matches():
    """test_interp.cpp:151-168: iteration order does not change legal results."""
    for c in CASES:
        if c.error or not c.name.startswith("fx_") or "accum_rw" in c.name:
            continue
        st = {n: a for n, (b, a) in c.inputs.items()}
        a = Port.execute(c.text, st, order=0)
        b = Port.execute(c.text, st, order=1)
        for n in a:
            np.testing.assert_array_equal(a[n], b[n])
