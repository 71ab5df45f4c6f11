"""Parser/printer parity: the executor's front end reads every program the
reference prints, and prints it back byte-identically (text.cpp:453-567)."""
import pytest

import paper_1903_06498_b200 as sb
from harness import corpus
from oracle import OracleError, Port, Ref


@pytest.mark.parametrize("case", corpus(), ids=lambda c: c.name)
def test_roundtrip_golden(case):
    assert sb.print_program(sb.parse_program(case.text)) == case.text


def test_buffer_table():
    p = sb.parse_program("block [] ( in A[0, 0] i8(3, 4):(4, 1) out B[0]:add i32(5):(-2) ) {}")
    assert p.buffers["A"].elements == 12 and p.buffers["A"].dtype == 8
    assert p.buffers["B"].elements == 9 and p.buffers["B"].dir == sb.Dir.Out


BAD = [
    "block [x:1, y=x] () {}",              # alias at root refers to nothing
    "block [x:1] ( x + >= 0 ) {}",
    "block [] ( in A[0] i32(1):(1) in A[0] i32(1):(1) ) {}",
    "block [] ( in A[0]:add i32(1):(1) ) {}",
    "block [] () { $a = load(Q) }",
    "block [] ( x >= 0 ) {}",
    "block [x:2] ( x >= 1 ) {}",
    "block [] () {} trailing",
    "block [] ( in A[0] i32(1, 2):(1) ) {}",
    "block [] ( #tag in A[0] i32(1):(1) #t2 ) {}",
    "block [y=1, x:2] () {}",
]


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("text", BAD)
def test_error_codes_match_reference(text):
    try:
        Ref.parse(text)
        ref_code = None
    except OracleError as e:
        ref_code = e.code
    try:
        sb.parse_program(text)
        my_code = None
    except sb.ExecError as e:
        my_code = e.code
    assert my_code == ref_code


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_random_text_programs_roundtrip():
    state = 5
    for i in range(100):
        text, state = Ref.gen_random(state, text_variant=True)
        assert sb.print_program(sb.parse_program(text)) == text
        assert Port.print(text) == text
