"""The drop-in boundary: the C-ABI library loads and exports every symbol that
include/stripe_b200.h declares; status codes mirror the reference's codes."""
import os
import re

import pytest

import paper_1903_06498_b200 as sb

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "stripe_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sb_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_exported_list():
    assert declared() == sorted(sb.EXPORTED)


@pytest.mark.parametrize("sym", declared())
def test_symbol_exported(sym):
    assert hasattr(sb.lib(), sym), sym


def test_status_names_match_reference_codes():
    L = sb.lib()
    assert L.sb_abi_version() == 1
    names = [L.sb_status_name(i).decode() for i in range(14)]
    assert names == sb.STATUS_NAMES
    for code in ["MissingBuffer", "UnknownIntrinsic", "UnknownSpecial", "UndefinedTemp", "OutOfBoundsAccess",
                 "UnboundIndex", "SyntaxError", "ScopeError"]:
        assert code in names


def test_parse_errors_have_reference_codes():
    with pytest.raises(sb.ExecError) as e:
        sb.parse_program("block [x:0] () {}")
    assert e.value.code == "SyntaxError"
    with pytest.raises(sb.ExecError) as e:
        sb.parse_program("block [] ( in A[q] i32(1):(1) ) {}")
    assert e.value.code == "ScopeError"
    with pytest.raises(sb.ExecError) as e:
        sb.parse_program("block [] ( in A[0] f64(1):(1) ) {}")
    assert e.value.code == "SyntaxError"


def test_no_cpu_fallback_without_gpu():
    from harness import gpu_available
    if gpu_available():
        pytest.skip("GPU present")
    with pytest.raises(sb.ExecError) as e:
        sb.Context(0)
    assert e.value.code == "CudaError"
