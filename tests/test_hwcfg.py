"""B200 hardware configs for the reference's KEPT pass pipeline
(configs/b200_*.hwcfg: HBM + 227 KB SMEM with 128-byte lines, the tcgen05 UMMA tile as a
stencil unit).  The reference's autotile/stencil/scalarize/schedule passes tile the program
(oracle: the unmodified pipeline, passes.cpp:905-1000); the executor's dimension merging maps
the tiled nest back onto ONE tensor-core launch, bit-exact vs the reference."""
import os

import numpy as np
import pytest

from harness import gpu_available, run_device
from oracle import Ref, random_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cfg(name):
    with open(os.path.join(ROOT, "configs", name)) as f:
        return f.read()


def cases():
    from paper_1903_06498_b200 import workloads as W
    return [
        ("matmul_i8", W.matmul(256, 256, 256, in_dtype="i8", out_dtype="i32"), "b200_matmul.hwcfg", "gemm_i8_tc"),
        ("matmul_i32", W.matmul(128, 256, 128, in_dtype="i32", out_dtype="i32"), "b200_matmul.hwcfg", "gemm_i8_tc"),
        ("conv", W.conv2d(2, 8, 8, 64, 64), "b200_conv.hwcfg", "conv_i8_tc"),
        ("conv_rows", W.conv2d(1, 12, 10, 64, 128), "b200_conv.hwcfg", "conv_i8_tc"),
    ]


@pytest.fixture(scope="module")
def tiled():
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    return {name: (text, Ref.pipeline(text, cfg(c)), kern) for name, text, c, kern in cases()}


def test_pipeline_output_plans_onto_tensor_cores(tiled):
    import paper_1903_06498_b200 as sb
    for name, (orig, t, kern) in tiled.items():
        assert "@SMEM" in t, name  # the pass pipeline really tiled and placed the program
        plan = sb.parse_program(t).describe_plan(True)
        assert f"kernel={kern}" in plan, (name, plan)


@pytest.mark.gpu
def test_pipeline_output_parity(tiled):
    if not gpu_available():
        pytest.skip("no B200")
    for name, (orig, t, kern) in tiled.items():
        prog = Ref.parse(t)
        store = Ref.random_inputs(prog, 2001)
        exp = Ref.execute(prog, store)
        # the reference's own property: the pipeline preserves execution
        exp0 = Ref.execute(Ref.parse(orig), Ref.random_inputs(Ref.parse(orig), 2001))
        for n in exp:
            np.testing.assert_array_equal(exp[n][1], exp0[n][1], err_msg=name)
        got = run_device(t, {n: (b, a) for n, (b, a) in store.items() if n != "C" and n != "O"})
        for n, (b, a) in exp.items():
            np.testing.assert_array_equal(got[n], a, err_msg=f"{name}:{n}")
