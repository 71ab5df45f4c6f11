"""Windowed max/min leaves on the pool kernel (kernels/pool.cu), bit-exact.

Checkers: the reference interpreter via its golden-pinned CPU restatement (oracle/port)
on small shapes; an exact PyTorch restatement at ResNet-stem size.
"""
import numpy as np
import pytest

from harness import gpu_available
from oracle import Port, reference_execute

CASES = [
    # N, H, W, C, R, S, stride, pad, agg, dtype
    (2, 9, 11, 16, 3, 3, 2, 1, "max", "i8"),
    (1, 8, 8, 32, 2, 2, 2, 0, "min", "i8"),
    (2, 7, 7, 8, 3, 3, 1, 1, "max", "i16"),
    (1, 10, 6, 4, 3, 3, 2, 1, "min", "i32"),
    (3, 12, 12, 64, 5, 5, 3, 2, "max", "i8"),
    # 3x3 / stride-2 i8: the row-strip kernel (odd and even sizes, no padding, min)
    (3, 13, 10, 48, 3, 3, 2, 1, "min", "i8"),
    (2, 15, 15, 32, 3, 3, 2, 0, "max", "i8"),
    (5, 40, 38, 16, 3, 3, 2, 1, "max", "i8"),
    # 3x3 / stride-2, other widths and a single-window image
    (2, 17, 19, 8, 3, 3, 2, 1, "max", "i16"),
    (2, 33, 9, 4, 3, 3, 2, 1, "min", "i32"),
    (1, 3, 3, 16, 3, 3, 2, 1, "max", "i8"),
]


def test_pool_planned():
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    for c in CASES:
        plan = sb.parse_program(W.pool2d(*c)).describe_plan()
        assert "kernel=pool" in plan or "kernel=reduce" in plan, plan


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c)))
def test_pool_vs_port(case):
    if not gpu_available():
        pytest.skip("no B200")
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.pool2d(*case)
    prog = sb.parse_program(text)
    bits = int(prog.buffers["I"].dtype)
    rng = np.random.default_rng(sum(case[:8]))
    x = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), prog.buffers["I"].elements, dtype=np.int64)
    store = {"I": sb.Buffer(prog.buffers["I"].dtype, x.copy())}
    sb.prepare_outputs(prog, store)
    o0 = store["O"].data.copy()
    sb.execute(prog, store)
    ref = reference_execute(text, {"I": x, "O": o0})
    np.testing.assert_array_equal(store["O"].data, ref["O"])


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["pair", "single"])
@pytest.mark.parametrize("case", [c for c in CASES if c[4:7] == (3, 3, 2)], ids=lambda c: "x".join(map(str, c)))
def test_pool_3x3s2_accumulates_into_existing(case, kernel, monkeypatch):
    """max/min into an output that already holds values (no fill absorbed): the pair kernel
    and the per-pixel kernel (SB_POOL_SINGLE)."""
    if not gpu_available():
        pytest.skip("no B200")
    if kernel == "single":
        monkeypatch.setenv("SB_POOL_SINGLE", "1")
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.pool2d(*case)
    prog = sb.parse_program(text)
    bits = int(prog.buffers["I"].dtype)
    rng = np.random.default_rng(7 + sum(case[:4]))
    lim = 1 << (bits - 1)
    x = rng.integers(-lim, lim, prog.buffers["I"].elements, dtype=np.int64)
    o0 = rng.integers(-lim, lim, prog.buffers["O"].elements, dtype=np.int64)
    store = {"I": sb.Buffer(prog.buffers["I"].dtype, x.copy()), "O": sb.Buffer(prog.buffers["O"].dtype, o0.copy())}
    sb.execute(prog, store)
    ref = reference_execute(text, {"I": x, "O": o0})
    np.testing.assert_array_equal(store["O"].data, ref["O"])


@pytest.mark.gpu
def test_stem_pool_vs_torch():
    if not gpu_available():
        pytest.skip("no B200")
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, C = 16, 112, 64
    text = W.pool2d(N, H, H, C)
    prog = sb.parse_program(text)
    assert "kernel=pool" in prog.describe_plan()
    x = np.random.default_rng(3).integers(-128, 128, N * H * H * C, dtype=np.int64)
    store = {"I": sb.Buffer(prog.buffers["I"].dtype, x.copy())}
    sb.prepare_outputs(prog, store)  # identity -128 (dtype min)
    sb.execute(prog, store)
    t = torch.as_tensor(x.reshape(N, H, H, C)).permute(0, 3, 1, 2).double()
    exp = torch.nn.functional.max_pool2d(t, 3, 2, 1).permute(0, 2, 3, 1).long().numpy().ravel()
    np.testing.assert_array_equal(store["O"].data, exp)
