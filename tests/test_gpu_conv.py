"""tcgen05 implicit-GEMM convolution path vs the reference semantics (bit-exact).

Small shapes: reference interpreter (oracle/_ref) or the pinned port.
Full BASELINE config-2 shape: size-independent checks against an exact float64
convolution (products <= 2^14, sums < 2^24: float64 is exact) and against the
generic block kernel.
"""
import numpy as np
import pytest

from harness import gpu_available, run_device
from oracle import Port, Ref, random_inputs, reference_execute
from paper_1903_06498_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def inputs_for(text, seed):
    import paper_1903_06498_b200 as sb
    p = sb.parse_program(text)
    bufs = [(n, d.dtype, d.elements, int(d.dir)) for n, d in p.buffers.items()]
    return p, {n: (p.buffers[n].dtype, a) for n, a in random_inputs(bufs, seed).items()}


def expected(text, inputs):
    import paper_1903_06498_b200 as sb
    p = sb.parse_program(text)
    store = {n: a for n, (b, a) in inputs.items()}
    for n, d in p.buffers.items():
        if n not in store:
            store[n] = np.full(d.elements, p.output_identity(n), np.int64)
    if Ref.available():
        r = Ref.parse(text)
        out = Ref.execute(r, {n: (p.buffers[n].dtype, a) for n, a in store.items()})
        return {n: v[1] for n, v in out.items()}
    return reference_execute(text, store)


SHAPES = [
    # N, H, W, C, K, out dtype
    (2, 16, 16, 64, 64, "i32"),
    (1, 7, 7, 64, 128, "i32"),
    (3, 14, 14, 64, 32, "i32"),
    (2, 13, 20, 64, 96, "i32"),
    (1, 9, 30, 128, 64, "i32"),
    (2, 8, 8, 64, 64, "i8"),
    (2, 8, 8, 64, 32, "i16"),
    (1, 3, 60, 64, 256, "i32"),
    (2, 5, 7, 192, 64, "i32"),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_conv_tc_small(shape):
    N, H, Wd, C, K, od = shape
    text = W.conv2d(N, H, Wd, C, K, out_dtype=od)
    import paper_1903_06498_b200 as sb
    assert "conv_i8_tc" in sb.parse_program(text).describe_plan(True)
    _, inp = inputs_for(text, N * 1000 + H)
    exp = expected(text, inp)
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["O"], exp["O"])


def test_conv_tc_accumulates_into_existing_output():
    """O:add accumulates into existing contents when the output is supplied (README.md:104-110)."""
    text = W.conv2d(2, 10, 12, 64, 64)
    p, inp = inputs_for(text, 5)
    rng = np.random.default_rng(0)
    inp["O"] = (32, rng.integers(-2**31, 2**31, size=p.buffers["O"].elements).astype(np.int64))
    exp = expected(text, inp)
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["O"], exp["O"])


def test_conv_tc_matches_generic_kernel():
    text = W.conv2d(2, 12, 12, 64, 64)
    _, inp = inputs_for(text, 9)
    a = run_device(text, inp)
    b = run_device(text, inp, disable_tc=True)
    np.testing.assert_array_equal(a["O"], b["O"])


def test_conv_tc_fig6a_constraint_window():
    """Constraint tighter than the buffer (fig6a.stripe's `12 - y - j >= 0`) is honoured."""
    text = W.conv2d(1, 12, 16, 64, 64).replace("-j - y + 16 >= 0", "-j - y + 12 >= 0")
    _, inp = inputs_for(text, 4)
    exp = expected(text, inp)
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["O"], exp["O"])


def test_conv_tc_full_config2_exact():
    """BASELINE config 2 (3x3 NHWC 56x56x64->64, batch 32) through the device-resident API,
    checked against an exact float64 convolution on the GPU."""
    import torch
    import paper_1903_06498_b200 as sb
    N, H, Wd, C, K = 32, 56, 56, 64, 64
    text = W.conv2d(N, H, Wd, C, K)
    prog = sb.parse_program(text)
    g = torch.Generator(device="cuda").manual_seed(1)
    I = torch.randint(-128, 128, (N, H, Wd, C), dtype=torch.int8, device="cuda", generator=g)
    F = torch.randint(-128, 128, (3, 3, K, C), dtype=torch.int8, device="cuda", generator=g)
    O = torch.full((N, H, Wd, K), 12345, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()  # the context's own stream does not wait for torch's
    ctx = sb.default_context(0)
    ctx.execute_device(prog, {"I": (I.data_ptr(), I.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                              "O": (O.data_ptr(), O.numel(), sb.SB_BUF_PREPARE)})
    ctx.sync()
    ref = torch.nn.functional.conv2d(I.permute(0, 3, 1, 2).double(), F.permute(2, 3, 0, 1).double(), padding=1)
    ref = ref.permute(0, 2, 3, 1).to(torch.int64)
    assert torch.equal(O.to(torch.int64), ref)


@pytest.mark.parametrize("shape", [(2, 8, 8, 64, 64), (1, 6, 20, 128, 32), (3, 4, 9, 64, 96)],
                         ids=lambda s: "x".join(map(str, s)))
def test_fused_conv_bias_relu(shape):
    """BASELINE config 3 structure: conv into a per-tile local accumulator, then
    O = max(T + Bias[k], 0); the epilogue is fused into the tcgen05 kernel."""
    import paper_1903_06498_b200 as sb
    N, H, Wd, C, K = shape
    text = W.conv_bias_relu(N, H, Wd, C, K)
    plan = sb.parse_program(text).describe_plan(True)
    assert "epilogue of" in plan and "conv_i8_tc" in plan, plan
    _, inp = inputs_for(text, 77 + N)
    exp = expected(text, inp)
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["O"], exp["O"])


def test_fused_epilogue_int64_semantics_near_overflow():
    """max(T + Bias, 0) is evaluated on unwrapped int64 temps (interp.cpp:515-537) and
    wrapped only at the store: biases near 2^31 must wrap exactly like the reference."""
    text = W.conv_bias_relu(1, 4, 8, 64, 32)
    p, inp = inputs_for(text, 5)
    inp["Bias"] = (32, np.array([2**31 - 1 - 3 * i for i in range(16)] + [-(2**31) + 7 * i for i in range(16)],
                                dtype=np.int64))
    exp = expected(text, inp)
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["O"], exp["O"])


@pytest.mark.parametrize("ordered", [False, True])
def test_async_two_context_pingpong_matches_sync(ordered):
    """sb_execute_async on two contexts (the bench's e2e pattern) gives the sync results."""
    import ctypes

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.conv2d(4, 10, 10, 64, 64)
    prog = sb.parse_program(text)
    ctxs = [sb.Context(0), sb.Context(0)]
    for c in ctxs:  # sb_context_set_kernel_order: kernels one step at a time, copies overlap
        c.set_kernel_order(ordered)
    pins = []

    def pinned(n, ct):
        p = ctypes.c_void_p()
        sb._check(sb.lib().sb_host_alloc_pinned(n * ctypes.sizeof(ct), ctypes.byref(p)))
        pins.append(p)
        return np.ctypeslib.as_array((ct * n).from_address(p.value))

    rng = np.random.default_rng(5)
    steps = []
    for i in range(4):
        I = pinned(4 * 10 * 10 * 64, ctypes.c_int8)
        F = pinned(9 * 64 * 64, ctypes.c_int8)
        O = pinned(4 * 10 * 10 * 64, ctypes.c_int32)
        I[:] = rng.integers(-128, 128, I.size, dtype=np.int8)
        F[:] = rng.integers(-128, 128, F.size, dtype=np.int8)
        steps.append((I, F, O))
        ctxs[i % 2].execute_native_async(prog, {"I": I, "F": F, "O": O}, prepare=("O",))
    for c in ctxs:
        c.sync()
    for I, F, O in steps:
        ref = np.empty_like(O)
        sb.default_context(0).execute_native(prog, {"I": I.copy(), "F": F.copy(), "O": ref}, prepare=("O",))
        np.testing.assert_array_equal(O, ref)
    for p in pins:
        sb.lib().sb_host_free_pinned(p)
