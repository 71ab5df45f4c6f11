"""General im2col-TMA implicit-GEMM conv (kernels/conv_igemm.cu): strided, 1x1, streamed
filters, any output-channel count, fused bias/ReLU epilogue to i8 -- bit-exact.

Checkers: the CPU restatement (oracle/port) on small cases, which pins the exact
PyTorch restatement (tests/intmodel.py) used at larger shapes.
"""
import numpy as np
import pytest

from harness import gpu_available
from oracle import Port, reference_execute

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def rand_inputs(prog, seed):
    import paper_1903_06498_b200 as sb
    rng = np.random.default_rng(seed)
    store = {}
    for name, d in prog.buffers.items():
        if d.dir == sb.Dir.Out:
            continue
        bits = int(d.dtype)
        lo, hi = -(1 << (bits - 1)), (1 << (bits - 1))
        store[name] = sb.Buffer(d.dtype, rng.integers(lo, hi, d.elements, dtype=np.int64))
    return store


def run(text, seed=0):
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(text)
    store = rand_inputs(prog, seed)
    inputs = {n: b.data.copy() for n, b in store.items()}
    sb.prepare_outputs(prog, store)
    sb.execute(prog, store)
    return prog, inputs, {n: b.data for n, b in store.items()}


CONVS = [
    # N, H, W, C, K, R, S, stride, pad
    (2, 16, 16, 64, 64, 3, 3, 2, 1),      # strided 3x3 (ResNet v1.5 stage entry)
    (2, 14, 14, 256, 256, 3, 3, 1, 1),    # filter too large for shared memory
    (2, 8, 8, 128, 512, 1, 1, 1, 0),      # 1x1, K > 256
    (2, 16, 16, 64, 256, 1, 1, 2, 0),     # strided 1x1 projection
    (1, 7, 7, 512, 2048, 1, 1, 1, 0),     # stage-4 1x1
    (3, 9, 11, 64, 320, 3, 3, 1, 1),      # ragged tiles, K not a multiple of 128
    (1, 32, 32, 64, 64, 7, 7, 2, 3),      # 7x7/2 (stem shape with 64 channels)
    (2, 15, 13, 128, 64, 3, 3, 2, 1),     # odd extents with stride 2
    (2, 16, 15, 64, 64, 3, 3, 2, 1),      # im2col corners differ in H and W (upper -2 vs -1)
    (1, 6, 17, 64, 128, 1, 3, 2, 0),      # 1x3 filter, no padding, wide rows
]


@pytest.mark.parametrize("shape", CONVS, ids=lambda s: "x".join(map(str, s)))
def test_igemm_conv_exact(shape):
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_exact, wrap
    N, H, Wd, C, K, R, S, st, pad = shape
    text = W.conv2d(N, H, Wd, C, K, R, S, pad=pad, stride=st)
    plan = sb.parse_program(text).describe_plan()
    assert "conv_igemm_tc" in plan or "conv_i8_tc" in plan or "gemm_i8_tc" in plan, plan
    prog, inp, out = run(text, seed=sum(shape))
    x = inp["I"].reshape(N, H, Wd, C)
    w = inp["F"].reshape(R, S, K, C)
    exp = wrap(32, conv_exact(x, w, st, pad, "cuda")).cpu().numpy().ravel()
    np.testing.assert_array_equal(out["O"], exp)


def test_igemm_pinned_against_port():
    from paper_1903_06498_b200 import workloads as W
    text = W.conv2d(1, 9, 7, 64, 192, 3, 3, pad=1, stride=2)
    prog, inp, out = run(text, seed=5)
    ref = reference_execute(text, {**inp, "O": np.zeros_like(out["O"])})
    np.testing.assert_array_equal(out["O"], ref["O"])


FUSED = [
    # N, H, W, C, K, R, S, stride, pad, relu, residual
    (2, 16, 16, 64, 64, 3, 3, 2, 1, True, False),
    (2, 8, 8, 256, 512, 1, 1, 1, 0, True, False),
    (2, 14, 14, 256, 256, 3, 3, 1, 1, False, False),
    (2, 8, 8, 64, 256, 1, 1, 1, 0, True, True),   # residual add fused (TMA-loaded tile)
    (3, 7, 9, 128, 192, 3, 3, 1, 1, True, True),  # residual with ragged M and N tiles
    (2, 14, 14, 256, 512, 1, 1, 1, 0, True, True),  # 256-wide tiles + tensor-core residual
    # large M with N <= 128: two 128-row sub-tiles per tile (M = 2 x 128 rows, one stage handshake)
    (32, 56, 56, 64, 64, 3, 3, 1, 1, True, False),
    (27, 56, 56, 64, 128, 1, 1, 1, 0, True, True),  # + residual per sub-tile, ragged last tile
    (2, 14, 14, 64, 320, 1, 1, 1, 0, True, True),   # 256-wide tiles, last n-tile 64 wide + residual
    (4, 14, 14, 256, 256, 3, 3, 1, 1, True, False),  # streamed 3x3 filter, 18 k-blocks
]


@pytest.mark.parametrize("case", FUSED, ids=lambda s: "x".join(map(str, s)))
def test_igemm_fused_epilogue_i8(case):
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_layer_exact
    import torch
    N, H, Wd, C, K, R, S, st, pad, relu, res = case
    text = W.conv_fused(N, H, Wd, C, K, R, S, st, pad, relu=relu, residual=res)
    plan = sb.parse_program(text).describe_plan()
    assert "fused" in plan, plan
    prog, inp, out = run(text, seed=sum(case[:9]))
    P = (H + 2 * pad - R) // st + 1
    Q = (Wd + 2 * pad - S) // st + 1
    r = torch.as_tensor(inp["Res"].reshape(N, P, Q, K), device="cuda") if res else None
    exp = conv_layer_exact(inp["I"].reshape(N, H, Wd, C), inp["F"].reshape(R, S, K, C), inp["Bias"], st, pad,
                           relu, r, 8, "cuda").cpu().numpy().ravel()
    np.testing.assert_array_equal(out["O"], exp)


@pytest.mark.parametrize("lo", [-5, 1000, -(1 << 33), (1 << 33)])
def test_igemm_fused_clamp_constants(lo):
    """max(x, lo) with lo away from 0 and outside the i32 range (int64 temps)."""
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_layer_exact
    import torch
    N, H, Wd, C, K = 2, 8, 8, 64, 128
    for res in (False, True):
        for od, bits in (("i8", 8), ("i32", 32)):
            if res and od == "i32":
                continue
            text = W.conv_fused(N, H, Wd, C, K, 3, 3, 1, 1, relu=True, residual=res, out_dtype=od, lo=lo)
            assert "fused" in sb.parse_program(text).describe_plan()
            prog, inp, out = run(text, seed=lo & 0xFFFF)
            r = torch.as_tensor(inp["Res"].reshape(N, H, Wd, K), device="cuda") if res else None
            exp = conv_layer_exact(inp["I"].reshape(N, H, Wd, C), inp["F"].reshape(3, 3, K, C), inp["Bias"], 1, 1,
                                   True, r, bits, "cuda", lo=lo).cpu().numpy().ravel()
            np.testing.assert_array_equal(out["O"], exp, err_msg=f"lo={lo} res={res} out={od}")


def test_fused_small_pinned_against_port():
    from paper_1903_06498_b200 import workloads as W
    text = W.conv_fused(1, 6, 6, 64, 128, 3, 3, 2, 1)
    prog, inp, out = run(text, seed=9)
    ref = reference_execute(text, {**inp, "O": np.zeros_like(out["O"])})
    np.testing.assert_array_equal(out["O"], ref["O"])


SMALL_C = [
    # N, H, W, C, K, R, S, stride, pad  (phase fold, or gather mode: taps x channels per pixel in smem)
    (2, 32, 32, 3, 64, 7, 7, 2, 3),       # ResNet stem shape
    (1, 9, 13, 16, 96, 3, 3, 1, 1),
    (2, 10, 10, 24, 128, 5, 5, 2, 2),
    (1, 8, 8, 3, 200, 3, 3, 1, 0),        # no padding, K > 128
    (2, 13, 18, 3, 64, 7, 7, 2, 3),       # odd/even extents under the 2x2 fold
    (1, 11, 9, 5, 32, 3, 5, 3, 1),        # stride 3 fold (45 bytes per folded pixel)
    (3, 15, 17, 3, 64, 7, 7, 2, 3),       # odd extents, materialised fold rows
]


@pytest.fixture(params=["fold", "gather"])
def small_c_mode(request, monkeypatch):
    if request.param == "gather":
        monkeypatch.setenv("SB_NO_FOLD", "1")
    else:
        monkeypatch.delenv("SB_NO_FOLD", raising=False)
    return request.param


@pytest.mark.parametrize("shape", SMALL_C, ids=lambda s: "x".join(map(str, s)))
def test_gather_conv_exact(shape, small_c_mode):
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_exact, wrap
    N, H, Wd, C, K, R, S, st, pad = shape
    text = W.conv2d(N, H, Wd, C, K, R, S, pad=pad, stride=st)
    plan = sb.parse_program(text).describe_plan()
    assert "packed" in plan, plan
    if small_c_mode == "fold":
        assert "phase-folded" in plan, plan
    elif "phase-folded" in plan:
        pytest.fail(plan)
    prog, inp, out = run(text, seed=sum(shape))
    exp = wrap(32, conv_exact(inp["I"].reshape(N, H, Wd, C), inp["F"].reshape(R, S, K, C), st, pad, "cuda"))
    np.testing.assert_array_equal(out["O"], exp.cpu().numpy().ravel())


def test_gather_stem_fused_vs_port(small_c_mode):
    from paper_1903_06498_b200 import workloads as W
    text = W.conv_fused(1, 12, 12, 3, 64, 7, 7, 2, 3)
    prog, inp, out = run(text, seed=21)
    ref = reference_execute(text, {**inp, "O": np.zeros_like(out["O"])})
    np.testing.assert_array_equal(out["O"], ref["O"])


BAND = [
    # N, H, W, C, K, R, S, stride, pad, relu: strided small-channel convs into fresh i8 activations
    (2, 32, 32, 3, 64, 7, 7, 2, 3, True),     # ResNet stem shape
    (3, 28, 36, 3, 64, 7, 7, 2, 3, True),     # non-square, several images
    (1, 224, 224, 3, 64, 7, 7, 2, 3, True),   # the full stem: 112-pixel rows in 128-row tiles
    (2, 256, 250, 3, 64, 7, 7, 2, 3, False),  # 125-pixel rows (junk-row tail reads), no clamp
    (2, 20, 20, 3, 128, 7, 7, 2, 3, True),    # K = 128: N = 256 per instruction, one store per row
    (2, 16, 24, 3, 64, 5, 5, 2, 2, True),     # 3x3 folded taps (4 k-blocks)
    # rows of whole 16-byte chunks (band_raw-eligible; see test_band_raw_matches_folded)
    (2, 64, 48, 3, 64, 7, 7, 2, 3, True),
    (2, 20, 32, 3, 128, 7, 7, 2, 3, True),    # K = 128
    (2, 16, 32, 3, 64, 5, 5, 2, 2, True),     # 5x5 / pad 2: 4 folded rows, 8 raw rows per band
    (1, 36, 16, 3, 64, 7, 7, 2, 3, False),    # 8-pixel output rows, no clamp
]


@pytest.mark.parametrize("case", BAND, ids=lambda c: "x".join(map(str, c)))
def test_band_fold_conv_exact(case):
    """Band tiles (ConvPlan::fold_band): compact folded rows in shared memory read by
    overlapping-row UMMA descriptors, two output rows stacked along N against the banded
    filter, 4-D clipped TMA store -- bit-exact vs the exact restatement."""
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_layer_exact
    N, H, Wd, C, K, R, S, st, pad, relu = case
    text = W.conv_fused(N, H, Wd, C, K, R, S, st, pad, relu=relu)
    plan = sb.parse_program(text).describe_plan()
    assert "band tiles of 2 output rows" in plan, plan
    prog, inp, out = run(text, seed=N + H + K)
    exp = conv_layer_exact(inp["I"].reshape(N, H, Wd, C), inp["F"].reshape(R, S, K, C), inp["Bias"], st, pad, relu,
                           None, 8, "cuda").cpu().numpy().ravel()
    np.testing.assert_array_equal(out["O"], exp)


STRIP = [
    # N, H, W, K, pad, relu: stride-1 3x3 over 64 channels into a fresh i8 activation
    (2, 56, 56, 64, 1, True),      # the ResNet stage-1 shape
    (3, 13, 17, 64, 1, True),      # odd rows (last strip clipped), 17-pixel rows in the 64 pitch
    (2, 9, 62, 128, 1, False),     # widest row the pitch holds, K = 128, no clamp
    (1, 20, 30, 256, 1, True),     # K = 256 (two store boxes per sub-tile)
    (2, 10, 12, 64, 0, True),      # no padding (valid conv, different window corner)
]


@pytest.mark.parametrize("case", STRIP, ids=lambda c: "x".join(map(str, c)))
def test_strip_conv_exact(case):
    """Strip mode (IgKParams::strip): one haloed 4-D TMA strip per tile, the 9 taps as
    descriptor shifts, 4-D clipped TMA store -- bit-exact vs the exact restatement."""
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_layer_exact
    N, H, Wd, K, pad, relu = case
    text = W.conv_fused(N, H, Wd, 64, K, 3, 3, 1, pad, relu=relu)
    prog, inp, out = run(text, seed=N + H + K + pad)
    exp = conv_layer_exact(inp["I"].reshape(N, H, Wd, 64), inp["F"].reshape(3, 3, K, 64), inp["Bias"], 1, pad, relu,
                           None, 8, "cuda").cpu().numpy().ravel()
    np.testing.assert_array_equal(out["O"], exp)


def test_strip_off_matches(monkeypatch):
    """SB_IG_NOSTRIP keeps the im2col path: same bytes."""
    from paper_1903_06498_b200 import workloads as W
    text = W.conv_fused(2, 14, 14, 64, 64, 3, 3, 1, 1)
    _, _, out_strip = run(text, seed=9)
    monkeypatch.setenv("SB_IG_NOSTRIP", "1")
    _, _, out_i2c = run(text, seed=9)
    np.testing.assert_array_equal(out_strip["O"], out_i2c["O"])


@pytest.mark.parametrize("shape", [(2, 32, 32), (3, 64, 48), (1, 224, 224)], ids=lambda c: "x".join(map(str, c)))
def test_band_raw_matches_folded(monkeypatch, shape):
    """band_raw (SB_BAND_RAW=1: the fold inside the conv's producer warps) writes the same bytes
    as the default band path over a materialised folded copy."""
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, Wd = shape
    text = W.conv_fused(N, H, Wd, 3, 64, 7, 7, 2, 3)
    monkeypatch.setenv("SB_BAND_RAW", "1")  # opt-in (measured slower than the separate fold)
    assert "folded in the producer warps" in sb.parse_program(text).describe_plan()
    _, _, out_raw = run(text, seed=H)
    monkeypatch.delenv("SB_BAND_RAW")
    plan = sb.parse_program(text).describe_plan()
    assert "band tiles" in plan and "producer warps" not in plan, plan
    _, _, out_fold = run(text, seed=H)
    np.testing.assert_array_equal(out_raw["O"], out_fold["O"])


def test_band_fold_off_matches(monkeypatch):
    """SB_NO_BAND keeps the materialised-rows fold: same bytes as the band path."""
    from paper_1903_06498_b200 import workloads as W
    text = W.conv_fused(2, 30, 30, 3, 64, 7, 7, 2, 3)
    _, _, out_band = run(text, seed=3)
    monkeypatch.setenv("SB_NO_BAND", "1")
    import paper_1903_06498_b200 as sb
    plan = sb.parse_program(text).describe_plan()
    assert "band tiles" not in plan and "phase-folded" in plan, plan
    _, _, out_rows = run(text, seed=3)
    np.testing.assert_array_equal(out_band["O"], out_rows["O"])


@pytest.mark.parametrize("case", [(2, 16, 16, 64, 64, True), (3, 9, 11, 64, 128, True), (2, 14, 14, 64, 192, False)],
                         ids=lambda c: "x".join(map(str, c)))
def test_resident_filter_conv_fused_i8(case):
    """Stride-1 3x3 with C = 64: the resident-filter kernel's i8 TMA-store epilogue (opt-in
    routing SB_TC_I8_EPI; the default keeps these layers on the im2col kernel)."""
    import os

    import paper_1903_06498_b200 as sb
    os.environ["SB_TC_I8_EPI"] = "1"
    from paper_1903_06498_b200 import workloads as W
    from intmodel import conv_layer_exact
    N, H, Wd, C, K, relu = case
    text = W.conv_fused(N, H, Wd, C, K, 3, 3, 1, 1, relu=relu)
    plan = sb.parse_program(text).describe_plan()
    assert "kernel=conv_i8_tc" in plan and "fused" in plan, plan
    prog, inp, out = run(text, seed=N + H + K)
    del os.environ["SB_TC_I8_EPI"]
    exp = conv_layer_exact(inp["I"].reshape(N, H, Wd, C), inp["F"].reshape(3, 3, K, C), inp["Bias"], 1, 1, relu,
                           None, 8, "cuda").cpu().numpy().ravel()
    np.testing.assert_array_equal(out["O"], exp)
