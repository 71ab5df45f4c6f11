"""tcgen05 GEMM path (kernels/gemm_tc.cu) vs the reference semantics, bit-exact."""
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


def check(text, seed=3, provide_out=False):
    import paper_1903_06498_b200 as sb
    p = sb.parse_program(text)
    assert "gemm_i8_tc" in p.describe_plan(not provide_out), p.describe_plan(True)
    bufs = [(n, d.dtype, d.elements, int(d.dir)) for n, d in p.buffers.items()]
    inp = {n: (p.buffers[n].dtype, a) for n, a in random_inputs(bufs, seed).items()}
    if provide_out:
        rng = np.random.default_rng(seed)
        d = p.buffers["C"]
        lim = 2 ** (d.dtype - 1)
        inp["C"] = (d.dtype, rng.integers(-lim, lim, size=d.elements).astype(np.int64))
    store = {n: a for n, (b, a) in inp.items()}
    for n, d in p.buffers.items():
        if n not in store:
            store[n] = np.full(d.elements, p.output_identity(n), np.int64)
    if Ref.available():
        exp = {n: v[1] for n, v in Ref.execute(Ref.parse(text), {n: (p.buffers[n].dtype, a) for n, a in store.items()}).items()}
    else:
        exp = reference_execute(text, store)
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["C"], exp["C"])


@pytest.mark.parametrize("mnk", [(64, 64, 64), (256, 128, 512), (200, 176, 320), (130, 304, 48), (3, 16, 16),
                                 (128, 128, 384), (1008, 608, 1008), (130, 1104, 4096)],
                         ids=lambda s: "x".join(map(str, s)))
def test_matmul_i8_to_i32(mnk):
    check(W.matmul(*mnk, in_dtype="i8", out_dtype="i32"))


@pytest.mark.parametrize("od", ["i8", "i16"])
def test_matmul_narrow_outputs_wrap(od):
    check(W.matmul(128, 128, 256, in_dtype="i8", out_dtype=od))


@pytest.mark.parametrize("mnk", [(256, 128, 512), (128, 128, 384), (1008, 608, 1008), (1024, 1024, 1024)],
                         ids=lambda s: "x".join(map(str, s)))
def test_matmul_pair_split_path(monkeypatch, mnk):
    """The opt-in CTA-pair split-K (SB_GEMM_SPLIT: rank 1's partial tile added over DSMEM by
    rank 0) stays bit-exact, odd k-block counts included."""
    monkeypatch.setenv("SB_GEMM_SPLIT", "1")
    check(W.matmul(*mnk, in_dtype="i8", out_dtype="i32"))


def check_exact_np(text, a_shape, b_shape, bt=False, seed=5):
    """Large shapes: the exact int64 product (numpy) wrapped to i32 is the reference's value
    (i8 x i8 products summed in int64, stored with i32 wrap; interp.cpp / ir.cpp:79-97)."""
    import paper_1903_06498_b200 as sb
    p = sb.parse_program(text)
    assert "gemm_i8_tc" in p.describe_plan(True)
    rng = np.random.default_rng(seed)
    a = rng.integers(-128, 128, a_shape, dtype=np.int64)
    b = rng.integers(-128, 128, b_shape, dtype=np.int64)
    store = {"A": sb.Buffer(p.buffers["A"].dtype, a.ravel().copy()), "B": sb.Buffer(p.buffers["B"].dtype, b.ravel().copy())}
    sb.prepare_outputs(p, store)
    sb.execute(p, store)
    exp = (a @ (b.T if bt else b)).astype(np.int32).astype(np.int64)
    np.testing.assert_array_equal(store["C"].data.reshape(exp.shape), exp)


@pytest.mark.parametrize("shape", [(2048, 4864, 256, "n"), (2048, 4800, 384, "n"), (2048, 4864, 256, "k"),
                                   (1920, 5120, 128, "n")], ids=lambda s: "x".join(map(str, s)))
def test_matmul_wide_tiles(shape):
    """128 x 256 tiles (N = 256 MMAs, two 128-element MN boxes of B per stage or one 256-row
    K-major box, the staged i32 output stored in two 128-column halves), chosen when every SM
    gets at least two of them; ragged N included."""
    M, N, K, major = shape
    if major == "n":
        check_exact_np(W.matmul(M, N, K, in_dtype="i8", out_dtype="i32"), (M, K), (K, N))
    else:
        check_exact_np(W.matmul_bt(M, N, K), (M, K), (N, K), bt=True)


def test_matmul_wide_tiles_forced_and_accumulating(monkeypatch):
    monkeypatch.setenv("SB_GEMM_BN", "256")
    check(W.matmul(384, 512, 256, in_dtype="i8", out_dtype="i32"))
    check(W.matmul(256, 768, 128, in_dtype="i8", out_dtype="i32"), provide_out=True)
    check(W.matmul(128, 400, 256, in_dtype="i8", out_dtype="i16"))


def test_matmul_b_k_major():
    check(W.matmul_bt(192, 160, 256))


def test_matmul_accumulates_into_existing():
    check(W.matmul(128, 256, 128, in_dtype="i8", out_dtype="i32"), provide_out=True)


def test_matmul_config1_shape_exact():
    """BASELINE config 1 shape (1024^3) in the i8 integer mode, checked against numpy int64."""
    import paper_1903_06498_b200 as sb
    rng = np.random.default_rng(1)
    A = rng.integers(-128, 128, size=(1024, 1024)).astype(np.int64)
    B = rng.integers(-128, 128, size=(1024, 1024)).astype(np.int64)
    got = run_device(W.matmul(1024, 1024, 1024, "i8", "i32"), {"A": (8, A.ravel()), "B": (8, B.ravel())})
    np.testing.assert_array_equal(got["C"].reshape(1024, 1024), A @ B)


# ---- byte-limb mode: i16 / i32 operands, exact modulo 2^bits(C) on u8 tensor cores ----------

LIMB = [
    # M, N, K, in dtype, out dtype, B transposed
    (64, 48, 32, "i32", "i32", False),
    (130, 96, 80, "i16", "i32", False),
    (128, 64, 48, "i32", "i16", True),
    (96, 112, 64, "i16", "i8", True),
    (33, 16, 16, "i32", "i32", True),
    (256, 208, 2048, "i32", "i32", False),  # few tiles, long K: split-K partials added with red.global.add
    (300, 128, 1008, "i16", "i32", True),   # K not a multiple of the 64-byte k-block (zero-padded planes)
]


@pytest.mark.parametrize("case", LIMB, ids=lambda c: "x".join(map(str, c)))
def test_limb_gemm_vs_reference(case):
    M, N, K, dt, od, bt = case
    text = (W.matmul_bt if bt else W.matmul)(M, N, K, in_dtype=dt, out_dtype=od)
    check(text, seed=M + N + K)
    check(text, seed=M + N + K + 1, provide_out=True)


def test_limb_gemm_unfused_path(monkeypatch):
    """SB_LIMB_UNFUSED keeps the per-sum GEMMs + combine pass: same bytes."""
    monkeypatch.setenv("SB_LIMB_UNFUSED", "1")
    text = W.matmul(130, 96, 80, in_dtype="i32", out_dtype="i32")
    check(text, seed=5)


def test_limb_gemm_config1_i32_exact():
    """Config 1 in the reference's exact integer mode: 1024^3 i32 x i32 -> i32 (mod 2^32)."""
    import torch
    import paper_1903_06498_b200 as sb
    text = W.matmul(1024, 1024, 1024, in_dtype="i32", out_dtype="i32")
    p = sb.parse_program(text)
    assert "byte limbs" in p.describe_plan(True)
    rng = np.random.default_rng(1001)
    a = rng.integers(-2**31, 2**31, 1024 * 1024, dtype=np.int64)
    b = rng.integers(-2**31, 2**31, 1024 * 1024, dtype=np.int64)
    store = {"A": sb.Buffer(32, a.copy()), "B": sb.Buffer(32, b.copy())}
    sb.prepare_outputs(p, store)
    sb.execute(p, store)
    # exact reference: 16-bit halves on the GPU in float64 (every partial sum < 2^53)
    A = torch.as_tensor(a.reshape(1024, 1024) & 0xFFFFFFFF, device="cuda")
    B = torch.as_tensor(b.reshape(1024, 1024) & 0xFFFFFFFF, device="cuda")
    al, ah = (A & 0xFFFF).double(), (A >> 16).double()
    bl, bh = (B & 0xFFFF).double(), (B >> 16).double()
    ll = (al @ bl).long()
    mid = ((al @ bh) + (ah @ bl)).long()
    c = (ll + (mid << 16)) & 0xFFFFFFFF
    c = torch.where(c >= 2**31, c - 2**32, c).cpu().numpy().ravel()
    np.testing.assert_array_equal(store["C"].data, c)


@pytest.mark.parametrize("dt", ["i8", "i32"])
def test_config1_autotiled_program_exact(dt):
    """BASELINE config 1 as one autotiled Stripe block (configs/c1_autotiled_*.stripe: the
    reference's tile_rewrite of the device autotile choice) collapses onto the tensor-core GEMM
    and equals the exact int64 product wrapped to i32."""
    import os
    import paper_1903_06498_b200 as sb
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "configs", f"c1_autotiled_{dt}.stripe")) as f:
        text = f.read()
    p = sb.parse_program(text)
    assert "gemm_i8_tc" in p.describe_plan(True)
    bits = 8 if dt == "i8" else 32
    rng = np.random.default_rng(11)
    a = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), (1024, 1024), dtype=np.int64)
    b = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), (1024, 1024), dtype=np.int64)
    store = {"A": sb.Buffer(p.buffers["A"].dtype, a.ravel().copy()), "B": sb.Buffer(p.buffers["B"].dtype, b.ravel().copy())}
    sb.prepare_outputs(p, store)
    sb.execute(p, store)
    # exact product modulo 2^32 (uint64 wrap-around arithmetic), as the reference's i32 store wraps
    exp = (a.astype(np.uint64) @ b.astype(np.uint64)).astype(np.uint32).astype(np.int32).astype(np.int64)
    np.testing.assert_array_equal(store["C"].data.reshape(1024, 1024), exp)
