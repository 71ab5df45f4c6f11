"""fp32 numeric mode (the north_star's floating-point extension; the reference's DType has
no float, proj/include/stripe/ir.h:25).

Oracle: the CPU restatement's F32 policy (oracle/port, same interpreter structure as
interp.cpp with float temps and float store aggregation), plus a plain PyTorch fp32
reference for the conv workload.  Tolerance policy (stated per test):
  * owner / serial launches: bitwise equal to the F32 oracle (each output address sees
    its contributions in lexicographic order, uncontracted fp32 ops on both sides);
  * atomic launches (non-injective commutative aggregation) reorder fp32 sums:
    rtol 1e-5 / atol 1e-5 * sum|terms| against the oracle;
  * vs torch fp32 conv (different summation order): rtol 1e-4, atol 1e-4.
"""
import re

import numpy as np
import pytest

from harness import corpus, gpu_available
from oracle import Port

F32_RE = re.compile(r"\b(i8|i16|i32)\(")


def to_f32(text):
    return F32_RE.sub("f32(", text)


def f32_cases():
    out = []
    for c in corpus():
        if c.error or "gather(" in c.text or "scatter(" in c.text:
            continue
        out.append(c)
    return out


CASES = f32_cases()


def random_f32_inputs(prog, seed):
    import paper_1903_06498_b200 as sb
    rng = np.random.default_rng(seed)
    store = {}
    for name, d in prog.buffers.items():
        if d.dir == sb.Dir.Out:
            continue
        store[name] = sb.Buffer(d.dtype, rng.standard_normal(d.elements).astype(np.float32))
    return store


# ---- CPU: plan + oracle -------------------------------------------------------------------

def test_f32_plan_marks_launches():
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    p = sb.parse_program(W.conv2d(1, 4, 4, 4, 4, in_dtype="f32", out_dtype="f32"))
    plan = p.describe_plan()
    assert "kernel=generic" in plan and " f32" in plan, plan
    assert "conv_i8_tc" not in plan


def test_f32_identity_bits():
    import paper_1903_06498_b200 as sb
    t = """block []:1 (
\tin I[0] f32(8):(1)
\tout O[0]:assign f32(1):(1)
) {
\t0:
\tblock [i:8]:8 (
\t\tin I[i] f32(1):(1)
\t\tout O[0]:max f32(1):(1)
\t) {
\t\t0: $I = load(I)
\t\t1: O = store($I)
\t}
}
"""
    p = sb.parse_program(t)
    store = {}
    sb.prepare_outputs(p, store)
    assert store["O"].data.dtype == np.float32 and np.isneginf(store["O"].data[0])


def test_f32_mixed_dtypes_rejected():
    import paper_1903_06498_b200 as sb
    t = """block []:1 (
\tin I[0] i32(8):(1)
\tout O[0]:assign f32(8):(1)
) {
\t0:
\tblock [i:8]:8 (
\t\tin I[i] i32(1):(1)
\t\tout O[i] f32(1):(1)
\t) {
\t\t0: $I = load(I)
\t\t1: O = store($I)
\t}
}
"""
    p = sb.parse_program(t)
    with pytest.raises(sb.ExecError) as e:
        p.describe_plan()
    assert e.value.code == "Unsupported"


# ---- GPU parity ---------------------------------------------------------------------------

def run_both(text, seed=0):
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(text)
    store = random_f32_inputs(prog, seed)
    sb.prepare_outputs(prog, store)
    ref = Port.execute(text, {n: b.data.copy() for n, b in store.items()}, f32=True)
    sb.execute(prog, store)
    return prog, store, ref


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
def test_f32_corpus_vs_oracle(case):
    if not gpu_available():
        pytest.skip("no B200")
    text = to_f32(case.text)
    prog, store, ref = run_both(text, seed=len(case.name))
    atomic = "mode=atomic" in prog.describe_plan()
    for n, b in store.items():
        if prog.buffers[n].dir == 0:
            continue
        if atomic:
            np.testing.assert_allclose(b.data, ref[n], rtol=1e-5, atol=1e-4, err_msg=f"{case.name}:{n}")
        else:
            np.testing.assert_array_equal(b.data.view(np.uint32), np.asarray(ref[n], np.float32).view(np.uint32),
                                          err_msg=f"{case.name}:{n}")


@pytest.mark.gpu
def test_f32_conv_vs_torch():
    if not gpu_available():
        pytest.skip("no B200")
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, Wd, C, K = 2, 8, 8, 16, 16
    text = W.conv2d(N, H, Wd, C, K, in_dtype="f32", out_dtype="f32")
    prog, store, ref = run_both(text, seed=3)
    # bitwise vs the F32 oracle (owner mode: taps and channels summed in lex order)
    np.testing.assert_array_equal(store["O"].data.view(np.uint32), np.asarray(ref["O"], np.float32).view(np.uint32))
    x = torch.from_numpy(store["I"].data.reshape(N, H, Wd, C)).permute(0, 3, 1, 2).double()
    w = torch.from_numpy(store["F"].data.reshape(3, 3, K, C)).permute(2, 3, 0, 1).double()
    o = torch.nn.functional.conv2d(x, w, padding=1).permute(0, 2, 3, 1).float().numpy().ravel()
    np.testing.assert_allclose(store["O"].data, o, rtol=1e-4, atol=1e-4)


# ---- fp32 matmul (config 1 "fp32 matmul contraction") on the exact-order SIMT GEMM ----------

GEMMS = [(64, 48, 32, False), (130, 96, 80, False), (200, 72, 333, True), (1, 1, 1, False)]


def test_f32_gemm_planned():
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    p = sb.parse_program(W.matmul(128, 128, 128, in_dtype="f32", out_dtype="f32"))
    assert "kernel=gemm_f32" in p.describe_plan(True)


@pytest.mark.gpu
@pytest.mark.parametrize("case", GEMMS, ids=lambda c: "x".join(map(str, c)))
def test_f32_gemm_bitwise_vs_oracle(case):
    """Owner mode, k folded in order with rounded mul then add: bitwise equal to the oracle."""
    if not gpu_available():
        pytest.skip("no B200")
    from paper_1903_06498_b200 import workloads as W
    M, N, K, bt = case
    text = (W.matmul_bt if bt else W.matmul)(M, N, K, in_dtype="f32", out_dtype="f32")
    for accumulate in (False, True):
        import paper_1903_06498_b200 as sb
        prog = sb.parse_program(text)
        store = random_f32_inputs(prog, M + K)
        if accumulate:
            store["C"] = sb.Buffer(prog.buffers["C"].dtype,
                                   np.random.default_rng(1).standard_normal(M * N).astype(np.float32))
        sb.prepare_outputs(prog, store)
        ref = Port.execute(text, {n: b.data.copy() for n, b in store.items()}, f32=True)
        sb.execute(prog, store)
        np.testing.assert_array_equal(store["C"].data.view(np.uint32),
                                      np.asarray(ref["C"], np.float32).view(np.uint32))


@pytest.mark.gpu
def test_f32_gemm_config1_vs_torch():
    """1024^3 fp32: stated bound |c - exact| <= 1e-5 * sum_k |a||b| (sequential fp32 fold)."""
    if not gpu_available():
        pytest.skip("no B200")
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.matmul(1024, 1024, 1024, in_dtype="f32", out_dtype="f32")
    prog = sb.parse_program(text)
    store = random_f32_inputs(prog, 1001)
    sb.prepare_outputs(prog, store)
    a = torch.as_tensor(store["A"].data.reshape(1024, 1024), device="cuda").double()
    b = torch.as_tensor(store["B"].data.reshape(1024, 1024), device="cuda").double()
    sb.execute(prog, store)
    exact = (a @ b).cpu().numpy().ravel()
    scale = (a.abs() @ b.abs()).cpu().numpy().ravel()
    err = np.abs(store["C"].data.astype(np.float64) - exact)
    assert np.all(err <= 1e-5 * scale), float((err / scale).max())


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1024, 1024, 1024, False), (256, 384, 512, True), (130, 96, 80, False)],
                         ids=lambda c: "x".join(map(str, c)))
def test_f32_gemm_tf32x3_stated_bound(shape):
    """Opt-in SB_FP32_TF32X3: one kind::tf32 GEMM over [hi|hi|lo] x [hi;lo;hi];
    stated bound |c - exact| <= 1e-5 * sum_k |a||b| (fresh and accumulating outputs)."""
    if not gpu_available():
        pytest.skip("no B200")
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    M, N, K, bt = shape
    text = (W.matmul_bt if bt else W.matmul)(M, N, K, in_dtype="f32", out_dtype="f32")
    prog = sb.parse_program(text)
    assert "3xTF32" in prog.describe_plan(True, fp32_mode=1)
    for accumulate in (False, True):
        store = random_f32_inputs(prog, 7 + M)
        c0 = np.random.default_rng(2).standard_normal(M * N).astype(np.float32) if accumulate else None
        if accumulate:
            store["C"] = sb.Buffer(prog.buffers["C"].dtype, c0.copy())
        sb.prepare_outputs(prog, store)
        a = torch.as_tensor(store["A"].data.reshape(M, K), device="cuda").double()
        bm = store["B"].data.reshape(N, K).T if bt else store["B"].data.reshape(K, N)
        b = torch.as_tensor(np.ascontiguousarray(bm), device="cuda").double()
        sb.execute(prog, store, sb.ExecOptions(fp32_mode=1))
        exact = (a @ b).cpu().numpy().ravel() + (c0.astype(np.float64) if accumulate else 0)
        scale = (a.abs() @ b.abs()).cpu().numpy().ravel() + (np.abs(c0) if accumulate else 0)
        err = np.abs(store["C"].data.astype(np.float64) - exact)
        assert np.all(err <= 1e-5 * scale + 1e-30), float((err / (scale + 1e-30)).max())
