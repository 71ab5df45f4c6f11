"""Vectorised map/reduce kernel (kernels/map.cu) vs the reference semantics, bit-exact."""
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


def check(text, seed=1, expect_kernel="map"):
    import paper_1903_06498_b200 as sb
    p = sb.parse_program(text)
    if expect_kernel:
        kinds = expect_kernel if isinstance(expect_kernel, tuple) else (expect_kernel,)
        plan = p.describe_plan(True)
        assert any(f"kernel={k}" in plan for k in kinds), plan
    bufs = [(n, d.dtype, d.elements, int(d.dir)) for n, d in p.buffers.items()]
    inp = {n: (p.buffers[n].dtype, a) for n, a in random_inputs(bufs, seed).items()}
    store = {n: a for n, (b, a) in inp.items()}
    for n, d in p.buffers.items():
        if n not in store:
            store[n] = np.full(d.elements, p.output_identity(n), np.int64)
    if Ref.available():
        exp = {n: v[1] for n, v in Ref.execute(Ref.parse(text), {n: (p.buffers[n].dtype, a) for n, a in store.items()}).items()}
    else:
        exp = reference_execute(text, store)
    got = run_device(text, inp)
    for n in exp:
        np.testing.assert_array_equal(got[n], exp[n], err_msg=n)


@pytest.mark.parametrize("dt", ["i8", "i16", "i32"])
def test_maxpool(dt):
    check(W.maxpool2x2(3, 16, 18, 24, dtype=dt), expect_kernel=("reduce", "map"))


def test_maxpool_identity_fused_into_reduce():
    check(W.maxpool2x2(2, 8, 8, 64, dtype="i8"), expect_kernel="reduce")


@pytest.mark.parametrize("shape", [(4, 7, 7, 64), (3, 5, 3, 30), (2, 1, 9, 1027)])
def test_global_sum(shape):
    check(W.global_sum(*shape), expect_kernel=None)


def test_global_sum_i8_to_i16_wraps():
    check(W.global_sum(8, 7, 7, 1024, in_dtype="i8", out_dtype="i16"), expect_kernel="reduce")


@pytest.mark.parametrize("agg", ["assign", "add", "max", "min", "mul"])
def test_reduce_all_aggregations(agg):
    check(W.global_sum(4, 3, 5, 256).replace("O[n, c]:add", f"O[n, c]:{agg}"), expect_kernel="reduce")


@pytest.mark.parametrize("dt", ["i8", "i16", "i32"])
@pytest.mark.parametrize("agg", ["add", "max", "min", "mul"])
@pytest.mark.parametrize("prefill", [False, True])
def test_reduce_row_split(dt, agg, prefill):
    """Few outputs x many rows (the ResNet global sum shape): rows folded in 8 phases and
    combined in shared memory (order-free for add/max/min/mul); with a prefilled output the
    partials fold onto its old values."""
    import paper_1903_06498_b200 as sb
    text = W.global_sum(4, 5, 7, 256, in_dtype=dt, out_dtype=dt).replace("O[n, c]:add", f"O[n, c]:{agg}")
    p = sb.parse_program(text)
    assert "kernel=reduce" in p.describe_plan(True)
    bufs = [(n, d.dtype, d.elements, int(d.dir)) for n, d in p.buffers.items()]
    inp = {n: (p.buffers[n].dtype, a) for n, a in random_inputs(bufs, 17).items()}
    if prefill:  # an existing output: the reduction accumulates onto it
        o = random_inputs([("O", p.buffers["O"].dtype, p.buffers["O"].elements, 0)], 23)["O"]
        inp["O"] = (p.buffers["O"].dtype, o)
    store = {n: a for n, (b, a) in inp.items()}
    if "O" not in store:
        store["O"] = np.full(p.buffers["O"].elements, p.output_identity("O"), np.int64)
    exp = reference_execute(text, {n: a.copy() for n, a in store.items()})
    got = run_device(text, inp)
    np.testing.assert_array_equal(got["O"], exp["O"])


def _eltwise(N, C, body, out_agg="assign", dt="i32", extra_cons=""):
    return f"""block []:1 (
	in A[0, 0] {dt}({N}, {C}):({C}, 1)
	in Bias[0] {dt}({C}):(1)
	out O[0, 0]:assign {dt}({N}, {C}):({C}, 1)
) {{
	0:
	block [n:{N}, c:{C}]:{N * C} (
{extra_cons}		in A[n, c] {dt}(1, 1):({C}, 1)
		in Bias[c] {dt}(1):(1)
		out O[n, c]:{out_agg} {dt}(1, 1):({C}, 1)
	) {{
{body}
	}}
}}
"""


BIAS_RELU = "\t\t$a = load(A)\n\t\t$b = load(Bias)\n\t\t$s = add($a, $b)\n\t\t$z = constant(0)\n\t\t$r = max($s, $z)\n\t\tO = store($r)"
SELECT = ("\t\t$a = load(A)\n\t\t$b = load(Bias)\n\t\t$c = cmp_lt($a, $b)\n\t\t$m = mul($a, $b)\n"
          "\t\t$r = select($c, $m, $b)\n\t\tO = store($r)")


@pytest.mark.parametrize("dt", ["i8", "i32"])
@pytest.mark.parametrize("C", [64, 66])
def test_bias_relu_broadcast(dt, C):
    check(_eltwise(257, C, BIAS_RELU, dt=dt), expect_kernel="map" if C % 4 == 0 else "generic")


def test_select_chain_and_constraint_on_vector_dim():
    # the constraint cuts the vector dim mid-vector: lanes must be masked individually
    check(_eltwise(300, 64, SELECT, extra_cons="\t\t-c + 41 >= 0\n"))


def test_accumulating_output_add():
    check(_eltwise(128, 128, BIAS_RELU, out_agg="add"))
