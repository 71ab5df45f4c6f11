"""Device executor vs the reference interpreter, bit-exact (integer programs).

Ground truth: tests/golden (made by the unmodified reference) and, when
oracle/_ref is present, live reference runs over fresh generator programs.
"""
import numpy as np
import pytest

from harness import corpus, gpu_available, run_device
from oracle import OracleError, Ref

pytestmark = pytest.mark.gpu
CASES = corpus()


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def check_case(case, disable_tc=False, order=0):
    import paper_1903_06498_b200 as sb
    if case.error:
        with pytest.raises(sb.ExecError) as e:
            run_device(case.text, case.inputs, disable_tc=disable_tc, order=order)
        assert e.value.code == case.error.split(":")[0], str(e.value)
        return
    out = run_device(case.text, case.inputs, disable_tc=disable_tc, order=order)
    for n, exp in case.expected.items():
        np.testing.assert_array_equal(out[n], exp, err_msg=f"{case.name}:{n}")


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
def test_golden(case):
    check_case(case)


@pytest.mark.parametrize("case", [c for c in CASES if c.name.startswith(("fx_", "gen_", "tile_", "pipe_"))],
                         ids=lambda c: c.name)
def test_golden_generic_kernels_only(case):
    check_case(case, disable_tc=True)


def test_iteration_order_option_accepted():
    for c in CASES:
        if c.name in ("fx_maxpool", "fx_conv_relu", "fx_fig6a_fixed_i32"):
            check_case(c, order=1)
            check_case(c, order=2)


def test_missing_and_wrong_size_buffers():
    import paper_1903_06498_b200 as sb
    c = next(x for x in CASES if x.name == "fx_copy16")
    prog = sb.parse_program(c.text)
    with pytest.raises(sb.ExecError) as e:
        sb.execute(prog, {})
    assert e.value.code == "MissingBuffer"
    with pytest.raises(sb.ExecError) as e:
        sb.execute(prog, {"A": sb.Buffer(32, np.zeros(3, np.int64)), "B": sb.Buffer(32, np.zeros(16, np.int64))})
    assert e.value.code == "MissingBuffer"


def test_observer_rejected():
    import paper_1903_06498_b200 as sb
    c = next(x for x in CASES if x.name == "fx_copy16")
    prog = sb.parse_program(c.text)
    store = {n: sb.Buffer(b, a.copy()) for n, (b, a) in c.inputs.items()}
    sb.prepare_outputs(prog, store)
    with pytest.raises(sb.ExecError) as e:
        sb.execute(prog, store, sb.ExecOptions(observer=object()))
    assert e.value.code == "Unsupported"


def test_inputs_untouched():
    """test_interp.cpp:170-177."""
    c = next(x for x in CASES if x.name == "fx_conv_relu")
    out = run_device(c.text, c.inputs)
    for n in ("I", "F"):
        np.testing.assert_array_equal(out[n], c.inputs[n][1])


ref = pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not present")


@ref
def test_live_random_programs():
    state = 4242
    for i in range(150):
        text, state = Ref.gen_random(state, text_variant=bool(i % 2))
        prog = Ref.parse(text)
        st = Ref.random_inputs(prog, 10_000 + i)
        exp = Ref.execute(prog, st)
        got = run_device(text, st)
        for n in exp:
            np.testing.assert_array_equal(got[n], exp[n][1], err_msg=f"program {i}\n{text}")


@ref
def test_live_tilings():
    """test_tile.cpp:94-113: random tilings preserve execution."""
    rng = np.random.default_rng(3131)
    for kind, args, bits in [("matmul", (20, 18, 22), 32), ("conv", (9, 11, 3, 5), 8), ("maxpool", (12, 10, 3), 16)]:
        base = Ref.gen(kind, *args, bits=bits)
        idx = {"matmul": lambda: dict(m=args[0], n=args[1], k=args[2]),
               "conv": lambda: dict(x=args[0], y=args[1], c=args[2], k=args[3]),
               "maxpool": lambda: dict(x=args[0] // 2, y=args[1] // 2, c=args[2])}[kind]()
        for t in range(6):
            tiles = ",".join(f"{n}:{int(rng.integers(1, min(6, r) + 1))}" for n, r in idx.items() if rng.random() < 0.7)
            tiles = tiles or f"{next(iter(idx))}:2"
            text = Ref.tile_rewrite(base, "0", tiles)
            prog = Ref.parse(text)
            st = Ref.random_inputs(prog, t)
            exp = Ref.execute(prog, st)
            got = run_device(text, st)
            for n in exp:
                np.testing.assert_array_equal(got[n], exp[n][1], err_msg=f"{kind} {tiles}")


def test_concurrent_host_threads_distinct_contexts():
    """SPEC.md:263 / SURVEY §8(b) threading: execute is reentrant; one context per host
    thread, the same parsed program shared (plans built under the program's lock)."""
    import threading

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    text = W.conv2d(2, 12, 12, 64, 64)
    prog = sb.parse_program(text)
    rng = np.random.default_rng(3)
    I = rng.integers(-128, 128, 2 * 12 * 12 * 64).astype(np.int64)
    F = rng.integers(-128, 128, 9 * 64 * 64).astype(np.int64)
    ref = {"I": sb.Buffer(8, I.copy()), "F": sb.Buffer(8, F.copy())}
    sb.prepare_outputs(prog, ref)
    sb.execute(prog, ref)
    errors, results = [], []

    def worker():
        try:
            ctx = sb.Context(0)
            for _ in range(5):
                st = {"I": sb.Buffer(8, I.copy()), "F": sb.Buffer(8, F.copy())}
                sb.prepare_outputs(prog, st)
                ctx.execute(prog, st)
                results.append(np.array_equal(st["O"].data, ref["O"].data))
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker) for _ in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors and len(results) == 20 and all(results)
