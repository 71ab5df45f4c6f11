"""Config 5: the ResNet-50-shaped Stripe program (workloads.resnet50) end to end.

CPU: the generated program is validate_static clean in the reference, and the reference
and the CPU restatement agree on a reduced-width variant.  GPU: bit-exact logits against
the reference's golden logits (tests/golden/resnet/, made by make_golden_resnet.py from
the unmodified interpreter) at full widths, and the exact PyTorch restatement
(tests/intmodel.py) pinned on the same case.
"""
import os

import numpy as np
import pytest

from harness import GOLDEN, gpu_available
from oracle import Port, Ref, random_inputs, reference_execute

TINY = dict(image=32, width=8, stages=(1, 1, 1, 1), classes=10)


def test_tiny_resnet_reference_vs_port():
    from paper_1903_06498_b200 import workloads as W
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    text, info = W.resnet50(1, **TINY)
    prog = Ref.parse(text)
    assert prog.validate()[0] == 0
    store = Ref.random_inputs(prog, 1005)
    out = Ref.execute(prog, store)
    port = Port.execute(text, {n: a for n, (b, a) in store.items()})
    np.testing.assert_array_equal(out["Logits"][1], port["Logits"])


def test_resnet_structure():
    from paper_1903_06498_b200 import workloads as W
    import paper_1903_06498_b200 as sb
    text, info = W.resnet50(2)
    assert len(info["convs"]) == 53
    assert abs(info["macs"] / 2 - 4.09e9) / 4.09e9 < 0.05  # 3.95e9 useful MAC/img (+fc)
    plan = sb.parse_program(text).describe_plan()
    assert plan.count("kernel=conv_igemm_tc") + plan.count("kernel=conv_i8_tc") >= 40, plan
    # the 7x7/2 stem on 3 channels runs phase-folded (2x2 fold, 16-byte folded pixels) on the
    # im2col tensor-core kernel; the max-pool absorbs its output's zero fill
    assert "small-channel conv phase-folded (2x2, 16 bytes per folded pixel)" in plan, plan
    assert "kernel=pool" in plan and "(elided) fill alloc:0:Pool" in plan, plan
    # bias + residual + ReLU fuse into the producing conv (the residual add runs on the
    # tensor core inside the kernel): one per bottleneck block
    assert plan.count("epilogue=vec+res+clamp") == 16, plan


def golden(name):
    path = os.path.join(GOLDEN, "resnet", name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} golden not generated")
    return np.load(path)


def run_device(text, prog_buffers, seed):
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(text)
    bufs = [(n, int(d.dtype), d.elements, int(d.dir)) for n, d in prog.buffers.items()]
    inputs = random_inputs(bufs, seed)
    store = {n: sb.Buffer(prog.buffers[n].dtype, a.copy()) for n, a in inputs.items()}
    sb.prepare_outputs(prog, store)
    sb.execute(prog, store)
    return inputs, store["Logits"].data


@pytest.mark.gpu
def test_tiny_resnet_gpu_vs_reference():
    if not gpu_available():
        pytest.skip("no B200")
    from paper_1903_06498_b200 import workloads as W
    text, info = W.resnet50(1, **TINY)
    _, logits = run_device(text, None, 1005)
    port_inputs = None
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(text)
    bufs = [(n, int(d.dtype), d.elements, int(d.dir)) for n, d in prog.buffers.items()]
    store = random_inputs(bufs, 1005)
    store["Logits"] = np.zeros(prog.buffers["Logits"].elements, dtype=np.int64)
    port = reference_execute(text, store)
    np.testing.assert_array_equal(logits, port["Logits"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["resnet50_img32_b2", "resnet50_img224_b1"])
def test_resnet_gpu_vs_reference_golden(name):
    if not gpu_available():
        pytest.skip("no B200")
    from paper_1903_06498_b200 import workloads as W
    from intmodel import resnet_exact
    g = golden(name)
    N, image = int(g["N"]), int(g["image"])
    text, info = W.resnet50(N, image=image)
    inputs, logits = run_device(text, None, int(g["seed"]))
    np.testing.assert_array_equal(logits, g["logits"])
    # the torch restatement agrees with the reference too (pins it for larger batches)
    exp = resnet_exact(info, inputs, image, 64, (3, 4, 6, 3), 1000).ravel()
    np.testing.assert_array_equal(exp, g["logits"])


@pytest.mark.gpu
def test_resnet_batch8_vs_intmodel():
    if not gpu_available():
        pytest.skip("no B200")
    from paper_1903_06498_b200 import workloads as W
    from intmodel import resnet_exact
    text, info = W.resnet50(8)
    inputs, logits = run_device(text, None, 77)
    exp = resnet_exact(info, inputs, 224, 64, (3, 4, 6, 3), 1000).ravel()
    np.testing.assert_array_equal(logits, exp)
