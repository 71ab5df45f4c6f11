"""Parity at the EXACT shapes the bench lines are quoted on (VERDICT r1 "what's weak" 1).

* C3, batch 128: conv_i8_tc with the fused bias/ReLU epilogue runs ~24 tiles per CTA, so
  both epilogue groups and the TMEM double-buffer phase flips run with the fused epilogue;
  full-range int32 biases take the exact threshold form, small ones the fast form.
* C4a, 128x112x112x64 i32 max-pool: the reduce kernel's grid-stride loop (~10 iterations
  per thread at this size).
* C4b, 1024x7x7x2048 global sum at full shape.
* C5, the ResNet-50 program at the 128 images one GPU runs in the 8-GPU split of batch 1024,
  against the exact restatement (tests/intmodel.py, pinned on the reference's golden logits
  in test_resnet.py).
Checkers are exact integer restatements in PyTorch (int64 / float64 below 2^53)."""
import numpy as np
import pytest

from harness import gpu_available

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def _ctx():
    """A context on its own (non-blocking) stream: every execute below is preceded by
    torch.cuda.synchronize() so the inputs torch wrote on its stream are complete."""
    import torch
    import paper_1903_06498_b200 as sb
    torch.cuda.synchronize()
    return sb.Context(0)


def _wrap(bits, x):
    import torch
    m = 1 << bits
    return torch.remainder(x + (m >> 1), m) - (m >> 1)


@pytest.mark.parametrize("bias", ["full_range", "small"])
def test_c3_b128_fused_epilogue_full_shape(bias):
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, Wd, C, K = 128, 56, 56, 64, 64
    prog = sb.parse_program(W.conv_bias_relu(N, H, Wd, C, K))
    plan = prog.describe_plan(True)
    assert "conv_i8_tc" in plan and "epilogue of" in plan, plan
    g = torch.Generator(device="cuda").manual_seed(1003)
    I = torch.randint(-128, 128, (N, H, Wd, C), dtype=torch.int8, device="cuda", generator=g)
    F = torch.randint(-128, 128, (3, 3, K, C), dtype=torch.int8, device="cuda", generator=g)
    if bias == "full_range":
        B = torch.randint(-2**31, 2**31 - 1, (K,), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    else:
        B = torch.randint(-5000, 5000, (K,), dtype=torch.int32, device="cuda", generator=g)
    O = torch.full((N, H, Wd, K), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    ctx = _ctx()
    ctx.execute_device(prog, {"I": (I.data_ptr(), I.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                              "Bias": (B.data_ptr(), B.numel(), 0),
                              "O": (O.data_ptr(), O.numel(), sb.SB_BUF_PREPARE)})
    ctx.sync()
    t = torch.nn.functional.conv2d(I.permute(0, 3, 1, 2).double(), F.permute(2, 3, 0, 1).double(), padding=1)
    t = _wrap(32, t.permute(0, 2, 3, 1).round().long())
    exp = _wrap(32, torch.clamp(t + B.long(), min=0))
    assert torch.equal(O.long(), exp)


def test_c4a_maxpool_full_shape():
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, Wd, C = 128, 112, 112, 64
    prog = sb.parse_program(W.maxpool2x2(N, H, Wd, C))
    assert "kernel=reduce" in prog.describe_plan(True) or "kernel=pool" in prog.describe_plan(True)
    g = torch.Generator(device="cuda").manual_seed(1004)
    I = torch.randint(-2**31, 2**31 - 1, (N, H, Wd, C), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    O = torch.full((N, H // 2, Wd // 2, C), 777, dtype=torch.int32, device="cuda")
    ctx = _ctx()
    ctx.execute_device(prog, {"I": (I.data_ptr(), I.numel(), 0), "O": (O.data_ptr(), O.numel(), sb.SB_BUF_PREPARE)})
    ctx.sync()
    exp = I.view(N, H // 2, 2, Wd // 2, 2, C).amax(dim=(2, 4))
    assert torch.equal(O, exp)
    # accumulate into existing contents (no prepare): max(old, window)
    O2 = torch.randint(-2**31, 2**31 - 1, O.shape, dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    old = O2.clone()
    torch.cuda.synchronize()
    ctx.execute_device(prog, {"I": (I.data_ptr(), I.numel(), 0), "O": (O2.data_ptr(), O2.numel(), 0)})
    ctx.sync()
    assert torch.equal(O2, torch.maximum(old, exp))


def test_c4b_global_sum_full_shape():
    import torch
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, Wd, C = 1024, 7, 7, 2048
    prog = sb.parse_program(W.global_sum(N, H, Wd, C))
    g = torch.Generator(device="cuda").manual_seed(1004)
    I = torch.randint(-2**31, 2**31 - 1, (N, H, Wd, C), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    O = torch.full((N, C), -1, dtype=torch.int32, device="cuda")
    ctx = _ctx()
    ctx.execute_device(prog, {"I": (I.data_ptr(), I.numel(), 0), "O": (O.data_ptr(), O.numel(), sb.SB_BUF_PREPARE)})
    ctx.sync()
    exp = _wrap(32, I.long().sum(dim=(1, 2)))
    assert torch.equal(O.long(), exp)


def test_c5_resnet50_128_images_vs_exact():
    """The bench's per-GPU C5 shard (128 images of batch 1024) end to end, bit-exact."""
    import paper_1903_06498_b200 as sb
    from intmodel import resnet_exact
    from oracle import random_inputs
    from paper_1903_06498_b200 import workloads as W
    text, info = W.resnet50(128)
    prog = sb.parse_program(text)
    bufs = [(n, int(d.dtype), d.elements, int(d.dir)) for n, d in prog.buffers.items()]
    inputs = random_inputs(bufs, 1005)
    store = {n: sb.Buffer(prog.buffers[n].dtype, a.copy()) for n, a in inputs.items()}
    sb.prepare_outputs(prog, store)
    sb.execute(prog, store)
    exp = resnet_exact(info, inputs, 224, 64, (3, 4, 6, 3), 1000).ravel()
    np.testing.assert_array_equal(store["Logits"].data, exp)
