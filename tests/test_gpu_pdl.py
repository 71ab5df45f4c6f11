"""Programmatic-dependent-launch ordering across back-to-back executes on one stream.

The tensor-core kernels release their dependents only after their own griddepcontrol.wait
(capi.cpp run_plan / conv_tc.cu), and an immutable filter is fetched before the wait only
when no launch that may still run writes it.  These chains would read stale data if either
rule broke: step 3 reads step 1's output with an independent step 2 in between, and a
program whose FILTER is the previous execute's output."""
import numpy as np
import pytest

from harness import gpu_available

pytestmark = pytest.mark.gpu


def _dev():
    if not gpu_available():
        pytest.skip("no B200")
    import torch
    return torch


def _run_chain(torch, steps, sync_each):
    import paper_1903_06498_b200 as sb
    torch.cuda.synchronize()  # inputs written on torch's stream are complete
    ctx = sb.Context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        for prog, bufs in steps:
            ctx.execute_device(prog, bufs)
            if sync_each:
                ctx.sync()
        ctx.sync()
    torch.cuda.synchronize()


def _t(torch, shape, dtype, gen):
    if dtype == torch.int32:
        return torch.randint(-2**20, 2**20, shape, dtype=dtype, device="cuda", generator=gen)
    return torch.randint(-128, 128, shape, dtype=dtype, device="cuda", generator=gen)


def test_three_step_chain_step3_reads_step1():
    """step 1: fused conv (im2col kernel) writes X1 (i8); step 2: an independent resident-filter
    conv; step 3: a resident-filter conv reading X1 -- launched load-early (its window holds
    only step 2), so it must not start before step 1 has completed."""
    torch = _dev()
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    N, H, C = 8, 56, 64
    p1 = sb.parse_program(W.conv_fused(N, H, H, C, C))
    p2 = sb.parse_program(W.conv2d(N, H, H, C, C))
    assert "conv_i8_tc" in p2.describe_plan(True)
    g = torch.Generator(device="cuda").manual_seed(5)
    for trial in range(3):
        X0, Y0 = _t(torch, (N, H, H, C), torch.int8, g), _t(torch, (N, H, H, C), torch.int8, g)
        F, Bias = _t(torch, (3, 3, C, C), torch.int8, g), _t(torch, (C,), torch.int32, g)
        outs = {}
        for mode in (True, False):
            X1 = torch.empty((N, H, H, C), dtype=torch.int8, device="cuda")
            Y1, X2 = (torch.empty((N, H, H, C), dtype=torch.int32, device="cuda") for _ in range(2))
            s1 = {"I": (X0.data_ptr(), X0.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                  "Bias": (Bias.data_ptr(), Bias.numel(), 0), "O": (X1.data_ptr(), X1.numel(), sb.SB_BUF_PREPARE)}

            def conv(i, o):
                return {"I": (i.data_ptr(), i.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                        "O": (o.data_ptr(), o.numel(), sb.SB_BUF_PREPARE)}
            _run_chain(torch, [(p1, s1), (p2, conv(Y0, Y1)), (p2, conv(X1, X2))], sync_each=mode)
            outs[mode] = (X1.cpu().numpy(), Y1.cpu().numpy(), X2.cpu().numpy())
        for a, b in zip(outs[True], outs[False]):
            assert np.array_equal(a, b), f"trial {trial}: back-to-back executes differ from synced ones"


def test_filter_written_by_previous_execute():
    """Program B's filter F is program A's output: B must not fetch F early."""
    torch = _dev()
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    C = K = 64
    # A: conv_fused over a 3 x 3 x 64 x 64 "image" -> i8 output of the filter's shape (R, S, K, C)
    pa = sb.parse_program(W.conv_fused(3, 3, 64, C, K))
    pb = sb.parse_program(W.conv2d(16, 56, 56, C, K))
    assert "conv_i8_tc" in pb.describe_plan(True)
    g = torch.Generator(device="cuda").manual_seed(9)
    for trial in range(3):
        IA, FA, BA = _t(torch, (3, 3, 64, C), torch.int8, g), _t(torch, (3, 3, K, C), torch.int8, g), \
            _t(torch, (K,), torch.int32, g)
        IB = _t(torch, (16, 56, 56, C), torch.int8, g)
        res = {}
        for mode in (True, False):
            Fz = torch.full((3, 3, K, C), 7, dtype=torch.int8, device="cuda")
            OB = torch.empty((16, 56, 56, K), dtype=torch.int32, device="cuda")
            OB0 = torch.empty((16, 56, 56, K), dtype=torch.int32, device="cuda")
            steps = [(pb, {"I": (IB.data_ptr(), IB.numel(), 0), "F": (Fz.data_ptr(), Fz.numel(), 0),
                           "O": (OB0.data_ptr(), OB0.numel(), sb.SB_BUF_PREPARE)}),
                     (pa, {"I": (IA.data_ptr(), IA.numel(), 0), "F": (FA.data_ptr(), FA.numel(), 0),
                           "Bias": (BA.data_ptr(), BA.numel(), 0), "O": (Fz.data_ptr(), Fz.numel(), sb.SB_BUF_PREPARE)}),
                     (pb, {"I": (IB.data_ptr(), IB.numel(), 0), "F": (Fz.data_ptr(), Fz.numel(), 0),
                           "O": (OB.data_ptr(), OB.numel(), sb.SB_BUF_PREPARE)})]
            _run_chain(torch, steps, sync_each=mode)
            res[mode] = OB.cpu().numpy()
        assert np.array_equal(res[True], res[False]), f"trial {trial}"
