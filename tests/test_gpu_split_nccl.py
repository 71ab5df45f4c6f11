"""The split-aggregation combine through the C ABI (sb_split_allreduce over NCCL, SURVEY
§8(e)) on the B200.  One GPU is available here, so the communicator has one rank: the
all-reduce leaves each partial unchanged and the test pins that the NCCL path loads, runs
stream-ordered after the shard's kernels, keeps every output dtype (i8 direct, i16 widened to
i32 and narrowed back, i32) bit-exact, and refuses what it must.  The multi-rank arithmetic of
the combine (sum/max/min/prod with wrap) is covered by tests/test_multiproc.py (gloo, world 2)."""
import numpy as np
import pytest

from harness import gpu_available
from oracle import reference_execute
from paper_1903_06498_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def _run_shard_and_combine(text, path, idx, extent):
    import torch

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200.parallel import NcclComm, allreduce_outputs_device, shard_aggregation
    prog = sb.parse_program(text)
    shard = shard_aggregation(prog, path, idx, extent, 1, 0)
    rng = np.random.default_rng(3)
    ctx = sb.Context(0)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    dev, host_in = {}, {}
    torch_dt = {8: torch.int8, 16: torch.int16, 32: torch.int32}
    for n, d in prog.buffers.items():
        bits = int(d.dtype)
        if d.dir == sb.Dir.In:
            x = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), d.elements, dtype=np.int64)
            host_in[n] = x
            t = torch.from_numpy(x).to(torch_dt[bits]).cuda()
        else:
            t = torch.empty(d.elements, dtype=torch_dt[bits], device="cuda")
        dev[n] = t
    bufs = {n: (t.data_ptr(), t.numel(), sb.SB_BUF_PREPARE if prog.buffers[n].dir != sb.Dir.In else 0)
            for n, t in dev.items()}
    comm = NcclComm(ctx)
    with torch.cuda.stream(s):
        ctx.bind_device(shard, bufs)()
        outs = {n: (dev[n].data_ptr(), dev[n].numel()) for n, d in prog.buffers.items() if d.dir != sb.Dir.In}
        allreduce_outputs_device(ctx, prog, outs, comm)
        ctx.sync()
    comm.close()
    store = dict(host_in)
    for n, d in prog.buffers.items():
        if d.dir != sb.Dir.In:
            store[n] = np.full(d.elements, prog.output_identity(n), np.int64)
    exp = reference_execute(text, store)
    for n in outs:
        np.testing.assert_array_equal(dev[n].cpu().numpy().astype(np.int64), exp[n])
    return prog, ctx, dev


@pytest.mark.parametrize("case", [
    ("matmul_i32", lambda: W.matmul(64, 48, 96, in_dtype="i32", out_dtype="i32"), "0", "k", 96),
    ("matmul_i8_i16", lambda: W.matmul(64, 48, 96, in_dtype="i8", out_dtype="i16"), "0", "k", 96),
    ("gsum_i8", lambda: W.global_sum(4, 7, 5, 64, in_dtype="i8", out_dtype="i8"), "0", "x", 7),
    ("pool_max", lambda: W.maxpool2x2(2, 6, 8, 16), "0", "i", 2),
], ids=lambda c: c[0])
def test_split_combine_through_c_abi(case):
    _, make, path, idx, extent = case
    _run_shard_and_combine(make(), path, idx, extent)


def test_split_combine_refusals():
    import ctypes

    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200.parallel import NcclComm
    ctx = sb.Context(0)
    comm = NcclComm(ctx)
    prog = sb.parse_program(W.matmul(8, 8, 8, in_dtype="i32", out_dtype="i32"))
    buf = ctypes.c_void_p()
    sb._check(sb.lib().sb_device_alloc(ctx.handle, 64 * 4, ctypes.byref(buf)))
    with pytest.raises(sb.ExecError) as e:  # wrong element count
        sb._check(sb.lib().sb_split_allreduce(ctx.handle, prog.handle, b"C", buf, 63, comm.handle))
    assert e.value.code == "MissingBuffer"
    with pytest.raises(sb.ExecError) as e:  # an input is not combined
        sb._check(sb.lib().sb_split_allreduce(ctx.handle, prog.handle, b"A", buf, 64, comm.handle))
    assert e.value.code == "Unsupported"
    # the root output of a matmul is `assign`ed, its writer aggregates with add: combinable
    sb._check(sb.lib().sb_split_allreduce(ctx.handle, prog.handle, b"C", buf, 64, comm.handle))
    ctx.sync()
    sb._check(sb.lib().sb_device_free(ctx.handle, buf))
    comm.close()
