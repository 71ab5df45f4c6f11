"""Config programs produced by the reference's own passes.

* configs/c3_pipeline_b{2,128}.stripe: config 3 after tile_rewrite -> fuse -> localize ->
  scalarize (tests/golden/make_pipeline_programs.py, test_passes.cpp:357-379) plans onto the
  resident-filter tensor-core conv with the bias/ReLU epilogue fused, and runs bit-exact.
* configs/c2_partition_n8_b{8,32}.stripe: config 2 after `partition index=n n=8`
  (tile.cpp:644-691): the banked program plans onto the same kernel, and each bank is a shard
  (restrict_index on the bank index) whose outputs are disjoint -- the multi-GPU carrier.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from harness import HERE, gpu_available

CONFIGS = os.path.join(os.path.dirname(HERE), "configs")


def _text(name):
    return open(os.path.join(CONFIGS, name)).read()


def test_c3_pipeline_program_plans_fused():
    import paper_1903_06498_b200 as sb
    for n in (2, 128):
        text = _text(f"c3_pipeline_b{n}.stripe")
        plan = sb.parse_program(text).describe_plan(True)
        assert "kernel=conv_i8_tc" in plan and "epilogue=vec+clamp" in plan, plan
        assert "never materialised" in plan, plan


def test_c3_pipeline_regenerates_identically():
    """The committed text is what the reference's passes produce (small case here)."""
    from oracle import Ref, reference_execute
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    import sys
    sys.path.insert(0, os.path.join(HERE, "golden"))
    import make_pipeline_programs as M
    assert M.make(2) == _text("c3_pipeline_b2.stripe")
    from paper_1903_06498_b200 import workloads as W
    assert Ref.pipeline(W.conv2d(8, 56, 56, 64, 64), M.PARTITION) == _text("c2_partition_n8_b8.stripe")


def test_c2_partition_program_plans_tc():
    import paper_1903_06498_b200 as sb
    plan = sb.parse_program(_text("c2_partition_n8_b32.stripe")).describe_plan(True)
    assert "kernel=conv_i8_tc" in plan, plan
    prog = sb.parse_program(_text("c2_partition_n8_b32.stripe"))
    shard = prog.restrict_index("0", "n", 3, 4)
    assert "kernel=conv_i8_tc" in shard.describe_plan(True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bank_worker(rank, world, port, out):
    import torch

    import paper_1903_06498_b200 as sb
    from oracle import Port, Ref, reference_execute
    from paper_1903_06498_b200 import workloads as W
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    text = Ref.pipeline(W.conv2d(4, 6, 6, 8, 4, in_dtype="i32"),
                        "mem HBM cap=1048576 line=128 banks=4\npass partition block=0 index=n n=4 unit=HBM\n")
    prog = sb.parse_program(text)
    store = Ref.random_inputs(Ref.parse(text), 17)
    base = {n: a for n, (b, a) in store.items()}
    o = base["O"].copy()
    for bank in range(rank, 4, world):  # this rank's banks: disjoint slices of O
        shard = sb.print_program(prog.restrict_index("0", "n", bank, bank + 1))
        part = reference_execute(shard, dict(base))["O"]
        changed = part != base["O"]
        o[changed] = part[changed]
    t = torch.from_numpy(o - base["O"])
    dist.all_reduce(t)  # disjoint banks: the sum of the deltas assembles the output
    if rank == 0:
        full = Ref.execute(Ref.parse(text), store)["O"][1]
        out["ok"] = bool(np.array_equal(base["O"] + t.numpy(), full))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_partition_banks_as_shards_gloo_world2():
    from oracle import Port, Ref, reference_execute
    if not (Port.available() and Ref.available()):
        pytest.skip("oracles not built")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bank_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["ok"]


def _dev():
    if not gpu_available():
        pytest.skip("no B200")
    import torch
    return torch


def _wrap(bits, x):
    import torch
    m = 1 << bits
    return torch.remainder(x + (m >> 1), m) - (m >> 1)


@pytest.mark.gpu
def test_c3_pipeline_b128_on_device_exact():
    torch = _dev()
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(_text("c3_pipeline_b128.stripe"))
    N, H, C, K = 128, 56, 64, 64
    g = torch.Generator(device="cuda").manual_seed(33)
    I = torch.randint(-128, 128, (N, H, H, C), dtype=torch.int8, device="cuda", generator=g)
    F = torch.randint(-128, 128, (3, 3, K, C), dtype=torch.int8, device="cuda", generator=g)
    B = torch.randint(-2**31, 2**31 - 1, (K,), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    O = torch.full((N, H, H, K), 3, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()  # the context's own stream does not wait for torch's
    ctx = sb.Context(0)
    ctx.execute_device(prog, {"I": (I.data_ptr(), I.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                              "Bias": (B.data_ptr(), B.numel(), 0), "O": (O.data_ptr(), O.numel(), sb.SB_BUF_PREPARE)})
    ctx.sync()
    t = torch.nn.functional.conv2d(I.permute(0, 3, 1, 2).double(), F.permute(2, 3, 0, 1).double(), padding=1)
    t = _wrap(32, t.permute(0, 2, 3, 1).round().long())
    assert torch.equal(O.long(), _wrap(32, torch.clamp(t + B.long(), min=0)))


@pytest.mark.gpu
def test_c3_pipeline_b2_vs_reference():
    _dev()
    from harness import run_device
    from oracle import Ref, reference_execute
    text = _text("c3_pipeline_b2.stripe")
    r = Ref.parse(text)
    store = Ref.random_inputs(r, 32)
    exp = Ref.execute(r, store)
    got = run_device(text, store)
    np.testing.assert_array_equal(got["O"], exp["O"][1])


@pytest.mark.gpu
def test_c2_partition_banks_on_device():
    torch = _dev()
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(_text("c2_partition_n8_b32.stripe"))
    N, H, C, K = 32, 56, 64, 64
    g = torch.Generator(device="cuda").manual_seed(8)
    I = torch.randint(-128, 128, (N, H, H, C), dtype=torch.int8, device="cuda", generator=g)
    F = torch.randint(-128, 128, (3, 3, K, C), dtype=torch.int8, device="cuda", generator=g)
    ref = torch.nn.functional.conv2d(I.permute(0, 3, 1, 2).double(), F.permute(2, 3, 0, 1).double(), padding=1)
    ref = ref.permute(0, 2, 3, 1).round().to(torch.int32)
    ctx = sb.Context(0)

    def run(p, O, flags):
        torch.cuda.synchronize()  # the context's own stream does not wait for torch's
        ctx.execute_device(p, {"I": (I.data_ptr(), I.numel(), 0), "F": (F.data_ptr(), F.numel(), 0),
                               "O": (O.data_ptr(), O.numel(), flags)})
        ctx.sync()
    O = torch.empty((N, H, H, K), dtype=torch.int32, device="cuda")
    run(prog, O, sb.SB_BUF_PREPARE)
    assert torch.equal(O, ref)
    # every bank as its own shard (what one rank of eight runs), accumulating into zeros
    O2 = torch.zeros_like(O)
    for b in range(8):
        run(prog.restrict_index("0", "n", b, b + 1), O2, 0)
        lo, hi = 4 * b, 4 * b + 4
        assert torch.equal(O2[lo:hi], ref[lo:hi]) and not O2[hi:].any()
