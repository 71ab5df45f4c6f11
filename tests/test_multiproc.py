"""N>1 host logic on CPU (gloo, world_size 2): batch sharding of a conv program is exact
(each rank's shard program over its slice == the corresponding slice of the full program),
and the max-over-ranks reduction the bench uses."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_06498_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch

    from oracle import Port, Rng, wrap, reference_execute
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, H, Wd, C, K = 4, 5, 6, 8, 4
    rng = Rng(99)
    I = wrap(8, rng.bulk(N * H * Wd * C)).reshape(N, H * Wd * C)
    F = wrap(8, rng.bulk(9 * K * C))
    lo, hi = W.shard_range(N, world, rank)
    text = W.conv2d(hi - lo, H, Wd, C, K)
    o = reference_execute(text, {"I": I[lo:hi].ravel(), "F": F, "O": np.zeros((hi - lo) * H * Wd * K, np.int64)})["O"]
    objs = [None] * world
    dist.all_gather_object(objs, o)
    gathered = [torch.from_numpy(x.astype(np.float64)) for x in objs]
    elapsed = torch.tensor([1.0 + rank])  # bench.py: device time reduced with MAX over ranks
    dist.all_reduce(elapsed, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = reference_execute(W.conv2d(N, H, Wd, C, K), {"I": I.ravel(), "F": F,
                                                       "O": np.zeros(N * H * Wd * K, np.int64)})["O"]
        out["ok"] = bool(np.array_equal(torch.cat(gathered).numpy().astype(np.int64), full))
        out["max"] = float(elapsed.item())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_batch_sharding_gloo_world2():
    from oracle import Port, reference_execute
    if not Port.available():
        pytest.skip("oracle/_port not built")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["ok"]
    assert out["max"] == 2.0


def test_shard_range_partitions():
    for total in (1, 5, 32, 1024):
        for world in (1, 2, 3, 8):
            spans = [W.shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


# ---- split aggregation (SURVEY §8(e) optional demo): shards + all-reduce -----------------

def _split_worker(rank, world, port, out):
    import torch

    import paper_1903_06498_b200 as sb
    from oracle import Port, Rng, wrap, reference_execute
    from paper_1903_06498_b200.parallel import allreduce_outputs, shard_aggregation
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cases = {
        # split-K of an i32 matmul (add -> SUM, wrap mod 2^32)
        "matmul": (W.matmul(12, 10, 37, in_dtype="i32", out_dtype="i32"), "0", "k", 37),
        # a global sum split over rows (add)
        "gsum": (W.global_sum(3, 7, 5, 16), "0", "x", 7),
        # max-pool taps split across ranks (max -> MAX)
        "pool": (W.maxpool2x2(2, 6, 8, 16), "0", "i", 2),
    }
    ok = {}
    for name, (text, path, idx, extent) in cases.items():
        prog = sb.parse_program(text)
        rng = Rng(500 + len(name))
        inputs = {}
        for n, d in prog.buffers.items():
            if d.dir == sb.Dir.Out:
                continue
            inputs[n] = wrap(int(d.dtype), rng.bulk(d.elements))
        shard = shard_aggregation(prog, path, idx, extent, world, rank)
        store = dict(inputs)
        for n, d in prog.buffers.items():
            if d.dir != sb.Dir.In:
                store[n] = np.full(d.elements, prog.output_identity(n), np.int64)  # fresh on every rank
        part = reference_execute(sb.print_program(shard), store)
        outs = {n: torch.from_numpy(part[n].copy()) for n, d in prog.buffers.items() if d.dir != sb.Dir.In}
        allreduce_outputs(prog, outs)
        full_store = dict(inputs)
        for n, d in prog.buffers.items():
            if d.dir != sb.Dir.In:
                full_store[n] = np.full(d.elements, prog.output_identity(n), np.int64)
        full = reference_execute(text, full_store)
        ok[name] = all(np.array_equal(outs[n].numpy(), full[n]) for n in outs)
    if rank == 0:
        out.update(ok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_split_aggregation_gloo_world2():
    from oracle import Port, reference_execute
    if not Port.available():
        pytest.skip("oracle/_port not built")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_split_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert dict(out) == {"matmul": True, "gsum": True, "pool": True}, dict(out)


def test_restrict_index_rejects_assign_outputs():
    import torch  # noqa: F401
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200.parallel import AGG_OPS
    prog = sb.parse_program(W.matmul(4, 4, 4))
    assert AGG_OPS[prog.output_aggregation("C")] == "SUM"
    with pytest.raises(sb.ExecError):
        prog.restrict_index("0", "q", 0, 1)


@pytest.mark.gpu
def test_split_k_shards_on_device():
    """The shard programs of a split-K i8 matmul run on the B200 kernels (16-aligned k slices
    stay on the tcgen05 GEMM) and their wrapped sum equals the full product."""
    from harness import gpu_available
    if not gpu_available():
        pytest.skip("no B200")
    import paper_1903_06498_b200 as sb
    from oracle import Rng, wrap, reference_execute
    from paper_1903_06498_b200.parallel import shard_aggregation
    text = W.matmul(256, 128, 512, in_dtype="i8", out_dtype="i32")
    prog = sb.parse_program(text)
    rng = Rng(77)
    A = wrap(8, rng.bulk(256 * 512))
    B = wrap(8, rng.bulk(512 * 128))
    total = np.zeros(256 * 128, np.int64)
    for r in range(4):
        shard = shard_aggregation(prog, "0", "k", 512, 4, r)
        assert "gemm_i8_tc" in shard.describe_plan(True)
        st = {"A": sb.Buffer(8, A.copy()), "B": sb.Buffer(8, B.copy())}
        sb.prepare_outputs(shard, st)
        sb.execute(shard, st)
        total += st["C"].data
    full = (A.reshape(256, 512) @ B.reshape(512, 128)).ravel()
    np.testing.assert_array_equal(wrap(32, total.astype(np.uint64)), wrap(32, full.astype(np.uint64)))


def test_check_split_accepts_linear_and_rejects_nonlinear():
    """a split is exact only when every path from the index to an output is a
    combine with the output's own aggregation (sb_program_check_split)."""
    import paper_1903_06498_b200 as sb
    ok = [(W.matmul(12, 10, 37), "0", "k"), (W.global_sum(3, 7, 5, 16), "0", "x"),
          (W.maxpool2x2(2, 6, 8, 16), "0", "i"), (W.conv2d(2, 6, 6, 8, 4, in_dtype="i32"), "0", "c")]
    for text, path, idx in ok:
        sb.parse_program(text).check_split(path, idx)
    # conv -> local T (declared above the leaf) -> bias + relu -> O:assign: relu(partial) != partial
    fused = sb.parse_program(W.conv_fused(1, 6, 6, 64, 64))
    with pytest.raises(sb.ExecError) as e:
        fused.check_split("0.0", "c")
    assert e.value.code == "Unsupported"
    # the epilogue block's own index writes an assigned output
    with pytest.raises(sb.ExecError):
        fused.check_split("0.1", "k")
    # unknown index
    with pytest.raises(sb.ExecError) as e:
        fused.check_split("0.0", "zz")
    assert e.value.code == "UnboundIndex"


def test_restrict_index_shifts_tile_aliases_fig6b():
    """restrict_index on the outer tile index of a tile_rewrite output shifts the
    child's `xo = 3*x` alias even though the child's own ranged x is declared before it.
    Shards of x (a partition index here) run one after the other over the same store must
    equal the full program (reference fixture testdata/fig6b.stripe)."""
    import paper_1903_06498_b200 as sb
    from harness import corpus
    from oracle import Ref, reference_execute
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    case = next(c for c in corpus() if c.name == "fx_fig6b")
    prog = sb.parse_program(case.text)
    # the unmodified reference runs both the full program and the shards
    full = Ref.execute(Ref.parse(case.text), dict(case.inputs))
    for cuts in ((0, 2, 4), (0, 1, 3, 4)):
        store = dict(case.inputs)
        for lo, hi in zip(cuts, cuts[1:]):
            shard = prog.restrict_index("0", "x", lo, hi)
            store = Ref.execute(Ref.parse(sb.print_program(shard)), store)
        for n in full:
            assert np.array_equal(store[n][1], full[n][1]), (cuts, n)
    assert not np.array_equal(full["O"][1], case.inputs["O"][1])
