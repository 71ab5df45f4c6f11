"""Multi-GPU sharding of Stripe programs, one process per GPU.

* Partitioned indexes (batch n, output channels, rows m): each rank runs the program over
  its contiguous slice (workloads.shard_range); outputs are disjoint, no collective.
* Split aggregation (optional demo: split-K of a matmul, a huge global sum): each rank runs
  `shard_aggregation(...)` — the program with the aggregation index restricted to its slice
  (sb_program_restrict_index) — into FRESH outputs (prepare_outputs' identity), and
  `allreduce_outputs` combines the partials with the output's aggregation: add -> SUM,
  max -> MAX, min -> MIN, mul -> PRODUCT (NCCL over NVLink on B200; gloo on CPU).  Integer
  outputs wrap modulo 2^bits exactly like the reference's store (the wrapping sum of wrapped
  partials is the wrapped total), so the split is bit-exact.
"""
from typing import Dict

import numpy as np

from . import Dir, Program
from .workloads import shard_range

AGG_OPS = {1: "SUM", 2: "MAX", 3: "MIN", 4: "PRODUCT"}


def shard_aggregation(program: Program, block_path: str, index: str, extent: int, world: int, rank: int) -> Program:
    program.check_split(block_path, index)  # exact only when every path is a linear combine
    lo, hi = shard_range(extent, world, rank)
    return program.restrict_index(block_path, index, lo, hi)


def _wrap(x: np.ndarray, bits: int) -> np.ndarray:
    m = 1 << bits
    return ((x + (m >> 1)) % m) - (m >> 1)


def allreduce_outputs(program: Program, outputs: Dict[str, object], group=None) -> None:
    """outputs: name -> torch tensor (int64 carriers on CPU/gloo, or native-width on GPU/NCCL),
    reduced in place across `group` with each output's aggregation.  The shards must come
    from shard_aggregation (whose check_split proves the combine exact)."""
    import torch
    import torch.distributed as dist
    for name, t in outputs.items():
        decl = program.buffers[name]
        if decl.dir == Dir.In:
            continue
        agg = program.output_aggregation(name)
        if agg not in AGG_OPS:
            raise ValueError(f"output '{name}' is assigned, not aggregated: it cannot be split")
        dist.all_reduce(t, op=getattr(dist.ReduceOp, AGG_OPS[agg]), group=group)
        if t.dtype == torch.int64 and int(decl.dtype) in (8, 16, 32):
            t.copy_(torch.from_numpy(_wrap(t.cpu().numpy(), int(decl.dtype))).to(t.device))


class NcclComm:
    """An NCCL communicator made through the C ABI (sb_nccl_unique_id on rank 0, broadcast
    with torch.distributed -- gloo or nccl -- then sb_nccl_comm_init on every rank)."""

    def __init__(self, ctx, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _check, lib
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _check(lib().sb_nccl_unique_id(uid))
        box = [uid.raw]
        if world > 1:
            dist.broadcast_object_list(box, src=0, group=group)
        h = ctypes.c_void_p()
        _check(lib().sb_nccl_comm_init(ctx.handle, world, box[0], rank, ctypes.byref(h)))
        self.handle, self.ctx, self.world, self.rank = h.value, ctx, world, rank

    def close(self):
        from . import _check, lib
        if self.handle:
            _check(lib().sb_nccl_comm_destroy(self.handle))
            self.handle = None


def allreduce_outputs_device(ctx, program: Program, outputs: Dict[str, tuple], comm: NcclComm) -> None:
    """The C-ABI combine (sb_split_allreduce): outputs name -> (device_ptr, count) at native
    width, reduced in place on ctx's stream with each output's aggregation over NCCL."""
    from . import _check, lib
    for name, (ptr, count) in outputs.items():
        _check(lib().sb_split_allreduce(ctx.handle, program.handle, name.encode(), ptr, count, comm.handle))
