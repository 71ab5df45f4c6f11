"""B200-native execution backend for the Stripe IR (arXiv 1903.06498 reference).

Python mirror of the reference's executor API (proj/include/stripe/interp.h,
text.h) over the C ABI in include/stripe_b200.h:

    parse_program(text)                     text.h:20     -> Program
    print_program(program)                  text.h:23
    prepare_outputs(program, store)         interp.h:73
    execute(program, store, opts=None)      interp.h:68   (store updated in place)
    Buffer(dtype, data) / BufferStore       interp.h:14-20
    ExecOptions / IterOrder                 interp.h:58-64
    ExecError(code, message)                interp.h:22-26

All compute runs in libstripe_b200.so (hand-written sm_100a kernels).  There is
no CPU fallback: without the built library, or without a Blackwell GPU,
execute() raises.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SB_LIBRARY: development override (e.g. the `make trace` build); default the in-tree library
LIB_PATH = os.environ.get("SB_LIBRARY") or os.path.join(_HERE, "libstripe_b200.so")

SB_I8, SB_I16, SB_I32, SB_F32 = 8, 16, 32, 0x20F
SB_CARRIER_I64, SB_CARRIER_NATIVE = 0, 1
SB_BUF_PREPARE = 1
STATUS_NAMES = [
    "Ok", "MissingBuffer", "UnknownIntrinsic", "UnknownSpecial", "UndefinedTemp",
    "OutOfBoundsAccess", "UnboundIndex", "SyntaxError", "ScopeError", "Unsupported",
    "CudaError", "NcclError", "Invalid", "PassError",
]

# Every symbol include/stripe_b200.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "sb_last_error", "sb_status_name", "sb_abi_version",
    "sb_program_parse", "sb_program_free", "sb_program_print", "sb_program_buffer_count",
    "sb_program_buffer_info", "sb_program_output_identity", "sb_program_describe_plan",
    "sb_program_output_aggregation", "sb_program_restrict_index", "sb_program_check_split", "sb_count_valid_points",
    "sb_tile_cost", "sb_autotile", "sb_nccl_unique_id", "sb_nccl_comm_init", "sb_nccl_comm_destroy",
    "sb_split_allreduce",
    "sb_context_create", "sb_context_destroy", "sb_context_set_stream", "sb_context_stream",
    "sb_context_set_kernel_order",
    "sb_context_sync", "sb_context_launch_count", "sb_context_set_profile", "sb_context_profile_read", "sb_device_alloc", "sb_device_free",
    "sb_host_alloc_pinned", "sb_host_free_pinned", "sb_execute", "sb_execute_device", "sb_execute_async",
    "sb_graph_begin", "sb_graph_end", "sb_graph_launch", "sb_graph_free",
]


class HostBuffer(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("carrier", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("data", ctypes.c_void_p), ("count", ctypes.c_int64)]


class TileReport(ctypes.Structure):
    """TileCostReport (passes.h:42-50): cost() = lines_total / useful_ops; excluded = "MemCap"."""
    _fields_ = [("lines_total", ctypes.c_int64), ("useful_ops", ctypes.c_int64), ("tile_elements", ctypes.c_int64),
                ("_excluded", ctypes.c_int32)]

    @property
    def excluded(self):
        return "MemCap" if self._excluded else None

    def as_tuple(self):
        return (self.lines_total, self.useful_ops, self.tile_elements, bool(self._excluded))


class AutotileResult:
    """AutotileResult (passes.h:76-83) without the rewritten block: apply the reference's
    tile_rewrite to `chosen` (TileShape::to_string text, or None when every candidate was
    excluded: the reference's NoFeasibleTile warning)."""

    def __init__(self, chosen, report, candidates, excluded):
        self.chosen, self.report, self.candidates, self.excluded = chosen, report, candidates, excluded


class DeviceBuffer(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("dptr", ctypes.c_void_p), ("count", ctypes.c_int64)]


class _Opts(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("observer", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("disable_tensor_cores", ctypes.c_int32), ("fp32_mode", ctypes.c_int32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Loads the in-tree library; raises loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_1903_06498_b200)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.sb_last_error.restype = ctypes.c_char_p
        L.sb_status_name.restype = ctypes.c_char_p
        L.sb_program_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
        L.sb_program_free.argtypes = [vp]
        L.sb_program_free.restype = None
        L.sb_program_print.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.sb_program_buffer_count.argtypes = [vp]
        L.sb_program_buffer_info.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(i32),
                                             ctypes.POINTER(i64), ctypes.POINTER(i32)]
        L.sb_program_output_identity.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(i64)]
        L.sb_program_output_aggregation.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(i32)]
        L.sb_program_restrict_index.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p, i64, i64, ctypes.POINTER(vp)]
        L.sb_program_check_split.argtypes = [vp, ctypes.c_char_p, ctypes.c_char_p]
        L.sb_count_valid_points.argtypes = [vp, vp, ctypes.c_char_p, ctypes.POINTER(i64)]
        L.sb_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.sb_nccl_comm_init.argtypes = [vp, i32, ctypes.c_char_p, i32, ctypes.POINTER(vp)]
        L.sb_nccl_comm_destroy.argtypes = [vp]
        L.sb_split_allreduce.argtypes = [vp, vp, ctypes.c_char_p, vp, i64, vp]
        L.sb_tile_cost.argtypes = [vp, vp, ctypes.c_char_p, ctypes.c_char_p, i32, i64, i64, ctypes.POINTER(TileReport)]
        L.sb_autotile.argtypes = [vp, vp, ctypes.c_char_p, i64, i64, i32, ctypes.c_char_p, ctypes.c_size_t,
                                  ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(i32), ctypes.POINTER(TileReport),
                                  ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.sb_program_describe_plan.argtypes = [vp, i32, i32, ctypes.c_char_p, ctypes.c_size_t,
                                               ctypes.POINTER(ctypes.c_size_t)]
        L.sb_context_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.sb_context_destroy.argtypes = [vp]
        L.sb_context_destroy.restype = None
        L.sb_context_set_stream.argtypes = [vp, vp]
        L.sb_context_set_kernel_order.argtypes = [vp, i32]
        L.sb_context_stream.argtypes = [vp]
        L.sb_context_stream.restype = vp
        L.sb_context_sync.argtypes = [vp]
        L.sb_context_launch_count.argtypes = [vp]
        L.sb_context_launch_count.restype = ctypes.c_uint64
        L.sb_context_set_profile.argtypes = [vp, i32]
        L.sb_context_profile_read.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.sb_device_alloc.argtypes = [vp, i64, ctypes.POINTER(vp)]
        L.sb_device_free.argtypes = [vp, vp]
        L.sb_host_alloc_pinned.argtypes = [i64, ctypes.POINTER(vp)]
        L.sb_host_free_pinned.argtypes = [vp]
        L.sb_execute.argtypes = [vp, vp, ctypes.POINTER(HostBuffer), i32, ctypes.POINTER(_Opts)]
        L.sb_execute_device.argtypes = [vp, vp, ctypes.POINTER(DeviceBuffer), i32, ctypes.POINTER(_Opts)]
        L.sb_execute_async.argtypes = [vp, vp, ctypes.POINTER(HostBuffer), i32, ctypes.POINTER(_Opts)]
        L.sb_graph_begin.argtypes = [vp]
        L.sb_graph_end.argtypes = [vp, ctypes.POINTER(vp)]
        L.sb_graph_launch.argtypes = [vp, vp]
        L.sb_graph_free.argtypes = [vp]
        L.sb_graph_free.restype = None
        _lib = L
    return _lib


class ExecError(RuntimeError):
    """Mirror of stripe::ExecError / ParseError: `.code` is the reference's code string."""

    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().sb_last_error().decode(errors="replace")
        code = STATUS_NAMES[rc] if 0 <= rc < len(STATUS_NAMES) else "Invalid"
        if code == "PassError":  # PassError{code}: InvalidTile / NotTileable (passes.h)
            code = msg.split(":", 1)[0]
        raise ExecError(code, msg)


class DType(enum.IntEnum):
    i8 = 8
    i16 = 16
    i32 = 32
    f32 = SB_F32


_NP = {8: np.int8, 16: np.int16, 32: np.int32, SB_F32: np.float32}


class Dir(enum.IntEnum):
    In = 0
    Out = 1
    InOut = 2


@dataclass
class BufferDecl:
    dtype: int
    elements: int
    dir: Dir


class Program:
    """A parsed Stripe program (owning an sb_program handle)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        L = lib()
        self.buffers: Dict[str, BufferDecl] = {}
        for i in range(L.sb_program_buffer_count(self._h)):
            name = ctypes.c_char_p()
            dt, el, dr = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int()
            _check(L.sb_program_buffer_info(self._h, i, ctypes.byref(name), ctypes.byref(dt), ctypes.byref(el),
                                            ctypes.byref(dr)))
            self.buffers[name.value.decode()] = BufferDecl(dt.value, el.value, Dir(dr.value))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.sb_program_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def output_identity(self, name: str) -> int:
        v = ctypes.c_int64()
        _check(lib().sb_program_output_identity(self._h, name.encode(), ctypes.byref(v)))
        return v.value

    def output_aggregation(self, name: str) -> int:
        """0 assign, 1 add, 2 max, 3 min, 4 mul (interp.cpp:620-632)."""
        v = ctypes.c_int()
        _check(lib().sb_program_output_aggregation(self._h, name.encode(), ctypes.byref(v)))
        return v.value

    def restrict_index(self, block_path: str, index: str, lo: int, hi: int) -> "Program":
        """Split-aggregation shard: ranged `index` of the block at `block_path` over [lo, hi)."""
        h = ctypes.c_void_p()
        _check(lib().sb_program_restrict_index(self._h, block_path.encode(), index.encode(), lo, hi, ctypes.byref(h)))
        return Program(h.value)

    def check_split(self, block_path: str, index: str) -> None:
        """Raises ExecError('Unsupported') unless shards of `index` combine exactly
        (sb_program_check_split)."""
        _check(lib().sb_program_check_split(self._h, block_path.encode(), index.encode()))

    def text(self) -> str:
        return print_program(self)

    def count_valid_points(self, block_path: str = "0", ctx: "Context" = None) -> int:
        """tile.cpp:338-370 on the device (closed form per innermost row)."""
        v = ctypes.c_int64()
        _check(lib().sb_count_valid_points((ctx or default_context(0)).handle, self._h, block_path.encode(),
                                           ctypes.byref(v)))
        return v.value

    def tile_cost(self, block_path: str, tiles: str, line: int, mem_cap: int, interleaved: bool = False,
                  ctx: "Context" = None) -> TileReport:
        """tile_cost(block, parse_tile_shape(tiles), CacheModel{line}, mem_cap) (tile.cpp:380-455),
        line counts on the device (sb_tile_cost)."""
        r = TileReport()
        _check(lib().sb_tile_cost((ctx or default_context(0)).handle, self._h, block_path.encode(), tiles.encode(),
                                  int(interleaved), line, mem_cap, ctypes.byref(r)))
        return r

    def autotile(self, block_path: str, line: int, mem_cap: int, power_of_two: bool = False,
                 ctx: "Context" = None) -> AutotileResult:
        """autotile(block, CacheModel{line}, AutotileOptions{mem_cap, power_of_two}) (tile.cpp:475-535):
        every candidate evaluated on the device (sb_autotile)."""
        buf = ctypes.create_string_buffer(4096)
        n, found, r = ctypes.c_size_t(), ctypes.c_int32(), TileReport()
        cands, excl = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().sb_autotile((ctx or default_context(0)).handle, self._h, block_path.encode(), line, mem_cap,
                                 int(power_of_two), buf, len(buf), ctypes.byref(n), ctypes.byref(found),
                                 ctypes.byref(r), ctypes.byref(cands), ctypes.byref(excl)))
        return AutotileResult(buf.value.decode() if found.value else None, r, cands.value, excl.value)

    def describe_plan(self, fresh_outputs: bool = False, tensor_cores: bool = True, fp32_mode: int = 0) -> str:
        n = ctypes.c_size_t()
        flags = int(not tensor_cores) | (2 if fp32_mode == 1 else 0)
        _check(lib().sb_program_describe_plan(self._h, int(fresh_outputs), flags, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(lib().sb_program_describe_plan(self._h, int(fresh_outputs), flags, buf, len(buf), ctypes.byref(n)))
        return buf.value.decode()


def parse_program(text: str) -> Program:
    h = ctypes.c_void_p()
    _check(lib().sb_program_parse(text.encode(), ctypes.byref(h)))
    return Program(h.value)


def print_program(p: Program) -> str:
    n = ctypes.c_size_t()
    _check(lib().sb_program_print(p.handle, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(lib().sb_program_print(p.handle, buf, len(buf), ctypes.byref(n)))
    return buf.value.decode()


@dataclass
class Buffer:
    """interp.h:14-17: dtype plus int64 carriers (values always wrapped to dtype).

    f32 extension: an F32 buffer carries float32 values instead."""
    dtype: int
    data: np.ndarray


BufferStore = Dict[str, Buffer]


class IterOrder(enum.IntEnum):
    Lex = 0
    Reversed = 1
    Shuffled = 2


@dataclass
class ExecOptions:
    order: IterOrder = IterOrder.Lex
    seed: int = 0
    observer: Optional[object] = None
    disable_tensor_cores: bool = False
    fp32_mode: int = 0  # 0 exact (bitwise = CPU F32 policy), 1 3xTF32 tensor cores (stated bound)

    def _c(self) -> _Opts:
        return _Opts(int(self.order), 1 if self.observer is not None else 0, self.seed,
                     int(self.disable_tensor_cores), int(self.fp32_mode))


def prepare_outputs(program: Program, store: BufferStore) -> None:
    """interp.cpp:617-642: create missing out/inout buffers filled with the aggregation identity."""
    for name, decl in program.buffers.items():
        if decl.dir == Dir.In or name in store:
            continue
        ident = program.output_identity(name)
        if decl.dtype == SB_F32:  # f32 extension: identity returned as IEEE-754 bits
            data = np.full(decl.elements, ident & 0xFFFFFFFF, dtype=np.uint32).view(np.float32)
        else:
            data = np.full(decl.elements, ident, dtype=np.int64)
        store[name] = Buffer(decl.dtype, data)


class Context:
    """One device context (stream, error word, cached device buffers)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        _check(lib().sb_context_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.sb_context_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        _check(lib().sb_context_set_stream(self._h, ctypes.c_void_p(stream_ptr or 0)))

    def sync(self) -> None:
        _check(lib().sb_context_sync(self._h))

    def set_kernel_order(self, enable: bool) -> None:
        """sb_context_set_kernel_order: kernels queue behind other ordered contexts' kernels."""
        _check(lib().sb_context_set_kernel_order(self._h, int(enable)))

    def set_profile(self, enable: bool) -> None:
        _check(lib().sb_context_set_profile(self._h, int(enable)))

    def read_profile(self):
        """[(step, ms, kernel, path, points)] of the executes since the last read."""
        n = ctypes.c_size_t()
        _check(lib().sb_context_profile_read(self._h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _check(lib().sb_context_profile_read(self._h, buf, len(buf), ctypes.byref(n)))
        out = []
        for line in buf.value.decode().splitlines():
            f = line.split()
            out.append((int(f[0]), float(f[1]), f[2], f[3], int(f[4])))
        return out

    @property
    def launch_count(self) -> int:
        return int(lib().sb_context_launch_count(self._h))

    def execute(self, program: Program, store: BufferStore, opts: Optional[ExecOptions] = None) -> None:
        opts = opts or ExecOptions()
        arrs, hb = [], []
        for name, buf in store.items():
            if buf.dtype == SB_F32:  # f32 buffers travel as native float32 carriers
                a = np.ascontiguousarray(buf.data, dtype=np.float32)
                arrs.append(a)
                hb.append(HostBuffer(name.encode(), SB_CARRIER_NATIVE, 0, a.ctypes.data, a.size))
                continue
            a = np.ascontiguousarray(buf.data, dtype=np.int64)
            arrs.append(a)
            hb.append(HostBuffer(name.encode(), SB_CARRIER_I64, 0, a.ctypes.data, a.size))
        arr = (HostBuffer * len(hb))(*hb)
        _check(lib().sb_execute(self._h, program.handle, arr, len(hb), ctypes.byref(opts._c())))
        for (name, buf), a in zip(store.items(), arrs):
            if a is not buf.data:
                buf.data[...] = a

    def execute_native(self, program: Program, arrays: Dict[str, np.ndarray], prepare=(),
                       opts: Optional[ExecOptions] = None) -> None:
        """Native-width host arrays (int8/int16/int32); names in `prepare` are created on device."""
        opts = opts or ExecOptions()
        hb = []
        for name, a in arrays.items():
            assert a.flags["C_CONTIGUOUS"]
            hb.append(HostBuffer(name.encode(), SB_CARRIER_NATIVE, SB_BUF_PREPARE if name in prepare else 0,
                                 a.ctypes.data, a.size))
        arr = (HostBuffer * len(hb))(*hb)
        _check(lib().sb_execute(self._h, program.handle, arr, len(hb), ctypes.byref(opts._c())))

    def execute_native_async(self, program: Program, arrays: Dict[str, np.ndarray], prepare=(),
                             opts: Optional[ExecOptions] = None) -> None:
        """sb_execute_async: arrays must live in pinned host memory; results after sync()."""
        opts = opts or ExecOptions()
        hb = []
        for name, a in arrays.items():
            assert a.flags["C_CONTIGUOUS"]
            hb.append(HostBuffer(name.encode(), SB_CARRIER_NATIVE, SB_BUF_PREPARE if name in prepare else 0,
                                 a.ctypes.data, a.size))
        arr = (HostBuffer * len(hb))(*hb)
        _check(lib().sb_execute_async(self._h, program.handle, arr, len(hb), ctypes.byref(opts._c())))

    def execute_device(self, program: Program, buffers: Dict[str, tuple], opts: Optional[ExecOptions] = None) -> None:
        """buffers: name -> (device_ptr, count, flags).  Asynchronous on the context stream."""
        self.bind_device(program, buffers, opts)()

    def bind_device(self, program: Program, buffers: Dict[str, tuple], opts: Optional[ExecOptions] = None):
        """Pre-marshals an HBM-resident execute; the returned callable enqueues it."""
        opts = opts or ExecOptions()
        names = [n.encode() for n in buffers]
        db = [DeviceBuffer(nm, int(f), 0, int(p), int(c)) for nm, (p, c, f) in zip(names, buffers.values())]
        arr = (DeviceBuffer * len(db))(*db)
        copts = opts._c()
        fn, h, ph, n, po = lib().sb_execute_device, self._h, program.handle, len(db), ctypes.byref(copts)

        def run():
            rc = fn(h, ph, arr, n, po)
            if rc:
                _check(rc)
        run._keep = (names, arr, copts, program)
        return run


class Graph:
    """A captured sequence of HBM-resident executes (sb_graph_*), replayed with one launch."""

    def __init__(self, ctx: "Context", fn):
        self.ctx = ctx
        _check(lib().sb_graph_begin(ctx.handle))
        try:
            fn()
        finally:
            h = ctypes.c_void_p()
            rc = lib().sb_graph_end(ctx.handle, ctypes.byref(h))
        _check(rc)
        self._h = h

    def launch(self) -> None:
        _check(lib().sb_graph_launch(self.ctx.handle, self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.sb_graph_free(self._h)
            self._h = None


_default_ctx: Dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def execute(program: Program, store: BufferStore, opts: Optional[ExecOptions] = None) -> None:
    """interp.h:68: run `program` over `store` on the B200 (store updated in place)."""
    default_context(0).execute(program, store, opts)


__all__ = [
    "parse_program", "print_program", "prepare_outputs", "execute", "Program", "Buffer", "BufferStore",
    "ExecOptions", "IterOrder", "ExecError", "DType", "Dir", "Context", "default_context", "lib",
]
