"""oracle — TEST INFRASTRUCTURE ONLY (the checker; never the product).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg import this package.  Two checkers:

* ``Ref``  — the UNMODIFIED reference interpreter (Stripe Kit) compiled from
  /root/reference/proj by oracle/Makefile into oracle/_ref/libstripe_ref.so
  (built here; the .so travels to the GPU box).  Bit-exact ground truth.
* ``Port`` — oracle/port: a CPU restatement of interp.cpp's semantics,
  templated on a scalar policy (int64-wrap: pinned bit-exact against Ref on the
  whole corpus by tests/test_oracle.py; f32: the fp32 extension).

Plus ``random_inputs``: a numpy restatement of tests/support.h:29-70 (splitmix64
Rng + wrap_value), pinned against Ref.random_inputs.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libstripe_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libstripe_port.so")

_vp, _i64, _i32, _cp, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t

BITS = {"i8": 8, "i16": 16, "i32": 32}


class OracleError(RuntimeError):
    def __init__(self, text: str):
        super().__init__(text)
        self.code = text.split(":", 1)[0]


# --------------------------------------------------------------------------------------
# splitmix64 (tests/support.h:29-40) and random_inputs (support.h:55-70)
MASK = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int):
        self.state = seed & MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def bulk(self, n: int) -> np.ndarray:
        """n successive next() values as uint64 (vectorised)."""
        with np.errstate(over="ignore"):
            k = np.arange(1, n + 1, dtype=np.uint64)
            z = np.uint64(self.state) + k * np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * 0x9E3779B97F4A7C15) & MASK
        return z


def wrap(bits: int, values: np.ndarray) -> np.ndarray:
    """ir.cpp:39-48 wrap_value on uint64/int64 arrays -> int64."""
    v = values.astype(np.uint64, copy=False)
    if bits == 8:
        return v.astype(np.uint8).view(np.int8).astype(np.int64)
    if bits == 16:
        return v.astype(np.uint16).view(np.int16).astype(np.int64)
    return v.astype(np.uint32).view(np.int32).astype(np.int64)


def random_inputs(buffers, seed: int) -> Dict[str, np.ndarray]:
    """buffers: ordered iterable of (name, bits, elements, dir) root refinements.
    Returns int64 carriers for every non-`out` buffer, exactly as support.h:55-70."""
    rng = Rng(seed)
    out = {}
    for name, bits, elements, d in buffers:
        if d == 1:  # Dir::Out
            continue
        out[name] = wrap(bits, rng.bulk(elements))
    return out


def native(bits: int, carrier: np.ndarray) -> np.ndarray:
    return carrier.astype({8: np.int8, 16: np.int16, 32: np.int32}[bits])


# --------------------------------------------------------------------------------------
class Ref:
    """ctypes view of oracle/_ref/libstripe_ref.so (the reference itself)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise RuntimeError(f"{REF_SO} missing; build with `make -C oracle ref`")
            L = ctypes.CDLL(REF_SO)
            L.sr_parse.argtypes = [_cp, _cp, _sz]
            L.sr_parse.restype = _vp
            L.sr_free_program.argtypes = [_vp]
            L.sr_print.argtypes = [_vp, _cp, _sz]
            L.sr_validate.argtypes = [_vp, _cp, _sz]
            L.sr_buffer_count.argtypes = [_vp]
            L.sr_buffer_info.argtypes = [_vp, _i32, _cp, _sz, ctypes.POINTER(_i32), ctypes.POINTER(_i64),
                                         ctypes.POINTER(_i32)]
            L.sr_store_new.restype = _vp
            L.sr_store_free.argtypes = [_vp]
            L.sr_store_clone.argtypes = [_vp]
            L.sr_store_clone.restype = _vp
            L.sr_store_set.argtypes = [_vp, _cp, _i32, _vp, _i64]
            L.sr_store_get.argtypes = [_vp, _cp, _vp, _i64]
            L.sr_store_get.restype = _i64
            L.sr_random_inputs.argtypes = [_vp, ctypes.c_uint64, _vp]
            L.sr_prepare_outputs.argtypes = [_vp, _vp, _cp, _sz]
            L.sr_execute.argtypes = [_vp, _vp, _i32, ctypes.c_uint64, _cp, _sz]
            L.sr_execute_many.argtypes = [ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i32, _i32]
            L.sr_conflicts.argtypes = [_vp, _vp, _cp, _sz]
            L.sr_conflicts.restype = _i64
            L.sr_gen.argtypes = [_cp, _i64, _i64, _i64, _i64, _i32, _cp, _sz]
            L.sr_gen_random.argtypes = [_i32, ctypes.POINTER(ctypes.c_uint64), _cp, _sz]
            L.sr_gen_oracle.argtypes = [_cp, _i64, _i64, _i64, _i64, _i32, _vp]
            L.sr_tile_rewrite.argtypes = [_vp, _cp, _cp, _cp, _sz, _cp, _sz]
            L.sr_pipeline.argtypes = [_vp, _cp, _cp, _sz, _cp, _sz]
            L.sr_useful_ops.argtypes = [_vp, _cp, ctypes.POINTER(_i64), _cp, _sz]
            L.sr_tile_cost.argtypes = [_vp, _cp, _cp, _i32, _i64, _i64, _i64, _vp, _cp, _sz]
            L.sr_autotile.argtypes = [_vp, _cp, _i64, _i64, _i32, _cp, _sz, _vp, _cp, _sz]
            cls._lib = L
        return cls._lib

    # ---- programs ----
    class Program:
        def __init__(self, handle):
            self.h = handle

        def __del__(self):
            if self.h and Ref._lib is not None:
                Ref._lib.sr_free_program(self.h)
                self.h = None

        def text(self) -> str:
            return Ref._text(lambda b, n: Ref.lib().sr_print(self.h, b, n))

        def buffers(self):
            L = Ref.lib()
            out = []
            for i in range(L.sr_buffer_count(self.h)):
                name = ctypes.create_string_buffer(256)
                bits, el, d = _i32(), _i64(), _i32()
                L.sr_buffer_info(self.h, i, name, 256, ctypes.byref(bits), ctypes.byref(el), ctypes.byref(d))
                out.append((name.value.decode(), bits.value, el.value, d.value))
            return out

        def validate(self):
            buf = ctypes.create_string_buffer(1 << 16)
            n = Ref.lib().sr_validate(self.h, buf, len(buf))
            return n, buf.value.decode()

    @staticmethod
    def _text(fn) -> str:
        n = fn(None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        fn(buf, n + 1)
        return buf.value.decode()

    @classmethod
    def parse(cls, text: str) -> "Ref.Program":
        err = ctypes.create_string_buffer(4096)
        h = cls.lib().sr_parse(text.encode(), err, len(err))
        if not h:
            raise OracleError(err.value.decode())
        return Ref.Program(h)

    @classmethod
    def gen(cls, kind: str, a: int, b: int, c: int, d: int = 0, bits: int = 32) -> str:
        return cls._text(lambda buf, n: cls.lib().sr_gen(kind.encode(), a, b, c, d, bits, buf, n))

    @classmethod
    def gen_random(cls, state: int, text_variant: bool = False):
        st = ctypes.c_uint64(state)
        n = cls.lib().sr_gen_random(int(text_variant), ctypes.byref(ctypes.c_uint64(state)), None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        cls.lib().sr_gen_random(int(text_variant), ctypes.byref(st), buf, n + 1)
        return buf.value.decode(), st.value

    @classmethod
    def tile_rewrite(cls, text: str, path: str, tiles: str) -> str:
        p = cls.parse(text)
        err = ctypes.create_string_buffer(4096)
        n = cls.lib().sr_tile_rewrite(p.h, path.encode(), tiles.encode(), None, 0, err, len(err))
        if n < 0:
            raise OracleError(err.value.decode())
        buf = ctypes.create_string_buffer(n + 1)
        cls.lib().sr_tile_rewrite(p.h, path.encode(), tiles.encode(), buf, n + 1, err, len(err))
        return buf.value.decode()

    @classmethod
    def useful_ops(cls, text: str, path: str) -> int:
        """count_valid_points of the block at `path` via tile_cost (tile.cpp:404-411)."""
        p = cls.parse(text)
        err = ctypes.create_string_buffer(4096)
        v = _i64()
        if cls.lib().sr_useful_ops(p.h, path.encode(), ctypes.byref(v), err, len(err)):
            raise OracleError(err.value.decode())
        return v.value

    @classmethod
    def tile_cost(cls, text: str, path: str, tiles: str, line: int, mem_cap: int, interleaved: bool = False,
                  hint: int = -1):
        """tile_cost (tile.cpp:380-455) -> (lines_total, useful_ops, tile_elements, excluded)."""
        p = cls.parse(text)
        err = ctypes.create_string_buffer(4096)
        out = np.zeros(4, dtype=np.int64)
        if cls.lib().sr_tile_cost(p.h, path.encode(), tiles.encode(), int(interleaved), line, mem_cap, hint,
                                  out.ctypes.data, err, len(err)):
            raise OracleError(err.value.decode())
        return int(out[0]), int(out[1]), int(out[2]), bool(out[3])

    @classmethod
    def autotile(cls, text: str, path: str, line: int, mem_cap: int, power_of_two: bool = False):
        """autotile (tile.cpp:475-535) -> (chosen text or None, (lines, ops, tile_elements), candidates, excluded)."""
        p = cls.parse(text)
        err = ctypes.create_string_buffer(4096)
        buf = ctypes.create_string_buffer(4096)
        out = np.zeros(6, dtype=np.int64)
        if cls.lib().sr_autotile(p.h, path.encode(), line, mem_cap, int(power_of_two), buf, len(buf),
                                 out.ctypes.data, err, len(err)):
            raise OracleError(err.value.decode())
        return (buf.value.decode() if out[5] else None, (int(out[0]), int(out[1]), int(out[2])), int(out[3]),
                int(out[4]))

    @classmethod
    def pipeline(cls, text: str, hwcfg: str) -> str:
        p = cls.parse(text)
        err = ctypes.create_string_buffer(8192)
        n = cls.lib().sr_pipeline(p.h, hwcfg.encode(), None, 0, err, len(err))
        if n < 0:
            raise OracleError(err.value.decode())
        buf = ctypes.create_string_buffer(n + 1)
        cls.lib().sr_pipeline(p.h, hwcfg.encode(), buf, n + 1, err, len(err))
        return buf.value.decode()

    # ---- stores: dict name -> (bits, int64 array) ----
    @classmethod
    def _store(cls, store: Dict[str, tuple]):
        L = cls.lib()
        s = L.sr_store_new()
        for name, (bits, arr) in store.items():
            a = np.ascontiguousarray(arr, dtype=np.int64)
            L.sr_store_set(s, name.encode(), bits, a.ctypes.data, a.size)
        return s

    @classmethod
    def _read(cls, s, names_bits) -> Dict[str, tuple]:
        L = cls.lib()
        out = {}
        for name, bits in names_bits:
            n = L.sr_store_get(s, name.encode(), None, 0)
            if n < 0:
                continue
            a = np.empty(n, dtype=np.int64)
            L.sr_store_get(s, name.encode(), a.ctypes.data, n)
            out[name] = (bits, a)
        return out

    @classmethod
    def random_inputs(cls, prog: "Ref.Program", seed: int) -> Dict[str, tuple]:
        """support.h:55-70 incl. prepare_outputs."""
        L = cls.lib()
        s = L.sr_store_new()
        L.sr_random_inputs(prog.h, seed, s)
        out = cls._read(s, [(b[0], b[1]) for b in prog.buffers()])
        L.sr_store_free(s)
        return out

    @classmethod
    def prepare_outputs(cls, prog: "Ref.Program", store: Dict[str, tuple]) -> Dict[str, tuple]:
        L = cls.lib()
        s = cls._store(store)
        err = ctypes.create_string_buffer(4096)
        if L.sr_prepare_outputs(prog.h, s, err, len(err)):
            L.sr_store_free(s)
            raise OracleError(err.value.decode())
        out = cls._read(s, [(b[0], b[1]) for b in prog.buffers()])
        L.sr_store_free(s)
        return out

    @classmethod
    def execute(cls, prog: "Ref.Program", store: Dict[str, tuple], order: int = 0, seed: int = 0):
        """Returns the updated store (dict name -> (bits, int64 array)); raises OracleError."""
        L = cls.lib()
        s = cls._store(store)
        err = ctypes.create_string_buffer(4096)
        rc = L.sr_execute(prog.h, s, order, seed, err, len(err))
        out = cls._read(s, [(n, b[0]) for n, b in store.items()])
        L.sr_store_free(s)
        if rc:
            raise OracleError(err.value.decode())
        return out

    @classmethod
    def conflicts(cls, prog: "Ref.Program", store: Dict[str, tuple]):
        L = cls.lib()
        s = cls._store(store)
        buf = ctypes.create_string_buffer(1 << 16)
        n = L.sr_conflicts(prog.h, s, buf, len(buf))
        L.sr_store_free(s)
        return n, buf.value.decode()


class Port:
    """ctypes view of oracle/_port/libstripe_port.so (CPU restatement)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(PORT_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(PORT_SO):
                raise RuntimeError(f"{PORT_SO} missing; build with `make -C oracle port`")
            L = ctypes.CDLL(PORT_SO)
            L.sp_last_error.restype = _cp
            L.sp_parse.argtypes = [_cp]
            L.sp_parse.restype = _vp
            L.sp_free_program.argtypes = [_vp]
            L.sp_print.argtypes = [_vp, _cp, _sz]
            L.sp_store_new.restype = _vp
            L.sp_store_free.argtypes = [_vp]
            L.sp_store_set.argtypes = [_vp, _cp, _vp, _i64]
            L.sp_store_set_f32.argtypes = [_vp, _cp, _vp, _i64]
            L.sp_store_get.argtypes = [_vp, _cp, _vp, _i64]
            L.sp_store_get.restype = _i64
            L.sp_store_get_f32.argtypes = [_vp, _cp, _vp, _i64]
            L.sp_store_get_f32.restype = _i64
            L.sp_execute.argtypes = [_vp, _vp, _i32, _i32]
            L.sp_output_identity.argtypes = [_vp, _cp]
            L.sp_output_identity.restype = _i64
            cls._lib = L
        return cls._lib

    @classmethod
    def parse(cls, text: str):
        h = cls.lib().sp_parse(text.encode())
        if not h:
            raise OracleError(cls.lib().sp_last_error().decode())
        return h

    @classmethod
    def print(cls, text: str) -> str:
        h = cls.parse(text)
        L = cls.lib()
        n = L.sp_print(h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        L.sp_print(h, buf, n + 1)
        L.sp_free_program(h)
        return buf.value.decode()

    @classmethod
    def execute(cls, text: str, store: Dict[str, np.ndarray], order: int = 0, f32: bool = False):
        """store: name -> int64 carriers (or float32 in f32 mode).  Returns updated copy."""
        L = cls.lib()
        h = cls.parse(text)
        s = L.sp_store_new()
        for name, arr in store.items():
            if f32:
                a = np.ascontiguousarray(arr, dtype=np.float32)
                L.sp_store_set_f32(s, name.encode(), a.ctypes.data, a.size)
            else:
                a = np.ascontiguousarray(arr, dtype=np.int64)
                L.sp_store_set(s, name.encode(), a.ctypes.data, a.size)
        rc = L.sp_execute(h, s, 1 if f32 else 0, order)
        out = {}
        for name, arr in store.items():
            if f32:
                o = np.empty(arr.size, dtype=np.float32)
                L.sp_store_get_f32(s, name.encode(), o.ctypes.data, o.size)
            else:
                o = np.empty(arr.size, dtype=np.int64)
                L.sp_store_get(s, name.encode(), o.ctypes.data, o.size)
            out[name] = o
        err = L.sp_last_error().decode()
        L.sp_store_free(s)
        L.sp_free_program(h)
        if rc:
            raise OracleError(err)
        return out


def reference_execute(text: str, store: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
    """The parity checker the GPU tests use: the UNMODIFIED reference (its own parser and
    interpreter, oracle/_ref) when it was built, so the checker shares no code with the
    product; the port restatement (which shares the product's parser) only as a fallback.
    store: name -> int64 carriers; returns name -> int64 arrays after execute()."""
    if Ref.available():
        p = Ref.parse(text)
        bits = {b[0]: b[1] for b in p.buffers()}
        out = Ref.execute(p, {n: (bits.get(n, 32), np.ascontiguousarray(a, dtype=np.int64)) for n, a in store.items()})
        return {n: v[1] for n, v in out.items()}
    return Port.execute(text, store)
