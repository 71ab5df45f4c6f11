// Generic block kernel (K4 in SURVEY §2.1): executes one flat launch of the
// plan for ANY leaf body, bit-exact with the reference interpreter.
//
// One thread owns one point of the thread-mapped dims (pdims); it walks the
// remaining dims (rdims) serially in declaration order, which is the
// lexicographic order restricted to that thread (interp.cpp:365-384), so
// last-writer-wins `assign`, read-modify-write bodies and non-commutative
// chains reproduce serial results exactly.  Per point: constraints are the
// skip predicate (interp.cpp:426-428), temps are zeroed (interp.cpp:454),
// leaf allocs are zeroed cells (interp.cpp:442-447), loads/stores hit the
// single element at the composed view base (interp.cpp:497-504) and stores
// aggregate with wrap at the refinement dtype (ir.cpp:79-97).  Owned output
// cells stay in registers for the whole R loop and are written once.
#include <cuda_runtime.h>

#include <cstdint>

#include "../desc.hpp"

namespace sb {
namespace {

__device__ __forceinline__ std::int64_t wrap_dt(int dt, std::int64_t v) {
  switch (dt) {
    case 0: return static_cast<std::int8_t>(v);
    case 1: return static_cast<std::int16_t>(v);
    case 2: return static_cast<std::int32_t>(v);
    default: return v;  // -1: int64 spill carrier
  }
}

__device__ __forceinline__ std::int64_t agg_apply(int agg, std::int64_t cur, std::int64_t in, int dt) {
  std::int64_t v = wrap_dt(dt, in);
  switch (agg) {
    case 0: return v;
    case 1: return wrap_dt(dt, static_cast<std::int64_t>(static_cast<unsigned long long>(cur) +
                                                        static_cast<unsigned long long>(v)));
    case 2: return cur > v ? cur : v;
    case 3: return cur < v ? cur : v;
    default:
      return wrap_dt(dt, static_cast<std::int64_t>(static_cast<unsigned long long>(cur) *
                                                  static_cast<unsigned long long>(v)));
  }
}

__device__ __forceinline__ std::int64_t ld(const void* p, int kind, std::int64_t i) {
  switch (kind) {
    case kI8: return static_cast<const std::int8_t*>(p)[i];
    case kI16: return static_cast<const std::int16_t*>(p)[i];
    case kI32: return static_cast<const std::int32_t*>(p)[i];
    default: return static_cast<const long long*>(p)[i];
  }
}

__device__ __forceinline__ void st(void* p, int kind, std::int64_t i, std::int64_t v) {
  switch (kind) {
    case kI8: static_cast<std::int8_t*>(p)[i] = static_cast<std::int8_t>(v); break;
    case kI16: static_cast<std::int16_t*>(p)[i] = static_cast<std::int16_t>(v); break;
    case kI32: static_cast<std::int32_t*>(p)[i] = static_cast<std::int32_t>(v); break;
    default: static_cast<long long*>(p)[i] = v; break;
  }
}

// Commutative aggregation through device atomics.  32-bit add/max/min use the
// native ops (two's-complement add wraps exactly like wrap_value at i32);
// sub-word elements and mul use a CAS loop on the enclosing aligned word
// (device buffers are padded to 16 bytes, so that word is always in bounds).
__device__ void atomic_agg(void* p, int kind, std::int64_t i, int agg, std::int64_t in, int dt) {
  std::int64_t v = wrap_dt(dt, in);
  if (kind == kI32) {
    int* a = static_cast<int*>(p) + i;
    if (agg == 1) { atomicAdd(a, static_cast<int>(v)); return; }
    if (agg == 2) { atomicMax(a, static_cast<int>(v)); return; }
    if (agg == 3) { atomicMin(a, static_cast<int>(v)); return; }
    int old = *a, assumed;
    do {
      assumed = old;
      int nv = static_cast<int>(agg_apply(agg, assumed, v, dt));
      old = atomicCAS(a, assumed, nv);
    } while (old != assumed);
    return;
  }
  int bytes = kind == kI8 ? 1 : 2;
  std::uintptr_t addr = reinterpret_cast<std::uintptr_t>(p) + static_cast<std::uintptr_t>(i) * bytes;
  unsigned int* word = reinterpret_cast<unsigned int*>(addr & ~std::uintptr_t{3});
  int shift = static_cast<int>(addr & 3) * 8;
  unsigned int mask = (bytes == 1 ? 0xffu : 0xffffu) << shift;
  unsigned int old = *word, assumed;
  do {
    assumed = old;
    unsigned int raw = (assumed & mask) >> shift;
    std::int64_t cur = bytes == 1 ? static_cast<std::int8_t>(raw) : static_cast<std::int16_t>(raw);
    std::int64_t nv = agg_apply(agg, cur, v, dt);
    unsigned int next = (assumed & ~mask) | ((static_cast<unsigned int>(nv) << shift) & mask);
    old = atomicCAS(word, assumed, next);
  } while (old != assumed);
}

__device__ __forceinline__ std::int64_t eval_aff(const DAff& a, const std::int64_t* coord, int nd) {
  std::int64_t v = a.c;
  for (int d = 0; d < nd; d++) v += a.k[d] * coord[d];
  return v;
}

__device__ void report(DevError* err, int code, int launch, std::int64_t addr, int buf) {
  if (atomicCAS(&err->code, 0, code) == 0) {
    err->launch = launch;
    err->addr = addr;
    err->buf = buf;
  }
}

__global__ void __launch_bounds__(128) generic_block_kernel(const GenericDesc* __restrict__ D,
                                                            BufTable T, DevError* err, int launch_id) {
  const GenericDesc& d = *D;
  const int nd = d.ndims;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t lin = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       lin < d.pcount; lin += stride) {
    std::int64_t coord[kMaxDims];
    for (int i = 0; i < nd; i++) coord[i] = 0;
    std::int64_t rest = lin;
    for (int i = 0; i < d.npdims; i++) {
      int dim = d.pdims[i];
      coord[dim] = rest % d.range[dim];
      rest /= d.range[dim];
    }
    std::int64_t cell[kMaxCells];
    std::int64_t cell_addr[kMaxCells];
    int cell_slot[kMaxCells];
    unsigned loaded = 0, dirty = 0;
    std::int64_t t[kMaxTemps];
    std::int64_t priv[kMaxCells];

    auto cell_get = [&](const DAccess& a) -> std::int64_t& {
      int c = a.cell;
      if (!(loaded >> c & 1u)) {
        std::int64_t addr = eval_aff(a.addr, coord, nd);
        cell_addr[c] = addr;
        cell_slot[c] = a.buf;
        if (addr < 0 || addr >= T.elems[a.buf]) {
          report(err, 1, launch_id, addr, a.buf);
          cell[c] = 0;
          cell_slot[c] = -1;
        } else {
          cell[c] = ld(T.ptr[a.buf], T.kind[a.buf], addr);
        }
        loaded |= 1u << c;
      }
      return cell[c];
    };
    auto opv = [&](int x) -> std::int64_t { return x >= 0 ? t[x] : d.consts[-1 - x]; };

    for (;;) {
      bool ok = true;
      for (int c = 0; c < d.ncons && ok; c++) ok = eval_aff(d.cons[c], coord, nd) >= 0;
      if (ok) {
        for (int i = 0; i < d.ntemps; i++) t[i] = 0;
        for (int i = 0; i < d.npriv; i++) priv[i] = 0;
        for (int pc = 0; pc < d.ncode; pc++) {
          const DInstr ins = d.code[pc];
          switch (ins.op) {
            case kOpLoad: {
              const DAccess& a = d.acc[ins.acc];
              if (a.mode == kAccOwned) {
                t[ins.dst] = cell_get(a);
              } else {
                std::int64_t addr = eval_aff(a.addr, coord, nd);
                if (addr < 0 || addr >= T.elems[a.buf]) {
                  report(err, 1, launch_id, addr, a.buf);
                  t[ins.dst] = 0;
                } else {
                  t[ins.dst] = ld(T.ptr[a.buf], T.kind[a.buf], addr);
                }
              }
              break;
            }
            case kOpStore: {
              const DAccess& a = d.acc[ins.acc];
              std::int64_t v = t[ins.a];
              if (a.mode == kAccOwned) {
                std::int64_t& c = cell_get(a);
                c = ins.dtype < 0 ? v : agg_apply(ins.agg, c, v, ins.dtype);
                dirty |= 1u << a.cell;
                break;
              }
              std::int64_t addr = eval_aff(a.addr, coord, nd);
              if (addr < 0 || addr >= T.elems[a.buf]) {
                report(err, 1, launch_id, addr, a.buf);
                break;
              }
              if (a.mode == kAccAtomic) {
                atomic_agg(T.ptr[a.buf], T.kind[a.buf], addr, ins.agg, v, ins.dtype);
              } else {
                std::int64_t cur = ld(T.ptr[a.buf], T.kind[a.buf], addr);
                st(T.ptr[a.buf], T.kind[a.buf], addr,
                   ins.dtype < 0 ? v : agg_apply(ins.agg, cur, v, ins.dtype));
              }
              break;
            }
            case kOpLoadPriv: t[ins.dst] = priv[ins.acc]; break;
            case kOpStorePriv:
              priv[ins.acc] = agg_apply(d.priv_agg[ins.acc], priv[ins.acc], t[ins.a], d.priv_dtype[ins.acc]);
              break;
            case kOpAdd:
              t[ins.dst] = static_cast<std::int64_t>(static_cast<unsigned long long>(opv(ins.a)) +
                                                     static_cast<unsigned long long>(opv(ins.b)));
              break;
            case kOpSub:
              t[ins.dst] = static_cast<std::int64_t>(static_cast<unsigned long long>(opv(ins.a)) -
                                                     static_cast<unsigned long long>(opv(ins.b)));
              break;
            case kOpMul:
              t[ins.dst] = static_cast<std::int64_t>(static_cast<unsigned long long>(opv(ins.a)) *
                                                     static_cast<unsigned long long>(opv(ins.b)));
              break;
            case kOpNeg:
              t[ins.dst] = static_cast<std::int64_t>(0ull - static_cast<unsigned long long>(opv(ins.a)));
              break;
            case kOpMax: { std::int64_t x = opv(ins.a), y = opv(ins.b); t[ins.dst] = x > y ? x : y; break; }
            case kOpMin: { std::int64_t x = opv(ins.a), y = opv(ins.b); t[ins.dst] = x < y ? x : y; break; }
            case kOpCmpEq: t[ins.dst] = opv(ins.a) == opv(ins.b); break;
            case kOpCmpNe: t[ins.dst] = opv(ins.a) != opv(ins.b); break;
            case kOpCmpLt: t[ins.dst] = opv(ins.a) < opv(ins.b); break;
            case kOpCmpLe: t[ins.dst] = opv(ins.a) <= opv(ins.b); break;
            case kOpCmpGt: t[ins.dst] = opv(ins.a) > opv(ins.b); break;
            case kOpCmpGe: t[ins.dst] = opv(ins.a) >= opv(ins.b); break;
            case kOpSelect: t[ins.dst] = opv(ins.a) != 0 ? opv(ins.b) : opv(ins.c); break;
            case kOpConst: t[ins.dst] = opv(ins.a); break;
            case kOpGather:
            case kOpScatter: {
              // gather: dst[v] = src[idx[v], v1..]; scatter: dst[idx[v], v1..] agg= src[v]
              // (interp.cpp:539-600).  Serial mode only.
              const DSpecial& s = d.special[ins.acc];
              const DAccess& ad = d.acc[s.dst];
              const DAccess& as = d.acc[s.src];
              const DAccess& ai = d.acc[s.idx];
              std::int64_t bd = eval_aff(ad.addr, coord, nd), bs = eval_aff(as.addr, coord, nd),
                           bi = eval_aff(ai.addr, coord, nd);
              std::int64_t total = 1;
              for (int r = 0; r < s.rank; r++) total *= s.walk[r];
              bool gather = ins.op == kOpGather;
              for (std::int64_t n = 0; n < total; n++) {
                std::int64_t co[kMaxRank];
                std::int64_t rr = n;
                for (int r = s.rank - 1; r >= 0; r--) {
                  co[r] = rr % s.walk[r];
                  rr /= s.walk[r];
                }
                std::int64_t ia = bi;
                for (int r = 0; r < s.rank; r++) ia += co[r] * s.sidx[r];
                if (ia < 0 || ia >= T.elems[ai.buf]) { report(err, 1, launch_id, ia, ai.buf); return; }
                std::int64_t pick = ld(T.ptr[ai.buf], T.kind[ai.buf], ia);
                if (pick < 0 || pick >= s.bound) { report(err, 2, launch_id, pick, ai.buf); return; }
                std::int64_t sa = bs, da = bd;
                if (gather) {
                  sa += pick * s.ssrc[0];
                  for (int r = 1; r < s.rank; r++) sa += co[r] * s.ssrc[r];
                  for (int r = 0; r < s.rank; r++) da += co[r] * s.sdst[r];
                } else {
                  da += pick * s.sdst[0];
                  for (int r = 0; r < s.rank; r++) sa += co[r] * s.ssrc[r];
                  for (int r = 1; r < s.rank; r++) da += co[r] * s.sdst[r];
                }
                if (sa < 0 || sa >= T.elems[as.buf]) { report(err, 1, launch_id, sa, as.buf); return; }
                if (da < 0 || da >= T.elems[ad.buf]) { report(err, 1, launch_id, da, ad.buf); return; }
                std::int64_t v = ld(T.ptr[as.buf], T.kind[as.buf], sa);
                std::int64_t cur = ld(T.ptr[ad.buf], T.kind[ad.buf], da);
                st(T.ptr[ad.buf], T.kind[ad.buf], da, agg_apply(s.dst_agg, cur, v, s.dst_dtype));
              }
              break;
            }
          }
        }
      }
      // odometer over the serial dims, last fastest
      bool more = false;
      for (int i = d.nrdims - 1; i >= 0; i--) {
        int dim = d.rdims[i];
        if (++coord[dim] < d.range[dim]) {
          more = true;
          break;
        }
        coord[dim] = 0;
      }
      if (!more) break;
    }
    for (int c = 0; c < d.ncells; c++)
      if ((dirty >> c & 1u) && cell_slot[c] >= 0) st(T.ptr[cell_slot[c]], T.kind[cell_slot[c]], cell_addr[c], cell[c]);
  }
}

// Identity fill (prepare_outputs, interp.cpp:617-642; alloc zero-fill, interp.cpp:442-447).
template <typename E>
__global__ void fill_kernel(E* p, std::int64_t n, E v) {
  std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
}

int grid_for(std::int64_t work, int block) {
  std::int64_t g = (work + block - 1) / block;
  std::int64_t cap = 148 * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

cudaError_t launch_generic(const GenericDesc* d_desc, std::int64_t pcount, const BufTable& t,
                           DevError* err, int launch_id, cudaStream_t s) {
  int block = pcount >= 128 ? 128 : 32;
  generic_block_kernel<<<grid_for(pcount, block), block, 0, s>>>(d_desc, t, err, launch_id);
  return cudaGetLastError();
}

cudaError_t launch_fill(void* p, int kind, std::int64_t n, std::int64_t v, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (v == 0) return cudaMemsetAsync(p, 0, static_cast<std::size_t>(n) * (kind == kI8 ? 1 : kind == kI16 ? 2 : kind == kI64 ? 8 : 4), s);
  int block = 256;
  switch (kind) {
    case kI8: fill_kernel<<<grid_for(n, block), block, 0, s>>>(static_cast<std::int8_t*>(p), n, static_cast<std::int8_t>(v)); break;
    case kI16: fill_kernel<<<grid_for(n, block), block, 0, s>>>(static_cast<std::int16_t*>(p), n, static_cast<std::int16_t>(v)); break;
    case kI32: case kF32: fill_kernel<<<grid_for(n, block), block, 0, s>>>(static_cast<std::int32_t*>(p), n, static_cast<std::int32_t>(v)); break;
    default: fill_kernel<<<grid_for(n, block), block, 0, s>>>(static_cast<long long*>(p), n, static_cast<long long>(v)); break;
  }
  return cudaGetLastError();
}

}  // namespace sb
