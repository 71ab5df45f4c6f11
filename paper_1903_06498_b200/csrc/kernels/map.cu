// Vectorised block kernel for memory-bound Stripe blocks (K1 map / K2 reduce in
// SURVEY §2.1): element-wise maps, pooling windows, global reductions.
//
// Same semantics and bytecode as the generic kernel (kernels/generic.cu) in owner
// mode — a thread owns output points and walks the serial dims in declaration order
// (interp.cpp:365-384), so assign / add / max / min / mul aggregation is exact — but a
// thread owns kVec consecutive points of the fastest thread dim: every access is a
// broadcast, an aligned contiguous vector (one 4/8/16-byte load per access and point)
// or a per-lane gather, and the owned output vectors stay in registers for the whole
// reduction walk and are written once.
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
    default: return v;
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

__device__ __forceinline__ std::int64_t ld1(const void* p, int kind, std::int64_t i) {
  switch (kind) {
    case kI8: return static_cast<const std::int8_t*>(p)[i];
    case kI16: return static_cast<const std::int16_t*>(p)[i];
    case kI32: return static_cast<const std::int32_t*>(p)[i];
    default: return static_cast<const long long*>(p)[i];
  }
}

__device__ __forceinline__ void st1(void* p, int kind, std::int64_t i, std::int64_t v) {
  switch (kind) {
    case kI8: static_cast<std::int8_t*>(p)[i] = static_cast<std::int8_t>(v); break;
    case kI16: static_cast<std::int16_t*>(p)[i] = static_cast<std::int16_t>(v); break;
    case kI32: static_cast<std::int32_t*>(p)[i] = static_cast<std::int32_t>(v); break;
    default: static_cast<long long*>(p)[i] = v; break;
  }
}

// kVec (=4) consecutive elements starting at an index that is a multiple of 4.
__device__ __forceinline__ void ldv(const void* p, int kind, std::int64_t i, std::int64_t (&o)[kVec]) {
  switch (kind) {
    case kI8: {
      unsigned w = __ldg(reinterpret_cast<const unsigned*>(static_cast<const std::int8_t*>(p) + i));
#pragma unroll
      for (int l = 0; l < kVec; l++) o[l] = static_cast<std::int8_t>(w >> (8 * l));
      break;
    }
    case kI16: {
      uint2 w = __ldg(reinterpret_cast<const uint2*>(static_cast<const std::int16_t*>(p) + i));
      o[0] = static_cast<std::int16_t>(w.x);
      o[1] = static_cast<std::int16_t>(w.x >> 16);
      o[2] = static_cast<std::int16_t>(w.y);
      o[3] = static_cast<std::int16_t>(w.y >> 16);
      break;
    }
    case kI32: {
      int4 w = __ldg(reinterpret_cast<const int4*>(static_cast<const std::int32_t*>(p) + i));
      o[0] = w.x;
      o[1] = w.y;
      o[2] = w.z;
      o[3] = w.w;
      break;
    }
    default: {
      const longlong2* q = reinterpret_cast<const longlong2*>(static_cast<const long long*>(p) + i);
      longlong2 a = q[0], b = q[1];
      o[0] = a.x;
      o[1] = a.y;
      o[2] = b.x;
      o[3] = b.y;
    }
  }
}

__device__ __forceinline__ void stv(void* p, int kind, std::int64_t i, const std::int64_t (&v)[kVec]) {
  switch (kind) {
    case kI8: {
      unsigned w = 0;
#pragma unroll
      for (int l = 0; l < kVec; l++) w |= (static_cast<unsigned>(v[l]) & 0xffu) << (8 * l);
      *reinterpret_cast<unsigned*>(static_cast<std::int8_t*>(p) + i) = w;
      break;
    }
    case kI16: {
      uint2 w;
      w.x = (static_cast<unsigned>(v[0]) & 0xffffu) | (static_cast<unsigned>(v[1]) << 16);
      w.y = (static_cast<unsigned>(v[2]) & 0xffffu) | (static_cast<unsigned>(v[3]) << 16);
      *reinterpret_cast<uint2*>(static_cast<std::int16_t*>(p) + i) = w;
      break;
    }
    case kI32:
      *reinterpret_cast<int4*>(static_cast<std::int32_t*>(p) + i) =
          make_int4(static_cast<int>(v[0]), static_cast<int>(v[1]), static_cast<int>(v[2]), static_cast<int>(v[3]));
      break;
    default: {
      longlong2* q = reinterpret_cast<longlong2*>(static_cast<long long*>(p) + i);
      q[0] = make_longlong2(v[0], v[1]);
      q[1] = make_longlong2(v[2], v[3]);
    }
  }
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

__global__ void __launch_bounds__(256) map_block_kernel(const GenericDesc* __restrict__ D, BufTable T, DevError* err,
                                                        int launch_id) {
  const GenericDesc& d = *D;
  const int nd = d.ndims;
  const int vdim = d.vdim;
  const std::int64_t rv = d.range[vdim];
  const std::int64_t nchunk = (rv + kVec - 1) / kVec;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t lin = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; lin < d.vcount;
       lin += stride) {
    std::int64_t coord[kMaxDims];
    for (int i = 0; i < nd; i++) coord[i] = 0;
    std::int64_t rest = lin;
    coord[vdim] = (rest % nchunk) * kVec;
    rest /= nchunk;
    for (int i = 1; i < d.npdims; i++) {
      int dim = d.pdims[i];
      coord[dim] = rest % d.range[dim];
      rest /= d.range[dim];
    }
    const int nlane = static_cast<int>(rv - coord[vdim] < kVec ? rv - coord[vdim] : kVec);
    const unsigned full = (1u << nlane) - 1;

    std::int64_t cell[kVecMaxCells][kVec];
    std::int64_t cell_addr[kVecMaxCells];
    int cell_buf[kVecMaxCells];
    unsigned loaded = 0, dirty = 0;
    std::int64_t t[kVecMaxTemps][kVec];
    std::int64_t priv[kVecMaxCells][kVec];

    auto owned = [&](const DAccess& a) -> std::int64_t(&)[kVec] {
      int c = a.cell;
      if (!(loaded >> c & 1u)) {
        std::int64_t base = eval_aff(a.addr, coord, nd);
        cell_addr[c] = base;
        cell_buf[c] = a.buf;
        if (base < 0 || base + nlane > T.elems[a.buf]) {
          report(err, 1, launch_id, base, a.buf);
          cell_buf[c] = -1;
          for (int l = 0; l < kVec; l++) cell[c][l] = 0;
        } else if (nlane == kVec) {
          ldv(T.ptr[a.buf], T.kind[a.buf], base, cell[c]);
        } else {
          for (int l = 0; l < kVec; l++) cell[c][l] = l < nlane ? ld1(T.ptr[a.buf], T.kind[a.buf], base + l) : 0;
        }
        loaded |= 1u << c;
      }
      return cell[c];
    };
    auto opv = [&](int x, int l) -> std::int64_t { return x >= 0 ? t[x][l] : d.consts[-1 - x]; };

    for (;;) {
      unsigned mask = full;
      for (int c = 0; c < d.ncons && mask; c++) {
        std::int64_t b = eval_aff(d.cons[c], coord, nd);
        std::int64_t kv = d.cons[c].k[vdim];
        for (int l = 0; l < kVec; l++)
          if (b + kv * l < 0) mask &= ~(1u << l);
      }
      if (mask) {
        for (int i = 0; i < d.ntemps; i++)
          for (int l = 0; l < kVec; l++) t[i][l] = 0;
        for (int i = 0; i < d.npriv; i++)
          for (int l = 0; l < kVec; l++) priv[i][l] = 0;
        for (int pc = 0; pc < d.ncode; pc++) {
          const DInstr ins = d.code[pc];
          switch (ins.op) {
            case kOpLoad: {
              const DAccess& a = d.acc[ins.acc];
              if (a.mode == kAccOwned) {
                std::int64_t(&c)[kVec] = owned(a);
                for (int l = 0; l < kVec; l++) t[ins.dst][l] = c[l];
                break;
              }
              std::int64_t base = eval_aff(a.addr, coord, nd);
              const std::int8_t vk = d.vkind[ins.acc];
              const std::int64_t n = T.elems[a.buf];
              if (vk == 0) {
                std::int64_t x = 0;
                if (base < 0 || base >= n) report(err, 1, launch_id, base, a.buf);
                else x = ld1(T.ptr[a.buf], T.kind[a.buf], base);
                for (int l = 0; l < kVec; l++) t[ins.dst][l] = x;
              } else if (vk == 1 && mask == full && nlane == kVec && base >= 0 && base + kVec <= n) {
                ldv(T.ptr[a.buf], T.kind[a.buf], base, t[ins.dst]);
              } else {
                std::int64_t kv = vk == 1 ? 1 : a.addr.k[vdim];
                for (int l = 0; l < kVec; l++) {
                  t[ins.dst][l] = 0;
                  if (!(mask >> l & 1u)) continue;
                  std::int64_t ad = base + kv * l;
                  if (ad < 0 || ad >= n) report(err, 1, launch_id, ad, a.buf);
                  else t[ins.dst][l] = ld1(T.ptr[a.buf], T.kind[a.buf], ad);
                }
              }
              break;
            }
            case kOpStore: {
              const DAccess& a = d.acc[ins.acc];
              if (a.mode == kAccOwned) {
                std::int64_t(&c)[kVec] = owned(a);
                for (int l = 0; l < kVec; l++)
                  if (mask >> l & 1u) c[l] = ins.dtype < 0 ? t[ins.a][l] : agg_apply(ins.agg, c[l], t[ins.a][l], ins.dtype);
                dirty |= 1u << a.cell;
              } else {  // thread-owned but not register cached (kAccDirect)
                std::int64_t base = eval_aff(a.addr, coord, nd);
                for (int l = 0; l < kVec; l++) {
                  if (!(mask >> l & 1u)) continue;
                  std::int64_t ad = base + l;
                  if (ad < 0 || ad >= T.elems[a.buf]) {
                    report(err, 1, launch_id, ad, a.buf);
                    continue;
                  }
                  std::int64_t cur = ld1(T.ptr[a.buf], T.kind[a.buf], ad);
                  st1(T.ptr[a.buf], T.kind[a.buf], ad,
                      ins.dtype < 0 ? t[ins.a][l] : agg_apply(ins.agg, cur, t[ins.a][l], ins.dtype));
                }
              }
              break;
            }
            case kOpLoadPriv:
              for (int l = 0; l < kVec; l++) t[ins.dst][l] = priv[ins.acc][l];
              break;
            case kOpStorePriv:
              for (int l = 0; l < kVec; l++)
                priv[ins.acc][l] = agg_apply(d.priv_agg[ins.acc], priv[ins.acc][l], t[ins.a][l], d.priv_dtype[ins.acc]);
              break;
            default:
              for (int l = 0; l < kVec; l++) {
                std::int64_t x = opv(ins.a, l), y = ins.op == kOpNeg || ins.op == kOpConst ? 0 : opv(ins.b, l);
                std::int64_t r;
                switch (ins.op) {
                  case kOpAdd: r = static_cast<std::int64_t>(static_cast<unsigned long long>(x) + static_cast<unsigned long long>(y)); break;
                  case kOpSub: r = static_cast<std::int64_t>(static_cast<unsigned long long>(x) - static_cast<unsigned long long>(y)); break;
                  case kOpMul: r = static_cast<std::int64_t>(static_cast<unsigned long long>(x) * static_cast<unsigned long long>(y)); break;
                  case kOpNeg: r = static_cast<std::int64_t>(0ull - static_cast<unsigned long long>(x)); break;
                  case kOpMax: r = x > y ? x : y; break;
                  case kOpMin: r = x < y ? x : y; break;
                  case kOpCmpEq: r = x == y; break;
                  case kOpCmpNe: r = x != y; break;
                  case kOpCmpLt: r = x < y; break;
                  case kOpCmpLe: r = x <= y; break;
                  case kOpCmpGt: r = x > y; break;
                  case kOpCmpGe: r = x >= y; break;
                  case kOpSelect: r = x != 0 ? y : opv(ins.c, l); break;
                  default: r = x; break;  // constant
                }
                t[ins.dst][l] = r;
              }
              break;
          }
        }
      }
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
    for (int c = 0; c < d.ncells; c++) {
      if (!(dirty >> c & 1u) || cell_buf[c] < 0) continue;
      if (nlane == kVec) {
        stv(T.ptr[cell_buf[c]], T.kind[cell_buf[c]], cell_addr[c], cell[c]);
      } else {
        for (int l = 0; l < nlane; l++) st1(T.ptr[cell_buf[c]], T.kind[cell_buf[c]], cell_addr[c] + l, cell[c][l]);
      }
    }
  }
}

}  // namespace

cudaError_t launch_map(const GenericDesc* d_desc, std::int64_t vcount, const BufTable& t, DevError* err,
                       int launch_id, cudaStream_t s) {
  int block = 256;
  std::int64_t g = (vcount + block - 1) / block;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  map_block_kernel<<<static_cast<int>(g), block, 0, s>>>(d_desc, t, err, launch_id);
  return cudaGetLastError();
}

}  // namespace sb
