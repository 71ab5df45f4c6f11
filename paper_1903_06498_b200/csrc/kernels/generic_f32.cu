// f32 numeric mode of the generic block kernel (the reference's DType has
// no float, ir.h:25; this is the additive fp32 extension the north_star asks for).
//
// Same control flow, owner/atomic/serial modes and bytecode as kernels/generic.cu, with
// fp32 temps and fp32 store-time aggregation.  In owner and serial mode a thread applies
// every point's operations in lexicographic order with correctly rounded, uncontracted
// fp32 operations (this file is compiled with -fmad=false), so results are bitwise equal
// to the CPU restatement's F32 policy (oracle/port).  Atomic mode reorders fp32 sums and
// is tolerance-checked instead.
#include <cuda_runtime.h>

#include <cstdint>

#include "../desc.hpp"

namespace sb {
namespace {

__device__ __forceinline__ float fmax_ref(float a, float b) { return a < b ? b : a; }  // std::max
__device__ __forceinline__ float fmin_ref(float a, float b) { return b < a ? b : a; }  // std::min

__device__ __forceinline__ float agg_f(int agg, float cur, float in) {
  switch (agg) {
    case 0: return in;
    case 1: return __fadd_rn(cur, in);
    case 2: return fmax_ref(cur, in);
    case 3: return fmin_ref(cur, in);
    default: return __fmul_rn(cur, in);
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

// f32 buffers hold floats; spill buffers (kI64) hold the float's bits.
__device__ __forceinline__ float ldf(const void* p, int kind, std::int64_t i) {
  if (kind == kI64) return __int_as_float(static_cast<int>(static_cast<const long long*>(p)[i]));
  return static_cast<const float*>(p)[i];
}
__device__ __forceinline__ void stf(void* p, int kind, std::int64_t i, float v) {
  if (kind == kI64) static_cast<long long*>(p)[i] = __float_as_int(v);
  else static_cast<float*>(p)[i] = v;
}

__device__ void atomic_agg_f(float* a, int agg, float v) {
  if (agg == 1) {
    atomicAdd(a, v);
    return;
  }
  int* ai = reinterpret_cast<int*>(a);
  int old = *ai, assumed;
  do {
    assumed = old;
    float nv = agg_f(agg, __int_as_float(assumed), v);
    old = atomicCAS(ai, assumed, __float_as_int(nv));
  } while (old != assumed);
}

__global__ void __launch_bounds__(128) generic_f32_kernel(const GenericDesc* __restrict__ D, BufTable T, DevError* err,
                                                          int launch_id) {
  const GenericDesc& d = *D;
  const int nd = d.ndims;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t lin = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; lin < d.pcount;
       lin += stride) {
    std::int64_t coord[kMaxDims];
    for (int i = 0; i < nd; i++) coord[i] = 0;
    std::int64_t rest = lin;
    for (int i = 0; i < d.npdims; i++) {
      int dim = d.pdims[i];
      coord[dim] = rest % d.range[dim];
      rest /= d.range[dim];
    }
    float cell[kMaxCells];
    std::int64_t cell_addr[kMaxCells];
    int cell_slot[kMaxCells];
    unsigned loaded = 0, dirty = 0;
    float t[kMaxTemps];
    float priv[kMaxCells];
    auto cell_get = [&](const DAccess& a) -> float& {
      int c = a.cell;
      if (!(loaded >> c & 1u)) {
        std::int64_t addr = eval_aff(a.addr, coord, nd);
        cell_addr[c] = addr;
        cell_slot[c] = a.buf;
        if (addr < 0 || addr >= T.elems[a.buf]) {
          report(err, 1, launch_id, addr, a.buf);
          cell[c] = 0.0f;
          cell_slot[c] = -1;
        } else {
          cell[c] = ldf(T.ptr[a.buf], T.kind[a.buf], addr);
        }
        loaded |= 1u << c;
      }
      return cell[c];
    };
    auto opv = [&](int x) -> float { return x >= 0 ? t[x] : static_cast<float>(d.consts[-1 - x]); };
    for (;;) {
      bool ok = true;
      for (int c = 0; c < d.ncons && ok; c++) ok = eval_aff(d.cons[c], coord, nd) >= 0;
      if (ok) {
        for (int i = 0; i < d.ntemps; i++) t[i] = 0.0f;
        for (int i = 0; i < d.npriv; i++) priv[i] = 0.0f;
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
                  t[ins.dst] = 0.0f;
                } else {
                  t[ins.dst] = ldf(T.ptr[a.buf], T.kind[a.buf], addr);
                }
              }
              break;
            }
            case kOpStore: {
              const DAccess& a = d.acc[ins.acc];
              float v = t[ins.a];
              if (a.mode == kAccOwned) {
                float& c = cell_get(a);
                c = ins.dtype < 0 ? v : agg_f(ins.agg, c, v);
                dirty |= 1u << a.cell;
                break;
              }
              std::int64_t addr = eval_aff(a.addr, coord, nd);
              if (addr < 0 || addr >= T.elems[a.buf]) {
                report(err, 1, launch_id, addr, a.buf);
                break;
              }
              if (a.mode == kAccAtomic) {
                atomic_agg_f(static_cast<float*>(T.ptr[a.buf]) + addr, ins.agg, v);
              } else {
                float cur = ldf(T.ptr[a.buf], T.kind[a.buf], addr);
                stf(T.ptr[a.buf], T.kind[a.buf], addr, ins.dtype < 0 ? v : agg_f(ins.agg, cur, v));
              }
              break;
            }
            case kOpLoadPriv: t[ins.dst] = priv[ins.acc]; break;
            case kOpStorePriv: priv[ins.acc] = agg_f(d.priv_agg[ins.acc], priv[ins.acc], t[ins.a]); break;
            case kOpAdd: t[ins.dst] = __fadd_rn(opv(ins.a), opv(ins.b)); break;
            case kOpSub: t[ins.dst] = __fsub_rn(opv(ins.a), opv(ins.b)); break;
            case kOpMul: t[ins.dst] = __fmul_rn(opv(ins.a), opv(ins.b)); break;
            case kOpNeg: t[ins.dst] = __fsub_rn(0.0f, opv(ins.a)); break;
            case kOpMax: t[ins.dst] = fmax_ref(opv(ins.a), opv(ins.b)); break;
            case kOpMin: t[ins.dst] = fmin_ref(opv(ins.a), opv(ins.b)); break;
            case kOpCmpEq: t[ins.dst] = opv(ins.a) == opv(ins.b) ? 1.0f : 0.0f; break;
            case kOpCmpNe: t[ins.dst] = opv(ins.a) != opv(ins.b) ? 1.0f : 0.0f; break;
            case kOpCmpLt: t[ins.dst] = opv(ins.a) < opv(ins.b) ? 1.0f : 0.0f; break;
            case kOpCmpLe: t[ins.dst] = opv(ins.a) <= opv(ins.b) ? 1.0f : 0.0f; break;
            case kOpCmpGt: t[ins.dst] = opv(ins.a) > opv(ins.b) ? 1.0f : 0.0f; break;
            case kOpCmpGe: t[ins.dst] = opv(ins.a) >= opv(ins.b) ? 1.0f : 0.0f; break;
            case kOpSelect: t[ins.dst] = opv(ins.a) != 0.0f ? opv(ins.b) : opv(ins.c); break;
            case kOpConst: t[ins.dst] = opv(ins.a); break;
            default: report(err, 3, launch_id, pc, -1); break;  // specials are integer-only
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
    for (int c = 0; c < d.ncells; c++)
      if ((dirty >> c & 1u) && cell_slot[c] >= 0) stf(T.ptr[cell_slot[c]], T.kind[cell_slot[c]], cell_addr[c], cell[c]);
  }
}

}  // namespace

cudaError_t launch_generic_f32(const GenericDesc* d_desc, std::int64_t pcount, const BufTable& t, DevError* err,
                               int launch_id, cudaStream_t s) {
  int block = pcount >= 128 ? 128 : 32;
  std::int64_t g = (pcount + block - 1) / block;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  generic_f32_kernel<<<static_cast<int>(g), block, 0, s>>>(d_desc, t, err, launch_id);
  return cudaGetLastError();
}

}  // namespace sb
