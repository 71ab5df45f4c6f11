// POD launch descriptors shared by the host planner and the sm_100a kernels.
// Everything here is plain data so it can be memcpy'd to HBM once per plan.
#pragma once

#include <cstdint>

namespace sb {

constexpr int kMaxDims = 24;     // flattened nest depth (ranged indexes along one root-to-leaf chain)
constexpr int kMaxAccess = 32;   // distinct (buffer, affine) accesses in one launch
constexpr int kMaxCons = 24;     // constraints in one launch
constexpr int kMaxCode = 160;    // bytecode instructions in one leaf body
constexpr int kMaxConsts = 64;   // immediate pool
constexpr int kMaxTemps = 64;    // int64 temps per point
constexpr int kMaxCells = 16;    // owned output cells / private allocs per thread
constexpr int kMaxBufs = 48;     // buffers visible to one launch (roots + scratch)
constexpr int kMaxSpecial = 4;   // gather/scatter statements per body
constexpr int kMaxRank = 8;      // refinement rank for specials

// Device element kinds (storage width); I64 is the temp-spill carrier.
enum : std::int8_t { kI8 = 0, kI16 = 1, kI32 = 2, kF32 = 3, kI64 = 4 };

// Dense affine over the launch's dims: addr = c + sum_d k[d] * coord[d].
struct DAff {
  std::int64_t c;
  std::int64_t k[kMaxDims];
};

// How one access reaches memory.
enum : std::int8_t {
  kAccRead = 0,    // read-only in this launch: direct load
  kAccOwned = 1,   // owner-computes: the thread's private cell (register) for this address
  kAccAtomic = 2,  // commutative aggregation via device atomics
  kAccDirect = 3,  // serial mode: plain read-modify-write
};

struct DAccess {
  std::int16_t buf;
  std::int8_t mode;
  std::int8_t cell;  // owned cell index (kAccOwned)
  DAff addr;
};

// Bytecode.  Operands >= 0 are temps; < 0 are const-pool entries (-1 - i).
enum : std::uint8_t {
  kOpLoad = 0,      // t[dst] = mem[acc]
  kOpStore = 1,     // mem[acc] = agg(mem[acc], wrap(t[a]))
  kOpLoadPriv = 2,  // t[dst] = priv[cell]
  kOpStorePriv = 3, // priv[cell] = agg(priv[cell], wrap(t[a]))
  kOpAdd, kOpSub, kOpMul, kOpNeg, kOpMax, kOpMin,
  kOpCmpEq, kOpCmpNe, kOpCmpLt, kOpCmpLe, kOpCmpGt, kOpCmpGe,
  kOpSelect, kOpConst,
  kOpGather, kOpScatter,  // special; `acc` indexes the special table
};

struct DInstr {
  std::uint8_t op;
  std::int8_t agg;    // store aggregation (Agg)
  std::int8_t dtype;  // store wrap dtype (DType)
  std::int8_t acc;    // access / private cell / special index
  std::int16_t dst;
  std::int16_t a, b, c;
};

struct DSpecial {
  std::int8_t dst, src, idx;  // access indices (view bases)
  std::int8_t rank;
  std::int8_t dst_agg, dst_dtype;
  std::int64_t walk[kMaxRank];
  std::int64_t sdst[kMaxRank], ssrc[kMaxRank], sidx[kMaxRank];
  std::int64_t bound;  // sizes[0] of the picked operand
};

enum : std::int8_t { kModeOwner = 0, kModeAtomic = 1, kModeSerial = 2 };

// One flat launch of the generic block kernel.
struct GenericDesc {
  std::int32_t ndims, ncons, nacc, ncode, nconsts, ntemps, ncells, npriv, nspecial;
  std::int8_t mode;
  std::int8_t npdims, nrdims;
  std::int8_t pdims[kMaxDims];  // thread-mapped dims, fastest first
  std::int8_t rdims[kMaxDims];  // serial dims, declaration (outer->inner) order
  std::int64_t range[kMaxDims];
  std::int64_t pcount;          // product of pdim ranges
  std::int64_t cell_elem_dummy;
  std::int8_t priv_agg[kMaxCells], priv_dtype[kMaxCells];
  DAff cons[kMaxCons];
  DAccess acc[kMaxAccess];
  DInstr code[kMaxCode];
  std::int64_t consts[kMaxConsts];
  DSpecial special[kMaxSpecial];
  // vectorised owner-mode variant (kernels/map.cu): one thread owns kVec consecutive
  // points of the fastest thread dim `vdim`
  std::int8_t vdim;
  std::int8_t vkind[kMaxAccess];  // 0 broadcast (coef 0), 1 contiguous aligned vector, 2 per-lane
  std::int64_t vcount;            // threads: pcount / range[vdim] * ceil(range[vdim] / kVec)
  std::int8_t is_float;           // f32 numeric mode: temps, cells and aggregation in fp32
};

constexpr int kVec = 4;            // lanes per thread in the map kernel
constexpr int kVecMaxTemps = 8;
constexpr int kVecMaxCells = 4;

// Per-run buffer table (kernel parameter, by value).
struct BufTable {
  void* ptr[kMaxBufs];
  std::int64_t elems[kMaxBufs];
  std::int8_t kind[kMaxBufs];
};

// Device-side error report (first error wins).
struct DevError {
  int code;  // 0 none, 1 OutOfBoundsAccess (load/store), 2 gather/scatter index
  int launch;
  long long addr;
  long long buf;
};

}  // namespace sb
