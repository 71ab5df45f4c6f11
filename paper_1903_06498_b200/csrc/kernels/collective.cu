// Split-aggregation combine over NCCL: the one collective of the executor.
//
// When an aggregation index is split across GPUs (sb_program_restrict_index, checked exact by
// sb_program_check_split), every rank runs its shard into fresh outputs and the partial
// outputs are all-reduced with the output's aggregation (add -> sum, max -> max, min -> min,
// mul -> prod).  Integer outputs wrap exactly like the reference's store (ir.cpp:79-97): the
// wrapping sum / product of wrapped partials is the wrapped total, max / min are order-free.
// NCCL has no 16-bit integer type, so i16 partials are widened to i32 in a device scratch,
// reduced, and narrowed back (exact for all four operations modulo 2^16).
//
// NCCL is loaded at first use (dlopen "libnccl.so.2": the torch-bundled or the system
// library), so the executor library keeps no link dependency on it; the communicator comes
// from sb_nccl_comm_init (a unique id from sb_nccl_unique_id on rank 0, broadcast by the
// caller's own launcher) or from the caller (any ncclComm_t).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <algorithm>
#include <string>

#include "../ir.hpp"

namespace sb {
namespace {

// the slice of nccl.h this file uses (ABI-stable since NCCL 2.0)
typedef int ncclResult_t;
typedef void* ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
enum { ncclInt8 = 0, ncclInt32 = 2, ncclFloat32 = 7 };
enum { ncclSum = 0, ncclProd = 1, ncclMax = 2, ncclMin = 3 };

struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, std::size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      n.load_error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_reduce || !n.error_string)
      n.load_error = "libnccl.so.2 lacks a required symbol";
  });
  if (!n.load_error.empty()) throw Error("NcclError", n.load_error);
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r != 0) throw Error("NcclError", std::string(what) + ": " + nccl().error_string(r));
}

__global__ void widen16(const std::int16_t* in, std::int32_t* out, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}
__global__ void narrow16(const std::int32_t* in, std::int16_t* out, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = static_cast<std::int16_t>(in[i]);
}

}  // namespace

void nccl_unique_id(char (&id)[128]) {
  ncclUniqueId u;
  check(nccl().get_unique_id(&u), "ncclGetUniqueId");
  std::memcpy(id, u.internal, 128);
}

void* nccl_comm_init(int nranks, const char* id, int rank) {
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  ncclComm_t c = nullptr;
  check(nccl().comm_init_rank(&c, nranks, u, rank), "ncclCommInitRank");
  return c;
}

void nccl_comm_destroy(void* comm) { check(nccl().comm_destroy(comm), "ncclCommDestroy"); }

// In-place all-reduce of one output's partials (native width on the device) with its
// aggregation; stream-ordered on `s`.
void split_allreduce(void* comm, void* data, long long count, DType dt, Agg agg, cudaStream_t s) {
  int op;
  switch (agg) {
    case Agg::Add: op = ncclSum; break;
    case Agg::Max: op = ncclMax; break;
    case Agg::Min: op = ncclMin; break;
    case Agg::Mul: op = ncclProd; break;
    default: throw Error("Unsupported", "an assigned output cannot be combined across shards");
  }
  if (count <= 0) return;
  const Nccl& n = nccl();
  if (dt == DType::I16) {
    std::int32_t* wide = nullptr;
    if (cudaMallocAsync(&wide, count * sizeof(std::int32_t), s) != cudaSuccess)
      throw Error("CudaError", "cudaMallocAsync(i16 widen)");
    const int grid = static_cast<int>(std::min<long long>((count + 255) / 256, 148 * 8));
    widen16<<<grid, 256, 0, s>>>(static_cast<const std::int16_t*>(data), wide, count);
    const ncclResult_t r = n.all_reduce(wide, wide, static_cast<std::size_t>(count), ncclInt32, op, comm, s);
    if (r == 0) narrow16<<<grid, 256, 0, s>>>(wide, static_cast<std::int16_t*>(data), count);
    cudaFreeAsync(wide, s);
    check(r, "ncclAllReduce");
    if (cudaGetLastError() != cudaSuccess) throw Error("CudaError", "i16 widen/narrow");
    return;
  }
  const int type = dt == DType::I8 ? ncclInt8 : dt == DType::F32 ? ncclFloat32 : ncclInt32;
  check(n.all_reduce(data, data, static_cast<std::size_t>(count), type, op, comm, s), "ncclAllReduce");
}

}  // namespace sb
