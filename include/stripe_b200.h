/*
 * stripe_b200.h — C ABI of the B200-native Stripe block executor.
 *
 * Drop-in boundary for the reference's block executor (Stripe Kit,
 * arXiv 1903.06498 reference).  The reference exposes a C++ free-function API
 * with no FFI; each entry point below replaces one reference interface, cited
 * file:line relative to /root/reference/proj:
 *
 *   sb_program_parse / sb_program_print    parse_program / print_program   include/stripe/text.h:20-25
 *   sb_program_buffer_*                    Program::buffers, rebind_buffers include/stripe/ir.h:146-160
 *   sb_program_output_identity             prepare_outputs' fill value      include/stripe/interp.h:70-73
 *   sb_execute                             execute(Program, BufferStore*, ExecOptions)
 *                                                                           include/stripe/interp.h:68
 *   sb_execute_device                      same, buffers already resident in HBM (benchmarks)
 *   sb_exec_options                        ExecOptions / IterOrder          include/stripe/interp.h:58-64
 *   sb_last_error / SB_ERR_*               ExecError{code}                  include/stripe/interp.h:22-26
 *
 * Plain C types only: no C++ or torch types cross this boundary, and no
 * exceptions: every call returns an SB_ERR_* status and sb_last_error()
 * holds "Code: message" for the calling thread.  There is no CPU fallback:
 * without a usable sm_100 device, sb_context_create fails.
 */
#ifndef STRIPE_B200_H
#define STRIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_ABI_VERSION 1

/* Status codes; names match the reference's ExecError / ParseError codes. */
enum {
  SB_OK = 0,
  SB_ERR_MISSING_BUFFER = 1,     /* "MissingBuffer"      interp.cpp:187-192, 312 */
  SB_ERR_UNKNOWN_INTRINSIC = 2,  /* "UnknownIntrinsic"   interp.cpp:270 */
  SB_ERR_UNKNOWN_SPECIAL = 3,    /* "UnknownSpecial"     interp.cpp:289-293, 546-549 */
  SB_ERR_UNDEFINED_TEMP = 4,     /* "UndefinedTemp"      interp.cpp:321 */
  SB_ERR_OUT_OF_BOUNDS = 5,      /* "OutOfBoundsAccess"  interp.cpp:463-478, 560-578 */
  SB_ERR_UNBOUND_INDEX = 6,      /* "UnboundIndex"       affine.h:46-50 */
  SB_ERR_SYNTAX = 7,             /* "SyntaxError"        text.h:12-18 */
  SB_ERR_SCOPE = 8,              /* "ScopeError"         text.h:12-18 */
  SB_ERR_UNSUPPORTED = 9,        /* outside this executor's contract (e.g. observers) */
  SB_ERR_CUDA = 10,              /* CUDA runtime / driver failure */
  SB_ERR_NCCL = 11,              /* NCCL failure (split aggregations) */
  SB_ERR_INVALID = 12,           /* bad argument at the ABI */
  SB_ERR_PASS = 13               /* PassError{code} "InvalidTile"/"NotTileable" (passes.h, tile.cpp:104-133) */
};

/* Element dtypes (bit widths; ir.h:25) plus the fp32 extension. */
enum { SB_I8 = 8, SB_I16 = 16, SB_I32 = 32, SB_F32 = 0x20F };

/* Buffer directions of root refinements. */
enum { SB_IN = 0, SB_OUT = 1, SB_INOUT = 2 };

/* Host carriers: the reference's int64 BufferStore vectors (interp.h:14-20),
 * or native-width arrays (int8/int16/int32/float). */
enum { SB_CARRIER_I64 = 0, SB_CARRIER_NATIVE = 1 };

/* Buffer flags. */
enum {
  SB_BUF_PREPARE = 1 /* output absent from the store: create it with prepare_outputs' identity
                        (interp.cpp:617-642) on the device; input contents are ignored */
};

typedef struct sb_host_buffer {
  const char* name;
  int32_t carrier; /* SB_CARRIER_* */
  int32_t flags;   /* SB_BUF_* */
  void* data;      /* int64_t[count] or native[count]; outputs are written back in place */
  int64_t count;   /* element count; must equal the program's buffer table entry */
} sb_host_buffer;

typedef struct sb_device_buffer {
  const char* name;
  int32_t flags; /* SB_BUF_* */
  int32_t reserved;
  void* dptr;    /* native-width device array; allocation padded to 16 bytes */
  int64_t count;
} sb_device_buffer;

enum { SB_FP32_EXACT = 0, SB_FP32_TF32X3 = 1 };

typedef struct sb_exec_options {
  int32_t order;     /* IterOrder: 0 Lex, 1 Reversed, 2 Shuffled — accepted, result is order-free */
  int32_t observer;  /* nonzero = caller wants an ExecObserver: rejected (SB_ERR_UNSUPPORTED) */
  uint64_t seed;     /* Shuffled seed (ignored) */
  int32_t disable_tensor_cores; /* force the generic kernel family (testing) */
  int32_t fp32_mode; /* SB_FP32_EXACT (0): fp32 matmuls bitwise equal to the CPU F32 policy;
                        SB_FP32_TF32X3 (1): 3xTF32 tensor cores, |err| <= 1e-5 * sum|a||b| */
} sb_exec_options;

typedef struct sb_context sb_context;
typedef struct sb_program sb_program;

const char* sb_last_error(void);
const char* sb_status_name(int status);
int sb_abi_version(void);

/* ---- programs (host only; no GPU needed) ---- */
int sb_program_parse(const char* text, sb_program** out);
void sb_program_free(sb_program* p);
int sb_program_print(const sb_program* p, char* buf, size_t cap, size_t* len);
int sb_program_buffer_count(const sb_program* p);
int sb_program_buffer_info(const sb_program* p, int i, const char** name, int* dtype,
                           int64_t* elements, int* dir);
int sb_program_output_identity(const sb_program* p, const char* name, int64_t* value);
/* Aggregation of a root output (0 assign, 1 add, 2 max, 3 min, 4 mul) as prepare_outputs
 * resolves it (interp.cpp:620-632). */
int sb_program_output_aggregation(const sb_program* p, const char* name, int* agg);
/* Constraint-satisfying points of the block at `block_path` (its own ranged indexes and
 * constraints), the reference's count_valid_points (tile.cpp:338-370) evaluated on the
 * device in closed form per innermost row. */
int sb_count_valid_points(sb_context* ctx, const sb_program* p, const char* block_path, int64_t* count);
/* TileCostReport (passes.h:42-50); excluded = 1 for "MemCap". */
typedef struct sb_tile_report {
  int64_t lines_total;
  int64_t useful_ops;
  int64_t tile_elements;
  int32_t excluded;
} sb_tile_report;
/* tile_cost(block, parse_tile_shape(tiles), CacheModel{line}, mem_cap) (passes.h:60-67,
 * tile.cpp:380-455) of the block at `block_path`, evaluated on the device: same report, same
 * PassError codes (SB_ERR_PASS, sb_last_error "InvalidTile: ..."/"NotTileable: ...").
 * `interleaved` = TileShape::interleaved.  line <= 4096 elements. */
int sb_tile_cost(sb_context* ctx, const sb_program* p, const char* block_path, const char* tiles, int interleaved,
                 int64_t line, int64_t mem_cap, sb_tile_report* out);
/* autotile(block, CacheModel{line}, AutotileOptions{mem_cap, power_of_two}) (passes.h:85-89,
 * tile.cpp:475-535): the exhaustive divisor (or power-of-two) search, every candidate's lines
 * counted on the device.  *found = 0 when every candidate exceeds the cap (the reference's
 * "NoFeasibleTile" warning); otherwise `chosen` gets TileShape::to_string ("m:32,n:64", names
 * sorted), *len its length.  The caller applies the reference's tile_rewrite to it. */
int sb_autotile(sb_context* ctx, const sb_program* p, const char* block_path, int64_t line, int64_t mem_cap,
                int power_of_two, char* chosen, size_t cap, size_t* len, int* found, sb_tile_report* report,
                int64_t* candidates, int64_t* excluded);
/* Split-aggregation sharding: a copy of `p` whose ranged index `index` in the
 * block at dot path `block_path` ("" = root, "0", "0.1", ...) runs over [lo, hi) only.
 * Shards' outputs combine with the output's aggregation (all-reduce sum/max/min/prod). */
int sb_program_restrict_index(const sb_program* p, const char* block_path, const char* index, int64_t lo,
                              int64_t hi, sb_program** out);
/* The split-aggregation combine over NCCL (the reference has no split,
 * tile.cpp:668-685): every rank runs its shard (sb_program_restrict_index) into fresh
 * outputs, then sb_split_allreduce all-reduces each output's partials in place on the
 * context stream with the output's aggregation (add -> sum, max -> max, min -> min,
 * mul -> prod; integer wrap exact; i16 reduced as i32).  `data` = the output's device buffer
 * at native width, `count` its element count.  NCCL (libnccl.so.2) is loaded at first use;
 * the communicator is any ncclComm_t, or one from sb_nccl_comm_init with the 128-byte id
 * sb_nccl_unique_id made on rank 0 and broadcast by the caller.  SB_ERR_NCCL on NCCL
 * failures. */
int sb_nccl_unique_id(char* id /* [128] */);
int sb_nccl_comm_init(sb_context* ctx, int nranks, const char* id, int rank, void** comm);
int sb_nccl_comm_destroy(void* comm);
int sb_split_allreduce(sb_context* ctx, const sb_program* p, const char* name, void* data, int64_t count,
                       void* nccl_comm);
/* SB_OK when splitting ranged `index` of the block at `block_path` across shards and
 * combining the shards' outputs with each output's aggregation is exact; otherwise
 * SB_ERR_UNSUPPORTED with the reason (an assigned output, a store whose aggregation differs
 * from the output's, a read of an output or a write to an outer local inside the block, or
 * an output written outside it).  The reference has no split (tile.cpp:668-685 refuses
 * aggregation indexes in `partition`); this states the condition under which one is exact. */
int sb_program_check_split(const sb_program* p, const char* block_path, const char* index);
/* Human-readable launch plan (which kernel family / execution mode per block).
 * `disable_tensor_cores` bit 0: generic kernels only; bit 1: plan for SB_FP32_TF32X3. */
int sb_program_describe_plan(sb_program* p, int fresh_outputs, int disable_tensor_cores, char* buf,
                             size_t cap, size_t* len);

/* ---- device contexts ---- */
int sb_context_create(int device, sb_context** out);
void sb_context_destroy(sb_context* ctx);
/* Launch on an external cudaStream_t (e.g. torch's current stream); NULL = own stream. */
int sb_context_set_stream(sb_context* ctx, void* cuda_stream);
void* sb_context_stream(sb_context* ctx);
/* Kernel order across contexts (host-buffer executes, sb_execute / sb_execute_async): while
 * enabled, this context's kernels start only after the kernels of the previous execute of any
 * ordered context on the same device; its host<->device copies are not held back.  Two
 * contexts ping-ponging steps then overlap one step's copies with the other's kernels
 * without running both steps' kernels at once. */
int sb_context_set_kernel_order(sb_context* ctx, int enable);
/* Waits for the stream and reports any device-side error (OutOfBoundsAccess ...). */
int sb_context_sync(sb_context* ctx);
/* Number of kernels this library launched on the context so far. */
/* Per-step device timing (development and bench aid): while enabled, every execute runs its
 * steps serially on the context stream bracketed by CUDA events and appends one line per
 * step, "step ms kernel path points", read (and cleared) by sb_context_profile_read. */
int sb_context_set_profile(sb_context* ctx, int enable);
int sb_context_profile_read(sb_context* ctx, char* buf, size_t cap, size_t* len);
uint64_t sb_context_launch_count(sb_context* ctx);
int sb_device_alloc(sb_context* ctx, int64_t bytes, void** dptr);
int sb_device_free(sb_context* ctx, void* dptr);
int sb_host_alloc_pinned(int64_t bytes, void** ptr);
int sb_host_free_pinned(void* ptr);

/* ---- execution ---- */
/* Reference-compatible execute: host buffers in, outputs written back; synchronous. */
int sb_execute(sb_context* ctx, sb_program* p, sb_host_buffer* bufs, int n,
               const sb_exec_options* opts);
/* HBM-resident execute: enqueues on the context stream and returns (call sb_context_sync). */
int sb_execute_device(sb_context* ctx, sb_program* p, const sb_device_buffer* bufs, int n,
                      const sb_exec_options* opts);

/* ---- CUDA graphs (launch overhead off the critical path) ---- */
/* Asynchronous sb_execute: native-width carriers in pinned host memory (sb_host_alloc_pinned),
 * H2D + kernels + D2H enqueued on the context stream and the call returns; results and
 * device errors are available after sb_context_sync.  Two contexts ping-ponging steps
 * overlap one step's device-to-host copy with the next step's host-to-device copy. */
int sb_execute_async(sb_context* ctx, sb_program* p, sb_host_buffer* bufs, int n,
                     const sb_exec_options* opts);

typedef struct sb_graph sb_graph;
/* Starts capturing everything this thread enqueues on the context stream
 * (sb_execute_device calls; plans must have run once outside capture). */
int sb_graph_begin(sb_context* ctx);
int sb_graph_end(sb_context* ctx, sb_graph** out);
int sb_graph_launch(sb_context* ctx, sb_graph* g);
void sb_graph_free(sb_graph* g);

#ifdef __cplusplus
}
#endif

#endif /* STRIPE_B200_H */
