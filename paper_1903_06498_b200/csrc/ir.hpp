// Stripe IR data model for the B200 block executor.
//
// This is the executor's INPUT model: a restatement of the reference's
// Program/Block/Index/Constraint/Refinement/Statement structures
// (reference: proj/include/stripe/ir.h:18-156, affine.h:13-42) with the same
// field meaning, so that the canonical text produced by the reference's
// print_program (text.cpp:453-567) round-trips through parse()/print() here
// byte-for-byte.  The executor itself never walks this tree at run time: the
// planner (planner.cpp) lowers it once into flat launch descriptors.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sb {

// Error with a reference-compatible code string ("MissingBuffer", "SyntaxError",
// "OutOfBoundsAccess", ...): interp.h:22-26, text.h:12-18.
struct Error : std::runtime_error {
  Error(std::string code_in, const std::string& message)
      : std::runtime_error(message), code(std::move(code_in)) {}
  std::string code;
};

// Element types.  I8/I16/I32 are the reference's (ir.h:25).  F32 is an
// additive extension for the fp32 numeric mode; the reference
// parser rejects it (text.cpp:257-260), so programs using it only run here.
enum class DType : std::int8_t { I8 = 0, I16 = 1, I32 = 2, F32 = 3 };
enum class Dir : std::int8_t { In = 0, Out = 1, InOut = 2 };
enum class Agg : std::int8_t { Assign = 0, Add = 1, Max = 2, Min = 3, Mul = 4 };

int dtype_bits(DType d);
int dtype_bytes(DType d);
const char* dtype_name(DType d);
const char* agg_name(Agg a);
const char* dir_name(Dir d);
bool is_float(DType d);
std::int64_t dtype_min(DType d);
std::int64_t dtype_max(DType d);

// Two's-complement wrap at the dtype width, sign extended (ir.cpp:39-48).
inline std::int64_t wrap(DType d, std::int64_t v) {
  switch (d) {
    case DType::I8: return static_cast<std::int8_t>(static_cast<std::uint64_t>(v));
    case DType::I16: return static_cast<std::int16_t>(static_cast<std::uint64_t>(v));
    case DType::I32: return static_cast<std::int32_t>(static_cast<std::uint64_t>(v));
    default: return v;
  }
}

// Store-time aggregation on int64 carriers (ir.cpp:79-97).
inline std::int64_t aggregate(Agg op, std::int64_t cur, std::int64_t in, DType d) {
  std::int64_t v = wrap(d, in);
  switch (op) {
    case Agg::Assign: return v;
    case Agg::Add:
      return wrap(d, static_cast<std::int64_t>(static_cast<std::uint64_t>(cur) +
                                               static_cast<std::uint64_t>(v)));
    case Agg::Max: return cur > v ? cur : v;
    case Agg::Min: return cur < v ? cur : v;
    case Agg::Mul:
      return wrap(d, static_cast<std::int64_t>(static_cast<std::uint64_t>(cur) *
                                               static_cast<std::uint64_t>(v)));
  }
  return v;
}

// Integer affine form over named indexes; terms kept sorted by name with no
// zero coefficients (affine.h:11-42).
struct Affine {
  std::vector<std::pair<std::string, std::int64_t>> terms;
  std::int64_t constant = 0;

  Affine() = default;
  explicit Affine(std::int64_t c) : constant(c) {}
  static Affine term(const std::string& name, std::int64_t coeff);

  bool is_constant() const { return terms.empty(); }
  std::int64_t coeff(const std::string& name) const;
  Affine& add(const Affine& rhs, std::int64_t scale = 1);
  bool operator==(const Affine& o) const { return terms == o.terms && constant == o.constant; }
  std::string str() const;  // canonical form, as affine.cpp:52-82 prints it
};

struct Index {
  std::string name;
  std::int64_t range = 1;
  bool is_alias = false;
  Affine alias;  // over the parent scope's indexes
};

struct Location {
  std::string unit;
  Affine bank;
  std::int64_t address = 0;
};

struct Refinement {
  Dir dir = Dir::In;
  std::string name;  // buffer name; children bind parents by name
  std::vector<Affine> offsets;
  bool has_agg = false;
  Agg agg = Agg::Assign;
  DType dtype = DType::I32;
  std::vector<std::int64_t> sizes;
  std::vector<std::int64_t> strides;
  bool has_location = false;
  Location location;
  std::set<std::string> tags;

  std::size_t rank() const { return sizes.size(); }
  // Element count of the flat extent 1 + sum (size-1)*|stride| (ir.cpp:146-155).
  std::int64_t extent() const;
};

struct Block;

// Scalar operand: a $temp or an integer immediate.
struct Operand {
  bool is_imm = false;
  std::int64_t imm = 0;
  std::string temp;
};

enum class StmtKind : std::int8_t { Load, Store, Intrinsic, Special, Block };

struct Statement {
  StmtKind kind = StmtKind::Load;
  std::string into;               // Load: $temp; Store: refinement; Intrinsic: $temp
  std::string from;               // Load: refinement; Store: $temp
  std::string op;                 // Intrinsic / Special name
  std::vector<Operand> args;      // Intrinsic operands
  std::vector<std::string> refs;  // Special operands (refinement names)
  std::unique_ptr<Block> block;   // Block statement

  Statement() = default;
  Statement(const Statement& o);
  Statement& operator=(const Statement& o);
  Statement(Statement&&) = default;
  Statement& operator=(Statement&&) = default;
};

struct Block {
  std::vector<Index> indexes;
  std::vector<Affine> constraints;  // each: expr >= 0
  std::vector<Refinement> refs;
  std::vector<Statement> stmts;
  std::set<std::string> tags;
  bool has_annotation = false;
  std::int64_t annotation = 0;

  std::int64_t range_product() const;
  const Refinement* find_ref(const std::string& name) const;
  const Index* find_index(const std::string& name) const;
};

struct BufferDecl {
  std::string name;
  DType dtype = DType::I32;
  Dir dir = Dir::In;
  std::int64_t elements = 0;
};

struct Program {
  Block root;
  std::vector<BufferDecl> buffers;  // root refinement order
  int buffer_index(const std::string& name) const;
};

// Text format (text.h:20-25).  parse() throws Error("SyntaxError"/"ScopeError").
Program parse_program(const std::string& text);
std::string print_program(const Program& p);
void rebind_buffers(Program* p);

// prepare_outputs' fill value for root buffer `name` (interp.cpp:617-642):
// the identity of the deepest aggregation writing it.
std::int64_t output_identity(const Program& p, const std::string& name);
// The aggregation prepare_outputs keys on (deepest re-declaration, interp.cpp:620-632).
Agg output_aggregation(const Program& p, const std::string& name);
// Split-aggregation sharding: the program with ranged index `idx` of the block at dot path
// `path` restricted to [lo, hi) (idx -> idx + lo below it).  Partial results of the shards
// combine with the output's aggregation (add: sum, max, min, mul: product).
Program restrict_index(const Program& p, const std::string& path, const std::string& idx, std::int64_t lo,
                       std::int64_t hi);
// Throws Error("Unsupported") unless the shards of ranged index `idx` of the block at `path`
// combine exactly with each output's aggregation: every write inside the block's subtree
// goes to a root output whose aggregation (add/max/min/mul) the store uses, or to a local
// declared at or below the block; nothing inside reads an output; nothing outside writes
// one (it would run on every shard).
void check_split(const Program& p, const std::string& path, const std::string& idx);

}  // namespace sb
