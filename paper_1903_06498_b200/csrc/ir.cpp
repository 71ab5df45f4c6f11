// IR helpers, canonical printer and buffer table for the B200 executor.
// Printer output format follows the reference printer (text.cpp:453-567) so
// the two round-trip identically; the code is an independent implementation.
#include "ir.hpp"

#include <algorithm>
#include <sstream>

namespace sb {

int dtype_bits(DType d) {
  switch (d) {
    case DType::I8: return 8;
    case DType::I16: return 16;
    case DType::I32: return 32;
    case DType::F32: return 32;
  }
  return 0;
}
int dtype_bytes(DType d) { return dtype_bits(d) / 8; }
bool is_float(DType d) { return d == DType::F32; }

const char* dtype_name(DType d) {
  switch (d) {
    case DType::I8: return "i8";
    case DType::I16: return "i16";
    case DType::I32: return "i32";
    case DType::F32: return "f32";
  }
  return "?";
}

const char* agg_name(Agg a) {
  static const char* names[] = {"assign", "add", "max", "min", "mul"};
  return names[static_cast<int>(a)];
}

const char* dir_name(Dir d) {
  static const char* names[] = {"in", "out", "inout"};
  return names[static_cast<int>(d)];
}

std::int64_t dtype_min(DType d) { return -(std::int64_t{1} << (dtype_bits(d) - 1)); }
std::int64_t dtype_max(DType d) { return (std::int64_t{1} << (dtype_bits(d) - 1)) - 1; }

Affine Affine::term(const std::string& name, std::int64_t coeff) {
  Affine a;
  if (coeff != 0) a.terms.emplace_back(name, coeff);
  return a;
}

std::int64_t Affine::coeff(const std::string& name) const {
  for (const auto& [n, c] : terms)
    if (n == name) return c;
  return 0;
}

Affine& Affine::add(const Affine& rhs, std::int64_t scale) {
  if (scale == 0) return *this;
  std::vector<std::pair<std::string, std::int64_t>> merged;
  merged.reserve(terms.size() + rhs.terms.size());
  std::size_t i = 0, j = 0;
  while (i < terms.size() || j < rhs.terms.size()) {
    if (j == rhs.terms.size() || (i < terms.size() && terms[i].first < rhs.terms[j].first)) {
      merged.push_back(terms[i++]);
    } else if (i == terms.size() || rhs.terms[j].first < terms[i].first) {
      merged.emplace_back(rhs.terms[j].first, rhs.terms[j].second * scale);
      j++;
    } else {
      std::int64_t c = terms[i].second + rhs.terms[j].second * scale;
      if (c != 0) merged.emplace_back(terms[i].first, c);
      i++;
      j++;
    }
  }
  terms.swap(merged);
  constant += rhs.constant * scale;
  return *this;
}

std::string Affine::str() const {
  std::ostringstream os;
  bool lead = true;
  for (const auto& [name, c] : terms) {
    if (lead) {
      if (c == -1) os << "-";
      else if (c != 1) os << c << "*";
    } else {
      os << (c < 0 ? " - " : " + ");
      std::int64_t m = c < 0 ? -c : c;
      if (m != 1) os << m << "*";
    }
    os << name;
    lead = false;
  }
  if (lead) os << constant;
  else if (constant > 0) os << " + " << constant;
  else if (constant < 0) os << " - " << -constant;
  return os.str();
}

std::int64_t Refinement::extent() const {
  std::int64_t e = 1;
  for (std::size_t d = 0; d < sizes.size(); d++) {
    std::int64_t s = strides[d] < 0 ? -strides[d] : strides[d];
    e += (sizes[d] - 1) * s;
  }
  return e;
}

Statement::Statement(const Statement& o)
    : kind(o.kind), into(o.into), from(o.from), op(o.op), args(o.args), refs(o.refs),
      block(o.block ? std::make_unique<Block>(*o.block) : nullptr) {}

Statement& Statement::operator=(const Statement& o) {
  if (this != &o) {
    Statement tmp(o);
    *this = std::move(tmp);
  }
  return *this;
}

std::int64_t Block::range_product() const {
  std::int64_t p = 1;
  for (const auto& idx : indexes)
    if (!idx.is_alias) p *= idx.range;
  return p;
}

const Refinement* Block::find_ref(const std::string& name) const {
  for (const auto& r : refs)
    if (r.name == name) return &r;
  return nullptr;
}

const Index* Block::find_index(const std::string& name) const {
  for (const auto& i : indexes)
    if (i.name == name) return &i;
  return nullptr;
}

int Program::buffer_index(const std::string& name) const {
  for (std::size_t i = 0; i < buffers.size(); i++)
    if (buffers[i].name == name) return static_cast<int>(i);
  return -1;
}

void rebind_buffers(Program* p) {
  p->buffers.clear();
  for (const auto& r : p->root.refs) {
    BufferDecl d;
    d.name = r.name;
    d.dtype = r.dtype;
    d.dir = r.dir;
    d.elements = r.extent();
    p->buffers.push_back(d);
  }
}

namespace {

void tabs(std::ostringstream& os, int n) {
  for (int i = 0; i < n; i++) os << '\t';
}

void print_ints(std::ostringstream& os, const std::vector<std::int64_t>& v) {
  os << '(';
  for (std::size_t i = 0; i < v.size(); i++) os << (i ? ", " : "") << v[i];
  os << ')';
}

void print_block(std::ostringstream& os, const Block& b, int depth) {
  tabs(os, depth);
  os << "block [";
  for (std::size_t i = 0; i < b.indexes.size(); i++) {
    const auto& idx = b.indexes[i];
    if (i) os << ", ";
    if (idx.is_alias) os << idx.name << '=' << idx.alias.str();
    else os << idx.name << ':' << idx.range;
  }
  os << "]:" << (b.has_annotation ? b.annotation : b.range_product()) << " (\n";
  for (const auto& t : b.tags) {
    tabs(os, depth + 1);
    os << '#' << t << '\n';
  }
  for (const auto& c : b.constraints) {
    tabs(os, depth + 1);
    os << c.str() << " >= 0\n";
  }
  for (const auto& r : b.refs) {
    tabs(os, depth + 1);
    os << dir_name(r.dir) << ' ' << r.name << '[';
    for (std::size_t d = 0; d < r.offsets.size(); d++) os << (d ? ", " : "") << r.offsets[d].str();
    os << ']';
    if (r.has_agg) os << ':' << agg_name(r.agg);
    os << ' ' << dtype_name(r.dtype);
    print_ints(os, r.sizes);
    os << ':';
    print_ints(os, r.strides);
    if (r.has_location)
      os << " @" << r.location.unit << '[' << r.location.bank.str() << "]:" << r.location.address;
    for (const auto& t : r.tags) os << " #" << t;
    os << '\n';
  }
  tabs(os, depth);
  os << ") {\n";
  for (std::size_t i = 0; i < b.stmts.size(); i++) {
    const auto& s = b.stmts[i];
    tabs(os, depth + 1);
    os << i << ':';
    switch (s.kind) {
      case StmtKind::Block:
        os << '\n';
        print_block(os, *s.block, depth + 1);
        continue;
      case StmtKind::Load: os << ' ' << s.into << " = load(" << s.from << ')'; break;
      case StmtKind::Store: os << ' ' << s.into << " = store(" << s.from << ')'; break;
      case StmtKind::Intrinsic:
        os << ' ' << s.into << " = " << s.op << '(';
        for (std::size_t a = 0; a < s.args.size(); a++) {
          if (a) os << ", ";
          if (s.args[a].is_imm) os << s.args[a].imm;
          else os << s.args[a].temp;
        }
        os << ')';
        break;
      case StmtKind::Special:
        os << " special " << s.op << '(';
        for (std::size_t a = 0; a < s.refs.size(); a++) os << (a ? ", " : "") << s.refs[a];
        os << ')';
        break;
    }
    os << '\n';
  }
  tabs(os, depth);
  os << "}\n";
}

}  // namespace

std::string print_program(const Program& p) {
  std::ostringstream os;
  print_block(os, p.root, 0);
  return os.str();
}

Agg output_aggregation(const Program& p, const std::string& name) {
  const Refinement* root_ref = p.root.find_ref(name);
  if (!root_ref) throw Error("MissingBuffer", "no root refinement '" + name + "'");
  Agg agg = root_ref->has_agg ? root_ref->agg : Agg::Assign;
  std::vector<const Block*> stack = {&p.root};
  while (!stack.empty()) {
    const Block* b = stack.back();
    stack.pop_back();
    const Refinement* r = b->find_ref(name);
    if (b != &p.root && (r == nullptr || !r->has_agg)) continue;
    if (r && r->has_agg) agg = r->agg;
    for (const auto& s : b->stmts)
      if (s.kind == StmtKind::Block) stack.push_back(s.block.get());
  }
  return agg;
}

namespace {

// idx -> idx + lo in every affine that sees `idx` (the block's own constraints and
// refinement offsets, and the subtree below it until a block redeclares the name).
void shift_index(Block* b, const std::string& idx, std::int64_t lo, bool own) {
  auto fix = [&](Affine& a) {
    const std::int64_t k = a.coeff(idx);
    if (k) a.constant += k * lo;
  };
  if (!own) {
    // every alias reads the parent scope (interp.cpp:210), whatever its position among the
    // block's indexes -- tile_rewrite emits `[x:3, ..., xo = 3*x]` with the child's ranged x
    // declared before the alias that reads the parent's x (testdata/fig6b.stripe)
    for (auto& i : b->indexes)
      if (i.is_alias) fix(i.alias);
    for (const auto& i : b->indexes)
      if (i.name == idx) return;  // shadowed below this point
  }
  for (auto& c : b->constraints) fix(c);
  for (auto& r : b->refs)
    for (auto& o : r.offsets) fix(o);
  for (auto& s : b->stmts)
    if (s.kind == StmtKind::Block) shift_index(s.block.get(), idx, lo, false);
}

}  // namespace

Program restrict_index(const Program& p, const std::string& path, const std::string& idx, std::int64_t lo,
                       std::int64_t hi) {
  Program q = p;
  Block* b = &q.root;
  std::stringstream ss(path);
  std::string part;
  while (!path.empty() && std::getline(ss, part, '.')) {
    const std::size_t k = static_cast<std::size_t>(std::stoll(part));
    if (k >= b->stmts.size() || b->stmts[k].kind != StmtKind::Block)
      throw Error("Unsupported", "no block at path '" + path + "'");
    b = b->stmts[k].block.get();
  }
  Index* target = nullptr;
  for (auto& i : b->indexes)
    if (i.name == idx && !i.is_alias) target = &i;
  if (!target) throw Error("UnboundIndex", "block '" + path + "' has no ranged index '" + idx + "'");
  if (lo < 0 || hi > target->range || lo >= hi) throw Error("Unsupported", "bad index range");
  target->range = hi - lo;
  shift_index(b, idx, lo, true);
  if (b->has_annotation) b->annotation = b->range_product();
  return q;
}

namespace {

// Binding of a refinement name in some scope: a root buffer, or a local allocation
// (declared in the block `owner`, interp.cpp:234-247).
struct Bound {
  int root = -1;                 // root buffer index, else local
  const Block* owner = nullptr;  // declaring block of a local
  bool local_inside = false;     // local declared at or below the split block
};


struct SplitCheck {
  const Program& p;
  const Block* split;
  std::string why;

  void fail(const std::string& w) {
    if (why.empty()) why = w;
  }

  void walk(const Block& b, const std::map<std::string, Bound>& parent, bool inside) {
    inside = inside || &b == split;
    std::map<std::string, Bound> env;
    for (const auto& r : b.refs) {
      Bound x;
      if (&b == &p.root) {
        x.root = p.buffer_index(r.name);
      } else {
        auto it = parent.find(r.name);
        if (it != parent.end()) {
          x = it->second;
        } else {
          x.owner = &b;
          x.local_inside = inside;
        }
      }
      env[r.name] = x;
    }
    auto agg_of = [&](const std::string& name) {
      const Refinement* r = b.find_ref(name);
      return r && r->has_agg ? r->agg : Agg::Assign;
    };
    auto on_write = [&](const std::string& name) {
      auto it = env.find(name);
      if (it == env.end()) return;
      const Bound& x = it->second;
      const bool out = x.root >= 0 && p.buffers[x.root].dir != Dir::In;
      if (!inside) {
        if (out) fail("a statement outside the split block writes output '" + name + "' (it would run on every shard)");
        return;
      }
      if (x.root >= 0) {
        const Agg a = output_aggregation(p, p.buffers[x.root].name);
        if (a == Agg::Assign)
          fail("output '" + p.buffers[x.root].name + "' is assigned, not aggregated: it cannot be split");
        else if (agg_of(name) != a)
          fail("a store into '" + name + "' aggregates differently from the output's combine");
      } else if (!x.local_inside) {
        fail("local '" + name + "' declared outside the split block would carry partial results");
      }
    };
    auto on_read = [&](const std::string& name) {
      if (!inside) return;
      auto it = env.find(name);
      if (it != env.end() && it->second.root >= 0 && p.buffers[it->second.root].dir != Dir::In)
        fail("the split block reads output '" + name + "' (a partial value on each shard)");
    };
    for (const auto& st : b.stmts) {
      switch (st.kind) {
        case StmtKind::Load: on_read(st.from); break;
        case StmtKind::Store: on_write(st.into); break;
        case StmtKind::Special:
          if (!st.refs.empty()) on_write(st.refs[0]);
          for (std::size_t k = 1; k < st.refs.size(); k++) on_read(st.refs[k]);
          break;
        case StmtKind::Block: walk(*st.block, env, inside); break;
        default: break;
      }
    }
  }
};

}  // namespace

void check_split(const Program& p, const std::string& path, const std::string& idx) {
  const Block* b = &p.root;
  std::stringstream ss(path);
  std::string part;
  while (!path.empty() && std::getline(ss, part, '.')) {
    const std::size_t k = static_cast<std::size_t>(std::stoll(part));
    if (k >= b->stmts.size() || b->stmts[k].kind != StmtKind::Block)
      throw Error("Unsupported", "no block at path '" + path + "'");
    b = b->stmts[k].block.get();
  }
  bool ranged = false;
  for (const auto& i : b->indexes) ranged |= i.name == idx && !i.is_alias;
  if (!ranged) throw Error("UnboundIndex", "block '" + path + "' has no ranged index '" + idx + "'");
  SplitCheck c{p, b, {}};
  c.walk(p.root, {}, false);
  if (!c.why.empty()) throw Error("Unsupported", "index '" + idx + "' cannot be split across shards: " + c.why);
}

std::int64_t output_identity(const Program& p, const std::string& name) {
  const Refinement* root_ref = p.root.find_ref(name);
  if (!root_ref) throw Error("MissingBuffer", "no root refinement '" + name + "'");
  Agg agg = root_ref->has_agg ? root_ref->agg : Agg::Assign;
  // Walk the refinement chain of `name` through every block that re-declares
  // it with an aggregation; the last such block in a depth-first, last-child-
  // first traversal decides, matching interp.cpp:620-632.
  std::vector<const Block*> stack = {&p.root};
  while (!stack.empty()) {
    const Block* b = stack.back();
    stack.pop_back();
    const Refinement* r = b->find_ref(name);
    if (b != &p.root && (r == nullptr || !r->has_agg)) continue;
    if (r && r->has_agg) agg = r->agg;
    for (const auto& s : b->stmts)
      if (s.kind == StmtKind::Block) stack.push_back(s.block.get());
  }
  if (is_float(root_ref->dtype)) {
    // f32 extension: the identity's IEEE-754 bit pattern (-inf, +inf, 1.0f, 0.0f)
    switch (agg) {
      case Agg::Max: return static_cast<std::int32_t>(0xFF800000u);
      case Agg::Min: return 0x7F800000;
      case Agg::Mul: return 0x3F800000;
      default: return 0;
    }
  }
  switch (agg) {
    case Agg::Max: return dtype_min(root_ref->dtype);
    case Agg::Min: return dtype_max(root_ref->dtype);
    case Agg::Mul: return 1;
    default: return 0;
  }
}

}  // namespace sb
