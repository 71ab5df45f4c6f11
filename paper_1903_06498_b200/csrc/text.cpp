// Parser for the .stripe text format (grammar: proj/README.md "The text format").
// This follows the reference parser (proj/src/text.cpp:135-451) production by production
// and keeps its diagnostic strings and error codes (SyntaxError for malformed input,
// ScopeError for undeclared indexes/buffers) so error parity holds at the C ABI, which
// carries programs as canonical text.  It is the drop-in surface's parser restated, not
// part of the hot path: the reference's own parse_program stays the front end of the
// binding (include/stripe_b200_binding.hpp prints the Program and this re-reads it).
#include <cctype>
#include <cstdlib>

#include "ir.hpp"

namespace sb {
namespace {

enum class T { Ident, Int, Punct, Ge, End };

struct Tok {
  T kind = T::End;
  std::string text;  // identifier / punctuation character
  std::int64_t value = 0;
  int line = 1, col = 1;
};

class Scanner {
 public:
  explicit Scanner(const std::string& s) : s_(s) { cur_ = scan(pos_, line_, col_); }

  const Tok& peek() const { return cur_; }
  // Second token of lookahead, computed on demand from a saved cursor.
  Tok peek2() const {
    std::size_t p = pos_;
    int l = line_, c = col_;
    if (cur_.kind == T::End) return cur_;
    return scan(p, l, c);
  }
  Tok next() {
    Tok t = cur_;
    if (cur_.kind != T::End) cur_ = scan(pos_, line_, col_);
    return t;
  }
  bool is_punct(char c) const { return cur_.kind == T::Punct && cur_.text[0] == c; }
  bool is_word(const char* w) const { return cur_.kind == T::Ident && cur_.text == w; }

  [[noreturn]] void fail(const std::string& msg, const char* code = "SyntaxError") const {
    throw Error(code, msg + " at line " + std::to_string(cur_.line) + ":" +
                          std::to_string(cur_.col));
  }

 private:
  Tok scan(std::size_t& p, int& line, int& col) const {
    auto adv = [&] {
      if (s_[p] == '\n') {
        line++;
        col = 1;
      } else {
        col++;
      }
      p++;
    };
    for (;;) {
      if (p >= s_.size()) break;
      char c = s_[p];
      if (c == '/' && p + 1 < s_.size() && s_[p + 1] == '/') {
        while (p < s_.size() && s_[p] != '\n') adv();
      } else if (std::isspace(static_cast<unsigned char>(c))) {
        adv();
      } else {
        break;
      }
    }
    Tok t;
    t.line = line;
    t.col = col;
    if (p >= s_.size()) return t;
    char c = s_[p];
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      t.kind = T::Ident;
      while (p < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[p])) || s_[p] == '_')) {
        t.text += s_[p];
        adv();
      }
      return t;
    }
    if (std::isdigit(static_cast<unsigned char>(c))) {
      t.kind = T::Int;
      while (p < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p]))) {
        t.text += s_[p];
        adv();
      }
      errno = 0;
      t.value = std::strtoll(t.text.c_str(), nullptr, 10);
      if (errno == ERANGE)
        throw Error("SyntaxError", "integer literal out of range at line " + std::to_string(t.line));
      return t;
    }
    if (c == '>' && p + 1 < s_.size() && s_[p + 1] == '=') {
      t.kind = T::Ge;
      t.text = ">=";
      adv();
      adv();
      return t;
    }
    static const std::string punct = "[](){}:,=*+-$#@";
    if (punct.find(c) == std::string::npos)
      throw Error("SyntaxError", std::string("unexpected character '") + c + "' at line " +
                                     std::to_string(line) + ":" + std::to_string(col));
    t.kind = T::Punct;
    t.text = std::string(1, c);
    adv();
    return t;
  }

  const std::string& s_;
  std::size_t pos_ = 0;
  int line_ = 1, col_ = 1;
  Tok cur_;
};

class Parser {
 public:
  explicit Parser(const std::string& text) : sc_(text) {}

  Program run() {
    if (!sc_.is_word("block")) sc_.fail("expected 'block'");
    Program p;
    p.root = block();
    if (sc_.peek().kind != T::End) sc_.fail("trailing input after program");
    if (!p.root.has_annotation) {
      p.root.has_annotation = true;
      p.root.annotation = p.root.range_product();
    }
    rebind_buffers(&p);
    return p;
  }

 private:
  void punct(char c, const char* what) {
    if (!sc_.is_punct(c)) sc_.fail(std::string("expected ") + what);
    sc_.next();
  }
  bool accept(char c) {
    if (!sc_.is_punct(c)) return false;
    sc_.next();
    return true;
  }
  std::string ident(const char* what) {
    if (sc_.peek().kind != T::Ident) sc_.fail(std::string("expected ") + what);
    return sc_.next().text;
  }
  std::int64_t integer() {
    bool neg = accept('-');
    if (sc_.peek().kind != T::Int) sc_.fail("expected integer");
    std::int64_t v = sc_.next().value;
    return neg ? -v : v;
  }

  Affine affine() {
    Affine out;
    bool first = true;
    for (;;) {
      std::int64_t sign = 1;
      if (accept('-')) sign = -1;
      else if (accept('+')) sign = 1;
      else if (!first) break;
      const Tok& t = sc_.peek();
      if (t.kind == T::Int) {
        std::int64_t v = sc_.next().value;
        if (accept('*')) out.add(Affine::term(ident("index name"), sign * v));
        else out.constant += sign * v;
      } else if (t.kind == T::Ident) {
        std::string name = sc_.next().text;
        std::int64_t c = sign;
        if (accept('*')) {
          if (sc_.peek().kind != T::Int) sc_.fail("expected coefficient");
          c = sign * sc_.next().value;
        }
        out.add(Affine::term(name, c));
      } else {
        sc_.fail("expected affine term");
      }
      first = false;
    }
    return out;
  }

  void scope_check(const Affine& a, const std::set<std::string>* scope) {
    for (const auto& [name, c] : a.terms) {
      (void)c;
      if (!scope || !scope->count(name))
        sc_.fail("index '" + name + "' is not in scope", "ScopeError");
    }
  }

  std::vector<std::int64_t> int_list() {
    std::vector<std::int64_t> v;
    punct('(', "'('");
    if (!accept(')')) {
      v.push_back(integer());
      while (accept(',')) v.push_back(integer());
      punct(')', "')'");
    }
    return v;
  }

  Refinement refinement(Dir dir, const Block& owner) {
    Refinement r;
    r.dir = dir;
    r.name = ident("buffer name");
    punct('[', "'['");
    if (!accept(']')) {
      r.offsets.push_back(affine());
      while (accept(',')) r.offsets.push_back(affine());
      punct(']', "']'");
    }
    for (const auto& o : r.offsets) scope_check(o, &scopes_.back());
    if (accept(':')) {
      std::string a = ident("aggregation op");
      static const char* names[] = {"assign", "add", "max", "min", "mul"};
      int found = -1;
      for (int i = 0; i < 5; i++)
        if (a == names[i]) found = i;
      if (found < 0) sc_.fail("unknown aggregation op '" + a + "'");
      if (dir == Dir::In) sc_.fail("aggregation op not allowed on an in refinement");
      r.has_agg = true;
      r.agg = static_cast<Agg>(found);
    }
    std::string dt = ident("dtype");
    if (dt == "i8") r.dtype = DType::I8;
    else if (dt == "i16") r.dtype = DType::I16;
    else if (dt == "i32") r.dtype = DType::I32;
    else if (dt == "f32") r.dtype = DType::F32;  // fp32 extension (not accepted by the reference)
    else sc_.fail("unknown dtype '" + dt + "'");
    r.sizes = int_list();
    punct(':', "':'");
    r.strides = int_list();
    if (r.sizes.size() != r.offsets.size() || r.strides.size() != r.offsets.size())
      sc_.fail("refinement rank mismatch between offsets, sizes and strides");
    if (accept('@')) {
      r.has_location = true;
      r.location.unit = ident("memory unit name");
      punct('[', "'['");
      r.location.bank = affine();
      scope_check(r.location.bank, &scopes_.back());
      punct(']', "']'");
      punct(':', "':'");
      r.location.address = integer();
    }
    while (accept('#')) r.tags.insert(ident("tag name"));
    if (owner.find_ref(r.name)) sc_.fail("duplicate refinement '" + r.name + "'");
    return r;
  }

  void need_ref(const Block& b, const std::string& name, const char* what) {
    if (!b.find_ref(name))
      throw Error("ScopeError", std::string(what) + " names undeclared buffer '" + name + "'");
  }

  Statement statement(const Block& owner) {
    Statement s;
    if (sc_.peek().kind == T::Int) {
      Tok t2 = sc_.peek2();
      if (t2.kind == T::Punct && t2.text == ":") {
        sc_.next();
        sc_.next();
      }
    }
    const Tok& t = sc_.peek();
    if (t.kind == T::Ident && t.text == "block") {
      Tok t2 = sc_.peek2();
      if (t2.kind == T::Punct && t2.text == "[") {
        s.kind = StmtKind::Block;
        s.block = std::make_unique<Block>(block());
        return s;
      }
    }
    if (t.kind == T::Ident && t.text == "special" && sc_.peek2().kind == T::Ident) {
      sc_.next();
      s.kind = StmtKind::Special;
      s.op = ident("special name");
      punct('(', "'('");
      s.refs.push_back(ident("refinement name"));
      while (accept(',')) s.refs.push_back(ident("refinement name"));
      punct(')', "')'");
      for (const auto& r : s.refs) need_ref(owner, r, "special");
      return s;
    }
    if (accept('$')) {
      s.into = "$" + ident("temp name");
      punct('=', "'='");
      std::string op = ident("intrinsic name");
      punct('(', "'('");
      if (op == "load") {
        s.kind = StmtKind::Load;
        s.from = ident("refinement name");
        punct(')', "')'");
        need_ref(owner, s.from, "load");
        return s;
      }
      s.kind = StmtKind::Intrinsic;
      s.op = op;
      if (!accept(')')) {
        do {
          Operand o;
          if (accept('$')) {
            o.temp = "$" + ident("temp name");
          } else {
            o.is_imm = true;
            o.imm = integer();
          }
          s.args.push_back(o);
        } while (accept(','));
        punct(')', "')'");
      }
      return s;
    }
    if (t.kind == T::Ident) {
      Tok t2 = sc_.peek2();
      if (t2.kind == T::Punct && t2.text == "=") {
        s.kind = StmtKind::Store;
        s.into = sc_.next().text;
        sc_.next();
        if (ident("'store'") != "store") sc_.fail("expected 'store'");
        punct('(', "'('");
        punct('$', "'$'");
        s.from = "$" + ident("temp name");
        punct(')', "')'");
        need_ref(owner, s.into, "store");
        return s;
      }
    }
    sc_.fail("expected statement");
  }

  Block block() {
    Block b;
    if (ident("'block'") != "block") sc_.fail("expected 'block'");
    punct('[', "'['");
    bool saw_alias = false;
    if (!accept(']')) {
      do {
        Index idx;
        idx.name = ident("index name");
        if (b.find_index(idx.name)) sc_.fail("duplicate index '" + idx.name + "'");
        if (accept(':')) {
          if (saw_alias) sc_.fail("ranged index after alias index");
          idx.range = integer();
          if (idx.range < 1) sc_.fail("index range must be >= 1");
        } else {
          punct('=', "':' or '='");
          idx.is_alias = true;
          idx.alias = affine();
          scope_check(idx.alias, scopes_.empty() ? nullptr : &scopes_.back());
          saw_alias = true;
        }
        b.indexes.push_back(std::move(idx));
      } while (accept(','));
      punct(']', "']'");
    }
    if (accept(':')) {
      b.has_annotation = true;
      b.annotation = integer();
    }
    scopes_.emplace_back();
    for (const auto& idx : b.indexes) scopes_.back().insert(idx.name);
    punct('(', "'('");
    bool saw_body = false;
    while (!accept(')')) {
      if (sc_.is_punct('#')) {
        if (saw_body) sc_.fail("block tags must precede constraints and refinements");
        sc_.next();
        b.tags.insert(ident("tag name"));
        continue;
      }
      saw_body = true;
      if (sc_.is_word("in") || sc_.is_word("out") || sc_.is_word("inout")) {
        std::string w = sc_.next().text;
        Dir d = w == "in" ? Dir::In : w == "out" ? Dir::Out : Dir::InOut;
        b.refs.push_back(refinement(d, b));
        continue;
      }
      Affine c = affine();
      scope_check(c, &scopes_.back());
      if (sc_.peek().kind != T::Ge) sc_.fail("expected '>='");
      sc_.next();
      if (sc_.peek().kind != T::Int) sc_.fail("expected '0'");
      if (sc_.next().value != 0) sc_.fail("constraint right-hand side must be 0");
      b.constraints.push_back(std::move(c));
    }
    punct('{', "'{'");
    while (!accept('}')) b.stmts.push_back(statement(b));
    scopes_.pop_back();
    return b;
  }

  Scanner sc_;
  std::vector<std::set<std::string>> scopes_;
};

}  // namespace

Program parse_program(const std::string& text) { return Parser(text).run(); }

}  // namespace sb
