// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A C-ABI shim over the UNMODIFIED reference interpreter (Stripe Kit,
// /root/reference/proj), compiled from the reference's own sources by
// oracle/Makefile into oracle/_ref/libstripe_ref.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load it.  Nothing here is copied from the reference: every function is a thin
// adapter that calls the reference's public API:
//   parse_program / print_program          proj/include/stripe/text.h:20-25
//   validate_static                         proj/include/stripe/validate.h:15
//   execute / prepare_outputs               proj/include/stripe/interp.h:68-73
//   check_parallel_semantics                proj/include/stripe/conflicts.h:39
//   random_inputs, gen_*                    proj/tests/support.h:55-70, 163-170
//   tile_rewrite / apply_pipeline           proj/include/stripe/passes.h:60, 140
//   load_config                             proj/include/stripe/hwconfig.h:81
// Errors cross the ABI as "Code: message" strings (no exceptions).
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "stripe/conflicts.h"
#include "stripe/hwconfig.h"
#include "stripe/interp.h"
#include "stripe/passes.h"
#include "stripe/text.h"
#include "stripe/validate.h"
#include "support.h"

using namespace stripe;

namespace {

int put(const std::string& s, char* buf, std::size_t cap) {
  if (buf && cap) {
    std::size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return static_cast<int>(s.size());
}

DType dt(int v) { return v == 8 ? DType::i8 : v == 16 ? DType::i16 : DType::i32; }
int dt_bits(DType d) { return dtype_bits(d); }

template <typename F>
int guarded(char* err, std::size_t cap, F&& f) {
  try {
    f();
    put("", err, cap);
    return 0;
  } catch (const ExecError& e) {
    put(e.code + ": " + e.what(), err, cap);
  } catch (const ParseError& e) {
    put(e.code + ": " + e.what(), err, cap);
  } catch (const PassError& e) {
    put(e.code + ": " + e.what(), err, cap);
  } catch (const ConfigError& e) {
    put(e.code + ": " + e.what(), err, cap);
  } catch (const UnboundIndex& e) {
    put(std::string("UnboundIndex: ") + e.what(), err, cap);
  } catch (const std::exception& e) {
    put(std::string("Exception: ") + e.what(), err, cap);
  }
  return 1;
}

}  // namespace

extern "C" {

void* sr_parse(const char* text, char* err, std::size_t cap) {
  Program* out = nullptr;
  guarded(err, cap, [&] { out = new Program(parse_program(text)); });
  return out;
}

void sr_free_program(void* p) { delete static_cast<Program*>(p); }

int sr_print(void* p, char* buf, std::size_t cap) {
  return put(print_program(*static_cast<Program*>(p)), buf, cap);
}

// Returns the number of error diagnostics; renders all diagnostics into buf.
int sr_validate(void* p, char* buf, std::size_t cap) {
  auto diags = validate_static(*static_cast<Program*>(p));
  std::string all;
  int errors = 0;
  for (const auto& d : diags) {
    all += d.render("prog") + "\n";
    if (d.severity == Diagnostic::Severity::Error) errors++;
  }
  put(all, buf, cap);
  return errors;
}

int sr_buffer_count(void* p) {
  return static_cast<int>(static_cast<Program*>(p)->root.refinements.size());
}

// Root refinement i: name, dtype bits, element count (buffer table), dir (0 in, 1 out, 2 inout).
int sr_buffer_info(void* p, int i, char* name, std::size_t cap, int* bits, std::int64_t* elements,
                   int* dir) {
  auto* prog = static_cast<Program*>(p);
  const auto& ref = prog->root.refinements.at(i);
  put(ref.buffer, name, cap);
  *bits = dt_bits(ref.dtype);
  *elements = prog->buffers.at(ref.buffer).elements;
  *dir = ref.dir == Dir::In ? 0 : ref.dir == Dir::Out ? 1 : 2;
  return 0;
}

void* sr_store_new() { return new BufferStore(); }
void sr_store_free(void* s) { delete static_cast<BufferStore*>(s); }
void* sr_store_clone(void* s) { return new BufferStore(*static_cast<BufferStore*>(s)); }

int sr_store_set(void* s, const char* name, int bits, const std::int64_t* data, std::int64_t n) {
  Buffer b;
  b.dtype = dt(bits);
  b.data.assign(data, data + n);
  (*static_cast<BufferStore*>(s))[name] = std::move(b);
  return 0;
}

std::int64_t sr_store_get(void* s, const char* name, std::int64_t* data, std::int64_t cap) {
  auto* store = static_cast<BufferStore*>(s);
  auto it = store->find(name);
  if (it == store->end()) return -1;
  std::int64_t n = static_cast<std::int64_t>(it->second.data.size());
  if (data) std::memcpy(data, it->second.data.data(), sizeof(std::int64_t) * std::min(n, cap));
  return n;
}

// tests/support.h:55-70 random_inputs (splitmix64 Rng seeded with `seed`) incl. prepare_outputs.
int sr_random_inputs(void* p, std::uint64_t seed, void* s) {
  testing::Rng rng(seed);
  *static_cast<BufferStore*>(s) = testing::random_inputs(*static_cast<Program*>(p), &rng);
  return 0;
}

int sr_prepare_outputs(void* p, void* s, char* err, std::size_t cap) {
  return guarded(err, cap, [&] {
    prepare_outputs(*static_cast<Program*>(p), static_cast<BufferStore*>(s));
  });
}

// order: 0 Lex, 1 Reversed, 2 Shuffled (interp.h:58-64)
int sr_execute(void* p, void* s, int order, std::uint64_t seed, char* err, std::size_t cap) {
  return guarded(err, cap, [&] {
    ExecOptions opts;
    opts.order = order == 1 ? IterOrder::Reversed : order == 2 ? IterOrder::Shuffled : IterOrder::Lex;
    opts.seed = seed;
    execute(*static_cast<Program*>(p), static_cast<BufferStore*>(s), opts);
  });
}

// Runs execute() over several independent (program, store) pairs on host threads;
// execute is reentrant.  Used for the multi-core CPU baseline.
int sr_execute_many(void** progs, void** stores, int n, int threads) {
  std::vector<std::thread> pool;
  std::vector<int> status(n, 0);
  int next = 0;
  std::mutex* mu = new std::mutex();
  auto worker = [&] {
    for (;;) {
      int i;
      {
        std::lock_guard<std::mutex> lock(*mu);
        if (next >= n) return;
        i = next++;
      }
      try {
        execute(*static_cast<Program*>(progs[i]), static_cast<BufferStore*>(stores[i]));
      } catch (...) {
        status[i] = 1;
      }
    }
  };
  for (int t = 0; t < threads; t++) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  delete mu;
  int bad = 0;
  for (int v : status) bad += v;
  return bad;
}

// check_parallel_semantics (conflicts.cpp:158-167): returns total conflicts.
std::int64_t sr_conflicts(void* p, void* s, char* buf, std::size_t cap) {
  auto report = check_parallel_semantics(*static_cast<Program*>(p), *static_cast<BufferStore*>(s));
  std::string all;
  for (const auto& c : report.conflicts) all += c.to_string() + "\n";
  put(all, buf, cap);
  return report.total;
}

// Reference generators (tests/support.cpp:50-155) rendered as canonical text.
int sr_gen(const char* kind, std::int64_t a, std::int64_t b, std::int64_t c, std::int64_t d,
           int bits, char* buf, std::size_t cap) {
  std::string k = kind;
  testing::GeneratedProgram g;
  if (k == "matmul") g = testing::gen_matmul(a, b, c, dt(bits));
  else if (k == "conv") g = testing::gen_conv(a, b, c, d, dt(bits));
  else if (k == "maxpool") g = testing::gen_maxpool(a, b, c, dt(bits));
  else return -1;
  return put(print_program(g.program), buf, cap);
}

// gen_random_program / gen_random_text_program with an externally held Rng state.
int sr_gen_random(int text_variant, std::uint64_t* state, char* buf, std::size_t cap) {
  testing::Rng rng(*state);
  std::string out;
  if (text_variant) {
    out = print_program(testing::gen_random_text_program(&rng));
  } else {
    out = print_program(testing::gen_random_program(&rng).program);
  }
  *state = rng.state;
  return put(out, buf, cap);
}

// The brute-force oracle of a generated program (support.h:101-152) applied to a store.
int sr_gen_oracle(const char* kind, std::int64_t a, std::int64_t b, std::int64_t c, std::int64_t d,
                  int bits, void* s) {
  std::string k = kind;
  testing::GeneratedProgram g;
  if (k == "matmul") g = testing::gen_matmul(a, b, c, dt(bits));
  else if (k == "conv") g = testing::gen_conv(a, b, c, d, dt(bits));
  else if (k == "maxpool") g = testing::gen_maxpool(a, b, c, dt(bits));
  else return -1;
  g.oracle(static_cast<BufferStore*>(s));
  return 0;
}

// tile_rewrite (tile.cpp:100-235) of the block at `path`, e.g. "0"; tiles "m:32,n:32".
int sr_tile_rewrite(void* p, const char* path, const char* tiles, char* buf, std::size_t cap,
                    char* err, std::size_t ecap) {
  std::string out;
  int rc = guarded(err, ecap, [&] {
    Program prog = *static_cast<Program*>(p);
    Block* blk = block_at_path(&prog.root, path);
    if (!blk) throw std::runtime_error("bad block path");
    *blk = tile_rewrite(*blk, parse_tile_shape(tiles));
    rebind_buffers(&prog);
    out = print_program(prog);
  });
  if (rc) return -1;
  return put(out, buf, cap);
}

// useful_ops of tile_cost (tile.cpp:404-411) = count_valid_points(block) (tile.cpp:338-370).
int sr_useful_ops(void* p, const char* path, std::int64_t* out, char* err, std::size_t ecap) {
  return guarded(err, ecap, [&] {
    const Program& prog = *static_cast<Program*>(p);
    const Block* blk = block_at_path(&prog.root, path);
    if (!blk) throw std::runtime_error("bad block path");
    TileShape ts;
    *out = tile_cost(*blk, ts, CacheModel{8, std::int64_t{1} << 40}, std::int64_t{1} << 40).useful_ops;
  });
}

// tile_cost (tile.cpp:380-455) of the block at `path`; hint < 0: no useful_ops hint.
// out = {lines_total, useful_ops, tile_elements, excluded}.
int sr_tile_cost(void* p, const char* path, const char* tiles, int interleaved, std::int64_t line,
                 std::int64_t mem_cap, std::int64_t hint, std::int64_t* out, char* err, std::size_t ecap) {
  return guarded(err, ecap, [&] {
    const Program& prog = *static_cast<Program*>(p);
    const Block* blk = block_at_path(&prog.root, path);
    if (!blk) throw std::runtime_error("bad block path");
    TileShape ts = parse_tile_shape(tiles);
    ts.interleaved = interleaved != 0;
    CacheModel cm{line, std::int64_t{1} << 40};
    TileCostReport r = hint < 0 ? tile_cost(*blk, ts, cm, mem_cap) : tile_cost(*blk, ts, cm, mem_cap, hint);
    out[0] = r.lines_total;
    out[1] = r.useful_ops;
    out[2] = r.tile_elements;
    out[3] = r.excluded ? 1 : 0;
  });
}

// autotile (tile.cpp:475-535); chosen gets TileShape::to_string() ("" when none feasible).
// out = {lines_total, useful_ops, tile_elements, candidates, excluded, found}.
int sr_autotile(void* p, const char* path, std::int64_t line, std::int64_t mem_cap, int power_of_two,
                char* chosen, std::size_t cap, std::int64_t* out, char* err, std::size_t ecap) {
  return guarded(err, ecap, [&] {
    const Program& prog = *static_cast<Program*>(p);
    const Block* blk = block_at_path(&prog.root, path);
    if (!blk) throw std::runtime_error("bad block path");
    AutotileOptions opts;
    opts.mem_cap = mem_cap;
    opts.power_of_two = power_of_two != 0;
    AutotileResult r = autotile(*blk, CacheModel{line, std::int64_t{1} << 40}, opts);
    put(r.chosen ? r.chosen->to_string() : std::string(), chosen, cap);
    out[0] = r.report.lines_total;
    out[1] = r.report.useful_ops;
    out[2] = r.report.tile_elements;
    out[3] = r.candidates;
    out[4] = r.excluded;
    out[5] = r.chosen ? 1 : 0;
  });
}

// apply_pipeline (passes.cpp:905-1023) with a .hwcfg text.
int sr_pipeline(void* p, const char* hwcfg, char* buf, std::size_t cap, char* err,
                std::size_t ecap) {
  std::string out;
  int rc = guarded(err, ecap, [&] {
    auto [hw, pipeline] = load_config(hwcfg);
    PipelineResult res = apply_pipeline(*static_cast<Program*>(p), pipeline, hw);
    if (!res.ok) {
      std::string msg;
      for (const auto& dg : res.diags) msg += dg.render("pipeline") + "; ";
      throw std::runtime_error("PassFailed " + msg);
    }
    out = print_program(res.program);
  });
  if (rc) return -1;
  return put(out, buf, cap);
}

}  // extern "C"
