// oracle/dropin/dropin_test.cpp — TEST INFRASTRUCTURE: the drop-in check from the
// reference's side.  Built against the UNMODIFIED reference sources (parser, interpreter,
// tests/support.h random_inputs) and include/stripe_b200_binding.hpp; for each program
// file given it runs stripe::execute (the reference) and stripe::b200::execute (the B200
// executor through the C ABI) on the same random inputs and compares every buffer.
//
//   dropin_test [--seed S] [--threads T] [--autotile LINE:CAP] prog1.stripe [prog2.stripe ...]
// With --threads T (> 1) every program is additionally run by T concurrent host threads,
// each through stripe::b200::execute on its own copy of the store (disjoint stores, the
// reference's reentrancy contract SPEC.md:263), every copy compared with the reference.
// Prints one line per program ("OK <name>" / "DIFF <name> ..." / "ERR <name> code code");
// exit status = number of mismatches.  Error parity: when the reference throws ExecError,
// the binding must throw the same code.  With --autotile, block 0 of every program is also
// searched by stripe::autotile and stripe::b200::autotile (divisor and power-of-two spaces,
// CacheModel{LINE}, mem_cap CAP): chosen shape, report, candidate counts, the rewritten block's
// text and PassError/UnboundIndex codes must match ("OK autotile <name> ...").
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "stripe/interp.h"
#include "stripe/passes.h"
#include "stripe/text.h"
#include "stripe_b200_binding.hpp"
#include "support.h"

static bool same_store(const stripe::BufferStore& a, const stripe::BufferStore& b) {
  if (a.size() != b.size()) return false;
  for (const auto& [name, buf] : b) {
    const auto it = a.find(name);
    if (it == a.end() || it->second.data != buf.data) return false;
  }
  return true;
}

template <typename F>
static std::string run_search(F&& f, std::string* err) {
  try {
    return f();
  } catch (const stripe::PassError& e) {
    *err = e.code;
  } catch (const stripe::UnboundIndex& e) {
    *err = "UnboundIndex";
  }
  return "";
}

static std::string describe(const stripe::AutotileResult& r) {
  std::string s = (r.chosen ? r.chosen->to_string() : "none") + " " + r.report.to_string() + " candidates=" +
                  std::to_string(r.candidates) + " excluded=" + std::to_string(r.excluded);
  stripe::Program wrap;
  wrap.root = r.block;
  return s + "\n" + stripe::print_program(wrap);
}

static int autotile_check(const stripe::Program& prog, const std::string& name, std::int64_t line, std::int64_t cap) {
  if (prog.root.stmts.empty() || !prog.root.stmts[0].is_block()) return 0;
  int bad = 0;
  for (bool p2 : {false, true}) {
    stripe::AutotileOptions opts;
    opts.mem_cap = cap;
    opts.power_of_two = p2;
    const stripe::CacheModel cm{line, cap};
    std::string ref_err, dev_err;
    const std::string ref = run_search([&] { return describe(stripe::autotile(prog.root.stmts[0].block(), cm, opts)); },
                                       &ref_err);
    const std::string dev = run_search([&] { return describe(stripe::b200::autotile(prog, "0", cm, opts)); }, &dev_err);
    const bool same = ref == dev && ref_err == dev_err;
    std::printf("%s autotile %s p2=%d %s%s\n", same ? "OK" : "DIFF", name.c_str(), p2 ? 1 : 0,
                ref_err.empty() ? ref.substr(0, ref.find('\n')).c_str() : ("error " + ref_err).c_str(),
                same ? "" : (" | b200: " + (dev_err.empty() ? dev.substr(0, dev.find('\n')) : "error " + dev_err)).c_str());
    bad += same ? 0 : 1;
  }
  return bad;
}

int main(int argc, char** argv) {
  std::uint64_t seed = 1001;
  int threads = 1;
  int bad = 0;
  std::int64_t at_line = 0, at_cap = 0;
  for (int i = 1; i < argc; i++) {
    std::string arg = argv[i];
    if (arg == "--seed" && i + 1 < argc) {
      seed = std::strtoull(argv[++i], nullptr, 10);
      continue;
    }
    if (arg == "--autotile" && i + 1 < argc) {
      const std::string v = argv[++i];
      at_line = std::stoll(v.substr(0, v.find(':')));
      at_cap = std::stoll(v.substr(v.find(':') + 1));
      continue;
    }
    if (arg == "--threads" && i + 1 < argc) {
      threads = std::atoi(argv[++i]);
      continue;
    }
    std::ifstream f(arg);
    std::stringstream ss;
    ss << f.rdbuf();
    stripe::Program prog;
    try {
      prog = stripe::parse_program(ss.str());
    } catch (const std::exception& e) {
      std::printf("SKIP %s parse: %s\n", arg.c_str(), e.what());
      continue;
    }
    if (at_line > 0) bad += autotile_check(prog, arg, at_line, at_cap);
    stripe::testing::Rng rng(seed);
    stripe::BufferStore ref = stripe::testing::random_inputs(prog, &rng);
    stripe::BufferStore dev = ref;
    std::string ref_err, dev_err;
    try {
      stripe::execute(prog, &ref);
    } catch (const stripe::ExecError& e) {
      ref_err = e.code;
    }
    try {
      stripe::b200::execute(prog, &dev);
    } catch (const stripe::ExecError& e) {
      dev_err = e.code;
    }
    if (!ref_err.empty() || !dev_err.empty()) {
      const bool same = ref_err == dev_err;
      std::printf("%s %s error ref=%s b200=%s\n", same ? "OK" : "ERR", arg.c_str(), ref_err.c_str(),
                  dev_err.c_str());
      bad += same ? 0 : 1;
      continue;
    }
    std::string diff;
    for (const auto& [name, buf] : ref) {
      const auto it = dev.find(name);
      if (it == dev.end() || it->second.data != buf.data) {
        std::size_t first = 0;
        if (it != dev.end())
          while (first < buf.data.size() && buf.data[first] == it->second.data[first]) first++;
        diff += " " + name + "@" + std::to_string(first);
      }
    }
    std::printf("%s %s%s\n", diff.empty() ? "OK" : "DIFF", arg.c_str(), diff.c_str());
    bad += diff.empty() ? 0 : 1;
    if (threads > 1) {
      // T host threads, disjoint stores, all at once through the binding
      stripe::testing::Rng rng2(seed);
      const stripe::BufferStore inputs = stripe::testing::random_inputs(prog, &rng2);
      std::vector<stripe::BufferStore> stores(threads, inputs);
      std::vector<std::string> errs(threads);
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; t++)
        pool.emplace_back([&, t] {
          try {
            for (int rep = 0; rep < 3; rep++) {
              stores[t] = inputs;
              stripe::b200::execute(prog, &stores[t]);
            }
          } catch (const stripe::ExecError& e) {
            errs[t] = e.code;
          }
        });
      for (auto& th : pool) th.join();
      int tbad = 0;
      for (int t = 0; t < threads; t++)
        if (!errs[t].empty() || !same_store(stores[t], ref)) tbad++;
      std::printf("%s %s threads=%d mismatching=%d\n", tbad ? "DIFF" : "OK", arg.c_str(), threads, tbad);
      bad += tbad ? 1 : 0;
    }
  }
  return bad;
}
