// stripe_b200_binding.hpp — the reference-side C++ binding of the B200 block executor.
//
// Drop-in for `stripe::execute(const Program&, BufferStore*, const ExecOptions&)`
// (proj/include/stripe/interp.h:68, proj/src/interp.cpp:613-615) with the identical
// signature, in namespace stripe::b200 so the reference interpreter can stay linked next
// to it.  Header-only; include it in ONE translation unit of the reference
// build (it needs the reference's headers: stripe/interp.h, stripe/text.h) and link
// paper_1903_06498_b200/libstripe_b200.so.  The program crosses the C ABI
// (include/stripe_b200.h) as its canonical text (print_program, text.h:23-24).
//
// Semantics: the store is updated in place exactly as stripe::execute does (int64
// carriers holding dtype-wrapped values, interp.h:14-17); missing buffers raise
// ExecError("MissingBuffer", ...); observers are rejected (device execution cannot call
// back per access) with ExecError("Unsupported", ...); device errors map to the reference's
// codes (sb_status_name).
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "stripe/interp.h"
#include "stripe/passes.h"
#include "stripe/text.h"
#include "stripe_b200.h"

namespace stripe::b200 {

inline void check(int rc) {
  if (rc == SB_OK) return;
  const std::string msg = sb_last_error();  // "Code: message"
  const auto colon = msg.find(':');
  throw ExecError(colon == std::string::npos ? sb_status_name(rc) : msg.substr(0, colon), msg);
}

// One device context per host thread (and device): concurrent execute calls on disjoint
// stores run on their own streams, staging and device buffers -- "execute is reentrant; a
// single invocation owns its BufferStore exclusively".  Each context is
// destroyed when its thread exits.
inline sb_context* context(int device = 0) {
  struct Holder {
    std::map<int, sb_context*> ctx;
    ~Holder() {
      for (auto& [d, c] : ctx) sb_context_destroy(c);
    }
  };
  thread_local Holder h;
  auto it = h.ctx.find(device);
  if (it != h.ctx.end()) return it->second;
  sb_context* c = nullptr;
  check(sb_context_create(device, &c));
  h.ctx.emplace(device, c);
  return c;
}

// Parsed programs cached by canonical text (plans and device state live with them).
inline sb_program* compiled(const Program& program) {
  static std::mutex mu;
  static std::map<std::string, std::unique_ptr<sb_program, void (*)(sb_program*)>> cache;
  std::string text = print_program(program);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(text);
  if (it == cache.end()) {
    sb_program* p = nullptr;
    check(sb_program_parse(text.c_str(), &p));
    it = cache.emplace(std::move(text), std::unique_ptr<sb_program, void (*)(sb_program*)>(p, sb_program_free)).first;
  }
  return it->second.get();
}

inline void execute(const Program& program, BufferStore* store, const ExecOptions& opts = {}) {
  sb_program* p = compiled(program);
  std::vector<sb_host_buffer> bufs;
  bufs.reserve(store->size());
  for (auto& [name, buf] : *store)
    bufs.push_back({name.c_str(), SB_CARRIER_I64, 0, buf.data.data(), static_cast<std::int64_t>(buf.data.size())});
  sb_exec_options o{};
  o.order = static_cast<std::int32_t>(opts.order);
  o.seed = opts.seed;
  o.observer = opts.observer != nullptr ? 1 : 0;
  check(sb_execute(context(), p, bufs.data(), static_cast<int>(bufs.size()), &o));
}

// ---- the autotile search on the device ------------------------------
// tile_cost / autotile (passes.h:60-89) of the block at dot path `block_path` ("0", "0.1", ...)
// of `program`, with the same reports, choices and exceptions (PassError "InvalidTile" /
// "NotTileable", UnboundIndex); the candidates' line counts run on the GPU.  autotile applies
// the reference's own tile_rewrite to the chosen shape.

inline void check_pass(int rc) {
  if (rc == SB_OK) return;
  const std::string msg = sb_last_error();  // "Code: message"
  const auto colon = msg.find(':');
  const std::string code = colon == std::string::npos ? sb_status_name(rc) : msg.substr(0, colon);
  const std::string text = colon == std::string::npos ? msg : msg.substr(colon + 2);
  if (rc == SB_ERR_PASS) throw PassError(code, text);
  if (rc == SB_ERR_UNBOUND_INDEX) {
    const auto q0 = text.find('\''), q1 = text.rfind('\'');
    throw UnboundIndex(q0 < q1 ? text.substr(q0 + 1, q1 - q0 - 1) : text);
  }
  check(rc);
}

inline const Block& block_at(const Program& program, const std::string& block_path) {
  const Block* b = &program.root;
  std::size_t pos = 0;
  while (pos < block_path.size()) {
    const std::size_t dot = block_path.find('.', pos);
    const std::size_t k = std::stoul(block_path.substr(pos, dot == std::string::npos ? std::string::npos : dot - pos));
    b = &b->stmts.at(k).block();
    pos = dot == std::string::npos ? block_path.size() : dot + 1;
  }
  return *b;
}

inline TileCostReport tile_cost(const Program& program, const std::string& block_path, const TileShape& ts,
                                const CacheModel& cm, std::int64_t mem_cap) {
  sb_tile_report r{};
  check_pass(sb_tile_cost(context(), compiled(program), block_path.c_str(), ts.to_string().c_str(),
                          ts.interleaved ? 1 : 0, cm.line, mem_cap, &r));
  TileCostReport out;
  out.lines_total = r.lines_total;
  out.useful_ops = r.useful_ops;
  out.tile_elements = r.tile_elements;
  if (r.excluded) out.excluded = "MemCap";
  return out;
}

inline AutotileResult autotile(const Program& program, const std::string& block_path, const CacheModel& cm,
                               const AutotileOptions& opts) {
  const Block& block = block_at(program, block_path);
  if (opts.pinned) {  // tile.cpp:477-483
    AutotileResult res;
    res.chosen = opts.pinned;
    res.report = tile_cost(program, block_path, *opts.pinned, cm, opts.mem_cap);
    res.block = tile_rewrite(block, *opts.pinned);
    res.candidates = 1;
    return res;
  }
  char chosen[4096];
  std::size_t len = 0;
  int found = 0;
  sb_tile_report r{};
  std::int64_t cands = 0, excl = 0;
  check_pass(sb_autotile(context(), compiled(program), block_path.c_str(), cm.line, opts.mem_cap,
                         opts.power_of_two ? 1 : 0, chosen, sizeof chosen, &len, &found, &r, &cands, &excl));
  AutotileResult res;
  res.candidates = cands;
  res.excluded = excl;
  if (!found) {  // tile.cpp:523-529
    res.block = block;
    res.diags.push_back({Diagnostic::Severity::Warning, "NoFeasibleTile",
                         "every tile candidate exceeded the memory cap", block.span});
    return res;
  }
  res.chosen = parse_tile_shape(std::string(chosen, len));
  res.report.lines_total = r.lines_total;
  res.report.useful_ops = r.useful_ops;
  res.report.tile_elements = r.tile_elements;
  res.block = tile_rewrite(block, *res.chosen);
  return res;
}

}  // namespace stripe::b200
