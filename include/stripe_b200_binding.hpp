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

}  // namespace stripe::b200
