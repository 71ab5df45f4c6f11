// oracle/port — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// CPU restatement of the reference interpreter's semantics
// (proj/src/interp.cpp:178-642), templated on a scalar policy so that the
// same control flow serves:
//   * IntPolicy  — int64 temps, wrap-at-store (bit-exact vs stripe::execute;
//                  pinned against oracle/_ref on the whole corpus in tests/),
//   * F32Policy  — the fp32 numeric-mode extension the reference lacks
//                  (SURVEY §8(c)); it is "parity unpinned" by the reference
//                  except through its shared control flow with IntPolicy.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "ir.hpp"

namespace sbport {

struct Store {
  // name -> int64 carriers (integer mode) / float values (f32 mode)
  std::map<std::string, std::vector<std::int64_t>> ints;
  std::map<std::string, std::vector<float>> floats;
};

// Order: 0 lexicographic, 1 reversed (interp.cpp:365-417).
void execute_int(const sb::Program& p, Store* s, int order);
void execute_f32(const sb::Program& p, Store* s, int order);

}  // namespace sbport
