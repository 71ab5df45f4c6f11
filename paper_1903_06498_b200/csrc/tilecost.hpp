// tile_cost / autotile evaluated on the device (tilecost.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "ir.hpp"
#include "kernels.hpp"

namespace sb {

// TileCostReport (passes.h:42-50); excluded = "MemCap".
struct TileReport {
  std::int64_t lines_total = 0, useful_ops = 0, tile_elements = 0;
  bool excluded = false;
};

// AutotileResult (passes.h:76-83) without the rewritten block: the caller applies the
// reference's tile_rewrite to `chosen` (tile sizes per ranged index, declaration order).
struct AutotileResult {
  bool found = false;
  std::vector<std::int64_t> chosen;
  TileReport report;
  std::int64_t candidates = 0, excluded = 0;
};

class TileCoster {
 public:
  TileCoster(const Block& b, std::int64_t line, std::int64_t mem_cap, cudaStream_t s);
  TileReport tile_cost(const std::map<std::string, std::int64_t>& shape, bool interleaved);
  AutotileResult autotile(bool power_of_two);
  std::string shape_text(const std::vector<std::int64_t>& tiles) const;

 private:
  struct Dim {
    std::int64_t c = 0, size = 1, stride = 0, clip = 0;
    std::vector<std::int64_t> k;  // coefficient per ranged index
  };
  struct Ref {
    bool untiled = false;
    std::vector<Dim> dims;
  };
  struct Batch {
    std::vector<TileLineItem> items;
    std::vector<long long> values;
    std::vector<std::vector<std::int64_t>> hists;
    long long scratch_words = 0;
  };
  struct Pending {
    std::size_t slot, first;
  };
  void validate(const std::map<std::string, std::int64_t>& shape, std::vector<std::int64_t>* tiles) const;
  std::int64_t useful_ops();
  bool footprint(const std::vector<std::int64_t>& t, bool interleaved, TileReport* rep) const;
  void stage(const std::vector<std::int64_t>& t, bool interleaved, Batch* b) const;
  void flush(Batch* b, std::vector<Pending>* pend, std::vector<TileReport>* out);
  std::vector<TileReport> evaluate(const std::vector<std::vector<std::int64_t>>& cands, bool interleaved);

  const Block& blk_;
  std::int64_t line_, mem_cap_;
  cudaStream_t stream_;
  std::vector<std::string> names_;
  std::vector<std::int64_t> ranges_;
  std::vector<Ref> refs_;
  bool has_alias_ = false, has_special_ = false, useful_known_ = false;
  std::int64_t useful_ = 0;
};

std::map<std::string, std::int64_t> parse_tile_shape_text(const std::string& text);

}  // namespace sb
