// tile_cost and the autotile search on the B200.
//
// Reference: tile_cost (tile.cpp:380-455), autotile (tile.cpp:475-535), with tile_rewrite's
// window arithmetic (tile.cpp:100-235), tile_elements_of (tile.cpp:239-336) and the
// validator's bound_affine (validate.cpp:43-137) for the memory-cap footprint.  The reference
// evaluates one candidate at a time: it rewrites the block, enumerates every tile element of
// every refinement into std::sets (one set per distinct base residue) and every outer point.
// That is what makes the search infeasible at config scale.
//
// Here nothing is rewritten or enumerated on the host beyond per-dimension offset lists:
//   * the per-candidate window arithmetic is closed form (outer offset c + lo + sum k*T*xo,
//     window size hi - lo + size, tile-relative offset rel - lo);
//   * the outer points only matter through their base residue mod L, whose histogram is a
//     cyclic convolution of one arithmetic progression per tiled index (O(L * period));
//   * the distinct-line counts per residue (the expensive part) run on the device, one CTA per
//     (candidate, refinement), all residues at once (kernels/tilecost.cu);
//   * useful_ops is the device count_valid_points (kernels/count.cu), once per search.
// lines_total = sum over refinements and residues of histogram x line count: the same integer
// the reference accumulates point by point.
#include "tilecost.hpp"

#include <algorithm>
#include <limits>
#include <map>
#include <numeric>
#include <sstream>

#include "kernels.hpp"

namespace sb {
namespace {

using Int = __int128;

Int fdiv128(Int a, Int b) {
  Int q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

std::int64_t fdiv(std::int64_t a, std::int64_t b) {
  std::int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

std::int64_t clamp64(Int v) {
  const Int lo = std::numeric_limits<std::int64_t>::min(), hi = std::numeric_limits<std::int64_t>::max();
  return static_cast<std::int64_t>(v < lo ? lo : v > hi ? hi : v);
}

// The validator's interval bound of an affine form over a box under constraints g >= 0
// (validate.cpp:57-137): start from the box extreme, then repeatedly add the one nonnegative
// rational multiple of a constraint that cancels one shared variable and improves the bound
// most (at most 8 rounds, strict improvement, first best kept).
struct Wide {
  std::map<std::string, Int> terms;
  Int constant = 0;
};

Int extreme(const Wide& w, const std::map<std::string, std::pair<std::int64_t, std::int64_t>>& box, bool maximize) {
  Int total = w.constant;
  for (const auto& [name, c] : w.terms) {
    auto it = box.find(name);
    const Int lo = it == box.end() ? 0 : it->second.first, hi = it == box.end() ? 0 : it->second.second;
    total += c * ((c > 0) == maximize ? hi : lo);
  }
  return total;
}

Int bound_side(const Affine& expr, const std::map<std::string, std::pair<std::int64_t, std::int64_t>>& box,
               const std::vector<Affine>& cons, bool maximize) {
  Wide cur;
  cur.constant = expr.constant;
  for (const auto& [n, c] : expr.terms) cur.terms[n] = c;
  Int denom = 1;
  auto score = [&](const Wide& w, Int d) {
    const Int e = extreme(w, box, maximize);
    return maximize ? fdiv128(e, d) : -fdiv128(-e, d);
  };
  Int best = score(cur, denom);
  for (int round = 0; round < 8; round++) {
    Wide pick;
    Int pick_denom = 1;
    bool improved = false;
    for (const Affine& g : cons) {
      for (const auto& [name, gc] : g.terms) {
        auto it = cur.terms.find(name);
        if (it == cur.terms.end() || it->second == 0) continue;
        Int a = -it->second, b = denom * gc;  // b*cur + a*denom*g cancels `name`
        if (b < 0) a = -a, b = -b;
        if (maximize ? a < 0 : a > 0) continue;
        if (a == 0) continue;
        Wide next;
        next.constant = b * cur.constant + a * denom * g.constant;
        for (const auto& [tn, tc] : cur.terms) next.terms[tn] = b * tc;
        for (const auto& [tn, tc] : g.terms) next.terms[tn] += a * denom * tc;
        for (auto t = next.terms.begin(); t != next.terms.end();) t = t->second == 0 ? next.terms.erase(t) : std::next(t);
        const Int nd = b * denom, cand = score(next, nd);
        if (maximize ? cand < best : cand > best) {
          best = cand;
          pick = std::move(next);
          pick_denom = nd;
          improved = true;
        }
      }
    }
    if (!improved) break;
    cur = std::move(pick);
    denom = pick_denom;
  }
  return best;
}

}  // namespace

std::string TileCoster::shape_text(const std::vector<std::int64_t>& tiles) const {
  std::map<std::string, std::int64_t> m;  // TileShape::to_string order (tile.cpp:13-23)
  for (std::size_t x = 0; x < names_.size(); x++) m[names_[x]] = tiles[x];
  std::string s;
  for (const auto& [n, t] : m) s += (s.empty() ? "" : ",") + n + ":" + std::to_string(t);
  return s;
}

TileCoster::TileCoster(const Block& b, std::int64_t line, std::int64_t mem_cap, cudaStream_t s)
    : blk_(b), line_(line), mem_cap_(mem_cap), stream_(s) {
  if (line < 1) throw Error("Invalid", "cache line must be >= 1 element");
  if (line > 4096) throw Error("Unsupported", "cache lines above 4096 elements");
  for (const auto& idx : b.indexes) {
    if (idx.is_alias) {
      has_alias_ = true;
      continue;
    }
    names_.push_back(idx.name);
    ranges_.push_back(idx.range);
  }
  for (const auto& st : b.stmts) has_special_ = has_special_ || st.kind == StmtKind::Special;
  std::map<std::string, std::pair<std::int64_t, std::int64_t>> box;
  for (std::size_t x = 0; x < names_.size(); x++) box[names_[x]] = {0, ranges_[x] - 1};
  for (const auto& ref : b.refs) {
    Ref r;
    r.untiled = ref.tags.count("untiled") != 0;
    for (std::size_t d = 0; d < ref.rank(); d++) {
      Dim dm;
      dm.c = ref.offsets[d].constant;
      dm.size = ref.sizes[d];
      dm.stride = ref.strides[d];
      dm.k.assign(names_.size(), 0);
      for (const auto& [n, c] : ref.offsets[d].terms) {
        auto it = std::find(names_.begin(), names_.end(), n);
        if (it != names_.end()) dm.k[it - names_.begin()] = c;  // alias terms cancel in the window
      }
      const std::int64_t lo = clamp64(bound_side(ref.offsets[d], box, b.constraints, false));
      const std::int64_t hi = clamp64(bound_side(ref.offsets[d], box, b.constraints, true));
      dm.clip = hi + dm.size - lo;  // tile.cpp:402-403
      r.dims.push_back(std::move(dm));
    }
    refs_.push_back(std::move(r));
  }
}

void TileCoster::validate(const std::map<std::string, std::int64_t>& shape, std::vector<std::int64_t>* tiles) const {
  tiles->assign(names_.size(), 0);
  for (std::size_t x = 0; x < names_.size(); x++) {  // tile.cpp:104-115
    auto it = shape.find(names_[x]);
    const std::int64_t t = it == shape.end() ? ranges_[x] : it->second;
    if (t < 1 || t > ranges_[x])
      throw Error("InvalidTile", "tile " + std::to_string(t) + " invalid for index '" + names_[x] + "' of range " +
                                     std::to_string(ranges_[x]));
    (*tiles)[x] = t;
  }
  for (const auto& [n, t] : shape) {  // tile.cpp:124-129
    (void)t;
    if (std::find(names_.begin(), names_.end(), n) == names_.end())
      throw Error("InvalidTile", "no ranged index '" + n + "' to tile");
  }
}

std::int64_t TileCoster::useful_ops() {
  if (has_alias_) throw Error("InvalidTile", "tile_cost requires alias-free blocks");  // tile.cpp:341-344
  if (useful_known_) return useful_;
  std::vector<long long> ranges(ranges_.begin(), ranges_.end());
  std::int64_t total = 1;
  for (auto r : ranges) total *= r;
  if (ranges.empty()) ranges.push_back(1);
  const int nd = static_cast<int>(ranges.size()), nc = static_cast<int>(blk_.constraints.size());
  std::vector<long long> cc(nc), ck(static_cast<std::size_t>(nc) * nd, 0);
  for (int c = 0; c < nc; c++) {
    cc[c] = blk_.constraints[c].constant;
    for (const auto& [n, k] : blk_.constraints[c].terms) {
      auto it = std::find(names_.begin(), names_.end(), n);
      if (it == names_.end()) throw Error("UnboundIndex", "unbound index '" + n + "'");
      ck[static_cast<std::size_t>(c) * nd + (it - names_.begin())] = k;
    }
  }
  useful_ = 0;
  if (total != 0) {
    void* scratch = nullptr;
    if (cudaMalloc(&scratch, count_points_scratch_bytes()) != cudaSuccess) throw Error("CudaError", "cudaMalloc(count)");
    unsigned long long h = 0;
    const cudaError_t e = launch_count_points(nd, ranges.data(), nc, cc.data(), ck.data(), scratch, &h, stream_);
    cudaFree(scratch);
    if (e != cudaSuccess) throw Error("CudaError", std::string("count_points: ") + cudaGetErrorString(e));
    useful_ = static_cast<std::int64_t>(h);
  }
  useful_known_ = true;
  return useful_;
}

// Footprint of one candidate (tile.cpp:384-410); false when it exceeds the memory cap.
bool TileCoster::footprint(const std::vector<std::int64_t>& t, bool interleaved, TileReport* rep) const {
  bool any_tiled = false;
  for (std::size_t x = 0; x < t.size(); x++) any_tiled = any_tiled || t[x] != ranges_[x];
  if (has_special_ && any_tiled) throw Error("NotTileable", "block contains a special spanning tiled indexes");
  rep->tile_elements = 0;
  for (const Ref& r : refs_) {
    if (r.untiled) continue;
    std::int64_t elements = 1;
    for (const Dim& d : r.dims) {
      std::int64_t lo = 0, hi = 0;
      for (std::size_t x = 0; x < t.size(); x++) {
        const std::int64_t o = (ranges_[x] + t[x] - 1) / t[x];
        const std::int64_t kk = interleaved ? d.k[x] * o : d.k[x];
        (kk > 0 ? hi : lo) += kk * (t[x] - 1);
      }
      elements *= std::min(hi - lo + d.size, d.clip);
    }
    rep->tile_elements += elements;
  }
  rep->excluded = rep->tile_elements > mem_cap_;
  return !rep->excluded;
}

// Device work items of one candidate's refinements + the host residue histograms.
void TileCoster::stage(const std::vector<std::int64_t>& t, bool interleaved, Batch* b) const {
  const std::int64_t L = line_;
  const std::size_t nx = t.size();
  std::vector<std::int64_t> outer(nx);
  for (std::size_t x = 0; x < nx; x++) outer[x] = (ranges_[x] + t[x] - 1) / t[x];
  for (const Ref& r : refs_) {
    // tile-relative offsets: rel - lo with rel = sum kk * x over the inner box (tile.cpp:195-203)
    const std::size_t nd = r.dims.size();
    std::vector<std::vector<std::int64_t>> kk(nd, std::vector<std::int64_t>(nx, 0));
    std::vector<std::int64_t> lo(nd, 0);
    for (std::size_t d = 0; d < nd; d++)
      for (std::size_t x = 0; x < nx; x++) {
        kk[d][x] = interleaved ? r.dims[d].k[x] * outer[x] : r.dims[d].k[x];
        if (kk[d][x] < 0) lo[d] += kk[d][x] * (t[x] - 1);
      }
    // element set F as axes (tile_elements_of, tile.cpp:239-336)
    std::vector<int> uses(nx, 0);
    for (std::size_t d = 0; d < nd; d++)
      for (std::size_t x = 0; x < nx; x++) uses[x] += kk[d][x] != 0;
    const bool disjoint = std::all_of(uses.begin(), uses.end(), [](int u) { return u <= 1; });
    std::vector<std::vector<std::int64_t>> axes;
    std::int64_t cst = 0;
    if (disjoint) {
      for (std::size_t d = 0; d < nd; d++) {
        std::vector<std::int64_t> offs{-lo[d]};
        for (std::size_t x = 0; x < nx; x++) {
          if (kk[d][x] == 0) continue;
          std::vector<std::int64_t> next;
          next.reserve(offs.size() * static_cast<std::size_t>(t[x]));
          for (std::int64_t v : offs)
            for (std::int64_t p = 0; p < t[x]; p++) next.push_back(v + kk[d][x] * p);
          std::sort(next.begin(), next.end());
          next.erase(std::unique(next.begin(), next.end()), next.end());
          offs.swap(next);
        }
        std::vector<std::int64_t> wide;
        wide.reserve(offs.size() * static_cast<std::size_t>(r.dims[d].size));
        for (std::int64_t v : offs)
          for (std::int64_t w = 0; w < r.dims[d].size; w++) wide.push_back((v + w) * r.dims[d].stride);
        axes.push_back(std::move(wide));
      }
    } else {
      // The reference enumerates the inner box here (tile.cpp:306-333) with enumerate_points,
      // which evaluates the inner block's tile aliases (xo = T*x, tile.cpp:220-226) against an
      // empty parent scope: UnboundIndex whenever a pushed or overflow constraint uses one.
      for (std::size_t x = 0; x < nx; x++) {
        if (outer[x] == 1) continue;
        bool used = outer[x] * t[x] != ranges_[x];
        for (const Affine& c : blk_.constraints) used = used || c.coeff(names_[x]) != 0;
        if (used) throw Error("UnboundIndex", "unbound index '" + names_[x] + "'");
      }
      for (std::size_t d = 0; d < nd; d++) cst += -lo[d] * r.dims[d].stride;
      for (std::size_t x = 0; x < nx; x++) {
        std::int64_t kf = 0;
        for (std::size_t d = 0; d < nd; d++) kf += kk[d][x] * r.dims[d].stride;
        std::vector<std::int64_t> a;
        for (std::int64_t p = 0; p < t[x]; p++) a.push_back(kf * p);
        axes.push_back(std::move(a));
      }
      for (std::size_t d = 0; d < nd; d++) {
        std::vector<std::int64_t> a;
        for (std::int64_t w = 0; w < r.dims[d].size; w++) a.push_back(w * r.dims[d].stride);
        axes.push_back(std::move(a));
      }
    }
    // dedupe, fold single values into the constant, pick the longest unit-step run as last axis
    std::vector<std::vector<std::int64_t>> kept;
    for (auto& a : axes) {
      std::sort(a.begin(), a.end());
      a.erase(std::unique(a.begin(), a.end()), a.end());
      if (a.size() == 1) cst += a[0];
      else if (!a.empty()) kept.push_back(std::move(a));
    }
    int run = -1;
    for (std::size_t a = 0; a < kept.size(); a++) {
      if (kept[a].back() - kept[a].front() + 1 != static_cast<std::int64_t>(kept[a].size())) continue;
      if (run < 0 || kept[a].size() > kept[run].size()) run = static_cast<int>(a);
    }
    if (run >= 0) std::swap(kept[run], kept.back());
    if (kept.size() > static_cast<std::size_t>(kTileMaxAxes)) throw Error("Unsupported", "more than 32 tile axes");
    TileLineItem it{};
    it.cst = cst;
    it.naxes = static_cast<int>(kept.size());
    it.run = run >= 0 ? 1 : 0;
    it.val_off = static_cast<int>(b->values.size());
    std::int64_t fmin = cst, fmax = cst;
    it.prefixes = 1;
    for (std::size_t a = 0; a < kept.size(); a++) {
      fmin += kept[a].front();
      fmax += kept[a].back();
      it.len[a] = static_cast<int>(kept[a].size());
      const bool is_run = it.run && a + 1 == kept.size();
      if (is_run) {
        b->values.push_back(kept[a].front());
      } else {
        it.prefixes *= static_cast<std::int64_t>(kept[a].size());
        b->values.insert(b->values.end(), kept[a].begin(), kept[a].end());
      }
    }
    it.qbase = fdiv(fmin, L);
    const std::int64_t nq = fdiv(fmax, L) - it.qbase + 1;
    if (nq > (std::int64_t{1} << 28)) throw Error("Unsupported", "tile spans more than 2^28 cache lines");
    it.nq = static_cast<int>(nq);
    it.scratch_off = -1;
    if (nq > tile_lines_smem_q()) {
      it.scratch_off = b->scratch_words;
      b->scratch_words += 2 * nq;
    }
    b->items.push_back(it);
    // residue histogram of the outer bases: B0 + sum_x g_x * xo, xo in [0, outer_x)
    // (rc.base over the outer block's points, tile.cpp:430-452)
    std::int64_t b0 = 0;
    std::vector<std::int64_t> g(nx, 0);
    for (std::size_t d = 0; d < nd; d++) {
      b0 += (r.dims[d].c + lo[d]) * r.dims[d].stride;
      for (std::size_t x = 0; x < nx; x++)
        if (outer[x] > 1) g[x] += r.dims[d].k[x] * (interleaved ? 1 : t[x]) * r.dims[d].stride;
    }
    std::vector<std::int64_t> hist(static_cast<std::size_t>(L), 0), step(static_cast<std::size_t>(L));
    hist[static_cast<std::size_t>(((b0 % L) + L) % L)] = 1;
    for (std::size_t x = 0; x < nx; x++) {
      if (outer[x] == 1) continue;
      const std::int64_t gm = ((g[x] % L) + L) % L;
      const std::int64_t period = gm == 0 ? 1 : L / std::gcd(gm, L);
      // residues of gm * j for j < period, each hit floor(outer / period) (+1 for j < outer % period)
      std::vector<std::pair<std::int64_t, std::int64_t>> h;
      for (std::int64_t j = 0; j < period && j < outer[x]; j++)
        h.emplace_back((gm * j) % L, outer[x] / period + (j < outer[x] % period ? 1 : 0));
      std::fill(step.begin(), step.end(), 0);
      for (std::int64_t q = 0; q < L; q++) {
        if (!hist[q]) continue;
        for (const auto& [res, n] : h) step[(q + res) % L] += hist[q] * n;
      }
      hist.swap(step);
    }
    b->hists.push_back(std::move(hist));
  }
}

void TileCoster::flush(Batch* b, std::vector<Pending>* pend, std::vector<TileReport>* out) {
  if (pend->empty()) return;
  std::vector<long long> counts;
  const cudaError_t e = launch_tile_lines(b->items, b->values, b->scratch_words, static_cast<int>(line_), &counts,
                                          stream_);
  if (e != cudaSuccess) throw Error("CudaError", std::string("tile_lines: ") + cudaGetErrorString(e));
  for (const Pending& p : *pend) {
    TileReport& rep = (*out)[p.slot];
    rep.lines_total = 0;
    for (std::size_t i = p.first; i < p.first + refs_.size(); i++)
      for (std::int64_t q = 0; q < line_; q++)
        rep.lines_total += b->hists[i][q] * counts[i * static_cast<std::size_t>(line_) + q];
  }
  *b = Batch{};
  pend->clear();
}

std::vector<TileReport> TileCoster::evaluate(const std::vector<std::vector<std::int64_t>>& cands, bool interleaved) {
  std::vector<TileReport> out(cands.size());
  Batch b;
  std::vector<Pending> pend;
  bool counted = false;
  for (std::size_t c = 0; c < cands.size(); c++) {
    if (!footprint(cands[c], interleaved, &out[c])) continue;
    if (!counted) {  // the reference counts once per tile_cost call that gets this far
      useful_ops();
      counted = true;
    }
    out[c].useful_ops = useful_;
    pend.push_back({c, b.items.size()});
    stage(cands[c], interleaved, &b);
    if (b.items.size() >= 16384 || b.values.size() >= (std::size_t{1} << 24) || b.scratch_words >= (1ll << 27))
      flush(&b, &pend, &out);
  }
  flush(&b, &pend, &out);
  return out;
}

TileReport TileCoster::tile_cost(const std::map<std::string, std::int64_t>& shape, bool interleaved) {
  std::vector<std::int64_t> t;
  validate(shape, &t);
  return evaluate({t}, interleaved)[0];
}

AutotileResult TileCoster::autotile(bool power_of_two) {
  AutotileResult res;
  useful_ops();  // tile.cpp:491, before any candidate
  std::vector<std::vector<std::int64_t>> cand(names_.size());
  for (std::size_t x = 0; x < names_.size(); x++) {  // tile_candidates (tile.cpp:459-471)
    if (power_of_two)
      for (std::int64_t v = 1; v <= ranges_[x]; v *= 2) cand[x].push_back(v);
    else
      for (std::int64_t v = 1; v <= ranges_[x]; v++)
        if (ranges_[x] % v == 0) cand[x].push_back(v);
  }
  std::vector<std::size_t> pos(names_.size(), 0);
  std::vector<std::vector<std::int64_t>> chunk;
  bool have = false;
  std::int64_t best_lines = 0;
  auto consume = [&] {
    const std::vector<TileReport> reps = evaluate(chunk, false);
    for (std::size_t i = 0; i < chunk.size(); i++) {
      res.candidates++;
      if (reps[i].excluded) {
        res.excluded++;
        continue;
      }
      // Rational{lines, ops} < best (passes.h:37): lines * ops_best < lines_best * ops, int64 as there
      const std::uint64_t lhs = static_cast<std::uint64_t>(reps[i].lines_total) * static_cast<std::uint64_t>(useful_);
      const std::uint64_t rhs = static_cast<std::uint64_t>(best_lines) * static_cast<std::uint64_t>(useful_);
      if (!have || static_cast<std::int64_t>(lhs) < static_cast<std::int64_t>(rhs)) {
        have = true;
        best_lines = reps[i].lines_total;
        res.report = reps[i];
        res.chosen = chunk[i];
      }
    }
    chunk.clear();
  };
  for (;;) {
    std::vector<std::int64_t> t(names_.size());
    for (std::size_t x = 0; x < names_.size(); x++) t[x] = cand[x][pos[x]];
    chunk.push_back(std::move(t));
    if (chunk.size() == 8192) consume();
    std::size_t d = names_.size();
    bool done = true;
    while (d > 0) {
      d--;
      if (++pos[d] < cand[d].size()) {
        done = false;
        break;
      }
      pos[d] = 0;
    }
    if (done || names_.empty()) break;
  }
  consume();
  res.found = have;
  if (!have) res.report = TileReport{};
  return res;
}

std::map<std::string, std::int64_t> parse_tile_shape_text(const std::string& text) {
  std::map<std::string, std::int64_t> m;  // parse_tile_shape (tile.cpp:47-60)
  std::istringstream is(text);
  std::string piece;
  while (std::getline(is, piece, ',')) {
    if (piece.empty()) continue;
    const std::size_t sep = piece.find_first_of(":=");
    if (sep == std::string::npos) throw Error("InvalidTile", "malformed tile entry '" + piece + "'");
    m[piece.substr(0, sep)] = std::stoll(piece.substr(sep + 1));
  }
  return m;
}

}  // namespace sb
