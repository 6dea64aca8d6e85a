// rrgpu.hpp -- C++17 adapter over the C ABI (include/rrgpu.h).
//
// Mirrors the reference's operator API (rrflow 0.1.0, proj/include/rrflow) so a
// caller such as proj/tools/rrflow.cpp:104 switches by swapping one include
// and namespace. Same defaults, slot/stream semantics, side
// effects and exception classes:
//   RRG_EINVAL -> std::invalid_argument   RRG_ENOMEM -> rrgpu::BatchOutOfMemory
//   RRG_ECUDA  -> std::runtime_error
// Header-only; link with librrgpu.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../rrgpu.h"

namespace rrgpu {

enum class DiffusionModel { IC, LT };  // graph.hpp:19

// sampling.hpp:148-154
struct BatchOutOfMemory : std::runtime_error {
  explicit BatchOutOfMemory(uint64_t generated, const std::string& why)
      : std::runtime_error("out of memory after generating " + std::to_string(generated) +
                           " RRR sets: " + why),
        sets_generated(generated) {}
  uint64_t sets_generated;
};

inline void check(rrg_status st, uint64_t generated = 0) {
  if (st == RRG_OK) return;
  const std::string msg = rrg_last_error();
  if (st == RRG_EINVAL) throw std::invalid_argument(msg);
  if (st == RRG_ENOMEM) throw BatchOutOfMemory(generated, msg);
  throw std::runtime_error(msg);
}

inline rrg_model to_c(DiffusionModel m) { return m == DiffusionModel::IC ? RRG_IC : RRG_LT; }

// Device-resident transpose of rrflow::Graph (graph.hpp:34-59). Build it from the
// reference graph's reverse arrays verbatim: Graph g(rg.num_vertices,
// rg.reverse_offsets, rg.reverse_sources, rg.reverse_weights).
class Graph {
 public:
  Graph(uint32_t n, const std::vector<uint64_t>& reverse_offsets,
        const std::vector<uint32_t>& reverse_sources, const std::vector<float>& reverse_weights)
      : Graph(n, reverse_offsets, reverse_sources, reverse_weights, -1) {}
  // With the diffusion model the graph will be sampled under, the upload and
  // the model's device layouts overlap (rrg_graph_create_for); same results.
  Graph(uint32_t n, const std::vector<uint64_t>& reverse_offsets,
        const std::vector<uint32_t>& reverse_sources, const std::vector<float>& reverse_weights,
        DiffusionModel model)
      : Graph(n, reverse_offsets, reverse_sources, reverse_weights, static_cast<int>(to_c(model))) {}

 private:
  Graph(uint32_t n, const std::vector<uint64_t>& reverse_offsets,
        const std::vector<uint32_t>& reverse_sources, const std::vector<float>& reverse_weights,
        int model_hint) {
    if (reverse_offsets.size() != static_cast<size_t>(n) + 1)
      throw std::invalid_argument("reverse_offsets must hold n + 1 entries");
    if (reverse_sources.size() != reverse_weights.size())
      throw std::invalid_argument("reverse_sources and reverse_weights differ in length");
    rrg_graph* h = nullptr;
    check(rrg_graph_create_for(n, reverse_sources.size(), reverse_offsets.data(),
                               reverse_sources.data(), reverse_weights.data(), model_hint, &h));
    h_.reset(h);
  }

 public:
  uint32_t num_vertices() const { return rrg_graph_num_vertices(h_.get()); }
  uint64_t num_edges() const { return rrg_graph_num_edges(h_.get()); }
  rrg_graph* handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(rrg_graph* g) const { rrg_graph_destroy(g); }
  };
  std::unique_ptr<rrg_graph, Del> h_;
};

// RRRStore + the fused Counter of generate_batch_fused (rrr_store.hpp, counter.hpp).
class RRRStore {
 public:
  explicit RRRStore(const Graph& g) : n_(g.num_vertices()) {
    rrg_store* h = nullptr;
    check(rrg_store_create(g.handle(), &h));
    h_.reset(h);
  }
  uint64_t size() const {
    uint64_t s = 0;
    check(rrg_store_info(h_.get(), &s, nullptr, nullptr));
    return s;
  }
  uint64_t total_member_count() const {
    uint64_t m = 0;
    check(rrg_store_info(h_.get(), nullptr, &m, nullptr));
    return m;
  }
  uint32_t max_set_size() const {
    uint32_t x = 0;
    check(rrg_store_info(h_.get(), nullptr, nullptr, &x));
    return x;
  }
  // Members of set `idx` in visit order (root first).
  std::vector<uint32_t> set(uint64_t idx) const {
    uint64_t off[2];
    check(rrg_store_export(h_.get(), idx, 1, off, nullptr));
    std::vector<uint32_t> out(off[1]);
    check(rrg_store_export(h_.get(), idx, 1, off, out.data()));
    return out;
  }
  // rrr_store.hpp:84: sets the last select_seeds left uncovered (appends revive all)
  uint64_t live_count() const {
    uint64_t x = 0;
    check(rrg_store_live_count(h_.get(), &x));
    return x;
  }
  // rrr_store.hpp:62
  bool is_live(uint64_t idx) const {
    uint8_t f = 0;
    check(rrg_store_live_flags(h_.get(), idx, 1, &f));
    return f != 0;
  }
  // Counter::get for every vertex (counter.hpp:29)
  std::vector<uint64_t> counter() const {
    std::vector<uint64_t> out(n_);
    check(rrg_store_counter(h_.get(), out.data()));
    return out;
  }
  rrg_store* handle() const { return h_.get(); }

 private:
  struct Del {
    void operator()(rrg_store* s) const { rrg_store_destroy(s); }
  };
  uint32_t n_;
  std::unique_ptr<rrg_store, Del> h_;
};

// sampling.hpp:159-199. `fused` plays the role of the Counter* argument.
inline void generate_batch(const Graph& g, DiffusionModel model, uint64_t run_seed,
                           uint64_t count, RRRStore& store, bool fused = true,
                           uint32_t density_divisor = 64) {
  uint64_t made = 0;
  check(rrg_generate_batch(g.handle(), to_c(model), run_seed, count, store.handle(),
                           fused ? 1 : 0, density_divisor, &made),
        made);
}

// work_pool.hpp: the device's persistent grids replace the fork-join pool; a
// WorkPool keeps the reference's signatures and its worker-count contract.
class WorkPool {
 public:
  explicit WorkPool(unsigned workers = 1) : workers_(workers) {
    if (workers < 1) throw std::invalid_argument("WorkPool: workers must be >= 1");
  }
  unsigned workers() const { return workers_; }

 private:
  unsigned workers_;
};

// counter.hpp:15-62: a caller-owned per-vertex tally (host values).
class Counter {
 public:
  explicit Counter(uint32_t n) : c_(n, 0) {}
  uint32_t size() const { return static_cast<uint32_t>(c_.size()); }
  uint64_t get(uint32_t v) const { return c_.at(v); }
  void add(uint32_t v, uint64_t d = 1) { c_.at(v) += d; }
  void sub(uint32_t v, uint64_t d = 1) { c_.at(v) -= d; }
  void zero() { std::fill(c_.begin(), c_.end(), 0); }
  Counter clone() const { return *this; }
  const std::vector<uint64_t>& values() const { return c_; }
  std::vector<uint64_t>& values() { return c_; }

 private:
  std::vector<uint64_t> c_;
};

// sampling.hpp:159-199 with the reference's signature: counter == nullptr samples
// unfused; otherwise every member of the new sets is added to *counter (the
// store's fused tally grows by exactly those counts on the device).
inline void generate_batch(const Graph& g, DiffusionModel model, uint64_t run_seed,
                           uint64_t count, WorkPool& /*pool*/, RRRStore& store, Counter* counter,
                           uint32_t density_divisor = 64) {
  if (counter && counter->size() != g.num_vertices())
    throw std::invalid_argument("generate_batch: counter size != vertex count");
  std::vector<uint64_t> before;
  if (counter) before = store.counter();
  uint64_t made = 0;
  const rrg_status st = rrg_generate_batch(g.handle(), to_c(model), run_seed, count,
                                           store.handle(), counter ? 1 : 0, density_divisor,
                                           &made);
  if (counter) {  // also on BatchOutOfMemory: the sets that made it in are counted
    const std::vector<uint64_t> after = store.counter();
    for (size_t v = 0; v < after.size(); ++v) counter->values()[v] += after[v] - before[v];
  }
  check(st, made);
}

// sampling.hpp:201-206
inline void generate_batch_fused(const Graph& g, DiffusionModel model, uint64_t run_seed,
                                 uint64_t count, Counter& counter, WorkPool& pool,
                                 RRRStore& store, uint32_t density_divisor = 64) {
  generate_batch(g, model, run_seed, count, pool, store, &counter, density_divisor);
}

// selection.hpp:45-49. touches (the reference's CPU touch tally) has no device
// counterpart and stays 0; the per-round counter snapshots are exact.
struct SelectionStats {
  uint64_t touches = 0;
  bool capture_round_counters = false;
  std::vector<std::vector<uint64_t>> round_counters;
};

// selection.hpp:19-22
struct SeedSet {
  std::vector<uint32_t> seeds;
  std::vector<uint64_t> marginal_counts;
};

// selection.hpp:209-243 (prebuilt = the store's fused counter).
inline SeedSet select_seeds(RRRStore& store, uint32_t n, uint32_t k,
                            double adaptive_threshold = 0.25, bool prebuilt = true) {
  if (k < 1) throw std::invalid_argument("select_seeds: k must be >= 1");
  if (k > n) throw std::invalid_argument("select_seeds: k exceeds vertex count");
  SeedSet out;
  out.seeds.resize(k);
  out.marginal_counts.resize(k);
  check(rrg_select_seeds(store.handle(), k, adaptive_threshold, prebuilt ? 1 : 0,
                         out.seeds.data(), out.marginal_counts.data(), nullptr, nullptr,
                         nullptr));
  return out;
}

// selection.hpp:209-243 with the reference's signature: prebuilt == nullptr
// recounts the store (build_counter, :79-95), else *prebuilt is the starting tally.
inline SeedSet select_seeds(RRRStore& store, uint32_t n, uint32_t k, WorkPool& /*pool*/,
                            double adaptive_threshold = 0.25, const Counter* prebuilt = nullptr,
                            SelectionStats* stats = nullptr) {
  if (k < 1) throw std::invalid_argument("select_seeds: k must be >= 1");
  if (k > n) throw std::invalid_argument("select_seeds: k exceeds vertex count");
  if (prebuilt) {
    if (prebuilt->size() != n) throw std::invalid_argument("select_seeds: prebuilt size != n");
    check(rrg_store_set_counter(store.handle(), prebuilt->values().data()));
  }
  SeedSet out;
  out.seeds.resize(k);
  out.marginal_counts.resize(k);
  const bool capture = stats && stats->capture_round_counters;
  std::vector<uint64_t> snaps(capture ? static_cast<size_t>(k) * n : 0);
  uint32_t rounds = 0;
  check(rrg_select_seeds(store.handle(), k, adaptive_threshold, prebuilt ? 1 : 0,
                         out.seeds.data(), out.marginal_counts.data(),
                         capture ? snaps.data() : nullptr, &rounds, nullptr));
  if (capture) {
    for (uint32_t r = 0; r < rounds; ++r)
      stats->round_counters.emplace_back(snaps.begin() + static_cast<size_t>(r) * n,
                                         snaps.begin() + static_cast<size_t>(r + 1) * n);
  }
  return out;
}

// selection.hpp:340-358
inline double fraction_covered(RRRStore& store, const std::vector<uint32_t>& seeds) {
  double f = 0.0;
  check(rrg_fraction_covered(store.handle(), seeds.data(), static_cast<uint32_t>(seeds.size()),
                             &f));
  return f;
}

// imm.hpp:15-24
enum class Strategy { fused, baseline };
inline Strategy parse_strategy(const std::string& s) {
  if (s == "fused") return Strategy::fused;
  if (s == "baseline") return Strategy::baseline;
  throw std::invalid_argument("unknown strategy: " + s);
}

// imm.hpp:27-54
struct ImmConfig {
  uint32_t k = 50;
  double epsilon = 0.5;
  DiffusionModel model = DiffusionModel::IC;
  unsigned workers = 1;
  uint64_t rng_seed = 1;
  double ell = 1.0;
  double adaptive_threshold = 0.25;
  Strategy strategy = Strategy::fused;
};

struct ImmTimings {
  double generate_rrrsets = 0.0;
  double find_most_influential = 0.0;
  double total = 0.0;
};

struct ImmResult {
  SeedSet seeds;
  uint64_t theta = 0;
  uint64_t theta_prime = 0;
  double lower_bound = 0.0;
  ImmTimings timings;
  uint64_t sets_generated = 0;
  double mean_set_size = 0.0;
  uint32_t max_set_size = 0;
  double mean_coverage_fraction = 0.0;
};

inline rrg_imm_config to_c(const ImmConfig& cfg) {
  rrg_imm_config c;
  rrg_imm_config_default(&c);
  c.k = cfg.k;
  c.epsilon = cfg.epsilon;
  c.model = to_c(cfg.model);
  c.workers = cfg.workers;
  c.rng_seed = cfg.rng_seed;
  c.ell = cfg.ell;
  c.adaptive_threshold = cfg.adaptive_threshold;
  c.strategy = cfg.strategy == Strategy::fused ? RRG_STRATEGY_FUSED : RRG_STRATEGY_BASELINE;
  return c;
}

// imm.hpp:157-162 (the store's fused counter is the phase's Counter)
struct SamplingPhaseResult {
  RRRStore store;
  double lower_bound = 0.0;
  uint64_t theta_prime = 0;
};

// imm.hpp:169-209
inline SamplingPhaseResult sampling_phase(const Graph& g, const ImmConfig& cfg,
                                          ImmTimings* timings = nullptr) {
  const rrg_imm_config c = to_c(cfg);
  SamplingPhaseResult out{RRRStore(g)};
  rrg_imm_result t{};
  check(rrg_sampling_phase(g.handle(), &c, out.store.handle(), &out.lower_bound,
                           &out.theta_prime, &t));
  if (timings) {
    timings->generate_rrrsets += t.t_generate;
    timings->find_most_influential += t.t_select;
  }
  return out;
}

// imm.hpp:214-251
inline ImmResult run_imm(const Graph& g, const ImmConfig& cfg) {
  const rrg_imm_config c = to_c(cfg);
  ImmResult r;
  const uint32_t k = cfg.k ? cfg.k : 1;
  r.seeds.seeds.resize(k);
  r.seeds.marginal_counts.resize(k);
  rrg_imm_result out{};
  check(rrg_run_imm(g.handle(), &c, r.seeds.seeds.data(), r.seeds.marginal_counts.data(), &out));
  r.theta = out.theta;
  r.theta_prime = out.theta_prime;
  r.lower_bound = out.lower_bound;
  r.timings = {out.t_generate, out.t_select, out.t_total};
  r.sets_generated = out.sets_generated;
  r.mean_set_size = out.mean_set_size;
  r.max_set_size = out.max_set_size;
  r.mean_coverage_fraction = out.mean_coverage_fraction;
  return r;
}

}  // namespace rrgpu
