// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED reference headers.
// TEST INFRASTRUCTURE ONLY (kind "reference").
//
// Compiled by oracle/Makefile with -I/root/reference/proj/include into
// oracle/_ref/librrflow_ref.so (git-ignored, travels to the GPU box as a
// built artefact). No reference source is copied: every algorithm below is a
// call into rrflow::*. The shim only converts between the transpose arrays of
// oracle.h and rrflow::Graph / RRRStore.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "oracle.h"
#include "rrflow/graph.hpp"
#include "rrflow/imm.hpp"
#include "rrflow/oracle.hpp"
#include "rrflow/sampling.hpp"
#include "rrflow/selection.hpp"

namespace {
thread_local std::string g_err;

rrflow::DiffusionModel to_model(int m) {
  return m == 0 ? rrflow::DiffusionModel::IC : rrflow::DiffusionModel::LT;
}

void export_reverse(const rrflow::Graph& g, uint64_t* roff, uint32_t* rsrc, float* rw) {
  std::memcpy(roff, g.reverse_offsets.data(), (g.num_vertices + 1) * 8ull);
  std::memcpy(rsrc, g.reverse_sources.data(), g.num_edges * 4ull);
  std::memcpy(rw, g.reverse_weights.data(), g.num_edges * 4ull);
}
}  // namespace

struct orc_graph {
  rrflow::Graph g;
};

struct orc_store {
  uint32_t n = 0;
  std::vector<uint64_t> off;
  std::vector<uint32_t> mem;
  std::vector<uint32_t> roots;
  std::vector<uint64_t> counter;
};

extern "C" {

const char* orc_kind(void) { return "reference"; }
const char* orc_last_error(void) { return g_err.c_str(); }

// Rebuilds an rrflow::Graph whose transpose equals the given arrays. The
// reference orders each in-list by source id (graph.hpp:96-113), so inputs
// produced by detail::build_graph round-trip exactly; anything else is refused.
orc_graph* orc_graph_new(uint32_t n, uint64_t m, const uint64_t* roff, const uint32_t* rsrc,
                         const float* rw) {
  try {
    std::vector<rrflow::detail::EdgeTriple> edges;
    edges.reserve(m);
    std::vector<uint64_t> order(m);
    std::vector<uint32_t> dst_of(m);
    for (uint32_t v = 0; v < n; ++v)
      for (uint64_t j = roff[v]; j < roff[v + 1]; ++j) dst_of[j] = v;
    for (uint64_t j = 0; j < m; ++j) order[j] = j;
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
      if (rsrc[a] != rsrc[b]) return rsrc[a] < rsrc[b];
      return dst_of[a] < dst_of[b];
    });
    for (uint64_t j : order) edges.push_back({rsrc[j], dst_of[j], rw[j]});
    auto* h = new orc_graph;
    h->g = rrflow::detail::build_graph(n, std::move(edges), {});
    for (uint64_t j = 0; j < m; ++j) {
      if (h->g.reverse_sources[j] != rsrc[j] || h->g.reverse_weights[j] != rw[j]) {
        delete h;
        g_err = "transpose order not representable by rrflow::Graph";
        return nullptr;
      }
    }
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_graph_free(orc_graph* g) { delete g; }

uint64_t orc_derive_stream_seed(uint64_t run_seed, uint64_t stream) {
  return rrflow::derive_stream_seed(run_seed, stream);
}

void orc_prng_draws(uint64_t seed, uint64_t count, uint64_t* out) {
  rrflow::Prng r(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

uint64_t orc_uniform_below(uint64_t seed, uint64_t bound, double* next_u01) {
  rrflow::Prng r(seed);
  const uint64_t v = r.uniform_below(bound);
  if (next_u01) *next_u01 = r.uniform01();
  return v;
}

// first_slot == 0 goes through generate_batch_fused on a WorkPool (the
// reference's own batch path, sampling.hpp:159-206); other offsets replay
// the per-slot stream exactly as generate_batch does (:177-183).
orc_store* orc_sample(orc_graph* h, int model, uint64_t run_seed, uint64_t first_slot,
                      uint64_t count, uint32_t workers) {
  try {
    const rrflow::Graph& g = h->g;
    const uint32_t n = g.num_vertices;
    auto* st = new orc_store;
    st->n = n;
    st->off.assign(count + 1, 0);
    st->roots.assign(count, 0);
    st->counter.assign(n, 0);
    std::vector<std::vector<uint32_t>> sets(count);
    if (first_slot == 0) {
      rrflow::WorkPool pool(std::max<uint32_t>(1, workers));
      rrflow::RRRStore store(n, pool.workers());
      rrflow::Counter counter(n);
      rrflow::generate_batch_fused(g, to_model(model), run_seed, count, counter, pool, store);
      for (uint64_t k = 0; k < count; ++k) {
        const rrflow::RRRSet& r = store.set(k);
        st->roots[k] = r.root;
        r.for_each_member([&](uint32_t v) { sets[k].push_back(v); });
      }
      for (uint32_t v = 0; v < n; ++v) st->counter[v] = counter.get(v);
    } else {
      if (n == 0) throw std::invalid_argument("generate_batch: empty graph");
      rrflow::SamplerState state(n, 0);
      for (uint64_t k = 0; k < count; ++k) {
        state.reseed(rrflow::derive_stream_seed(run_seed, first_slot + k));
        const uint32_t root = rrflow::sample_root(state, n);
        const rrflow::RRRSet r = model == 0 ? rrflow::generate_rrr_ic(g, root, state)
                                            : rrflow::generate_rrr_lt(g, root, state);
        st->roots[k] = r.root;
        r.for_each_member([&](uint32_t v) {
          sets[k].push_back(v);
          st->counter[v]++;
        });
      }
    }
    for (uint64_t k = 0; k < count; ++k) st->off[k + 1] = st->off[k] + sets[k].size();
    st->mem.resize(st->off[count]);
    for (uint64_t k = 0; k < count; ++k)
      std::copy(sets[k].begin(), sets[k].end(), st->mem.begin() + st->off[k]);
    return st;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

uint64_t orc_store_sets(const orc_store* s) { return s->off.size() - 1; }
uint64_t orc_store_members(const orc_store* s) { return s->mem.size(); }
void orc_store_export(const orc_store* s, uint64_t* offsets, uint32_t* members) {
  std::memcpy(offsets, s->off.data(), s->off.size() * 8);
  std::memcpy(members, s->mem.data(), s->mem.size() * 4);
}
void orc_store_counter(const orc_store* s, uint64_t* counts) {
  std::memcpy(counts, s->counter.data(), s->counter.size() * 8);
}
void orc_store_roots(const orc_store* s, uint32_t* roots) {
  std::memcpy(roots, s->roots.data(), s->roots.size() * 4);
}
uint64_t orc_store_inspected(const orc_store*) { return UINT64_MAX; }
void orc_store_free(orc_store* s) { delete s; }

// select_seeds on a store built like proj/tests/test_util.hpp:55-63.
int orc_select(uint32_t n, uint64_t nsets, const uint64_t* offsets, const uint32_t* members,
               uint32_t k, double threshold, uint32_t workers, uint32_t* seeds,
               uint64_t* marginals, uint64_t* round_counters, uint32_t* rounds_done) {
  try {
    rrflow::RRRStore store(n, 1);
    for (uint64_t s = 0; s < nsets; ++s) {
      std::vector<uint32_t> mem(members + offsets[s], members + offsets[s + 1]);
      store.append(rrflow::make_repr(std::move(mem), n));
    }
    rrflow::WorkPool pool(std::max<uint32_t>(1, workers));
    rrflow::SelectionStats stats;
    stats.capture_round_counters = round_counters != nullptr;
    const rrflow::SeedSet out =
        rrflow::select_seeds(store, n, k, pool, threshold, nullptr, &stats);
    for (size_t i = 0; i < out.seeds.size(); ++i) {
      seeds[i] = out.seeds[i];
      marginals[i] = out.marginal_counts[i];
    }
    if (round_counters) {
      for (size_t r = 0; r < stats.round_counters.size(); ++r)
        std::memcpy(round_counters + r * n, stats.round_counters[r].data(), 8ull * n);
    }
    if (rounds_done) *rounds_done = static_cast<uint32_t>(stats.round_counters.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int orc_imm(orc_graph* h, const orc_imm_config* c, uint32_t* seeds, uint64_t* marginals,
            orc_imm_result* out) {
  try {
    rrflow::ImmConfig cfg;
    cfg.k = c->k;
    cfg.epsilon = c->epsilon;
    cfg.model = to_model(c->model);
    cfg.workers = c->workers;
    cfg.rng_seed = c->rng_seed;
    cfg.ell = c->ell;
    cfg.adaptive_threshold = c->adaptive_threshold;
    cfg.strategy = c->strategy ? rrflow::Strategy::baseline : rrflow::Strategy::fused;
    const rrflow::ImmResult r = rrflow::run_imm(h->g, cfg);
    for (size_t i = 0; i < r.seeds.seeds.size(); ++i) {
      seeds[i] = r.seeds.seeds[i];
      marginals[i] = r.seeds.marginal_counts[i];
    }
    out->theta = r.theta;
    out->theta_prime = r.theta_prime;
    out->lower_bound = r.lower_bound;
    out->sets_generated = r.sets_generated;
    out->mean_set_size = r.mean_set_size;
    out->max_set_size = r.max_set_size;
    out->mean_coverage_fraction = r.mean_coverage_fraction;
    out->t_generate = r.timings.generate_rrrsets;
    out->t_select = r.timings.find_most_influential;
    out->t_total = r.timings.total;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int orc_sampling_phase(orc_graph* h, const orc_imm_config* c, double* lower_bound,
                       uint64_t* theta_prime, uint64_t* counter) {
  try {
    rrflow::ImmConfig cfg;
    cfg.k = c->k;
    cfg.epsilon = c->epsilon;
    cfg.model = to_model(c->model);
    cfg.workers = c->workers;
    cfg.rng_seed = c->rng_seed;
    cfg.ell = c->ell;
    cfg.adaptive_threshold = c->adaptive_threshold;
    cfg.strategy = c->strategy ? rrflow::Strategy::baseline : rrflow::Strategy::fused;
    rrflow::WorkPool pool(std::max<uint32_t>(1, c->workers));
    const rrflow::SamplingPhaseResult r = rrflow::sampling_phase(h->g, cfg, pool);
    *lower_bound = r.lower_bound;
    *theta_prime = r.theta_prime;
    if (counter)
      for (uint32_t v = 0; v < h->g.num_vertices; ++v) counter[v] = r.counter.get(v);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double orc_log_binomial(uint64_t n, uint64_t k) { return rrflow::log_binomial(n, k); }
double orc_effective_ell(double ell, uint64_t n) { return rrflow::effective_ell(ell, n); }
double orc_lambda_prime(uint64_t n, uint64_t k, double e, double l) {
  return rrflow::lambda_prime(n, k, e, l);
}
uint32_t orc_sampling_rounds(uint64_t n) { return rrflow::sampling_rounds(n); }
uint64_t orc_theta_for_round(uint64_t n, uint64_t k, double e, double l, uint32_t i) {
  return rrflow::theta_for_round(n, k, e, l, i);
}
double orc_lambda_star(uint64_t n, uint64_t k, double e, double l) {
  return rrflow::lambda_star(n, k, e, l);
}
uint64_t orc_set_theta(uint64_t n, uint64_t k, double e, double l, double lb) {
  return rrflow::set_theta(n, k, e, l, lb);
}

int orc_build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                    const float* w, uint64_t* roff, uint32_t* rsrc, float* rw) {
  try {
    std::vector<rrflow::detail::EdgeTriple> edges(m);
    for (uint64_t e = 0; e < m; ++e) edges[e] = {src[e], dst[e], w[e]};
    const rrflow::Graph g = rrflow::detail::build_graph(n, std::move(edges), {});
    export_reverse(g, roff, rsrc, rw);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// normalize_lt_weights on a graph whose transpose is (roff, rsrc-less, rw): the
// reference normalizes per in-list and mirrors into the forward view; only the
// transpose weights are read back.
int orc_normalize_lt(uint32_t n, const uint64_t* roff, float* rw) {
  try {
    rrflow::Graph g;
    g.num_vertices = n;
    g.num_edges = roff[n];
    g.reverse_offsets.assign(roff, roff + n + 1);
    g.reverse_weights.assign(rw, rw + roff[n]);
    g.forward_weights.assign(roff[n], 0.0f);
    g.reverse_edge_index.resize(roff[n]);
    for (uint64_t j = 0; j < roff[n]; ++j) g.reverse_edge_index[j] = j;
    rrflow::normalize_lt_weights(g);
    std::memcpy(rw, g.reverse_weights.data(), roff[n] * 4ull);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double orc_activation_probability(orc_graph* h, const uint32_t* sources, uint32_t nsrc,
                                  uint32_t target, int model, uint64_t trials, uint64_t seed) {
  std::vector<uint32_t> s(sources, sources + nsrc);
  return rrflow::activation_probability(h->g, s, target, to_model(model), trials, seed);
}

double orc_exact_spread(orc_graph* h, const uint32_t* seeds, uint32_t k, int model) {
  std::vector<uint32_t> s(seeds, seeds + k);
  return rrflow::exact_spread(h->g, s, to_model(model)).value;
}

uint64_t orc_synth_graph(int kind, uint32_t n, double param, uint64_t seed, int with_ic,
                         uint64_t ic_seed, uint64_t* roff, uint32_t* rsrc, float* rw) {
  try {
    rrflow::Graph g = rrflow::synth_graph(
        kind == 0 ? rrflow::SynthKind::erdos_renyi : rrflow::SynthKind::scc_core, n, param, seed);
    if (with_ic) rrflow::generate_ic_weights(g, ic_seed);
    if (roff) export_reverse(g, roff, rsrc, rw);
    return g.num_edges;
  } catch (const std::exception& e) {
    g_err = e.what();
    return UINT64_MAX;
  }
}

}  // extern "C"
