// port.cpp -- CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
//
// This is the "port" checker: the reference algorithm (rrflow 0.1.0,
// /root/reference/proj/include/rrflow) re-expressed in plain C++17, one
// function per reference function, each citing the file:line it follows.
// It is pinned against the reference itself (oracle/_ref, built from the
// unmodified headers by oracle/Makefile) and against the golden vectors in
// tests/golden/ (tests/test_oracle_pin.py). Nothing in paper_2411_09473_b200/
// links or calls this file; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg load it.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oracle.h"

namespace {

thread_local std::string g_err;

// ---- prng.hpp:8-13 splitmix64, :17-20 derive_stream_seed -------------------
inline uint64_t sm64_next(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline uint64_t stream_seed(uint64_t run_seed, uint64_t stream) {
  uint64_t s = run_seed ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  return sm64_next(s);
}

// ---- prng.hpp:23-70 xoshiro256** ------------------------------------------
struct Xoshiro {
  uint64_t s[4];
  void seed(uint64_t v) {  // prng.hpp:28-31: four successive splitmix64 outputs
    for (int i = 0; i < 4; ++i) s[i] = sm64_next(v);
  }
  static uint64_t rol(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {  // prng.hpp:33-43
    const uint64_t out = rol(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rol(s[3], 45);
    return out;
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // prng.hpp:46
  uint64_t below(uint64_t bound) {  // prng.hpp:49-60 (Lemire, rejection below threshold)
    unsigned __int128 prod = static_cast<unsigned __int128>(next()) * bound;
    uint64_t low = static_cast<uint64_t>(prod);
    if (low < bound) {
      const uint64_t thr = (0 - bound) % bound;
      while (low < thr) {
        prod = static_cast<unsigned __int128>(next()) * bound;
        low = static_cast<uint64_t>(prod);
      }
    }
    return static_cast<uint64_t>(prod >> 64);
  }
};

}  // namespace

struct orc_graph {
  uint32_t n = 0;
  uint64_t m = 0;
  std::vector<uint64_t> off;
  std::vector<uint32_t> src;
  std::vector<float> w;
};

struct orc_store {
  uint32_t n = 0;
  std::vector<uint64_t> off;   // slot-ordered offsets
  std::vector<uint32_t> mem;   // ascending per set (rrr_set.hpp:73-90 sparse form)
  std::vector<uint32_t> roots;
  std::vector<uint64_t> counter;
  uint64_t inspected = 0;
};

namespace {

// One reverse sketch, following sampling.hpp:90-111 (IC) and :117-145 (LT).
// `mark` is an n-entry byte map cleared through the member list afterwards
// (sampling.hpp:34-38). Returns members in visit order (root first).
void one_sketch(const orc_graph& g, int model, Xoshiro& rng, uint32_t root,
                std::vector<uint8_t>& mark, std::vector<uint32_t>& order,
                uint64_t& inspected) {
  order.clear();
  order.push_back(root);
  mark[root] = 1;
  if (model == 0) {
    for (size_t head = 0; head < order.size(); ++head) {
      const uint32_t u = order[head];
      for (uint64_t j = g.off[u]; j < g.off[u + 1]; ++j) {
        ++inspected;
        const uint32_t v = g.src[j];
        // sampling.hpp:102 -- the draw happens only for unvisited sources
        if (mark[v]) continue;
        if (rng.u01() < static_cast<double>(g.w[j])) {
          mark[v] = 1;
          order.push_back(v);
        }
      }
    }
  } else {
    uint32_t u = root;
    for (;;) {
      const double draw = rng.u01();  // sampling.hpp:127: one draw per step
      double acc = 0.0;               // sampling.hpp:128: double running sum
      uint32_t pick = g.n;
      for (uint64_t j = g.off[u]; j < g.off[u + 1]; ++j) {
        ++inspected;
        acc += g.w[j];
        if (draw < acc) {
          pick = g.src[j];
          break;
        }
      }
      if (pick == g.n || mark[pick]) break;  // sampling.hpp:137
      mark[pick] = 1;
      order.push_back(pick);
      u = pick;
    }
  }
  for (uint32_t v : order) mark[v] = 0;
}

}  // namespace

extern "C" {

const char* orc_kind(void) { return "port"; }
const char* orc_last_error(void) { return g_err.c_str(); }

orc_graph* orc_graph_new(uint32_t n, uint64_t m, const uint64_t* roff, const uint32_t* rsrc,
                         const float* rw) {
  auto* g = new orc_graph;
  g->n = n;
  g->m = m;
  g->off.assign(roff, roff + n + 1);
  g->src.assign(rsrc, rsrc + m);
  g->w.assign(rw, rw + m);
  return g;
}

void orc_graph_free(orc_graph* g) { delete g; }

uint64_t orc_derive_stream_seed(uint64_t run_seed, uint64_t stream) {
  return stream_seed(run_seed, stream);
}

void orc_prng_draws(uint64_t seed, uint64_t count, uint64_t* out) {
  Xoshiro r;
  r.seed(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = r.next();
}

uint64_t orc_uniform_below(uint64_t seed, uint64_t bound, double* next_u01) {
  Xoshiro r;
  r.seed(seed);
  const uint64_t v = r.below(bound);
  if (next_u01) *next_u01 = r.u01();
  return v;
}

// generate_batch (sampling.hpp:159-199): slot j <- stream derive(run_seed, j),
// root = uniform_below(n) right after reseed (:179-180), fused counter (:184-186).
orc_store* orc_sample(orc_graph* g, int model, uint64_t run_seed, uint64_t first_slot,
                      uint64_t count, uint32_t workers) {
  if (g->n == 0) {
    g_err = "generate_batch: empty graph";
    return nullptr;
  }
  auto* st = new orc_store;
  st->n = g->n;
  std::vector<std::vector<uint32_t>> sets(count);
  st->roots.assign(count, 0);
  const unsigned w = std::max<uint32_t>(1, workers);
  std::atomic<uint64_t> next{0}, insp{0};
  auto body = [&]() {
    std::vector<uint8_t> mark(g->n, 0);
    std::vector<uint32_t> order;
    uint64_t local = 0;
    for (;;) {
      const uint64_t i = next.fetch_add(64);
      if (i >= count) break;
      const uint64_t e = std::min<uint64_t>(count, i + 64);
      for (uint64_t k = i; k < e; ++k) {
        Xoshiro rng;
        rng.seed(stream_seed(run_seed, first_slot + k));
        const uint32_t root = static_cast<uint32_t>(rng.below(g->n));
        one_sketch(*g, model, rng, root, mark, order, local);
        st->roots[k] = root;
        sets[k] = order;
        std::sort(sets[k].begin(), sets[k].end());
      }
    }
    insp += local;
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < w; ++t) pool.emplace_back(body);
  body();
  for (auto& t : pool) t.join();
  st->inspected = insp.load();
  st->off.assign(count + 1, 0);
  for (uint64_t k = 0; k < count; ++k) st->off[k + 1] = st->off[k] + sets[k].size();
  st->mem.resize(st->off[count]);
  st->counter.assign(g->n, 0);
  for (uint64_t k = 0; k < count; ++k) {
    std::copy(sets[k].begin(), sets[k].end(), st->mem.begin() + st->off[k]);
    for (uint32_t v : sets[k]) st->counter[v]++;
  }
  return st;
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
uint64_t orc_store_inspected(const orc_store* s) { return s->inspected; }
void orc_store_free(orc_store* s) { delete s; }

// select_seeds (selection.hpp:209-243) with decrement_update (:130-156) as the
// only update: rebuild_update (:161-203) is observationally identical
// (proj/tests/test_selection.cpp:116-137), so the threshold changes no output.
// parallel_argmax tie rule: highest count, then lowest id (:113, :119-120).
int orc_select(uint32_t n, uint64_t nsets, const uint64_t* offsets, const uint32_t* members,
               uint32_t k, double /*threshold*/, uint32_t /*workers*/, uint32_t* seeds,
               uint64_t* marginals, uint64_t* round_counters, uint32_t* rounds_done) {
  if (k < 1) {
    g_err = "select_seeds: k must be >= 1";
    return -1;
  }
  if (k > n) {
    g_err = "select_seeds: k exceeds vertex count";
    return -1;
  }
  std::vector<uint64_t> cnt(n, 0);
  for (uint64_t s = 0; s < nsets; ++s)
    for (uint64_t j = offsets[s]; j < offsets[s + 1]; ++j) cnt[members[j]]++;
  // vertex -> sets index, so each round touches only the sets holding v
  std::vector<uint64_t> ioff(n + 1, 0);
  for (uint32_t v = 0; v < n; ++v) ioff[v + 1] = ioff[v] + cnt[v];
  std::vector<uint64_t> inv(ioff[n]);
  {
    std::vector<uint64_t> cur(ioff.begin(), ioff.end() - 1);
    for (uint64_t s = 0; s < nsets; ++s)
      for (uint64_t j = offsets[s]; j < offsets[s + 1]; ++j) inv[cur[members[j]]++] = s;
  }
  std::vector<uint8_t> dead(nsets, 0), chosen(n, 0);
  uint32_t filled = 0;
  uint32_t captured = 0;
  for (uint32_t r = 0; r < k; ++r) {
    uint32_t best = 0;
    for (uint32_t v = 1; v < n; ++v)
      if (cnt[v] > cnt[best]) best = v;
    if (cnt[best] == 0) {
      // selection.hpp:61-72: lowest unselected ids at zero marginal
      for (uint32_t v = 0; v < n && filled < k; ++v) {
        if (!chosen[v]) {
          chosen[v] = 1;
          seeds[filled] = v;
          marginals[filled] = 0;
          ++filled;
        }
      }
      break;
    }
    uint64_t killed = 0;
    for (uint64_t t = ioff[best]; t < ioff[best + 1]; ++t) {
      const uint64_t s = inv[t];
      if (dead[s]) continue;
      dead[s] = 1;
      ++killed;
      for (uint64_t j = offsets[s]; j < offsets[s + 1]; ++j) cnt[members[j]]--;
    }
    chosen[best] = 1;
    seeds[filled] = best;
    marginals[filled] = killed;
    ++filled;
    if (round_counters) {
      std::memcpy(round_counters + static_cast<uint64_t>(captured) * n, cnt.data(), 8ull * n);
      ++captured;
    }
  }
  if (rounds_done) *rounds_done = captured;
  return 0;
}

// ---- imm.hpp:57-120 theta math, same expression order ---------------------
double orc_log_binomial(uint64_t n, uint64_t k) {
  double acc = 0.0;
  for (uint64_t j = n - k + 1; j <= n; ++j) acc += std::log(static_cast<double>(j));
  for (uint64_t j = 1; j <= k; ++j) acc -= std::log(static_cast<double>(j));
  return acc;
}
double orc_effective_ell(double ell, uint64_t n) {
  if (n < 2) return ell;
  return ell * (1.0 + std::log(2.0) / std::log(static_cast<double>(n)));
}
double orc_lambda_prime(uint64_t n, uint64_t k, double eps, double ell) {
  const double nd = static_cast<double>(n);
  const double ep = std::sqrt(2.0) * eps;
  const double l2 = std::max(1.0, std::log2(nd));
  const double terms = orc_log_binomial(n, k) + ell * std::log(nd) + std::log(l2);
  return (2.0 + (2.0 / 3.0) * ep) * terms * nd / (ep * ep);
}
uint32_t orc_sampling_rounds(uint64_t n) {
  if (n <= 4) return 1;
  const int r = static_cast<int>(std::floor(std::log2(static_cast<double>(n)))) - 1;
  return r < 1 ? 1u : static_cast<uint32_t>(r);
}
static double round_target(uint64_t n, unsigned i) {
  if (n <= 4) return std::max(1.0, static_cast<double>(n) / 2.0);
  return static_cast<double>(n) / std::exp2(static_cast<double>(i));
}
uint64_t orc_theta_for_round(uint64_t n, uint64_t k, double eps, double ell, uint32_t i) {
  const double t = std::ceil(orc_lambda_prime(n, k, eps, ell) / round_target(n, i));
  if (!(t >= 1.0)) return 1;
  return static_cast<uint64_t>(t);
}
double orc_lambda_star(uint64_t n, uint64_t k, double eps, double ell) {
  const double nd = static_cast<double>(n);
  const double c = 1.0 - 1.0 / std::exp(1.0);
  const double a = std::sqrt(ell * std::log(nd) + std::log(2.0));
  const double b = std::sqrt(c * (orc_log_binomial(n, k) + ell * std::log(nd) + std::log(2.0)));
  const double s = c * a + b;
  return 2.0 * nd * s * s / (eps * eps);
}
uint64_t orc_set_theta(uint64_t n, uint64_t k, double eps, double ell, double lb) {
  const double t = std::ceil(orc_lambda_star(n, k, eps, ell) / lb);
  if (!(t >= 1.0)) return 1;
  return static_cast<uint64_t>(t);
}

// sampling_phase (imm.hpp:169-209) alone: the same rounds as orc_imm below.
int orc_sampling_phase(orc_graph* g, const orc_imm_config* cfg, double* lower_bound,
                       uint64_t* theta_prime, uint64_t* counter) {
  const uint32_t n = g->n;
  if (n == 0 || !(cfg->epsilon > 0.0 && cfg->epsilon < 1.0) || cfg->k < 1 || cfg->k > n ||
      cfg->workers < 1) {
    g_err = "invalid configuration";  // imm.hpp:136-145
    return -1;
  }
  const double ell = orc_effective_ell(cfg->ell, n);
  const double eps_prime = std::sqrt(2.0) * cfg->epsilon;
  std::vector<uint64_t> off{0};
  std::vector<uint32_t> mem;
  std::vector<uint32_t> sd(cfg->k);
  std::vector<uint64_t> mg(cfg->k);
  const uint32_t rounds = orc_sampling_rounds(n);
  double spread = 0.0;
  bool triggered = false;
  for (uint32_t i = 1; i <= rounds; ++i) {
    const uint64_t target = orc_theta_for_round(n, cfg->k, cfg->epsilon, ell, i);
    const uint64_t have = off.size() - 1;
    if (target > have) {
      orc_store* st = orc_sample(g, cfg->model, cfg->rng_seed, have, target - have, cfg->workers);
      for (uint64_t s = 0; s < target - have; ++s)
        off.push_back(off.back() + (st->off[s + 1] - st->off[s]));
      mem.insert(mem.end(), st->mem.begin(), st->mem.end());
      orc_store_free(st);
    }
    orc_select(n, off.size() - 1, off.data(), mem.data(), cfg->k, cfg->adaptive_threshold, 1,
               sd.data(), mg.data(), nullptr, nullptr);
    uint64_t covered = 0;
    for (uint32_t r = 0; r < cfg->k; ++r) covered += mg[r];
    spread = static_cast<double>(n) * (static_cast<double>(covered) / static_cast<double>(off.size() - 1));
    if (spread >= (1.0 + eps_prime) * round_target(n, i)) {
      triggered = true;
      break;
    }
  }
  *lower_bound = triggered ? spread / (1.0 + eps_prime)
                           : std::max(spread / (1.0 + eps_prime), static_cast<double>(cfg->k));
  *theta_prime = off.size() - 1;
  if (counter) {
    std::fill(counter, counter + n, 0);
    if (!cfg->strategy)  // the fused strategy's counter; baseline samples unfused
      for (uint32_t v : mem) ++counter[v];
  }
  return 0;
}

// run_imm (imm.hpp:214-251) with sampling_phase (imm.hpp:169-209).
int orc_imm(orc_graph* g, const orc_imm_config* cfg, uint32_t* seeds, uint64_t* marginals,
            orc_imm_result* out) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const uint32_t n = g->n;
  if (n == 0 || !(cfg->epsilon > 0.0 && cfg->epsilon < 1.0) || cfg->k < 1 || cfg->k > n ||
      cfg->workers < 1) {
    g_err = "invalid configuration";  // imm.hpp:136-145
    return -1;
  }
  const double ell = orc_effective_ell(cfg->ell, n);
  const double eps_prime = std::sqrt(2.0) * cfg->epsilon;
  std::vector<uint64_t> off{0};
  std::vector<uint32_t> mem;
  double tg = 0, ts = 0;
  auto top_up = [&](uint64_t target) {
    const uint64_t have = off.size() - 1;
    if (target <= have) return;
    const auto a = clk::now();
    orc_store* st = orc_sample(g, cfg->model, cfg->rng_seed, have, target - have, cfg->workers);
    for (uint64_t s = 0; s < target - have; ++s) {
      off.push_back(off.back() + (st->off[s + 1] - st->off[s]));
    }
    mem.insert(mem.end(), st->mem.begin(), st->mem.end());
    orc_store_free(st);
    tg += std::chrono::duration<double>(clk::now() - a).count();
  };
  auto select = [&](uint32_t* sd, uint64_t* mg) {
    const auto a = clk::now();
    orc_select(n, off.size() - 1, off.data(), mem.data(), cfg->k, cfg->adaptive_threshold, 1,
               sd, mg, nullptr, nullptr);
    ts += std::chrono::duration<double>(clk::now() - a).count();
  };
  std::vector<uint32_t> sd(cfg->k);
  std::vector<uint64_t> mg(cfg->k);
  const uint32_t rounds = orc_sampling_rounds(n);
  double spread = 0.0;
  bool triggered = false;
  for (uint32_t i = 1; i <= rounds; ++i) {
    top_up(orc_theta_for_round(n, cfg->k, cfg->epsilon, ell, i));
    select(sd.data(), mg.data());
    uint64_t covered = 0;
    for (uint32_t r = 0; r < cfg->k; ++r) covered += mg[r];
    const double frac = static_cast<double>(covered) / static_cast<double>(off.size() - 1);
    spread = static_cast<double>(n) * frac;
    if (spread >= (1.0 + eps_prime) * round_target(n, i)) {
      triggered = true;
      break;
    }
  }
  const double lb = triggered ? spread / (1.0 + eps_prime)
                              : std::max(spread / (1.0 + eps_prime), static_cast<double>(cfg->k));
  out->theta_prime = off.size() - 1;
  out->lower_bound = lb;
  out->theta = orc_set_theta(n, cfg->k, cfg->epsilon, ell, lb);
  top_up(out->theta);
  select(seeds, marginals);
  out->sets_generated = off.size() - 1;
  uint32_t mx = 0;
  for (uint64_t s = 0; s + 1 < off.size(); ++s)
    mx = std::max<uint32_t>(mx, static_cast<uint32_t>(off[s + 1] - off[s]));
  out->mean_set_size = static_cast<double>(mem.size()) / static_cast<double>(off.size() - 1);
  out->max_set_size = mx;
  out->mean_coverage_fraction = out->mean_set_size / static_cast<double>(n);
  out->t_generate = tg;
  out->t_select = ts;
  out->t_total = std::chrono::duration<double>(clk::now() - t0).count();
  return 0;
}

// detail::build_graph (graph.hpp:69-115): forward CSR by stable counting sort on
// source; transpose filled by walking sources ascending and forward slots in order.
int orc_build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                    const float* w, uint64_t* roff, uint32_t* rsrc, float* rw) {
  std::vector<uint64_t> foff(n + 1, 0);
  for (uint64_t e = 0; e < m; ++e) foff[src[e] + 1]++;
  for (uint32_t v = 0; v < n; ++v) foff[v + 1] += foff[v];
  std::vector<uint32_t> ft(m);
  std::vector<float> fw(m);
  {
    std::vector<uint64_t> cur(foff.begin(), foff.end() - 1);
    for (uint64_t e = 0; e < m; ++e) {
      const uint64_t p = cur[src[e]]++;
      ft[p] = dst[e];
      fw[p] = w[e];
    }
  }
  std::fill(roff, roff + n + 1, 0);
  for (uint64_t e = 0; e < m; ++e) roff[dst[e] + 1]++;
  for (uint32_t v = 0; v < n; ++v) roff[v + 1] += roff[v];
  std::vector<uint64_t> cur(roff, roff + n);
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t j = foff[u]; j < foff[u + 1]; ++j) {
      const uint64_t p = cur[ft[j]]++;
      rsrc[p] = u;
      rw[p] = fw[j];
    }
  return 0;
}

// normalize_lt_weights (graph.hpp:207-235), applied to the transpose weights.
int orc_normalize_lt(uint32_t n, const uint64_t* roff, float* rw) {
  for (uint32_t v = 0; v < n; ++v) {
    double sum = 0.0;
    for (uint64_t j = roff[v]; j < roff[v + 1]; ++j) {
      if (rw[j] < 0.0f) {
        g_err = "negative edge weight";
        return -1;
      }
      sum += rw[j];
    }
    if (sum <= 1.0) continue;
    double scale = 1.0 / sum;
    for (int attempt = 0; attempt < 64; ++attempt) {
      double ss = 0.0;
      for (uint64_t j = roff[v]; j < roff[v + 1]; ++j)
        ss += static_cast<float>(rw[j] * scale);
      if (ss <= 1.0) break;
      scale *= 1.0 - 0x1.0p-20;
    }
    for (uint64_t j = roff[v]; j < roff[v + 1]; ++j) rw[j] = static_cast<float>(rw[j] * scale);
  }
  return 0;
}

double orc_activation_probability(orc_graph*, const uint32_t*, uint32_t, uint32_t, int, uint64_t,
                                  uint64_t) {
  g_err = "activation_probability: reference library only";
  return -1.0;
}
double orc_exact_spread(orc_graph*, const uint32_t*, uint32_t, int) {
  g_err = "exact_spread: reference library only";
  return -1.0;
}
uint64_t orc_synth_graph(int, uint32_t, double, uint64_t, int, uint64_t, uint64_t*, uint32_t*,
                         float*) {
  g_err = "synth_graph: reference library only";
  return UINT64_MAX;
}

}  // extern "C"
