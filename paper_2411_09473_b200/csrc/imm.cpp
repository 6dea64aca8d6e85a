// imm.cpp -- the IMM driver (host C++17). Re-expresses imm.hpp:57-251 with the
// same expression order and libm calls, so theta, theta', LB and the seeds are
// bit-identical to the reference; every sampling and selection call goes through
// the C ABI into the device (rrg_generate_batch / rrg_select_seeds). Between
// rounds only the scalar coverage crosses back to the host (imm.hpp:194-201).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/rrgpu.h"

namespace rrgpu {
void set_error(const std::string& msg);
// shard.cu (multi-GPU): NCCL exchange of this rank's shard + ordered append
rrg_status exchange_and_append(rrg_store* side, rrg_store* dst, void* comm);
void nccl_comm_shape(void* comm, int* nranks, int* rank);
void store_keep_host_offsets(rrg_store* s, bool on);  // capi.cu
double graph_ic_mean_inspected(const rrg_graph* g);   // capi.cu
// select_seeds that stops once the coverage provably cannot reach `need` sets
rrg_status select_seeds_until(rrg_store* s, uint32_t k, double adaptive_threshold,
                              int use_prebuilt, uint32_t* seeds, uint64_t* marginals,
                              uint64_t* covered_total, uint64_t need, bool* aborted);  // capi.cu
}

#ifndef RRG_IMM_FREE_EDGES
#define RRG_IMM_FREE_EDGES 67108864.0  // 2^26 inspected edges: ~1.5 ms of IC sampler throughput
#endif

namespace {

// imm.hpp:57-63
double log_binomial(uint64_t n, uint64_t k) {
  double sum = 0.0;
  for (uint64_t j = n - k + 1; j <= n; ++j) sum += std::log(static_cast<double>(j));
  for (uint64_t j = 1; j <= k; ++j) sum -= std::log(static_cast<double>(j));
  return sum;
}

// imm.hpp:66-69
double effective_ell(double ell, uint64_t n) {
  if (n < 2) return ell;
  return ell * (1.0 + std::log(2.0) / std::log(static_cast<double>(n)));
}

// imm.hpp:72-79
double lambda_prime(uint64_t n, uint64_t k, double epsilon, double ell) {
  const double nd = static_cast<double>(n);
  const double eps_prime = std::sqrt(2.0) * epsilon;
  const double log2n = std::max(1.0, std::log2(nd));
  const double terms = log_binomial(n, k) + ell * std::log(nd) + std::log(log2n);
  return (2.0 + (2.0 / 3.0) * eps_prime) * terms * nd / (eps_prime * eps_prime);
}

// imm.hpp:82-86
unsigned sampling_rounds(uint64_t n) {
  if (n <= 4) return 1;
  const auto r = static_cast<int>(std::floor(std::log2(static_cast<double>(n)))) - 1;
  return r < 1 ? 1u : static_cast<unsigned>(r);
}

// imm.hpp:89-92
double round_target(uint64_t n, unsigned i) {
  if (n <= 4) return std::max(1.0, static_cast<double>(n) / 2.0);
  return static_cast<double>(n) / std::exp2(static_cast<double>(i));
}

// imm.hpp:95-100
uint64_t theta_for_round(uint64_t n, uint64_t k, double epsilon, double ell, unsigned i) {
  const double theta = std::ceil(lambda_prime(n, k, epsilon, ell) / round_target(n, i));
  if (!(theta >= 1.0)) return 1;
  return static_cast<uint64_t>(theta);
}

// imm.hpp:103-112
double lambda_star(uint64_t n, uint64_t k, double epsilon, double ell) {
  const double nd = static_cast<double>(n);
  const double one_minus_inv_e = 1.0 - 1.0 / std::exp(1.0);
  const double alpha = std::sqrt(ell * std::log(nd) + std::log(2.0));
  const double beta =
      std::sqrt(one_minus_inv_e * (log_binomial(n, k) + ell * std::log(nd) + std::log(2.0)));
  const double s = one_minus_inv_e * alpha + beta;
  return 2.0 * nd * s * s / (epsilon * epsilon);
}

// imm.hpp:115-120
uint64_t set_theta(uint64_t n, uint64_t k, double epsilon, double ell, double lower_bound) {
  const double theta = std::ceil(lambda_star(n, k, epsilon, ell) / lower_bound);
  if (!(theta >= 1.0)) return 1;
  return static_cast<uint64_t>(theta);
}

// RRGPU_IMM_EARLY_EXIT=0 runs every trial selection to the end (tests, A/B)
bool early_exit_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RRGPU_IMM_EARLY_EXIT");
    return !e || *e != '0';
  }();
  return on;
}

double seconds_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

struct StoreGuard {
  rrg_store* s = nullptr;
  ~StoreGuard() { rrg_store_destroy(s); }
};

// validate_config (imm.hpp:136-145)
rrg_status validate(rrg_graph* g, const rrg_imm_config* cfg) {
  const uint32_t n = rrg_graph_num_vertices(g);
  if (n == 0) {
    rrgpu::set_error("empty graph");
    return RRG_EINVAL;
  }
  if (!(cfg->epsilon > 0.0 && cfg->epsilon < 1.0)) {
    rrgpu::set_error("epsilon must lie in (0, 1)");
    return RRG_EINVAL;
  }
  if (cfg->k < 1 || cfg->k > n) {
    rrgpu::set_error("k must lie in [1, n]");
    return RRG_EINVAL;
  }
  if (cfg->workers < 1) {
    rrgpu::set_error("workers must be >= 1");
    return RRG_EINVAL;
  }
  if (cfg->model != RRG_IC && cfg->model != RRG_LT) {
    rrgpu::set_error("unknown diffusion model");
    return RRG_EINVAL;
  }
  if (cfg->strategy != RRG_STRATEGY_FUSED && cfg->strategy != RRG_STRATEGY_BASELINE) {
    rrgpu::set_error("unknown strategy");  // parse_strategy (imm.hpp:20-24)
    return RRG_EINVAL;
  }
  return RRG_OK;
}

// The IMM driver over one caller-visible store: top-ups (with speculation) and
// selections, timed like ImmTimings (imm.hpp:38-42).
class Driver {
 public:
  Driver(rrg_graph* g, const rrg_imm_config* cfg, rrg_store* store, void* comm = nullptr,
         int sim_ranks = 0)
      : g_(g), cfg_(cfg), store_(store), n_(rrg_graph_num_vertices(g)),
        ell_(effective_ell(cfg->ell, n_)), fused_(cfg->strategy == RRG_STRATEGY_FUSED),
        comm_(comm), sim_ranks_(sim_ranks), trial_seeds_(cfg->k), trial_marg_(cfg->k) {}

  double ell() const { return ell_; }
  uint64_t size() const { return size_; }
  double t_generate = 0.0, t_select = 0.0;

  // Top-ups. Slot j's set depends only on (rng_seed, j) (sampling.hpp:179), so
  // sets for slots a later round may need can be sampled ahead into a side
  // store and committed only when (and if) a top-up reaches them: the main
  // store ends up with exactly the reference's sets. Small batches are bound by
  // the latency of their largest set, so one batch covering the next rounds
  // costs about what one round's batch does.
  // Multi-GPU top-up: the new slots [size, target) split into
  // contiguous shards, rank r samples shard r (no communication), the shards are
  // exchanged over NCCL and appended in rank (= slot) order on every rank.
  // comm == nullptr with sim_ranks >= 1: the same split and ordered assembly in
  // one process (parity of the shard arithmetic without a second GPU).
  rrg_status top_up_sharded(uint64_t target) {
    const auto t = std::chrono::steady_clock::now();
    const uint64_t count = target - size_;
    int nranks = sim_ranks_, rank = 0;
    if (comm_) rrgpu::nccl_comm_shape(comm_, &nranks, &rank);
    rrg_status s = RRG_OK;
    if (!ahead_.s) s = rrg_store_create(g_, &ahead_.s);
    for (int r = comm_ ? rank : 0; s == RRG_OK && r < (comm_ ? rank + 1 : nranks); ++r) {
      const uint64_t a = count * static_cast<uint64_t>(r) / nranks;
      const uint64_t b = count * static_cast<uint64_t>(r + 1) / nranks;
      s = rrg_store_clear(ahead_.s);
      uint64_t made = 0;
      if (s == RRG_OK && b > a)
        s = rrg_generate_slots(g_, static_cast<rrg_model>(cfg_->model), cfg_->rng_seed,
                               size_ + a, b - a, ahead_.s, fused_ ? 1 : 0, 64, &made);
      if (s == RRG_OK && !comm_) s = rrg_store_append_from(store_, ahead_.s, 0, b - a);
    }
    if (s == RRG_OK && comm_) s = rrgpu::exchange_and_append(ahead_.s, store_, comm_);
    if (s == RRG_OK) size_ = target;
    t_generate += seconds_since(t);
    return s;
  }

  rrg_status ensure_ahead() {
    if (ahead_.s) return RRG_OK;
    const rrg_status s = rrg_store_create(g_, &ahead_.s);
    if (s == RRG_OK) rrgpu::store_keep_host_offsets(ahead_.s, true);  // appends need no read-back
    return s;
  }

  // A graph that has not sampled IC yet has no mean-inspected-edges estimate, so
  // its first top-up could not tell which later rounds are free to sample along
  // (ahead_for). Its first slots go out as a small pilot batch -- the sampler
  // splits a fresh graph's first batch at 2,048 sets anyway, to choose its
  // schedule -- and the first top-up then extends the side store knowing the
  // mean: cfg3 from host arrays samples 2,048 + 90,456 sets instead of 2,048 +
  // 21,078 + 69,378.
  rrg_status prime() {
    if (cfg_->model != RRG_IC || comm_ || sim_ranks_ > 0) return RRG_OK;
    if (rrgpu::graph_ic_mean_inspected(g_) >= 0.0) return RRG_OK;
    const auto t = std::chrono::steady_clock::now();
    rrg_status s = ensure_ahead();
    if (s != RRG_OK) return s;
    const uint64_t pilot =
        std::min<uint64_t>(2048, theta_for_round(n_, cfg_->k, cfg_->epsilon, ell_, 1));
    uint64_t made = 0;
    s = rrg_generate_slots(g_, static_cast<rrg_model>(cfg_->model), cfg_->rng_seed, 0, pilot,
                           ahead_.s, fused_ ? 1 : 0, 64, &made);
    ahead_first_ = 0;
    ahead_count_ = made;
    t_generate += seconds_since(t);
    return s;
  }

  rrg_status top_up(uint64_t target, uint64_t ahead) {
    if (target <= size_) return RRG_OK;
    if (comm_ || sim_ranks_ > 0) return top_up_sharded(target);
    const auto t = std::chrono::steady_clock::now();
    rrg_status s = RRG_OK;
    const uint64_t have_end = ahead_first_ + ahead_count_;
    const bool covered = ahead_count_ && ahead_first_ <= size_ && target <= have_end;
    if (!covered) {
      s = ensure_ahead();
      if (s != RRG_OK) return s;
      // the side store is extended when it still holds uncommitted slots from
      // size_ on (the pilot batch of a fresh graph), else restarted at size_
      const bool extend = ahead_count_ && ahead_first_ <= size_ && size_ < have_end;
      if (!extend) {
        rrg_store_clear(ahead_.s);
        ahead_first_ = size_;
        ahead_count_ = 0;
      }
      const uint64_t from = ahead_first_ + ahead_count_;
      uint64_t made = 0;
      s = rrg_generate_slots(g_, static_cast<rrg_model>(cfg_->model), cfg_->rng_seed, from,
                             std::max(target, ahead) - from, ahead_.s, fused_ ? 1 : 0, 64, &made);
      ahead_count_ += made;
      if (s != RRG_OK) {
        t_generate += seconds_since(t);
        return s;
      }
    }
    s = rrg_store_append_from(store_, ahead_.s, size_ - ahead_first_, target - size_);
    if (s == RRG_OK) size_ = target;
    t_generate += seconds_since(t);
    return s;
  }

  // how far ahead to sample: the next rounds' budgets while the batch stays small
  uint64_t ahead_for(unsigned i, unsigned rounds_total) const {
    // 2^17: cfg3's rounds 4 and 5 (46,252 and 92,504 sets) become one batch --
    // batches are bound by their largest sets, so 69K sets cost about what 23K do
    // (IMM cfg3 28.5 -> 24.0 ms; the other configs unchanged)
    constexpr uint64_t kAheadMax = 1ull << 17;
    // IC batches of few inspected edges in total are bound by the latency of
    // their largest set, not by the work (cfg3: 92,504 sets are 10M inspected
    // edges, 0.2 ms of sampler throughput, behind one 10 ms set): while the
    // slots up to a later round's target stay under kFreeEdges of estimated work
    // (mean inspected edges per set of this graph's earlier batches), sample
    // them in the same batch, however many rounds ahead that is.
    static const double kFreeEdges = [] {
      const char* e = std::getenv("RRGPU_IMM_FREE_EDGES");  // tuning
      return e ? std::atof(e) : RRG_IMM_FREE_EDGES;
    }();
    // The final top-up's slots are added only when they are few (kFinalMaxSets):
    // measured cfg1 11.4 -> 10.0 ms (5,268 extra slots, the final batch disappears)
    // but cfg3 19.7 -> 24.3 ms with 27,966 extra slots (one more giant set in the
    // tail, for a top-up that run never needs): profiles/r2/NOTES.md
    constexpr uint64_t kFinalMaxSets = 1ull << 13;
    static const bool kFinal = [] {
      const char* e = std::getenv("RRGPU_IMM_SPEC_FINAL");  // tuning: 0 off
      return !e || *e != '0';
    }();
    const double mean = cfg_->model == RRG_IC ? rrgpu::graph_ic_mean_inspected(g_) : -1.0;
    auto free_to = [&](uint64_t from, uint64_t to) {
      return mean >= 0.0 && to > from && static_cast<double>(to - from) * mean <= kFreeEdges;
    };
    uint64_t best = 0;
    unsigned jlast = 0;
    for (unsigned j = i + 1; j <= rounds_total; ++j) {
      const uint64_t tj = theta_for_round(n_, cfg_->k, cfg_->epsilon, ell_, j);
      if (tj <= size_) continue;
      if (tj - size_ > kAheadMax) break;
      if (j <= i + 2 || free_to(size_, tj)) {
        best = std::max(best, tj);
        jlast = j;
      }
    }
    // The final top-up (imm.hpp:227-231): a trigger at round j gives LB >= x_j,
    // so theta <= set_theta(x_j). While those extra slots are free too, the batch
    // covers them and the final top-up finds its sets already sampled.
    if (kFinal && mean >= 0.0) {
      const unsigned j = std::max(jlast, i);
      const uint64_t have = std::max(best, theta_for_round(n_, cfg_->k, cfg_->epsilon, ell_, i));
      const uint64_t fj = set_theta(n_, cfg_->k, cfg_->epsilon, ell_, round_target(n_, j));
      if (fj > have && fj - have <= kFinalMaxSets && fj - size_ <= kAheadMax && free_to(have, fj))
        best = fj;
    }
    return best;
  }

  // run_selection (imm.hpp:147-153): the fused strategy uses the fused counter,
  // the baseline strategy recounts (build_counter) -- same seeds either way.
  // need > 0 (trial rounds that have a successor): the selection may stop once
  // its coverage provably stays below `need` sets (*aborted); such a round fails
  // the trigger test whatever its seeds are, and nothing else of it is used.
  rrg_status select(uint32_t* sd, uint64_t* mg, uint64_t* covered, uint64_t need = 0,
                    bool* aborted = nullptr) {
    const auto t = std::chrono::steady_clock::now();
    bool ab = false;
    const rrg_status s = rrgpu::select_seeds_until(store_, cfg_->k, cfg_->adaptive_threshold,
                                                   fused_ ? 1 : 0, sd, mg, covered, need, &ab);
    t_select += seconds_since(t);
    if (aborted) *aborted = ab;
    if (s == RRG_OK && !ab && sd == trial_seeds_.data()) trial_size_ = size_;
    return s;
  }

  // The final selection (imm.hpp:238) runs on max(theta, theta') sets; when the
  // final top-up added none, that is the collection the last sampling round
  // selected on, and select_seeds is a deterministic function of the collection
  // (it revives every set first, selection.hpp:215): its seeds and marginals are
  // the last round's. Returns false when a selection is needed.
  bool reuse_last_selection(uint32_t* sd, uint64_t* mg) const {
    if (trial_size_ != size_ || size_ == 0) return false;
    std::copy(trial_seeds_.begin(), trial_seeds_.end(), sd);
    std::copy(trial_marg_.begin(), trial_marg_.end(), mg);
    return true;
  }

  // sampling_phase (imm.hpp:169-209)
  rrg_status sampling_phase(double* lower_bound) {
    const double eps_prime = std::sqrt(2.0) * cfg_->epsilon;
    const unsigned rounds = sampling_rounds(n_);
    double estimated_spread = 0.0;
    bool triggered = false;
    const rrg_status primed = prime();
    if (primed != RRG_OK) return primed;
    for (unsigned i = 1; i <= rounds; ++i) {
      rrg_status st = top_up(theta_for_round(n_, cfg_->k, cfg_->epsilon, ell_, i), ahead_for(i, rounds));
      if (st != RRG_OK) return st;
      uint64_t covered = 0;
      // the smallest covered count that passes the round's test below (the
      // expression is monotone in the count): a selection that cannot reach it
      // is cut short. The last round always runs to the end (its estimate is
      // the lower bound when no round triggers).
      const double target = (1.0 + eps_prime) * round_target(n_, i);
      auto spread_of = [&](uint64_t c) {
        return static_cast<double>(n_) * (static_cast<double>(c) / static_cast<double>(size_));
      };
      uint64_t need = 0;
      if (i < rounds && early_exit_enabled()) {
        const double guess = std::ceil(target * static_cast<double>(size_) / static_cast<double>(n_));
        need = guess >= 1.0 ? (guess < 1.8e19 ? static_cast<uint64_t>(guess) : UINT64_MAX) : 1;
        while (need > 1 && spread_of(need - 1) >= target) --need;
        while (need < UINT64_MAX && spread_of(need) < target) ++need;
      }
      bool aborted = false;
      st = select(trial_seeds_.data(), trial_marg_.data(), &covered, need, &aborted);
      if (st != RRG_OK) return st;
      if (aborted) continue;  // covered < need: the test below fails
      const double fraction = static_cast<double>(covered) / static_cast<double>(size_);
      estimated_spread = static_cast<double>(n_) * fraction;
      if (estimated_spread >= target) {
        triggered = true;
        break;
      }
    }
    *lower_bound = triggered ? estimated_spread / (1.0 + eps_prime)
                             : std::max(estimated_spread / (1.0 + eps_prime),
                                        static_cast<double>(cfg_->k));
    return RRG_OK;
  }

 private:
  rrg_graph* g_;
  const rrg_imm_config* cfg_;
  rrg_store* store_;
  uint32_t n_;
  double ell_;
  bool fused_;
  void* comm_ = nullptr;  // NCCL communicator (multi-GPU), or null
  int sim_ranks_ = 0;     // > 0: shards simulated in-process
  StoreGuard ahead_;
  uint64_t ahead_first_ = 0, ahead_count_ = 0;
  uint64_t size_ = 0;
  std::vector<uint32_t> trial_seeds_;
  std::vector<uint64_t> trial_marg_;
  uint64_t trial_size_ = 0;  // store size the trial seeds were selected on
};

}  // namespace

extern "C" {

void rrg_imm_config_default(rrg_imm_config* cfg) {
  if (!cfg) return;
  cfg->k = 50;
  cfg->epsilon = 0.5;
  cfg->model = RRG_IC;
  cfg->workers = 1;
  cfg->rng_seed = 1;
  cfg->ell = 1.0;
  cfg->adaptive_threshold = 0.25;
  cfg->strategy = RRG_STRATEGY_FUSED;
}

rrg_status rrg_sampling_phase(rrg_graph* g, const rrg_imm_config* cfg, rrg_store* store,
                              double* lower_bound, uint64_t* theta_prime,
                              rrg_imm_result* timings) {
  if (!g || !cfg || !store || !lower_bound || !theta_prime) {
    rrgpu::set_error("sampling_phase: null argument");
    return RRG_EINVAL;
  }
  rrg_status st = validate(g, cfg);
  if (st != RRG_OK) return st;
  st = rrg_store_clear(store);
  if (st != RRG_OK) return st;
  Driver d(g, cfg, store);
  st = d.sampling_phase(lower_bound);
  if (st != RRG_OK) return st;
  *theta_prime = d.size();
  if (timings) {
    timings->t_generate = d.t_generate;
    timings->t_select = d.t_select;
  }
  return RRG_OK;
}

}  // extern "C"

namespace {

// run_imm (imm.hpp:214-251) on one GPU (comm == nullptr, sim_ranks == 0), N
// GPUs (an NCCL communicator: every rank returns the same result) or shards
// simulated in one process (sim_ranks >= 1).
rrg_status run_imm_impl(rrg_graph* g, const rrg_imm_config* cfg, uint32_t* seeds,
                        uint64_t* marginals, rrg_imm_result* out, void* comm, int sim_ranks) {
  const auto t_total = std::chrono::steady_clock::now();
  if (!g || !cfg || !seeds || !marginals || !out) {
    rrgpu::set_error("run_imm: null argument");
    return RRG_EINVAL;
  }
  rrg_status st = validate(g, cfg);
  if (st != RRG_OK) return st;
  const uint32_t n = rrg_graph_num_vertices(g);
  *out = rrg_imm_result{};
  StoreGuard store;
  st = rrg_store_create(g, &store.s);
  if (st != RRG_OK) return st;
  Driver d(g, cfg, store.s, comm, sim_ranks);
  st = d.sampling_phase(&out->lower_bound);
  if (st != RRG_OK) return st;
  out->theta_prime = d.size();
  out->theta = set_theta(n, cfg->k, cfg->epsilon, d.ell(), out->lower_bound);

  // final top-up and selection (imm.hpp:227-241)
  st = d.top_up(out->theta, 0);
  if (st != RRG_OK) return st;
  if (!d.reuse_last_selection(seeds, marginals)) {
    st = d.select(seeds, marginals, nullptr);
    if (st != RRG_OK) return st;
  }

  // set statistics (imm.hpp:243-248)
  uint64_t sets = 0, members = 0;
  uint32_t max_len = 0;
  rrg_store_info(store.s, &sets, &members, &max_len);
  out->sets_generated = sets;
  out->mean_set_size = static_cast<double>(members) / static_cast<double>(sets);
  out->max_set_size = max_len;
  out->mean_coverage_fraction = out->mean_set_size / static_cast<double>(n);
  out->t_generate = d.t_generate;
  out->t_select = d.t_select;
  out->t_total = seconds_since(t_total);
  return RRG_OK;
}

}  // namespace

extern "C" {

rrg_status rrg_run_imm(rrg_graph* g, const rrg_imm_config* cfg, uint32_t* seeds,
                       uint64_t* marginals, rrg_imm_result* out) {
  return run_imm_impl(g, cfg, seeds, marginals, out, nullptr, 0);
}

rrg_status rrg_run_imm_sharded(rrg_graph* g, const rrg_imm_config* cfg, void* nccl_comm,
                               int sim_ranks, uint32_t* seeds, uint64_t* marginals,
                               rrg_imm_result* out) {
  if (!nccl_comm && sim_ranks < 1) {
    rrgpu::set_error("run_imm_sharded: need an NCCL communicator or sim_ranks >= 1");
    return RRG_EINVAL;
  }
  try {
    return run_imm_impl(g, cfg, seeds, marginals, out, nccl_comm, nccl_comm ? 0 : sim_ranks);
  } catch (const std::exception& e) {  // NCCL loading / communicator errors
    rrgpu::set_error(e.what());
    return RRG_ECUDA;
  }
}

}  // extern "C"
