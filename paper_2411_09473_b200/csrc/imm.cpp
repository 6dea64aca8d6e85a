// imm.cpp -- the IMM driver (host C++17). Re-expresses imm.hpp:57-251 with the
// same expression order and libm calls, so theta, theta', LB and the seeds are
// bit-identical to the reference; every sampling and selection call goes through
// the C ABI into the device (rrg_generate_batch / rrg_select_seeds). Between
// rounds only the scalar coverage crosses back to the host (imm.hpp:194-201).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rrgpu.h"

namespace rrgpu {
void set_error(const std::string& msg);
}

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

double seconds_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

struct StoreGuard {
  rrg_store* s = nullptr;
  ~StoreGuard() { rrg_store_destroy(s); }
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
}

// run_imm (imm.hpp:214-251) + sampling_phase (imm.hpp:169-209), fused strategy.
rrg_status rrg_run_imm(rrg_graph* g, const rrg_imm_config* cfg, uint32_t* seeds,
                       uint64_t* marginals, rrg_imm_result* out) {
  const auto t_total = std::chrono::steady_clock::now();
  if (!g || !cfg || !seeds || !marginals || !out) {
    rrgpu::set_error("run_imm: null argument");
    return RRG_EINVAL;
  }
  // validate_config (imm.hpp:136-145)
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
  const rrg_model model = static_cast<rrg_model>(cfg->model);
  *out = rrg_imm_result{};
  const double ell = effective_ell(cfg->ell, n);
  const double eps_prime = std::sqrt(2.0) * cfg->epsilon;

  StoreGuard store;
  rrg_status st = rrg_store_create(g, &store.s);
  if (st != RRG_OK) return st;

  // Top-ups. Slot j's set depends only on (rng_seed, j) (sampling.hpp:179), so
  // sets for slots a later round may need can be sampled ahead into a side
  // store and committed only when (and if) a top-up reaches them: the main
  // store ends up with exactly the reference's sets. Small batches are bound by
  // the latency of their largest set, so one batch covering the next rounds
  // costs about what one round's batch does.
  StoreGuard ahead_store;
  uint64_t ahead_first = 0, ahead_count = 0;
  uint64_t size = 0;
  auto top_up = [&](uint64_t target, uint64_t ahead) -> rrg_status {
    if (target <= size) return RRG_OK;
    const auto t = std::chrono::steady_clock::now();
    rrg_status s = RRG_OK;
    const bool covered = ahead_count && ahead_first <= size && target <= ahead_first + ahead_count;
    if (!covered) {
      if (!ahead_store.s) {
        s = rrg_store_create(g, &ahead_store.s);
        if (s != RRG_OK) return s;
      } else {
        rrg_store_clear(ahead_store.s);
      }
      const uint64_t want = std::max(target, ahead) - size;
      uint64_t made = 0;
      s = rrg_generate_slots(g, model, cfg->rng_seed, size, want, ahead_store.s, /*fused=*/0, 64,
                             &made);
      ahead_first = size;
      ahead_count = made;
      if (s != RRG_OK) {
        out->t_generate += seconds_since(t);
        return s;
      }
    }
    s = rrg_store_append_from(store.s, ahead_store.s, size - ahead_first, target - size);
    if (s == RRG_OK) size = target;
    out->t_generate += seconds_since(t);
    return s;
  };
  // how far ahead to sample: the next rounds' budgets while the batch stays small
  constexpr uint64_t kAheadMax = 1ull << 16;
  auto ahead_for = [&](unsigned i, unsigned rounds_total) -> uint64_t {
    uint64_t best = 0;
    for (unsigned j = i + 1; j <= std::min(rounds_total, i + 2); ++j) {
      const uint64_t tj = theta_for_round(n, cfg->k, cfg->epsilon, ell, j);
      if (tj > size && tj - size <= kAheadMax) best = std::max(best, tj);
    }
    return best;
  };
  std::vector<uint32_t> trial_seeds(cfg->k);
  std::vector<uint64_t> trial_marg(cfg->k);
  auto select = [&](uint32_t* sd, uint64_t* mg, uint64_t* covered) -> rrg_status {
    const auto t = std::chrono::steady_clock::now();
    const rrg_status s = rrg_select_seeds(store.s, cfg->k, cfg->adaptive_threshold,
                                          /*use_prebuilt=*/1, sd, mg, nullptr, nullptr, covered);
    out->t_select += seconds_since(t);
    return s;
  };

  // sampling phase: top up to theta_i, trial selection, stop once the estimate
  // certifies the round target (imm.hpp:182-206)
  const unsigned rounds = sampling_rounds(n);
  double estimated_spread = 0.0;
  bool triggered = false;
  for (unsigned i = 1; i <= rounds; ++i) {
    st = top_up(theta_for_round(n, cfg->k, cfg->epsilon, ell, i), ahead_for(i, rounds));
    if (st != RRG_OK) return st;
    uint64_t covered = 0;
    st = select(trial_seeds.data(), trial_marg.data(), &covered);
    if (st != RRG_OK) return st;
    const double fraction = static_cast<double>(covered) / static_cast<double>(size);
    estimated_spread = static_cast<double>(n) * fraction;
    if (estimated_spread >= (1.0 + eps_prime) * round_target(n, i)) {
      triggered = true;
      break;
    }
  }
  out->lower_bound = triggered ? estimated_spread / (1.0 + eps_prime)
                               : std::max(estimated_spread / (1.0 + eps_prime),
                                          static_cast<double>(cfg->k));
  out->theta_prime = size;
  out->theta = set_theta(n, cfg->k, cfg->epsilon, ell, out->lower_bound);

  // final top-up and selection (imm.hpp:227-241)
  st = top_up(out->theta, 0);
  if (st != RRG_OK) return st;
  st = select(seeds, marginals, nullptr);
  if (st != RRG_OK) return st;

  // set statistics (imm.hpp:243-248)
  uint64_t sets = 0, members = 0;
  uint32_t max_len = 0;
  rrg_store_info(store.s, &sets, &members, &max_len);
  out->sets_generated = sets;
  out->mean_set_size = static_cast<double>(members) / static_cast<double>(sets);
  out->max_set_size = max_len;
  out->mean_coverage_fraction = out->mean_set_size / static_cast<double>(n);
  out->t_total = seconds_since(t_total);
  return RRG_OK;
}

}  // extern "C"
