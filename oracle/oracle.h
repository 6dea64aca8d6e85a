/*
 * oracle.h -- C ABI of the CPU checkers. TEST INFRASTRUCTURE ONLY.
 *
 * Two shared libraries export this identical API:
 *   oracle/liboracle_port.so     -- oracle/port.cpp, a C++17 restatement of the
 *                                   reference algorithm (kind "port");
 *   oracle/_ref/librrflow_ref.so -- oracle/ref_shim.cpp, the UNMODIFIED reference
 *                                   headers of /root/reference/proj/include compiled
 *                                   by include path (kind "reference").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load either library. The product path
 * (paper_2411_09473_b200/) never links or calls them.
 *
 * Graphs are passed as the reference's transpose CSR (graph.hpp:45-47):
 * reverse_offsets u64[n+1], reverse_sources u32[m], reverse_weights f32[m].
 */
#ifndef RRGPU_ORACLE_H
#define RRGPU_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_graph orc_graph;
typedef struct orc_store orc_store;

typedef struct {
  uint32_t k;
  double epsilon;
  int model; /* 0 = IC, 1 = LT */
  uint32_t workers;
  uint64_t rng_seed;
  double ell;
  double adaptive_threshold;
  int strategy; /* 0 = fused, 1 = baseline (imm.hpp:15-24) */
} orc_imm_config;

typedef struct {
  uint64_t theta;
  uint64_t theta_prime;
  double lower_bound;
  uint64_t sets_generated;
  double mean_set_size;
  uint32_t max_set_size;
  double mean_coverage_fraction;
  double t_generate;
  double t_select;
  double t_total;
} orc_imm_result;

const char* orc_kind(void);
const char* orc_last_error(void);

/* graph handle (arrays are copied) */
orc_graph* orc_graph_new(uint32_t n, uint64_t m, const uint64_t* roff,
                         const uint32_t* rsrc, const float* rw);
void orc_graph_free(orc_graph* g);

/* PRNG known-answer helpers (prng.hpp) */
uint64_t orc_derive_stream_seed(uint64_t run_seed, uint64_t stream);
void orc_prng_draws(uint64_t seed, uint64_t count, uint64_t* out);
uint64_t orc_uniform_below(uint64_t seed, uint64_t bound, double* next_uniform01);

/* sampling of slots [first_slot, first_slot + count), fused counter */
orc_store* orc_sample(orc_graph* g, int model, uint64_t run_seed, uint64_t first_slot,
                      uint64_t count, uint32_t workers);
uint64_t orc_store_sets(const orc_store* s);
uint64_t orc_store_members(const orc_store* s);
/* offsets u64[sets+1]; members sorted ascending within each set */
void orc_store_export(const orc_store* s, uint64_t* offsets, uint32_t* members);
void orc_store_counter(const orc_store* s, uint64_t* counts);
void orc_store_roots(const orc_store* s, uint32_t* roots);
/* reference-equivalent inspected in-edges (port only; the reference returns UINT64_MAX) */
uint64_t orc_store_inspected(const orc_store* s);
void orc_store_free(orc_store* s);

/* select_seeds over literal lists (selection.hpp:209-243); round_counters may be NULL,
 * else u64[k*n] per-round counter snapshots. Returns 0, or -1 with orc_last_error(). */
int orc_select(uint32_t n, uint64_t nsets, const uint64_t* offsets, const uint32_t* members,
               uint32_t k, double threshold, uint32_t workers, uint32_t* seeds,
               uint64_t* marginals, uint64_t* round_counters, uint32_t* rounds_done);

/* run_imm (imm.hpp:214-251). seeds u32[k], marginals u64[k]. */
int orc_imm(orc_graph* g, const orc_imm_config* cfg, uint32_t* seeds, uint64_t* marginals,
            orc_imm_result* out);
/* sampling_phase (imm.hpp:169-209): lower_bound, theta_prime and the phase's
 * counter u64[n] (zeros under the baseline strategy, which samples unfused) */
int orc_sampling_phase(orc_graph* g, const orc_imm_config* cfg, double* lower_bound,
                       uint64_t* theta_prime, uint64_t* counter);

/* theta math (imm.hpp:57-120) */
double orc_log_binomial(uint64_t n, uint64_t k);
double orc_effective_ell(double ell, uint64_t n);
double orc_lambda_prime(uint64_t n, uint64_t k, double eps, double ell);
uint32_t orc_sampling_rounds(uint64_t n);
uint64_t orc_theta_for_round(uint64_t n, uint64_t k, double eps, double ell, uint32_t i);
double orc_lambda_star(uint64_t n, uint64_t k, double eps, double ell);
uint64_t orc_set_theta(uint64_t n, uint64_t k, double eps, double ell, double lb);

/* graph preparation (graph.hpp:69-115, 207-235) */
int orc_build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                    const float* w, uint64_t* roff, uint32_t* rsrc, float* rw);
int orc_normalize_lt(uint32_t n, const uint64_t* roff, float* rw);

/* forward-simulation ground truth (oracle.hpp; reference library only, port returns -1) */
double orc_activation_probability(orc_graph* g, const uint32_t* sources, uint32_t nsrc,
                                  uint32_t target, int model, uint64_t trials, uint64_t seed);
double orc_exact_spread(orc_graph* g, const uint32_t* seeds, uint32_t k, int model);
/* reference synthetic graphs (graph.hpp:245-306); returns m, arrays may be NULL to query */
uint64_t orc_synth_graph(int kind, uint32_t n, double param, uint64_t seed, int ic_weights_seed_valid,
                         uint64_t ic_weights_seed, uint64_t* roff, uint32_t* rsrc, float* rw);

#ifdef __cplusplus
}
#endif

#endif
