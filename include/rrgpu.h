/*
 * rrgpu.h -- C ABI of the B200-native IMM hot path (librrgpu.so).
 *
 * Drop-in boundary for the reference rrflow 0.1.0 (/root/reference/proj/include/rrflow).
 * The reference has no FFI; its operator API is a set of free C++ functions.
 * Each entry point below replaces one of them (file:line cited per symbol) with the
 * same argument meaning, slot/stream semantics, side effects and error classes:
 *   RRG_EINVAL <-> std::invalid_argument, RRG_ENOMEM <-> BatchOutOfMemory /
 *   std::bad_alloc, RRG_ECUDA <-> std::runtime_error. Messages via rrg_last_error().
 * The C++17 adapter include/rrgpu/rrgpu.hpp maps these back onto exceptions and
 * reference-shaped types; INTEGRATION.md shows the caller-side switch.
 *
 * All calls are synchronous at return (the reference's WorkPool barrier semantics,
 * work_pool.hpp:14-19). Host arrays are borrowed for the duration of a call.
 * A graph and the stores created on it are NOT thread-safe (one orchestrator
 * thread, as SPEC.md:420 states for the reference driver).
 */
#ifndef RRGPU_H
#define RRGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { RRG_OK = 0, RRG_EINVAL = 1, RRG_ENOMEM = 2, RRG_ECUDA = 3 } rrg_status;

/* rrflow::DiffusionModel (graph.hpp:19) */
typedef enum { RRG_IC = 0, RRG_LT = 1 } rrg_model;

typedef struct rrg_graph rrg_graph; /* device-resident transpose CSR (rrflow::Graph, graph.hpp:34-59) */
typedef struct rrg_store rrg_store; /* RRRStore + fused Counter (rrr_store.hpp:20-120, counter.hpp:15-62) */

/* ---- graph ---------------------------------------------------------------
 * Replaces the transpose view of rrflow::Graph (graph.hpp:45-47): reverse_offsets
 * u64[n+1], reverse_sources u32[m], reverse_weights f32[m], in the reference's
 * in-list order (graph.hpp:96-113), which is the draw order. m must be < 2^32.
 * n == 0 is accepted here; sampling on it fails like generate_batch (sampling.hpp:165). */
rrg_status rrg_graph_create(uint32_t n, uint64_t m, const uint64_t* rev_offsets,
                            const uint32_t* rev_sources, const float* rev_weights,
                            rrg_graph** out);
/* Frees the graph; while stores of it are alive it is only marked, and the last
 * rrg_store_destroy frees it (destruction order is the caller's choice). */
void rrg_graph_destroy(rrg_graph* g);
/* Builds the per-model device layout up front (otherwise done on first use):
 * IC -> interleaved {source, weight} records; LT -> sequential fp64 CDF (K0). */
rrg_status rrg_graph_prepare(rrg_graph* g, rrg_model model);
/* Runs every subsequent call of this graph and its stores on `cuda_stream`
 * (a cudaStream_t; NULL restores the graph's private stream). */
/* rrg_graph_create with the diffusion model the graph will be sampled under
 * (RRG_IC, RRG_LT, or -1 = unknown: exactly rrg_graph_create). With RRG_LT the
 * weight-only LT layouts (the exact sequential fp64 CDF, sampling.hpp:130-136)
 * are built on the device while the sources are still being uploaded; results
 * are identical, only the time from host arrays to the first batch changes (and
 * the LT layouts -- 8 B per in-edge of CDF, 16 B of lite guide table -- are
 * resident from creation on, also if the graph is then only sampled under IC). */
rrg_status rrg_graph_create_for(uint32_t n, uint64_t m, const uint64_t* rev_offsets,
                                const uint32_t* rev_sources, const float* rev_weights,
                                int model_hint, rrg_graph** out);
/* On-device graph preparation: uploads an edge list
 * (src[i] -> dst[i], weight w[i]) and builds the transpose on the device in the
 * in-list order of detail::build_graph (graph.hpp:69-115: sources ascending,
 * parallel edges in input order), then, if normalize_lt != 0, applies
 * normalize_lt_weights (graph.hpp:207-235) to it -- bit-identical to
 * rrg_build_transpose + rrg_normalize_lt_weights + rrg_graph_create. Errors:
 * RRG_EINVAL for an id >= n or (normalize) a negative weight, like the
 * reference's std::runtime_error. m < 2^31. */
rrg_status rrg_graph_create_from_edges(uint32_t n, uint64_t m, const uint32_t* src,
                                       const uint32_t* dst, const float* w, int normalize_lt,
                                       rrg_graph** out);
/* The device transpose back on the host: roff u64[n+1], rsrc u32[m], rw f32[m]. */
rrg_status rrg_graph_export_transpose(const rrg_graph* g, uint64_t* roff, uint32_t* rsrc,
                                      float* rw);
rrg_status rrg_graph_set_stream(rrg_graph* g, void* cuda_stream);
uint32_t rrg_graph_num_vertices(const rrg_graph* g);
uint64_t rrg_graph_num_edges(const rrg_graph* g);

/* Tuning knobs; none changes any output bit. */
typedef enum {
  RRG_OPT_LT_SCAN = 0,  /* 0 = linear CDF scan (reference trip count), 1 = search tree
                           (picks the identical index in ~log32(deg) node loads), 2 = guide
                           table (default; identical index, one 32-byte load per step;
                           falls back to 1 when the table does not fit in free HBM) */
  RRG_OPT_LT_COOP_MIN = 1, /* in-list length from which LT scans go warp-cooperative */
  RRG_OPT_IC_INNER = 2, /* IC edge steps per scheduling round (1..64) */
  RRG_OPT_IC_COOP_MIN = 3, /* IC in-list length from which the warp expands it cooperatively
                             (GF(2) jump-ahead segments); UINT32_MAX disables */
  RRG_OPT_LT_KARY = 4,  /* arity of the LT CDF search: 2, 4, 8 or 16 (default 8) */
  RRG_OPT_IC_MODE = 5,  /* IC schedule: 0 auto (pilot-measured), 1 lane per sample,
                           2 warp per sample, 3 thread block per sample */
  RRG_OPT_IC_WARP_MIN_INSP = 6, /* auto: warp per sample once the mean inspected
                                   in-edges per set reaches this value */
  RRG_OPT_IC_RNG = 7 /* IC randomness: 0 (default) the reference's per-slot stream,
                        sets bit-identical; 1 FAST: counter-based per-edge draws with
                        geometric skipping over equal-weight in-lists -- same set
                        distribution, statistical parity only */,
  RRG_OPT_LT_GUIDE_MULT = 8, /* LT guide buckets per in-edge, 1..16 (default 4; table =
                               32 B x mult x m; larger = fewer multi-entry buckets) */
  RRG_OPT_IC_WARP_BUDGET = 9 /* IC warp schedule: 512-edge windows a set may take before it
                                is handed to the block schedule (0 = no budget) */
} rrg_option;
rrg_status rrg_graph_set_option(rrg_graph* g, rrg_option opt, int64_t value);

/* ---- store -------------------------------------------------------------- */
rrg_status rrg_store_create(rrg_graph* g, rrg_store** out);
void rrg_store_destroy(rrg_store* s);
/* Drops every set and zeroes the fused counter. */
rrg_status rrg_store_clear(rrg_store* s);
/* RRRStore::size / total_member_count / max_set_size (rrr_store.hpp:29, :100-110) */
rrg_status rrg_store_info(const rrg_store* s, uint64_t* sets, uint64_t* members,
                          uint32_t* max_set_size);

/* RRRStore::live_count (rrr_store.hpp:84): sets not covered by the last
 * rrg_select_seeds (the store stays tombstoned, imm.hpp:194-195); every append
 * (generate_batch, import, append_from) revives all sets, as finalize does. */
rrg_status rrg_store_live_count(const rrg_store* s, uint64_t* live);
/* RRRStore::is_live (rrr_store.hpp:62) for sets [first, first+count): out u8[count]. */
rrg_status rrg_store_live_flags(const rrg_store* s, uint64_t first, uint64_t count, uint8_t* out);
/* Replaces the store's occurrence counter with a caller-held tally u64[n] (each
 * < 2^32): the `prebuilt` Counter of select_seeds (selection.hpp:209-218). */
rrg_status rrg_store_set_counter(rrg_store* s, const uint64_t* counts);
/* A budget for the store: a batch chunk that would take it past max_members
 * members fails with RRG_ENOMEM; the sets of earlier chunks stay, the fused
 * counter matches them, *sets_generated counts them (BatchOutOfMemory,
 * sampling.hpp:148-154). 0: no limit (device allocation failures behave alike). */
rrg_status rrg_store_set_member_limit(rrg_store* s, uint64_t max_members);

/* The dense arm (rrr_set.hpp:10-13, :73-90): sets of >= n / density_divisor
 * members are held as n-bit maps (rows), the rest as id lists. *dense_sets rows
 * holding *dense_members members in *dense_bytes of HBM; *rebuild_rounds = rounds
 * of the last rrg_select_seeds on this store that rebuilt the counter from the
 * surviving sets (rebuild_update, selection.hpp:161-203). Any pointer may be NULL. */
rrg_status rrg_store_dense_info(const rrg_store* s, uint64_t* dense_sets,
                                uint64_t* dense_members, uint64_t* dense_bytes,
                                uint64_t* rebuild_rounds);

/* ---- sampling: generate_batch (sampling.hpp:159-199) --------------------
 * Appends exactly `count` sets at slots [size, size+count); set j is sampled from
 * stream derive_stream_seed(run_seed, j) (sampling.hpp:179, prng.hpp:17-20), so the
 * sets are bit-identical to the reference's. fused != 0 adds every member to the
 * store's occurrence counter (sampling.hpp:184-186). density_divisor selects the
 * in-memory representation exactly as the reference's make_repr / pack_sketch
 * (rrr_set.hpp:73-90, sampling.hpp:68-84): a set of >= n / density_divisor members
 * is an n-bit map row (0: never); exports list every set either way (root first,
 * a row's other members ascending). On RRG_ENOMEM, *sets_generated holds
 * the number of sets that were appended (BatchOutOfMemory, sampling.hpp:148-154). */
rrg_status rrg_generate_batch(rrg_graph* g, rrg_model model, uint64_t run_seed, uint64_t count,
                              rrg_store* s, int fused, uint32_t density_divisor,
                              uint64_t* sets_generated);

/* Same, but the appended sets come from streams [first_slot, first_slot+count)
 * instead of [size, size+count): one shard of a slot range split across GPUs
 * (slot j depends only on (run_seed, j), sampling.hpp:179). */
rrg_status rrg_generate_slots(rrg_graph* g, rrg_model model, uint64_t run_seed,
                              uint64_t first_slot, uint64_t count, rrg_store* s, int fused,
                              uint32_t density_divisor, uint64_t* sets_generated);

/* Per-call counters of the last rrg_generate_batch on this graph. */
typedef struct {
  uint64_t sets;               /* sets appended */
  uint64_t members;            /* members appended */
  uint64_t edges_inspected;    /* reference-equivalent in-edges inspected */
  uint64_t entries_read;       /* adjacency entries the kernels actually loaded */
  uint64_t deferred;           /* sets routed to the big-set path */
  float sample_ms;             /* device time of the sampler kernels (CUDA events) */
  float total_ms;              /* device time of the whole call incl. compaction */
} rrg_batch_stats;
rrg_status rrg_last_batch_stats(const rrg_graph* g, rrg_batch_stats* out);

/* ---- selection: select_seeds (selection.hpp:209-243) ---------------------
 * k in [1, n] else RRG_EINVAL (:213-214). Revives every set first (:215). With
 * use_prebuilt the fused counter is the starting tally (:217-218), else it is
 * recounted (build_counter, :79-95). k greedy rounds run on the device with no host
 * round-trip: argmax with ties to the lowest id (:100-125), exhaustion fill with the
 * lowest unselected ids at zero gain (:61-72), decrement through an on-device
 * inverted index (:130-156), or -- when the round's seed covers more than
 * adaptive_threshold of the live sets -- a rebuild of the counter from the
 * surviving sets (rebuild_update, :161-203; the same rule, :226-231). Both give
 * the same counts (test_selection.cpp:116-137). Dense rows are tested bit by bit
 * and counted by column sums.
 * seeds u32[k], marginals u64[k]; round_counters (nullable) u64[k*n] receives the
 * per-round counter snapshots (SelectionStats::capture_round_counters, :237-239).
 * *rounds_done (nullable) = rounds that produced a snapshot. The store stays
 * tombstoned: *covered_total (nullable) = size - live_count (imm.hpp:194-195). */
rrg_status rrg_select_seeds(rrg_store* s, uint32_t k, double adaptive_threshold, int use_prebuilt,
                            uint32_t* seeds, uint64_t* marginals, uint64_t* round_counters,
                            uint32_t* rounds_done, uint64_t* covered_total);

/* fraction_covered (selection.hpp:340-358) */
rrg_status rrg_fraction_covered(rrg_store* s, const uint32_t* seeds, uint32_t nseeds,
                                double* out);

/* ---- IMM driver: run_imm (imm.hpp:214-251) -------------------------------- */
typedef struct {
  uint32_t k;                 /* ImmConfig defaults (imm.hpp:27-36): 50 */
  double epsilon;             /* 0.5 */
  int model;                  /* RRG_IC */
  uint32_t workers;           /* 1; validated (>= 1) but the device ignores it */
  uint64_t rng_seed;          /* 1 */
  double ell;                 /* 1.0 */
  double adaptive_threshold;  /* 0.25 */
  int strategy;               /* RRG_STRATEGY_FUSED (Strategy::fused, imm.hpp:33); BASELINE =
                                 unfused sampling + recount before each selection: the
                                 reference's baseline_select returns the same seeds and
                                 marginals (test_selection.cpp:188-200), so the device
                                 runs its one selection on both */
} rrg_imm_config;
enum { RRG_STRATEGY_FUSED = 0, RRG_STRATEGY_BASELINE = 1 };

typedef struct {
  uint64_t theta;
  uint64_t theta_prime;
  double lower_bound;
  uint64_t sets_generated;
  double mean_set_size;
  uint32_t max_set_size;
  double mean_coverage_fraction;
  double t_generate;          /* ImmTimings (imm.hpp:38-42), seconds */
  double t_select;
  double t_total;
} rrg_imm_result;

void rrg_imm_config_default(rrg_imm_config* cfg);
/* seeds u32[k], marginals u64[k] */
rrg_status rrg_run_imm(rrg_graph* g, const rrg_imm_config* cfg, uint32_t* seeds,
                       uint64_t* marginals, rrg_imm_result* out);
/* sampling_phase (imm.hpp:169-209): rounds of top-ups + trial selections into
 * `store` (cleared first) until the estimate certifies the round target.
 * Outputs SamplingPhaseResult's lower_bound and theta_prime (= store size; the
 * store's counter is the phase's fused Counter); `timings` (nullable) receives
 * t_generate / t_select. */
rrg_status rrg_sampling_phase(rrg_graph* g, const rrg_imm_config* cfg, rrg_store* store,
                              double* lower_bound, uint64_t* theta_prime,
                              rrg_imm_result* timings);

/* ---- multi-GPU IMM ----------------------------------------
 * One process per GPU sharing an NCCL communicator (NCCL is loaded at first use:
 * libnccl.so.2). rrg_nccl_unique_id on one rank, the 128 bytes passed to every
 * rank (e.g. over torch.distributed), rrg_nccl_comm_create on each with the
 * rank's device current. rrg_run_imm_sharded: every top-up's new slots are split
 * into nranks contiguous shards, rank r samples shard r with no communication
 * (slot j depends only on (run_seed, j), sampling.hpp:179), the shards' device
 * buffers are broadcast over NCCL and appended in slot order on every rank; the
 * selection runs replicated. Every rank returns the result of rrg_run_imm.
 * nccl_comm == NULL with sim_ranks >= 1: the same shard split and ordered
 * assembly in one process (no transport; parity of the sharding). */
rrg_status rrg_nccl_unique_id(uint8_t* id /* [128] */);
rrg_status rrg_nccl_comm_create(const uint8_t* id, int nranks, int rank, void** comm);
void rrg_nccl_comm_destroy(void* comm);
rrg_status rrg_run_imm_sharded(rrg_graph* g, const rrg_imm_config* cfg, void* nccl_comm,
                               int sim_ranks, uint32_t* seeds, uint64_t* marginals,
                               rrg_imm_result* out);

/* ---- parity / interop --------------------------------------------------- */
/* Copies sets [first, first+count) to the host: offsets u64[count+1] (relative to
 * the first set), members in visit order (root first, sampling.hpp:93-94). */
rrg_status rrg_store_export(const rrg_store* s, uint64_t first, uint64_t count, uint64_t* offsets,
                            uint32_t* members);
/* Appends literal sets (e.g. the oracle's), updating the fused counter. */
rrg_status rrg_store_import(rrg_store* s, uint64_t count, const uint64_t* offsets,
                            const uint32_t* members);
/* Appends sets [first, first+count) of `src` to `dst` (device to device, same graph),
 * adding them to dst's fused counter. Slot j's set depends only on (run_seed, j), so
 * sets sampled ahead of need into a side store are exactly the sets a later top-up of
 * dst would draw for those slots (the IMM driver's speculative top-ups use this). */
rrg_status rrg_store_append_from(rrg_store* dst, const rrg_store* src, uint64_t first,
                                 uint64_t count);
/* Fused occurrence counter as u64[n] (Counter::get, counter.hpp:29). */
rrg_status rrg_store_counter(const rrg_store* s, uint64_t* counts);
/* Enqueues, on `stream` (a cudaStream_t), the device-to-host copies of the whole
 * store: offsets u64[nsets+1], members u32[total] and, if `counts` is non-null, the
 * counter as u64[n]; returns without waiting. Host buffers should be pinned. The
 * store must not be modified or destroyed until `stream` has completed. Lets a
 * caller overlap one batch's export with the next batch's sampling. */
rrg_status rrg_store_export_all_async(const rrg_store* s, uint64_t* offsets, uint32_t* members,
                                      uint64_t* counts, void* stream);
/* The same with 32-bit offsets and counts (offsets u32[nsets+1], counts u32[n]):
 * 7 % fewer bytes over PCIe for a store below 2^32 members (else RRG_EINVAL). */
rrg_status rrg_store_export_all_async32(const rrg_store* s, uint32_t* offsets, uint32_t* members,
                                        uint32_t* counts, void* stream);

/* ---- host-side graph preparation (plumbing that feeds both sides) ---------- */
/* detail::build_graph (graph.hpp:69-115): transpose of an edge list in the
 * reference's in-list order. roff u64[n+1], rsrc u32[m], rw f32[m]. */
rrg_status rrg_build_transpose(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                               const float* w, uint64_t* roff, uint32_t* rsrc, float* rw);
/* normalize_lt_weights (graph.hpp:207-235) on transpose weights, in place. */
rrg_status rrg_normalize_lt_weights(uint32_t n, const uint64_t* roff, float* rw);

/* ---- misc ------------------------------------------------------------------ */
const char* rrg_last_error(void);
const char* rrg_version(void);
/* Kernels this library has launched in the process so far (all graphs). */
uint64_t rrg_launch_count(void);
/* Host waits on the device (stream synchronizations) by this library so far. */
uint64_t rrg_host_sync_count(void);
/* Test hook: the integer Bernoulli threshold used by the IC kernel
 * (uniform01() < (double)w  <=>  (next_u64() >> 11) < threshold(w)). */
uint64_t rrg_debug_bernoulli_threshold(uint32_t weight_bits);
/* The 32-bit threshold stored in IC edge records: T >> 21, saturated at 2^32-1. */
uint32_t rrg_debug_bernoulli_thr_hi(uint32_t weight_bits);
/* Test hook: the LT running sums cdf[j] = acc after in-edge j (sampling.hpp:130-136:
 * acc = 0.0 per vertex, acc += (double)w[j] in CSR order) as the device built them;
 * f64[m]. Must equal the host's sequential sums bit for bit. */
rrg_status rrg_debug_export_lt_cdf(rrg_graph* g, double* cdf);
/* Test hook: advances a xoshiro256** state (4 words) by k draws with the GF(2)
 * jump matrices the IC hub expansion uses (csrc/jump.cpp). */
void rrg_debug_jump(const uint64_t* state_in, uint64_t k, uint64_t* state_out);

#ifdef __cplusplus
}
#endif

#endif /* RRGPU_H */
