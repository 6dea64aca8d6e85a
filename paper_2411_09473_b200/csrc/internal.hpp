// internal.hpp -- host-side context objects and kernel launchers (not exported).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rrgpu.h"
#include "common.cuh"

namespace rrgpu {

void set_error(const std::string& msg);

struct CudaError {
  cudaError_t err;
  std::string where;
};

#define RRG_CUDA(call)                                                   \
  do {                                                                   \
    cudaError_t e_ = (call);                                             \
    if (e_ != cudaSuccess) throw ::rrgpu::CudaError{e_, #call};          \
  } while (0)

// cudaStreamSynchronize + a process-wide count of host round trips (evidence of
// how often the host waits on the device per IMM run; rrg_host_sync_count).
void host_sync(cudaStream_t s);
uint64_t host_syncs();

// Process-wide caching allocator (per device): freed blocks are kept and reused
// for requests of 1/2..1x their size, so graph/store churn (the e2e path creates
// a graph per call) does not pay cudaMalloc/cudaFree every time.
void* pool_alloc(size_t bytes, size_t* granted);
void pool_free(void* p, size_t bytes);

// Owning device buffer, grow-only.
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) pool_free(ptr, bytes);
    ptr = nullptr;
    cap = 0;
    bytes = 0;
  }
  // Ensures capacity >= n elements; contents are NOT preserved.
  void reserve_discard(size_t n) {
    if (n <= cap) return;
    release();
    size_t got = 0;
    ptr = static_cast<T*>(pool_alloc(n * sizeof(T), &got));
    bytes = got;
    cap = got / sizeof(T);
  }
  // Ensures capacity >= n elements, preserving the first `keep` elements.
  void reserve_keep(size_t n, size_t keep, cudaStream_t s) {
    if (n <= cap) return;
    size_t got = 0;
    T* np = static_cast<T*>(pool_alloc(n * sizeof(T), &got));
    if (keep) RRG_CUDA(cudaMemcpyAsync(np, ptr, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    host_sync((s));
    release();
    ptr = np;
    bytes = got;
    cap = got / sizeof(T);
  }
};

enum LtScan : int { kLtLinear = 0, kLtBsearch = 1, kLtGuide = 2 };

// IC whole-list expansion (sample.cu): 32-edge chunks per lane of a sub-window
#ifndef RRG_LX_CPL
#define RRG_LX_CPL 1
#endif
constexpr uint32_t kLxWin = 1024u * RRG_LX_CPL;  // edges per list-expansion sub-window
#ifndef RRG_LIST_MIN
#define RRG_LIST_MIN 8192
#endif
constexpr uint32_t kListMin = RRG_LIST_MIN;  // in-lists at least this long are expanded whole

// Per-lane sampler scratch: visit-order list + tagged hash table + tag.
// Tagged tables are never cleared; that is sound because the region layouts
// draw tags from disjoint ranges: lane regions (IC lane mode, LT) use tags in
// [1, 2^31) from `tags`; warp regions of 32 lanes use [2^31, 3*2^30) and of 256
// lanes [3*2^30, 2^32), both counted in `wtags`. Zeroed memory matches none.
struct LaneScratch {
  uint64_t lanes = 0;
  DevBuf<uint32_t> lists;
  DevBuf<uint64_t> tabs;
  DevBuf<uint32_t> xhi;  // block IC schedule: a window's draw high words, per block (kCtaWin each)
  DevBuf<uint32_t> tags;
  DevBuf<uint32_t> wtags;
};

// Giant CTA schedule scratch (sample_ic.cu k_sample_ic_cta<true>): per block a
// list of kGiantCap members and an n-bit visited map.
struct GiantScratch {
  uint32_t ctas = 0;
  DevBuf<uint32_t> lists;
  DevBuf<uint32_t> bits;  // per block: an n-bit visited map, zero between sets
  DevBuf<uint32_t> tags;
};

// Big-set path scratch: one n-bit map and one n-entry list per worker warp.
struct BigScratch {
  uint32_t workers = 0;
  DevBuf<uint32_t> bitmaps;
  DevBuf<uint32_t> lists;
};

}  // namespace rrgpu

struct rrg_graph {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint32_t n = 0;
  uint64_t m = 0;
  rrgpu::DevBuf<uint32_t> off;   // u32[n+1] transpose offsets
  rrgpu::DevBuf<uint32_t> src;   // u32[m]   transpose sources (CSR order = draw order)
  rrgpu::DevBuf<float> w;        // f32[m]   transpose weights
  rrgpu::DevBuf<uint2> rec;      // IC: {source, weight bits} per in-edge (lazy)
  rrgpu::DevBuf<double> cdf;     // LT: sequential fp64 prefix per in-list (lazy, +2 pad)
  rrgpu::DevBuf<uint32_t> ltrec; // LT: 64-byte vertex records (k_build_ltrec), monotone CDF only
  rrgpu::DevBuf<uint64_t> ltnodeoff;  // LT: first search-tree slot per vertex (u64[n+1])
  rrgpu::DevBuf<uint32_t> ltnodes;    // LT: search-tree nodes, 32 floats (31 pivots) each
  rrgpu::DevBuf<uint4> ltguide;  // LT: guide table, 32 bytes per bucket (common.cuh), lazy
  rrgpu::DevBuf<uint2> ltlite;   // LT: lite guide table, 8 bytes per bucket (small batches before the full table)
  uint32_t lt_guide_mult = 4;    // LT: guide buckets per in-edge (4: 0.74 vs 0.85 ms at 2, cfg4 65K walks)
  uint32_t lt_guide_built = 0;   // multiplier the current table was built with (0: none)
  uint64_t lt_light_walks = 0;   // walks sampled on the lite guide table so far
  bool lt_guide_mult_explicit = false;  // set through RRG_OPT_LT_GUIDE_MULT: no light table
  bool lt_search_ready = false;  // LT: records + search trees built
  const uint64_t* jtab = nullptr;  // IC: byte tables of T^(32 l), l = 1..31 (7.75 MB)
  const uint64_t* jtab16 = nullptr;  // IC: byte tables of T^(16 l), l = 1..31 (7.75 MB)
  const uint64_t* jtab256 = nullptr;  // IC: byte tables of T^(256 a), a = 1..15 (3.75 MB)
  const uint64_t* jtabhi = nullptr;   // IC: byte tables of T^(16^k a), k = 3, 4, 5, a = 1..15 (11.25 MB)
  const uint64_t* jtab64 = nullptr;   // IC: byte tables of T^(kLxPer l), l = 1..31 (list expansion)
  uint32_t max_indeg = 0;           // IC: largest in-list (list-expansion scratch sizing)
  rrgpu::DevBuf<uint32_t> lx;       // IC: per-CTA list-expansion scratch (masks, counts)
  rrgpu::DevBuf<uint8_t> dupfree;  // IC: per-vertex strictly-increasing-sources flag
  rrgpu::DevBuf<uint8_t> uniformw; // IC fast mode: per-vertex "all in-weights equal" flag
  bool uniform_ready = false;
  int ic_rng = 0;                // IC: 0 the reference's stream (exact), 1 fast (statistical)
  uint32_t ic_coop_min = 256;    // IC: in-lists at least this long expand warp-cooperatively
  int ic_mode = 0;               // IC: 0 auto, 1 lane, 2 warp, 3 block per sample
  bool ic_giant = false;         // IC auto: run the block schedule over the giant scratch
  uint32_t ic_warp_budget = 0;   // IC: warp-schedule windows per set before the block pass (0: off)
  double ic_mean_insp = -1.0;    // IC: running mean of inspected in-edges per set
  double ic_hub_insp = 1e5;       // auto: warp per sample from this mean on (cfg5 ~1M)
  double ic_cta_max_edges = 1.0e8;  // auto: block per sample up to this many expected
                                    // inspected edges per batch (cfg1: the block schedule
                                    // wins up to ~18K sets = 1e8 edges -- 16,631 sets 6.65 vs
                                    // 7.2 ms -- the warp schedule beyond -- 21,899 sets 7.5
                                    // vs 8.0 ms, 66,523 sets 12.9 vs 20.5 ms)
  double ic_warp_min_insp = 1024.0;  // auto: warp per sample from this mean on (cfg1 5.5K
                                     // and cfg5 986K run faster per warp; cfg3 237 per lane)
  bool rec_ready = false;
  bool cdf_ready = false;
  bool cdf_monotone = true;
  int lt_scan = rrgpu::kLtGuide;  // guide table (falls back to the search tree, then linear)
  uint32_t coop_min = 64;        // LT: in-lists at least this long are scanned warp-cooperatively
  int lt_kary = 8;               // LT: arity of the CDF search (8 measured best at cfg4)
  uint32_t ic_inner = 8;         // IC: edge steps per flat-loop iteration
  rrgpu::LaneScratch scratch;
  rrgpu::BigScratch big;
  rrgpu::GiantScratch giant;
  rrgpu::DevBuf<rrgpu::SampleCtl> ctl;
  rrg_batch_stats last{};
  int nstores = 0;               // stores alive on this graph
  bool destroyed = false;        // rrg_graph_destroy ran while stores were alive
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

struct rrg_store {
  rrg_graph* g = nullptr;
  uint64_t nsets = 0;
  uint64_t total = 0;            // members stored
  uint32_t max_len = 0;
  bool counter_complete = true;  // every batch so far was fused
  rrgpu::DevBuf<uint64_t> off;   // u64[nsets+1], slot order
  rrgpu::DevBuf<uint32_t> mem;   // u32[total], visit order within a set (root first)
  rrgpu::DevBuf<uint32_t> counter;  // fused occurrence histogram u32[n]
  rrgpu::DevBuf<uint32_t> maxlen_dev;
  // staging for one batch
  rrgpu::DevBuf<uint32_t> stage;
  rrgpu::DevBuf<uint64_t> slot_start;
  rrgpu::DevBuf<uint32_t> slot_len;
  rrgpu::DevBuf<uint32_t> deferred;
  rrgpu::DevBuf<uint32_t> deferred2;
  rrgpu::DevBuf<uint32_t> restage;
  rrgpu::DevBuf<uint32_t> restage2;
  rrgpu::DevBuf<uint32_t> bigre;
  rrgpu::DevBuf<uint64_t> scan;
  rrgpu::DevBuf<uint64_t> scan_tmp;
  // selection scratch
  rrgpu::DevBuf<uint32_t> wcnt;
  rrgpu::DevBuf<uint64_t> ioff;
  rrgpu::DevBuf<unsigned long long> icur;
  rrgpu::DevBuf<uint32_t> inv;
  rrgpu::DevBuf<uint32_t> covered;
  rrgpu::DevBuf<unsigned long long> keys;
  rrgpu::DevBuf<unsigned long long> marg;
  rrgpu::DevBuf<uint32_t> seeds;
  rrgpu::DevBuf<uint8_t> selected;
  rrgpu::DevBuf<uint32_t> snap;
  rrgpu::DevBuf<uint32_t> status;
  rrgpu::DevBuf<unsigned long long> tmax;  // selection: per-tile max keys
  rrgpu::DevBuf<uint32_t> tdirty;          // selection: per-tile dirty flags
  rrgpu::DevBuf<uint64_t> span;            // selection (scan mode): member -> set span
  rrgpu::DevBuf<uint64_t> wide;  // u64 staging of counter exports
  rrgpu::DevBuf<uint32_t> narrow;  // u32 offsets of compact exports
  // ---- dense arm (rrr_set.hpp:10-13, :73-90; pack_sketch, sampling.hpp:68-84) ----
  // A set of >= n / density_divisor members is a row of the n-bit map pool
  // instead of a list: its list range in mem/off is EMPTY (a list set always
  // holds its root), dix maps the set to its row. Rows of one batch are a
  // contiguous range (allocation order within it is arbitrary).
  uint32_t dwords = 0;                 // u32 words per row: ceil(n/32) rounded up to 4
  uint64_t ndense = 0;                 // rows in use
  uint64_t dense_members = 0;          // sum of the rows' member counts
  uint32_t dense_max = 0;              // largest row
  rrgpu::DevBuf<uint32_t> dbits;       // ndense x dwords
  rrgpu::DevBuf<uint32_t> dlen;        // per row: member count
  rrgpu::DevBuf<uint32_t> droot;       // per row: the set's root (RRRSet::root)
  rrgpu::DevBuf<uint32_t> dslot;       // per row: its set index in the store
  rrgpu::DevBuf<uint32_t> dix;         // per set: its row, or kNoRow (list set)
  rrgpu::DevBuf<uint32_t> bdix;        // per batch slot: its row, or kNoRow
  rrgpu::DevBuf<uint32_t> dreq;        // batch-local slots to convert at commit
  rrgpu::DevBuf<unsigned long long> dctl;  // [0] rows requested [1] members [2] max
  rrgpu::DevBuf<uint32_t> dcov;        // selection: per row, covered
  rrgpu::DevBuf<uint32_t> dkill;       // selection: rows killed in the current round
  rrgpu::DevBuf<uint32_t> dkn;         // selection: per round, rows killed
  rrgpu::DevBuf<uint32_t> lcnt;        // selection (index mode): list-only counts
  rrgpu::DevBuf<uint32_t> xlen;        // export: per set, its member count
  rrgpu::DevBuf<uint64_t> xoff;        // export: materialized offsets
  rrgpu::DevBuf<uint32_t> xmem;        // export: materialized members
  uint64_t last_rebuilds = 0;          // rounds of the last select_seeds that rebuilt
  // host copy of the offsets (side stores the IMM driver appends from): filled
  // from the commit's scan, so appends need no device read-back
  bool keep_hoff = false;
  std::vector<uint64_t> hoff{0};
  uint64_t live = 0;                   // RRRStore::live_count (rrr_store.hpp:84)
  int sel_mode = 0;                    // liveness held by: 0 none (all live), 1 scan copy, 2 covered[]
  uint64_t member_limit = 0;           // 0: none; else RRG_ENOMEM past it (tests, budgets)
  rrgpu::DevBuf<uint32_t> csnap;       // fused counter before the current chunk
  uint64_t members() const { return total + dense_members; }
};

namespace rrgpu {

// ---- launchers (sample.cu) ------------------------------------------------
struct SampleParams {
  uint32_t n;
  const uint32_t* off;
  const uint2* rec;
  const uint32_t* src;
  const float* w;        // IC: f32 weights (Bernoulli ties, big-set path)
  const double* cdf;
  const uint4* ltrec;    // LT vertex records (search mode), 4 x uint4 per vertex
  const uint32_t* ltnodes;  // LT search-tree nodes (32 floats each)
  const uint4* ltguide;     // LT guide table (guide mode), 2 x uint4 per bucket
  const uint2* ltlite;      // LT lite guide table (set INSTEAD of ltguide), 8 bytes per bucket
  uint32_t lt_guide_mult;   // LT guide buckets per in-edge
  uint64_t run_seed;
  uint64_t base_slot;
  uint64_t count;
  uint32_t* lists;
  uint64_t* tabs;
  uint32_t* xhi;  // per block: 4096 draw high words of the current window
  uint32_t* tags;
  uint32_t* wtags;       // warp-region tag counters (IC warp mode)
  uint64_t lanes;        // lane scratch regions allocated
  uint32_t* stage;
  uint64_t stage_cap;
  uint64_t* slot_start;
  uint32_t* slot_len;
  uint32_t* counter;
  const uint32_t* list;  // optional batch-local slot list (reruns); count = its length
  uint32_t idx_base;     // range mode: batch-local index of dispenser item 0
  uint32_t* deferred;    // out: slots for the big-set path
  uint32_t* restage;     // out: slots refused for lack of staging
  SampleCtl* ctl;
  int lt_scan;
  uint32_t coop_min;
  int lt_kary;              // LT search arity (2, 4, 8, 16)
  // IC cooperative expansion of long in-lists
  const uint64_t* jtab;     // byte tables of T^(32 l), l = 1..31 (jump.cpp segment_tables)
  const uint64_t* jtab16;   // byte tables of T^(16 l), l = 1..31 (warp-schedule windows)
  const uint64_t* jtab256;  // byte tables of T^(256 a), a = 1..15 (CTA-schedule windows)
  const uint64_t* jtabhi;   // byte tables of T^(16^k a), k = 3..5, a = 1..15 (list expansion)
  const uint64_t* jtab64;   // byte tables of T^(kLxPer l), l = 1..31 (list-expansion lanes)
  uint32_t* lx;             // per-CTA list-expansion scratch (CTA schedule), or null
  uint32_t lx_wmax;         // sub-windows of 512 edges the scratch holds per CTA
  const uint8_t* dupfree;   // per vertex: in-list sources strictly increasing
  const uint8_t* uniformw;  // IC fast mode: per vertex, all in-weights equal
  uint32_t ic_coop_min;     // in-lists at least this long go warp-cooperative
  uint32_t warp_win_budget; // IC warp schedule: windows per set before deferring it (0: none)
  // dense arm: the big-set path writes sets of >= dense_thr members as rows
  uint32_t dense_thr;       // kNoDense: never
  uint32_t dwords;
  uint32_t* dbits;
  uint32_t* dlen;
  uint32_t* droot;
  uint32_t* dslot;
  uint32_t* bdix;           // per batch slot: its row (kNoRow: list)
  uint64_t drow_base;       // first row of this batch
  uint64_t drow_avail;      // rows allocated after drow_base
  uint64_t set_base;        // store index of batch slot 0
  // giant CTA schedule: per block kGiantCap list entries, 2 kGiantCap table entries
  uint32_t* glists;
  uint32_t* gbits;          // per block: an n-bit visited map (gwords words)
  uint64_t gwords;
  uint32_t* gtags;
  uint32_t gctas;
};

// graph_dev.cu: device transpose (+ normalize_lt_weights) of an edge list on the
// device into g->off/src/w; 0 ok, 1 vertex out of range, 2 + v negative weight at v.
// d_w may still be in flight: w_ready (if set) is waited on before it is read.
uint64_t build_transpose_device(rrg_graph* g, const uint32_t* d_src, const uint32_t* d_dst,
                                const float* d_w, bool normalize, cudaEvent_t w_ready = nullptr);
void prepare_ic(rrg_graph* g);
void prepare_ic_fast(rrg_graph* g);
// IC fast (statistical) sampler: warp region tables, or n-bit maps (bitmap)
void launch_fast(const SampleParams& p, int grid, bool bitmap, uint32_t* bitmaps, uint32_t* lists,
                 uint32_t workers, cudaStream_t s);
void launch_fast_lane(const SampleParams& p, int grid, cudaStream_t s);
void prepare_lt(rrg_graph* g);  // fp64 CDF + monotone flag
// prepare_lt + what the graph's LT scan mode needs; returns the mode to launch
// (guide falls back to search when the table does not fit, both to linear
// when the CDF is not monotone)
// batch_sets 0: explicit prepare (full structures). *lite: launches use the lite
// guide table (g->ltlite, kGuideLiteMult buckets per in-edge) instead of the full one.
int prepare_lt_mode(rrg_graph* g, uint64_t batch_sets, bool* lite);
bool prepare_lt_lite(rrg_graph* g);  // the lite guide table (needs the CDF only)
uint32_t lt_lite_mult();
// converts d_off64 into g->off and validates offsets/sources on the device;
// returns a bit mask of violations (1 offsets, 2 sources), 0 if clean
// which: 1 = offsets, 2 = sources (sample.cu)
uint32_t upload_checks(rrg_graph* g, const uint64_t* d_off64, uint32_t which);
void upload_checks_async(rrg_graph* g, const uint64_t* d_off64, uint32_t which,
                         DevBuf<uint32_t>& bad);
int sampler_block();
int sampler_blocks_per_sm(int model, uint32_t ic_inner, int lt_mode = 1);
// IC schedules: lane per sample; warp per sample over its 32 lanes' scratch
// (sets up to 32K members); CTA per sample over its 256 lanes' scratch (256K).
enum Schedule : int { kSchedLane = 0, kSchedWarp = 1, kSchedCta = 2, kSchedCtaGiant = 3 };
constexpr uint32_t kGiantCap = 1u << 20;  // members per block of the giant CTA schedule
void launch_sampler(int model, const SampleParams& p, int grid, uint32_t ic_inner, int schedule,
                    cudaStream_t s);
// per-model halves of the two above (sample_ic.cu, sample_lt.cu)
int ic_blocks_per_sm();
void launch_ic_sampler(const SampleParams& p, int grid, uint32_t ic_inner, int schedule,
                       cudaStream_t s);
int lt_blocks_per_sm(int lt_mode);
void launch_lt_sampler(const SampleParams& p, int grid, cudaStream_t s);
void launch_big(int model, const SampleParams& p, const uint32_t* list, uint32_t nlist,
                uint32_t* bitmaps, uint32_t* lists, uint32_t workers, cudaStream_t s);
std::vector<uint64_t> segment_matrices(uint64_t seg, int count);  // jump.cpp
std::vector<uint64_t> segment_tables(uint64_t seg, int count);    // jump.cpp (byte tables)
uint64_t launches();  // kernels launched by this library so far (bench evidence)
void count_launch(uint64_t k = 1);

// ---- dense.cu ---------------------------------------------------------------
constexpr uint32_t kNoRow = 0xffffffffu;
constexpr uint32_t kNoDense = 0xffffffffu;
// smallest member count with (double)len >= (double)n / divisor (make_repr's
// switch, rrr_set.hpp:82-83); kNoDense when no set can be dense (divisor 0)
uint32_t dense_threshold(uint32_t n, uint32_t divisor);
// batch slots with slot_len >= thr -> dreq (count in dctl[0])
void launch_dense_mark(const uint32_t* slot_len, uint64_t count, uint32_t thr, uint32_t* dreq,
                       unsigned long long* dctl, cudaStream_t s);
// the requested slots' staged lists -> rows [row0, row0 + nreq); their slot_len
// becomes 0 (empty list range), bdix names the row; members/max into dctl[1..2]
void launch_densify(const uint32_t* dreq, uint64_t nreq, const uint32_t* stage,
                    const uint64_t* slot_start, uint32_t* slot_len, uint32_t* bdix, uint64_t row0,
                    uint64_t set_base, uint32_t* dbits, uint32_t dwords, uint32_t* dlen,
                    uint32_t* droot, uint32_t* dslot, unsigned long long* dctl, cudaStream_t s);
// counter[v] += sign * #{rows r in [row0, row0 + nrows) with bit v} (rows given
// directly, or through `rows` when not null); column sums, no per-member atomics
void launch_dense_colsum(const uint32_t* dbits, uint32_t dwords, uint32_t n, const uint32_t* rows,
                         uint64_t row0, uint64_t nrows, uint32_t* counter, int sign,
                         cudaStream_t s);
// per set of [first, first + count): its member count (list or row) -> xlen
void launch_set_lengths(const uint64_t* off, const uint32_t* dix, const uint32_t* dlen,
                        uint64_t first, uint64_t count, uint32_t* xlen, cudaStream_t s);
// sets [first, first + count) as lists at xoff (relative): list sets copied,
// rows decoded root first, then ascending
void launch_materialize(const uint64_t* off, const uint32_t* mem, const uint32_t* dix,
                        const uint32_t* dbits, uint32_t dwords, const uint32_t* droot,
                        uint64_t first, uint64_t count, const uint64_t* xoff, uint32_t* xmem,
                        cudaStream_t s);
// is_live per set of [first, first + count) after a selection: rows by dcov,
// list sets by the blanked scan copy (scan) or covered[] (index)
void launch_live_flags(const uint64_t* off, const uint32_t* dix, const uint32_t* wmem,
                       const uint32_t* covered, const uint32_t* dcov, bool scan, uint64_t first,
                       uint64_t count, uint8_t* out, cudaStream_t s);
// fraction_covered over rows: rows holding a flagged vertex -> hits
void launch_dense_fraction(const uint32_t* dbits, uint32_t dwords, uint64_t nrows,
                           const uint32_t* seeds, uint32_t nseeds, unsigned long long* hits,
                           cudaStream_t s);
// gathers rows src_rows[i] of src into consecutive rows from dst_row0 of dst
void launch_gather_rows(const uint32_t* src, uint32_t dwords, const uint32_t* src_rows,
                        uint64_t nrows, uint32_t* dst, uint64_t dst_row0, cudaStream_t s);

// ---- store.cu ---------------------------------------------------------------
// out[i] = sum_{t<i} in[t] for i in [0, count]; tmp grows as needed.
void exclusive_scan_u32(const uint32_t* in, uint64_t* out, uint64_t count, DevBuf<uint64_t>& tmp,
                        cudaStream_t s);
void launch_compact(const uint32_t* stage, const uint64_t* slot_start, const uint32_t* slot_len,
                    const uint64_t* scan, uint64_t base_total, uint64_t count, uint32_t* mem_out,
                    uint64_t* off_out, uint32_t* maxlen, cudaStream_t s);
void launch_recount(const uint64_t* off, const uint32_t* mem, uint64_t nsets, uint32_t* counter,
                    cudaStream_t s);
void launch_set_spans(const uint64_t* off, const uint32_t* mem, uint64_t nsets, uint64_t* span,
                      uint32_t* wmem, cudaStream_t s);
void launch_invert(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                   unsigned long long* icur, const uint64_t* ioff, uint32_t* inv,
                   uint32_t* status, cudaStream_t s);
void launch_fraction(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                     const uint8_t* in_seed_set, unsigned long long* hits, cudaStream_t s);
void launch_widen(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s);
void launch_narrow(const uint64_t* in, uint32_t* out, uint64_t n, cudaStream_t s);
void launch_rebase(const uint64_t* in, uint64_t count, uint64_t base, uint64_t* out,
                   uint32_t* maxlen, cudaStream_t s);

// ---- select.cu --------------------------------------------------------------
struct SelectParams {
  uint32_t n;
  uint32_t k;
  uint32_t* cnt;
  const uint64_t* ioff;
  const uint32_t* inv;
  const uint64_t* span;  // scan mode: per member, its set's start << 32 | length
  uint32_t* wmem;        // scan mode: working copy of the members, covered sets blanked
  const uint64_t* off;
  const uint32_t* mem;
  uint32_t* covered;
  unsigned long long* keys;
  unsigned long long* marg;
  uint32_t* seeds;
  uint8_t* selected;
  uint32_t* snap;      // k*n or null
  uint32_t* status;    // [0] = rounds completed
  uint64_t nsets;
  uint64_t total;      // members stored (scan mode reads mem[0, total) each round)
  unsigned long long* tmax;  // per-tile max packed key (kSelTile vertices per tile)
  uint32_t* dirty;     // per tile: a count in it changed this round
  int scan;            // 1: find the sets holding v by scanning the flat members
                       // (no inverted index); 0: inverted index ioff/inv
  // dense arm: rows of the n-bit map pool (their list ranges are empty)
  uint64_t nd;                 // rows
  uint32_t dwords;
  const uint32_t* dbits;
  uint32_t* dcov;              // per row: covered
  uint32_t* dkill;             // rows killed this round (kill order)
  uint32_t* dkn;               // per round: rows killed
  double adaptive_threshold;   // rebuild_update when top_count / live exceeds it
  unsigned long long* rebuilds;  // rounds that rebuilt (stats)
  // Early exit for the IMM driver's trial selections: when, at the start of a
  // round r, covered so far + (k - r) x the round's top count cannot reach
  // `need` sets, the selection stops (status[0] = r | kSelAborted). Every later
  // marginal is at most this round's top count (counts only fall), so the final
  // coverage provably stays below `need`. 0: run all k rounds.
  unsigned long long need;
};
constexpr uint32_t kSelAborted = 0x80000000u;
constexpr uint32_t kSelTileLog = 11;  // 2048 vertices per argmax tile
void launch_select(const SelectParams& p, int num_sms, cudaStream_t s);
// whether the cluster-resident selection may run this store (no dense rows, no
// per-round snapshots, not disabled by RRGPU_SELECT_CLUSTER=0)
bool select_cluster_eligible(const SelectParams& p);

}  // namespace rrgpu
