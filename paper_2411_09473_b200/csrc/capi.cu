// capi.cu -- the extern "C" boundary (include/rrgpu.h): device graph, store,
// generate_batch, select_seeds, export/import. Every call is synchronous at
// return, mirroring the reference's fork-join barriers (work_pool.hpp:14-19).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "internal.hpp"

namespace rrgpu {

namespace {
thread_local std::string t_err;
}

void set_error(const std::string& msg) { t_err = msg; }

namespace {
std::atomic<uint64_t> g_launches{0};

// Free blocks per device, keyed by size. Blocks are only ever reused for requests
// between half and all of their size, so waste stays bounded.
struct Pool {
  std::mutex mu;
  std::map<int, std::multimap<size_t, void*>> free_blocks;
};
Pool& pool() {
  static Pool* p = new Pool;  // never destroyed: outlives every static DevBuf
  return *p;
}
}  // namespace

uint64_t launches() { return g_launches.load(); }

std::atomic<uint64_t> g_syncs{0};
void host_sync(cudaStream_t s) {
  g_syncs += 1;
  RRG_CUDA(cudaStreamSynchronize(s));
}
uint64_t host_syncs() { return g_syncs.load(); }
void count_launch(uint64_t k) { g_launches += k; }

void* pool_alloc(size_t bytes, size_t* granted) {
  if (bytes == 0) bytes = 1;
  bytes = (bytes + 255) & ~static_cast<size_t>(255);
  int dev = 0;
  RRG_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lock(pool().mu);
    auto& fb = pool().free_blocks[dev];
    auto it = fb.lower_bound(bytes);
    if (it != fb.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      *granted = it->first;
      fb.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    // release every cached block of this device and retry once
    cudaGetLastError();
    std::lock_guard<std::mutex> lock(pool().mu);
    for (auto& kv : pool().free_blocks[dev]) cudaFree(kv.second);
    pool().free_blocks[dev].clear();
    e = cudaMalloc(&p, bytes);
  }
  if (e != cudaSuccess) throw CudaError{e, "cudaMalloc"};
  *granted = bytes;
  return p;
}

void pool_free(void* p, size_t bytes) {
  if (!p) return;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) == cudaSuccess) dev = attr.device;
  std::lock_guard<std::mutex> lock(pool().mu);
  pool().free_blocks[dev].emplace(bytes, p);
}

// Converts exceptions at the C boundary into status codes.
// A store limit (rrg_store_set_member_limit) reached: RRG_ENOMEM, like a failed
// device allocation (BatchOutOfMemory, sampling.hpp:148-154).
struct OutOfMemory : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename Fn>
rrg_status guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const OutOfMemory& e) {
    set_error(e.what());
    return RRG_ENOMEM;
  } catch (const CudaError& e) {
    set_error(std::string(e.where) + ": " + cudaGetErrorString(e.err));
    if (e.err == cudaErrorMemoryAllocation) {
      cudaGetLastError();  // clear the sticky-free allocation error
      return RRG_ENOMEM;
    }
    return RRG_ECUDA;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return RRG_ENOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return RRG_ECUDA;
  }
}

rrg_status invalid(const char* msg) {
  set_error(msg);
  return RRG_EINVAL;
}

}  // namespace rrgpu

using namespace rrgpu;

namespace {

constexpr int kMaxBlocksPerSm = 4;
constexpr uint32_t kBigWorkersMax = 1024;

// RRGPU_DEBUG=1 prints one line per sampler launch to stderr.
bool debug_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RRGPU_DEBUG");
    return e && *e && *e != '0';
  }();
  return on;
}

void ensure_lane_scratch(rrg_graph* g, uint64_t lanes) {
  LaneScratch& sc = g->scratch;
  if (sc.lanes >= lanes) return;
  sc.lists.release();
  sc.tabs.release();
  sc.xhi.release();
  sc.tags.release();
  sc.wtags.release();
  sc.lists.reserve_discard(lanes * kMemCap);
  sc.tabs.reserve_discard(lanes * kTabCap);
  sc.xhi.reserve_discard((lanes / 256 + 1) * 4096);  // blocks of 256 lanes x kCtaWin
  sc.tags.reserve_discard(lanes);
  sc.wtags.reserve_discard(lanes / 32 + 1);
  RRG_CUDA(cudaMemsetAsync(sc.tabs.ptr, 0, lanes * kTabCap * sizeof(uint64_t), g->stream));
  RRG_CUDA(cudaMemsetAsync(sc.tags.ptr, 0, lanes * sizeof(uint32_t), g->stream));
  RRG_CUDA(cudaMemsetAsync(sc.wtags.ptr, 0, (lanes / 32 + 1) * sizeof(uint32_t), g->stream));
  sc.lanes = lanes;
}

// Worker warps of the big-set path for n_items sets: up to 4 per SM, capped so
// their n-bit maps + n-entry lists take at most a quarter of the free device
// memory (the kernel's grid-stride loop takes the remaining sets); >= 1.
uint32_t big_workers(rrg_graph* g, uint64_t n_items) {
  uint64_t w = std::min<uint64_t>(n_items, std::min<uint64_t>(kBigWorkersMax, 4ull * g->num_sms));
  if (g->big.workers >= w) return static_cast<uint32_t>(std::max<uint64_t>(1, w));
  size_t free_b = 0, total_b = 0;
  RRG_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t per = ((static_cast<uint64_t>(g->n) + 31) / 32) * 4 + static_cast<uint64_t>(g->n) * 4;
  const uint64_t budget = (free_b + static_cast<uint64_t>(g->big.workers) * per) / 4;
  w = std::min<uint64_t>(w, budget / std::max<uint64_t>(per, 1));
  return static_cast<uint32_t>(std::max<uint64_t>(1, w));
}

void ensure_giant_scratch(rrg_graph* g, uint32_t ctas) {
  GiantScratch& gs = g->giant;
  if (gs.ctas >= ctas) return;
  gs.lists.release();
  gs.bits.release();
  gs.tags.release();
  const uint64_t words = (static_cast<uint64_t>(g->n) + 31) / 32;
  gs.lists.reserve_discard(static_cast<uint64_t>(ctas) * kGiantCap);
  gs.bits.reserve_discard(static_cast<uint64_t>(ctas) * words);
  gs.tags.reserve_discard(ctas);
  RRG_CUDA(cudaMemsetAsync(gs.bits.ptr, 0, static_cast<uint64_t>(ctas) * words * 4, g->stream));
  RRG_CUDA(cudaMemsetAsync(gs.tags.ptr, 0, ctas * 4ull, g->stream));
  gs.ctas = ctas;
}

void ensure_big_scratch(rrg_graph* g, uint32_t workers) {
  BigScratch& b = g->big;
  if (b.workers >= workers) return;
  const uint64_t words = (static_cast<uint64_t>(g->n) + 31) / 32;
  b.bitmaps.release();
  b.lists.release();
  b.bitmaps.reserve_discard(words * workers);
  b.lists.reserve_discard(static_cast<uint64_t>(g->n) * workers);
  RRG_CUDA(cudaMemsetAsync(b.bitmaps.ptr, 0, words * workers * 4, g->stream));
  b.workers = workers;
}

template <typename T>
void d2h(T* dst, const T* src, size_t count, cudaStream_t s) {
  if (!count) return;
  RRG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
}

void sync(rrg_graph* g) { host_sync((g->stream)); }

// Grows the row pool of the dense arm to hold `need` rows, keeping the rows in use.
}  // namespace

namespace rrgpu {
// The IMM driver's side stores keep their offsets on the host (csrc/imm.cpp).
void store_keep_host_offsets(rrg_store* s, bool on) {
  s->keep_hoff = on;
  if (on && s->hoff.size() != s->nsets + 1) s->hoff.clear();  // valid again after a clear
}
// IC: running mean of inspected in-edges per set on this graph (< 0: no batch
// sampled yet) -- the IMM driver's estimate of what sampling ahead costs.
double graph_ic_mean_inspected(const rrg_graph* g) { return g->ic_mean_insp; }
}  // namespace rrgpu

namespace {

// Grows the row pool of the dense arm to hold `need` rows, keeping the first
// `keep` (default: the rows in use).
void ensure_rows(rrg_store* s, uint64_t need, uint64_t keep = UINT64_MAX) {
  rrg_graph* g = s->g;
  if (keep == UINT64_MAX) keep = s->ndense;
  // (the caching allocator may grant any of the four more than asked: check each)
  if (need * s->dwords <= s->dbits.cap && need <= s->dlen.cap && need <= s->droot.cap &&
      need <= s->dslot.cap)
    return;
  const uint64_t rows = std::max<uint64_t>(need, std::max<uint64_t>(16, s->dlen.cap + s->dlen.cap / 2));
  s->dbits.reserve_keep(rows * s->dwords, keep * s->dwords, g->stream);
  s->dlen.reserve_keep(rows, keep, g->stream);
  s->droot.reserve_keep(rows, keep, g->stream);
  s->dslot.reserve_keep(rows, keep, g->stream);
}

uint64_t rows_cap(const rrg_store* s) {
  if (!s->dwords) return 0;
  return std::min<uint64_t>(std::min<uint64_t>(s->dbits.cap / s->dwords, s->dlen.cap),
                            std::min<uint64_t>(s->droot.cap, s->dslot.cap));
}

// Appends `count` already-staged sets (slot_len/slot_start in the store's staging
// arrays, bdix per slot: the row the big-set path wrote, else kNoRow) to the
// slot-ordered buffer: staged lists of >= thr members become rows of the dense
// arm (make_repr, rrr_set.hpp:82-83), then K3 scan + compaction of the lists.
// rows_big rows from s->ndense on were written by the big-set path.
// list_max: the batch's longest staged list when the sampler reported it (then
// no list can become a row below thr and the store's maximum needs no read-back),
// UINT32_MAX when unknown (imports).
void commit_staged(rrg_store* s, uint64_t count, uint32_t thr, uint64_t rows_big = 0,
                   uint64_t big_members = 0, uint32_t big_max = 0,
                   uint32_t list_max = UINT32_MAX) {
  rrg_graph* g = s->g;
  uint64_t nreq = 0;
  unsigned long long dc[3] = {0, 0, 0};
  if (thr != kNoDense && count && list_max >= thr) {
    s->dreq.reserve_discard(count);
    s->dctl.reserve_discard(3);
    RRG_CUDA(cudaMemsetAsync(s->dctl.ptr, 0, 3 * sizeof(unsigned long long), g->stream));
    launch_dense_mark(s->slot_len.ptr, count, thr, s->dreq.ptr, s->dctl.ptr, g->stream);
    d2h(dc, s->dctl.ptr, 1, g->stream);
    sync(g);
    nreq = dc[0];
    if (nreq) {
      ensure_rows(s, s->ndense + rows_big + nreq, s->ndense + rows_big);
      launch_densify(s->dreq.ptr, nreq, s->stage.ptr, s->slot_start.ptr, s->slot_len.ptr,
                     s->bdix.ptr, s->ndense + rows_big, s->nsets, s->dbits.ptr, s->dwords,
                     s->dlen.ptr, s->droot.ptr, s->dslot.ptr, s->dctl.ptr, g->stream);
      d2h(dc, s->dctl.ptr, 3, g->stream);
    }
  }
  s->scan.reserve_discard(count + 1);
  exclusive_scan_u32(s->slot_len.ptr, s->scan.ptr, count, s->scan_tmp, g->stream);
  uint64_t added = 0;
  std::vector<uint64_t> scan_h;
  const bool mirror = s->keep_hoff && s->hoff.size() == s->nsets + 1;
  if (mirror) {  // the whole scan in the same round trip: the host offsets
    scan_h.resize(count + 1);
    d2h(scan_h.data(), s->scan.ptr, count + 1, g->stream);
  } else {
    d2h(&added, s->scan.ptr + count, 1, g->stream);
  }
  sync(g);
  if (mirror) added = scan_h[count];
  if (s->member_limit &&
      s->members() + added + big_members + dc[1] > s->member_limit)
    throw OutOfMemory("store member limit reached (" + std::to_string(s->member_limit) +
                      " members)");
  const uint64_t need_mem = s->total + added;
  if (need_mem > s->mem.cap)
    s->mem.reserve_keep(std::max<uint64_t>(need_mem, s->mem.cap + s->mem.cap / 2), s->total,
                        g->stream);
  const uint64_t need_off = s->nsets + count + 1;
  if (need_off > s->off.cap)
    s->off.reserve_keep(std::max<uint64_t>(need_off, s->off.cap + s->off.cap / 2), s->nsets + 1,
                        g->stream);
  if (s->nsets + count > s->dix.cap)
    s->dix.reserve_keep(std::max<uint64_t>(s->nsets + count, s->dix.cap + s->dix.cap / 2),
                        s->nsets, g->stream);
  if (count)
    RRG_CUDA(cudaMemcpyAsync(s->dix.ptr + s->nsets, s->bdix.ptr, count * 4,
                             cudaMemcpyDeviceToDevice, g->stream));
  launch_compact(s->stage.ptr, s->slot_start.ptr, s->slot_len.ptr, s->scan.ptr, s->total, count,
                 s->mem.ptr, s->off.ptr + s->nsets, s->maxlen_dev.ptr, g->stream);
  uint32_t mx = list_max;
  if (list_max == UINT32_MAX) {  // not reported: read the compaction's maximum back
    d2h(&mx, s->maxlen_dev.ptr, 1, g->stream);
    sync(g);
  }
  if (mirror) {
    for (uint64_t i = 1; i <= count; ++i) s->hoff.push_back(s->total + scan_h[i]);
  } else if (s->keep_hoff) {
    s->hoff.clear();  // unknown: invalid until the next clear
  }
  s->nsets += count;
  s->total += added;
  s->max_len = std::max(s->max_len, mx);
  s->ndense += rows_big + nreq;
  s->dense_members += big_members + dc[1];
  s->dense_max = std::max<uint32_t>(s->dense_max, std::max<uint32_t>(big_max,
                                                                     static_cast<uint32_t>(dc[2])));
  s->live = s->nsets;  // finalize revives every set (rrr_store.hpp:49-59)
  s->sel_mode = 0;
}

// bdix[0, count) = kNoRow (every slot of a new batch starts as a list set)
void reset_batch_rows(rrg_store* s, uint64_t count) {
  s->bdix.reserve_discard(count ? count : 1);
  if (count) RRG_CUDA(cudaMemsetAsync(s->bdix.ptr, 0xff, count * 4, s->g->stream));
}

// counter += occurrences over sets [first, nsets) (build_counter, selection.hpp:79-95):
// list sets by per-member atomics, rows [row0, ndense) by column sums
void recount_into(rrg_store* s, uint64_t first, uint64_t row0, uint32_t* counter) {
  rrg_graph* g = s->g;
  launch_recount(s->off.ptr + first, s->mem.ptr, s->nsets - first, counter, g->stream);
  launch_dense_colsum(s->dbits.ptr, s->dwords, g->n, nullptr, row0, s->ndense - row0, counter, +1,
                      g->stream);
}

// Materializes sets [first, first + count) as lists (rows decoded root first)
// into s->xoff (relative offsets, count + 1) / s->xmem; returns the members.
uint64_t materialize(rrg_store* s, uint64_t first, uint64_t count, cudaStream_t st) {
  s->xlen.reserve_discard(count ? count : 1);
  s->xoff.reserve_discard(count + 1);
  launch_set_lengths(s->off.ptr, s->dix.ptr, s->dlen.ptr, first, count, s->xlen.ptr, st);
  exclusive_scan_u32(s->xlen.ptr, s->xoff.ptr, count, s->scan_tmp, st);
  uint64_t tot = 0;
  d2h(&tot, s->xoff.ptr + count, 1, st);
  host_sync((st));
  s->xmem.reserve_discard(tot ? tot : 1);
  launch_materialize(s->off.ptr, s->mem.ptr, s->dix.ptr, s->dbits.ptr, s->dwords, s->droot.ptr,
                     first, count, s->xoff.ptr, s->xmem.ptr, st);
  return tot;
}

}  // namespace

extern "C" {

const char* rrg_last_error(void) { return rrgpu::t_err.c_str(); }
uint64_t rrg_host_sync_count(void) { return rrgpu::host_syncs(); }

uint64_t rrg_launch_count(void) { return rrgpu::launches(); }
const char* rrg_version(void) { return "rrgpu 0.1.0 (sm_100a; reference rrflow 0.1.0)"; }
uint64_t rrg_debug_bernoulli_threshold(uint32_t bits) { return bernoulli_threshold(bits); }
uint32_t rrg_debug_bernoulli_thr_hi(uint32_t bits) { return bern_thr_hi(bits); }

rrg_status rrg_graph_create(uint32_t n, uint64_t m, const uint64_t* roff, const uint32_t* rsrc,
                            const float* rw, rrg_graph** out) {
  return rrg_graph_create_for(n, m, roff, rsrc, rw, -1, out);
}

// model_hint = RRG_LT: the LT layouts that need only offsets and weights (the
// exact sequential fp64 CDF: k_build_cdf, and the hubs' serial chains,
// k_build_cdf_long) are built on a second stream WHILE the sources are still
// crossing PCIe: upload order offsets, weights, sources; the CDF kernels start
// at the weights' arrival. At cfg4 the 5.9 ms of CDF chains hide behind the
// 5.1 ms source upload (IMM from host arrays 24 -> ~17 ms).
rrg_status rrg_graph_create_for(uint32_t n, uint64_t m, const uint64_t* roff, const uint32_t* rsrc,
                                const float* rw, int model_hint, rrg_graph** out) {
  if (!out) return invalid("rrg_graph_create: null output");
  *out = nullptr;
  if (m >= (1ull << 32)) return invalid("rrg_graph_create: m must be < 2^32");
  if (n && !roff) return invalid("rrg_graph_create: null offsets");
  if (m && (!rsrc || !rw)) return invalid("rrg_graph_create: null edge arrays");
  if (n == UINT32_MAX) return invalid("rrg_graph_create: n must be < 2^32 - 1");
  if (n == 0 && m != 0) return invalid("rrg_graph_create: edges without vertices");
  if (model_hint != -1 && model_hint != RRG_IC && model_hint != RRG_LT)
    return invalid("rrg_graph_create_for: unknown model hint");
  auto* g = new (std::nothrow) rrg_graph;
  if (!g) return RRG_ENOMEM;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_off = nullptr, ev_w = nullptr;
  const rrg_status st = guarded([&]() -> rrg_status {
    RRG_CUDA(cudaGetDevice(&g->device));
    RRG_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device));
    RRG_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->own_stream = true;
    RRG_CUDA(cudaEventCreate(&g->ev0));
    RRG_CUDA(cudaEventCreate(&g->ev1));
    g->n = n;
    g->m = m;
    g->off.reserve_discard(static_cast<size_t>(n) + 1);
    g->src.reserve_discard(m ? m : 1);
    g->w.reserve_discard(m ? m : 1);
    g->ctl.reserve_discard(1);
    if (n == 0) {
      RRG_CUDA(cudaMemsetAsync(g->off.ptr, 0, 4, g->stream));
      host_sync((g->stream));
      return RRG_OK;
    }
    // offsets travel as u64 and are narrowed + validated on the device
    DevBuf<uint64_t> off64;
    off64.reserve_discard(static_cast<size_t>(n) + 1);
    RRG_CUDA(cudaMemcpyAsync(off64.ptr, roff, (static_cast<size_t>(n) + 1) * 8,
                             cudaMemcpyHostToDevice, g->stream));
    const bool overlap = model_hint == RRG_LT && m != 0;
    if (!overlap) {
      if (m) {
        RRG_CUDA(cudaMemcpyAsync(g->src.ptr, rsrc, m * 4, cudaMemcpyHostToDevice, g->stream));
        RRG_CUDA(cudaMemcpyAsync(g->w.ptr, rw, m * 4, cudaMemcpyHostToDevice, g->stream));
      }
      const uint32_t bad = upload_checks(g, off64.ptr, 3u);
      if (bad & 1u) return invalid("rrg_graph_create: offsets must run 0..m, non-decreasing");
      if (bad & 2u) return invalid("rrg_graph_create: source id out of range");
      return RRG_OK;
    }
    RRG_CUDA(cudaEventCreateWithFlags(&ev_off, cudaEventDisableTiming));
    RRG_CUDA(cudaEventCreateWithFlags(&ev_w, cudaEventDisableTiming));
    RRG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    // main stream: offsets (checked), weights, sources (checked)
    DevBuf<uint32_t> bad;
    // pinned flag words (kept per thread): a pageable read would be staged
    // behind the uploads
    thread_local uint32_t* hbad = nullptr;
    if (!hbad) RRG_CUDA(cudaMallocHost(&hbad, 8));
    hbad[0] = hbad[1] = 0;
    upload_checks_async(g, off64.ptr, 1u, bad);
    RRG_CUDA(cudaMemcpyAsync(hbad, bad.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
    RRG_CUDA(cudaEventRecord(ev_off, g->stream));
    RRG_CUDA(cudaMemcpyAsync(g->w.ptr, rw, m * 4, cudaMemcpyHostToDevice, g->stream));
    RRG_CUDA(cudaEventRecord(ev_w, g->stream));
    RRG_CUDA(cudaMemcpyAsync(g->src.ptr, rsrc, m * 4, cudaMemcpyHostToDevice, g->stream));
    DevBuf<uint32_t> bad2;
    upload_checks_async(g, off64.ptr, 2u, bad2);
    RRG_CUDA(cudaMemcpyAsync(hbad + 1, bad2.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
    // the CDF kernels index the weights through the offsets: only valid ones
    RRG_CUDA(cudaEventSynchronize(ev_off));
    g_syncs += 1;
    if (hbad[0] & 1u) {
      host_sync((g->stream));
      return invalid("rrg_graph_create: offsets must run 0..m, non-decreasing");
    }
    // side stream: the CDF, from the weights' arrival on
    RRG_CUDA(cudaStreamWaitEvent(side, ev_w, 0));
    const cudaStream_t main_stream = g->stream;
    g->stream = side;
    try {
      prepare_lt(g);  // ends with a host sync of the side stream
      if (g->cdf_monotone) prepare_lt_lite(g);  // CDF only: also before the sources land
    } catch (...) {
      g->stream = main_stream;
      cudaStreamSynchronize(main_stream);
      throw;
    }
    g->stream = main_stream;
    host_sync((g->stream));
    if (hbad[1] & 2u) return invalid("rrg_graph_create: source id out of range");
    return RRG_OK;
  });
  if (side) cudaStreamDestroy(side);
  if (ev_off) cudaEventDestroy(ev_off);
  if (ev_w) cudaEventDestroy(ev_w);
  if (st != RRG_OK) {
    rrg_graph_destroy(g);
    return st;
  }
  *out = g;
  return RRG_OK;
}

rrg_status rrg_graph_create_from_edges(uint32_t n, uint64_t m, const uint32_t* src,
                                       const uint32_t* dst, const float* w, int normalize_lt,
                                       rrg_graph** out) {
  if (!out) return invalid("rrg_graph_create_from_edges: null output");
  *out = nullptr;
  if (m >= (1ull << 31)) return invalid("rrg_graph_create_from_edges: m must be < 2^31");
  if (m && (!src || !dst || !w)) return invalid("rrg_graph_create_from_edges: null edge arrays");
  if (n == UINT32_MAX) return invalid("rrg_graph_create_from_edges: n must be < 2^32 - 1");
  if (n == 0 && m != 0) return invalid("rrg_graph_create_from_edges: edges without vertices");
  auto* g = new (std::nothrow) rrg_graph;
  if (!g) return RRG_ENOMEM;
  const rrg_status st = guarded([&]() -> rrg_status {
    RRG_CUDA(cudaGetDevice(&g->device));
    RRG_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device));
    RRG_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->own_stream = true;
    RRG_CUDA(cudaEventCreate(&g->ev0));
    RRG_CUDA(cudaEventCreate(&g->ev1));
    g->n = n;
    g->m = m;
    g->ctl.reserve_discard(1);
    DevBuf<uint32_t> d_src, d_dst;
    DevBuf<float> d_w;
    d_src.reserve_discard(m ? m : 1);
    d_dst.reserve_discard(m ? m : 1);
    d_w.reserve_discard(m ? m : 1);
    // The weights are only read after the sort: their copy (queued behind the
    // ids on the link) overlaps the key build and the radix sort.
    cudaStream_t side = nullptr;
    cudaEvent_t ids_in = nullptr, w_in = nullptr;
    struct Release {
      cudaStream_t& s;
      cudaEvent_t& a;
      cudaEvent_t& b;
      ~Release() {
        if (s) cudaStreamSynchronize(s);
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
        if (s) cudaStreamDestroy(s);
      }
    } release{side, ids_in, w_in};
    if (m) {
      RRG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      RRG_CUDA(cudaEventCreateWithFlags(&ids_in, cudaEventDisableTiming));
      RRG_CUDA(cudaEventCreateWithFlags(&w_in, cudaEventDisableTiming));
      RRG_CUDA(cudaMemcpyAsync(d_src.ptr, src, m * 4, cudaMemcpyHostToDevice, g->stream));
      RRG_CUDA(cudaMemcpyAsync(d_dst.ptr, dst, m * 4, cudaMemcpyHostToDevice, g->stream));
      RRG_CUDA(cudaEventRecord(ids_in, g->stream));
      RRG_CUDA(cudaStreamWaitEvent(side, ids_in, 0));
      RRG_CUDA(cudaMemcpyAsync(d_w.ptr, w, m * 4, cudaMemcpyHostToDevice, side));
      RRG_CUDA(cudaEventRecord(w_in, side));
    }
    const uint64_t r = build_transpose_device(g, d_src.ptr, d_dst.ptr, d_w.ptr, normalize_lt != 0,
                                              w_in);
    if (r == 1) return invalid("rrg_graph_create_from_edges: vertex id out of range");
    if (r >= 2)
      return invalid(("normalize_lt_weights: negative edge weight on vertex " +
                      std::to_string(r - 2)).c_str());
    return RRG_OK;
  });
  if (st != RRG_OK) {
    rrg_graph_destroy(g);
    return st;
  }
  *out = g;
  return RRG_OK;
}

rrg_status rrg_graph_export_transpose(const rrg_graph* g, uint64_t* roff, uint32_t* rsrc,
                                      float* rw) {
  if (!g || !roff || (g->m && (!rsrc || !rw))) return invalid("null argument");
  return guarded([&]() -> rrg_status {
    std::vector<uint32_t> off(static_cast<size_t>(g->n) + 1);
    d2h(off.data(), g->off.ptr, off.size(), g->stream);
    if (g->m) {
      d2h(rsrc, g->src.ptr, g->m, g->stream);
      d2h(rw, g->w.ptr, g->m, g->stream);
    }
    sync(const_cast<rrg_graph*>(g));
    for (size_t i = 0; i < off.size(); ++i) roff[i] = off[i];
    return RRG_OK;
  });
}

// Test hook: the LT CDF as built on the device (prepares the LT layout first).
rrg_status rrg_debug_export_lt_cdf(rrg_graph* g, double* cdf) {
  if (!g || (g->m && !cdf)) return invalid("null argument");
  return guarded([&]() -> rrg_status {
    prepare_lt(g);
    if (g->m) d2h(cdf, g->cdf.ptr, g->m, g->stream);
    sync(g);
    return RRG_OK;
  });
}

namespace {
void graph_free(rrg_graph* g) {
  if (g->stream) cudaStreamSynchronize(g->stream);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
  delete g;
}
}  // namespace

// A graph outlives its stores: destroying it while stores remain (a caller's
// garbage collector may run the two in any order) only marks it, and the last
// store's destroy frees it.
void rrg_graph_destroy(rrg_graph* g) {
  if (!g) return;
  if (g->nstores > 0) {
    g->destroyed = true;
    return;
  }
  graph_free(g);
}

rrg_status rrg_graph_prepare(rrg_graph* g, rrg_model model) {
  if (!g) return invalid("null graph");
  if (model != RRG_IC && model != RRG_LT) return invalid("unknown diffusion model");
  return guarded([&]() -> rrg_status {
    if (model == RRG_IC) prepare_ic(g);
    else {
      bool lite = false;
      prepare_lt_mode(g, 0, &lite);
    }
    return RRG_OK;
  });
}

rrg_status rrg_graph_set_stream(rrg_graph* g, void* stream) {
  if (!g) return invalid("null graph");
  return guarded([&]() -> rrg_status {
    host_sync((g->stream));
    if (g->own_stream) {
      RRG_CUDA(cudaStreamDestroy(g->stream));
      g->own_stream = false;
    }
    if (stream) {
      g->stream = static_cast<cudaStream_t>(stream);
    } else {
      RRG_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      g->own_stream = true;
    }
    return RRG_OK;
  });
}

uint32_t rrg_graph_num_vertices(const rrg_graph* g) { return g ? g->n : 0; }
uint64_t rrg_graph_num_edges(const rrg_graph* g) { return g ? g->m : 0; }

rrg_status rrg_graph_set_option(rrg_graph* g, rrg_option opt, int64_t value) {
  if (!g) return invalid("null graph");
  switch (opt) {
    case RRG_OPT_LT_SCAN:
      if (value != kLtLinear && value != kLtBsearch && value != kLtGuide)
        return invalid("LT scan must be 0 (linear), 1 (search tree) or 2 (guide table)");
      g->lt_scan = static_cast<int>(value);
      return RRG_OK;
    case RRG_OPT_LT_GUIDE_MULT:
      if (value < 1 || value > 16) return invalid("lt_guide_mult must be in [1, 16]");
      g->lt_guide_mult = static_cast<uint32_t>(value);
      g->lt_guide_mult_explicit = true;
      return RRG_OK;
    case RRG_OPT_LT_COOP_MIN:
      if (value < 2) return invalid("coop_min must be >= 2");
      g->coop_min = static_cast<uint32_t>(std::min<int64_t>(value, UINT32_MAX));
      return RRG_OK;
    case RRG_OPT_IC_INNER:
      if (value < 1 || value > 64) return invalid("ic_inner must be in [1, 64]");
      g->ic_inner = static_cast<uint32_t>(value);
      return RRG_OK;
    case RRG_OPT_IC_MODE:
      if (value < 0 || value > 3)
        return invalid("ic_mode must be 0 (auto), 1 (lane), 2 (warp) or 3 (block)");
      g->ic_mode = static_cast<int>(value);
      return RRG_OK;
    case RRG_OPT_IC_WARP_MIN_INSP:
      if (value < 0) return invalid("ic_warp_min_insp must be >= 0");
      g->ic_warp_min_insp = static_cast<double>(value);
      return RRG_OK;
    case RRG_OPT_LT_KARY:
      if (value != 2 && value != 4 && value != 8 && value != 16)
        return invalid("lt_kary must be 2, 4, 8 or 16");
      g->lt_kary = static_cast<int>(value);
      return RRG_OK;
    case RRG_OPT_IC_RNG:
      if (value != 0 && value != 1) return invalid("ic_rng must be 0 (exact) or 1 (fast)");
      g->ic_rng = static_cast<int>(value);
      return RRG_OK;
    case RRG_OPT_IC_WARP_BUDGET:
      if (value < 0) return invalid("ic_warp_budget must be >= 0");
      g->ic_warp_budget = static_cast<uint32_t>(std::min<int64_t>(value, UINT32_MAX));
      return RRG_OK;
    case RRG_OPT_IC_COOP_MIN:
      if (value < 1) return invalid("ic_coop_min must be >= 1");
      g->ic_coop_min = static_cast<uint32_t>(std::min<int64_t>(value, UINT32_MAX));
      return RRG_OK;
  }
  return invalid("unknown option");
}

rrg_status rrg_store_create(rrg_graph* g, rrg_store** out) {
  if (!g || !out) return invalid("rrg_store_create: null argument");
  *out = nullptr;
  auto* s = new (std::nothrow) rrg_store;
  if (!s) return RRG_ENOMEM;
  s->g = g;
  const rrg_status st = guarded([&]() -> rrg_status {
    s->off.reserve_discard(1024);
    s->dix.reserve_discard(1024);
    s->dctl.reserve_discard(3);
    s->dwords = static_cast<uint32_t>(((static_cast<uint64_t>(g->n) + 31) / 32 + 3) & ~3ull);
    s->mem.reserve_discard(1 << 16);
    s->counter.reserve_discard(g->n ? g->n : 1);
    s->maxlen_dev.reserve_discard(1);
    s->status.reserve_discard(2);
    RRG_CUDA(cudaMemsetAsync(s->off.ptr, 0, 8, g->stream));
    RRG_CUDA(cudaMemsetAsync(s->counter.ptr, 0, 4ull * (g->n ? g->n : 1), g->stream));
    RRG_CUDA(cudaMemsetAsync(s->maxlen_dev.ptr, 0, 4, g->stream));
    sync(g);
    return RRG_OK;
  });
  if (st != RRG_OK) {
    delete s;
    return st;
  }
  ++g->nstores;
  *out = s;
  return RRG_OK;
}

void rrg_store_destroy(rrg_store* s) {
  if (!s) return;
  rrg_graph* g = s->g;
  cudaStreamSynchronize(g->stream);
  delete s;
  if (--g->nstores == 0 && g->destroyed) graph_free(g);
}

rrg_status rrg_store_clear(rrg_store* s) {
  if (!s) return invalid("null store");
  return guarded([&]() -> rrg_status {
    rrg_graph* g = s->g;
    RRG_CUDA(cudaMemsetAsync(s->counter.ptr, 0, 4ull * (g->n ? g->n : 1), g->stream));
    RRG_CUDA(cudaMemsetAsync(s->maxlen_dev.ptr, 0, 4, g->stream));
    sync(g);
    s->nsets = s->total = 0;
    s->max_len = 0;
    s->ndense = s->dense_members = 0;
    s->dense_max = 0;
    s->live = 0;
    s->sel_mode = 0;
    s->hoff.assign(1, 0);
    s->counter_complete = true;
    return RRG_OK;
  });
}

rrg_status rrg_store_dense_info(const rrg_store* s, uint64_t* dense_sets,
                                uint64_t* dense_members, uint64_t* dense_bytes,
                                uint64_t* rebuild_rounds) {
  if (!s) return invalid("null store");
  if (dense_sets) *dense_sets = s->ndense;
  if (dense_members) *dense_members = s->dense_members;
  if (dense_bytes) *dense_bytes = s->ndense * s->dwords * 4ull;
  if (rebuild_rounds) *rebuild_rounds = s->last_rebuilds;
  return RRG_OK;
}

rrg_status rrg_store_live_count(const rrg_store* s, uint64_t* live) {
  if (!s || !live) return invalid("null argument");
  *live = s->live;
  return RRG_OK;
}

rrg_status rrg_store_live_flags(const rrg_store* s, uint64_t first, uint64_t count,
                                uint8_t* out) {
  if (!s || (count && !out)) return invalid("null argument");
  if (count > s->nsets || first > s->nsets - count) return invalid("live_flags: range out of bounds");
  if (!count) return RRG_OK;
  if (s->sel_mode == 0) {
    std::fill(out, out + count, uint8_t{1});
    return RRG_OK;
  }
  return guarded([&]() -> rrg_status {
    rrg_graph* g = s->g;
    auto* ms = const_cast<rrg_store*>(s);  // scratch only
    ms->xlen.reserve_discard((count + 3) / 4 + 1);
    launch_live_flags(s->off.ptr, s->dix.ptr, s->inv.ptr, s->covered.ptr, s->dcov.ptr,
                      s->sel_mode == 1, first, count,
                      reinterpret_cast<uint8_t*>(ms->xlen.ptr), g->stream);
    d2h(out, reinterpret_cast<const uint8_t*>(ms->xlen.ptr), count, g->stream);
    sync(g);
    return RRG_OK;
  });
}

rrg_status rrg_store_set_counter(rrg_store* s, const uint64_t* counts) {
  if (!s || !counts) return invalid("null argument");
  rrg_graph* g = s->g;
  std::vector<uint32_t> c32(g->n);
  for (uint32_t v = 0; v < g->n; ++v) {
    if (counts[v] > UINT32_MAX) return invalid("set_counter: count exceeds 2^32 - 1");
    c32[v] = static_cast<uint32_t>(counts[v]);
  }
  return guarded([&]() -> rrg_status {
    if (g->n)
      RRG_CUDA(cudaMemcpyAsync(s->counter.ptr, c32.data(), 4ull * g->n, cudaMemcpyHostToDevice,
                               g->stream));
    sync(g);
    s->counter_complete = true;  // the caller's tally is the prebuilt counter
    return RRG_OK;
  });
}

rrg_status rrg_store_set_member_limit(rrg_store* s, uint64_t max_members) {
  if (!s) return invalid("null store");
  s->member_limit = max_members;
  return RRG_OK;
}

rrg_status rrg_store_info(const rrg_store* s, uint64_t* sets, uint64_t* members,
                          uint32_t* max_set_size) {
  if (!s) return invalid("null store");
  if (sets) *sets = s->nsets;
  if (members) *members = s->members();
  if (max_set_size) *max_set_size = std::max(s->max_len, s->dense_max);
  return RRG_OK;
}

rrg_status rrg_generate_batch(rrg_graph* g, rrg_model model, uint64_t run_seed, uint64_t count,
                              rrg_store* s, int fused, uint32_t density_divisor,
                              uint64_t* sets_generated) {
  if (!s) return invalid("generate_batch: null store");
  return rrg_generate_slots(g, model, run_seed, s->nsets, count, s, fused, density_divisor,
                            sets_generated);
}

rrg_status rrg_generate_slots(rrg_graph* g, rrg_model model, uint64_t run_seed,
                              uint64_t first_slot, uint64_t count, rrg_store* s, int fused,
                              uint32_t density_divisor, uint64_t* sets_generated) {
  if (sets_generated) *sets_generated = 0;
  if (!g || !s || s->g != g) return invalid("generate_batch: graph/store mismatch");
  if (model != RRG_IC && model != RRG_LT) return invalid("unknown diffusion model");
  if (g->n == 0) return invalid("generate_batch: empty graph");
  g->last = rrg_batch_stats{};
  if (count == 0) return RRG_OK;
  return guarded([&]() -> rrg_status {
    int lt_mode = kLtLinear;
    bool lt_lite = false;
    if (model == RRG_IC) prepare_ic(g);
    else lt_mode = prepare_lt_mode(g, count, &lt_lite);
    const bool ic_fast = model == RRG_IC && g->ic_rng == 1;
    if (model == RRG_IC) prepare_ic_fast(g);  // uniform-weight flags (fast mode, list expansion)
    if (!fused) s->counter_complete = false;
    const cudaStream_t st = g->stream;
    const int block = sampler_block();
    const int per_sm = std::min(kMaxBlocksPerSm, sampler_blocks_per_sm(model, g->ic_inner, lt_mode));
    const uint64_t full_grid = static_cast<uint64_t>(g->num_sms) * per_sm;
    ensure_lane_scratch(g, full_grid * block);
    const uint64_t kChunk = 1ull << 30;  // batch-local indices are u32
    const uint32_t dense_thr = dense_threshold(g->n, density_divisor);
    float sample_ms = 0.0f;
    const auto t0 = std::chrono::steady_clock::now();
    rrg_batch_stats acc{};
    // The fused counter is restored to its value before a chunk that fails
    // (device allocation or the store's member limit): the store then holds
    // exactly the sets counted, *sets_generated of them (BatchOutOfMemory,
    // sampling.hpp:148-154, :190-198).
    bool snap = false;
    try {
    for (uint64_t done = 0; done < count;) {
      uint64_t c = std::min(kChunk, count - done);
      if (s->member_limit) c = std::min<uint64_t>(c, 1024);  // partial progress before the limit
      if (fused) {
        s->csnap.reserve_discard(g->n ? g->n : 1);
        RRG_CUDA(cudaMemcpyAsync(s->csnap.ptr, s->counter.ptr, 4ull * g->n,
                                 cudaMemcpyDeviceToDevice, st));
        snap = true;
      }
      // IC execution mode. Auto mode measures a pilot chunk on a new graph first
      // (block schedule: bounded latency whatever the set sizes); sub-batches
      // append in slot order, so splitting changes nothing. Then: hub-dominated
      // sets (mean inspected >= ic_hub_insp) -> warp per sample (per-edge
      // throughput); batches of few inspected edges in total -> block per sample
      // (latency: the largest sets finish 4-8x sooner); heavy large batches ->
      // warp; light large batches -> lane.
      if (model == RRG_IC && !ic_fast && g->ic_mode == 0 && g->ic_mean_insp < 0)
        c = std::min<uint64_t>(c, 2048);
      bool ic_warp = false, ic_cta = false;
      if (model == RRG_IC) {
        const double mean = g->ic_mean_insp;
        if (g->ic_mode == 2) ic_warp = true;
        else if (g->ic_mode == 3) ic_cta = true;
        else if (g->ic_mode == 0) {
          if (mean < 0) ic_cta = true;
          else if (mean >= g->ic_hub_insp) {
            // hub-dominated sets: block per sample when its long in-lists are
            // expanded whole (cfg5 IMM 0.60 s vs 0.80 s per warp), else warp
            if (g->max_indeg >= kListMin && g->max_indeg < (1u << 24)) ic_cta = true;
            else ic_warp = true;
          }
          else if (static_cast<double>(c) * mean <= g->ic_cta_max_edges) ic_cta = true;
          else ic_warp = mean >= g->ic_warp_min_insp;
        }
      }
      // staging sized from the running mean set size (first batch: a guess;
      // sets that do not fit are re-run once staging has grown)
      const double per_set = s->nsets ? static_cast<double>(s->total) / s->nsets * 1.5 + 8 : 96.0;
      // guide-mode LT warps allocate staging in kStageChunk (2048) member chunks:
      // slack for one partly used chunk per warp of the grid
      const uint64_t slack = lt_mode == kLtGuide ? full_grid * (block / 32) * 2048 : 0;
      const uint64_t want = std::min<uint64_t>(static_cast<uint64_t>(c * per_set) + (1u << 20) + slack,
                                               1ull << 31);
      if (want > s->stage.cap) s->stage.reserve_discard(want);
      s->slot_start.reserve_discard(c);
      s->slot_len.reserve_discard(c);
      s->deferred.reserve_discard(c);
      s->deferred2.reserve_discard(c);
      s->restage.reserve_discard(c);
      s->restage2.reserve_discard(c);
      s->bigre.reserve_discard(c);
      reset_batch_rows(s, c);
      SampleCtl ctl{};
      SampleParams p{};
      p.n = g->n;
      p.off = g->off.ptr;
      p.rec = g->rec.ptr;
      p.src = g->src.ptr;
      p.w = g->w.ptr;
      p.cdf = g->cdf.ptr;
      p.ltrec = reinterpret_cast<const uint4*>(g->ltrec.ptr);
      p.ltnodes = g->ltnodes.ptr;
      p.run_seed = run_seed;
      p.base_slot = first_slot + done;
      p.count = c;
      p.lists = g->scratch.lists.ptr;
      p.tabs = g->scratch.tabs.ptr;
      p.xhi = g->scratch.xhi.ptr;
      p.tags = g->scratch.tags.ptr;
      p.wtags = g->scratch.wtags.ptr;
      p.lanes = g->scratch.lanes;
      p.stage = s->stage.ptr;
      p.stage_cap = s->stage.cap;
      p.slot_start = s->slot_start.ptr;
      p.slot_len = s->slot_len.ptr;
      p.counter = fused ? s->counter.ptr : nullptr;
      p.ctl = g->ctl.ptr;
      p.lt_scan = lt_mode;
      p.ltguide = lt_lite ? nullptr : g->ltguide.ptr;
      p.ltlite = lt_lite ? g->ltlite.ptr : nullptr;
      p.lt_guide_mult = lt_lite ? lt_lite_mult() : g->lt_guide_built;
      p.coop_min = g->coop_min;
      p.jtab = g->jtab;
      p.jtab16 = g->jtab16;
      p.jtab256 = g->jtab256;
      p.jtabhi = g->jtabhi;
      p.jtab64 = g->jtab64;
      p.lx = nullptr;
      p.lx_wmax = 0;
      if (model == RRG_IC && !ic_fast && g->max_indeg >= kListMin &&
          g->max_indeg < (1u << 24)) {
        // list expansion of long duplicate-free in-lists (CTA schedule): per CTA
        // 2 x (kLxWin / 32) + 2 words per sub-window of the largest in-list
        const uint32_t wmax = (g->max_indeg + kLxWin - 1) / kLxWin;
        const uint64_t ctas = g->scratch.lanes / block;
        g->lx.reserve_discard(ctas * (wmax * (2ull * kLxWin / 32 + 2) + 2));
        p.lx = g->lx.ptr;
        p.lx_wmax = wmax;
      }
      p.lt_kary = g->lt_kary;
      p.dupfree = g->dupfree.ptr;
      p.uniformw = g->uniformw.ptr;
      p.ic_coop_min = g->ic_coop_min;
      p.warp_win_budget = 0;
      // dense arm: the big-set path writes rows from s->ndense on
      uint64_t drow_avail = rows_cap(s) - s->ndense;
      p.dense_thr = dense_thr;
      p.dwords = s->dwords;
      p.bdix = s->bdix.ptr;
      p.drow_base = s->ndense;
      p.set_base = s->nsets;
      auto set_rows = [&]() {
        p.dbits = s->dbits.ptr;
        p.dlen = s->dlen.ptr;
        p.droot = s->droot.ptr;
        p.dslot = s->dslot.ptr;
        p.drow_avail = drow_avail;
      };
      set_rows();
      bool dense_short = false;

      // One launch of `kind` over `list` (nullptr: the range [0, n_items)). The
      // per-launch counters reset here; the deferral list accumulates over a pass.
      enum Kind { kMain, kMainWarp, kCta, kBig, kFast, kFastBig, kFastLane, kCtaGiant };
      auto launch = [&](Kind kind, const uint32_t* list, uint64_t n_items, uint32_t* restage_out) {
        ctl.next = 0;
        ctl.restage_members = 0;
        ctl.nrestage = 0;
        RRG_CUDA(cudaMemcpyAsync(g->ctl.ptr, &ctl, sizeof(SampleCtl), cudaMemcpyHostToDevice, st));
        p.restage = restage_out;
        RRG_CUDA(cudaEventRecord(g->ev0, st));
        if (kind == kFastLane) {
          p.list = list;
          p.count = n_items;
          const uint64_t grid_need = (n_items + block - 1) / block;
          launch_fast_lane(p, static_cast<int>(std::max<uint64_t>(1, std::min(full_grid, grid_need))),
                           st);
        } else if (kind == kFast || kind == kFastBig) {
          p.list = list;
          p.count = n_items;
          uint32_t workers = 0;
          if (kind == kFastBig) {
            workers = big_workers(g, n_items);
            ensure_big_scratch(g, workers);
          }
          const uint64_t grid_need = (n_items + block / 32 - 1) / (block / 32);
          launch_fast(p, static_cast<int>(std::max<uint64_t>(1, std::min(full_grid, grid_need))),
                      kind == kFastBig, g->big.bitmaps.ptr, g->big.lists.ptr, workers, st);
        } else if (kind == kBig) {
          const uint32_t workers = big_workers(g, n_items);
          ensure_big_scratch(g, workers);
          launch_big(model, p, list, static_cast<uint32_t>(n_items), g->big.bitmaps.ptr,
                     g->big.lists.ptr, workers, st);
        } else {
          p.warp_win_budget = kind == kMainWarp ? g->ic_warp_budget : 0;
          const int sched = kind == kMainWarp ? kSchedWarp : kind == kCta ? kSchedCta
                            : kind == kCtaGiant ? kSchedCtaGiant : kSchedLane;
          p.list = list;
          p.count = n_items;
          const uint64_t per_block = sched == kSchedLane ? block : sched == kSchedWarp ? block / 32 : 1;
          uint64_t grid_cap = full_grid;
          if (sched == kSchedCta) grid_cap = g->scratch.lanes / block;
          if (sched == kSchedCtaGiant) {
            grid_cap = std::min<uint64_t>(g->scratch.lanes / block, n_items);
            ensure_giant_scratch(g, static_cast<uint32_t>(grid_cap));
            p.glists = g->giant.lists.ptr;
            p.gbits = g->giant.bits.ptr;
            p.gwords = (static_cast<uint64_t>(g->n) + 31) / 32;
            p.gtags = g->giant.tags.ptr;
            p.gctas = g->giant.ctas;
          }
          const uint64_t grid_need = (n_items + per_block - 1) / per_block;
          launch_sampler(model, p,
                         static_cast<int>(std::max<uint64_t>(1, std::min(grid_cap, grid_need))),
                         g->ic_inner, sched, st);
        }
        RRG_CUDA(cudaEventRecord(g->ev1, st));
        d2h(&ctl, g->ctl.ptr, 1, st);
        sync(g);
        // rows requested past the pool were not written (those slots restaged)
        dense_short = ctl.ndense > p.drow_avail;
        if (dense_short) ctl.ndense = p.drow_avail;
        float ms = 0.0f;
        RRG_CUDA(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
        sample_ms += ms;
        if (debug_enabled())
          std::fprintf(stderr, "[rrgpu] launch kind=%d model=%d items=%llu ms=%.3f deferred=%u "
                               "restage=%u cursor=%llu cap=%zu windows=%llu cuts=%llu repairs=%llu "
                               "blocks/SM=%d\n",
                       static_cast<int>(kind), static_cast<int>(model),
                       static_cast<unsigned long long>(n_items), ms, ctl.ndeferred, ctl.nrestage,
                       static_cast<unsigned long long>(ctl.cursor), s->stage.cap, ctl.windows,
                       ctl.cuts, ctl.repairs, per_sm);
      };
      auto grow_staging = [&]() {
        const uint64_t ncap = std::max<uint64_t>(
            s->stage.cap + s->stage.cap / 2, ctl.cursor + 2 * ctl.restage_members + (1u << 20));
        s->stage.reserve_keep(ncap, s->stage.cap, st);
        p.stage = s->stage.ptr;
        p.stage_cap = s->stage.cap;
      };
      // A pass: `kind` over `list`, then over its staging refusals (after staging
      // has grown) until none remain. Returns the number of deferred slots, which
      // are in `defer_out`.
      auto pass = [&](Kind kind, const uint32_t* list, uint64_t n_items,
                      uint32_t* defer_out) -> uint64_t {
        ctl.ndeferred = 0;
        p.deferred = defer_out;
        uint32_t* rb[2] = {s->restage.ptr, s->restage2.ptr};
        for (int it = 0; n_items > 0; ++it) {
          if (it > 64) throw std::runtime_error("staging did not converge");
          launch(kind, list, n_items, rb[it & 1]);
          n_items = ctl.nrestage;
          list = rb[it & 1];
          if (dense_short) {  // the big-set path ran out of rows
            ensure_rows(s, s->ndense + std::max<uint64_t>(ctl.ndense + n_items, 2 * drow_avail),
                        s->ndense + ctl.ndense);
            drow_avail = rows_cap(s) - s->ndense;
            set_rows();
          }
          if (n_items && ctl.restage_members) grow_staging();
        }
        return ctl.ndeferred;
      };
      // main schedule, then the wider schedules for the sets it could not hold:
      // lane (1K members) or warp (32K) -> block (256K, IC) -> big-set path (n)
      // fast IC: lane per sample (ic_mode 1) or warp per sample (2, 3); auto: lane
      // for large batches (throughput), warp for small ones (latency of the
      // largest sets: cfg5 32K sets 5.1 ms per warp vs 9.2 ms per lane)
      const bool fast_lane = ic_fast && (g->ic_mode == 1 || (g->ic_mode == 0 && c >= (1u << 17)));
      // the giant / big-set passes get the largest sets of the batch: reserve a
      // row for each when they are dense-sized (bounded by a quarter of the free
      // memory; a slot that finds no row is re-run after the pool grows)
      auto reserve_rows_for = [&](uint64_t nsets_big) {
        if (dense_thr == kNoDense || dense_thr > static_cast<uint32_t>(block) * kMemCap) return;
        size_t free_b = 0, total_b = 0;
        RRG_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const uint64_t fit = free_b / 4 / (static_cast<uint64_t>(s->dwords) * 4 + 16);
        const uint64_t want = std::min<uint64_t>(nsets_big, fit);
        if (drow_avail - ctl.ndense < want) {
          ensure_rows(s, s->ndense + ctl.ndense + want, s->ndense + ctl.ndense);
          drow_avail = rows_cap(s) - s->ndense;
          set_rows();
        }
      };
      // giant-component graphs (auto mode: a block pass deferred >= 5 % of its
      // sets past the 256K-member block scratch) run the block schedule over the
      // giant scratch from the start: no set is run twice
      const bool giant_main = ic_cta && g->ic_giant && g->ic_mode == 0;
      const Kind main_kind = fast_lane ? kFastLane : ic_fast ? kFast
                             : giant_main ? kCtaGiant
                             : ic_cta ? kCta : ic_warp ? kMainWarp : kMain;
      if (giant_main) reserve_rows_for(c / 2);
      uint64_t ndef = pass(main_kind, nullptr, c, s->deferred.ptr);
      if (main_kind == kCta && g->n > static_cast<uint32_t>(block) * kMemCap && ndef * 20 >= c)
        g->ic_giant = true;
      uint32_t* dlist = s->deferred.ptr;
      uint32_t* dspare = s->deferred2.ptr;
      if (ic_fast) {
        if (ndef && fast_lane) {
          acc.deferred += ndef;
          ndef = pass(kFast, dlist, ndef, dspare);
          std::swap(dlist, dspare);
        }
        if (ndef) {
          acc.deferred += ndef;
          pass(kFastBig, dlist, ndef, dspare);
          ndef = 0;
        }
      }
      if (!ic_fast && model == RRG_IC) {
        if (ndef && main_kind != kCta && main_kind != kCtaGiant) {
          acc.deferred += ndef;
          ndef = pass(kCta, dlist, ndef, dspare);
          std::swap(dlist, dspare);
        }
        // sets past the block scratch (256K members): the same block schedule
        // over a private 1M-member scratch per block
        if (ndef && main_kind != kCtaGiant && g->n > static_cast<uint32_t>(block) * kMemCap) {
          acc.deferred += ndef;
          reserve_rows_for(ndef);
          ndef = pass(kCtaGiant, dlist, ndef, dspare);
          std::swap(dlist, dspare);
        }
      }
      if (ndef) {
        acc.deferred += ndef;
        reserve_rows_for(ndef);
        pass(kBig, dlist, ndef, s->bigre.ptr);
      }
      acc.edges_inspected += ctl.inspected;
      if (model == RRG_IC && !ic_fast) {
        const double mean = static_cast<double>(ctl.inspected) / static_cast<double>(c);
        g->ic_mean_insp = g->ic_mean_insp < 0 ? mean : 0.5 * (g->ic_mean_insp + mean);
      }
      acc.entries_read += ctl.entries;
      const uint64_t before = s->members();
      commit_staged(s, c, dense_thr, ctl.ndense, ctl.dense_members, ctl.dense_max, ctl.max_len);
      acc.members += s->members() - before;
      acc.sets += c;
      done += c;
      if (sets_generated) *sets_generated = done;
    }
    } catch (...) {
      if (snap) {
        cudaMemcpyAsync(s->counter.ptr, s->csnap.ptr, 4ull * g->n, cudaMemcpyDeviceToDevice, st);
        cudaStreamSynchronize(st);
      }
      throw;
    }
    acc.sample_ms = sample_ms;
    acc.total_ms = static_cast<float>(
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    g->last = acc;
    return RRG_OK;
  });
}

rrg_status rrg_last_batch_stats(const rrg_graph* g, rrg_batch_stats* out) {
  if (!g || !out) return invalid("null argument");
  *out = g->last;
  return RRG_OK;
}

}  // extern "C"

namespace {
rrg_status select_seeds_impl(rrg_store* s, uint32_t k, double adaptive_threshold,
                             int use_prebuilt, uint32_t* seeds, uint64_t* marginals,
                             uint64_t* round_counters, uint32_t* rounds_done,
                             uint64_t* covered_total, uint64_t need, bool* aborted);
}

extern "C" {

rrg_status rrg_select_seeds(rrg_store* s, uint32_t k, double adaptive_threshold,
                            int use_prebuilt, uint32_t* seeds, uint64_t* marginals,
                            uint64_t* round_counters, uint32_t* rounds_done,
                            uint64_t* covered_total) {
  return select_seeds_impl(s, k, adaptive_threshold, use_prebuilt, seeds, marginals,
                           round_counters, rounds_done, covered_total, 0, nullptr);
}

}  // extern "C"

namespace rrgpu {
// select_seeds for the IMM driver's trial rounds (csrc/imm.cpp): stops as soon as
// the coverage provably cannot reach `need` sets (*aborted = true; seeds and
// marginals then hold only the rounds done). need == 0: rrg_select_seeds.
rrg_status select_seeds_until(rrg_store* s, uint32_t k, double adaptive_threshold,
                              int use_prebuilt, uint32_t* seeds, uint64_t* marginals,
                              uint64_t* covered_total, uint64_t need, bool* aborted) {
  return select_seeds_impl(s, k, adaptive_threshold, use_prebuilt, seeds, marginals, nullptr,
                           nullptr, covered_total, need, aborted);
}
}  // namespace rrgpu

namespace {
rrg_status select_seeds_impl(rrg_store* s, uint32_t k, double adaptive_threshold,
                             int use_prebuilt, uint32_t* seeds, uint64_t* marginals,
                             uint64_t* round_counters, uint32_t* rounds_done,
                             uint64_t* covered_total, uint64_t need, bool* aborted) {
  if (aborted) *aborted = false;
  if (!s) return invalid("null store");
  rrg_graph* g = s->g;
  if (k < 1) return invalid("select_seeds: k must be >= 1");
  if (k > g->n) return invalid("select_seeds: k exceeds vertex count");
  if (!seeds || !marginals) return invalid("select_seeds: null output");
  return guarded([&]() -> rrg_status {
    const cudaStream_t st = g->stream;
    const uint32_t n = g->n;
    s->wcnt.reserve_discard(n);
    if (use_prebuilt && s->counter_complete) {
      RRG_CUDA(cudaMemcpyAsync(s->wcnt.ptr, s->counter.ptr, 4ull * n, cudaMemcpyDeviceToDevice,
                               st));
    } else {
      RRG_CUDA(cudaMemsetAsync(s->wcnt.ptr, 0, 4ull * n, st));
      recount_into(s, 0, 0, s->wcnt.ptr);
    }
    RRG_CUDA(cudaMemsetAsync(s->status.ptr, 0, 8, st));
    // Scan mode (stores up to kScanMaxMembers, 128 MB: every round re-reads the
    // flat members, L2-resident) needs no index; larger stores get K5, the
    // inverted index vertex -> sets from the starting tally (all sets live:
    // revive_all, selection.hpp:215).
    constexpr uint64_t kScanMaxMembers = 1ull << 25;
    const char* force_index = std::getenv("RRGPU_SELECT_INDEX");  // tests: the index path
    const bool scan = s->total <= kScanMaxMembers &&
                      !(force_index && *force_index && *force_index != '0');

    if (scan) {
      s->inv.reserve_discard(s->total ? s->total : 1);  // the blanked working copy
      s->span.reserve_discard(s->total ? s->total : 1);
      launch_set_spans(s->off.ptr, s->mem.ptr, s->nsets, s->span.ptr, s->inv.ptr, st);
    } else {
      s->ioff.reserve_discard(static_cast<uint64_t>(n) + 1);
      const uint32_t* lc = s->wcnt.ptr;
      if (s->ndense) {  // the index holds list sets only: their own counts
        s->lcnt.reserve_discard(n);
        RRG_CUDA(cudaMemsetAsync(s->lcnt.ptr, 0, 4ull * n, st));
        launch_recount(s->off.ptr, s->mem.ptr, s->nsets, s->lcnt.ptr, st);
        lc = s->lcnt.ptr;
      }
      exclusive_scan_u32(lc, s->ioff.ptr, n, s->scan_tmp, st);
      s->icur.reserve_discard(n);
      RRG_CUDA(cudaMemcpyAsync(s->icur.ptr, s->ioff.ptr, 8ull * n, cudaMemcpyDeviceToDevice, st));
      s->inv.reserve_discard(s->total ? s->total : 1);
      launch_invert(s->off.ptr, s->mem.ptr, s->nsets, s->icur.ptr, s->ioff.ptr, s->inv.ptr,
                    s->status.ptr, st);
    }
    s->covered.reserve_discard(s->nsets ? s->nsets : 1);
    RRG_CUDA(cudaMemsetAsync(s->covered.ptr, 0, 4ull * (s->nsets ? s->nsets : 1), st));
    s->keys.reserve_discard(k);
    s->marg.reserve_discard(k);
    s->seeds.reserve_discard(k);
    s->selected.reserve_discard(n);
    const uint64_t ntiles = (static_cast<uint64_t>(n) + (1u << kSelTileLog) - 1) >> kSelTileLog;
    s->tmax.reserve_discard(ntiles);
    s->tdirty.reserve_discard(ntiles);
    RRG_CUDA(cudaMemsetAsync(s->marg.ptr, 0, 8ull * k, st));
    RRG_CUDA(cudaMemsetAsync(s->selected.ptr, 0, n, st));
    if (round_counters) s->snap.reserve_discard(static_cast<uint64_t>(k) * n);
    SelectParams p{};
    p.n = n;
    p.k = k;
    p.cnt = s->wcnt.ptr;
    p.ioff = s->ioff.ptr;
    p.inv = s->inv.ptr;
    p.off = s->off.ptr;
    p.mem = s->mem.ptr;
    p.covered = s->covered.ptr;
    p.keys = s->keys.ptr;
    p.marg = s->marg.ptr;
    p.seeds = s->seeds.ptr;
    p.selected = s->selected.ptr;
    p.snap = round_counters ? s->snap.ptr : nullptr;
    p.status = s->status.ptr;
    p.nsets = s->nsets;
    p.total = s->total;
    p.tmax = s->tmax.ptr;
    p.dirty = s->tdirty.ptr;
    p.scan = scan ? 1 : 0;
    p.span = s->span.ptr;
    p.wmem = s->inv.ptr;
    // dense arm: rows are tested bit by bit; rebuild_update (selection.hpp:161-203)
    // when the round's seed covers more than adaptive_threshold of the live sets
    p.nd = s->ndense;
    p.dwords = s->dwords;
    p.dbits = s->dbits.ptr;
    s->dcov.reserve_discard(s->ndense ? s->ndense : 1);
    s->dkill.reserve_discard(s->ndense ? s->ndense : 1);
    s->dkn.reserve_discard(k + 1);
    s->dctl.reserve_discard(3);
    if (s->ndense) RRG_CUDA(cudaMemsetAsync(s->dcov.ptr, 0, 4ull * s->ndense, st));
    RRG_CUDA(cudaMemsetAsync(s->dkn.ptr, 0, 4ull * (k + 1), st));
    RRG_CUDA(cudaMemsetAsync(s->dctl.ptr, 0, 8, st));
    p.dcov = s->dcov.ptr;
    p.dkill = s->dkill.ptr;
    p.dkn = s->dkn.ptr;
    p.adaptive_threshold = adaptive_threshold;
    p.rebuilds = s->dctl.ptr;
    p.need = round_counters ? 0 : need;
    launch_select(p, g->num_sms, st);
    uint32_t status[2] = {0, 0};
    std::vector<unsigned long long> marg(k);
    d2h(status, s->status.ptr, 2, st);
    d2h(seeds, s->seeds.ptr, k, st);
    d2h(marg.data(), s->marg.ptr, k, st);
    unsigned long long rebuilds = 0;
    d2h(&rebuilds, s->dctl.ptr, 1, st);
    sync(g);
    s->last_rebuilds = rebuilds;
    if (status[1]) {
      set_error("select_seeds: prebuilt counter does not match the stored sets");
      return RRG_EINVAL;
    }
    uint64_t covered = 0;
    for (uint32_t r = 0; r < k; ++r) {
      marginals[r] = marg[r];
      covered += marg[r];
    }
    if (covered_total) *covered_total = covered;
    if (status[0] & kSelAborted) {
      status[0] &= ~kSelAborted;
      if (aborted) *aborted = true;
    }
    if (rounds_done) *rounds_done = status[0];
    s->live = s->nsets - covered;  // the store stays tombstoned (imm.hpp:194-195)
    s->sel_mode = scan ? 1 : 2;
    if (round_counters && status[0]) {
      std::vector<uint32_t> snap(static_cast<uint64_t>(status[0]) * n);
      d2h(snap.data(), s->snap.ptr, snap.size(), st);
      sync(g);
      for (size_t i = 0; i < snap.size(); ++i) round_counters[i] = snap[i];
    }
    return RRG_OK;
  });
}
}  // namespace

extern "C" {

rrg_status rrg_fraction_covered(rrg_store* s, const uint32_t* seeds, uint32_t nseeds,
                                double* out) {
  if (!s || !out) return invalid("null argument");
  if (nseeds && !seeds) return invalid("null seeds");
  rrg_graph* g = s->g;
  for (uint32_t i = 0; i < nseeds; ++i)
    if (seeds[i] >= g->n) return invalid("fraction_covered: seed out of range");
  if (s->nsets == 0) {
    *out = 0.0;
    return RRG_OK;
  }
  return guarded([&]() -> rrg_status {
    std::vector<uint8_t> flag(g->n, 0);
    for (uint32_t i = 0; i < nseeds; ++i) flag[seeds[i]] = 1;
    s->selected.reserve_discard(g->n);
    s->marg.reserve_discard(1);
    RRG_CUDA(cudaMemcpyAsync(s->selected.ptr, flag.data(), g->n, cudaMemcpyHostToDevice,
                             g->stream));
    RRG_CUDA(cudaMemsetAsync(s->marg.ptr, 0, 8, g->stream));
    launch_fraction(s->off.ptr, s->mem.ptr, s->nsets, s->selected.ptr, s->marg.ptr, g->stream);
    if (s->ndense && nseeds) {  // rows: a bit test per seed
      s->xlen.reserve_discard(nseeds);
      RRG_CUDA(cudaMemcpyAsync(s->xlen.ptr, seeds, 4ull * nseeds, cudaMemcpyHostToDevice,
                               g->stream));
      launch_dense_fraction(s->dbits.ptr, s->dwords, s->ndense, s->xlen.ptr, nseeds, s->marg.ptr,
                            g->stream);
    }
    unsigned long long hits = 0;
    d2h(&hits, s->marg.ptr, 1, g->stream);
    sync(g);
    *out = static_cast<double>(hits) / static_cast<double>(s->nsets);
    return RRG_OK;
  });
}

rrg_status rrg_store_export(const rrg_store* s, uint64_t first, uint64_t count, uint64_t* offsets,
                            uint32_t* members) {
  if (!s || !offsets) return invalid("null argument");
  if (count > s->nsets || first > s->nsets - count) return invalid("export range out of bounds");
  return guarded([&]() -> rrg_status {
    rrg_graph* g = s->g;
    if (s->ndense) {  // rows: materialized as lists (root first, then ascending)
      auto* ms = const_cast<rrg_store*>(s);  // scratch only
      const uint64_t tot = materialize(ms, first, count, g->stream);
      d2h(offsets, s->xoff.ptr, count + 1, g->stream);
      if (members) d2h(members, s->xmem.ptr, tot, g->stream);
      sync(g);
      return RRG_OK;
    }
    std::vector<uint64_t> off(count + 1);
    d2h(off.data(), s->off.ptr + first, count + 1, g->stream);
    sync(g);
    const uint64_t base = off[0];
    for (uint64_t i = 0; i <= count; ++i) offsets[i] = off[i] - base;
    if (members && off[count] > base) {
      d2h(members, s->mem.ptr + base, off[count] - base, g->stream);
      sync(g);
    }
    return RRG_OK;
  });
}

rrg_status rrg_store_append_from(rrg_store* dst, const rrg_store* src, uint64_t first,
                                 uint64_t count) {
  if (!dst || !src) return invalid("null store");
  if (dst->g != src->g) return invalid("append_from: stores of different graphs");
  if (dst == src) return invalid("append_from: source and destination are the same store");
  if (count > src->nsets || first > src->nsets - count)
    return invalid("append_from: range out of bounds");
  if (count == 0) return RRG_OK;
  return guarded([&]() -> rrg_status {
    rrg_graph* g = dst->g;
    const cudaStream_t st = g->stream;
    uint64_t ends[2] = {0, 0};
    const bool mirror = src->keep_hoff && src->hoff.size() == src->nsets + 1;
    uint32_t mirror_max = 0;
    if (mirror) {  // the source's offsets are on the host: no round trip
      ends[0] = src->hoff[first];
      ends[1] = src->hoff[first + count];
      for (uint64_t i = first; i < first + count; ++i)
        mirror_max = std::max<uint32_t>(mirror_max,
                                        static_cast<uint32_t>(src->hoff[i + 1] - src->hoff[i]));
    } else {
      d2h(ends, src->off.ptr + first, 1, st);
      d2h(ends + 1, src->off.ptr + first + count, 1, st);
      sync(g);
    }
    const uint64_t added = ends[1] - ends[0];
    if (dst->total + added > dst->mem.cap)
      dst->mem.reserve_keep(std::max<uint64_t>(dst->total + added, dst->mem.cap + dst->mem.cap / 2),
                            dst->total, st);
    if (dst->nsets + count + 1 > dst->off.cap)
      dst->off.reserve_keep(
          std::max<uint64_t>(dst->nsets + count + 1, dst->off.cap + dst->off.cap / 2),
          dst->nsets + 1, st);
    if (added)
      RRG_CUDA(cudaMemcpyAsync(dst->mem.ptr + dst->total, src->mem.ptr + ends[0], added * 4,
                               cudaMemcpyDeviceToDevice, st));
    launch_rebase(src->off.ptr + first, count, dst->total, dst->off.ptr + dst->nsets,
                  dst->maxlen_dev.ptr, st);
    // dense rows of the range: gathered into new rows of dst, dix rewritten
    std::vector<uint32_t> dix(count, kNoRow);
    if (src->ndense) {
      d2h(dix.data(), src->dix.ptr + first, count, st);
      sync(g);
    }
    std::vector<uint32_t> rows;
    for (uint64_t i = 0; i < count; ++i)
      if (dix[i] != kNoRow) rows.push_back(dix[i]);
    const uint64_t rows0 = dst->ndense;
    if (!rows.empty()) {
      const uint64_t nr = rows.size();
      std::vector<uint32_t> slen(src->ndense), sroot(src->ndense);
      d2h(slen.data(), src->dlen.ptr, src->ndense, st);
      d2h(sroot.data(), src->droot.ptr, src->ndense, st);
      sync(g);
      ensure_rows(dst, rows0 + nr);
      std::vector<uint32_t> nlen(nr), nroot(nr), nslot(nr);
      uint64_t j = 0;
      for (uint64_t i = 0; i < count; ++i) {
        if (dix[i] == kNoRow) continue;
        nlen[j] = slen[dix[i]];
        nroot[j] = sroot[dix[i]];
        nslot[j] = static_cast<uint32_t>(dst->nsets + i);
        dst->dense_members += nlen[j];
        dst->dense_max = std::max(dst->dense_max, nlen[j]);
        dix[i] = static_cast<uint32_t>(rows0 + j);
        ++j;
      }
      dst->dreq.reserve_discard(nr);
      RRG_CUDA(cudaMemcpyAsync(dst->dreq.ptr, rows.data(), nr * 4, cudaMemcpyHostToDevice, st));
      launch_gather_rows(src->dbits.ptr, src->dwords, dst->dreq.ptr, nr, dst->dbits.ptr, rows0, st);
      RRG_CUDA(cudaMemcpyAsync(dst->dlen.ptr + rows0, nlen.data(), nr * 4, cudaMemcpyHostToDevice, st));
      RRG_CUDA(cudaMemcpyAsync(dst->droot.ptr + rows0, nroot.data(), nr * 4, cudaMemcpyHostToDevice,
                               st));
      RRG_CUDA(cudaMemcpyAsync(dst->dslot.ptr + rows0, nslot.data(), nr * 4, cudaMemcpyHostToDevice,
                               st));
      dst->ndense += nr;
    }
    if (dst->nsets + count > dst->dix.cap)
      dst->dix.reserve_keep(std::max<uint64_t>(dst->nsets + count, dst->dix.cap + dst->dix.cap / 2),
                            dst->nsets, st);
    RRG_CUDA(cudaMemcpyAsync(dst->dix.ptr + dst->nsets, dix.data(), count * 4,
                             cudaMemcpyHostToDevice, st));
    launch_recount(dst->off.ptr + dst->nsets, dst->mem.ptr, count, dst->counter.ptr, st);
    launch_dense_colsum(dst->dbits.ptr, dst->dwords, g->n, nullptr, rows0, dst->ndense - rows0,
                        dst->counter.ptr, +1, st);
    uint32_t mx = mirror_max;
    if (!mirror) {
      d2h(&mx, dst->maxlen_dev.ptr, 1, st);
      sync(g);
    }
    if (dst->keep_hoff) {
      if (mirror && dst->hoff.size() == dst->nsets + 1) {
        for (uint64_t i = 1; i <= count; ++i)
          dst->hoff.push_back(dst->total + (src->hoff[first + i] - ends[0]));
      } else {
        dst->hoff.clear();  // unknown: invalid until the next clear
      }
    }
    dst->nsets += count;
    dst->total += added;
    dst->max_len = std::max(dst->max_len, mx);
    dst->live = dst->nsets;  // finalize revives every set
    dst->sel_mode = 0;
    return RRG_OK;
  });
}

rrg_status rrg_store_import(rrg_store* s, uint64_t count, const uint64_t* offsets,
                            const uint32_t* members) {
  if (!s) return invalid("null store");
  if (count == 0) return RRG_OK;
  if (!offsets) return invalid("null offsets");
  rrg_graph* g = s->g;
  const uint64_t total = offsets[count] - offsets[0];
  if (total && !members) return invalid("null members");
  for (uint64_t i = 0; i < count; ++i) {
    if (offsets[i + 1] < offsets[i]) return invalid("offsets must be non-decreasing");
    if (offsets[i + 1] - offsets[i] >= (1ull << 32)) return invalid("set too large");
  }
  for (uint64_t t = 0; t < total; ++t)
    if (members[offsets[0] + t] >= g->n) return invalid("member out of range");
  return guarded([&]() -> rrg_status {
    const cudaStream_t st = g->stream;
    std::vector<uint64_t> start(count);
    std::vector<uint32_t> len(count);
    for (uint64_t i = 0; i < count; ++i) {
      start[i] = offsets[i] - offsets[0];
      len[i] = static_cast<uint32_t>(offsets[i + 1] - offsets[i]);
    }
    s->stage.reserve_discard(total ? total : 1);
    s->slot_start.reserve_discard(count);
    s->slot_len.reserve_discard(count);
    if (total)
      RRG_CUDA(cudaMemcpyAsync(s->stage.ptr, members + offsets[0], total * 4,
                               cudaMemcpyHostToDevice, st));
    RRG_CUDA(cudaMemcpyAsync(s->slot_start.ptr, start.data(), count * 8, cudaMemcpyHostToDevice,
                             st));
    RRG_CUDA(cudaMemcpyAsync(s->slot_len.ptr, len.data(), count * 4, cudaMemcpyHostToDevice, st));
    const uint64_t nsets0 = s->nsets, rows0 = s->ndense;
    reset_batch_rows(s, count);
    // the reference's default representation switch (make_repr, rrr_set.hpp:73-90)
    commit_staged(s, count, dense_threshold(g->n, 64));
    // fused counter over the imported sets only
    recount_into(s, nsets0, rows0, s->counter.ptr);
    sync(g);
    return RRG_OK;
  });
}

rrg_status rrg_store_export_all_async(const rrg_store* s, uint64_t* offsets, uint32_t* members,
                                      uint64_t* counts, void* stream) {
  if (!s || !offsets || (s->members() && !members)) return invalid("null argument");
  return guarded([&]() -> rrg_status {
    rrg_graph* g = s->g;
    const cudaStream_t cs = static_cast<cudaStream_t>(stream);
    auto* ms = const_cast<rrg_store*>(s);  // scratch only; the store's sets are unchanged
    // the copies follow everything already enqueued on the graph's stream
    const uint64_t* off_src = s->off.ptr;
    const uint32_t* mem_src = s->mem.ptr;
    if (s->ndense) {  // rows materialized as lists on the graph's stream first
      materialize(ms, 0, s->nsets, g->stream);
      off_src = s->xoff.ptr;
      mem_src = s->xmem.ptr;
    }
    RRG_CUDA(cudaEventRecord(g->ev1, g->stream));
    RRG_CUDA(cudaStreamWaitEvent(cs, g->ev1, 0));
    RRG_CUDA(cudaMemcpyAsync(offsets, off_src, (s->nsets + 1) * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, cs));
    if (s->members())
      RRG_CUDA(cudaMemcpyAsync(members, mem_src, s->members() * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, cs));
    if (counts && g->n) {
      ms->wide.reserve_discard(g->n);
      launch_widen(s->counter.ptr, ms->wide.ptr, g->n, cs);
      RRG_CUDA(cudaMemcpyAsync(counts, ms->wide.ptr, g->n * sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, cs));
    }
    return RRG_OK;
  });
}

rrg_status rrg_store_export_all_async32(const rrg_store* s, uint32_t* offsets, uint32_t* members,
                                        uint32_t* counts, void* stream) {
  if (!s || !offsets || (s->members() && !members)) return invalid("null argument");
  if (s->members() >= (1ull << 32)) return invalid("export32: store exceeds 2^32 - 1 members");
  return guarded([&]() -> rrg_status {
    rrg_graph* g = s->g;
    const cudaStream_t cs = static_cast<cudaStream_t>(stream);
    auto* ms = const_cast<rrg_store*>(s);  // scratch only; the store's sets are unchanged
    const uint64_t* off_src = s->off.ptr;
    const uint32_t* mem_src = s->mem.ptr;
    if (s->ndense) {
      materialize(ms, 0, s->nsets, g->stream);
      off_src = s->xoff.ptr;
      mem_src = s->xmem.ptr;
    }
    ms->narrow.reserve_discard(s->nsets + 1);
    launch_narrow(off_src, ms->narrow.ptr, s->nsets + 1, g->stream);
    RRG_CUDA(cudaEventRecord(g->ev1, g->stream));
    RRG_CUDA(cudaStreamWaitEvent(cs, g->ev1, 0));
    RRG_CUDA(cudaMemcpyAsync(offsets, ms->narrow.ptr, (s->nsets + 1) * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, cs));
    if (s->members())
      RRG_CUDA(cudaMemcpyAsync(members, mem_src, s->members() * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, cs));
    if (counts && g->n)
      RRG_CUDA(cudaMemcpyAsync(counts, s->counter.ptr, g->n * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, cs));
    return RRG_OK;
  });
}

rrg_status rrg_store_counter(const rrg_store* s, uint64_t* counts) {
  if (!s || !counts) return invalid("null argument");
  return guarded([&]() -> rrg_status {
    rrg_graph* g = s->g;
    if (!g->n) return RRG_OK;
    auto* ms = const_cast<rrg_store*>(s);  // scratch only; the store's state is unchanged
    ms->wide.reserve_discard(g->n);
    launch_widen(s->counter.ptr, ms->wide.ptr, g->n, g->stream);
    d2h(counts, ms->wide.ptr, g->n, g->stream);
    sync(g);
    return RRG_OK;
  });
}

}  // extern "C"
