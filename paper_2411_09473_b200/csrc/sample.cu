// sample.cu -- K0 graph layouts and K1/K2 RRR samplers (IC / LT).
//
// Replaces generate_batch + generate_rrr_ic / generate_rrr_lt + fused
// Counter::add of the reference (proj/include/rrflow/sampling.hpp:90-199).
//
// Execution model: a persistent grid where every LANE owns one sample at a time
// and pulls the next batch-local slot from a warp-aggregated dispenser. The
// lane replays the slot's xoshiro256** stream exactly (common.cuh), so each
// set is bit-identical to the reference's whatever the schedule.
//   IC (K1): reverse BFS; the lane walks in-lists in CSR order, drawing only for
//            unvisited sources (sampling.hpp:102). Visited = 128-bit register
//            filter + per-lane tagged hash table.
//   LT (K2): reverse walk; one draw per step (sampling.hpp:127); "first j with
//            draw < acc_j" is found on a precomputed sequential fp64 CDF, so the
//            chosen index is bit-identical. Long in-lists are scanned by the
//            whole warp with 16-byte loads (coalesced), short ones per lane; an
//            optional binary-search mode picks the identical index.
// Sets that outgrow the per-lane budget (kMemCap) -- or find the staging buffer
// full -- are deferred to k_big (warp per set, n-bit visited map), which
// replays the same stream from the start.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_pipeline.h>

#include "internal.hpp"

namespace rrgpu {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void defer_slot(const SampleParams& p, uint32_t idx) {
  const unsigned q = atomicAdd(&p.ctl->ndeferred, 1u);
  p.deferred[q] = idx;  // at most one deferral per slot per launch: q < count
}

__device__ __forceinline__ void restage_slot(const SampleParams& p, uint32_t idx, uint32_t nmem) {
  atomicAdd(&p.ctl->restage_members, (unsigned long long)nmem);
  p.restage[atomicAdd(&p.ctl->nrestage, 1u)] = idx;
}

// Writes a finished set to staging, bumps the fused counter, records the slot.
// False when staging is full (the slot is re-run later and counted then).
__device__ __forceinline__ bool emit_set(const SampleParams& p, uint32_t idx, const uint32_t* mem,
                                         uint32_t nmem) {
  const unsigned long long pos = atomicAdd(&p.ctl->cursor, (unsigned long long)nmem);
  if (pos + nmem > p.stage_cap) {
    restage_slot(p, idx, nmem);
    return false;
  }
  uint32_t* out = p.stage + pos;
  uint32_t t = 0;
  for (; t + 8 <= nmem; t += 8) {  // eight member loads in flight per round trip
    uint32_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = mem[t + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      out[t + q] = v[q];
      if (p.counter) atomicAdd(p.counter + v[q], 1u);
    }
  }
  for (; t < nmem; ++t) {
    const uint32_t v = mem[t];
    out[t] = v;
    if (p.counter) atomicAdd(p.counter + v, 1u);
  }
  p.slot_start[idx] = pos;
  p.slot_len[idx] = nmem;
  return true;
}

__device__ __forceinline__ void flush_counters(const SampleParams& p, uint64_t insp,
                                               uint64_t ent) {
  for (int o = 16; o; o >>= 1) {
    insp += __shfl_xor_sync(kFull, insp, o);
    ent += __shfl_xor_sync(kFull, ent, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&p.ctl->inspected, (unsigned long long)insp);
    atomicAdd(&p.ctl->entries, (unsigned long long)ent);
  }
}

// Warp-aggregated slot dispenser. Lanes with `need` get a batch-local index or
// are marked exhausted.
__device__ __forceinline__ bool fetch_slot(const SampleParams& p, bool need, bool& exhausted,
                                           uint32_t& idx) {
  const unsigned nm = __ballot_sync(kFull, need);
  if (!nm) return false;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(nm) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&p.ctl->next, (unsigned long long)__popc(nm));
  base = __shfl_sync(kFull, base, leader);
  if (!need) return false;
  const uint64_t k = base + __popc(nm & lanemask_lt());
  if (k >= p.count) {
    exhausted = true;
    return false;
  }
  idx = p.list ? p.list[k] : p.idx_base + static_cast<uint32_t>(k);
  return true;
}

// Warp-queued slot dispenser: the warp takes kSlotChunk batch-local indices at a
// time (one atomic per chunk instead of one per walk; the dispenser word is a
// single L2 address every warp of the grid contends on) and hands them to its
// lanes in lane order. A lane that finds the queue short waits one iteration;
// `exhausted` only once the dispenser is empty too. wq_next/wq_end are
// warp-uniform.
constexpr uint32_t kSlotChunk = 32;
__device__ __forceinline__ bool fetch_slot_q(const SampleParams& p, bool need, bool& exhausted,
                                             uint32_t& idx, uint64_t& wq_next, uint64_t& wq_end) {
  const unsigned nm = __ballot_sync(kFull, need);
  if (!nm) return false;
  const int lane = threadIdx.x & 31;
  if (wq_next >= wq_end && wq_end < p.count) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&p.ctl->next, (unsigned long long)kSlotChunk);
    base = __shfl_sync(kFull, base, 0);
    wq_next = base;
    wq_end = base >= p.count ? p.count : min(static_cast<uint64_t>(base) + kSlotChunk, p.count);
  }
  const uint64_t k = wq_next + __popc(nm & lanemask_lt());
  wq_next = min(wq_next + __popc(nm), wq_end);
  if (!need) return false;
  if (k >= wq_end) {
    if (wq_end >= p.count) exhausted = true;
    return false;
  }
  idx = p.list ? p.list[k] : p.idx_base + static_cast<uint32_t>(k);
  return true;
}

// Inserts v into the lane's visited set (member list + table), growing the
// table by rehash when the load would exceed 1/2.
__device__ __forceinline__ void lane_insert(uint32_t* mem, uint64_t* tab, uint32_t& tag,
                                            uint32_t& lg, uint32_t& nmem, uint32_t v) {
  mem[nmem++] = v;
  if (2 * nmem > (1u << lg)) {
    ++lg;
    ++tag;
    for (uint32_t t = 0; t < nmem; ++t) tab_insert(tab, tag, lg, mem[t]);
  } else {
    tab_insert(tab, tag, lg, v);
  }
}

// ---------------------------------------------------------------------------
// Cooperative IC expansion of ONE lane's long in-list by the whole warp.
//
// The in-list of a dequeued vertex is consumed in windows of 1024 edges. With
// duplicate-free sources (K0 flag) the visited status of every edge is fixed
// at list start, so
//   1. the warp computes the unvisited mask of each 32-edge chunk (coalesced
//      record loads, four chunks in flight; visited = owner's filter + table,
//      or the n-bit map on the big-set path); chunk c -> lane c; the Bernoulli
//      thresholds of the window are staged in shared memory;
//   2. the window's U draws are the next U positions of the slot's stream:
//      lane l owns positions [32 l, 32 l + 32), reaches its first one with the
//      byte tables of T^(32 l) (csrc/jump.cpp) and draws for its unvisited
//      edges in CSR order -- exactly the draws the reference makes, in order;
//   3. accepted sources are appended in CSR order (ballot prefix) and marked
//      visited (owner's table by CAS + filter, or the bit map); the stream
//      continues from the state of the lane that made the window's last draw.
// Returns false when a lane set would exceed kMemCap (the slot is deferred).
// ---------------------------------------------------------------------------
struct CoopState {
  uint64_t a, b, c, d;  // owner's RNG state
  uint64_t flo, fhi;    // owner's filter (lane sets)
  uint32_t tag, lg, nmem;
};

struct CoopSmem {
  uint32_t mask[32];
  uint32_t pre[32];
  uint32_t acc[32];
  uint32_t thr[1024];  // weight bits of the window's edges
  unsigned long long st[4];
};

// Visited structures of coop_expand / the warp kernel:
//   kVisLane   owner lane's 128-bit register filter + tagged table (lane mode)
//   kVisBitmap exact n-bit map (big-set path)
//   kVisSmem   32K-bit shared-memory filter + tagged table (warp mode: sets of
//              thousands of members would saturate a register filter)
constexpr int kVisLane = 0, kVisBitmap = 1, kVisSmem = 2;
// records in flight per lane while classifying a window (one 256-byte chunk of
// the in-list per load per warp): the classification is one dependent round
// trip per kClassifyBatch chunks
#ifndef RRG_CLASSIFY_BATCH
#define RRG_CLASSIFY_BATCH 8
#endif
constexpr int kClassifyBatch = RRG_CLASSIFY_BATCH;
constexpr uint32_t kSmemFilterWords = 1024;  // 32K bits per warp
__device__ __forceinline__ uint32_t sfilt_bit(uint32_t v) { return (v * 0x2545F491u) >> 17; }
__device__ __forceinline__ bool sfilt_maybe(const uint32_t* sf, uint32_t v) {
  const uint32_t b = sfilt_bit(v);
  return (sf[b >> 5] >> (b & 31)) & 1u;
}
__device__ __forceinline__ void sfilt_add(uint32_t* sf, uint32_t v) {
  const uint32_t b = sfilt_bit(v);
  atomicOr(sf + (b >> 5), 1u << (b & 31));
}

// In-edge index of window position e: last list t with lpre[t] <= e (lists
// past the window carry lpre >= the window size). Only the rare Bernoulli tie
// needs it.
__device__ __noinline__ uint32_t win_edge(const uint32_t* lstart, const uint32_t* lpre,
                                          uint32_t nlists, uint32_t e) {
  uint32_t t = 0;
  for (uint32_t step = nlists / 2; step; step >>= 1)
    if (t + step < nlists && lpre[t + step] <= e) t += step;
  return lstart[t] + (e - lpre[t]);
}

template <int kVis>
__device__ bool coop_expand(const SampleParams& p, uint32_t jb, uint32_t je, uint32_t* mem,
                            uint64_t* tab, uint32_t* vis, CoopState& s, CoopSmem& sm,
                            uint32_t memcap = kMemCap, uint32_t* sfilt = nullptr) {
  constexpr bool kBitmap = kVis == kVisBitmap;
  const int lane = threadIdx.x & 31;
  const Filter f{s.flo, s.fhi};
  uint64_t add_lo = 0, add_hi = 0;
  for (uint32_t wb = jb; wb < je; wb += 1024) {
    const uint32_t nch = (min(1024u, je - wb) + 31) >> 5;
    // 1. unvisited mask per chunk, four chunks of records in flight
    uint32_t mymask = 0;
    for (uint32_t c0 = 0; c0 < nch; c0 += kClassifyBatch) {
      uint2 r[kClassifyBatch];
#pragma unroll
      for (int q = 0; q < kClassifyBatch; ++q) {
        const uint32_t j = wb + 32 * (c0 + q) + lane;
        r[q] = (c0 + q < nch && j < je) ? __ldg(p.rec + j) : make_uint2(0u, 0u);
      }
      uint32_t seen = 0;  // bit q: record q's source is visited
      if (kVis == kVisBitmap) {
#pragma unroll
        for (int q = 0; q < kClassifyBatch; ++q)
          seen |= ((vis[r[q].x >> 5] >> (r[q].x & 31)) & 1u) << q;
      } else {
        uint32_t vv[kClassifyBatch], maybe = 0;
#pragma unroll
        for (int q = 0; q < kClassifyBatch; ++q) {
          vv[q] = r[q].x;
          const uint32_t j = wb + 32 * (c0 + q) + lane;
          const bool hit = kVis == kVisSmem ? sfilt_maybe(sfilt, vv[q]) : f.maybe(vv[q]);
          maybe |= (c0 + q < nch && j < je && hit ? 1u : 0u) << q;
        }
        seen = tab_contains_batch<kClassifyBatch>(tab, s.tag, s.lg, vv, maybe);
      }
#pragma unroll
      for (int q = 0; q < kClassifyBatch; ++q) {
        const uint32_t c = c0 + q;
        if (c >= nch) break;
        const uint32_t j = wb + 32 * c + lane;
        bool unv = false;
        if (j < je) {
          unv = !((seen >> q) & 1u);
          sm.thr[32 * c + lane] = r[q].y;
        }
        const unsigned m = __ballot_sync(kFull, unv);
        if (lane == static_cast<int>(c)) mymask = m;
      }
    }
    const uint32_t cnt = __popc(mymask);
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t U = __shfl_sync(kFull, incl, 31);
    if (U == 0) continue;
    sm.mask[lane] = mymask;
    sm.pre[lane] = incl - cnt;
    sm.acc[lane] = 0;
    __syncwarp();
    // 2. lane l draws stream positions [32 l, min(U, 32 l + 32))
    const uint32_t r0 = 32u * lane;
    if (r0 < U) {
      Xoshiro st{s.a, s.b, s.c, s.d};
      if (lane)
        gf2_jump_tables(p.jtab + static_cast<size_t>(lane - 1) * (32 * 256 * 4), st.a, st.b, st.c,
                        st.d);
      uint32_t c = 0;  // chunk holding unvisited rank r0
      for (uint32_t step = 16; step; step >>= 1)
        if (c + step < nch && sm.pre[c + step] <= r0) c += step;
      uint32_t m = sm.mask[c];
      for (uint32_t k = r0 - sm.pre[c]; k; --k) m &= m - 1;
      const uint32_t need = min(32u, U - r0);
      uint32_t acc = 0;
      for (uint32_t done = 0; done < need;) {
        if (!m) {
          if (acc) atomicOr(&sm.acc[c], acc);
          acc = 0;
          m = sm.mask[++c];
          continue;
        }
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t x = st.next();
        const uint32_t kh = static_cast<uint32_t>(x >> 32), th = sm.thr[32 * c + bit];
        if (kh < th || (kh == th && bern_tie(x, p.w, wb + 32 * c + bit))) acc |= 1u << bit;
        ++done;
      }
      if (acc) atomicOr(&sm.acc[c], acc);
      if (r0 + need == U) {
        sm.st[0] = st.a;
        sm.st[1] = st.b;
        sm.st[2] = st.c;
        sm.st[3] = st.d;
      }
    }
    __syncwarp();
    s.a = sm.st[0];
    s.b = sm.st[1];
    s.c = sm.st[2];
    s.d = sm.st[3];
    // 3. append the accepted sources in CSR order
    const uint32_t am_lane = lane < static_cast<int>(nch) ? sm.acc[lane] : 0u;
    uint32_t A = __popc(am_lane);
    for (int o = 16; o; o >>= 1) A += __shfl_xor_sync(kFull, A, o);
    if (A) {
      if (!kBitmap) {
        if (s.nmem + A > memcap) return false;
        uint32_t lg2 = s.lg;
        while (2 * (s.nmem + A) > (1u << lg2)) ++lg2;
        if (lg2 != s.lg) {  // grow: re-insert the members under a fresh tag
          s.lg = lg2;
          ++s.tag;
          for (uint32_t t = lane; t < s.nmem; t += 32) tab_insert_atomic(tab, s.tag, s.lg, mem[t]);
          __syncwarp();
        }
      }
      unsigned cm = __ballot_sync(kFull, am_lane != 0);
      while (cm) {
        const int c = __ffs(cm) - 1;
        cm &= cm - 1;
        const uint32_t am = __shfl_sync(kFull, am_lane, c);
        if ((am >> lane) & 1u) {
          const uint32_t v = __ldg(p.src + wb + 32 * c + lane);
          mem[s.nmem + __popc(am & lanemask_lt())] = v;
          if (kVis == kVisBitmap) {
            atomicOr(vis + (v >> 5), 1u << (v & 31));
          } else {
            tab_insert_atomic(tab, s.tag, s.lg, v);
            if (kVis == kVisSmem) {
              sfilt_add(sfilt, v);
            } else {
              const uint32_t b = Filter::bit(v);
              if (b & 64) add_hi |= 1ull << (b & 63);
              else add_lo |= 1ull << (b & 63);
            }
          }
        }
        s.nmem += __popc(am);
      }
    }
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) {
    add_lo |= __shfl_xor_sync(kFull, add_lo, o);
    add_hi |= __shfl_xor_sync(kFull, add_hi, o);
  }
  s.flo |= add_lo;
  s.fhi |= add_hi;
  return true;
}

// ---------------------------------------------------------------------------
// K1: IC sampler (sampling.hpp:90-111 per slot, :177-189 per batch)
// ---------------------------------------------------------------------------
#ifndef RRG_IC_MIN_BLOCKS
#define RRG_IC_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(kBlock, RRG_IC_MIN_BLOCKS)
    k_sample_ic(const SampleParams p, const uint32_t inner) {
  __shared__ CoopSmem coop_sm[kBlock / 32];
  const int lane = threadIdx.x & 31;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t* mem = p.lists + gid * kMemCap;
  uint64_t* tab = p.tabs + gid * kTabCap;
  uint32_t tag = p.tags[gid];
  Xoshiro rng{0, 0, 0, 0};
  Filter flt;
  flt.clear();
  bool active = false, exhausted = false, want_coop = false;
  uint32_t idx = 0, nmem = 0, head = 0, lg = kTabLog0, j = 0, jend = 0;
  uint64_t insp = 0, sinsp = 0;  // committed / current sample's inspected in-edges

  for (;;) {
    if (fetch_slot(p, !active && !exhausted, exhausted, idx)) {
      rng.seed(stream_seed(p.run_seed, p.base_slot + idx));      // sampling.hpp:179
      const uint32_t root = static_cast<uint32_t>(rng.below(p.n));  // :180
      ++tag;
      lg = kTabLog0;
      flt.clear();
      mem[0] = root;
      nmem = 1;
      head = 0;
      sinsp = 0;
      j = jend = 0;
      tab_insert(tab, tag, lg, root);
      flt.add(root);
      active = true;
    }
    if (__all_sync(kFull, !active)) break;

    // long duplicate-free in-lists: the whole warp expands them, one lane at a time
    unsigned cm = __ballot_sync(kFull, active && want_coop);
    if (cm) __syncwarp();
    while (cm) {
      const int L = __ffs(cm) - 1;
      cm &= cm - 1;
      CoopState s;
      s.a = __shfl_sync(kFull, rng.a, L);
      s.b = __shfl_sync(kFull, rng.b, L);
      s.c = __shfl_sync(kFull, rng.c, L);
      s.d = __shfl_sync(kFull, rng.d, L);
      s.flo = __shfl_sync(kFull, flt.lo, L);
      s.fhi = __shfl_sync(kFull, flt.hi, L);
      s.tag = __shfl_sync(kFull, tag, L);
      s.lg = __shfl_sync(kFull, lg, L);
      s.nmem = __shfl_sync(kFull, nmem, L);
      const uint32_t jb = __shfl_sync(kFull, j, L), je = __shfl_sync(kFull, jend, L);
      const uint64_t gl = gid - lane + L;
      const bool ok = coop_expand<kVisLane>(p, jb, je, p.lists + gl * kMemCap, p.tabs + gl * kTabCap,
                                         nullptr, s, coop_sm[threadIdx.x >> 5]);
      if (lane == L) {
        want_coop = false;
        if (ok) {
          rng = Xoshiro{s.a, s.b, s.c, s.d};
          flt.lo = s.flo;
          flt.hi = s.fhi;
          tag = s.tag;
          lg = s.lg;
          nmem = s.nmem;
          j = jend;
        } else {
          defer_slot(p, idx);
          active = false;
        }
      }
    }
    if (!active) continue;

    if (j < jend) {
      // in-edges of the current vertex, CSR order (sampling.hpp:100-106)
      const uint32_t stop = min(jend, j + inner);
      for (; j < stop; ++j) {
        const uint2 r = p.rec[j];
        const uint32_t v = r.x;
        if (flt.maybe(v) && tab_contains(tab, tag, lg, v)) continue;  // visited: no draw
        const uint64_t x = rng.next();
        const uint32_t kh = static_cast<uint32_t>(x >> 32);
        if (kh < r.y || (kh == r.y && bern_tie(x, p.w, j))) {
          if (nmem == kMemCap) {
            defer_slot(p, idx);
            active = false;
            break;
          }
          lane_insert(mem, tab, tag, lg, nmem, v);
          flt.add(v);
        }
      }
    } else if (head < nmem) {
      const uint32_t u = mem[head++];  // FIFO dequeue (sampling.hpp:96-97)
      j = p.off[u];
      jend = p.off[u + 1];
      sinsp += jend - j;
      want_coop = jend - j >= p.ic_coop_min && p.dupfree[u];
    } else {
      if (emit_set(p, idx, mem, nmem)) insp += sinsp;
      active = false;
    }
  }
  p.tags[gid] = tag;
  flush_counters(p, insp, insp);
}

// ---------------------------------------------------------------------------
// K1w: IC sampler, WARP per sample. The warp keeps one sample's state
// warp-uniform and owns the scratch of all its 32 lanes as ONE region (32K
// members, 64K-entry table, 32K-bit shared-memory filter), so sets up to 32K
// members never leave the kernel.
//
// The sample's draw sequence is the concatenation, in FIFO order, of the
// in-lists of the queued vertices (sampling.hpp:96-106). The warp consumes it
// in WINDOWS of up to 512 in-edges that may span many in-lists:
//   1. window edges are loaded coalesced (32 per chunk, four chunks in flight);
//      unvisited = not in the visited set at window start;
//   2. lane l draws stream positions [16 l, 16 l + 16) of the window's
//      unvisited edges after a jump by T^(16 l) (byte tables, jump.cpp);
//   3. this is the reference's draw sequence exactly up to the first edge
//      whose source an earlier edge of the same window ACCEPTED (the reference
//      would not draw there). Accepted sources go into a shared-memory map
//      source -> first accepting position; the window is cut at the first
//      drawn edge that finds an earlier position, the stream state is
//      recomputed for the draws before the cut (jump + < 16 steps), and the
//      accepted sources before the cut are appended in window order.
// A repeated source only cuts when its earlier occurrence was accepted (about
// the edge probability), not whenever it repeats. The next window starts at
// the cut. Short in-lists of a giant near-critical set (cfg3) and hub
// in-lists (cfg5) go through the same path.
// ---------------------------------------------------------------------------
constexpr uint32_t kWarpMemCap = 32 * kMemCap;
constexpr uint32_t kWin = 512;
constexpr uint32_t kWinChunks = kWin / 32;
constexpr int kAmapLog = 9;
constexpr uint32_t kAmapSlots = 1u << kAmapLog;  // = kWin >= distinct accepted sources
struct WinFields {
  uint32_t mask[kWinChunks];
  uint32_t pre[kWinChunks];
  uint32_t acc[kWinChunks];
  uint32_t thr[kWin];
  uint32_t src[kWin];
  unsigned long long amap[kAmapSlots];  // accepted source -> first accepting position
  uint32_t lstart[32];
  uint32_t lpre[32];
  unsigned long long st[4];
};
// Accepted-source map of a window (2^kLog slots): slot = (source << 32 |
// position); the first accepting position wins by atomicMin (same key, smaller
// position). Full map (more distinct accepted sources than slots): false.
template <int kLog>
__device__ __forceinline__ bool amap_insert(unsigned long long* map, uint32_t v, uint32_t e) {
  constexpr uint32_t kSlots = 1u << kLog;
  const unsigned long long want = (static_cast<unsigned long long>(v) << 32) | e;
  uint32_t h = vhash(v) >> (32 - kLog);
  for (uint32_t probe = 0; probe < kSlots; ++probe, h = (h + 1) & (kSlots - 1)) {
    unsigned long long cur = map[h];
    if (cur == ~0ull) {
      cur = atomicCAS(map + h, ~0ull, want);
      if (cur == ~0ull) return true;
    }
    if ((cur >> 32) == v) {
      atomicMin(map + h, want);
      return true;
    }
  }
  return false;
}
// First accepting position of v in the window, or ~0u.
template <int kLog>
__device__ __forceinline__ uint32_t amap_first(const unsigned long long* map, uint32_t v) {
  constexpr uint32_t kSlots = 1u << kLog;
  uint32_t h = vhash(v) >> (32 - kLog);
  for (uint32_t probe = 0; probe < kSlots; ++probe, h = (h + 1) & (kSlots - 1)) {
    const unsigned long long cur = map[h];
    if (cur == ~0ull) return 0xffffffffu;
    if ((cur >> 32) == v) return static_cast<uint32_t>(cur);
  }
  return 0xffffffffu;
}
struct WinSmem {
  union {
    WinFields win;   // multi-list windows
    CoopSmem coop;   // one long duplicate-free in-list (coop_expand)
  } u;
  uint32_t filt[kSmemFilterWords];
};
constexpr size_t kWarpKernelDynSmem = (kBlock / 32) * sizeof(WinSmem);

// kRegionLanes: how many lane scratch regions one warp owns as ONE region --
// 32 (its own lanes: 32K members) or 256 (eight warps' lanes: 256K members,
// used for the few sets a 32-lane region could not hold). Each size draws its
// table tags from its own quarter of the tag space (see LaneScratch).
template <int kRegionLanes>
__global__ void __launch_bounds__(kBlock, RRG_IC_MIN_BLOCKS) k_sample_ic_warp(const SampleParams p) {
  constexpr uint32_t kRegionMemCap = kRegionLanes * kMemCap;
  constexpr uint32_t kTagBase = kRegionLanes == 32 ? 0x80000000u : 0xC0000000u;
  extern __shared__ __align__(16) unsigned char k_dsm[];
  const int lane = threadIdx.x & 31;
  const int wl = threadIdx.x >> 5;
  WinSmem& wsm = reinterpret_cast<WinSmem*>(k_dsm)[wl];
  WinFields& ws = wsm.u.win;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t region = gw * kRegionLanes;  // first lane region owned by this warp
  if (region + kRegionLanes > p.lanes) return;
  uint32_t* mem = p.lists + region * kMemCap;  // kRegionLanes lane regions, contiguous
  uint64_t* tab = p.tabs + region * kTabCap;
  uint32_t* sf = wsm.filt;
  for (uint32_t t = lane; t < kSmemFilterWords; t += 32) sf[t] = 0;
  const uint64_t tslot = region / 32;  // tag counter of this region (unique per size)
  uint32_t tag = kTagBase | (p.wtags[tslot] & 0x3fffffffu);
  uint64_t insp = 0;
  for (;;) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(&p.ctl->next, 1ull);
    k = __shfl_sync(kFull, k, 0);
    if (k >= p.count) break;
    const uint32_t idx = p.list ? p.list[k] : p.idx_base + static_cast<uint32_t>(k);
    Xoshiro rng;
    rng.seed(stream_seed(p.run_seed, p.base_slot + idx));
    const uint32_t root = static_cast<uint32_t>(rng.below(p.n));
    CoopState s{rng.a, rng.b, rng.c, rng.d, 0, 0, ++tag, kTabLog0, 1};
    if (lane == 0) {
      mem[0] = root;
      tab_insert(tab, s.tag, s.lg, root);
      sfilt_add(sf, root);
    }
    __syncwarp();
    bool ok = true;
    uint32_t qi = 0;             // queue position of the in-list being consumed
    uint32_t qj = p.off[root];   // its next in-edge
    while (qi < s.nmem && ok) {
      {  // a long duplicate-free in-list at the head: 1024-edge windows of one list
        const uint32_t u = mem[qi];
        const uint32_t je = p.off[u + 1];
        if (je - qj >= p.ic_coop_min && p.dupfree[u]) {
          ok = coop_expand<kVisSmem>(p, qj, je, mem, tab, nullptr, s, wsm.u.coop, kRegionMemCap,
                                     sf);
          ++qi;
          if (qi < s.nmem) qj = p.off[mem[qi]];
          __syncwarp();
          continue;
        }
      }
      // ---- window: up to 32 queued in-lists from (qi, qj), at most kWin edges
      const uint32_t nq = s.nmem;
      const bool lvalid = qi + lane < nq;
      uint32_t lb = 0, le = 0;
      if (lvalid) {
        const uint32_t v = mem[qi + lane];
        lb = lane == 0 ? qj : p.off[v];
        le = p.off[v + 1];
      }
      const uint32_t len = le - lb;
      uint32_t incl = len;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t total = __shfl_sync(kFull, incl, 31);
      ws.lstart[lane] = lb;
      ws.lpre[lane] = incl - len;
      __syncwarp();
      uint32_t ecur = min(kWin, total);
      for (uint32_t t = lane; t < kAmapSlots; t += 32) ws.amap[t] = ~0ull;
      // ---- 1. unvisited masks (status at window start)
      uint32_t mymask = 0;
      uint32_t thi = 0;  // in-list holding the window's last position
      if (ecur)
        for (uint32_t step = 16; step; step >>= 1)
          if (thi + step < 32 && ws.lpre[thi + step] <= ecur - 1) thi += step;
      const uint32_t top = thi ? 1u << (31 - __clz(thi)) : 0u;
      for (uint32_t c0 = 0; 32 * c0 < ecur; c0 += 4) {
        uint2 r[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t e = 32 * (c0 + q4) + lane;
          r[q4] = make_uint2(0xffffffffu, 0u);
          if (e < ecur) {
            uint32_t t = 0;  // in-list holding window position e: last t <= thi with lpre[t] <= e
            for (uint32_t step = top; step; step >>= 1)
              if (t + step <= thi && ws.lpre[t + step] <= e) t += step;
            r[q4] = __ldg(p.rec + ws.lstart[t] + (e - ws.lpre[t]));
          }
        }
        uint32_t vv[4], maybe = 0;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          vv[q4] = r[q4].x;
          maybe |= (32 * (c0 + q4) + lane < ecur && sfilt_maybe(sf, vv[q4]) ? 1u : 0u) << q4;
        }
        const uint32_t seen = tab_contains_batch<4>(tab, s.tag, s.lg, vv, maybe);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t c = c0 + q4;
          if (32 * c >= ecur) break;
          const uint32_t e = 32 * c + lane;
          const uint32_t v = r[q4].x;
          const bool unv = e < ecur && !((seen >> q4) & 1u);
          if (unv) {
            ws.thr[e] = r[q4].y;
            ws.src[e] = v;
          }
          const unsigned m = __ballot_sync(kFull, unv);
          if (lane == static_cast<int>(c)) mymask = m;
        }
      }
      uint32_t nch = (ecur + 31) >> 5;
      const uint32_t cnt = __popc(mymask);
      uint32_t ui = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, ui, o);
        if (lane >= o) ui += y;
      }
      const uint32_t U = __shfl_sync(kFull, ui, 31);
      if (lane < static_cast<int>(kWinChunks)) {
        ws.mask[lane] = mymask;
        ws.pre[lane] = ui - cnt;
        ws.acc[lane] = 0;
      }
      __syncwarp();
      bool cut = false;
      if (U) {
        // ---- 2. lane l draws positions [16 l, 16 l + 16) of the window
        const uint32_t r0 = 16u * lane;
        if (r0 < U) {
          Xoshiro st{s.a, s.b, s.c, s.d};
          if (lane)
            gf2_jump_tables(p.jtab16 + static_cast<size_t>(lane - 1) * (32 * 256 * 4), st.a, st.b,
                            st.c, st.d);
          uint32_t c = 0;
          for (uint32_t step = 8; step; step >>= 1)
            if (c + step < nch && ws.pre[c + step] <= r0) c += step;
          uint32_t m = ws.mask[c];
          for (uint32_t k2 = r0 - ws.pre[c]; k2; --k2) m &= m - 1;
          const uint32_t need = min(16u, U - r0);
          uint32_t acc = 0;
          for (uint32_t done = 0; done < need;) {
            if (!m) {
              if (acc) atomicOr(&ws.acc[c], acc);
              acc = 0;
              m = ws.mask[++c];
              continue;
            }
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const uint64_t x = st.next();
            const uint32_t kh = static_cast<uint32_t>(x >> 32), th = ws.thr[32 * c + bit];
            if (kh < th || (kh == th && bern_tie(x, p.w, win_edge(ws.lstart, ws.lpre, 32, 32 * c + bit))))
              acc |= 1u << bit;
            ++done;
          }
          if (acc) atomicOr(&ws.acc[c], acc);
          if (r0 + need == U) {
            ws.st[0] = st.a;
            ws.st[1] = st.b;
            ws.st[2] = st.c;
            ws.st[3] = st.d;
          }
        }
        __syncwarp();
        uint32_t am_lane = lane < static_cast<int>(nch) ? ws.acc[lane] : 0u;
        const unsigned acm = __ballot_sync(kFull, am_lane != 0);
        if (acm) {
          // ---- 3a. every edge drew as if its source were still unvisited. That
          // is the reference's draw sequence up to the first drawn edge whose
          // source an EARLIER edge of the window accepted: cut right there.
          uint32_t fail = 0xffffffffu;
          for (unsigned t = acm; t; t &= t - 1) {
            const int c = __ffs(t) - 1;
            const uint32_t am = __shfl_sync(kFull, am_lane, c);
            const uint32_t e = 32 * c + lane;
            if (((am >> lane) & 1u) && !amap_insert<kAmapLog>(ws.amap, ws.src[e], e)) fail = min(fail, e);
          }
          __syncwarp();
          uint32_t cpos = __reduce_min_sync(kFull, fail);
          for (uint32_t c = __ffs(acm) - 1; c < nch && 32 * c < cpos; ++c) {
            const uint32_t e = 32 * c + lane;
            const bool conf = ((ws.mask[c] >> lane) & 1u) && amap_first<kAmapLog>(ws.amap, ws.src[e]) < e;
            const unsigned b = __ballot_sync(kFull, conf);
            if (b) {
              cpos = min(cpos, 32 * c + __ffs(b) - 1);
              break;
            }
          }
          if (cpos < ecur) {
            // the stream resumes after the draws of the edges before the cut
            cut = true;
            const uint32_t cc = cpos >> 5, cb = cpos & 31;
            const uint32_t R = ws.pre[cc] + __popc(ws.mask[cc] & ((1u << cb) - 1u));
            if (lane == static_cast<int>(R >> 4)) {
              Xoshiro st{s.a, s.b, s.c, s.d};
              if (lane)
                gf2_jump_tables(p.jtab16 + static_cast<size_t>(lane - 1) * (32 * 256 * 4), st.a,
                                st.b, st.c, st.d);
              for (uint32_t k2 = R & 15u; k2; --k2) st.next();
              ws.st[0] = st.a;
              ws.st[1] = st.b;
              ws.st[2] = st.c;
              ws.st[3] = st.d;
            }
            if (lane > static_cast<int>(cc)) am_lane = 0;
            else if (lane == static_cast<int>(cc)) am_lane &= (1u << cb) - 1u;
            ecur = cpos;
            nch = (ecur + 31) >> 5;
            __syncwarp();
          }
        }
        s.a = ws.st[0];
        s.b = ws.st[1];
        s.c = ws.st[2];
        s.d = ws.st[3];
        // ---- 3. append the accepted sources in window order
        uint32_t A = __popc(am_lane);
        for (int o = 16; o; o >>= 1) A += __shfl_xor_sync(kFull, A, o);
        if (A) {
          if (s.nmem + A > kRegionMemCap) {
            ok = false;
          } else {
            uint32_t lg2 = s.lg;
            while (2 * (s.nmem + A) > (1u << lg2)) ++lg2;
            if (lg2 != s.lg) {  // grow: re-insert the members under a fresh tag
              s.lg = lg2;
              ++s.tag;
              for (uint32_t t = lane; t < s.nmem; t += 32) tab_insert_atomic(tab, s.tag, s.lg, mem[t]);
              __syncwarp();
            }
            unsigned cmk = __ballot_sync(kFull, am_lane != 0);
            while (cmk) {
              const int c = __ffs(cmk) - 1;
              cmk &= cmk - 1;
              const uint32_t am = __shfl_sync(kFull, am_lane, c);
              if ((am >> lane) & 1u) {
                const uint32_t v = ws.src[32 * c + lane];
                mem[s.nmem + __popc(am & lanemask_lt())] = v;
                tab_insert_atomic(tab, s.tag, s.lg, v);
                sfilt_add(sf, v);
              }
              s.nmem += __popc(am);
            }
          }
        }
      }
      if (lane == 0) {
        atomicAdd(&p.ctl->windows, 1ull);
        if (cut) atomicAdd(&p.ctl->cuts, 1ull);
      }
      // ---- advance past the ecur consumed edges
      const unsigned partial = __ballot_sync(kFull, lvalid && incl > ecur);
      if (partial) {
        const int t = __ffs(partial) - 1;
        qi += t;
        qj = ws.lstart[t] + (ecur - ws.lpre[t]);
      } else {
        qi += min(32u, nq - qi);
        if (qi < s.nmem) qj = p.off[mem[qi]];
      }
      __syncwarp();
    }
    // inspected in-edges of the set = sum of its members' in-degrees
    uint64_t sinsp = 0;
    if (ok) {
      for (uint32_t t = lane; t < s.nmem; t += 32) {
        const uint32_t v = mem[t];
        sinsp += p.off[v + 1] - p.off[v];
      }
      for (int o = 16; o; o >>= 1) sinsp += __shfl_xor_sync(kFull, sinsp, o);
    }
    tag = s.tag;
    for (uint32_t t = lane; t < kSmemFilterWords; t += 32) sf[t] = 0;  // filter per sample
    __syncwarp();
    if (!ok) {
      if (lane == 0) defer_slot(p, idx);
      continue;
    }
    // write-out: staging + fused counter, warp-parallel
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&p.ctl->cursor, (unsigned long long)s.nmem);
    pos = __shfl_sync(kFull, pos, 0);
    if (pos + s.nmem > p.stage_cap) {
      if (lane == 0) restage_slot(p, idx, s.nmem);
      continue;
    }
    for (uint32_t t = lane; t < s.nmem; t += 32) {
      const uint32_t v = mem[t];
      p.stage[pos + t] = v;
      if (p.counter) atomicAdd(p.counter + v, 1u);
    }
    if (lane == 0) {
      p.slot_start[idx] = pos;
      p.slot_len[idx] = s.nmem;
    }
    insp += sinsp;
    __syncwarp();
  }
  if (lane == 0) {
    p.wtags[tslot] = tag;
    atomicAdd(&p.ctl->inspected, (unsigned long long)insp);
    atomicAdd(&p.ctl->entries, (unsigned long long)insp);
  }
}

// ---------------------------------------------------------------------------
// K1c: IC sampler, CTA per sample, for the sets the warp schedule could not
// hold (up to 256K members: the block's 256 lane regions as one). Same window
// algorithm as K1w, eight times wider: a window holds up to 8 x 512 in-edges
// of up to 256 queued in-lists, warp w classifies positions [512 w, 512 w +
// 512) against the visited set at window start, a CTA scan of the warps'
// unvisited counts gives warp w its first stream position P_w (warp-
// cooperative jumps by T^(256 a) and T^(16 b), then c < 16 steps; P_w = 256 a +
// 16 b + c), and the accepted-source map is CTA-wide, so the conflict cut is
// the reference's across warps. The visited filter is 256K bits.
// ---------------------------------------------------------------------------
constexpr int kCtaWarps = kBlock / 32;
constexpr uint32_t kCtaWin = kCtaWarps * kWin;  // 4096 in-edges
constexpr int kCtaAmapLog = 11;                 // 2048 slots; a full map cuts the window
constexpr uint32_t kCtaFilterWords = 8192;      // 256K bits
constexpr uint32_t kCtaFastMin = 1024;          // single-list fast windows from this length
constexpr uint32_t kJumpTableWords = 32 * 256 * 4;
constexpr int kLxCpl = RRG_LX_CPL;            // list expansion: 32-edge chunks per lane
constexpr uint32_t kLxPer = 32u * kLxCpl;     // draws per lane per sub-window
constexpr uint32_t kLxWords = 32u * kLxCpl;   // mask words (chunks) per sub-window
struct CtaWarpFields {
  uint32_t mask[kWinChunks];
  uint32_t pre[kWinChunks];
  uint32_t acc[kWinChunks];
  union {
    struct {
      uint32_t thr[kWin];
      uint32_t src[kWin];
    };
    uint32_t lxthr[2 * kWin];  // list expansion: the sub-window's thresholds (unequal weights)
  };
  uint32_t lxmask[kLxWords], lxpre[kLxWords], lxacc[kLxWords];  // list expansion: per chunk
  unsigned long long st[4];  // list expansion: the warp's stream state after a sub-window
};
struct CtaSmem {
  CtaWarpFields w[kCtaWarps];
  unsigned long long amap[1u << kCtaAmapLog];
  uint32_t filt[kCtaFilterWords];
  uint32_t lstart[kBlock];
  uint32_t lpre[kBlock];
  unsigned long long st[4];
  unsigned long long next;
  uint32_t wsum[kCtaWarps];
  uint32_t wU[kCtaWarps];
  uint32_t wA[kCtaWarps];
  uint32_t cut;
  uint32_t adv_qi;
  uint32_t adv_qj;
  uint32_t any_acc;
};
constexpr size_t kCtaKernelDynSmem = sizeof(CtaSmem);
__device__ __forceinline__ uint32_t cfilt_bit(uint32_t v) { return (v * 0x2545F491u) >> 14; }
__device__ __forceinline__ bool cfilt_maybe(const uint32_t* sf, uint32_t v) {
  const uint32_t b = cfilt_bit(v);
  return (sf[b >> 5] >> (b & 31)) & 1u;
}
__device__ __forceinline__ void cfilt_add(uint32_t* sf, uint32_t v) {
  const uint32_t b = cfilt_bit(v);
  atomicOr(sf + (b >> 5), 1u << (b & 31));
}

// Warp-cooperative jump: every lane holds the same state; lane i looks up byte
// i of it in the byte tables (one 32-byte load) and the warp XOR-reduces.
__device__ __forceinline__ void warp_jump(const uint64_t* __restrict__ T, Xoshiro& st) {
  const int lane = threadIdx.x & 31;
  const uint64_t wv = lane < 8 ? st.a : lane < 16 ? st.b : lane < 24 ? st.c : st.d;
  const uint32_t byte = static_cast<uint32_t>(wv >> (8 * (lane & 7))) & 255u;
  const ulonglong2* e = reinterpret_cast<const ulonglong2*>(T + (static_cast<size_t>(lane) * 256 + byte) * 4);
  ulonglong2 x = __ldg(e), y = __ldg(e + 1);
  for (int o = 16; o; o >>= 1) {
    x.x ^= __shfl_xor_sync(kFull, x.x, o);
    x.y ^= __shfl_xor_sync(kFull, x.y, o);
    y.x ^= __shfl_xor_sync(kFull, y.x, o);
    y.y ^= __shfl_xor_sync(kFull, y.y, o);
  }
  st = Xoshiro{x.x, x.y, y.x, y.y};
}
// T^P st for P < 4096, warp-uniform.
__device__ __forceinline__ Xoshiro warp_advance(const SampleParams& p, Xoshiro st, uint32_t P) {
  const uint32_t a = P >> 8, b = (P >> 4) & 15u, c = P & 15u;
  if (a) warp_jump(p.jtab256 + static_cast<size_t>(a - 1) * kJumpTableWords, st);
  if (b) warp_jump(p.jtab16 + static_cast<size_t>(b - 1) * kJumpTableWords, st);
  for (uint32_t t = 0; t < c; ++t) st.next();
  return st;
}

// T^P st for P < 2^24, warp-uniform: one warp-cooperative table jump per
// nonzero base-16 digit above the first (jtab16, jtab256, jtabhi), then c < 16
// steps. The factors are powers of one matrix, so their order is free.
__device__ __forceinline__ Xoshiro warp_advance_far(const SampleParams& p, Xoshiro st, uint32_t P) {
  const uint32_t d5 = (P >> 20) & 15u, d4 = (P >> 16) & 15u, d3 = (P >> 12) & 15u;
  if (d5) warp_jump(p.jtabhi + static_cast<size_t>(30 + d5 - 1) * kJumpTableWords, st);
  if (d4) warp_jump(p.jtabhi + static_cast<size_t>(15 + d4 - 1) * kJumpTableWords, st);
  if (d3) warp_jump(p.jtabhi + static_cast<size_t>(d3 - 1) * kJumpTableWords, st);
  return warp_advance(p, st, P & 0xfffu);
}

// Block-wide exclusive scan of x[0, W) in place (global memory); x[W] = total,
// which is also returned. Thread t scans a contiguous run of the entries.
__device__ __forceinline__ uint32_t block_exscan_global(uint32_t* x, uint32_t W, uint32_t* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, wl = tid >> 5;
  const uint32_t per = (W + kBlock - 1) / kBlock;
  const uint32_t lo = min(W, per * tid), hi = min(W, lo + per);
  uint32_t sum = 0;
  for (uint32_t i = lo; i < hi; ++i) sum += x[i];
  uint32_t incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[wl] = incl;
  __syncthreads();
  uint32_t base = 0, total = 0;
  for (int w = 0; w < kBlock / 32; ++w) {
    const uint32_t v = wsum[w];
    if (w < wl) base += v;
    total += v;
  }
  uint32_t run = base + incl - sum;
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t t = x[i];
    x[i] = run;
    run += t;
  }
  if (tid == 0) x[W] = total;
  __syncthreads();  // prefix visible; wsum free again
  return total;
}

__global__ void __launch_bounds__(kBlock, RRG_IC_MIN_BLOCKS) k_sample_ic_cta(const SampleParams p) {
  constexpr uint32_t kCap = kBlock * kMemCap;
  extern __shared__ __align__(16) unsigned char k_dsm[];
  CtaSmem& cs = *reinterpret_cast<CtaSmem*>(k_dsm);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wl = tid >> 5;
  CtaWarpFields& ws = cs.w[wl];
  const uint64_t region = static_cast<uint64_t>(blockIdx.x) * kBlock;
  if (region + kBlock > p.lanes) return;  // uniform per block
  uint32_t* mem = p.lists + region * kMemCap;
  uint64_t* tab = p.tabs + region * kTabCap;
  uint32_t* sf = cs.filt;
  for (uint32_t t = tid; t < kCtaFilterWords; t += kBlock) sf[t] = 0;
  // same 256-lane regions and tag range as the 256-lane warp layout
  const uint64_t tslot = region / 32;
  uint32_t tag = 0xC0000000u | (p.wtags[tslot] & 0x3fffffffu);
  uint64_t insp = 0;
  const uint32_t wbase = kWin * wl;  // this warp's first window position
  for (;;) {
    __syncthreads();  // previous sample written out, filter cleared
    if (tid == 0) cs.next = atomicAdd(&p.ctl->next, 1ull);
    __syncthreads();
    const unsigned long long k = cs.next;
    if (k >= p.count) break;
    const uint32_t idx = p.list ? p.list[k] : p.idx_base + static_cast<uint32_t>(k);
    Xoshiro s;
    s.seed(stream_seed(p.run_seed, p.base_slot + idx));      // sampling.hpp:179
    const uint32_t root = static_cast<uint32_t>(s.below(p.n));  // :180
    uint32_t stag = ++tag, lg = kTabLog0, nmem = 1;
    if (tid == 0) {
      mem[0] = root;
      tab_insert(tab, stag, lg, root);
      cfilt_add(sf, root);
    }
    __syncthreads();
    bool ok = true;
    uint32_t qi = 0, qj = p.off[root];
    while (qi < nmem && ok) {
      // ---- whole-list expansion: a duplicate-free in-list with at least kListMin
      // remaining edges. Its unvisited edges draw consecutive stream positions in
      // CSR order whatever gets accepted inside it (no source repeats and the
      // visited set only changes when its accepted sources are appended), so the
      // list is cut into 1024-edge sub-windows that are classified in parallel
      // (1), prefix-summed into stream positions (2), drawn in parallel -- warp
      // wl walks a contiguous run of sub-windows, jumping once to its first
      // position (3) -- and appended in CSR order (4). Four barriers per list
      // instead of two per 4,096 edges.
      if (p.lx) {
        const uint32_t fv = mem[qi];
        const uint32_t fe = p.off[fv + 1];
        const uint32_t L = fe - qj;
        const bool uni = p.uniformw != nullptr && p.uniformw[fv];  // one threshold (WC)
        if (L >= kListMin && L < (1u << 24) && p.dupfree[fv] &&
            (uni || kLxWin <= 2 * kWin)) {  // uniform across the block
          const uint32_t W = (L + kLxWin - 1) / kLxWin;
          uint32_t* xm = p.lx + static_cast<size_t>(blockIdx.x) * (p.lx_wmax * (2ull * kLxWords + 2) + 2);
          uint32_t* xa = xm + static_cast<uint64_t>(kLxWords) * p.lx_wmax;
          uint32_t* xc = xa + static_cast<uint64_t>(kLxWords) * p.lx_wmax;
          uint32_t* xA = xc + p.lx_wmax + 1;
          const uint32_t t0 = (W * wl) / kCtaWarps, t1 = (W * (wl + 1)) / kCtaWarps;
          // (1) unvisited masks and counts per sub-window: lane c ends with the
          //     mask of 32-edge chunk c
          for (uint32_t t = t0; t < t1; ++t) {
            const uint32_t tb = t * kLxWin;
            const uint32_t wend = min(kLxWin, L - tb);
            uint32_t mymask[kLxCpl] = {};
            uint32_t cnt = 0;
#pragma unroll
            for (int part = 0; part < 2 * kLxCpl; ++part) {  // 16 loads in flight, then the probes
              uint32_t vv[16], maybe = 0;
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                const uint32_t el = 32 * (16 * part + q) + lane;
                vv[q] = el < wend ? __ldg(p.src + qj + tb + el) : 0u;
              }
#pragma unroll
              for (int q = 0; q < 16; ++q)
                maybe |= (32 * (16 * part + q) + lane < wend && cfilt_maybe(sf, vv[q]) ? 1u : 0u) << q;
              const uint32_t seen = tab_contains_batch<16>(tab, stag, lg, vv, maybe);
#pragma unroll
              for (int q = 0; q < 16; ++q) {
                const int c = 16 * part + q;
                const unsigned m = __ballot_sync(kFull, 32 * c + lane < wend && !((seen >> q) & 1u));
                cnt += __popc(m);
                if (lane == (c & 31)) mymask[c >> 5] = m;
              }
            }
#pragma unroll
            for (int i = 0; i < kLxCpl; ++i) xm[kLxWords * t + 32 * i + lane] = mymask[i];
            if (lane == 0) xc[t] = cnt;
          }
          __syncthreads();
          // (2) stream positions of the sub-windows
          const uint32_t U = block_exscan_global(xc, W, cs.wsum);
          // (3) draws; warp wl's state walks its sub-windows in order, lane l
          //     draws ranks [32 l, 32 l + 32) after one jump by T^(32 l)
          const uint32_t uthr = uni ? __ldg(&p.rec[qj].y) : 0u;  // every edge's threshold
          if (t0 < t1) {
            Xoshiro wst = warp_advance_far(p, s, xc[t0]);
            for (uint32_t t = t0; t < t1; ++t) {
              const uint32_t Ut = xc[t + 1] - xc[t];
              if (Ut == 0) {
#pragma unroll
                for (int i = 0; i < kLxCpl; ++i) xa[kLxWords * t + 32 * i + lane] = 0u;
                if (lane == 0) xA[t] = 0u;
                continue;
              }
              const uint32_t tb = t * kLxWin;
              const uint32_t wend = min(kLxWin, L - tb);
              const uint32_t nch = (wend + 31) >> 5;
              const uint32_t r0 = kLxPer * lane;
              Xoshiro st = wst;  // this lane's segment start, loads in flight with the masks'
              if (lane && r0 < Ut)
                gf2_jump_tables(p.jtab64 + static_cast<size_t>(lane - 1) * kJumpTableWords, st.a,
                                st.b, st.c, st.d);
              uint32_t mw[kLxCpl], run = 0;
#pragma unroll
              for (int i = 0; i < kLxCpl; ++i) mw[i] = xm[kLxWords * t + 32 * i + lane];
#pragma unroll
              for (int i = 0; i < kLxCpl; ++i) {  // chunk 32 i + lane: prefix over chunks
                uint32_t ui = __popc(mw[i]);
                for (int o = 1; o < 32; o <<= 1) {
                  const uint32_t y = __shfl_up_sync(kFull, ui, o);
                  if (lane >= o) ui += y;
                }
                ws.lxmask[32 * i + lane] = mw[i];
                ws.lxpre[32 * i + lane] = run + ui - __popc(mw[i]);
                ws.lxacc[32 * i + lane] = 0;
                run += __shfl_sync(kFull, ui, 31);
              }
              if (!uni) {  // unequal weights: the sub-window's thresholds to shared memory
                for (uint32_t c0 = 0; c0 < nch; c0 += kClassifyBatch) {
                  uint32_t th[kClassifyBatch];
#pragma unroll
                  for (int q = 0; q < kClassifyBatch; ++q) {
                    const uint32_t el = 32 * (c0 + q) + lane;
                    th[q] = el < wend ? __ldg(&p.rec[qj + tb + el].y) : 0u;
                  }
#pragma unroll
                  for (int q = 0; q < kClassifyBatch; ++q) {
                    const uint32_t el = 32 * (c0 + q) + lane;
                    if (el < wend) ws.lxthr[el] = th[q];
                  }
                }
              }
              __syncwarp();
              if (uni && Ut == kLxWin) {
                // every edge draws: lane l's ranks are exactly chunks kLxCpl l + i
#pragma unroll
                for (int c = 0; c < kLxCpl; ++c) {
                  uint32_t a32 = 0;
#pragma unroll 8
                  for (int i = 0; i < 32; ++i) {
                    const uint64_t x = st.next();
                    const uint32_t kh = static_cast<uint32_t>(x >> 32);
                    if (kh < uthr || (kh == uthr && bern_tie(x, p.w, qj + tb + r0 + 32 * c + i)))
                      a32 |= 1u << i;
                  }
                  ws.lxacc[kLxCpl * lane + c] = a32;
                }
                if (lane == 31) {
                  ws.st[0] = st.a;
                  ws.st[1] = st.b;
                  ws.st[2] = st.c;
                  ws.st[3] = st.d;
                }
              } else if (r0 < Ut) {
                uint32_t c = 0;
                for (uint32_t step = kLxWords / 2; step; step >>= 1)
                  if (c + step < nch && ws.lxpre[c + step] <= r0) c += step;
                uint32_t m = ws.lxmask[c];
                for (uint32_t k2 = r0 - ws.lxpre[c]; k2; --k2) m &= m - 1;
                const uint32_t need = min(kLxPer, Ut - r0);
                uint32_t acc = 0;
                for (uint32_t done = 0; done < need;) {
                  if (!m) {
                    if (acc) atomicOr(&ws.lxacc[c], acc);
                    acc = 0;
                    m = ws.lxmask[++c];
                    continue;
                  }
                  const int bit = __ffs(m) - 1;
                  m &= m - 1;
                  const uint64_t x = st.next();
                  const uint32_t kh = static_cast<uint32_t>(x >> 32);
                  const uint32_t th = uni ? uthr : ws.lxthr[32 * c + bit];
                  if (kh < th || (kh == th && bern_tie(x, p.w, qj + tb + 32 * c + bit)))
                    acc |= 1u << bit;
                  ++done;
                }
                if (acc) atomicOr(&ws.lxacc[c], acc);
                if (r0 + need == Ut) {
                  ws.st[0] = st.a;
                  ws.st[1] = st.b;
                  ws.st[2] = st.c;
                  ws.st[3] = st.d;
                }
              }
              __syncwarp();
              wst = Xoshiro{ws.st[0], ws.st[1], ws.st[2], ws.st[3]};
              uint32_t na = 0;
#pragma unroll
              for (int i = 0; i < kLxCpl; ++i) {
                const uint32_t aw = ws.lxacc[32 * i + lane];
                xa[kLxWords * t + 32 * i + lane] = aw;
                na += __popc(aw);
              }
              for (int o = 16; o; o >>= 1) na += __shfl_xor_sync(kFull, na, o);
              if (lane == 0) xA[t] = na;
              __syncwarp();
            }
            if (t1 == W && lane == 0) {  // the stream after the list
              cs.st[0] = wst.a;
              cs.st[1] = wst.b;
              cs.st[2] = wst.c;
              cs.st[3] = wst.d;
            }
          }
          __syncthreads();
          // (4) accepted sources, appended in CSR order
          const uint32_t A = block_exscan_global(xA, W, cs.wsum);
          if (U) s = Xoshiro{cs.st[0], cs.st[1], cs.st[2], cs.st[3]};
          if (A) {
            if (nmem + A > kCap) {
              ok = false;
            } else {
              uint32_t lg2 = lg;
              while (2 * (nmem + A) > (1u << lg2)) ++lg2;
              if (lg2 != lg) {  // grow: re-insert the members under a fresh tag
                lg = lg2;
                ++stag;
                for (uint32_t t = tid; t < nmem; t += kBlock) tab_insert_atomic(tab, stag, lg, mem[t]);
                __syncthreads();
              }
              for (uint32_t t = t0; t < t1; ++t) {
                uint32_t base = nmem + xA[t];
#pragma unroll
                for (int i = 0; i < kLxCpl; ++i) {  // chunks 32 i .. 32 i + 31, in order
                  const uint32_t aw = xa[kLxWords * t + 32 * i + lane];
                  unsigned cmk = __ballot_sync(kFull, aw != 0);
                  while (cmk) {
                    const int c = __ffs(cmk) - 1;
                    cmk &= cmk - 1;
                    const uint32_t am = __shfl_sync(kFull, aw, c);
                    if ((am >> lane) & 1u) {
                      const uint32_t v = __ldg(p.src + qj + t * kLxWin + 32 * (32 * i + c) + lane);
                      mem[base + __popc(am & lanemask_lt())] = v;
                      tab_insert_atomic(tab, stag, lg, v);
                      cfilt_add(sf, v);
                    }
                    base += __popc(am);
                  }
                }
              }
              nmem += A;
            }
          }
          if (tid == 0) atomicAdd(&p.ctl->windows, 1ull);
          __syncthreads();  // members appended; scratch and cs free
          ++qi;
          if (qi < nmem) qj = p.off[mem[qi]];
          continue;
        }
      }
      // ---- fast window: a slice of ONE duplicate-free in-list of at least
      // kCtaFastMin remaining edges (hub lists). The visited set is frozen
      // inside the window and no source repeats in it, so every unvisited edge
      // draws and no acceptance can void a later draw: no accepted-source map,
      // no conflict cut, no per-edge list search, three barriers.
      {
        const uint32_t fv = mem[qi];
        const uint32_t fe = p.off[fv + 1];
        if (fe - qj >= kCtaFastMin && p.dupfree[fv]) {  // uniform across the block
          const uint32_t E = min(fe - qj, kCtaWin);
          const uint32_t wend = wbase < E ? min(kWin, E - wbase) : 0u;
          const uint32_t nch = (wend + 31) >> 5;
          uint32_t mymask = 0;
          for (uint32_t c0 = 0; c0 < nch; c0 += kClassifyBatch) {
            uint2 r[kClassifyBatch];
#pragma unroll
            for (int q4 = 0; q4 < kClassifyBatch; ++q4) {
              const uint32_t el = 32 * (c0 + q4) + lane;
              r[q4] = el < wend ? __ldg(p.rec + qj + wbase + el) : make_uint2(0xffffffffu, 0u);
            }
            uint32_t vv[kClassifyBatch], maybe = 0;
#pragma unroll
            for (int q4 = 0; q4 < kClassifyBatch; ++q4) {
              vv[q4] = r[q4].x;
              maybe |= (32 * (c0 + q4) + lane < wend && cfilt_maybe(sf, vv[q4]) ? 1u : 0u) << q4;
            }
            const uint32_t seen = tab_contains_batch<kClassifyBatch>(tab, stag, lg, vv, maybe);
#pragma unroll
            for (int q4 = 0; q4 < kClassifyBatch; ++q4) {
              const uint32_t c = c0 + q4;
              if (c >= nch) break;
              const uint32_t el = 32 * c + lane;
              const uint32_t v = r[q4].x;
              const bool unv = el < wend && !((seen >> q4) & 1u);
              if (unv) {
                ws.thr[el] = r[q4].y;
                ws.src[el] = v;
              }
              const unsigned m = __ballot_sync(kFull, unv);
              if (lane == static_cast<int>(c)) mymask = m;
            }
          }
          const uint32_t cnt = __popc(mymask);
          uint32_t ui = cnt;
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, ui, o);
            if (lane >= o) ui += y;
          }
          const uint32_t Uw = __shfl_sync(kFull, ui, 31);
          if (lane < static_cast<int>(kWinChunks)) {
            ws.mask[lane] = mymask;
            ws.pre[lane] = ui - cnt;
            ws.acc[lane] = 0;
          }
          if (lane == 0) cs.wU[wl] = Uw;
          __syncthreads();  // (1) unvisited counts
          uint32_t Pw = 0, U = 0;
          for (int w = 0; w < kCtaWarps; ++w) {
            const uint32_t x = cs.wU[w];
            if (w < wl) Pw += x;
            U += x;
          }
          if (Uw) {  // warp wl draws stream positions [P_w, P_w + U_w); lane l the 16 from P_w + 16 l
            const Xoshiro wst = warp_advance(p, s, Pw);
            const uint32_t r0 = 16u * lane;
            if (r0 < Uw) {
              Xoshiro st = wst;
              if (lane) gf2_jump_tables(p.jtab16 + static_cast<size_t>(lane - 1) * kJumpTableWords,
                                        st.a, st.b, st.c, st.d);
              uint32_t c = 0;
              for (uint32_t step = 8; step; step >>= 1)
                if (c + step < nch && ws.pre[c + step] <= r0) c += step;
              uint32_t m = ws.mask[c];
              for (uint32_t k2 = r0 - ws.pre[c]; k2; --k2) m &= m - 1;
              const uint32_t need = min(16u, Uw - r0);
              uint32_t acc = 0;
              for (uint32_t done = 0; done < need;) {
                if (!m) {
                  if (acc) atomicOr(&ws.acc[c], acc);
                  acc = 0;
                  m = ws.mask[++c];
                  continue;
                }
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                const uint64_t x = st.next();
                const uint32_t kh = static_cast<uint32_t>(x >> 32), th = ws.thr[32 * c + bit];
                if (kh < th || (kh == th && bern_tie(x, p.w, qj + wbase + 32 * c + bit)))
                  acc |= 1u << bit;
                ++done;
              }
              if (acc) atomicOr(&ws.acc[c], acc);
              if (Pw + r0 + need == U) {
                cs.st[0] = st.a;
                cs.st[1] = st.b;
                cs.st[2] = st.c;
                cs.st[3] = st.d;
              }
            }
          }
          __syncwarp();
          const uint32_t am_lane = lane < static_cast<int>(nch) ? ws.acc[lane] : 0u;
          uint32_t Aw = __popc(am_lane);
          for (int o = 16; o; o >>= 1) Aw += __shfl_xor_sync(kFull, Aw, o);
          if (lane == 0) cs.wA[wl] = Aw;
          __syncthreads();  // (2) accepted counts, the stream after the window
          if (U) s = Xoshiro{cs.st[0], cs.st[1], cs.st[2], cs.st[3]};
          uint32_t Apre = 0, A = 0;
          for (int w = 0; w < kCtaWarps; ++w) {
            const uint32_t x = cs.wA[w];
            if (w < wl) Apre += x;
            A += x;
          }
          if (A) {
            if (nmem + A > kCap) {
              ok = false;
            } else {
              uint32_t lg2 = lg;
              while (2 * (nmem + A) > (1u << lg2)) ++lg2;
              if (lg2 != lg) {  // grow: re-insert the members under a fresh tag
                lg = lg2;
                ++stag;
                for (uint32_t t = tid; t < nmem; t += kBlock) tab_insert_atomic(tab, stag, lg, mem[t]);
                __syncthreads();
              }
              uint32_t base = nmem + Apre;
              unsigned cmk = __ballot_sync(kFull, am_lane != 0);
              while (cmk) {  // accepted sources in CSR order
                const int c = __ffs(cmk) - 1;
                cmk &= cmk - 1;
                const uint32_t am = __shfl_sync(kFull, am_lane, c);
                if ((am >> lane) & 1u) {
                  const uint32_t v = ws.src[32 * c + lane];
                  mem[base + __popc(am & lanemask_lt())] = v;
                  tab_insert_atomic(tab, stag, lg, v);
                  cfilt_add(sf, v);
                }
                base += __popc(am);
              }
              nmem += A;
            }
          }
          if (tid == 0) atomicAdd(&p.ctl->windows, 1ull);
          __syncthreads();  // (3) members appended; cs fields free for the next window
          qj += E;
          if (qj == fe) {
            ++qi;
            if (qi < nmem) qj = p.off[mem[qi]];
          }
          continue;
        }
      }
      // ---- window layout: up to 256 queued in-lists from (qi, qj). The
      // barrier closing the previous window made its members visible.
      const uint32_t nq = nmem;
      const bool lvalid = qi + tid < nq;
      uint32_t lb = 0, le = 0;
      if (lvalid) {
        const uint32_t v = mem[qi + tid];
        lb = tid == 0 ? qj : p.off[v];
        le = p.off[v + 1];
      }
      const uint32_t len = le - lb;
      uint32_t incl = len;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) cs.wsum[wl] = incl;
      for (uint32_t t = tid; t < (1u << kCtaAmapLog); t += kBlock) cs.amap[t] = ~0ull;
      __syncthreads();
      if (tid == 0) {  // after the barrier: every thread has read the previous window's
        cs.cut = 0xffffffffu;
        cs.adv_qi = 0xffffffffu;
        cs.any_acc = 0;
      }
      uint32_t total = 0;
      for (int w = 0; w < kCtaWarps; ++w) {
        const uint32_t x = cs.wsum[w];
        if (w < wl) incl += x;
        total += x;
      }
      cs.lstart[tid] = lb;
      cs.lpre[tid] = lvalid ? incl - len : 0xffffffffu;
      __syncthreads();
      uint32_t ecur = min(kCtaWin, total);
      // ---- 1. warp wl classifies positions [wbase, wbase + 512) (status at window start)
      uint32_t mymask = 0;
      const uint32_t wend = wbase < ecur ? min(kWin, ecur - wbase) : 0u;
      // lists holding this warp's first and last position (warp-uniform); the
      // per-edge search then only spans [tlo, thi] -- usually one list
      uint32_t tlo = 0, thi = 0;
      if (wend) {
        for (uint32_t step = kBlock / 2; step; step >>= 1) {
          if (cs.lpre[tlo + step] <= wbase) tlo += step;
          if (cs.lpre[thi + step] <= wbase + wend - 1) thi += step;
        }
      }
      const uint32_t span = thi - tlo;
      const uint32_t top = span ? 1u << (31 - __clz(span)) : 0u;
      for (uint32_t c0 = 0; 32 * c0 < wend; c0 += 4) {
        uint2 r[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t el = 32 * (c0 + q4) + lane;
          r[q4] = make_uint2(0xffffffffu, 0u);
          if (el < wend) {
            const uint32_t e = wbase + el;
            uint32_t t = tlo;  // last list t in [tlo, thi] with lpre[t] <= e
            for (uint32_t step = top; step; step >>= 1)
              if (t + step <= thi && cs.lpre[t + step] <= e) t += step;
            r[q4] = __ldg(p.rec + cs.lstart[t] + (e - cs.lpre[t]));
          }
        }
        uint32_t vv[4], maybe = 0;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          vv[q4] = r[q4].x;
          maybe |= (32 * (c0 + q4) + lane < wend && cfilt_maybe(sf, vv[q4]) ? 1u : 0u) << q4;
        }
        const uint32_t seen = tab_contains_batch<4>(tab, stag, lg, vv, maybe);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t c = c0 + q4;
          if (32 * c >= wend) break;
          const uint32_t el = 32 * c + lane;
          const uint32_t v = r[q4].x;
          const bool unv = el < wend && !((seen >> q4) & 1u);
          if (unv) {
            ws.thr[el] = r[q4].y;
            ws.src[el] = v;
          }
          const unsigned m = __ballot_sync(kFull, unv);
          if (lane == static_cast<int>(c)) mymask = m;
        }
      }
      const uint32_t cnt = __popc(mymask);
      uint32_t ui = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, ui, o);
        if (lane >= o) ui += y;
      }
      const uint32_t Uw = __shfl_sync(kFull, ui, 31);
      if (lane < static_cast<int>(kWinChunks)) {
        ws.mask[lane] = mymask;
        ws.pre[lane] = ui - cnt;
        ws.acc[lane] = 0;
      }
      if (lane == 0) cs.wU[wl] = Uw;
      __syncthreads();
      uint32_t Pw = 0, U = 0;
      for (int w = 0; w < kCtaWarps; ++w) {
        const uint32_t x = cs.wU[w];
        if (w < wl) Pw += x;
        U += x;
      }
      bool cut = false;
      if (U) {
        // ---- 2. warp wl draws stream positions [P_w, P_w + U_w); lane l the
        // 16 from P_w + 16 l
        const uint32_t nch = (wend + 31) >> 5;
        if (Uw) {
          const Xoshiro wst = warp_advance(p, s, Pw);
          const uint32_t r0 = 16u * lane;
          if (r0 < Uw) {
            Xoshiro st = wst;
            if (lane) gf2_jump_tables(p.jtab16 + static_cast<size_t>(lane - 1) * kJumpTableWords,
                                      st.a, st.b, st.c, st.d);
            uint32_t c = 0;
            for (uint32_t step = 8; step; step >>= 1)
              if (c + step < nch && ws.pre[c + step] <= r0) c += step;
            uint32_t m = ws.mask[c];
            for (uint32_t k2 = r0 - ws.pre[c]; k2; --k2) m &= m - 1;
            const uint32_t need = min(16u, Uw - r0);
            uint32_t acc = 0;
            for (uint32_t done = 0; done < need;) {
              if (!m) {
                if (acc) atomicOr(&ws.acc[c], acc);
                acc = 0;
                m = ws.mask[++c];
                continue;
              }
              const int bit = __ffs(m) - 1;
              m &= m - 1;
              const uint64_t x = st.next();
              const uint32_t kh = static_cast<uint32_t>(x >> 32), th = ws.thr[32 * c + bit];
              if (kh < th ||
                  (kh == th && bern_tie(x, p.w, win_edge(cs.lstart, cs.lpre, kBlock, wbase + 32 * c + bit))))
                acc |= 1u << bit;
              ++done;
            }
            if (acc) atomicOr(&ws.acc[c], acc);
            if (Pw + r0 + need == U) {
              cs.st[0] = st.a;
              cs.st[1] = st.b;
              cs.st[2] = st.c;
              cs.st[3] = st.d;
            }
          }
        }
        __syncwarp();
        // ---- 3a. accepted sources -> first accepting position (CTA-wide map)
        uint32_t am_lane = lane < static_cast<int>(nch) ? ws.acc[lane] : 0u;
        const unsigned acm = __ballot_sync(kFull, am_lane != 0);
        uint32_t fail = 0xffffffffu;
        for (unsigned t = acm; t; t &= t - 1) {
          const int c = __ffs(t) - 1;
          const uint32_t am = __shfl_sync(kFull, am_lane, c);
          const uint32_t el = 32 * c + lane;
          if (((am >> lane) & 1u) && !amap_insert<kCtaAmapLog>(cs.amap, ws.src[el], wbase + el))
            fail = min(fail, wbase + el);
        }
        fail = __reduce_min_sync(kFull, fail);
        if (lane == 0) {
          if (fail != 0xffffffffu) atomicMin(&cs.cut, fail);
          if (acm) cs.any_acc = 1;
        }
        __syncthreads();
        if (cs.any_acc) {
          // ---- 3b. the first drawn edge whose source an earlier edge accepted
          const uint32_t lim = cs.cut;
          for (uint32_t c = 0; c < nch && wbase + 32 * c < lim; ++c) {
            const uint32_t m = ws.mask[c];
            if (!m) continue;
            const uint32_t el = 32 * c + lane;
            const bool conf = ((m >> lane) & 1u) &&
                              amap_first<kCtaAmapLog>(cs.amap, ws.src[el]) < wbase + el;
            const unsigned b = __ballot_sync(kFull, conf);
            if (b) {
              if (lane == 0) atomicMin(&cs.cut, wbase + 32 * c + __ffs(b) - 1);
              break;
            }
          }
          __syncthreads();
          const uint32_t cpos = cs.cut;
          if (cpos < ecur) {
            cut = true;
            const uint32_t cw = cpos / kWin, cl = cpos % kWin, cc = cl >> 5, cb = cl & 31;
            if (wl == static_cast<int>(cw)) {
              // the stream resumes after the draws of the edges before the cut
              const uint32_t Rl = ws.pre[cc] + __popc(ws.mask[cc] & ((1u << cb) - 1u));
              const Xoshiro wst = warp_advance(p, s, Pw);
              if (lane == static_cast<int>(Rl >> 4)) {
                Xoshiro st = wst;
                if (lane) gf2_jump_tables(p.jtab16 + static_cast<size_t>(lane - 1) * kJumpTableWords,
                                          st.a, st.b, st.c, st.d);
                for (uint32_t k2 = Rl & 15u; k2; --k2) st.next();
                cs.st[0] = st.a;
                cs.st[1] = st.b;
                cs.st[2] = st.c;
                cs.st[3] = st.d;
              }
              if (lane > static_cast<int>(cc)) am_lane = 0;
              else if (lane == static_cast<int>(cc)) am_lane &= (1u << cb) - 1u;
            } else if (wl > static_cast<int>(cw)) {
              am_lane = 0;
            }
            ecur = cpos;
          }
        }
        // ---- 4. append the accepted sources in window order
        uint32_t Aw = __popc(am_lane);
        for (int o = 16; o; o >>= 1) Aw += __shfl_xor_sync(kFull, Aw, o);
        if (lane == 0) cs.wA[wl] = Aw;
        __syncthreads();
        s = Xoshiro{cs.st[0], cs.st[1], cs.st[2], cs.st[3]};
        uint32_t Apre = 0, A = 0;
        for (int w = 0; w < kCtaWarps; ++w) {
          const uint32_t x = cs.wA[w];
          if (w < wl) Apre += x;
          A += x;
        }
        if (A) {
          if (nmem + A > kCap) {
            ok = false;
          } else {
            uint32_t lg2 = lg;
            while (2 * (nmem + A) > (1u << lg2)) ++lg2;
            if (lg2 != lg) {  // grow: re-insert the members under a fresh tag
              lg = lg2;
              ++stag;
              for (uint32_t t = tid; t < nmem; t += kBlock) tab_insert_atomic(tab, stag, lg, mem[t]);
              __syncthreads();
            }
            uint32_t base = nmem + Apre;
            unsigned cmk = __ballot_sync(kFull, am_lane != 0);
            while (cmk) {
              const int c = __ffs(cmk) - 1;
              cmk &= cmk - 1;
              const uint32_t am = __shfl_sync(kFull, am_lane, c);
              if ((am >> lane) & 1u) {
                const uint32_t v = ws.src[32 * c + lane];
                mem[base + __popc(am & lanemask_lt())] = v;
                tab_insert_atomic(tab, stag, lg, v);
                cfilt_add(sf, v);
              }
              base += __popc(am);
            }
            nmem += A;
          }
        }
      }
      if (tid == 0) {
        atomicAdd(&p.ctl->windows, 1ull);
        if (cut) atomicAdd(&p.ctl->cuts, 1ull);
      }
      // ---- advance past the ecur consumed edges: the first list not wholly consumed
      if (lvalid && incl > ecur && incl - len <= ecur) {
        cs.adv_qi = qi + tid;
        cs.adv_qj = lb + (ecur - (incl - len));
      }
      __syncthreads();
      if (cs.adv_qi != 0xffffffffu) {
        qi = cs.adv_qi;
        qj = cs.adv_qj;
      } else {
        qi += min(static_cast<uint32_t>(kBlock), nq - qi);
        if (qi < nmem) qj = p.off[mem[qi]];
      }
    }
    __syncthreads();
    // inspected in-edges of the set = sum of its members' in-degrees
    uint64_t sinsp = 0;
    if (ok)
      for (uint32_t t = tid; t < nmem; t += kBlock) sinsp += p.off[mem[t] + 1] - p.off[mem[t]];
    tag = stag;
    for (uint32_t t = tid; t < kCtaFilterWords; t += kBlock) sf[t] = 0;  // filter per sample
    if (!ok) {
      if (tid == 0) defer_slot(p, idx);
      continue;
    }
    if (tid == 0) cs.next = atomicAdd(&p.ctl->cursor, (unsigned long long)nmem);
    __syncthreads();
    const unsigned long long pos = cs.next;
    if (pos + nmem > p.stage_cap) {
      if (tid == 0) restage_slot(p, idx, nmem);
      continue;
    }
    for (uint32_t t = tid; t < nmem; t += kBlock) {
      const uint32_t v = mem[t];
      p.stage[pos + t] = v;
      if (p.counter) atomicAdd(p.counter + v, 1u);
    }
    if (tid == 0) {
      p.slot_start[idx] = pos;
      p.slot_len[idx] = nmem;
    }
    insp += sinsp;
  }
  for (int o = 16; o; o >>= 1) insp += __shfl_xor_sync(kFull, insp, o);
  if (lane == 0 && insp) {
    atomicAdd(&p.ctl->inspected, (unsigned long long)insp);
    atomicAdd(&p.ctl->entries, (unsigned long long)insp);
  }
  if (tid == 0) p.wtags[tslot] = tag;
}

// ---------------------------------------------------------------------------
// K1f: opt-in FAST IC sampler (RRG_OPT_IC_RNG = 1). Not
// the reference's draw sequence: every in-edge's liveness comes from a
// counter-based stream keyed by (slot, vertex, edge), so the lists of one
// vertex need no serial order and runs of equal weights are sampled by
// geometric skipping (the next live edge after G ~ Geometric(p) dead ones).
// Each edge is live with probability w independently, so a set is distributed
// as the reference's (the RIS reverse-reachable set over live edges); parity is
// statistical (tests/test_gpu_fast.py). Roots are the reference's (slot stream).
// Warp per sample: the warp takes one dequeued vertex at a time; a weight-
// uniform in-list is cut into 32 lane segments, each skipping with its own
// substream; other lists are drawn 32 edges per round. kBitmap: n-bit visited
// map + n-entry list (big-set scratch, no size cap), else the warp's 32-lane
// region table (32K members, larger sets deferred to the bitmap variant).
// ---------------------------------------------------------------------------
// Equal-weight in-lists are cut into fixed segments, each skipped with its own
// substream, so every variant (lane, warp, bitmap) draws the same live edges
// and a deferred slot is re-run to the same set.
constexpr uint32_t kFastSeg = 1u << 16;
__device__ __forceinline__ uint64_t fast_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// uniform in (0, 1] from draw i of the (slot, vertex) stream ku
__device__ __forceinline__ double fast_u01(uint64_t ku, uint64_t i) {
  return static_cast<double>((fast_mix(ku + 0x9e3779b97f4a7c15ULL * (i + 1)) >> 11) + 1) * 0x1.0p-53;
}

template <bool kBitmap>
__global__ void __launch_bounds__(kBlock) k_sample_ic_fast(const SampleParams p, uint32_t* bitmaps,
                                                           uint32_t* lists, uint32_t workers) {
  constexpr uint32_t kCap = kBitmap ? 0xffffffffu : 32 * kMemCap;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  uint32_t* mem;
  uint32_t* vis = nullptr;
  uint64_t* tab = nullptr;
  uint64_t tslot = 0;
  uint32_t tag = 0;
  if (kBitmap) {
    if (gw >= workers) return;
    const uint64_t words = (static_cast<uint64_t>(p.n) + 31) / 32;
    vis = bitmaps + gw * words;
    mem = lists + gw * p.n;
  } else {
    const uint64_t region = gw * 32;
    if (region + 32 > p.lanes) return;
    mem = p.lists + region * kMemCap;
    tab = p.tabs + region * kTabCap;
    tslot = region / 32;  // same layout and tag range as the 32-lane warp schedule
    tag = 0x80000000u | (p.wtags[tslot] & 0x3fffffffu);
  }
  uint64_t insp = 0;
  for (;;) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(&p.ctl->next, 1ull);
    k = __shfl_sync(kFull, k, 0);
    if (k >= p.count) break;
    const uint32_t idx = p.list ? p.list[k] : p.idx_base + static_cast<uint32_t>(k);
    const uint64_t seed = stream_seed(p.run_seed, p.base_slot + idx);
    Xoshiro rng;
    rng.seed(seed);
    const uint32_t root = static_cast<uint32_t>(rng.below(p.n));  // the reference's root
    const uint64_t key = fast_mix(seed ^ 0xD1B54A32D192ED03ULL);
    uint32_t lg = kTabLog0, nmem = 1;
    if (!kBitmap) ++tag;
    if (lane == 0) {
      mem[0] = root;
      if (kBitmap) vis[root >> 5] |= 1u << (root & 31);
      else tab_insert(tab, tag, lg, root);
    }
    __syncwarp();
    bool ok = true;
    uint64_t sinsp = 0;
    for (uint32_t qi = 0; qi < nmem && ok; ++qi) {
      const uint32_t u = mem[qi];
      const uint32_t b = p.off[u], e = p.off[u + 1];
      if (b == e) continue;
      sinsp += e - b;
      const uint64_t ku = fast_mix(key ^ (0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(u) + 1)));
      bool uni = p.uniformw[u] != 0;
      bool all_live = false;  // equal weights >= 1: every edge live, no draws
      double pw = 0.0, lq = 0.0;
      uint32_t sg = lane, pos = 0, s1 = 0, cnum = 0;  // lane: segments lane, lane + 32, ...
      const uint32_t nseg = (e - b + kFastSeg - 1) / kFastSeg;
      if (uni) {
        pw = static_cast<double>(__ldg(p.w + b));
        if (!(pw > 0.0)) continue;  // 0, negative, NaN: never live (prng.hpp:62)
        if (pw >= 1.0) {
          uni = false;
          all_live = true;
        }
        lq = pw >= 1.0 ? 0.0 : log1p(-pw);
        pos = b + sg * kFastSeg;
        s1 = sg < nseg ? min(e, pos + kFastSeg) : pos;
      }
      for (uint32_t c0 = b;; c0 += 32) {
        // one candidate per lane per round: the lane's next live edge
        uint32_t cand = 0xffffffffu;
        if (uni) {
          while (sg < nseg) {
            if (pos < s1 && pw < 1.0) {
              const double g = floor(log(fast_u01(ku, (static_cast<uint64_t>(sg) << 32) | cnum++)) / lq);
              pos = g >= static_cast<double>(s1 - pos) ? s1 : pos + static_cast<uint32_t>(g);
            }
            if (pos < s1) {
              cand = pos++;
              break;
            }
            sg += 32;  // the lane's next segment
            pos = b + sg * kFastSeg;
            s1 = sg < nseg ? min(e, pos + kFastSeg) : pos;
            cnum = 0;
          }
        } else {
          if (c0 >= e) break;
          const uint32_t t = c0 + lane;
          if (t < e && (all_live || fast_u01(ku, t - b) <= static_cast<double>(__ldg(p.w + t))))
            cand = t;
        }
        if (uni && !__any_sync(kFull, cand != 0xffffffffu)) break;
        const uint32_t v = cand != 0xffffffffu ? __ldg(p.src + cand) : 0xffffffffu;
        const unsigned peers = __match_any_sync(kFull, v);
        bool fresh = cand != 0xffffffffu && (peers & lanemask_lt()) == 0;  // first lane with v
        if (fresh) fresh = kBitmap ? !((vis[v >> 5] >> (v & 31)) & 1u) : !tab_contains(tab, tag, lg, v);
        const unsigned fm = __ballot_sync(kFull, fresh);
        if (fm) {
          const uint32_t A = __popc(fm);
          if (nmem + A > kCap) {
            ok = false;
            break;
          }
          if (!kBitmap) {
            uint32_t lg2 = lg;
            while (2 * (nmem + A) > (1u << lg2)) ++lg2;
            if (lg2 != lg) {  // grow: re-insert the members under a fresh tag
              lg = lg2;
              ++tag;
              for (uint32_t t = lane; t < nmem; t += 32) tab_insert_atomic(tab, tag, lg, mem[t]);
              __syncwarp();
            }
          }
          if (fresh) {
            mem[nmem + __popc(fm & lanemask_lt())] = v;
            if (kBitmap) atomicOr(vis + (v >> 5), 1u << (v & 31));
            else tab_insert_atomic(tab, tag, lg, v);
          }
          nmem += A;
        }
        __syncwarp();
      }
    }
    if (!ok) {
      if (lane == 0) defer_slot(p, idx);
    } else {
      unsigned long long spos = 0;
      if (lane == 0) spos = atomicAdd(&p.ctl->cursor, (unsigned long long)nmem);
      spos = __shfl_sync(kFull, spos, 0);
      if (spos + nmem > p.stage_cap) {
        if (lane == 0) restage_slot(p, idx, nmem);
      } else {
        for (uint32_t t = lane; t < nmem; t += 32) {
          const uint32_t v = mem[t];
          p.stage[spos + t] = v;
          if (p.counter) atomicAdd(p.counter + v, 1u);
        }
        if (lane == 0) {
          p.slot_start[idx] = spos;
          p.slot_len[idx] = nmem;
        }
        insp += sinsp;
      }
    }
    if (kBitmap) {
      for (uint32_t t = lane; t < nmem; t += 32) {
        const uint32_t v = mem[t];
        atomicAnd(vis + (v >> 5), ~(1u << (v & 31)));
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (!kBitmap) p.wtags[tslot] = tag;
    atomicAdd(&p.ctl->inspected, (unsigned long long)insp);
    atomicAdd(&p.ctl->entries, (unsigned long long)insp);
  }
}

// Lane per sample variant of the fast sampler (light sets, e.g. cfg3): the lane
// walks its own BFS; an equal-weight in-list costs one geometric draw per live
// edge (+1), any other list one hash draw per edge. Sets beyond the lane's 1K
// members are deferred to the warp variant.
__global__ void __launch_bounds__(kBlock) k_sample_ic_fast_lane(const SampleParams p) {
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t* mem = p.lists + gid * kMemCap;
  uint64_t* tab = p.tabs + gid * kTabCap;
  uint32_t tag = p.tags[gid];
  bool exhausted = false;
  uint64_t insp = 0;
  for (;;) {
    uint32_t idx = 0;
    const bool got = fetch_slot(p, !exhausted, exhausted, idx);
    if (__all_sync(kFull, exhausted)) break;
    if (!got) continue;
    const uint64_t seed = stream_seed(p.run_seed, p.base_slot + idx);
    Xoshiro rng;
    rng.seed(seed);
    const uint32_t root = static_cast<uint32_t>(rng.below(p.n));  // the reference's root
    const uint64_t key = fast_mix(seed ^ 0xD1B54A32D192ED03ULL);
    ++tag;
    uint32_t lg = kTabLog0, nmem = 1;
    Filter flt;
    flt.clear();
    mem[0] = root;
    tab_insert(tab, tag, lg, root);
    flt.add(root);
    bool ok = true;
    uint64_t sinsp = 0;
    for (uint32_t qi = 0; qi < nmem && ok; ++qi) {
      const uint32_t u = mem[qi];
      const uint32_t b = p.off[u], e = p.off[u + 1];
      if (b == e) continue;
      sinsp += e - b;
      const uint64_t ku = fast_mix(key ^ (0x9e3779b97f4a7c15ULL * (static_cast<uint64_t>(u) + 1)));
      const bool uni = p.uniformw[u] != 0;
      double pw = 0.0, lq = 0.0;
      if (uni) {
        pw = static_cast<double>(__ldg(p.w + b));
        if (!(pw > 0.0)) continue;
        lq = pw >= 1.0 ? 0.0 : log1p(-pw);
      }
      uint32_t cnum = 0, send = min(e, b + kFastSeg);
      for (uint32_t t = b; t < e; ++t) {
        if (uni) {
          if (pw < 1.0) {  // the next live edge: skip G ~ Geometric(pw) dead ones
            const double g = floor(log(fast_u01(ku, (static_cast<uint64_t>((t - b) / kFastSeg) << 32) | cnum++)) / lq);
            if (g >= static_cast<double>(send - t)) {  // segment exhausted: the next one
              t = send - 1;
              send = min(e, send + kFastSeg);
              cnum = 0;
              continue;
            }
            t += static_cast<uint32_t>(g);
          }
        } else if (fast_u01(ku, t - b) > static_cast<double>(__ldg(p.w + t))) {
          continue;
        }
        const uint32_t v = __ldg(p.src + t);
        if (flt.maybe(v) && tab_contains(tab, tag, lg, v)) continue;
        if (nmem == kMemCap) {
          ok = false;
          break;
        }
        lane_insert(mem, tab, tag, lg, nmem, v);
        flt.add(v);
      }
    }
    if (!ok) {
      defer_slot(p, idx);
    } else if (emit_set(p, idx, mem, nmem)) {
      insp += sinsp;
    }
  }
  p.tags[gid] = tag;
  flush_counters(p, insp, insp);
}

// K0 for the fast sampler: 1 iff every in-weight of the vertex has the same bits.
__global__ void k_uniform_weights(const uint32_t* off, const float* w, uint32_t n, uint8_t* out) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t b = off[v], e = off[v + 1];
    const uint32_t w0 = b < e ? __float_as_uint(w[b]) : 0u;
    bool same = true;
    for (uint32_t t = b + lane; t < e && same; t += 32) same = __float_as_uint(w[t]) == w0;
    same = __all_sync(kFull, same);
    if (lane == 0) out[v] = (b < e && same) ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// K2: LT sampler (sampling.hpp:117-145 per slot)
// ---------------------------------------------------------------------------
constexpr uint32_t kLtTabLog0 = 8;        // walks average ~80 steps (cfg4): fewer rehashes

template <int KARY>
__global__ void __launch_bounds__(kBlock) k_sample_lt(const SampleParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t* mem = p.lists + gid * kMemCap;
  uint64_t* tab = p.tabs + gid * kTabCap;
  uint32_t tag = p.tags[gid];
  Xoshiro rng{0, 0, 0, 0};
  bool active = false, exhausted = false;
  uint32_t idx = 0, nmem = 0, lg = kTabLog0, u = 0;
  uint32_t nb = 0, ne = 0;  // in-list bounds of u, loaded as soon as u is known
  uint64_t insp = 0, sinsp = 0, ent = 0;
  const bool linear = p.lt_scan == kLtLinear;
  // search mode: u's 64-byte vertex record (k_build_ltrec), loaded as soon as
  // u is known -- bounds, and the whole list or the first search level
  const bool recs = !linear && p.ltrec != nullptr;
  uint4 rr[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) rr[i] = make_uint4(0, 0, 0, 0);

  for (;;) {
    if (fetch_slot(p, !active && !exhausted, exhausted, idx)) {
      rng.seed(stream_seed(p.run_seed, p.base_slot + idx));
      u = static_cast<uint32_t>(rng.below(p.n));
      if (recs) {
#pragma unroll
        for (int i = 0; i < 4; ++i) rr[i] = __ldg(p.ltrec + static_cast<size_t>(u) * 4 + i);
      } else {
        nb = p.off[u];
        ne = p.off[u + 1];
      }
      ++tag;
      lg = kLtTabLog0;
      mem[0] = u;
      nmem = 1;
      sinsp = 0;
      tab_insert(tab, tag, lg, u);
      active = true;
    }
    if (__all_sync(kFull, !active)) break;

    // one walk step for every active lane
    uint32_t b = 0, e = 0;
    double d = 0.0;
    if (active) {
      d = rng.u01();  // sampling.hpp:127 -- always consumed
      b = recs ? rr[0].x : nb;
      e = recs ? rr[0].x + rr[0].y : ne;
    }
    uint32_t vsel = 0;  // source of `pick` when the search already loaded it
    uint32_t pick = e;  // index of the first cdf entry > d, or e for "none"
    uint32_t slo = b, shi = e;  // search range: answer (first cdf > d, or e) in [slo, shi]
    bool picked = false;        // resolved from the vertex record alone
    if (recs && active) {
      const uint32_t deg = e - b;
      const uint32_t dbits = __float_as_uint(__double2float_rd(d));  // d in [0, 1)
      const uint32_t* w = reinterpret_cast<const uint32_t*>(rr);
      if (deg <= kLtRecSmall) {  // whole list in the record: count entries <= d
        const uint32_t cnt = lt_count_le<kLtRecSmall>(w + 2, dbits, d, p.cdf, b, 1);
#pragma unroll
        for (uint32_t t = 0; t < kLtRecSmall; ++t)
          if (t == cnt) vsel = w[8 + t];
        pick = b + cnt;
        ent += deg;
        picked = true;
      } else {  // the root's 13 pivots, then the vertex's search-tree nodes
        uint32_t lo = b, hi = e;
        const uint32_t st0 = lt_step(lo, hi, kLtRootPivots);
        const uint32_t below = lt_count_le<kLtRootPivots>(w + 3, dbits, d, p.cdf, lo + st0, st0);
        ent += kLtRootPivots;
        lt_child(lo, hi, kLtRootPivots, below);
        uint64_t level_base = w[2], idx = below, width = kLtRootFanout;
        while (hi - lo > kLtLeafMin) {  // one 128-byte node per level
          const uint4* nd = reinterpret_cast<const uint4*>(p.ltnodes + (level_base + idx) * 32);
          uint4 q[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) q[i] = __ldg(nd + i);
          const uint32_t* qw = reinterpret_cast<const uint32_t*>(q);
          if (hi - lo <= kLtLeafMax) {  // leaf: cdf[lo, hi) and src[lo, hi] resolve the step
            const uint32_t cnt = lt_count_le<kLtLeafMax>(qw, dbits, d, p.cdf, lo, 1);
#pragma unroll
            for (uint32_t t = 0; t <= kLtLeafMax; ++t)
              if (t == cnt) vsel = qw[kLtLeafMax + t];
            ent += hi - lo;
            pick = lo + cnt;
            picked = true;
            break;
          }
          const uint32_t st = lt_step(lo, hi, kLtNodePivots);
          const uint32_t bl = lt_count_le<kLtNodePivots>(qw, dbits, d, p.cdf, lo + st, st);
          ent += kLtNodePivots;
          lt_child(lo, hi, kLtNodePivots, bl);
          level_base += width;
          idx = idx * kLtFanout + bl;
          width *= kLtFanout;
        }
        slo = lo;
        shi = hi;
      }
    }
    const bool coop = active && linear && (e - b) >= p.coop_min;
    unsigned cm = __ballot_sync(kFull, coop);
    while (cm) {
      // warp-cooperative linear scan of one lane's long in-list: 4 x 64 entries
      // per iteration (four independent 16-byte loads per lane in flight), the
      // first hit located by ballot
      const int L = __ffs(cm) - 1;
      cm &= cm - 1;
      const uint32_t bL = __shfl_sync(kFull, b, L);
      const uint32_t eL = __shfl_sync(kFull, e, L);
      const double dL = __shfl_sync(kFull, d, L);
      uint32_t found = eL;
      uint64_t read = 0;
      for (uint32_t base = bL & ~1u; base < eL && found == eL; base += 256) {
        double2 c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i0 = base + 64 * u + 2 * lane;
          c[u] = i0 < eL ? __ldg(reinterpret_cast<const double2*>(p.cdf + i0))
                         : make_double2(0.0, 0.0);
        }
        read += min(256u, eL - base);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i0 = base + 64 * u + 2 * lane;
          const bool h0 = i0 < eL && i0 >= bL && dL < c[u].x;
          const bool h1 = i0 + 1 < eL && i0 + 1 >= bL && dL < c[u].y;
          const unsigned hm = __ballot_sync(kFull, h0 || h1);
          if (hm) {
            const int f = __ffs(hm) - 1;
            const unsigned first0 = __ballot_sync(kFull, h0);
            found = base + 64 * u + 2 * f + (((first0 >> f) & 1u) ? 0 : 1);
            break;
          }
        }
      }
      if (lane == L) {
        pick = found;
        ent += read;
      }
    }
    if (active && !coop && !picked) {
      if (linear) {
        for (uint32_t t = b; t < e; ++t) {
          if (d < p.cdf[t]) {
            pick = t;
            break;
          }
        }
        ent += (pick < e ? pick + 1 : e) - b;
      } else {
        // upper_bound (first cdf[t] > d; cdf non-decreasing) as a K-ary search:
        // K-1 independent pivot loads per level keep the dependent round trips
        // at logK(deg) instead of log2(deg). Invariant: answer in [lo, hi].
        uint32_t lo = slo, hi = shi;
        while (hi - lo > static_cast<uint32_t>(KARY)) {
          const uint32_t step = (hi - lo) / KARY;
          uint32_t below = 0;  // pivots with cdf <= d form a prefix
#pragma unroll
          for (uint32_t t = 1; t < KARY; ++t)
            below += __ldg(p.cdf + lo + t * step) <= d ? 1u : 0u;
          ent += KARY - 1;
          const uint32_t nlo = below ? lo + below * step + 1 : lo;
          hi = below < KARY - 1 ? lo + (below + 1) * step : hi;
          lo = nlo;
        }
        // last level: the <= K entries of [lo, hi) and the sources of [lo, hi]
        // in one round trip (independent loads); pick = lo + #(cdf <= d)
        uint32_t cnt = 0;
        uint32_t sv[KARY + 1];
#pragma unroll
        for (uint32_t t = 0; t <= static_cast<uint32_t>(KARY); ++t) {
          const uint32_t i = lo + t;
          sv[t] = i < e && i <= hi ? __ldg(p.src + i) : 0u;
          if (t < static_cast<uint32_t>(KARY) && i < hi && __ldg(p.cdf + i) <= d) ++cnt;
        }
        ent += hi - lo;
        pick = lo + cnt;
#pragma unroll
        for (uint32_t t = 0; t <= static_cast<uint32_t>(KARY); ++t)
          if (t == cnt) vsel = sv[t];
      }
    }
    if (!active) continue;
    sinsp += (pick < e ? pick + 1 : e) - b;  // reference trip count (sampling.hpp:130-136)
    bool stop = pick >= e;
    uint32_t v = 0;
    if (!stop) {
      v = (linear || coop) ? p.src[pick] : vsel;
      if (recs) {  // next step's record, in flight with the visited probe
#pragma unroll
        for (int i = 0; i < 4; ++i) rr[i] = __ldg(p.ltrec + static_cast<size_t>(v) * 4 + i);
      } else {
        nb = p.off[v];  // next step's list, in flight with the visited probe
        ne = p.off[v + 1];
      }
      stop = tab_find_or_insert(tab, tag, lg, v);  // chosen already visited (:137)
    }
    if (stop) {
      if (emit_set(p, idx, mem, nmem)) insp += sinsp;
      active = false;
    } else if (nmem == kMemCap) {
      defer_slot(p, idx);
      active = false;
    } else {  // v is in the table already (tab_find_or_insert)
      mem[nmem++] = v;
      if (2 * nmem > (1u << lg)) {  // grow: re-insert under a fresh tag
        ++lg;
        ++tag;
        for (uint32_t t = 0; t < nmem; ++t) tab_insert(tab, tag, lg, mem[t]);
      }
      u = v;
    }
  }
  p.tags[gid] = tag;
  flush_counters(p, insp, ent);
}

// Guide-mode LT step resolution (common.cuh, "LT guide table"): the bucket
// entry (e0, e1) of vertex u for draw x gives the chosen index `pick` (local;
// deg_u = none) and what the next step needs of the chosen source.
__device__ __forceinline__ void lt_guide_resolve(const SampleParams& p, const uint4 e0,
                                                 const uint4 e1, uint64_t x, uint32_t offu,
                                                 uint32_t degu, uint32_t& pick, uint32_t& v,
                                                 uint32_t& offv, uint32_t& degv, uint64_t& ent) {
  const uint32_t A = e0.x;
  const uint32_t pw = e0.y;
  if (pw & kGuideSpan0) {  // no CDF entry inside the bucket: index A_g whatever the draw
    pick = A;
    v = e0.z;
    offv = e0.w;
    degv = e1.x;
    return;
  }
  const double d = __ull2double_rn(x >> 11) * 0x1.0p-53;  // uniform01(), exact
  const uint32_t dbits = __float_as_uint(__double2float_rd(d));
  if (!(pw & kGuideSearch)) {  // one entry: pick A_g + [cdf[A_g] <= d]
    const uint32_t f = pw & kGuidePivot;
    const bool le = f < dbits || (f == dbits && __ldg(p.cdf + offu + A) <= d);
    if (le) {
      pick = A + 1;
      v = e1.y;
      offv = e1.z;
      degv = e1.w;
    } else {
      pick = A;
      v = e0.z;
      offv = e0.w;
      degv = e1.x;
    }
    return;
  }
  // span >= 2 (rare): count cdf[A_g, A_g + span) <= d, eight loads in flight
  const uint32_t span = e1.y;
  const double* c = p.cdf + offu + A;
  uint32_t cnt = 0;
  for (uint32_t t = 0; t < span; t += 8) {
    double q[8];
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) q[k] = t + k < span ? __ldg(c + t + k) : 2.0;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) cnt += q[k] <= d ? 1u : 0u;
    if (cnt < t + 8) break;  // the entries are sorted: the first one > d ends the count
  }
  ent += span;
  pick = A + cnt;
  if (pick < degu) {
    v = __ldg(p.src + offu + pick);
    offv = __ldg(p.off + v);
    degv = __ldg(p.off + v + 1) - offv;
  } else {
    v = kGuideNone;
  }
}

__device__ __forceinline__ void lt_guide_fetch(const SampleParams& p, uint32_t offu, uint32_t degu,
                                               uint64_t x, uint4& e0, uint4& e1) {
  if (!degu) return;
  const uint64_t G = static_cast<uint64_t>(degu) * p.lt_guide_mult;
  const uint64_t gi = static_cast<uint64_t>(offu) * p.lt_guide_mult + __umul64hi(x & ~0x7ffull, G);
  // one 256-bit load (sm_100: LDG.256), not allocated in L1: the entry is one
  // 32-byte sector and is never re-read by this SM
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(e0.x), "=r"(e0.y), "=r"(e0.z), "=r"(e0.w), "=r"(e1.x), "=r"(e1.y),
                 "=r"(e1.z), "=r"(e1.w)
               : "l"(p.ltguide + 2 * gi));
}

// Visited set of a guide-mode walk while it is short: a 2048-bit filter per lane
// (1024 in the A/B variant) in shared memory (two bits per member; lane words
// interleaved across the block, so every access is bank-conflict free) in front
// of the walk's member list. Only a filter hit scans the list (the whole warp, one round trip), so
// the common "not visited" answer never leaves the SM, and the per-lane hash
// tables (global memory, DRAM-bound once 150K lanes each own one) are used only
// by walks longer than kLtFiltMax members.
constexpr uint32_t kTabLog = 11;  // 2^11 = kTabCap entries: load <= 1/2 up to kMemCap members
static_assert((1u << kTabLog) == kTabCap, "guide-mode tables use the whole lane table");
// kFiltLog: log2 of the filter words per lane (5: 1024 bits, 6: 2048 bits)
template <int kFiltLog>
__device__ __forceinline__ void lfilt_bits(uint32_t v, uint32_t& w1, uint32_t& b1, uint32_t& w2,
                                           uint32_t& b2) {
  const uint32_t h = v * 0x9E3779B1u;
  w1 = h >> (32 - kFiltLog);
  b1 = (h >> (27 - kFiltLog)) & 31u;
  w2 = (h >> (22 - kFiltLog)) & ((1u << kFiltLog) - 1u);
  b2 = (h >> (17 - kFiltLog)) & 31u;
}
// Warp-cooperative emit (all 32 lanes, converged): every lane with `pending`
// has a finished set in its own member list; the warp copies them one after the
// other into staging -- each set's members loaded 32 per round trip by the whole
// warp (instead of 8 per round trip by its lane while the warp's other lanes
// wait at the reconvergence point) -- with the fused counter increments.
// Returns, to each pending lane, whether its set was written (false: staging
// full; the slot was recorded for a re-run).
// Staging positions come from a warp-private chunk of kStageChunk members
// (sc_next/sc_end, warp-uniform) refilled from the shared cursor, so the
// returning atomic on that one address is paid once per chunk, not per set;
// the host reserves grid-warps x kStageChunk of slack for the chunk tails.
constexpr uint32_t kStageChunk = 2048;
__device__ __forceinline__ bool warp_emit_pending(const SampleParams& p, bool pending,
                                                  uint32_t idx, uint32_t nmem,
                                                  const uint32_t* lists_warp,
                                                  uint64_t& sc_next, uint64_t& sc_end) {
  const int lane = threadIdx.x & 31;
  unsigned em = __ballot_sync(kFull, pending);
  bool mine = false;
  while (em) {
    const int L = __ffs(em) - 1;
    em &= em - 1;
    const uint32_t nL = __shfl_sync(kFull, nmem, L);
    const uint32_t iL = __shfl_sync(kFull, idx, L);
    unsigned long long pos = 0;
    if (sc_end - sc_next >= nL) {
      pos = sc_next;
      sc_next += nL;
    } else {
      const uint32_t take = nL > kStageChunk ? nL : kStageChunk;
      if (lane == L) pos = atomicAdd(&p.ctl->cursor, (unsigned long long)take);
      pos = __shfl_sync(kFull, pos, L);
      if (take == kStageChunk) {
        sc_next = pos + nL;
        sc_end = pos + take < p.stage_cap ? pos + take : p.stage_cap;
      }
    }
    if (pos + nL > p.stage_cap) {
      if (lane == L) restage_slot(p, iL, nL);
      continue;
    }
    const uint32_t* __restrict__ src = lists_warp + static_cast<size_t>(L) * kMemCap;
    uint32_t* __restrict__ out = p.stage + pos;
    for (uint32_t t = 0; t < nL; t += 128) {
      uint32_t v[4];
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) {
        const uint32_t i = t + 32 * k + lane;
        v[k] = i < nL ? src[i] : 0u;
      }
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) {
        const uint32_t i = t + 32 * k + lane;
        if (i < nL) {
          out[i] = v[k];
          if (p.counter) atomicAdd(p.counter + v[k], 1u);
        }
      }
    }
    if (lane == L) {
      p.slot_start[iL] = pos;
      p.slot_len[iL] = nL;
      mine = true;
    }
  }
  return mine;
}

// K2g: LT walk, guide mode. Lane per walk; every step is ONE 32-byte load (the
// bucket entry of the current vertex for this step's draw), issued as soon as
// the previous step chose its source; the draw of the step after is computed
// while it is in flight, and the chosen source's visited test runs against the
// shared-memory filter. Same index as the reference's linear scan
// (sampling.hpp:127-137), same draws in the same order.
template <int kFiltLog, uint32_t kLtFiltMax, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_sample_lt_guide(const SampleParams p) {
  constexpr uint32_t kLtFiltWords = 1u << kFiltLog;
  extern __shared__ uint32_t filt_all[];  // kLtFiltWords * kBlock words
  uint32_t* filt = filt_all + threadIdx.x;  // word w at filt[w * kBlock]
  const int lane = threadIdx.x & 31;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t* mem = p.lists + gid * kMemCap;
  const uint32_t* lists_warp = p.lists + (gid - lane) * kMemCap;
  uint64_t* tabs_warp = p.tabs + (gid - lane) * kTabCap;
  uint64_t* tab = p.tabs + gid * kTabCap;
  uint32_t tag = p.tags[gid];
  Xoshiro rng{0, 0, 0, 0};
  // per-lane walk state; `pending` / `check` / `rebuild` are resolved by the
  // whole warp at the top of the loop
  bool active = false, exhausted = false, big = false;
  bool pending = false;  // walk ended: its set waits for the cooperative emit
  bool check = false;    // chosen source vchk hit the filter: scan the members
  bool rebuild = false;  // walk reached kLtFiltMax members: fill its hash table
  uint32_t idx = 0, nmem = 0;
  uint32_t offu = 0, degu = 0, vchk = 0, offc = 0, degc = 0;
  uint64_t x = 0, xn = 0;  // this step's draw (its entry is in e0/e1) and the next step's
  uint4 e0 = make_uint4(0, 0, 0, 0), e1 = make_uint4(0, 0, 0, 0);
  uint64_t insp = 0, sinsp = 0, ent = 0;
  uint64_t wq_next = 0, wq_end = 0, sc_next = 0, sc_end = 0;  // warp-uniform queues

  for (;;) {
    // (1) filter hits: the warp scans each such lane's members (<= kLtFiltMax,
    //     one round trip) for its chosen source
    unsigned cm = __ballot_sync(kFull, check);
    while (cm) {
      const int L = __ffs(cm) - 1;
      cm &= cm - 1;
      const uint32_t nL = __shfl_sync(kFull, nmem, L);
      const uint32_t vL = __shfl_sync(kFull, vchk, L);
      const uint32_t* mL = lists_warp + static_cast<size_t>(L) * kMemCap;
      uint32_t q[kLtFiltMax / 32];
#pragma unroll
      for (uint32_t k = 0; k < kLtFiltMax / 32; ++k) {
        const uint32_t i = 32 * k + lane;
        q[k] = i < nL ? mL[i] : kGuideNone;
      }
      bool hit = false;
#pragma unroll
      for (uint32_t k = 0; k < kLtFiltMax / 32; ++k) hit |= q[k] == vL;
      hit = __any_sync(kFull, hit);
      if (lane == L) {
        check = false;
        if (hit) {  // chosen already visited (sampling.hpp:137): the walk ends
          pending = true;
          active = false;
        } else {  // a new member; its next step's entry is already in flight
          uint32_t w1, b1, w2, b2;
          lfilt_bits<kFiltLog>(vL, w1, b1, w2, b2);
          filt[w1 * kBlock] |= 1u << b1;
          filt[w2 * kBlock] |= 1u << b2;
          mem[nmem++] = vL;
          offu = offc;
          degu = degc;
          rebuild = nmem == kLtFiltMax;
        }
      }
    }
    // (2) finished walks -> staging (cooperative copy + fused counter)
    if (warp_emit_pending(p, pending, idx, nmem, lists_warp, sc_next, sc_end)) insp += sinsp;
    pending = false;
    // (3) walks that outgrew the filter: the warp inserts their members into
    //     their (fresh-tagged) per-lane tables, kTabCap entries, load <= 1/2
    unsigned rm = __ballot_sync(kFull, rebuild);
    if (rebuild) {
      ++tag;
      big = true;
      rebuild = false;
    }
    while (rm) {
      const int L = __ffs(rm) - 1;
      rm &= rm - 1;
      const uint32_t nL = __shfl_sync(kFull, nmem, L);
      const uint32_t tL = __shfl_sync(kFull, tag, L);
      const uint32_t* mL = lists_warp + static_cast<size_t>(L) * kMemCap;
      uint64_t* tL_tab = tabs_warp + static_cast<size_t>(L) * kTabCap;
      for (uint32_t i = lane; i < nL; i += 32) tab_insert_atomic(tL_tab, tL, kTabLog, mL[i]);
    }
    __syncwarp();

    if (fetch_slot_q(p, !active && !exhausted, exhausted, idx, wq_next, wq_end)) {
      rng.seed(stream_seed(p.run_seed, p.base_slot + idx));
      const uint32_t u = static_cast<uint32_t>(rng.below(p.n));
      offu = __ldg(p.off + u);
      degu = __ldg(p.off + u + 1) - offu;
      x = rng.next();  // the first step's draw (sampling.hpp:127)
      lt_guide_fetch(p, offu, degu, x, e0, e1);
      xn = rng.next();
#pragma unroll
      for (uint32_t w = 0; w < kLtFiltWords; ++w) filt[w * kBlock] = 0u;
      uint32_t w1, b1, w2, b2;
      lfilt_bits<kFiltLog>(u, w1, b1, w2, b2);
      filt[w1 * kBlock] |= 1u << b1;
      filt[w2 * kBlock] |= 1u << b2;
      big = false;
      mem[0] = u;
      nmem = 1;
      sinsp = 0;
      active = true;
    }
    if (__all_sync(kFull, !active)) break;
    if (!active) continue;

    uint32_t pick = degu, v = kGuideNone, offv = 0, degv = 0;
    if (degu) {
      lt_guide_resolve(p, e0, e1, x, offu, degu, pick, v, offv, degv, ent);
      ent += 4;  // the 32-byte bucket entry (in 8-byte units)
    }
    sinsp += pick < degu ? pick + 1 : degu;  // reference trip count (sampling.hpp:130-136)
    bool stop = v == kGuideNone;
    if (!stop) {
      lt_guide_fetch(p, offv, degv, xn, e0, e1);  // next step's entry, in flight now
      x = xn;
      xn = rng.next();
      if (big) {
        stop = tab_find_or_insert(tab, tag, kTabLog, v);  // chosen already visited (:137)
      } else {
        uint32_t w1, b1, w2, b2;
        lfilt_bits<kFiltLog>(v, w1, b1, w2, b2);
        const uint32_t f1 = filt[w1 * kBlock], f2 = filt[w2 * kBlock];
        if ((f1 >> b1) & (f2 >> b2) & 1u) {  // maybe visited: the warp scans (1)
          check = true;
          vchk = v;
          offc = offv;
          degc = degv;
          continue;
        }
        filt[w1 * kBlock] |= 1u << b1;
        filt[w2 * kBlock] |= 1u << b2;
      }
    }
    if (stop) {  // written by the warp at the top of the loop
      pending = true;
      active = false;
    } else if (nmem == kMemCap) {
      defer_slot(p, idx);
      active = false;
    } else {
      mem[nmem++] = v;
      rebuild = !big && nmem == kLtFiltMax;
      offu = offv;
      degu = degv;
    }
  }
  p.tags[gid] = tag;
  flush_counters(p, insp, ent);
}

// ---------------------------------------------------------------------------
// Big-set path: warp per deferred slot with an n-bit visited map. IC: the warp
// loads 32 in-edges per chunk (coalesced), tests visited and computes the
// Bernoulli thresholds in parallel, lane 0 (the slot's RNG) draws only for
// the unvisited edges in CSR order, and the accepted sources are appended in
// lane order. A chunk whose sources repeat falls back to lane 0 replaying it
// edge by edge against the live map, so the sequential semantics hold exactly.
// LT walks are replayed serially by lane 0. The warp writes out and clears.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_sample_big(const SampleParams p, const int model,
                                                       const uint32_t* list, const uint32_t nlist,
                                                       uint32_t* bitmaps, uint32_t* lists,
                                                       const uint32_t workers) {
  __shared__ uint64_t s_thr[kBlock / 32][32];
  __shared__ uint32_t s_src[kBlock / 32][32];
  __shared__ CoopSmem coop_sm[kBlock / 32];
  const int lane = threadIdx.x & 31;
  const int wl = threadIdx.x >> 5;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= workers) return;
  const uint64_t words = (static_cast<uint64_t>(p.n) + 31) / 32;
  uint32_t* vis = bitmaps + w * words;
  uint32_t* mem = lists + static_cast<uint64_t>(w) * p.n;
  uint64_t insp = 0;  // lane 0: committed; sinsp: this set
  for (uint32_t t = w; t < nlist; t += workers) {
    const uint32_t idx = list[t];
    uint32_t nmem = 0;
    uint64_t sinsp = 0;
    Xoshiro rng;
    rng.seed(stream_seed(p.run_seed, p.base_slot + idx));
    const uint32_t root = static_cast<uint32_t>(rng.below(p.n));
    if (model == RRG_IC) {
      if (lane == 0) {
        mem[0] = root;
        vis[root >> 5] |= 1u << (root & 31);
      }
      nmem = 1;
      __syncwarp();
      for (uint32_t head = 0; head < nmem; ++head) {
        const uint32_t uu = mem[head];
        const uint32_t jb = p.off[uu], je = p.off[uu + 1];
        sinsp += je - jb;
        if (je - jb >= p.ic_coop_min && p.dupfree[uu]) {
          CoopState s{rng.a, rng.b, rng.c, rng.d, 0, 0, 0, 0, nmem};
          coop_expand<kVisBitmap>(p, jb, je, mem, nullptr, vis, s, coop_sm[wl]);
          rng = Xoshiro{s.a, s.b, s.c, s.d};
          nmem = s.nmem;
          __syncwarp();
          continue;
        }
        for (uint32_t base = jb; base < je; base += 32) {
          const uint32_t j = base + lane;
          const bool valid = j < je;
          const uint2 r = valid ? p.rec[j] : make_uint2(0xffffffffu, 0);
          const bool unv = valid && !((vis[r.x >> 5] >> (r.x & 31)) & 1u);
          const unsigned peers = __match_any_sync(kFull, r.x);
          const bool dup = valid && (peers & lanemask_lt()) != 0;
          const unsigned um = __ballot_sync(kFull, unv);
          s_thr[wl][lane] = valid ? bernoulli_threshold(__float_as_uint(__ldg(p.w + j))) : 0ull;
          s_src[wl][lane] = r.x;
          __syncwarp();
          unsigned acc = 0;
          const bool any_dup = __any_sync(kFull, dup);
          if (lane == 0) {
            if (!any_dup) {
              for (unsigned mm = um; mm; mm &= mm - 1) {
                const int l = __ffs(mm) - 1;
                if (rng.u53() < s_thr[wl][l]) acc |= 1u << l;
              }
            } else {
              const int nv = static_cast<int>(min(32u, je - base));
              for (int l = 0; l < nv; ++l) {  // edge-by-edge against the live map
                const uint32_t v = s_src[wl][l];
                if ((vis[v >> 5] >> (v & 31)) & 1u) continue;
                if (rng.u53() < s_thr[wl][l]) {
                  vis[v >> 5] |= 1u << (v & 31);
                  acc |= 1u << l;
                }
              }
            }
          }
          acc = __shfl_sync(kFull, acc, 0);
          rng.a = __shfl_sync(kFull, rng.a, 0);  // keep the stream warp-uniform
          rng.b = __shfl_sync(kFull, rng.b, 0);
          rng.c = __shfl_sync(kFull, rng.c, 0);
          rng.d = __shfl_sync(kFull, rng.d, 0);
          if ((acc >> lane) & 1u) {
            mem[nmem + __popc(acc & lanemask_lt())] = r.x;
            atomicOr(vis + (r.x >> 5), 1u << (r.x & 31));
          }
          nmem += __popc(acc);
          __syncwarp();
        }
      }
    } else if (lane == 0) {
      mem[0] = root;
      nmem = 1;
      vis[root >> 5] |= 1u << (root & 31);
      {
        uint32_t uu = root;
        for (;;) {
          const double d = rng.u01();
          const uint32_t jb = p.off[uu], je = p.off[uu + 1];
          uint32_t pick = je;
          for (uint32_t j = jb; j < je; ++j) {
            if (d < p.cdf[j]) {
              pick = j;
              break;
            }
          }
          sinsp += (pick < je ? pick + 1 : je) - jb;
          if (pick >= je) break;
          const uint32_t v = p.src[pick];
          if ((vis[v >> 5] >> (v & 31)) & 1u) break;
          vis[v >> 5] |= 1u << (v & 31);
          mem[nmem++] = v;
          uu = v;
        }
      }
    }
    nmem = __shfl_sync(kFull, nmem, 0);
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&p.ctl->cursor, (unsigned long long)nmem);
    pos = __shfl_sync(kFull, pos, 0);
    __syncwarp();
    if (pos + nmem > p.stage_cap) {
      if (lane == 0) restage_slot(p, idx, nmem);
    } else {
      for (uint32_t i = lane; i < nmem; i += 32) {
        const uint32_t v = mem[i];
        p.stage[pos + i] = v;
        if (p.counter) atomicAdd(p.counter + v, 1u);
      }
      if (lane == 0) {
        p.slot_start[idx] = pos;
        p.slot_len[idx] = nmem;
        insp += sinsp;
      }
    }
    for (uint32_t i = lane; i < nmem; i += 32) {
      const uint32_t v = mem[i];
      atomicAnd(vis + (v >> 5), ~(1u << (v & 31)));
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(&p.ctl->inspected, (unsigned long long)insp);
    atomicAdd(&p.ctl->entries, (unsigned long long)insp);
  }
}

// ---------------------------------------------------------------------------
// K0: per-model layouts
// ---------------------------------------------------------------------------
__global__ void k_build_rec(const uint32_t* src, const float* w, uint2* rec, uint64_t m) {
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    rec[j] = make_uint2(src[j], bern_thr_hi(__float_as_uint(w[j])));
  }
}

// Warp per vertex: 1 iff the in-list's sources strictly increase (no duplicate
// sources), the precondition of the cooperative IC expansion.
__global__ void k_dupfree(const uint32_t* off, const uint32_t* src, uint32_t n, uint8_t* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  for (uint64_t v = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; v < n;
       v += warps) {
    bool bad = false;
    for (uint32_t j = off[v] + 1 + lane; j < off[v + 1]; j += 32) bad |= src[j] <= src[j - 1];
    bad = __any_sync(kFull, bad);
    if (lane == 0) out[v] = bad ? 0 : 1;
  }
}

// Sequential fp64 prefix per in-list, the exact add order of sampling.hpp:128-131.
// One thread per vertex; `bad` flags a non-monotone prefix (NaN / negative weight).
// Long in-lists stream through registers 32 weights at a time (eight 16-byte
// loads in flight, sixteen 16-byte stores), so a 540K-entry hub costs ~the
// dependent fp64 add chain rather than a memory round trip per entry.
__global__ void k_build_cdf(const uint32_t* off, const float* w, double* cdf, uint32_t n,
                            uint32_t* bad, uint32_t long_min, uint32_t* longv, uint32_t* nlong) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    double acc = 0.0;
    bool neg = false;
    uint32_t j = off[v];
    const uint32_t e = off[v + 1];
    if (e - j >= long_min) {  // hubs: warp per list (k_build_cdf_long)
      longv[atomicAdd(nlong, 1u)] = v;
      continue;
    }
    for (; j < e && (j & 3u); ++j) {  // head up to a 16-byte boundary
      const float x = w[j];
      neg |= !(x >= 0.0f);
      acc = __dadd_rn(acc, static_cast<double>(x));
      cdf[j] = acc;
    }
    for (; j + 32 <= e; j += 32) {
      float4 q[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) q[t] = __ldg(reinterpret_cast<const float4*>(w + j) + t);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float xs[4] = {q[t].x, q[t].y, q[t].z, q[t].w};
        double out[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          neg |= !(xs[u] >= 0.0f);
          acc = __dadd_rn(acc, static_cast<double>(xs[u]));
          out[u] = acc;
        }
        reinterpret_cast<double2*>(cdf + j)[2 * t] = make_double2(out[0], out[1]);
        reinterpret_cast<double2*>(cdf + j)[2 * t + 1] = make_double2(out[2], out[3]);
      }
    }
    for (; j < e; ++j) {
      const float x = w[j];
      neg |= !(x >= 0.0f);
      acc = __dadd_rn(acc, static_cast<double>(x));
      cdf[j] = acc;
    }
    if (neg) *bad = 1;
  }
}

// Hub in-lists: one warp per list. The warp streams the weights into shared
// memory with asynchronous copies (LDGSTS), double-buffered 512 entries ahead,
// while lane 0 runs the dependent fp64 add chain out of shared memory; the warp
// then writes the 512 prefix values back with coalesced stores. The chain
// itself -- the reference's sequential order -- is the only serial part.
constexpr int kCdfChunk = 512;
constexpr int kCdfWarps = 4;
__global__ void __launch_bounds__(kCdfWarps * 32)
    k_build_cdf_long(const uint32_t* off, const float* w, double* cdf, const uint32_t* longv,
                     const uint32_t* nlong, uint32_t* bad) {
  __shared__ float sw[kCdfWarps][2][kCdfChunk];
  __shared__ double sd[kCdfWarps][kCdfChunk];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint32_t nw = gridDim.x * kCdfWarps;
  for (uint32_t i = blockIdx.x * kCdfWarps + wl; i < *nlong; i += nw) {
    const uint32_t v = longv[i];
    const uint32_t b = off[v], e = off[v + 1];
    auto fetch = [&](uint32_t c0, int buf) {
      const uint32_t len = min(static_cast<uint32_t>(kCdfChunk), e - c0);
      for (uint32_t t = lane; t < len; t += 32)
        __pipeline_memcpy_async(&sw[wl][buf][t], w + c0 + t, sizeof(float));
      __pipeline_commit();
    };
    double acc = 0.0;
    bool neg = false;
    fetch(b, 0);
    int cur = 0;
    for (uint32_t c0 = b; c0 < e; c0 += kCdfChunk, cur ^= 1) {
      const uint32_t len = min(static_cast<uint32_t>(kCdfChunk), e - c0);
      if (c0 + kCdfChunk < e) {
        fetch(c0 + kCdfChunk, cur ^ 1);
        __pipeline_wait_prior(1);  // this chunk landed; the next stays in flight
      } else {
        __pipeline_wait_prior(0);
      }
      __syncwarp();
      if (lane == 0) {
        const float* x = sw[wl][cur];
        double* y = sd[wl];
        uint32_t t = 0;
        for (; t + 8 <= len; t += 8) {
          float xs[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) xs[u] = x[t + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            neg |= !(xs[u] >= 0.0f);
            acc = __dadd_rn(acc, static_cast<double>(xs[u]));
            y[t + u] = acc;
          }
        }
        for (; t < len; ++t) {
          neg |= !(x[t] >= 0.0f);
          acc = __dadd_rn(acc, static_cast<double>(x[t]));
          y[t] = acc;
        }
      }
      __syncwarp();
      for (uint32_t t = lane; t < len; t += 32) cdf[c0 + t] = sd[wl][t];
      __syncwarp();
    }
    if (lane == 0 && neg) *bad = 1;
  }
}

// Upload checks done on the device: offsets u64 -> u32 with monotonicity and
// range checks, sources < n. bad[0] |= 1 offsets, 2 sources.
__global__ void k_offsets_u32(const uint64_t* off64, uint32_t* off32, uint32_t n, uint64_t m,
                              uint32_t* bad) {
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v <= n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = off64[v];
    off32[v] = static_cast<uint32_t>(x);
    const bool ok = x <= m && (v == 0 ? x == 0 : off64[v - 1] <= x) && (v < n || x == m);
    if (!ok) atomicOr(bad, 1u);
  }
}

// LT vertex record (64 B): in-list start and degree, then for degree <= 6 the
// whole CDF (floats rounded down) and the sources, else the first slot of the
// vertex's search-tree nodes and the root's 13 pivots. One load per walk step
// replaces the offsets load and the first search level.
__device__ __forceinline__ uint32_t lt_fdown(double x) { return __float_as_uint(__double2float_rd(x)); }
constexpr uint32_t kLtSentinel = 0x40000000u;  // 2.0f: never <= a draw in [0, 1)

__global__ void k_build_ltrec(const uint32_t* off, const double* cdf, const uint32_t* src,
                              const uint64_t* nodeoff, uint32_t n, uint32_t* rec) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const uint32_t b = off[u], deg = off[u + 1] - b;
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = 0;
  w[0] = b;
  w[1] = deg;
  if (deg <= kLtRecSmall) {
    for (uint32_t t = 0; t < kLtRecSmall; ++t) {
      w[2 + t] = t < deg ? lt_fdown(cdf[b + t]) : kLtSentinel;
      w[8 + t] = t < deg ? src[b + t] : 0u;
    }
  } else {
    w[2] = static_cast<uint32_t>(nodeoff[u]);
    const uint32_t step = lt_step(0, deg, kLtRootPivots);
    for (uint32_t t = 1; t <= kLtRootPivots; ++t) {
      const uint32_t i = t * step;
      w[2 + t] = i < deg ? lt_fdown(cdf[b + i]) : kLtSentinel;
    }
  }
  uint4* out = reinterpret_cast<uint4*>(rec + static_cast<size_t>(u) * 16);
#pragma unroll
  for (int i = 0; i < 4; ++i) out[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}

// Node slots of a vertex's search tree: level 1 has 14, each deeper level 32x
// the one above, while the child ranges of the level above (<= its step) still
// exceed kLtLeafMin; a level whose ranges fit kLtLeafMax is the last (leaves).
__global__ void k_count_ltnodes(const uint32_t* off, uint32_t n, uint32_t* cnt) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint32_t len = off[u + 1] - off[u];
  uint64_t slots = 0, width = kLtRootFanout;
  uint32_t P = kLtRootPivots;
  if (len > kLtRecSmall) {
    for (;;) {
      const uint32_t cl = lt_step(0, len, P);  // longest child range
      if (cl <= kLtLeafMin) break;
      slots += width;
      if (cl <= kLtLeafMax) break;
      width *= kLtFanout;
      len = cl;
      P = kLtNodePivots;
    }
  }
  cnt[u] = static_cast<uint32_t>(slots);
}

// One block per vertex: slot s (node x = s + 1) follows its path from the root
// and stores its 31 pivots (unreachable slots: sentinels).
__global__ void k_build_ltnodes(const uint32_t* off, const double* cdf, const uint32_t* src,
                                const uint64_t* nodeoff, uint32_t n, uint32_t* nodes) {
  for (uint32_t u = blockIdx.x; u < n; u += gridDim.x) {
    const uint64_t base = nodeoff[u];
    const uint32_t cnt = static_cast<uint32_t>(nodeoff[u + 1] - base);
    if (!cnt) continue;
    const uint32_t b = off[u], e = off[u + 1];
    for (uint32_t s = threadIdx.x; s < cnt; s += blockDim.x) {
      // level and index of slot s (level 1: 14 slots, then x32 per level)
      uint64_t r = s, width = kLtRootFanout;
      int level = 1;
      while (r >= width) {
        r -= width;
        width *= kLtFanout;
        ++level;
      }
      uint32_t dig[8];  // child digits, root's first
      for (int k = level - 1; k >= 1; --k) {
        dig[k] = static_cast<uint32_t>(r % kLtFanout);
        r /= kLtFanout;
      }
      dig[0] = static_cast<uint32_t>(r);
      uint32_t lo = b, hi = e;
      bool ok = true;
      for (int k = 0; k < level && ok; ++k) {  // parents must be inner nodes (or the root)
        const uint32_t P = k == 0 ? kLtRootPivots : kLtNodePivots;
        if (dig[k] > P || (k > 0 && hi - lo <= kLtLeafMax)) {
          ok = false;
          break;
        }
        lt_child(lo, hi, P, dig[k]);
        if (lo > hi) ok = false;
      }
      ok = ok && hi - lo > kLtLeafMin;
      uint32_t* out = nodes + (base + s) * 32;
      if (ok && hi - lo <= kLtLeafMax) {  // leaf: cdf[lo, hi) and src[lo, hi]
        for (uint32_t t = 0; t < kLtLeafMax; ++t)
          out[t] = lo + t < hi ? lt_fdown(cdf[lo + t]) : kLtSentinel;
        for (uint32_t t = 0; t <= kLtLeafMax; ++t)
          out[kLtLeafMax + t] = lo + t <= hi && lo + t < e ? src[lo + t] : 0u;
        out[31] = 0u;
      } else {
        const uint32_t st = ok ? lt_step(lo, hi, kLtNodePivots) : 1u;
        for (uint32_t t = 1; t <= kLtNodePivots; ++t) {
          const uint32_t i = lo + t * st;
          out[t - 1] = ok && i < hi ? lt_fdown(cdf[i]) : kLtSentinel;
        }
        out[31] = kLtSentinel;
      }
    }
  }
}

// Guide table (common.cuh "LT guide table"): thread per chunk of kGuideChunk
// consecutive buckets of the flat bucket space [0, mult m) (vertex u owns
// [mult off[u], mult off[u+1])). The chunk finds its first vertex and A_g by
// binary search, then merges buckets against the CDF: A_{g+1} = #{cdf <= the
// smallest draw of bucket g+1}, that draw kept exactly as Q + (R > 0) with
// g 2^53 = Q G + R updated incrementally.
constexpr uint32_t kGuideChunk = 64;

__device__ __forceinline__ void guide_cand(const uint32_t* off, const uint32_t* src, uint32_t b,
                                           uint32_t deg, uint32_t j, uint32_t& v, uint32_t& ov,
                                           uint32_t& dv) {
  if (j < deg) {
    v = __ldg(src + b + j);
    ov = __ldg(off + v);
    dv = __ldg(off + v + 1) - ov;
  } else {
    v = kGuideNone;
    ov = 0;
    dv = 0;
  }
}

__global__ void k_build_ltguide(const uint32_t* off, const double* cdf, const uint32_t* src,
                                uint32_t n, uint64_t m, uint32_t mult, uint4* guide) {
  const uint64_t total = static_cast<uint64_t>(mult) * m;
  const uint64_t nchunks = (total + kGuideChunk - 1) / kGuideChunk;
  const uint64_t two53 = 1ull << 53;
  for (uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < nchunks;
       c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t i = c * kGuideChunk;
    const uint64_t iend = min(i + kGuideChunk, total);
    // the vertex owning bucket i: the largest u with off[u] <= i / mult
    const uint32_t q = static_cast<uint32_t>(i / mult);
    uint32_t lo = 0, hi = n - 1;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo + 1) / 2;
      if (__ldg(off + mid) <= q) lo = mid;
      else hi = mid - 1;
    }
    uint32_t u = lo;
    uint32_t b = __ldg(off + u), deg = __ldg(off + u + 1) - b;
    uint64_t G = static_cast<uint64_t>(mult) * deg;
    uint64_t g = i - static_cast<uint64_t>(mult) * b;
    uint64_t q0 = two53 / G, r0 = two53 % G;
    const unsigned __int128 N = static_cast<unsigned __int128>(g) << 53;
    uint64_t Q = static_cast<uint64_t>(N / G), R = static_cast<uint64_t>(N % G);
    // A_g = #{cdf <= dmin_g}: binary search on the sorted in-list
    const double d0 = static_cast<double>(Q + (R ? 1 : 0)) * 0x1.0p-53;
    uint32_t A = 0, ahi = deg;
    while (A < ahi) {
      const uint32_t mid = A + (ahi - A) / 2;
      if (__ldg(cdf + b + mid) <= d0) A = mid + 1;
      else ahi = mid;
    }
    uint32_t cu = 0xffffffffu, cA = 0xffffffffu;  // the vertex and index c0 describes
    bool cA1ok = false;                            // c1 describes index cA + 1
    uint3 c0 = make_uint3(0, 0, 0), c1 = make_uint3(0, 0, 0);
    for (; i < iend; ++i, ++g) {
      if (g == G) {  // next vertex with in-edges; its bucket 0 has the draw 0
        do {
          ++u;
          b = __ldg(off + u);
          deg = __ldg(off + u + 1) - b;
        } while (deg == 0);
        G = static_cast<uint64_t>(mult) * deg;
        g = 0;
        q0 = two53 / G;
        r0 = two53 % G;
        Q = 0;
        R = 0;
        A = 0;
        while (A < deg && __ldg(cdf + b + A) <= 0.0) ++A;
      }
      uint64_t Q1 = Q + q0, R1 = R + r0;
      if (R1 >= G) {
        R1 -= G;
        ++Q1;
      }
      const double d1 = static_cast<double>(Q1 + (R1 ? 1 : 0)) * 0x1.0p-53;  // 1.0 for g+1 = G
      uint32_t A1 = A;
      while (A1 < deg && __ldg(cdf + b + A1) <= d1) ++A1;
      const uint32_t span = A1 - A;
      uint4 e0, e1;
      e0.x = A;
      e0.y = (A < deg ? lt_fdown(__ldg(cdf + b + A)) : 0u) |
             (span == 0 ? kGuideSpan0 : span >= 2 ? kGuideSearch : 0u);
      // candidate infos, reused while consecutive buckets share A (about mult
      // buckets per CDF entry): the source's offsets are random L2 reads
      if (u != cu || A != cA) {
        if (u == cu && A == cA + 1 && cA1ok) {
          c0 = c1;
        } else {
          guide_cand(off, src, b, deg, A, c0.x, c0.y, c0.z);
        }
        cu = u;
        cA = A;
        cA1ok = false;
      }
      e0.z = c0.x;
      e0.w = c0.y;
      e1.x = c0.z;
      if (span == 1) {
        if (!cA1ok) {
          guide_cand(off, src, b, deg, A + 1, c1.x, c1.y, c1.z);
          cA1ok = true;
        }
        e1.y = c1.x;
        e1.z = c1.y;
        e1.w = c1.z;
      } else {
        e1.y = span >= 2 ? span : kGuideNone;
        e1.z = 0;
        e1.w = 0;
      }
      asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(guide + 2 * i),
                   "r"(e0.x), "r"(e0.y), "r"(e0.z), "r"(e0.w), "r"(e1.x), "r"(e1.y), "r"(e1.z),
                   "r"(e1.w)
                   : "memory");  // one 32-byte sector (STG.256)
      A = A1;
      Q = Q1;
      R = R1;
    }
  }
}

__global__ void k_max_degree(const uint32_t* off, uint32_t n, uint32_t* out) {
  uint32_t best = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    best = max(best, off[v + 1] - off[v]);
  for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(kFull, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void k_check_sources(const uint32_t* src, uint64_t m, uint32_t n, uint32_t* bad) {
  bool ok = true;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    ok &= src[j] < n;
  if (!__all_sync(kFull, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 2u);
}

}  // namespace

uint32_t upload_checks(rrg_graph* g, const uint64_t* d_off64) {
  DevBuf<uint32_t> bad;
  bad.reserve_discard(1);
  RRG_CUDA(cudaMemsetAsync(bad.ptr, 0, 4, g->stream));
  const int grid = g->num_sms * 8;
  k_offsets_u32<<<grid, 256, 0, g->stream>>>(d_off64, g->off.ptr, g->n, g->m, bad.ptr);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  if (g->m) {
    k_check_sources<<<grid, 256, 0, g->stream>>>(g->src.ptr, g->m, g->n, bad.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  }
  uint32_t h = 0;
  RRG_CUDA(cudaMemcpyAsync(&h, bad.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
  RRG_CUDA(cudaStreamSynchronize(g->stream));
  return h;
}

// Guide-mode walk variant. Default: 2048-bit filters, walks use the hash table
// from 384 members, 64 KB of shared memory per block, three blocks per SM (80
// registers, no spills): cfg4 2^20 walks 4.2 ms. RRGPU_LT_FILTER=0 selects the
// first design (1024 bits, table from 128 members, 32 KB, four blocks at 64
// registers with spills: 6.1 ms) for A/B runs.
using LtGuideFn = void (*)(SampleParams);
int lt_filter_variant() {
  static const int v = [] {
    const char* e = std::getenv("RRGPU_LT_FILTER");
    return e && *e == '0' ? 0 : 1;
  }();
  return v;
}
LtGuideFn lt_guide_kernel() {
  static bool attr = false;
  if (!attr) {
    RRG_CUDA(cudaFuncSetAttribute(k_sample_lt_guide<6, 384, 3>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr = true;
  }
  return lt_filter_variant() ? k_sample_lt_guide<6, 384, 3> : k_sample_lt_guide<5, 128, 4>;
}
size_t lt_guide_smem() { return (lt_filter_variant() ? 64u : 32u) * kBlock * 4u; }

int sampler_block() { return kBlock; }

int sampler_blocks_per_sm(int model, uint32_t, int lt_mode) {
  int b = 0;
  if (model == RRG_IC)
    RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample_ic, kBlock, 0));
  else if (lt_mode == kLtGuide)
    RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, lt_guide_kernel(), kBlock,
                                                           lt_guide_smem()));
  else
    RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample_lt<16>, kBlock, 0));
  return b < 1 ? 1 : b;
}

void launch_sampler(int model, const SampleParams& p, int grid, uint32_t ic_inner, int schedule,
                    cudaStream_t s) {
  if (model == RRG_IC) {
    if (schedule != kSchedLane) {
      static bool attr_set = false;  // > 48 KB of dynamic shared memory needs opting in
      if (!attr_set) {
        RRG_CUDA(cudaFuncSetAttribute(k_sample_ic_warp<32>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kWarpKernelDynSmem)));
        RRG_CUDA(cudaFuncSetAttribute(k_sample_ic_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(kCtaKernelDynSmem)));
        attr_set = true;
      }
      if (schedule == kSchedWarp) k_sample_ic_warp<32><<<grid, kBlock, kWarpKernelDynSmem, s>>>(p);
      else k_sample_ic_cta<<<grid, kBlock, kCtaKernelDynSmem, s>>>(p);
    } else {
      k_sample_ic<<<grid, kBlock, 0, s>>>(p, ic_inner);
    }
  } else if (p.lt_scan == kLtGuide) {
    lt_guide_kernel()<<<grid, kBlock, lt_guide_smem(), s>>>(p);
  } else {
    switch (p.lt_kary) {
      case 2: k_sample_lt<2><<<grid, kBlock, 0, s>>>(p); break;
      case 4: k_sample_lt<4><<<grid, kBlock, 0, s>>>(p); break;
      case 8: k_sample_lt<8><<<grid, kBlock, 0, s>>>(p); break;
      default: k_sample_lt<16><<<grid, kBlock, 0, s>>>(p); break;
    }
  }
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_big(int model, const SampleParams& p, const uint32_t* list, uint32_t nlist,
                uint32_t* bitmaps, uint32_t* lists, uint32_t workers, cudaStream_t s) {
  const int grid = static_cast<int>((workers * 32 + kBlock - 1) / kBlock);
  k_sample_big<<<grid, kBlock, 0, s>>>(p, model, list, nlist, bitmaps, lists, workers);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_fast_lane(const SampleParams& p, int grid, cudaStream_t s) {
  k_sample_ic_fast_lane<<<grid, kBlock, 0, s>>>(p);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_fast(const SampleParams& p, int grid, bool bitmap, uint32_t* bitmaps, uint32_t* lists,
                 uint32_t workers, cudaStream_t s) {
  if (bitmap) {
    k_sample_ic_fast<true><<<(workers * 32 + kBlock - 1) / kBlock, kBlock, 0, s>>>(p, bitmaps, lists,
                                                                                  workers);
  } else {
    k_sample_ic_fast<false><<<grid, kBlock, 0, s>>>(p, nullptr, nullptr, 0);
  }
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void prepare_ic_fast(rrg_graph* g) {
  if (g->uniform_ready) return;
  g->uniformw.reserve_discard(g->n ? g->n : 1);
  if (g->n) {
    k_uniform_weights<<<g->num_sms * 16, 256, 0, g->stream>>>(g->off.ptr, g->w.ptr, g->n,
                                                            g->uniformw.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    RRG_CUDA(cudaStreamSynchronize(g->stream));
  }
  g->uniform_ready = true;
}

void prepare_ic(rrg_graph* g) {
  if (g->rec_ready) return;
  g->rec.reserve_discard(g->m ? g->m : 1);
  if (g->m) {
    k_build_rec<<<g->num_sms * 8, 256, 0, g->stream>>>(g->src.ptr, g->w.ptr, g->rec.ptr, g->m);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  }
  g->dupfree.reserve_discard(g->n ? g->n : 1);
  if (g->n) {
    k_dupfree<<<g->num_sms * 16, 256, 0, g->stream>>>(g->off.ptr, g->src.ptr, g->n,
                                                      g->dupfree.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  }
  static const std::vector<uint64_t> jt = segment_tables(32, 31);  // host, built once
  static const std::vector<uint64_t> jt16 = segment_tables(16, 31);
  static const std::vector<uint64_t> jt256 = segment_tables(256, 15);
  static const std::vector<uint64_t> jt64 = segment_tables(kLxPer, 31);  // list-expansion lanes
  g->jtab64.reserve_discard(jt64.size());
  RRG_CUDA(cudaMemcpyAsync(g->jtab64.ptr, jt64.data(), jt64.size() * 8, cudaMemcpyHostToDevice,
                           g->stream));
  static const std::vector<uint64_t> jthi = [] {  // T^(4096 a), T^(65536 a), T^(2^20 a)
    std::vector<uint64_t> v;
    for (uint64_t seg : {4096ull, 65536ull, 1048576ull}) {
      const std::vector<uint64_t> t = segment_tables(seg, 15);
      v.insert(v.end(), t.begin(), t.end());
    }
    return v;
  }();
  g->jtabhi.reserve_discard(jthi.size());
  RRG_CUDA(cudaMemcpyAsync(g->jtabhi.ptr, jthi.data(), jthi.size() * 8, cudaMemcpyHostToDevice,
                           g->stream));
  {  // largest in-list: sizes the list-expansion scratch
    DevBuf<uint32_t> mx;
    mx.reserve_discard(1);
    RRG_CUDA(cudaMemsetAsync(mx.ptr, 0, 4, g->stream));
    if (g->n) {
      k_max_degree<<<g->num_sms * 8, 256, 0, g->stream>>>(g->off.ptr, g->n, mx.ptr);
      RRG_CUDA(cudaGetLastError());
      count_launch();
    }
    RRG_CUDA(cudaMemcpyAsync(&g->max_indeg, mx.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
    RRG_CUDA(cudaStreamSynchronize(g->stream));
  }
  g->jtab.reserve_discard(jt.size());
  g->jtab16.reserve_discard(jt16.size());
  g->jtab256.reserve_discard(jt256.size());
  RRG_CUDA(cudaMemcpyAsync(g->jtab256.ptr, jt256.data(), jt256.size() * 8, cudaMemcpyHostToDevice,
                           g->stream));
  RRG_CUDA(cudaMemcpyAsync(g->jtab.ptr, jt.data(), jt.size() * 8, cudaMemcpyHostToDevice,
                           g->stream));
  RRG_CUDA(cudaMemcpyAsync(g->jtab16.ptr, jt16.data(), jt16.size() * 8, cudaMemcpyHostToDevice,
                           g->stream));
  RRG_CUDA(cudaStreamSynchronize(g->stream));
  g->rec_ready = true;
}

void prepare_lt(rrg_graph* g) {
  if (g->cdf_ready) return;
  g->cdf.reserve_discard(g->m + 2);  // +2: the paired 16-byte loads may touch cdf[m]
  RRG_CUDA(cudaMemsetAsync(g->cdf.ptr + g->m, 0, 2 * sizeof(double), g->stream));
  DevBuf<uint32_t> bad;  // [0] bad flag, [1] number of hub lists
  bad.reserve_discard(2);
  RRG_CUDA(cudaMemsetAsync(bad.ptr, 0, 8, g->stream));
  if (g->m) {
    DevBuf<uint32_t> longv;
    longv.reserve_discard(g->n);
    const uint32_t long_min = 4096;
    const int blocks = (g->n + 127) / 128;
    k_build_cdf<<<blocks, 128, 0, g->stream>>>(g->off.ptr, g->w.ptr, g->cdf.ptr, g->n, bad.ptr,
                                              long_min, longv.ptr, bad.ptr + 1);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    k_build_cdf_long<<<g->num_sms * 4, kCdfWarps * 32, 0, g->stream>>>(
        g->off.ptr, g->w.ptr, g->cdf.ptr, longv.ptr, bad.ptr + 1, bad.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    RRG_CUDA(cudaStreamSynchronize(g->stream));  // longv is released at scope end
  }
  uint32_t hbad = 0;
  RRG_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
  RRG_CUDA(cudaStreamSynchronize(g->stream));
  g->cdf_monotone = hbad == 0;
  g->cdf_ready = true;
}

// LT search mode: vertex records + search trees (monotone CDF only).
void prepare_lt_search(rrg_graph* g) {
  if (g->lt_search_ready) return;
  g->lt_search_ready = true;
  if (!g->cdf_monotone || !g->n) return;
  DevBuf<uint32_t> cnt;
  cnt.reserve_discard(g->n);
  k_count_ltnodes<<<(g->n + 255) / 256, 256, 0, g->stream>>>(g->off.ptr, g->n, cnt.ptr);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  g->ltnodeoff.reserve_discard(static_cast<size_t>(g->n) + 1);
  DevBuf<uint64_t> tmp;
  exclusive_scan_u32(cnt.ptr, g->ltnodeoff.ptr, g->n, tmp, g->stream);
  uint64_t slots = 0;
  RRG_CUDA(cudaMemcpyAsync(&slots, g->ltnodeoff.ptr + g->n, 8, cudaMemcpyDeviceToHost,
                           g->stream));
  RRG_CUDA(cudaStreamSynchronize(g->stream));
  if (slots >= (1ull << 32)) {  // node slots are u32 in the records: use the plain search
    g->ltrec.release();
    g->ltnodes.release();
    return;
  }
  g->ltnodes.reserve_discard(slots ? slots * 32 : 32);
  if (slots) {
    k_build_ltnodes<<<std::min<uint32_t>(g->n, 65535u * 4), 128, 0, g->stream>>>(
        g->off.ptr, g->cdf.ptr, g->src.ptr, g->ltnodeoff.ptr, g->n, g->ltnodes.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  }
  g->ltrec.reserve_discard(static_cast<size_t>(g->n) * 16);
  k_build_ltrec<<<(g->n + 255) / 256, 256, 0, g->stream>>>(
      g->off.ptr, g->cdf.ptr, g->src.ptr, g->ltnodeoff.ptr, g->n, g->ltrec.ptr);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  RRG_CUDA(cudaStreamSynchronize(g->stream));
}

// LT guide mode: 32 bytes per bucket, mult buckets per in-edge. False (and no
// table) when the CDF is not monotone or the table would not fit in free HBM.
bool prepare_lt_guide(rrg_graph* g) {
  if (!g->cdf_monotone || !g->m) return false;
  if (g->lt_guide_built == g->lt_guide_mult && g->ltguide.ptr) return true;
  g->ltguide.release();
  g->lt_guide_built = 0;
  const uint64_t entries = static_cast<uint64_t>(g->lt_guide_mult) * g->m;
  size_t freeb = 0, totalb = 0;
  RRG_CUDA(cudaMemGetInfo(&freeb, &totalb));
  if (entries * 32 + (2ull << 30) > freeb) return false;
  g->ltguide.reserve_discard(2 * entries);
  const uint64_t chunks = (entries + kGuideChunk - 1) / kGuideChunk;
  const uint64_t grid = std::min<uint64_t>((chunks + 127) / 128, 1u << 20);
  k_build_ltguide<<<static_cast<unsigned>(grid), 128, 0, g->stream>>>(
      g->off.ptr, g->cdf.ptr, g->src.ptr, g->n, g->m, g->lt_guide_mult, g->ltguide.ptr);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  RRG_CUDA(cudaStreamSynchronize(g->stream));
  g->lt_guide_built = g->lt_guide_mult;
  return true;
}

// The structures the graph's LT scan mode needs; returns the mode launches use.
int prepare_lt_mode(rrg_graph* g) {
  prepare_lt(g);
  if (g->lt_scan == kLtGuide && prepare_lt_guide(g)) return kLtGuide;
  if (g->lt_scan == kLtLinear || !g->cdf_monotone) return kLtLinear;
  prepare_lt_search(g);
  return kLtBsearch;
}

}  // namespace rrgpu
