// sample_lt.cu -- K2: the LT samplers (sampling.hpp:117-145 per slot) -- the
// guide-table walk (default), the search-tree walk and the reference's linear
// CDF scan -- and the LT K0 layouts (fp64 CDF, vertex records and search trees,
// guide table). See sample.cu for the execution model shared by all samplers.
#include "sampler.cuh"

namespace rrgpu {

namespace {

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
      RRG_DCHECK(nmem < kMemCap && v < p.n, 5);
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
// kLite: the entry is {A_g, pivot | flags (span in the pivot bits when kGuideSearch)}
// only (ltlite, 8 bytes: built from the CDF alone, before the sources are on
// the device); the chosen source and its offsets are three dependent loads.
template <bool kLite>
__device__ __forceinline__ void lt_guide_resolve(const SampleParams& p, const uint4 e0,
                                                 const uint4 e1, uint64_t x, uint32_t offu,
                                                 uint32_t degu, uint32_t& pick, uint32_t& v,
                                                 uint32_t& offv, uint32_t& degv, uint64_t& ent) {
  const uint32_t A = e0.x;
  const uint32_t pw = e0.y;
  if (pw & kGuideSpan0) {  // no CDF entry inside the bucket: index A_g whatever the draw
    pick = A;
    if (!kLite) {
      v = e0.z;
      offv = e0.w;
      degv = e1.x;
      return;
    }
  } else {
    const double d = __ull2double_rn(x >> 11) * 0x1.0p-53;  // uniform01(), exact
    const uint32_t dbits = __float_as_uint(__double2float_rd(d));
    if (!(pw & kGuideSearch)) {  // one entry: pick A_g + [cdf[A_g] <= d]
      const uint32_t f = pw & kGuidePivot;
      const bool le = f < dbits || (f == dbits && __ldg(p.cdf + offu + A) <= d);
      pick = le ? A + 1 : A;
      if (!kLite) {
        if (le) {
          v = e1.y;
          offv = e1.z;
          degv = e1.w;
        } else {
          v = e0.z;
          offv = e0.w;
          degv = e1.x;
        }
        return;
      }
    } else {
      // span >= 2 (rare): count cdf[A_g, A_g + span) <= d, eight loads in flight
      const uint32_t span = kLite ? (pw & kGuidePivot) : e1.y;
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
    }
  }
  if (pick < degu) {
    v = __ldg(p.src + offu + pick);
    offv = __ldg(p.off + v);
    degv = __ldg(p.off + v + 1) - offv;
  } else {
    v = kGuideNone;
  }
}

#ifndef RRG_GUIDE_EVICT_FIRST
#define RRG_GUIDE_EVICT_FIRST 1
#endif
// L2 policy of the bucket-entry loads: evict first. The 8.8 GB table has no
// reuse worth keeping (a walk's buckets are uniformly likely), so its lines
// should not push the walks' member lists, hash tables and the fused counter
// out of L2 -- the kernel runs at the random-access DRAM ceiling, so every
// DRAM byte it does not move is time (profiles/r2/NOTES.md).
__device__ __forceinline__ uint64_t lt_guide_policy() {
  uint64_t pol = 0;
#if RRG_GUIDE_EVICT_FIRST
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}

template <bool kLite>
__device__ __forceinline__ void lt_guide_fetch(const SampleParams& p, uint32_t offu, uint32_t degu,
                                               uint64_t x, uint4& e0, uint4& e1, uint64_t pol) {
  if (!degu) return;
  const uint64_t G = static_cast<uint64_t>(degu) * p.lt_guide_mult;
  const uint64_t gi = static_cast<uint64_t>(offu) * p.lt_guide_mult + __umul64hi(x & ~0x7ffull, G);
  if (kLite) {
    const uint2 q = __ldg(p.ltlite + gi);
    e0.x = q.x;
    e0.y = q.y;
    (void)e1;
    (void)pol;
    return;
  }
  // one 256-bit load (sm_100: LDG.256), not allocated in L1: the entry is one
  // 32-byte sector and is never re-read by this SM
#if RRG_GUIDE_EVICT_FIRST
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(e0.x), "=r"(e0.y), "=r"(e0.z), "=r"(e0.w), "=r"(e1.x), "=r"(e1.y),
                 "=r"(e1.z), "=r"(e1.w)
               : "l"(p.ltguide + 2 * gi), "l"(pol));
#else
  (void)pol;
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(e0.x), "=r"(e0.y), "=r"(e0.z), "=r"(e0.w), "=r"(e1.x), "=r"(e1.y),
                 "=r"(e1.z), "=r"(e1.w)
               : "l"(p.ltguide + 2 * gi));
#endif
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
          RRG_DCHECK(v[k] < p.n && pos + i < p.stage_cap, 3);
          out[i] = v[k];
          if (p.counter) atomicAdd(p.counter + v[k], 1u);
        }
      }
    }
    if (lane == L) {
      p.slot_start[iL] = pos;
      p.slot_len[iL] = nL;
      note_len(p, nL);
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
template <int kFiltLog, uint32_t kLtFiltMax, int kMinBlocks, bool kLite = false>
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
  const uint64_t gpol = lt_guide_policy();

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
          RRG_DCHECK(nmem < kMemCap && vL < p.n, 4);
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
      lt_guide_fetch<kLite>(p, offu, degu, x, e0, e1, gpol);
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
      lt_guide_resolve<kLite>(p, e0, e1, x, offu, degu, pick, v, offv, degv, ent);
      ent += kLite ? 3 : 4;  // the 32-byte bucket entry (in 8-byte units); lite: 8 + 3 x 4 bytes
    }
    sinsp += pick < degu ? pick + 1 : degu;  // reference trip count (sampling.hpp:130-136)
    bool stop = v == kGuideNone;
    if (!stop) {
      lt_guide_fetch<kLite>(p, offv, degv, xn, e0, e1, gpol);  // next step's entry, in flight now
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
      RRG_DCHECK(nmem < kMemCap && v < p.n, 5);
      mem[nmem++] = v;
      rebuild = !big && nmem == kLtFiltMax;
      offu = offv;
      degu = degv;
    }
  }
  p.tags[gid] = tag;
  flush_counters(p, insp, ent);
}

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

// Hub in-lists: one warp per list. The reference's running sum acc += (double)w[j]
// (sampling.hpp:130-136) is a serial fp64 chain -- ~20 cycles per entry on one
// lane, 5.5 ms for cfg4's 542,861-entry hub -- but almost every one of its adds
// is EXACT (the weights are floats, the sum is < 2: an add rounds only when a
// weight has bits below the sum's last place, ~0.005 % of cfg4's hub entries).
// Exact adds are associative, so the warp scans 256 entries at a time in
// parallel -- eight per lane, a warp scan of the lane totals, the carry added
// last -- with every add checked by TwoSum: when all error terms are zero each
// value is the exact sum of its operands, hence representable, hence what the
// serial chain produces (by induction from the carry, which IS the chain's
// value). A chunk with any nonzero error term is redone by lane 0 as the plain
// serial chain. The weights stream into shared memory with asynchronous copies
// (LDGSTS), double-buffered one stage ahead.
constexpr int kCdfChunk = 512;  // staged entries (two scanned chunks of 256)
constexpr int kCdfWarps = 4;
// s = fl(a + b); err |= (a + b != s), Knuth's TwoSum (no ordering assumption)
__device__ __forceinline__ double cdf_add_checked(double a, double b, bool& err) {
  const double s = __dadd_rn(a, b);
  const double bb = __dadd_rn(s, -a);
  const double e = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
  err |= e != 0.0;
  return s;
}
__global__ void __launch_bounds__(kCdfWarps * 32)
    k_build_cdf_long(const uint32_t* off, const float* w, double* cdf, const uint32_t* longv,
                     const uint32_t* nlong, uint32_t* bad) {
  __shared__ __align__(16) float sw[kCdfWarps][2][kCdfChunk];
  __shared__ double sd[kCdfWarps][256];
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
    double acc = 0.0;  // the chain's value before the current chunk (warp-uniform)
    bool neg = false;
    fetch(b, 0);
    int cur = 0;
    for (uint32_t c0 = b; c0 < e; c0 += kCdfChunk, cur ^= 1) {
      const uint32_t len = min(static_cast<uint32_t>(kCdfChunk), e - c0);
      if (c0 + kCdfChunk < e) {
        fetch(c0 + kCdfChunk, cur ^ 1);
        __pipeline_wait_prior(1);  // this stage landed; the next stays in flight
      } else {
        __pipeline_wait_prior(0);
      }
      __syncwarp();
      for (uint32_t h0 = 0; h0 < len; h0 += 256) {
        const float* x = sw[wl][cur] + h0;
        const uint32_t hl = min(256u, len - h0);
        // lane l: entries [8 l, 8 l + 8) of the chunk (zeros past its end: exact)
        double loc[8];
        bool err = false;
        {
          const float4 q0 = *reinterpret_cast<const float4*>(x + 8 * lane);
          const float4 q1 = *reinterpret_cast<const float4*>(x + 8 * lane + 4);
          const float xs[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
          double run = 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool in = 8u * lane + u < hl;
            const float xv = in ? xs[u] : 0.0f;
            neg |= !(xv >= 0.0f);
            run = u == 0 ? static_cast<double>(xv)
                         : cdf_add_checked(run, static_cast<double>(xv), err);
            loc[u] = run;
          }
        }
        double incl = loc[7];  // inclusive scan of the lane totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl = cdf_add_checked(y, incl, err);
        }
        double base = __shfl_up_sync(kFull, incl, 1);  // exclusive prefix of the lane
        base = lane == 0 ? acc : cdf_add_checked(acc, base, err);
        double out[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) out[u] = cdf_add_checked(base, loc[u], err);
        if (!__any_sync(kFull, err)) {
          double* y = cdf + c0 + h0 + 8 * lane;
          if (8u * lane + 8 <= hl && ((c0 + h0) & 1u) == 0) {
#pragma unroll
            for (int u = 0; u < 8; u += 2)
              *reinterpret_cast<double2*>(y + u) = make_double2(out[u], out[u + 1]);
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (8u * lane + u < hl) y[u] = out[u];
          }
          // the chain after the chunk: its last entry's value
          const uint32_t last = hl - 1;
          double tail = out[0];
#pragma unroll
          for (int u = 1; u < 8; ++u) tail = (last & 7u) == static_cast<uint32_t>(u) ? out[u] : tail;
          acc = __shfl_sync(kFull, tail, last >> 3);
        } else {  // some add rounded: the serial chain, as the reference runs it
          if (lane == 0) {
            double a2 = acc;
            for (uint32_t t = 0; t < hl; ++t) {
              a2 = __dadd_rn(a2, static_cast<double>(x[t]));
              sd[wl][t] = a2;
            }
          }
          __syncwarp();
          for (uint32_t t = lane; t < hl; t += 32) cdf[c0 + h0 + t] = sd[wl][t];
          acc = sd[wl][hl - 1];
          __syncwarp();
        }
      }
      __syncwarp();  // the stage is free for the copy after next
    }
    if (__any_sync(kFull, neg) && lane == 0) *bad = 1;
  }
}

// Upload checks done on the device: offsets u64 -> u32 with monotonicity and
// range checks, sources < n. bad[0] |= 1 offsets, 2 sources.
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

// kLite: 8-byte entries {A_g, pivot | flags; the span in the pivot bits when
// kGuideSearch} into `lite` -- no candidate infos, so neither the sources nor
// their offsets are read: the table can be built while the sources upload.
template <bool kLite>
__global__ void k_build_ltguide(const uint32_t* off, const double* cdf, const uint32_t* src,
                                uint32_t n, uint64_t m, uint32_t mult, uint4* guide, uint2* lite) {
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
      if (kLite) {
        if (span >= 2) e0.y = kGuideSearch | span;  // span <= deg < 2^30 (checked by the host)
        lite[i] = make_uint2(e0.x, e0.y);
        A = A1;
        Q = Q1;
        R = R1;
        continue;
      }
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

}  // namespace

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
LtGuideFn lt_guide_kernel(bool lite) {
  static bool attr = false;
  if (!attr) {
    RRG_CUDA(cudaFuncSetAttribute(k_sample_lt_guide<6, 384, 3>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    RRG_CUDA(cudaFuncSetAttribute(k_sample_lt_guide<6, 384, 3, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr = true;
  }
  if (lite) return k_sample_lt_guide<6, 384, 3, true>;
  return lt_filter_variant() ? k_sample_lt_guide<6, 384, 3> : k_sample_lt_guide<5, 128, 4>;
}
size_t lt_guide_smem(bool lite) { return (lite || lt_filter_variant() ? 64u : 32u) * kBlock * 4u; }


int lt_blocks_per_sm(int lt_mode) {
  int b = 0;
  if (lt_mode == kLtGuide)
    RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, lt_guide_kernel(false), kBlock,
                                                           lt_guide_smem(false)));
  else
    RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample_lt<16>, kBlock, 0));
  return b;
}

void launch_lt_sampler(const SampleParams& p, int grid, cudaStream_t s) {
  if (p.lt_scan == kLtGuide) {
    const bool lite = p.ltlite != nullptr;  // the host passes exactly one of the two tables
    lt_guide_kernel(lite)<<<grid, kBlock, lt_guide_smem(lite), s>>>(p);
  } else {
    switch (p.lt_kary) {
      case 2: k_sample_lt<2><<<grid, kBlock, 0, s>>>(p); break;
      case 4: k_sample_lt<4><<<grid, kBlock, 0, s>>>(p); break;
      case 8: k_sample_lt<8><<<grid, kBlock, 0, s>>>(p); break;
      default: k_sample_lt<16><<<grid, kBlock, 0, s>>>(p); break;
    }
  }
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
    host_sync((g->stream));  // longv is released at scope end
  }
  uint32_t hbad = 0;
  RRG_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
  host_sync((g->stream));
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
  host_sync((g->stream));
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
  host_sync((g->stream));
}

// The lite guide table: 8 bytes per bucket, kGuideLiteMult buckets per in-edge,
// built from the offsets and the CDF alone (no candidate infos). It serves the
// small batches of a graph that has no full table yet: an IMM run from host
// arrays samples a few thousand walks, for which the full table's build (cfg4:
// 4.5 ms, 8.8 GB) costs more than it saves; with a model hint the lite table is
// built while the sources are still uploading (rrg_graph_create_for).
constexpr uint32_t kGuideLiteMult = 2;
bool prepare_lt_lite(rrg_graph* g) {
  if (!g->cdf_monotone || !g->m) return false;
  if (g->ltlite.ptr) return true;
  if (g->m >= (1ull << 30)) return false;  // a span (<= an in-degree) must fit the 30 pivot bits
  const uint64_t entries = static_cast<uint64_t>(kGuideLiteMult) * g->m;
  size_t freeb = 0, totalb = 0;
  RRG_CUDA(cudaMemGetInfo(&freeb, &totalb));
  if (entries * 8 + (2ull << 30) > freeb) return false;
  g->ltlite.reserve_discard(entries);
  const uint64_t chunks = (entries + kGuideChunk - 1) / kGuideChunk;
  const uint64_t grid = std::min<uint64_t>((chunks + 127) / 128, 1u << 20);
  k_build_ltguide<true><<<static_cast<unsigned>(grid), 128, 0, g->stream>>>(
      g->off.ptr, g->cdf.ptr, nullptr, g->n, g->m, kGuideLiteMult, nullptr, g->ltlite.ptr);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  host_sync((g->stream));
  return true;
}

// LT guide mode: 32 bytes per bucket, mult buckets per in-edge. False (and no
// table) when the CDF is not monotone or the table would not fit in free HBM.
// batch_sets (0: an explicit prepare) decides what a graph WITHOUT a full table
// does: a batch below kGuideLightSets walks runs on the lite table (*lite =
// true), and the first large batch -- or kGuideLightTotal walks of small ones
// -- builds the full table and drops the lite one. A multiplier set through
// RRG_OPT_LT_GUIDE_MULT always means the full table.
constexpr uint64_t kGuideLightSets = 1ull << 17;
constexpr uint64_t kGuideLightTotal = 1ull << 19;
bool prepare_lt_guide(rrg_graph* g, uint64_t batch_sets, bool* lite) {
  *lite = false;
  if (!g->cdf_monotone || !g->m) return false;
  if (g->lt_guide_built == g->lt_guide_mult && g->ltguide.ptr) return true;
  if (!g->lt_guide_mult_explicit && batch_sets && batch_sets < kGuideLightSets &&
      g->lt_light_walks + batch_sets <= kGuideLightTotal && prepare_lt_lite(g)) {
    g->lt_light_walks += batch_sets;
    *lite = true;
    return true;
  }
  g->ltlite.release();
  g->ltguide.release();
  g->lt_guide_built = 0;
  const uint64_t entries = static_cast<uint64_t>(g->lt_guide_mult) * g->m;
  size_t freeb = 0, totalb = 0;
  RRG_CUDA(cudaMemGetInfo(&freeb, &totalb));
  if (entries * 32 + (2ull << 30) > freeb) return false;
  g->ltguide.reserve_discard(2 * entries);
  const uint64_t chunks = (entries + kGuideChunk - 1) / kGuideChunk;
  const uint64_t grid = std::min<uint64_t>((chunks + 127) / 128, 1u << 20);
  k_build_ltguide<false><<<static_cast<unsigned>(grid), 128, 0, g->stream>>>(
      g->off.ptr, g->cdf.ptr, g->src.ptr, g->n, g->m, g->lt_guide_mult, g->ltguide.ptr, nullptr);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  host_sync((g->stream));
  g->lt_guide_built = g->lt_guide_mult;
  return true;
}

uint32_t lt_lite_mult() { return kGuideLiteMult; }

// The structures the graph's LT scan mode needs; returns the mode launches use.
int prepare_lt_mode(rrg_graph* g, uint64_t batch_sets, bool* lite) {
  *lite = false;
  prepare_lt(g);
  if (g->lt_scan == kLtGuide && prepare_lt_guide(g, batch_sets, lite)) return kLtGuide;
  if (g->lt_scan == kLtLinear || !g->cdf_monotone) return kLtLinear;
  prepare_lt_search(g);
  return kLtBsearch;
}

}  // namespace rrgpu
