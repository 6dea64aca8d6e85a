// sample_ic.cu -- K1: the IC samplers (sampling.hpp:90-111 per slot, :159-199
// per batch) in their three schedules (lane, warp, thread block per sample),
// the opt-in fast mode, and the IC K0 layouts (edge records, duplicate-free and
// uniform-weight flags, GF(2) jump tables, largest in-degree). See sample.cu
// for the execution model shared by all samplers.
#include <map>
#include <mutex>

#include "sampler.cuh"

namespace rrgpu {

namespace {

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
        // the expansion may have grown the table under a fresh tag before it
        // gave up: the lane's next tag must come after that one, or the next
        // sample would see the abandoned entries as its own (a full table, an
        // endless probe chain)
        tag = s.tag;
        if (ok) {
          rng = Xoshiro{s.a, s.b, s.c, s.d};
          flt.lo = s.flo;
          flt.hi = s.fhi;
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
// Epoch-tagged variant for the block schedule's in-window repairs: slot =
// (source << 32 | epoch << 12 | position), positions < 4096; entries of another
// epoch read as empty, so moving to the next epoch clears the map.
template <int kLog>
__device__ __forceinline__ bool amap_insert_ep(unsigned long long* map, uint32_t v, uint32_t e,
                                               uint32_t ep) {
  constexpr uint32_t kSlots = 1u << kLog;
  const unsigned long long want = (static_cast<unsigned long long>(v) << 32) | (ep << 12) | e;
  uint32_t h = vhash(v) >> (32 - kLog);
  for (uint32_t probe = 0; probe < kSlots; ++probe, h = (h + 1) & (kSlots - 1)) {
    unsigned long long cur = map[h];
    while (((cur >> 12) & 0xfffffu) != ep) {  // empty or stale: claim it
      const unsigned long long got = atomicCAS(map + h, cur, want);
      if (got == cur) return true;
      cur = got;
    }
    if ((cur >> 32) == v) {
      atomicMin(map + h, want);
      return true;
    }
  }
  return false;
}
template <int kLog>
__device__ __forceinline__ uint32_t amap_first_ep(const unsigned long long* map, uint32_t v,
                                                  uint32_t ep) {
  constexpr uint32_t kSlots = 1u << kLog;
  uint32_t h = vhash(v) >> (32 - kLog);
  for (uint32_t probe = 0; probe < kSlots; ++probe, h = (h + 1) & (kSlots - 1)) {
    const unsigned long long cur = map[h];
    if (((cur >> 12) & 0xfffffu) != ep) return 0xffffffffu;
    if ((cur >> 32) == v) return static_cast<uint32_t>(cur) & 0xfffu;
  }
  return 0xffffffffu;
}
// K lookups of amap_first_ep with their first probes in flight together.
template <int kLog, int K>
__device__ __forceinline__ void amap_first_ep_batch(const unsigned long long* map,
                                                    const uint32_t (&vs)[K], uint32_t want,
                                                    uint32_t ep, uint32_t (&out)[K]) {
  constexpr uint32_t kSlots = 1u << kLog;
  uint32_t h[K];
  unsigned long long x[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    h[q] = vhash(vs[q]) >> (32 - kLog);
    x[q] = ((want >> q) & 1u) ? map[h[q]] : 0ull;
  }
#pragma unroll
  for (int q = 0; q < K; ++q) {
    out[q] = 0xffffffffu;
    if (!((want >> q) & 1u)) continue;
    unsigned long long cur = x[q];
    uint32_t hh = h[q];
    for (uint32_t probe = 0; probe < kSlots; ++probe) {
      if (((cur >> 12) & 0xfffffu) != ep) break;
      if ((cur >> 32) == vs[q]) {
        out[q] = static_cast<uint32_t>(cur) & 0xfffu;
        break;
      }
      hh = (hh + 1) & (kSlots - 1);
      cur = map[hh];
    }
  }
}
// K inserts of amap_insert_ep with their probes and CASes in flight together;
// returns the mask of the ones that found the map full.
template <int kLog, int K>
__device__ __forceinline__ uint32_t amap_insert_ep_batch(unsigned long long* map,
                                                         const uint32_t (&vs)[K],
                                                         const uint32_t (&es)[K], uint32_t pend,
                                                         uint32_t ep) {
  constexpr uint32_t kSlots = 1u << kLog;
  uint32_t h[K], probes[K], failed = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    h[q] = vhash(vs[q]) >> (32 - kLog);
    probes[q] = 0;
  }
  while (pend) {
    unsigned long long cur[K], r[K];
#pragma unroll
    for (int q = 0; q < K; ++q)
      cur[q] = ((pend >> q) & 1u) ? *reinterpret_cast<volatile unsigned long long*>(map + h[q]) : 0ull;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      r[q] = ~cur[q];
      if (((pend >> q) & 1u) && ((cur[q] >> 12) & 0xfffffu) != ep)
        r[q] = atomicCAS(map + h[q], cur[q],
                         (static_cast<unsigned long long>(vs[q]) << 32) | (ep << 12) | es[q]);
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (!((pend >> q) & 1u)) continue;
      if (((cur[q] >> 12) & 0xfffffu) != ep) {
        if (r[q] == cur[q]) pend &= ~(1u << q);  // claimed (else: re-read the slot)
      } else if ((cur[q] >> 32) == vs[q]) {
        atomicMin(map + h[q], (static_cast<unsigned long long>(vs[q]) << 32) | (ep << 12) | es[q]);
        pend &= ~(1u << q);
      } else {
        h[q] = (h[q] + 1) & (kSlots - 1);
        if (++probes[q] >= kSlots) {
          failed |= 1u << q;
          pend &= ~(1u << q);
        }
      }
    }
  }
  return failed;
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
    uint32_t wspent = 0;         // windows spent on this set (edge budget, p.warp_win_budget)
    while (qi < s.nmem && ok) {
      if (p.warp_win_budget && ++wspent > p.warp_win_budget) {
        ok = false;  // a large set: handed to the block schedule (deferred pass)
        break;
      }
      {  // a long duplicate-free in-list at the head: 1024-edge windows of one list
        const uint32_t u = mem[qi];
        const uint32_t je = p.off[u + 1];
        if (je - qj >= p.ic_coop_min && p.dupfree[u]) {
          wspent += (je - qj) / kWin;
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
      note_len(p, s.nmem);
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
// Threads per block of this schedule: 256 (8 warps, 512 window positions each,
// two blocks per SM) or 512 (16 warps, 256 positions each, one block per SM; the
// block still owns the scratch of 256 lane regions). Measured (profiles/r2/
// NOTES.md): 512 threads run ONE set 1.2-1.3x faster (cfg3's 35,624-member set
// 10.1 -> 7.6 ms) but halve the sets in flight, and IMM-sized batches lose more
// than their tail gains (cfg1 IMM 11.4 -> 13.7 ms, cfg3 19.6 -> 20.9 ms, cfg3c
// 4.1 -> 5.2 s): 256 stays the default.
#ifndef RRG_CTA_THREADS
#define RRG_CTA_THREADS 256
#endif
constexpr int kCtaThreads = RRG_CTA_THREADS;
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr uint32_t kCtaWin = 4096;                       // in-edges per window
constexpr uint32_t kCtaSlice = kCtaWin / kCtaWarps;      // window positions per warp
constexpr uint32_t kCtaSliceChunks = kCtaSlice / 32;
static_assert(kCtaThreads == 256 || kCtaThreads == 512, "8 or 16 warps per block");
constexpr int kCtaAmapLog = 11;                 // 2048 slots; a full map cuts the window
#ifndef RRG_CTA_FILT_LOG
#define RRG_CTA_FILT_LOG 18
#endif
constexpr int kCtaFiltLog = RRG_CTA_FILT_LOG;  // visited filter: 2^18 bits = 32 KB
constexpr uint32_t kCtaFilterWords = 1u << (kCtaFiltLog - 5);
constexpr uint32_t kCtaFastMin = 1024;          // single-list fast windows from this length
constexpr uint32_t kJumpTableWords = 32 * 256 * 4;
constexpr int kLxCpl = RRG_LX_CPL;            // list expansion: 32-edge chunks per lane
constexpr uint32_t kLxPer = 32u * kLxCpl;     // draws per lane per sub-window
constexpr uint32_t kLxWords = 32u * kLxCpl;   // mask words (chunks) per sub-window
struct CtaWarpFields {
  uint32_t mask[kCtaSliceChunks];
  uint32_t pre[kCtaSliceChunks];
  uint32_t acc[kCtaSliceChunks];
  union {
    struct {
      uint32_t thr[kCtaSlice];
      uint32_t src[kCtaSlice];
    };
    uint32_t lxthr[kLxWin];  // list expansion: the sub-window's thresholds (unequal weights)
  };
  uint32_t lxmask[kLxWords], lxpre[kLxWords], lxacc[kLxWords];  // list expansion: per chunk
  unsigned long long st[4];  // list expansion: the warp's stream state after a sub-window
};
struct CtaSmem {
  CtaWarpFields w[kCtaWarps];
  unsigned long long amap[1u << kCtaAmapLog];
  uint32_t filt[kCtaFilterWords];
  uint32_t lstart[kCtaThreads];
  uint32_t lpre[kCtaThreads];
  unsigned long long st[4];
  unsigned long long next;
  uint32_t wsum[kCtaWarps];
  uint32_t wU[kCtaWarps];
  uint32_t wA[kCtaWarps];
  uint32_t cut;
  uint32_t fcut;  // first edge the window cannot settle (full map, or a repaired tie)
  uint32_t adv_qi;
  uint32_t adv_qj;
  uint32_t any_acc;
};
// The accepted edges of warp slice `ws` at positions [lo, hi) into the map
// (epoch ep), four chunks at a time; returns this lane's smallest position
// that found the map full (or ~0u).
__device__ __forceinline__ uint32_t warp_map_accepts(unsigned long long* amap,
                                                     const CtaWarpFields& ws, uint32_t wbase,
                                                     uint32_t nch, uint32_t lo, uint32_t hi,
                                                     uint32_t ep) {
  const int lane = threadIdx.x & 31;
  uint32_t fail = 0xffffffffu;
  for (uint32_t c0 = 0; c0 < nch && wbase + 32 * c0 < hi; c0 += 4) {
    if (wbase + 32 * (c0 + 4) <= lo) continue;
    uint32_t vs[4], es[4], pend = 0;
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      const uint32_t c = c0 + q, e = wbase + 32 * c + lane;
      const bool w = c < nch && ((ws.acc[c] >> lane) & 1u) && e >= lo && e < hi;
      vs[q] = w ? ws.src[32 * c + lane] : 0u;
      es[q] = e;
      pend |= (w ? 1u : 0u) << q;
    }
    if (!pend) continue;
    const uint32_t f = amap_insert_ep_batch<kCtaAmapLog, 4>(amap, vs, es, pend, ep);
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
      if ((f >> q) & 1u) fail = min(fail, es[q]);
  }
  return fail;
}

// The first window position in [lo, lim) of warp slice `ws` whose edge draws
// and whose source the map (epoch ep) holds at an earlier position, folded
// into *cut with atomicMin; four chunks' lookups in flight at a time.
__device__ __forceinline__ void warp_first_conflict(const unsigned long long* amap,
                                                    const CtaWarpFields& ws, uint32_t wbase,
                                                    uint32_t nch, uint32_t lo, uint32_t lim,
                                                    uint32_t ep, uint32_t* cut) {
  const int lane = threadIdx.x & 31;
  for (uint32_t c0 = 0; c0 < nch && wbase + 32 * c0 < lim; c0 += 4) {
    if (wbase + 32 * (c0 + 4) <= lo) continue;
    uint32_t vs[4], f[4], want = 0;
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      const uint32_t c = c0 + q, e = wbase + 32 * c + lane;
      const bool w = c < nch && ((ws.mask[c] >> lane) & 1u) && e >= lo && e < lim;
      vs[q] = w ? ws.src[32 * c + lane] : 0u;
      want |= (w ? 1u : 0u) << q;
    }
    if (!__any_sync(kFull, want != 0)) continue;
    amap_first_ep_batch<kCtaAmapLog, 4>(amap, vs, want, ep, f);
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
      const uint32_t e = wbase + 32 * (c0 + q) + lane;
      const unsigned b = __ballot_sync(kFull, ((want >> q) & 1u) && f[q] < e);
      if (b) {
        if (lane == 0) atomicMin(cut, wbase + 32 * (c0 + q) + __ffs(b) - 1);
        return;
      }
    }
  }
}
constexpr size_t kCtaKernelDynSmem = sizeof(CtaSmem);
static_assert(kCtaKernelDynSmem <= (kCtaThreads > 256 ? 200 : 97) * 1024,
              "one 512-thread block, or two 256-thread blocks, per SM within the shared-memory carveout");
constexpr uint32_t kMaxRepairs = 64;  // repairs per window before falling back to a cut
#ifndef RRG_REPAIR_MIN
#define RRG_REPAIR_MIN 1024
#endif
// A conflict is repaired only when at least this many window edges follow it;
// closer to the window's end a cut (and a fresh window) is cheaper.
constexpr uint32_t kRepairMin = RRG_REPAIR_MIN;
__device__ __forceinline__ uint32_t cfilt_bit(uint32_t v) { return (v * 0x2545F491u) >> (32 - kCtaFiltLog); }
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
#ifndef RRG_WARP_JUMP_CALL
#define RRG_WARP_JUMP_CALL 1
#endif
#if RRG_WARP_JUMP_CALL
// a real call: 22 inlined copies (40 shuffles each) were ~75 KB of the block
// schedule's 282 KB of code
#define RRG_WJ_INLINE __noinline__
#else
#define RRG_WJ_INLINE __forceinline__
#endif
__device__ RRG_WJ_INLINE Xoshiro warp_jump_fn(const uint64_t* __restrict__ T, uint64_t a, uint64_t b,
                                              uint64_t c, uint64_t d) {
  const int lane = threadIdx.x & 31;
  const uint64_t wv = lane < 8 ? a : lane < 16 ? b : lane < 24 ? c : d;
  const uint32_t byte = static_cast<uint32_t>(wv >> (8 * (lane & 7))) & 255u;
  const ulonglong2* e = reinterpret_cast<const ulonglong2*>(T + (static_cast<size_t>(lane) * 256 + byte) * 4);
  ulonglong2 x = __ldg(e), y = __ldg(e + 1);
  for (int o = 16; o; o >>= 1) {
    x.x ^= __shfl_xor_sync(kFull, x.x, o);
    x.y ^= __shfl_xor_sync(kFull, x.y, o);
    y.x ^= __shfl_xor_sync(kFull, y.x, o);
    y.y ^= __shfl_xor_sync(kFull, y.y, o);
  }
  return Xoshiro{x.x, x.y, y.x, y.y};
}
__device__ __forceinline__ void warp_jump(const uint64_t* __restrict__ T, Xoshiro& st) {
  st = warp_jump_fn(T, st.a, st.b, st.c, st.d);
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
  const uint32_t per = (W + kCtaThreads - 1) / kCtaThreads;
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
  for (int w = 0; w < kCtaThreads / 32; ++w) {
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

// Block-wide insert of mem[lo, hi) into the sample's table, four probe chains in
// flight per thread (the appends used to wait one CAS round trip per 32-edge
// chunk, the grows one per member).
__device__ __forceinline__ void cta_tab_insert(uint64_t* tab, uint32_t tag, uint32_t lg,
                                               const uint32_t* mem, uint32_t lo, uint32_t hi) {
  for (uint32_t b = lo + threadIdx.x; b < hi; b += 4 * kCtaThreads) {
    uint32_t vs[4], pend = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t i = b + q * kCtaThreads;
      vs[q] = i < hi ? mem[i] : 0u;
      pend |= (i < hi ? 1u : 0u) << q;
    }
    tab_insert_atomic_batch<4>(tab, tag, lg, vs, pend);
  }
}

// RRG_CTA_PHASES (diagnostic builds): thread 0 of each block accumulates the
// cycles between the schedule's barriers per phase and prints them at exit.
#ifdef RRG_CTA_PHASES
#define RRG_PH(k)                           \
  do {                                      \
    if (tid == 0) {                         \
      const long long t_ = clock64();       \
      ph_[k] += t_ - ph_t_;                 \
      ph_t_ = t_;                           \
    }                                       \
  } while (0)
#else
#define RRG_PH(k) \
  do {            \
  } while (0)
#endif
// Visited-set primitives of the block schedule: the tagged hash table + the
// shared-memory filter in front of it, or -- giant variant -- an n-bit map per
// block (L2-resident: 204 KB per block at n = 1.6M) with no filter: a giant set
// saturates any filter, and a 2M-entry hash table per block sends every probe
// to DRAM (ncu: 1.36 TB read for 2,048 cfg3c sets with tables).
template <bool kGiant, int K>
__device__ __forceinline__ uint32_t cta_contains(const uint64_t* tab, const uint32_t* gbits,
                                                 uint32_t tag, uint32_t lg,
                                                 const uint32_t (&vs)[K], uint32_t maybe) {
  if (!kGiant) return tab_contains_batch<K>(tab, tag, lg, vs, maybe);
  uint32_t w[K];
#pragma unroll
  for (int q = 0; q < K; ++q) w[q] = ((maybe >> q) & 1u) ? gbits[vs[q] >> 5] : 0u;
  uint32_t found = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) found |= ((w[q] >> (vs[q] & 31)) & 1u) << q;
  return found;
}

template <bool kGiant>
__device__ __forceinline__ void cta_insert_range(uint64_t* tab, uint32_t* gbits, uint32_t tag,
                                                 uint32_t lg, const uint32_t* mem, uint32_t lo,
                                                 uint32_t hi) {
  if (!kGiant) {
    cta_tab_insert(tab, tag, lg, mem, lo, hi);
    return;
  }
  for (uint32_t i = lo + threadIdx.x; i < hi; i += kCtaThreads) {
    const uint32_t v = mem[i];
    atomicOr(gbits + (v >> 5), 1u << (v & 31));
  }
}

template <bool kGiant>
__device__ __forceinline__ bool cta_filter_maybe(const uint32_t* sf, uint32_t v) {
  return kGiant ? true : cfilt_maybe(sf, v);
}

template <bool kGiant>
__device__ __forceinline__ void cta_filter_add(uint32_t* sf, uint32_t v) {
  if (!kGiant) cfilt_add(sf, v);
}

// kGiant: the same schedule for the sets the block scratch (256K members) could
// not hold -- the giant-component sets of supercritical graphs (cfg3c: ~1/3 of
// the sets, ~500K members each). Per block a private list of kGiantCap members
// and a table of 2 kGiantCap entries (own tag range); a set of >= dense_thr
// members is written straight into a row of the dense arm (rrr_set.hpp:82-83).
// Sets past kGiantCap go on to the big-set path.
template <bool kGiant>
__global__ void __launch_bounds__(kCtaThreads, kCtaThreads > 256 ? 1 : RRG_IC_MIN_BLOCKS)
    k_sample_ic_cta(const SampleParams p) {
  constexpr uint32_t kCap = kGiant ? kGiantCap : kBlock * kMemCap;
  extern __shared__ __align__(16) unsigned char k_dsm[];
  CtaSmem& cs = *reinterpret_cast<CtaSmem*>(k_dsm);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wl = tid >> 5;
  CtaWarpFields& ws = cs.w[wl];
  const uint64_t region = static_cast<uint64_t>(blockIdx.x) * kBlock;
  if (region + kBlock > p.lanes) return;  // uniform per block
  if (kGiant && blockIdx.x >= p.gctas) return;
  uint32_t* mem = kGiant ? p.glists + static_cast<uint64_t>(blockIdx.x) * kGiantCap
                         : p.lists + region * kMemCap;
  uint64_t* tab = kGiant ? nullptr : p.tabs + region * kTabCap;
  uint32_t* gbits = kGiant ? p.gbits + static_cast<uint64_t>(blockIdx.x) * p.gwords : nullptr;
  // general windows: high word of the draw at each stream rank (global: kept
  // out of shared memory so two blocks still leave L1 its share)
  uint32_t* xhi = p.xhi + static_cast<size_t>(blockIdx.x) * kCtaWin;
  uint32_t* sf = cs.filt;
  for (uint32_t t = tid; t < kCtaFilterWords; t += kCtaThreads) sf[t] = 0;
  // same 256-lane regions and tag range as the 256-lane warp layout; the giant
  // tables are private to the block and count their own tags
  const uint64_t tslot = region / 32;
  uint32_t tag = kGiant ? p.gtags[blockIdx.x] : 0xC0000000u | (p.wtags[tslot] & 0x3fffffffu);
  uint64_t insp = 0;
  const uint32_t wbase = kCtaSlice * wl;  // this warp's first window position
#ifdef RRG_CTA_PHASES
  long long ph_[16] = {0}, ph_t_ = clock64();
#endif
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
      if (kGiant) atomicOr(gbits + (root >> 5), 1u << (root & 31));
      else tab_insert(tab, stag, lg, root);
      cta_filter_add<kGiant>(sf, root);
    }
    __syncthreads();
    RRG_PH(0);
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
            (uni || kLxWin <= sizeof(ws.lxthr) / 4)) {  // uniform across the block
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
                maybe |= (32 * (16 * part + q) + lane < wend && cta_filter_maybe<kGiant>(sf, vv[q]) ? 1u : 0u) << q;
              const uint32_t seen = cta_contains<kGiant, 16>(tab, gbits, stag, lg, vv, maybe);
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
          RRG_PH(12);
          // (2) stream positions of the sub-windows
          const uint32_t U = block_exscan_global(xc, W, cs.wsum);
          RRG_PH(13);
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
          RRG_PH(14);
          // (4) accepted sources, appended in CSR order
          const uint32_t A = block_exscan_global(xA, W, cs.wsum);
          if (U) s = Xoshiro{cs.st[0], cs.st[1], cs.st[2], cs.st[3]};
          if (A) {
            if (nmem + A > kCap) {
              ok = false;
            } else {
              uint32_t lg2 = lg;
              while (2 * (nmem + A) > (1u << lg2)) ++lg2;
              if (!kGiant && lg2 != lg) {  // grow: re-insert the members under a fresh tag
                lg = lg2;
                ++stag;
                cta_tab_insert(tab, stag, lg, mem, 0, nmem);
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
                      cta_filter_add<kGiant>(sf, v);
                    }
                    base += __popc(am);
                  }
                }
              }
              __syncthreads();  // the appended members are visible block-wide
              cta_insert_range<kGiant>(tab, gbits, stag, lg, mem, nmem, nmem + A);
              nmem += A;
            }
          }
          if (tid == 0) atomicAdd(&p.ctl->windows, 1ull);
          __syncthreads();  // members appended; scratch and cs free
          RRG_PH(1);
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
          const uint32_t wend = wbase < E ? min(kCtaSlice, E - wbase) : 0u;
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
              maybe |= (32 * (c0 + q4) + lane < wend && cta_filter_maybe<kGiant>(sf, vv[q4]) ? 1u : 0u) << q4;
            }
            const uint32_t seen = cta_contains<kGiant, kClassifyBatch>(tab, gbits, stag, lg, vv, maybe);
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
          if (lane < static_cast<int>(kCtaSliceChunks)) {
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
              for (uint32_t step = kCtaSliceChunks / 2; step; step >>= 1)
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
              if (!kGiant && lg2 != lg) {  // grow: re-insert the members under a fresh tag
                lg = lg2;
                ++stag;
                cta_tab_insert(tab, stag, lg, mem, 0, nmem);
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
                  cta_filter_add<kGiant>(sf, v);
                }
                base += __popc(am);
              }
              __syncthreads();  // the appended members are visible block-wide
              cta_insert_range<kGiant>(tab, gbits, stag, lg, mem, nmem, nmem + A);
              nmem += A;
            }
          }
          if (tid == 0) atomicAdd(&p.ctl->windows, 1ull);
          __syncthreads();  // (3) members appended; cs fields free for the next window
          RRG_PH(2);
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
      for (uint32_t t = tid; t < (1u << kCtaAmapLog); t += kCtaThreads) cs.amap[t] = ~0ull;
      __syncthreads();
      if (tid == 0) {  // after the barrier: every thread has read the previous window's
        cs.cut = 0xffffffffu;
        cs.fcut = 0xffffffffu;
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
      RRG_PH(3);
      uint32_t ecur = min(kCtaWin, total);
      // ---- 1. warp wl classifies positions [wbase, wbase + 512) (status at window start)
      uint32_t mymask = 0;
      const uint32_t wend = wbase < ecur ? min(kCtaSlice, ecur - wbase) : 0u;
      // lists holding this warp's first and last position (warp-uniform); the
      // per-edge search then only spans [tlo, thi] -- usually one list
      uint32_t tlo = 0, thi = 0;
      if (wend) {
        for (uint32_t step = kCtaThreads / 2; step; step >>= 1) {
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
          maybe |= (32 * (c0 + q4) + lane < wend && cta_filter_maybe<kGiant>(sf, vv[q4]) ? 1u : 0u) << q4;
        }
        const uint32_t seen = cta_contains<kGiant, 4>(tab, gbits, stag, lg, vv, maybe);
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
      if (lane < static_cast<int>(kCtaSliceChunks)) {
        ws.mask[lane] = mymask;
        ws.pre[lane] = ui - cnt;
        ws.acc[lane] = 0;
      }
      if (lane == 0) cs.wU[wl] = Uw;
      __syncthreads();
      RRG_PH(4);
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
            for (uint32_t step = kCtaSliceChunks / 2; step; step >>= 1)
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
                  (kh == th && bern_tie(x, p.w, win_edge(cs.lstart, cs.lpre, kCtaThreads, wbase + 32 * c + bit))))
                acc |= 1u << bit;
              xhi[Pw + r0 + done] = kh;
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
        uint32_t fail = acm ? warp_map_accepts(cs.amap, ws, wbase, nch, 0u, 0xffffffffu, 0u) : 0xffffffffu;
        fail = __reduce_min_sync(kFull, fail);
        if (lane == 0) {
          if (fail != 0xffffffffu) atomicMin(&cs.fcut, fail);
          if (acm) cs.any_acc = 1;
        }
        __syncthreads();
        RRG_PH(5);
        if (cs.any_acc) {
          // ---- 3b. the first drawn edge whose source an earlier edge accepted
          const uint32_t lim = cs.fcut;
          warp_first_conflict(cs.amap, ws, wbase, nch, 0u, lim, 0u, &cs.cut);
          __syncthreads();
          RRG_PH(6);
          uint32_t rpos = cs.cut, fpos = cs.fcut;
          // ---- 3c. repair: the conflicting edge at rpos does not draw after all.
          // Everything before it is settled; after it, edges whose source a
          // settled edge accepted never draw, the others take the stored draws
          // at their new (lower) stream ranks, and the next conflict -- now only
          // possible against a re-decided acceptance -- is repaired in turn. Each
          // round uses the map under a new epoch (no clearing).
          uint32_t ep = 0;
          for (; rpos < fpos && rpos + kRepairMin < ecur && ep < kMaxRepairs;) {
            ++ep;
            if (lane < static_cast<int>(nch)) {
              const uint32_t e0 = wbase + 32 * lane;
              const uint32_t keep = e0 + 32 <= rpos ? ~0u : e0 >= rpos ? 0u : (1u << (rpos - e0)) - 1u;
              ws.acc[lane] &= keep;
              if (rpos >= e0 && rpos < e0 + 32) ws.mask[lane] &= ~(1u << (rpos - e0));
            }
            __syncwarp();
            warp_map_accepts(cs.amap, ws, wbase, nch, 0u, rpos, ep);  // settled accepts
            __syncthreads();
            if (tid == 0) cs.cut = 0xffffffffu;
            for (uint32_t c0 = 0; c0 < nch; c0 += 4) {  // edges after rpos with a settled source
              if (wbase + 32 * (c0 + 4) <= rpos + 1) continue;
              uint32_t vs[4], f[4], want = 0;
#pragma unroll
              for (uint32_t q = 0; q < 4; ++q) {
                const uint32_t c = c0 + q, el = 32 * c + lane;
                const bool w = c < nch && ((ws.mask[c] >> lane) & 1u) && wbase + el > rpos;
                vs[q] = w ? ws.src[el] : 0u;
                want |= (w ? 1u : 0u) << q;
              }
              amap_first_ep_batch<kCtaAmapLog, 4>(cs.amap, vs, want, ep, f);
#pragma unroll
              for (uint32_t q = 0; q < 4; ++q) {
                const unsigned b = __ballot_sync(kFull, ((want >> q) & 1u) && f[q] != 0xffffffffu);
                if (lane == 0 && b) ws.mask[c0 + q] &= ~b;
              }
              __syncwarp();
            }
            const uint32_t cnt2 = lane < static_cast<int>(nch) ? __popc(ws.mask[lane]) : 0u;
            uint32_t ui2 = cnt2;
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(kFull, ui2, o);
              if (lane >= o) ui2 += y;
            }
            if (lane < static_cast<int>(kCtaSliceChunks)) ws.pre[lane] = ui2 - cnt2;
            if (lane == 31) cs.wU[wl] = ui2;
            __syncthreads();
            Pw = 0;
            U = 0;
            for (int w = 0; w < kCtaWarps; ++w) {
              const uint32_t x = cs.wU[w];
              if (w < wl) Pw += x;
              U += x;
            }
            // acceptance after rpos from the stored draws, at the new ranks (lane =
            // position; four chunks' draw loads in flight)
            uint32_t fl = 0xffffffffu;
            for (uint32_t c0 = 0; c0 < nch; c0 += 4) {
              uint32_t kh[4];
#pragma unroll
              for (uint32_t q = 0; q < 4; ++q) {
                const uint32_t c = c0 + q;
                kh[q] = 0xffffffffu;
                if (c < nch && wbase + 32 * c + 31 > rpos) {
                  const uint32_t m = ws.mask[c];
                  if (((m >> lane) & 1u) && wbase + 32 * c + lane > rpos)
                    kh[q] = xhi[Pw + ws.pre[c] + __popc(m & lanemask_lt())];
                }
              }
#pragma unroll
              for (uint32_t q = 0; q < 4; ++q) {
                const uint32_t c = c0 + q;
                if (c >= nch) break;
                if (wbase + 32 * c + 31 <= rpos) continue;
                const uint32_t e = wbase + 32 * c + lane;
                const bool d = ((ws.mask[c] >> lane) & 1u) && e > rpos;
                const uint32_t th = ws.thr[32 * c + lane];
                if (d && kh[q] == th) fl = min(fl, e);  // needs the low bits: cut there
                const unsigned b = __ballot_sync(kFull, d && kh[q] < th);
                if (lane == 0 && b) ws.acc[c] |= b;
              }
            }
            __syncwarp();
            fl = min(fl, warp_map_accepts(cs.amap, ws, wbase, nch, rpos + 1, 0xffffffffu, ep));  // re-decided
            fl = __reduce_min_sync(kFull, fl);
            if (lane == 0 && fl != 0xffffffffu) atomicMin(&cs.fcut, fl);
            __syncthreads();
            const uint32_t lim2 = cs.fcut;
            warp_first_conflict(cs.amap, ws, wbase, nch, rpos + 1, lim2, ep, &cs.cut);  // the next one
            __syncthreads();
            rpos = cs.cut;
            fpos = cs.fcut;
          }
          RRG_PH(7);
          if (ep) {
            am_lane = lane < static_cast<int>(nch) ? ws.acc[lane] : 0u;
            if (tid == 0) atomicAdd(&p.ctl->repairs, static_cast<unsigned long long>(ep));
          }
          const uint32_t cpos = min(rpos, fpos);
          if (cpos >= ecur && ep && wl == 0) {
            // the stream resumes after the U draws the repaired window used
            Xoshiro st = warp_advance(p, s, min(U, kCtaWin - 1));
            if (U == kCtaWin) st.next();
            if (lane == 0) {
              cs.st[0] = st.a;
              cs.st[1] = st.b;
              cs.st[2] = st.c;
              cs.st[3] = st.d;
            }
          }
          if (cpos < ecur) {
            cut = true;
            const uint32_t cw = cpos / kCtaSlice, cl = cpos % kCtaSlice, cc = cl >> 5, cb = cl & 31;
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
        RRG_PH(8);
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
            if (!kGiant && lg2 != lg) {  // grow: re-insert the members under a fresh tag
              lg = lg2;
              ++stag;
              cta_tab_insert(tab, stag, lg, mem, 0, nmem);
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
                cta_filter_add<kGiant>(sf, v);
              }
              base += __popc(am);
            }
            __syncthreads();  // the appended members are visible block-wide
            cta_insert_range<kGiant>(tab, gbits, stag, lg, mem, nmem, nmem + A);
            nmem += A;
          }
        }
      }
      if (tid == 0) {
        atomicAdd(&p.ctl->windows, 1ull);
        if (cut) atomicAdd(&p.ctl->cuts, 1ull);
      }
      RRG_PH(9);
      // ---- advance past the ecur consumed edges: the first list not wholly consumed
      if (lvalid && incl > ecur && incl - len <= ecur) {
        cs.adv_qi = qi + tid;
        cs.adv_qj = lb + (ecur - (incl - len));
      }
      __syncthreads();
      RRG_PH(10);
      if (cs.adv_qi != 0xffffffffu) {
        qi = cs.adv_qi;
        qj = cs.adv_qj;
      } else {
        qi += min(static_cast<uint32_t>(kCtaThreads), nq - qi);
        if (qi < nmem) qj = p.off[mem[qi]];
      }
    }
    __syncthreads();
    RRG_PH(11);
    // inspected in-edges of the set = sum of its members' in-degrees
    uint64_t sinsp = 0;
    if (ok)
      for (uint32_t t = tid; t < nmem; t += kCtaThreads) sinsp += p.off[mem[t] + 1] - p.off[mem[t]];
    tag = stag;
    for (uint32_t t = tid; t < kCtaFilterWords; t += kCtaThreads) sf[t] = 0;  // filter per sample
    if (kGiant) {  // the block's n-bit map back to zero: exactly mem[0, nmem) is set
      __syncthreads();
      for (uint32_t t = tid; t < nmem; t += kCtaThreads) gbits[mem[t] >> 5] = 0u;
    }
    if (!ok) {
      if (tid == 0) defer_slot(p, idx);
      continue;
    }
    if (kGiant && nmem >= p.dense_thr) {
      // a row of the dense arm: zeroed, the members OR-ed in, counted
      if (tid == 0) cs.next = atomicAdd(&p.ctl->ndense, 1ull);
      __syncthreads();
      const unsigned long long row = cs.next;
      if (row >= p.drow_avail) {
        if (tid == 0) restage_slot(p, idx, 0);  // the row pool grows, then a re-run
        continue;
      }
      const uint64_t grow = p.drow_base + row;
      uint32_t* dst = p.dbits + grow * p.dwords;
      for (uint32_t t = tid; t < p.dwords; t += kCtaThreads) dst[t] = 0u;
      __syncthreads();
      for (uint32_t t = tid; t < nmem; t += kCtaThreads) {
        const uint32_t v = mem[t];
        RRG_DCHECK(v < p.n, 7);
        atomicOr(dst + (v >> 5), 1u << (v & 31));
        if (p.counter) atomicAdd(p.counter + v, 1u);
      }
      if (tid == 0) {
        p.dlen[grow] = nmem;
        p.droot[grow] = mem[0];
        p.dslot[grow] = static_cast<uint32_t>(p.set_base + idx);
        p.bdix[idx] = static_cast<uint32_t>(grow);
        p.slot_start[idx] = 0;
        p.slot_len[idx] = 0;  // empty list range
        atomicAdd(&p.ctl->dense_members, (unsigned long long)nmem);
        atomicMax(&p.ctl->dense_max, nmem);
      }
      insp += sinsp;
      continue;
    }
    if (tid == 0) cs.next = atomicAdd(&p.ctl->cursor, (unsigned long long)nmem);
    __syncthreads();
    const unsigned long long pos = cs.next;
    if (pos + nmem > p.stage_cap) {
      if (tid == 0) restage_slot(p, idx, nmem);
      continue;
    }
    for (uint32_t t = tid; t < nmem; t += kCtaThreads) {
      const uint32_t v = mem[t];
      RRG_DCHECK(v < p.n && nmem <= kCap, 6);
      p.stage[pos + t] = v;
      if (p.counter) atomicAdd(p.counter + v, 1u);
    }
    if (tid == 0) {
      p.slot_start[idx] = pos;
      p.slot_len[idx] = nmem;
      note_len(p, nmem);
    }
    insp += sinsp;
  }
  for (int o = 16; o; o >>= 1) insp += __shfl_xor_sync(kFull, insp, o);
  if (lane == 0 && insp) {
    atomicAdd(&p.ctl->inspected, (unsigned long long)insp);
    atomicAdd(&p.ctl->entries, (unsigned long long)insp);
  }
#ifdef RRG_CTA_PHASES
  if (tid == 0) {
    long long tot = 0;
    for (int k = 0; k < 16; ++k) tot += ph_[k];
    if (tot > 2000000 && blockIdx.x < 3)
      printf("[cta %d] Mcyc total %.2f: between %.2f list %.2f fast %.2f layout %.2f classify %.2f "
             "draw+3a %.2f 3b %.2f repair %.2f cut %.2f append %.2f advance %.2f tail %.2f\n",
             blockIdx.x, tot * 1e-6, ph_[0] * 1e-6, ph_[1] * 1e-6, ph_[2] * 1e-6, ph_[3] * 1e-6,
             ph_[4] * 1e-6, ph_[5] * 1e-6, ph_[6] * 1e-6, ph_[7] * 1e-6, ph_[8] * 1e-6,
             ph_[9] * 1e-6, ph_[10] * 1e-6, ph_[11] * 1e-6);
    if (tot > 2000000 && blockIdx.x < 3)
      printf("[cta %d] list: classify %.2f scan %.2f draws %.2f append %.2f\n", blockIdx.x,
             ph_[12] * 1e-6, ph_[13] * 1e-6, ph_[14] * 1e-6, ph_[1] * 1e-6);
  }
#endif
  if (tid == 0) {
    if (kGiant) p.gtags[blockIdx.x] = tag;
    else p.wtags[tslot] = tag;
  }
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
          note_len(p, nmem);
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
__global__ void k_max_degree(const uint32_t* off, uint32_t n, uint32_t* out) {
  uint32_t best = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    best = max(best, off[v + 1] - off[v]);
  for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(kFull, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

}  // namespace

int ic_blocks_per_sm() {
  int b = 0;
  RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_sample_ic, kBlock, 0));
  return b;
}

void launch_ic_sampler(const SampleParams& p, int grid, uint32_t ic_inner, int schedule,
                       cudaStream_t s) {
  if (schedule != kSchedLane) {
    static bool attr_set = false;  // > 48 KB of dynamic shared memory needs opting in
    if (!attr_set) {
      RRG_CUDA(cudaFuncSetAttribute(k_sample_ic_warp<32>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kWarpKernelDynSmem)));
      RRG_CUDA(cudaFuncSetAttribute(k_sample_ic_cta<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kCtaKernelDynSmem)));
      RRG_CUDA(cudaFuncSetAttribute(k_sample_ic_cta<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kCtaKernelDynSmem)));
      attr_set = true;
    }
    if (schedule == kSchedWarp) k_sample_ic_warp<32><<<grid, kBlock, kWarpKernelDynSmem, s>>>(p);
    else if (schedule == kSchedCtaGiant)
      k_sample_ic_cta<true><<<grid, kCtaThreads, kCtaKernelDynSmem, s>>>(p);
    else k_sample_ic_cta<false><<<grid, kCtaThreads, kCtaKernelDynSmem, s>>>(p);
  } else {
    k_sample_ic<<<grid, kBlock, 0, s>>>(p, ic_inner);
  }
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

// The GF(2) jump tables are constants of xoshiro256** (csrc/jump.cpp), ~39 MB:
// built on the host and uploaded ONCE per device and process, shared by every
// graph (they used to be re-uploaded from pageable memory by each graph's first
// IC batch: ~4 ms of every IMM run from host arrays). Never freed.
struct JumpTables {
  DevBuf<uint64_t> t32, t16, t256, thi, t64;
};
const JumpTables& jump_tables(int device, cudaStream_t st) {
  static std::mutex mu;
  static std::map<int, JumpTables*> per_device;
  std::lock_guard<std::mutex> lock(mu);
  JumpTables*& jt = per_device[device];
  if (jt) return *jt;
  jt = new JumpTables;
  auto up = [&](DevBuf<uint64_t>& d, const std::vector<uint64_t>& h) {
    d.reserve_discard(h.size());
    RRG_CUDA(cudaMemcpyAsync(d.ptr, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
  };
  up(jt->t32, segment_tables(32, 31));
  up(jt->t16, segment_tables(16, 31));
  up(jt->t256, segment_tables(256, 15));
  up(jt->t64, segment_tables(kLxPer, 31));  // list-expansion lanes
  std::vector<uint64_t> hi;  // T^(4096 a), T^(65536 a), T^(2^20 a)
  for (uint64_t seg : {4096ull, 65536ull, 1048576ull}) {
    const std::vector<uint64_t> t = segment_tables(seg, 15);
    hi.insert(hi.end(), t.begin(), t.end());
  }
  up(jt->thi, hi);
  host_sync(st);  // pageable sources: the copies are done when this returns
  return *jt;
}

void prepare_ic_fast(rrg_graph* g) {
  if (g->uniform_ready) return;
  g->uniformw.reserve_discard(g->n ? g->n : 1);
  if (g->n) {
    k_uniform_weights<<<g->num_sms * 16, 256, 0, g->stream>>>(g->off.ptr, g->w.ptr, g->n,
                                                            g->uniformw.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    host_sync((g->stream));
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
    host_sync((g->stream));
  }
  const JumpTables& jt = jump_tables(g->device, g->stream);
  g->jtab = jt.t32.ptr;
  g->jtab16 = jt.t16.ptr;
  g->jtab256 = jt.t256.ptr;
  g->jtabhi = jt.thi.ptr;
  g->jtab64 = jt.t64.ptr;
  g->rec_ready = true;
}

}  // namespace rrgpu
