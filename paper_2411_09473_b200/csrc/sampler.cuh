// sampler.cuh -- device building blocks shared by the sampler translation units
// (sample.cu core + big-set path, sample_ic.cu, sample_lt.cu): the slot
// dispensers, the staging emit, the per-lane visited inserts and the
// warp-cooperative IC in-list expansion (coop_expand). Everything is in an
// unnamed namespace: each translation unit gets its own copy.
#pragma once

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

// Fused-counter increment. North star (4) asks for warp-aggregated atomics; with
// RRG_WARP_AGG the lanes of the warp that are here together and add the same
// vertex issue one atomic with their count. Measured (profiles/r2/NOTES.md):
// +20 % on cfg2 (lane walks, search mode), +12 % on cfg4, +3 % on cfg3 -- the
// lanes of a warp emit different sets whose members rarely coincide at the
// same instant, so __match_any_sync costs more than the fire-and-forget L2
// reductions it saves. Default: one RED per member (the counter is L2-resident).
// Where counts do coincide -- dense rows -- they are aggregated by construction
// (bit-sliced column sums, one atomic per vertex and 32-row chunk, dense.cu).
__device__ __forceinline__ void counter_add(uint32_t* counter, uint32_t v) {
#ifndef RRG_WARP_AGG
  atomicAdd(counter + v, 1u);
  return;
#endif
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, v);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counter + v, __popc(peers));
}

// Records a staged set's length in the batch maximum: an atomic only when the
// set beats the maximum seen so far (a few per batch), so the host learns the
// batch's longest list without reading the store back.
__device__ __forceinline__ void note_len(const SampleParams& p, uint32_t n) {
  if (n > *reinterpret_cast<volatile unsigned*>(&p.ctl->max_len)) atomicMax(&p.ctl->max_len, n);
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
      RRG_DCHECK(v[q] < p.n, 1);
      out[t + q] = v[q];
      if (p.counter) counter_add(p.counter, v[q]);
    }
  }
  for (; t < nmem; ++t) {
    const uint32_t v = mem[t];
    RRG_DCHECK(v < p.n, 1);
    out[t] = v;
    if (p.counter) counter_add(p.counter, v);
  }
  p.slot_start[idx] = pos;
  p.slot_len[idx] = nmem;
  note_len(p, nmem);
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
  RRG_DCHECK(nmem < kMemCap, 2);
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
#define RRG_CLASSIFY_BATCH 2
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

#ifndef RRG_COOP_INLINE
#define RRG_COOP_INLINE
#endif
template <int kVis>
__device__ RRG_COOP_INLINE bool coop_expand(const SampleParams& p, uint32_t jb, uint32_t je, uint32_t* mem,
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

}  // namespace

}  // namespace rrgpu
