// common.cuh -- device-side building blocks shared by the rrgpu kernels.
//
//   * the per-slot xoshiro256** stream of the reference (prng.hpp:8-70),
//     reproduced bit-exactly so RRR sets match the CPU path slot for slot;
//   * the exact Bernoulli test of prng.hpp:62 rewritten as one integer compare;
//   * per-lane open-addressing visited sets (tagged, never cleared);
//   * the control block shared by the sampler launches.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rrgpu {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// RNG: prng.hpp:8-13 (splitmix64), :17-20 (derive_stream_seed), :28-31
// (reseed), :33-43 (next_u64), :46 (uniform01), :49-60 (uniform_below).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix_next(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_seed(uint64_t run_seed, uint64_t slot) {
  uint64_t s = run_seed ^ (0x9e3779b97f4a7c15ULL * (slot + 1));
  return splitmix_next(s);
}

struct Xoshiro {
  uint64_t a, b, c, d;

  __device__ __forceinline__ void seed(uint64_t v) {
    a = splitmix_next(v);
    b = splitmix_next(v);
    c = splitmix_next(v);
    d = splitmix_next(v);
  }
  __device__ __forceinline__ static uint64_t rol(uint64_t x, int k) {
    return (x << k) | (x >> (64 - k));
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t out = rol(b * 5, 7) * 9;
    const uint64_t t = b << 17;
    c ^= a;
    d ^= b;
    b ^= c;
    a ^= d;
    c ^= t;
    d = rol(d, 45);
    return out;
  }
  // 53-bit integer behind uniform01(): uniform01() == u53() * 2^-53 exactly.
  __device__ __forceinline__ uint64_t u53() { return next() >> 11; }
  __device__ __forceinline__ double u01() {
    return __ull2double_rn(next() >> 11) * 0x1.0p-53;
  }
  // Lemire multiply-shift with the reference's rejection rule.
  __device__ __forceinline__ uint64_t below(uint64_t bound) {
    uint64_t x = next();
    uint64_t lo = x * bound;
    uint64_t hi = __umul64hi(x, bound);
    if (lo < bound) {
      const uint64_t thr = (0 - bound) % bound;
      while (lo < thr) {
        x = next();
        lo = x * bound;
        hi = __umul64hi(x, bound);
      }
    }
    return hi;
  }
};

// ---------------------------------------------------------------------------
// Exact Bernoulli: uniform01() < (double)w  (prng.hpp:46, :62; sampling.hpp:102)
// uniform01() = k * 2^-53 with integer k < 2^53, and (double)w * 2^53 is exact,
// so the test is k < ceil(w * 2^53).  The threshold is derived from the f32
// bits with integer ops only; NaN and negatives never fire, >= 1 always fires.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t bernoulli_threshold(uint32_t bits) {
  if (bits & 0x80000000u) return 0;                    // negative or -0
  const uint32_t e = bits >> 23;
  const uint32_t f = bits & 0x7fffffu;
  if (e == 0xff) return f ? 0 : (1ull << 53);          // NaN never, +inf always
  if (e == 0) return f ? 1 : 0;                        // subnormal: k < tiny  <=> k == 0
  const uint64_t mant = f | 0x800000u;                 // w = mant * 2^(e-150)
  const int sh = static_cast<int>(e) - 97;             // w*2^53 = mant * 2^(e-97)
  if (sh >= 30) return 1ull << 53;                     // w >= 1: every k fires
  if (sh >= 0) return mant << sh;
  const int rs = -sh;
  if (rs >= 24) return 1;                              // 0 < w*2^53 < 1
  return ((mant - 1) >> rs) + 1;                       // ceil(mant / 2^rs)
}

// IC edge records carry T_hi = T >> 21 of T = ceil(w 2^53) (saturated at
// 2^32 - 1) instead of the weight: with k = x >> 11, x >> 32 = k >> 21, so
// x >> 32 < T_hi accepts and x >> 32 > T_hi rejects exactly; a tie
// (probability 2^-32) is settled from the f32 weight (bern_tie).
__host__ __device__ __forceinline__ uint32_t bern_thr_hi(uint32_t wbits) {
  const uint64_t hi = bernoulli_threshold(wbits) >> 21;
  return hi >= 0xffffffffull ? 0xffffffffu : static_cast<uint32_t>(hi);
}
__device__ __forceinline__ bool bern_tie(uint64_t x, const float* w, uint32_t j) {
  return (x >> 11) < bernoulli_threshold(__float_as_uint(__ldg(w + j)));
}

// ---------------------------------------------------------------------------
// Per-lane visited set: open addressing over u64 entries (tag << 32 | vertex).
// An entry is live only while its tag equals the lane's current tag, so a new
// sample (or a rehash into a larger table) just bumps the tag -- tables are
// never swept. Capacity grows 64 -> kTabCap keeping load <= 1/2.
// ---------------------------------------------------------------------------
constexpr uint32_t kMemCap = 1024;  // members per lane before deferring to the big path
constexpr uint32_t kTabCap = 2048;  // max table entries per lane (2 x kMemCap)
constexpr uint32_t kTabLog0 = 6;    // initial table log2 capacity
constexpr uint32_t kLtRecSmall = 6; // LT vertex record holds the whole in-list up to this degree
constexpr uint32_t kLtLeafMin = 2;  // child ranges up to this go to the plain final stage
constexpr uint32_t kLtLeafMax = 15; // ranges up to this get a LEAF: their CDF and sources

// LT search tree over one in-list's CDF (upper_bound: first cdf > d, or the
// list end). A node over candidate range [lo, hi] holds P pivots cdf[lo + t s],
// s = max(1, ceil((hi - lo) / (P + 1))), t = 1..P (a pivot at or past hi never
// counts); with `below` pivots <= d the answer lies in the child range below,
// of length <= s (so the tree depth follows from the degree alone). The root
// (P = 13) sits in the 64-byte vertex record; below it, 128-byte nodes exist
// for child ranges longer than kLtLeafMin: inner nodes (P = 31) while the range
// exceeds kLtLeafMax, else a leaf holding cdf[lo, hi) and src[lo, hi], which
// resolves the step with no further load. Level 1 has 14 slots (the root's
// children), each deeper level 32 times the one above (mixed-radix numbering).
// Pivots and leaf entries are floats rounded DOWN (f <= p < next(f)): counts are
// exact, an entry with f == the draw rounded down is re-read from the fp64 CDF.
constexpr uint32_t kLtRootPivots = 13;
constexpr uint32_t kLtNodePivots = 31;
constexpr uint32_t kLtFanout = 32;
constexpr uint32_t kLtRootFanout = kLtRootPivots + 1;
__device__ __host__ __forceinline__ uint32_t lt_step(uint32_t lo, uint32_t hi, uint32_t P) {
  const uint32_t s = (hi - lo + P) / (P + 1);
  return s ? s : 1u;
}
__device__ __host__ __forceinline__ void lt_child(uint32_t& lo, uint32_t& hi, uint32_t P,
                                                  uint32_t below) {
  const uint32_t s = lt_step(lo, hi, P);
  const uint32_t nlo = below ? lo + below * s + 1 : lo;
  const uint32_t cap = lo + (below + 1) * s;
  hi = below < P ? (cap < hi ? cap : hi) : hi;
  lo = nlo;
}
// Exact number of entries p_t <= d among P sorted entries stored as rounded-down
// floats w[t] (entry t at cdf[first + t * step]), given dbits = the bits of d
// rounded down to float. For non-negative floats the bit patterns order like
// the values, so f < fd proves p < next(f) <= fd <= d, f > fd proves p >= f > d,
// and only f == fd (d within one float ulp of p) is re-read from the fp64 CDF.
template <uint32_t P>
__device__ __forceinline__ uint32_t lt_count_le(const uint32_t* w, uint32_t dbits, double d,
                                                const double* cdf, uint32_t first, uint32_t step) {
  uint32_t sure = 0, maybe = 0;
#pragma unroll
  for (uint32_t t = 0; t < P; ++t) {
    sure += w[t] < dbits ? 1u : 0u;
    maybe += w[t] <= dbits ? 1u : 0u;
  }
  while (sure < maybe && __ldg(cdf + first + sure * step) <= d) ++sure;
  return sure;
}

// LT guide table (indexed search over each in-list's CDF). Vertex u with
// degree D gets G = mult * D buckets of equal width on the draw's 53-bit
// integer x53 (uniform01() = x53 * 2^-53): bucket g = floor(x53 * G / 2^53),
// i.e. x53 in [ceil(g 2^53 / G), ceil((g+1) 2^53 / G)). With A_g = #{cdf <= the
// bucket's smallest draw}, every draw of bucket g picks an index in
// [A_g, A_{g+1}] (the CDF is non-decreasing), so the entry of bucket g resolves
// the step by itself when the span A_{g+1} - A_g is 0 (no CDF entry falls in
// the bucket) or 1 (one compare against cdf[A_g], stored as a float rounded
// down; equality re-reads the fp64 CDF). Longer spans (rare: ~mult^-2 / 2 of
// the buckets) search cdf[A_g, A_{g+1}). The entry also carries what the NEXT
// step needs of the chosen source -- its id, in-list offset and degree -- so a
// walk step is one 32-byte load. Entry words (guide[2 i], guide[2 i + 1]):
//   x: A_g (local index)  y: pivot bits | kGuideSpan0 | kGuideSearch
//   z, w, x': candidate A_g     -> source id (kGuideNone past the list), off, deg
//   y', z', w': candidate A_g+1 -> source id, off, deg   (span 1)
//               or y' = span                              (kGuideSearch)
constexpr uint32_t kGuideNone = 0xffffffffu;
constexpr uint32_t kGuideSpan0 = 0x40000000u;   // pivots are floats in [0, 1]: bits 30, 31 free
constexpr uint32_t kGuideSearch = 0x80000000u;
constexpr uint32_t kGuidePivot = 0x3fffffffu;

__device__ __forceinline__ uint32_t vhash(uint32_t v) { return v * 0x9E3779B1u; }

// RRG_CHECKED builds (librrgpu_checked.so, tests/test_gpu_checked.py): bounds
// checks at the buffer writes that matter -- member ids < n, list positions
// within their scratch, staging / row / export positions within their buffers
// -- trap with a code instead of corrupting memory. compute-sanitizer is not
// available on the GPU pool; this build is what the parity fixtures run under.
#ifdef RRG_CHECKED
#define RRG_DCHECK(cond, code)                                                      \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("rrgpu check %d failed: blk %d thr %d at %s:%d\n", (code), blockIdx.x,   \
             threadIdx.x, __FILE__, __LINE__);                                      \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define RRG_DCHECK(cond, code) \
  do {                         \
  } while (0)
#endif

// RRG_PROBE_GUARD (debug builds): a probe chain longer than the table traps
// with a code naming the loop, instead of spinning forever.
#ifdef RRG_PROBE_GUARD
#define RRG_GUARD(cnt, lg, code)                                                   \
  if (++(cnt) > (2u << (lg))) {                                                    \
    uint32_t same = 0, minv = 0xffffffffu, maxv = 0;                               \
    for (uint32_t i_ = 0; i_ < (1u << (lg)); ++i_) {                               \
      const uint64_t e_ = tab[i_];                                                 \
      if (static_cast<uint32_t>(e_ >> 32) == tag) {                                \
        ++same;                                                                    \
        minv = min(minv, static_cast<uint32_t>(e_));                               \
        maxv = max(maxv, static_cast<uint32_t>(e_));                               \
      }                                                                            \
    }                                                                              \
    printf("rrgpu probe guard %d: blk %d thr %d tab %p lg %u tag %u v %u same %u "   \
           "vals %u..%u\n", (code), blockIdx.x, threadIdx.x, (const void*)tab,      \
           (lg), tag, v, same, minv, maxv);                                         \
    __trap();                                                                      \
  }
#else
#define RRG_GUARD(cnt, lg, code)
#endif

__device__ __forceinline__ bool tab_contains(const uint64_t* tab, uint32_t tag, uint32_t lg,
                                             uint32_t v) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = vhash(v) >> (32 - lg);
  uint32_t guard = 0;
  while (true) {
    const uint64_t e = tab[h];
    if (static_cast<uint32_t>(e >> 32) != tag) return false;
    if (static_cast<uint32_t>(e) == v) return true;
    h = (h + 1) & mask;
    RRG_GUARD(guard, lg, 1)
  }
}

// K membership tests with every first probe in flight at once (the classify
// loops used to wait one dependent round trip per 32-edge chunk): bit q of
// `maybe` asks for v[q] (a filter hit); returns bit q set when v[q] is present.
template <int K>
__device__ __forceinline__ uint32_t tab_contains_batch(const uint64_t* tab, uint32_t tag,
                                                       uint32_t lg, const uint32_t (&vs)[K],
                                                       uint32_t maybe) {
  if (!maybe) return 0u;
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h[K];
  uint64_t e[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    h[q] = vhash(vs[q]) >> (32 - lg);
    e[q] = ((maybe >> q) & 1u) ? tab[h[q]] : 0ull;
  }
  uint32_t found = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (!((maybe >> q) & 1u)) continue;
    const uint32_t v = vs[q];
    uint64_t x = e[q];
    uint32_t hh = h[q];
    uint32_t guard = 0;
    while (static_cast<uint32_t>(x >> 32) == tag) {
      RRG_GUARD(guard, lg, 4)
      if (static_cast<uint32_t>(x) == v) {
        found |= 1u << q;
        break;
      }
      hh = (hh + 1) & mask;
      x = tab[hh];
    }
  }
  return found;
}

__device__ __forceinline__ void tab_insert(uint64_t* tab, uint32_t tag, uint32_t lg, uint32_t v) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = vhash(v) >> (32 - lg);
  uint32_t guard = 0;
  while (static_cast<uint32_t>(tab[h] >> 32) == tag) {
    h = (h + 1) & mask;
    RRG_GUARD(guard, lg, 2)
  }
  tab[h] = (static_cast<uint64_t>(tag) << 32) | v;
}

// One probe chain for "visited?" and, if not, "insert": true when v was present.
__device__ __forceinline__ bool tab_find_or_insert(uint64_t* tab, uint32_t tag, uint32_t lg,
                                                   uint32_t v) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = vhash(v) >> (32 - lg);
  while (true) {
    const uint64_t e = tab[h];
    if (static_cast<uint32_t>(e >> 32) != tag) {
      tab[h] = (static_cast<uint64_t>(tag) << 32) | v;
      return false;
    }
    if (static_cast<uint32_t>(e) == v) return true;
    h = (h + 1) & mask;
  }
}

// Concurrent insert (several lanes filling one lane's table in the cooperative
// hub expansion). An entry with a stale tag is free; claim it with a CAS.
__device__ __forceinline__ void tab_insert_atomic(uint64_t* tab, uint32_t tag, uint32_t lg,
                                                  uint32_t v) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h = vhash(v) >> (32 - lg);
  const unsigned long long want = (static_cast<unsigned long long>(tag) << 32) | v;
  uint32_t guard = 0;
  while (true) {
    RRG_GUARD(guard, lg, 3)
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(tab + h);
    if (static_cast<uint32_t>(e >> 32) == tag) {
      h = (h + 1) & mask;
      continue;
    }
    if (atomicCAS(reinterpret_cast<unsigned long long*>(tab + h), e, want) == e) return;
  }
}

// K concurrent inserts (bit q of `pend`: insert vs[q]) with their probes and
// CASes in flight together: one round trip per probe step instead of K.
template <int K>
__device__ __forceinline__ void tab_insert_atomic_batch(uint64_t* tab, uint32_t tag, uint32_t lg,
                                                        const uint32_t (&vs)[K], uint32_t pend) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t h[K];
#pragma unroll
  for (int q = 0; q < K; ++q) h[q] = vhash(vs[q]) >> (32 - lg);
  while (pend) {
    unsigned long long e[K], r[K];
#pragma unroll
    for (int q = 0; q < K; ++q)
      e[q] = ((pend >> q) & 1u) ? *reinterpret_cast<volatile unsigned long long*>(tab + h[q]) : 0ull;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      r[q] = ~e[q];
      if (((pend >> q) & 1u) && static_cast<uint32_t>(e[q] >> 32) != tag)
        r[q] = atomicCAS(reinterpret_cast<unsigned long long*>(tab + h[q]), e[q],
                         (static_cast<unsigned long long>(tag) << 32) | vs[q]);
    }
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (!((pend >> q) & 1u)) continue;
      if (static_cast<uint32_t>(e[q] >> 32) == tag) h[q] = (h[q] + 1) & mask;  // taken: next slot
      else if (r[q] == e[q]) pend &= ~(1u << q);                               // claimed
    }
  }
}

// s <- M s over GF(2)^256 (state words a,b,c,d = bits 0..255), M column-major:
// column i = 4 words at M + 4 i (csrc/jump.cpp).
__device__ __forceinline__ void gf2_matvec(const uint64_t* __restrict__ M, uint64_t& a,
                                           uint64_t& b, uint64_t& c, uint64_t& d) {
  uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
  const uint64_t in[4] = {a, b, c, d};
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = in[w];
    while (bits) {
      const int i = __ffsll(static_cast<long long>(bits)) - 1;
      bits &= bits - 1;
      const ulonglong2* col = reinterpret_cast<const ulonglong2*>(M + 4 * (64 * w + i));
      const ulonglong2 x = __ldg(col), y = __ldg(col + 1);
      o0 ^= x.x;
      o1 ^= x.y;
      o2 ^= y.x;
      o3 ^= y.y;
    }
  }
  a = o0;
  b = o1;
  c = o2;
  d = o3;
}

// 32-byte table entry in one load (sm_100: LDG.256).
__device__ __forceinline__ void ld_u64x4(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                         uint64_t& d) {
  asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p));
}

#ifndef RRG_JUMP_CALL
#define RRG_JUMP_CALL 1
#endif
// Same product with byte tables (jump.cpp segment_tables): 32 independent
// 32-byte loads (one LDG.256 each), 16 in flight at a time, then XORs.
__device__ __forceinline__ void gf2_jump_tables_inl(const uint64_t* __restrict__ T, uint64_t& a,
                                                uint64_t& b, uint64_t& c, uint64_t& d) {
  const uint64_t in[4] = {a, b, c, d};
  uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll
  for (int g = 0; g < 4; g += 2) {  // two state words per group: 16 loads in flight
    uint64_t x0[16], x1[16], x2[16], x3[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int p = 8 * g + q;
      const uint32_t byte = static_cast<uint32_t>(in[g + (q >> 3)] >> (8 * (q & 7))) & 255u;
      ld_u64x4(T + (static_cast<size_t>(p) * 256 + byte) * 4, x0[q], x1[q], x2[q], x3[q]);
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      o0 ^= x0[q];
      o1 ^= x1[q];
      o2 ^= x2[q];
      o3 ^= x3[q];
    }
  }
  a = o0;
  b = o1;
  c = o2;
  d = o3;
}

// RRG_JUMP_CALL: the product as a real function call (one copy of its ~10 KB of
// code per kernel instead of one per call site; the block schedule's code was
// 282 KB, far past the instruction caches).
struct JumpState {
  uint64_t a, b, c, d;
};
static __device__ __noinline__ JumpState gf2_jump_call(const uint64_t* __restrict__ T, uint64_t a,
                                                uint64_t b, uint64_t c, uint64_t d) {
  gf2_jump_tables_inl(T, a, b, c, d);
  return JumpState{a, b, c, d};
}
__device__ __forceinline__ void gf2_jump_tables(const uint64_t* __restrict__ T, uint64_t& a,
                                                uint64_t& b, uint64_t& c, uint64_t& d) {
#if RRG_JUMP_CALL
  const JumpState r = gf2_jump_call(T, a, b, c, d);
  a = r.a;
  b = r.b;
  c = r.c;
  d = r.d;
#else
  gf2_jump_tables_inl(T, a, b, c, d);
#endif
}

// 128-bit register filter in front of the table: a clear bit proves absence.
struct Filter {
  uint64_t lo, hi;
  __device__ __forceinline__ void clear() { lo = hi = 0; }
  __device__ __forceinline__ static uint32_t bit(uint32_t v) { return (v * 0x2545F491u) >> 25; }
  __device__ __forceinline__ void add(uint32_t v) {
    const uint32_t b = bit(v);
    if (b & 64) hi |= 1ull << (b & 63);
    else lo |= 1ull << (b & 63);
  }
  __device__ __forceinline__ bool maybe(uint32_t v) const {
    const uint32_t b = bit(v);
    const uint64_t w = (b & 64) ? hi : lo;
    return (w >> (b & 63)) & 1;
  }
};

// ---------------------------------------------------------------------------
// Sampler control block (one per launch sequence of a generate_batch call).
// ---------------------------------------------------------------------------
struct SampleCtl {
  unsigned long long next;        // batch-local slot dispenser
  unsigned long long cursor;      // staging bump allocator (u32 units)
  unsigned long long inspected;   // reference-equivalent in-edges inspected
  unsigned long long entries;     // adjacency entries actually read by the kernel
  unsigned long long restage_members;  // members of sets refused for lack of staging
  unsigned long long windows;     // IC warp schedule: windows processed (diagnostics)
  unsigned long long cuts;        // IC warp schedule: windows cut at a repeated source
  unsigned long long repairs;     // IC block schedule: conflicts repaired inside a window
  unsigned int ndeferred;         // slots handed to the big-set path (set > kMemCap)
  unsigned int nrestage;          // slots to re-run once staging has grown
  unsigned int max_len;           // largest set written to staging (note_len)
  unsigned long long ndense;      // big-set path: rows requested (dense arm)
  unsigned long long dense_members;  // big-set path: members of the rows written
  unsigned int dense_max;         // big-set path: largest row written
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace rrgpu
