// select.cu -- K6: the k-round greedy max-coverage loop, resident on the GPU.
//
// Replaces select_seeds (selection.hpp:209-243) with parallel_argmax (:100-125),
// decrement_update (:130-156) and fill_remaining_seeds (:61-72). One cooperative
// persistent launch runs every round; the host sees nothing until all k rounds
// are done. The argmax is incremental: the vertices are cut into tiles of
// 2^kSelTileLog, each with its max packed key (count << 32 | ~v: max count wins,
// ties go to the lowest id -- the reference's rule, :113, :119-120), and a round
// only re-reduces the tiles whose counts changed. Sets of the dense arm (n-bit
// rows, dense.cu) are found by one bit test each and their counts move by
// column sums; a round whose seed covers more than adaptive_threshold of the
// live sets rebuilds the counter from the survivors instead (rebuild_update,
// selection.hpp:161-203, chosen as at :226-231). A round:
//   A) every block reduces the tile maxima (a few KB, L2) to the same key, so
//      the argmax needs no grid barrier of its own;
//   B) cover: each live set holding v is claimed once (atomicExch on its
//      covered flag); the claimer counts it in the round's marginal and the warp
//      decrements each member (Counter::sub, counter.hpp:28), flagging its tile.
//      The sets holding v are found by scanning the flat member buffer (scan
//      mode: a few MB per round at BASELINE sizes, L2-resident, and no index to
//      build) or through the inverted index vertex -> sets (index mode, for
//      stores too large to re-read every round);
//   -- grid barrier --
//   C) the dirty tiles are re-reduced;
//   -- grid barrier --
#include <cooperative_groups.h>

#include <cstdlib>

#include "internal.hpp"

namespace cg = cooperative_groups;

namespace rrgpu {

namespace {

constexpr int kSelBlock = 512;
constexpr uint32_t kSelTile = 1u << kSelTileLog;
constexpr uint32_t kBlank = 0xffffffffu;  // never a vertex id (ids < n <= 2^32 - 1)
constexpr uint32_t kAllTilesMax = 64;     // up to this many tiles: re-reduce all, no flags

__device__ __forceinline__ unsigned long long pack_key(uint32_t count, uint32_t v) {
  return (static_cast<unsigned long long>(count) << 32) | (0xffffffffu - v);
}

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

// Block-wide max; every thread gets the result. `red` holds kSelBlock/32 words.
__device__ __forceinline__ unsigned long long block_max(unsigned long long x,
                                                        unsigned long long* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) x = umax64(x, __shfl_xor_sync(kFull, x, o));
  __syncthreads();  // red may still be read by a previous call
  if (lane == 0) red[wid] = x;
  __syncthreads();
  x = lane < kSelBlock / 32 ? red[lane] : 0ull;
  for (int o = 16; o; o >>= 1) x = umax64(x, __shfl_xor_sync(kFull, x, o));
  return x;
}

// Max key of tile t by one warp (every lane gets it): 2048 counts as 16
// independent 16-byte loads per lane, shuffle reduction, no block barrier.
__device__ __forceinline__ unsigned long long tile_max_warp(const SelectParams& p, uint32_t t) {
  const int lane = threadIdx.x & 31;
  const uint32_t lo = t << kSelTileLog;
  unsigned long long best = 0;
  if (lo + kSelTile <= p.n) {
    const uint4* c4 = reinterpret_cast<const uint4*>(p.cnt + lo);
    uint4 q[kSelTile / 128];
#pragma unroll
    for (uint32_t i = 0; i < kSelTile / 128; ++i) q[i] = c4[i * 32 + lane];
#pragma unroll
    for (uint32_t i = 0; i < kSelTile / 128; ++i) {
      const uint32_t v = lo + (i * 32 + lane) * 4;
      best = umax64(best, pack_key(q[i].x, v));
      best = umax64(best, pack_key(q[i].y, v + 1));
      best = umax64(best, pack_key(q[i].z, v + 2));
      best = umax64(best, pack_key(q[i].w, v + 3));
    }
  } else {
    for (uint32_t v = lo + lane; v < p.n; v += 32) best = umax64(best, pack_key(p.cnt[v], v));
  }
  for (int o = 16; o; o >>= 1) best = umax64(best, __shfl_xor_sync(kFull, best, o));
  return best;
}

// The warp decrements every member of set s (claimed by one of its lanes).
__device__ __forceinline__ void warp_cover(const SelectParams& p, uint64_t s) {
  const int lane = threadIdx.x & 31;
  const uint64_t b = p.off[s], e = p.off[s + 1];
  for (uint64_t j = b + lane; j < e; j += 32) {
    const uint32_t u = p.mem[j];
    RRG_DCHECK(u < p.n, 11);
    atomicSub(p.cnt + u, 1u);
    p.dirty[u >> kSelTileLog] = 1u;
  }
}

// Column sums over rows of the dense arm, thread per (word, 32-row chunk): the
// rows' words are added into bit-sliced planes and each vertex of the word
// gets one atomic with its count. sign < 0: covered rows (rows = the round's
// kill list), flags the tiles; sign > 0: the live rows (rebuild recount).
__device__ __forceinline__ void sel_colsum(const SelectParams& p, const uint32_t* rows,
                                           uint64_t nrows, int sign, uint64_t tid,
                                           uint64_t nthreads) {
  const uint64_t nchunks = (nrows + 31) / 32;
  const uint64_t items = nchunks * p.dwords;
  for (uint64_t it = tid; it < items; it += nthreads) {
    const uint64_t c = it / p.dwords;
    const uint32_t w = static_cast<uint32_t>(it - c * p.dwords);
    if (static_cast<uint64_t>(w) * 32 >= p.n) continue;
    uint32_t pl[6] = {0, 0, 0, 0, 0, 0};
    const uint64_t d1 = c * 32 + 32 < nrows ? c * 32 + 32 : nrows;
    for (uint64_t d = c * 32; d < d1; ++d) {
      uint64_t row = d;
      if (rows) row = rows[d];
      else if (p.dcov[d]) continue;  // covered rows do not count in a rebuild
      uint32_t x = p.dbits[row * p.dwords + w];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const uint32_t cy = pl[i] & x;
        pl[i] ^= x;
        x = cy;
      }
    }
    uint32_t any = pl[0] | pl[1] | pl[2] | pl[3] | pl[4] | pl[5];
    if (any && sign < 0) p.dirty[(w * 32) >> kSelTileLog] = 1u;
    while (any) {
      const int b = __ffs(any) - 1;
      any &= any - 1;
      uint32_t cnt = 0;
#pragma unroll
      for (int i = 0; i < 6; ++i) cnt |= ((pl[i] >> b) & 1u) << i;
      if (sign < 0) atomicSub(p.cnt + w * 32 + b, cnt);
      else atomicAdd(p.cnt + w * 32 + b, cnt);
    }
  }
}

template <bool kScan>
__global__ void __launch_bounds__(kSelBlock, 1) k_select(const SelectParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long red[kSelBlock / 32];
  const int lane = threadIdx.x & 31;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t gwarp = tid >> 5;
  const uint64_t nwarps = nthreads >> 5;
  const uint32_t ntiles = (p.n + kSelTile - 1) >> kSelTileLog;

  for (uint64_t t = gwarp; t < ntiles; t += nwarps) {
    const unsigned long long m = tile_max_warp(p, static_cast<uint32_t>(t));
    if (lane == 0) {
      p.tmax[t] = m;
      p.dirty[t] = 0u;
    }
  }
  grid.sync();

  unsigned long long covered_sum = 0;  // sets covered in earlier rounds (every thread)
  for (uint32_t r = 0; r < p.k; ++r) {
    // ---- A: argmax over the tile maxima (every block, same answer) ---------
    unsigned long long best = 0;
    for (uint32_t t = threadIdx.x; t < ntiles; t += kSelBlock) best = umax64(best, p.tmax[t]);
    const unsigned long long key = block_max(best, red);
    const uint32_t top = static_cast<uint32_t>(key >> 32);
    const uint32_t v = 0xffffffffu - static_cast<uint32_t>(key);
    if (top == 0) {
      // exhaustion: lowest unselected ids at zero marginal (selection.hpp:61-72)
      if (tid == 0) {
        uint32_t filled = r;
        for (uint32_t u = 0; u < p.n && filled < p.k; ++u) {
          if (!p.selected[u]) {
            p.selected[u] = 1;
            p.seeds[filled] = u;
            p.marg[filled] = 0;
            ++filled;
          }
        }
        p.status[0] = r;  // rounds with a counter snapshot
      }
      return;  // uniform: every block computed the same key
    }
    if (p.need && covered_sum + static_cast<unsigned long long>(p.k - r) * top < p.need) {
      if (tid == 0) p.status[0] = r | kSelAborted;  // the coverage cannot reach `need`
      return;  // uniform: same key and covered_sum in every block
    }

    // rebuild_update vs decrement_update (selection.hpp:226-231): the same rule,
    // the same counts either way (test_selection.cpp:116-137)
    const unsigned long long live = p.nsets - covered_sum;
    const bool rebuild = live > 0 && static_cast<double>(top) / static_cast<double>(live) >
                                         p.adaptive_threshold;

    // ---- B: cover the live sets holding v ------------------------------------
    unsigned long long killed = 0;
    if (rebuild) {
      // kill only; the survivors are recounted below
      if (kScan) {
        const uint64_t nchunk = (p.total + 255) / 256;
        for (uint64_t c = gwarp; c < nchunk; c += nwarps) {
          const uint64_t base = c * 256 + static_cast<uint64_t>(lane) * 8;
          for (int j = 0; j < 8; ++j) {
            const uint64_t t = base + j;
            if (t >= p.total || p.wmem[t] != v) continue;
            ++killed;
            const uint64_t w = p.span[t];
            const uint64_t sb = w >> 32, se = sb + (w & 0xffffffffull);
            for (uint64_t q = sb; q < se; ++q) p.wmem[q] = kBlank;
          }
        }
      } else {
        const uint64_t ib = p.ioff[v], ie = p.ioff[v + 1];
        for (uint64_t t = ib + tid; t < ie; t += nthreads) {
          const uint32_t s = p.inv[t];
          if (!atomicExch(p.covered + s, 1u)) ++killed;
        }
      }
    } else if (kScan) {
      // warp w scans members [256 w', 256 w' + 256) of the working copy for v,
      // eight per lane. Covered sets are blanked there, so every match is a live
      // set, found by exactly one lane: no claim needed; that warp decrements and
      // blanks the set.
      const uint64_t nchunk = (p.total + 255) / 256;
      for (uint64_t c = gwarp; c < nchunk; c += nwarps) {
        const uint64_t base = c * 256 + static_cast<uint64_t>(lane) * 8;
        uint32_t q[8];
        if (base + 8 <= p.total) {
          const uint4 a = *reinterpret_cast<const uint4*>(p.wmem + base);
          const uint4 b = *reinterpret_cast<const uint4*>(p.wmem + base + 4);
          q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
          q[4] = b.x; q[5] = b.y; q[6] = b.z; q[7] = b.w;
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) q[j] = base + j < p.total ? p.wmem[base + j] : kBlank;
        }
        uint32_t hits = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) hits |= (q[j] == v ? 1u : 0u) << j;
        killed += __popc(hits);
        // matched sets: every matching lane loads the span of its lowest match at
        // once (one round trip for the warp), then the warp covers the sets one
        // after the other with the next set's first 128 members loaded while the
        // current one is decremented
        while (__any_sync(kFull, hits != 0)) {
          const uint64_t w = hits ? p.span[c * 256 + static_cast<uint64_t>(lane) * 8 + (__ffs(hits) - 1)]
                                  : 0ull;
          unsigned hm = __ballot_sync(kFull, hits != 0);
          if (hits) hits &= hits - 1;
          uint64_t wL = __shfl_sync(kFull, w, __ffs(hm) - 1);
          uint32_t pre[4];
          auto load4 = [&](uint64_t ww, uint32_t (&r)[4]) {
            const uint64_t sb = ww >> 32, len = ww & 0xffffffffull;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t i = static_cast<uint64_t>(lane) + 32u * k;
              r[k] = i < len ? p.wmem[sb + i] : kBlank;
            }
          };
          load4(wL, pre);
          while (hm) {
            hm &= hm - 1;
            uint32_t cur[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) cur[k] = pre[k];
            const uint64_t wC = wL;
            if (hm) {  // next set's members in flight during this set's decrements
              wL = __shfl_sync(kFull, w, __ffs(hm) - 1);
              load4(wL, pre);
            }
            const uint64_t sb = wC >> 32, se = sb + (wC & 0xffffffffull);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t t = sb + lane + 32u * k;
              if (t < se) {
                atomicSub(p.cnt + cur[k], 1u);
                p.dirty[cur[k] >> kSelTileLog] = 1u;
                p.wmem[t] = kBlank;
              }
            }
            for (uint64_t t = sb + lane + 128; t < se; t += 32) {  // sets past 128 members
              const uint32_t u = p.wmem[t];
              atomicSub(p.cnt + u, 1u);
              p.dirty[u >> kSelTileLog] = 1u;
              p.wmem[t] = kBlank;
            }
          }
        }
      }
    } else {
      const uint64_t ib = p.ioff[v], ie = p.ioff[v + 1];
      for (uint64_t t = ib + gwarp; t < ie; t += nwarps) {
        const uint32_t s = p.inv[t];
        uint32_t was = 0;
        if (lane == 0) was = atomicExch(p.covered + s, 1u);
        was = __shfl_sync(kFull, was, 0);
        if (was) continue;
        killed += lane == 0;
        warp_cover(p, s);
      }
    }
    // dense rows holding v: a bit test each; the round's kills are listed
    for (uint64_t d = tid; d < p.nd; d += nthreads) {
      if (p.dcov[d]) continue;
      if (!((p.dbits[d * p.dwords + (v >> 5)] >> (v & 31)) & 1u)) continue;
      p.dcov[d] = 1u;
      ++killed;
      p.dkill[atomicAdd(p.dkn + r, 1u)] = static_cast<uint32_t>(d);
    }
    for (int o = 16; o; o >>= 1) killed += __shfl_xor_sync(kFull, killed, o);
    if (lane == 0 && killed) atomicAdd(p.marg + r, killed);
    if (tid == 0) {
      p.keys[r] = key;
      p.seeds[r] = v;
      p.selected[v] = 1;
      if (rebuild) atomicAdd(p.rebuilds, 1ull);
    }
    grid.sync();
    covered_sum += p.marg[r];

    // ---- C0: the counts of the dense rows / the rebuild ----------------------
    if (rebuild) {
      for (uint64_t u = tid; u < p.n; u += nthreads) p.cnt[u] = 0u;
      grid.sync();
      sel_colsum(p, nullptr, p.nd, +1, tid, nthreads);  // live rows
      if (kScan) {  // live list sets: the non-blanked entries of the working copy
        for (uint64_t t = tid; t < p.total; t += nthreads) {
          const uint32_t u = p.wmem[t];
          if (u != kBlank) atomicAdd(p.cnt + u, 1u);
        }
      } else {
        for (uint64_t s = gwarp; s < p.nsets; s += nwarps) {
          if (p.covered[s]) continue;
          for (uint64_t t = p.off[s] + lane; t < p.off[s + 1]; t += 32) atomicAdd(p.cnt + p.mem[t], 1u);
        }
      }
      grid.sync();
    } else {
      const uint32_t ndk = p.dkn[r];
      if (ndk) {
        sel_colsum(p, p.dkill, ndk, -1, tid, nthreads);
        grid.sync();
      }
    }

    // ---- C: re-reduce the tiles whose counts changed -------------------------
    if (p.snap) {
      uint32_t* out = p.snap + static_cast<uint64_t>(r) * p.n;
      for (uint64_t u = tid; u < p.n; u += nthreads) out[u] = p.cnt[u];
    }
    for (uint64_t t = gwarp; t < ntiles; t += nwarps) {
      if (!rebuild && ntiles > kAllTilesMax && !p.dirty[t]) continue;  // uniform in the warp
      const unsigned long long m = tile_max_warp(p, static_cast<uint32_t>(t));
      if (lane == 0) {
        p.tmax[t] = m;
        p.dirty[t] = 0u;
      }
    }
    grid.sync();
  }
  if (tid == 0) p.status[0] = p.k;
}

// ---------------------------------------------------------------------------
// Cluster-resident variant (stores scanned per round, no dense rows, no counter
// snapshots): ONE cluster of kClCtas blocks runs all k rounds. Every block keeps
// a full replica of the tile maxima in shared memory, so the argmax of a round
// is a block-local reduction (no global round trip, same key in every block).
// The scan-mode cover is the grid kernel's; a decremented vertex flags its tile
// in the OWNER block's shared bitmap (tile t belongs to block t % kClCtas,
// a distributed-shared-memory atomic), and after the cluster barrier each block
// re-reduces its flagged tiles and writes the new maxima into all kClCtas
// replicas (DSMEM stores) before the second barrier. Two cluster barriers
// (~0.2 us each) per round instead of two grid barriers across 148 SMs.
// ---------------------------------------------------------------------------
constexpr int kClBlock = 1024;
constexpr int kClCtas = 16;

__device__ __forceinline__ unsigned long long cl_block_max(unsigned long long x,
                                                           unsigned long long* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) x = umax64(x, __shfl_xor_sync(kFull, x, o));
  __syncthreads();
  if (lane == 0) red[wid] = x;
  __syncthreads();
  x = lane < kClBlock / 32 ? red[lane] : 0ull;
  for (int o = 16; o; o >>= 1) x = umax64(x, __shfl_xor_sync(kFull, x, o));
  return x;
}

__global__ void __launch_bounds__(kClBlock, 1) k_select_cluster(const SelectParams p) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned crank = cl.block_rank();
  const uint32_t ntiles = (p.n + kSelTile - 1) >> kSelTileLog;
  extern __shared__ unsigned long long cl_smem[];
  unsigned long long* tmax = cl_smem;                                      // [ntiles]
  unsigned long long* red = tmax + ntiles;                                 // [32]
  // block b owns the contiguous tiles [b tpc, (b + 1) tpc): its dirty bitmap is
  // indexed by the tile's offset in that range; `touch` collects, per block, the
  // tiles its own decrements hit (local shared atomics), sent to the owners
  // one word at a time after the cover
  const uint32_t tpc = (ntiles + kClCtas - 1) / kClCtas;
  uint32_t* dirty = reinterpret_cast<uint32_t*>(red + kClBlock / 32);      // [tpc/32 + 1]
  const uint32_t dwords_t = (tpc >> 5) + 1;
  uint32_t* touch = dirty + dwords_t;                                      // [ntiles/32 + 1]
  const uint32_t twords = (ntiles >> 5) + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t tid = static_cast<uint64_t>(crank) * kClBlock + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(kClCtas) * kClBlock;
  const uint64_t gwarp = tid >> 5, nwarps = nthreads >> 5;
  for (uint32_t i = threadIdx.x; i < dwords_t; i += kClBlock) dirty[i] = 0u;
  for (uint32_t i = threadIdx.x; i < twords; i += kClBlock) touch[i] = 0u;
  // initial maxima: warp per tile across the cluster, broadcast to every replica
  for (uint64_t t = gwarp; t < ntiles; t += nwarps) {
    const unsigned long long m = tile_max_warp(p, static_cast<uint32_t>(t));
    if (lane < kClCtas) cl.map_shared_rank(tmax, lane)[t] = m;
  }
  cl.sync();

  auto flag_tile = [&](uint32_t u) {
    const uint32_t t = u >> kSelTileLog;
    atomicOr(touch + (t >> 5), 1u << (t & 31));
  };

  unsigned long long covered_sum = 0;
  for (uint32_t r = 0; r < p.k; ++r) {
    // ---- A: argmax over the local replica --------------------------------------
    unsigned long long best = 0;
    for (uint32_t t = threadIdx.x; t < ntiles; t += kClBlock) best = umax64(best, tmax[t]);
    const unsigned long long key = cl_block_max(best, red);
    const uint32_t top = static_cast<uint32_t>(key >> 32);
    const uint32_t v = 0xffffffffu - static_cast<uint32_t>(key);
    if (top == 0) {
      if (tid == 0) {  // exhaustion (selection.hpp:61-72)
        uint32_t filled = r;
        for (uint32_t u = 0; u < p.n && filled < p.k; ++u) {
          if (!p.selected[u]) {
            p.selected[u] = 1;
            p.seeds[filled] = u;
            p.marg[filled] = 0;
            ++filled;
          }
        }
        p.status[0] = r;
      }
      cl.sync();  // no block leaves while others may still write its shared memory
      return;
    }
    if (p.need && covered_sum + static_cast<unsigned long long>(p.k - r) * top < p.need) {
      if (tid == 0) p.status[0] = r | kSelAborted;  // the coverage cannot reach `need`
      cl.sync();
      return;
    }
    const unsigned long long live = p.nsets - covered_sum;
    const bool rebuild = live > 0 && static_cast<double>(top) / static_cast<double>(live) >
                                         p.adaptive_threshold;

    // ---- B: cover (scan mode as in k_select; index mode: warp per set of inv[v]) --
    unsigned long long killed = 0;
    if (!p.scan) {
      const uint64_t ib = p.ioff[v], ie = p.ioff[v + 1];
      for (uint64_t t = ib + gwarp; t < ie; t += nwarps) {
        const uint32_t sid = p.inv[t];
        uint32_t was = 0;
        if (lane == 0) was = atomicExch(p.covered + sid, 1u);
        was = __shfl_sync(kFull, was, 0);
        if (was) continue;
        killed += lane == 0;
        if (rebuild) continue;
        for (uint64_t j = p.off[sid] + lane; j < p.off[sid + 1]; j += 32) {
          const uint32_t u = p.mem[j];
          atomicSub(p.cnt + u, 1u);
          flag_tile(u);
        }
      }
    }
    const uint64_t nchunk = p.scan ? (p.total + 255) / 256 : 0;
    for (uint64_t c = gwarp; c < nchunk; c += nwarps) {
      const uint64_t base = c * 256 + static_cast<uint64_t>(lane) * 8;
      uint32_t q[8];
      if (base + 8 <= p.total) {
        const uint4 a = *reinterpret_cast<const uint4*>(p.wmem + base);
        const uint4 b = *reinterpret_cast<const uint4*>(p.wmem + base + 4);
        q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
        q[4] = b.x; q[5] = b.y; q[6] = b.z; q[7] = b.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = base + j < p.total ? p.wmem[base + j] : kBlank;
      }
      uint32_t hits = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) hits |= (q[j] == v ? 1u : 0u) << j;
      killed += __popc(hits);
      while (__any_sync(kFull, hits != 0)) {
        const uint64_t w = hits ? p.span[base + (__ffs(hits) - 1)] : 0ull;
        unsigned hm = __ballot_sync(kFull, hits != 0);
        if (hits) hits &= hits - 1;
        while (hm) {
          const int L = __ffs(hm) - 1;
          hm &= hm - 1;
          const uint64_t wL = __shfl_sync(kFull, w, L);
          const uint64_t sb = wL >> 32, se = sb + (wL & 0xffffffffull);
          for (uint64_t t = sb + lane; t < se; t += 32) {
            const uint32_t u = p.wmem[t];
            if (!rebuild) {
              atomicSub(p.cnt + u, 1u);
              flag_tile(u);
            }
            p.wmem[t] = kBlank;
          }
        }
      }
    }
    for (int o = 16; o; o >>= 1) killed += __shfl_xor_sync(kFull, killed, o);
    if (lane == 0 && killed) atomicAdd(p.marg + r, killed);
    if (tid == 0) {
      p.keys[r] = key;
      p.seeds[r] = v;
      p.selected[v] = 1;
      if (rebuild) atomicAdd(p.rebuilds, 1ull);
    }
    __syncthreads();
    // this block's touched tiles -> their owners' dirty bitmaps (DSMEM): thread
    // per tile, one remote atomic per touched tile
    for (uint32_t t = threadIdx.x; t < ntiles; t += kClBlock) {
      if (!((touch[t >> 5] >> (t & 31)) & 1u)) continue;
      const uint32_t owner = t / tpc, jo = t - owner * tpc;
      atomicOr(cl.map_shared_rank(dirty, owner) + (jo >> 5), 1u << (jo & 31));
    }
    __syncthreads();
    for (uint32_t i2 = threadIdx.x; i2 < twords; i2 += kClBlock) touch[i2] = 0u;
    cl.sync();
    covered_sum += p.marg[r];

    if (rebuild) {  // rebuild_update: zero, recount the surviving sets
      for (uint64_t u = tid; u < p.n; u += nthreads) p.cnt[u] = 0u;
      cl.sync();
      if (p.scan) {
        for (uint64_t t = tid; t < p.total; t += nthreads) {
          const uint32_t u = p.wmem[t];
          if (u != kBlank) atomicAdd(p.cnt + u, 1u);
        }
      } else {
        for (uint64_t sid = gwarp; sid < p.nsets; sid += nwarps) {
          if (p.covered[sid]) continue;
          for (uint64_t j = p.off[sid] + lane; j < p.off[sid + 1]; j += 32)
            atomicAdd(p.cnt + p.mem[j], 1u);
        }
      }
      cl.sync();
    }

    // ---- C: re-reduce this block's flagged tiles, broadcast the maxima ---------
    const uint32_t t0 = crank * tpc;
    const uint32_t owned = ntiles > t0 ? min(tpc, ntiles - t0) : 0;
    for (uint32_t j = wid; j < owned; j += kClBlock / 32) {
      const bool d = rebuild || ((dirty[j >> 5] >> (j & 31)) & 1u);
      if (!d) continue;  // uniform in the warp
      const uint32_t t = t0 + j;
      const unsigned long long m = tile_max_warp(p, t);
      if (lane < kClCtas) cl.map_shared_rank(tmax, lane)[t] = m;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < dwords_t; i += kClBlock) dirty[i] = 0u;
    cl.sync();
  }
  if (tid == 0) p.status[0] = p.k;
}

}  // namespace

// The cluster-resident selection when the store qualifies (scan mode, no dense
// rows, no per-round snapshots, tile maxima within shared memory) and the
// device can place a 16-block cluster; false otherwise (caller uses the grid).
// Measured (profiles/r2/sel_r2n.log, k = 50 over 8,192 sets): cfg2 (238K members)
// 0.42 vs 0.57 ms, cfg1 (114K) 0.39 vs 0.50, cfg3 (75K) 0.65 vs 0.75; cfg4
// (667K members, 2,367 tiles) 0.92 vs 0.65 -- 16 SMs re-scan a large store
// slower than 148; cfg4's first IMM selection (6,331 sets, ~500K members) 0.80
// vs ~0.50 ms -- the two cost lines cross near 390K members, so the cluster
// takes stores of up to 3 x 2^17 members.
constexpr uint64_t kClMaxMembers = 3ull << 17;

bool select_cluster_eligible(const SelectParams& p) {
  if (p.nd || p.snap) return false;
  if (const char* e = std::getenv("RRGPU_SELECT_CLUSTER"))  // tests / tuning: 0 off
    if (*e == '0') return false;
  return true;
}

bool launch_select_cluster(const SelectParams& p, cudaStream_t s) {
  if (!select_cluster_eligible(p)) return false;
  bool force = false;
  if (const char* e = std::getenv("RRGPU_SELECT_CLUSTER")) force = *e == '1';
  // scan mode re-reads the whole store every round: 16 SMs only for small stores;
  // index mode touches only the seed's sets (capi picks it for larger stores)
  if (p.scan && !force && p.total > kClMaxMembers) return false;
  const uint32_t ntiles = (p.n + kSelTile - 1) >> kSelTileLog;
  const uint32_t tpc = (ntiles + kClCtas - 1) / kClCtas;
  const size_t smem = static_cast<size_t>(ntiles) * 8 + (kClBlock / 32) * 8 +
                      ((tpc >> 5) + 1) * 4 + ((ntiles >> 5) + 1) * 4;
  if (smem > 200 * 1024) return false;
  static int ok = -1;
  if (ok < 0) {
    ok = cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                 cudaSuccess &&
         cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              200 * 1024) == cudaSuccess;
    cudaGetLastError();
  }
  if (!ok) return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClCtas);
  cfg.blockDim = dim3(kClBlock);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClCtas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, k_select_cluster, &cfg) != cudaSuccess ||
      clusters < 1) {
    cudaGetLastError();
    return false;
  }
  RRG_CUDA(cudaLaunchKernelEx(&cfg, k_select_cluster, p));
  count_launch();
  return true;
}

void launch_select(const SelectParams& p, int num_sms, cudaStream_t s) {
  if (launch_select_cluster(p, s)) return;
  const void* fn = p.scan ? reinterpret_cast<const void*>(k_select<true>)
                          : reinterpret_cast<const void*>(k_select<false>);
  int per_sm = 0;
  RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSelBlock, 0));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 2) per_sm = 2;
  if (const char* e = std::getenv("RRGPU_SELECT_BLOCKS_PER_SM")) {  // tuning
    const int v = std::atoi(e);
    if (v >= 1 && v <= per_sm) per_sm = v;
  }
  int grid = num_sms * per_sm;
  SelectParams args = p;
  void* kargs[] = {&args};
  RRG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSelBlock), kargs, 0, s));
  count_launch();
}

}  // namespace rrgpu
