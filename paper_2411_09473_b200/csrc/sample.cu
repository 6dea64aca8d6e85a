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
//
// This file: the big-set path (both models), the upload checks and the sampler
// dispatch; the IC samplers live in sample_ic.cu, the LT samplers in
// sample_lt.cu, their shared device building blocks in sampler.cuh.
#include "sampler.cuh"

namespace rrgpu {

namespace {

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
    if (nmem >= p.dense_thr) {
      // dense arm (pack_sketch, sampling.hpp:78-83): the visited map IS the
      // set's n-bit map -- copied into a row of the pool and cleared in the same
      // pass; the members only feed the fused counter
      unsigned long long row = 0;
      if (lane == 0) row = atomicAdd(&p.ctl->ndense, 1ull);
      row = __shfl_sync(kFull, row, 0);
      __syncwarp();
      if (row < p.drow_avail) {
        const uint64_t grow = p.drow_base + row;
        uint32_t* dst = p.dbits + grow * p.dwords;
        for (uint32_t wd = lane; wd < p.dwords; wd += 32) {
          uint32_t x = 0;
          if (wd < words) {
            x = vis[wd];
            vis[wd] = 0u;
          }
          dst[wd] = x;
        }
        if (p.counter)
          for (uint32_t i = lane; i < nmem; i += 32) atomicAdd(p.counter + mem[i], 1u);
        if (lane == 0) {
          p.dlen[grow] = nmem;
          p.droot[grow] = root;
          p.dslot[grow] = static_cast<uint32_t>(p.set_base + idx);
          p.bdix[idx] = static_cast<uint32_t>(grow);
          p.slot_start[idx] = 0;
          p.slot_len[idx] = 0;  // empty list range
          atomicAdd(&p.ctl->dense_members, (unsigned long long)nmem);
          atomicMax(&p.ctl->dense_max, nmem);
          insp += sinsp;
        }
      } else {
        if (lane == 0) restage_slot(p, idx, 0);  // the row pool grows, then a re-run
        for (uint32_t i = lane; i < nmem; i += 32) {
          const uint32_t v = mem[i];
          atomicAnd(vis + (v >> 5), ~(1u << (v & 31)));
        }
      }
      __syncwarp();
      continue;
    }
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&p.ctl->cursor, (unsigned long long)nmem);
    pos = __shfl_sync(kFull, pos, 0);
    __syncwarp();
    if (pos + nmem > p.stage_cap) {
      if (lane == 0) restage_slot(p, idx, nmem);
    } else {
      for (uint32_t i = lane; i < nmem; i += 32) {
        const uint32_t v = mem[i];
        RRG_DCHECK(v < p.n && nmem <= p.n, 8);
        p.stage[pos + i] = v;
        if (p.counter) atomicAdd(p.counter + v, 1u);
      }
      if (lane == 0) {
        p.slot_start[idx] = pos;
        p.slot_len[idx] = nmem;
        note_len(p, nmem);
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
__global__ void k_check_sources(const uint32_t* src, uint64_t m, uint32_t n, uint32_t* bad) {
  bool ok = true;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    ok &= src[j] < n;
  if (!__all_sync(kFull, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 2u);
}

}  // namespace

// which: 1 = offsets (u64 -> u32 + monotonicity / range), 2 = sources < n.
// Enqueues the checks on the graph's stream; `bad` receives the flag word.
void upload_checks_async(rrg_graph* g, const uint64_t* d_off64, uint32_t which,
                         DevBuf<uint32_t>& bad) {
  bad.reserve_discard(1);
  RRG_CUDA(cudaMemsetAsync(bad.ptr, 0, 4, g->stream));
  const int grid = g->num_sms * 8;
  if (which & 1u) {
    k_offsets_u32<<<grid, 256, 0, g->stream>>>(d_off64, g->off.ptr, g->n, g->m, bad.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  }
  if ((which & 2u) && g->m) {
    k_check_sources<<<grid, 256, 0, g->stream>>>(g->src.ptr, g->m, g->n, bad.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  }
}

uint32_t upload_checks(rrg_graph* g, const uint64_t* d_off64, uint32_t which) {
  DevBuf<uint32_t> bad;
  upload_checks_async(g, d_off64, which, bad);
  uint32_t h = 0;
  RRG_CUDA(cudaMemcpyAsync(&h, bad.ptr, 4, cudaMemcpyDeviceToHost, g->stream));
  host_sync((g->stream));
  return h;
}

int sampler_block() { return kBlock; }

int sampler_blocks_per_sm(int model, uint32_t, int lt_mode) {
  const int b = model == RRG_IC ? ic_blocks_per_sm() : lt_blocks_per_sm(lt_mode);
  return b < 1 ? 1 : b;
}

void launch_sampler(int model, const SampleParams& p, int grid, uint32_t ic_inner, int schedule,
                    cudaStream_t s) {
  if (model == RRG_IC) launch_ic_sampler(p, grid, ic_inner, schedule, s);
  else launch_lt_sampler(p, grid, s);
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

}  // namespace rrgpu
