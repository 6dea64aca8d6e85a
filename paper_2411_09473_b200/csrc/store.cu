// store.cu -- K3 stream compaction into the slot-ordered flat RRR buffer, the
// hand-written exclusive scan it uses, K4 standalone recount, K5 inverted index.
//
// Replaces RRRStore::place / finalize (rrr_store.hpp:41-60), build_counter
// (selection.hpp:79-95) and the membership probes of decrement_update
// (selection.hpp:137-149), which become a vertex -> set-id index.
#include <algorithm>

#include "internal.hpp"

namespace rrgpu {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr uint64_t kTile = static_cast<uint64_t>(kScanThreads) * kScanItems;

// Block-wide exclusive scan of one value per thread; returns the block total.
__device__ __forceinline__ uint64_t block_exclusive(uint64_t v, uint64_t& excl) {
  __shared__ uint64_t warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint64_t t = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  const uint64_t warp_base = wid ? warp_tot[wid - 1] : 0;
  const uint64_t total = warp_tot[kScanThreads / 32 - 1];
  excl = warp_base + incl - v;
  __syncthreads();
  return total;
}

// Tile-local exclusive scan; tile totals to `sums`.
template <typename TIn>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_tiles(const TIn* in, uint64_t* out, uint64_t count, uint64_t* sums) {
  const uint64_t base = blockIdx.x * kTile + static_cast<uint64_t>(threadIdx.x) * kScanItems;
  uint64_t vals[kScanItems];
  uint64_t local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i;
    vals[i] = idx < count ? static_cast<uint64_t>(in[idx]) : 0;
    local += vals[i];
  }
  uint64_t excl;
  const uint64_t total = block_exclusive(local, excl);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i;
    if (idx < count) out[idx] = excl;
    excl += vals[i];
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void k_scan_add(uint64_t* out, uint64_t count, const uint64_t* tile_prefix) {
  const uint64_t idx = blockIdx.x * kTile + threadIdx.x;
  const uint64_t add = tile_prefix[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t t = idx + static_cast<uint64_t>(i) * kScanThreads;
    if (t < count) out[t] += add;
  }
}

__global__ void k_set_total(uint64_t* out, uint64_t count, const uint64_t* sums_scan,
                            const uint64_t* sums, uint64_t ntiles) {
  out[count] = sums_scan[ntiles - 1] + sums[ntiles - 1];
}

// exclusive scan of u64 values (tile sums) -- recursion helper
void scan_u64_rec(const uint64_t* in, uint64_t* out, uint64_t count, DevBuf<uint64_t>& tmp,
                  uint64_t tmp_off, cudaStream_t s);

template <typename TIn>
void scan_impl(const TIn* in, uint64_t* out, uint64_t count, DevBuf<uint64_t>& tmp,
               uint64_t tmp_off, cudaStream_t s) {
  const uint64_t ntiles = (count + kTile - 1) / kTile;
  uint64_t* sums = tmp.ptr + tmp_off;
  uint64_t* sums_scan = sums + ntiles;
  k_scan_tiles<TIn><<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(in, out, count, sums);
  RRG_CUDA(cudaGetLastError());
  count_launch();
  if (ntiles > 1) {
    scan_u64_rec(sums, sums_scan, ntiles, tmp, tmp_off + 2 * ntiles + 1, s);
    k_scan_add<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(out, count, sums_scan);
    RRG_CUDA(cudaGetLastError());
    count_launch();
  } else {
    RRG_CUDA(cudaMemsetAsync(sums_scan, 0, sizeof(uint64_t), s));
  }
  k_set_total<<<1, 1, 0, s>>>(out, count, sums_scan, sums, ntiles);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void scan_u64_rec(const uint64_t* in, uint64_t* out, uint64_t count, DevBuf<uint64_t>& tmp,
                  uint64_t tmp_off, cudaStream_t s) {
  scan_impl<uint64_t>(in, out, count, tmp, tmp_off, s);
}

uint64_t scan_tmp_words(uint64_t count) {
  uint64_t words = 0;
  while (true) {
    const uint64_t ntiles = (count + kTile - 1) / kTile;
    words += 2 * ntiles + 2;
    if (ntiles <= 1) break;
    count = ntiles;
  }
  return words;
}

// K3: warp per set, copies staging -> slot-ordered buffer, writes offsets.
__global__ void k_compact(const uint32_t* stage, const uint64_t* slot_start,
                          const uint32_t* slot_len, const uint64_t* scan, uint64_t base_total,
                          uint64_t count, uint32_t* mem_out, uint64_t* off_out,
                          uint32_t* maxlen) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  uint32_t mx = 0;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < count;
       i += warps) {
    const uint32_t len = slot_len[i];
    const uint32_t* from = stage + slot_start[i];
    const uint64_t dst = base_total + scan[i];
    for (uint32_t t = lane; t < len; t += 32) mem_out[dst + t] = from[t];
    RRG_DCHECK(len < (1u << 31), 12);
    if (lane == 0) off_out[i + 1] = dst + len;
    mx = max(mx, len);
  }
  if (lane == 0 && mx) atomicMax(maxlen, mx);
}

// K3 for large batches: block per run of kCompactSets consecutive slots. Their
// outputs are one contiguous range of the store, so threads stride over OUTPUT
// positions (coalesced stores, four gathers in flight each) and find their slot
// by a binary search over the run's prefix in shared memory. The warp-per-set
// kernel above waits one round trip per set (~80 members); this one streams.
constexpr uint32_t kCompactSets = 128;
__global__ void __launch_bounds__(256) k_compact_runs(const uint32_t* stage, const uint64_t* slot_start,
                                                      const uint32_t* slot_len, const uint64_t* scan,
                                                      uint64_t base_total, uint64_t count,
                                                      uint32_t* mem_out, uint64_t* off_out,
                                                      uint32_t* maxlen) {
  __shared__ uint64_t s_pre[kCompactSets + 1];
  __shared__ uint64_t s_src[kCompactSets];
  const uint64_t s0 = static_cast<uint64_t>(blockIdx.x) * kCompactSets;
  const uint32_t ns = static_cast<uint32_t>(count - s0 < kCompactSets ? count - s0 : kCompactSets);
  uint32_t mx = 0;
  for (uint32_t i = threadIdx.x; i <= ns; i += blockDim.x) {
    s_pre[i] = scan[s0 + i];
    if (i < ns) {
      s_src[i] = slot_start[s0 + i];
      const uint32_t len = slot_len[s0 + i];
      off_out[s0 + i + 1] = base_total + scan[s0 + i] + len;
      mx = max(mx, len);
    }
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxlen, mx);
  __syncthreads();
  const uint64_t lo = s_pre[0], hi = s_pre[ns];
  for (uint64_t o0 = lo + threadIdx.x; o0 < hi; o0 += 4ull * blockDim.x) {
    uint32_t v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t o = o0 + static_cast<uint64_t>(q) * blockDim.x;
      v[q] = 0;
      if (o < hi) {
        uint32_t k = 0;  // last slot with s_pre[k] <= o
        for (uint32_t step = kCompactSets / 2; step; step >>= 1)
          if (k + step < ns && s_pre[k + step] <= o) k += step;
        v[q] = __ldg(stage + s_src[k] + (o - s_pre[k]));
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t o = o0 + static_cast<uint64_t>(q) * blockDim.x;
      if (o < hi) mem_out[base_total + o] = v[q];
    }
  }
}

// K4: occurrence histogram over stored sets (build_counter, selection.hpp:79-95).
__global__ void k_recount(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                          uint32_t* counter) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  for (uint64_t s = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < nsets;
       s += warps) {
    for (uint64_t t = off[s] + lane; t < off[s + 1]; t += 32) atomicAdd(counter + mem[t], 1u);
  }
}

// Scan-mode selection inputs: a working copy of the members (covered sets get
// blanked in it) and, per member, its set's span (start << 32 | length), so a
// member matching the round's seed names the whole set in one load.
__global__ void k_set_spans(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                            uint64_t* span, uint32_t* wmem) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  for (uint64_t s = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < nsets;
       s += warps) {
    const uint64_t b = off[s], e = off[s + 1];
    const uint64_t w = (b << 32) | (e - b);
    for (uint64_t t = b + lane; t < e; t += 32) {
      span[t] = w;
      wmem[t] = mem[t];
    }
  }
}

// K5: vertex -> ids of the sets containing it. icur starts at ioff[v].
__global__ void k_invert(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                         unsigned long long* icur, const uint64_t* ioff, uint32_t* inv,
                         uint32_t* status) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  for (uint64_t s = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < nsets;
       s += warps) {
    for (uint64_t t = off[s] + lane; t < off[s + 1]; t += 32) {
      const uint32_t v = mem[t];
      const unsigned long long pos = atomicAdd(icur + v, 1ull);
      if (pos < ioff[v + 1]) inv[pos] = static_cast<uint32_t>(s);
      else status[1] = 1;  // prebuilt counter disagrees with the stored sets
    }
  }
}

// fraction_covered helper: sets with a member flagged in `in_seed_set`.
__global__ void k_fraction(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                           const uint8_t* flag, unsigned long long* hits) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  unsigned long long local = 0;
  for (uint64_t s = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; s < nsets;
       s += warps) {
    bool hit = false;
    for (uint64_t t = off[s] + lane; t < off[s + 1] && !hit; t += 32) hit = flag[mem[t]] != 0;
    if (__any_sync(kFull, hit) && lane == 0) ++local;
  }
  if (lane == 0 && local) atomicAdd(hits, local);
}

// Offsets of sets copied from another store: out[i] = in[i] - in[0] + base for
// i in [1, count]; also the longest copied set.
__global__ void k_rebase(const uint64_t* in, uint64_t count, uint64_t base, uint64_t* out,
                         uint32_t* maxlen) {
  uint32_t mx = 0;
  const uint64_t zero = in[0];
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i <= count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    out[i] = in[i] - zero + base;
    mx = max(mx, static_cast<uint32_t>(in[i] - in[i - 1]));
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxlen, mx);
}

__global__ void k_widen(const uint32_t* in, uint64_t* out, uint64_t n) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__global__ void k_narrow(const uint64_t* in, uint32_t* out, uint64_t n) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(in[i]);
}

int grid_for(uint64_t warps_needed) {
  const uint64_t blocks = (warps_needed * 32 + 255) / 256;
  return static_cast<int>(blocks < 1 ? 1 : (blocks > 65535 ? 65535 : blocks));
}

}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint64_t* out, uint64_t count, DevBuf<uint64_t>& tmp,
                        cudaStream_t s) {
  if (count == 0) {
    RRG_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
    return;
  }
  tmp.reserve_discard(scan_tmp_words(count));
  scan_impl<uint32_t>(in, out, count, tmp, 0, s);
}

void launch_compact(const uint32_t* stage, const uint64_t* slot_start, const uint32_t* slot_len,
                    const uint64_t* scan, uint64_t base_total, uint64_t count, uint32_t* mem_out,
                    uint64_t* off_out, uint32_t* maxlen, cudaStream_t s) {
  if (!count) return;
  if (count >= 4096) {
    const uint64_t blocks = (count + kCompactSets - 1) / kCompactSets;
    k_compact_runs<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        stage, slot_start, slot_len, scan, base_total, count, mem_out, off_out, maxlen);
  } else {
    k_compact<<<grid_for(count), 256, 0, s>>>(stage, slot_start, slot_len, scan, base_total, count,
                                              mem_out, off_out, maxlen);
  }
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_recount(const uint64_t* off, const uint32_t* mem, uint64_t nsets, uint32_t* counter,
                    cudaStream_t s) {
  if (!nsets) return;
  k_recount<<<grid_for(nsets), 256, 0, s>>>(off, mem, nsets, counter);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_set_spans(const uint64_t* off, const uint32_t* mem, uint64_t nsets, uint64_t* span,
                      uint32_t* wmem, cudaStream_t s) {
  if (!nsets) return;
  k_set_spans<<<grid_for(nsets), 256, 0, s>>>(off, mem, nsets, span, wmem);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_invert(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                   unsigned long long* icur, const uint64_t* ioff, uint32_t* inv,
                   uint32_t* status, cudaStream_t s) {
  if (!nsets) return;
  k_invert<<<grid_for(nsets), 256, 0, s>>>(off, mem, nsets, icur, ioff, inv, status);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_rebase(const uint64_t* in, uint64_t count, uint64_t base, uint64_t* out,
                   uint32_t* maxlen, cudaStream_t s) {
  if (!count) return;
  const uint64_t blocks = std::min<uint64_t>((count + 255) / 256, 4096);
  k_rebase<<<static_cast<unsigned>(blocks), 256, 0, s>>>(in, count, base, out, maxlen);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_narrow(const uint64_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  k_narrow<<<1184, 256, 0, s>>>(in, out, n);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_widen(const uint32_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  k_widen<<<1184, 256, 0, s>>>(in, out, n);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_fraction(const uint64_t* off, const uint32_t* mem, uint64_t nsets,
                     const uint8_t* in_seed_set, unsigned long long* hits, cudaStream_t s) {
  if (!nsets) return;
  k_fraction<<<grid_for(nsets), 256, 0, s>>>(off, mem, nsets, in_seed_set, hits);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace rrgpu
