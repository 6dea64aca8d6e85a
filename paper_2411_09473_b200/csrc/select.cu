// select.cu -- K6: the k-round greedy max-coverage loop, resident on the GPU.
//
// Replaces select_seeds (selection.hpp:209-243) with parallel_argmax (:100-125),
// decrement_update (:130-156) and fill_remaining_seeds (:61-72). One cooperative
// persistent launch runs every round; grid-wide barriers separate
//   A) argmax: block max over packed keys (count << 32 | ~v) -> one 64-bit
//      atomicMax per block. Max count wins; ties go to the lowest id, exactly
//      the reference's rule (:113, :119-120).
//   B) cover: every set in inv[v] (inverted index, store.cu) is claimed once
//      with atomicExch on its covered flag; the winner counts it in the round's
//      marginal and decrements each member's count (Counter::sub, counter.hpp:28).
// The host sees nothing until all k rounds are done.
#include <cooperative_groups.h>

#include "internal.hpp"

namespace cg = cooperative_groups;

namespace rrgpu {

namespace {

constexpr int kSelBlock = 512;

__device__ __forceinline__ unsigned long long pack_key(uint32_t count, uint32_t v) {
  return (static_cast<unsigned long long>(count) << 32) | (0xffffffffu - v);
}

__global__ void __launch_bounds__(kSelBlock) k_select(const SelectParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long warp_best[kSelBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t gwarp = tid >> 5;
  const uint64_t nwarps = nthreads >> 5;

  for (uint32_t r = 0; r < p.k; ++r) {
    // ---- A: argmax over counts ------------------------------------------
    unsigned long long best = 0;
    for (uint64_t v = tid; v < p.n; v += nthreads) {
      const unsigned long long key = pack_key(p.cnt[v], static_cast<uint32_t>(v));
      best = key > best ? key : best;
    }
    for (int o = 16; o; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(kFull, best, o);
      best = y > best ? y : best;
    }
    if (lane == 0) warp_best[wid] = best;
    __syncthreads();
    if (wid == 0) {
      best = lane < kSelBlock / 32 ? warp_best[lane] : 0;
      for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(kFull, best, o);
        best = y > best ? y : best;
      }
      if (lane == 0) atomicMax(p.keys + r, best);
    }
    grid.sync();

    const unsigned long long key = p.keys[r];
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
      return;  // uniform: every block read the same key
    }

    // ---- B: cover the sets holding v --------------------------------------
    const uint64_t ib = p.ioff[v], ie = p.ioff[v + 1];
    unsigned long long killed = 0;
    for (uint64_t t = ib + gwarp; t < ie; t += nwarps) {
      const uint32_t s = p.inv[t];
      uint32_t was = 0;
      if (lane == 0) was = atomicExch(p.covered + s, 1u);
      was = __shfl_sync(kFull, was, 0);
      if (was) continue;
      killed += lane == 0;
      for (uint64_t j = p.off[s] + lane; j < p.off[s + 1]; j += 32) atomicSub(p.cnt + p.mem[j], 1u);
    }
    if (lane == 0 && killed) atomicAdd(p.marg + r, killed);
    if (tid == 0) {
      p.seeds[r] = v;
      p.selected[v] = 1;
    }
    grid.sync();
    if (p.snap) {
      uint32_t* out = p.snap + static_cast<uint64_t>(r) * p.n;
      for (uint64_t u = tid; u < p.n; u += nthreads) out[u] = p.cnt[u];
    }
  }
  if (tid == 0) p.status[0] = p.k;
}

}  // namespace

void launch_select(const SelectParams& p, int num_sms, cudaStream_t s) {
  int per_sm = 0;
  RRG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select, kSelBlock, 0));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 2) per_sm = 2;
  int grid = num_sms * per_sm;
  const uint64_t want = (static_cast<uint64_t>(p.n) + kSelBlock - 1) / kSelBlock;
  if (want < static_cast<uint64_t>(grid)) grid = static_cast<int>(want < 1 ? 1 : want);
  SelectParams args = p;
  void* kargs[] = {&args};
  RRG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_select), dim3(grid),
                                       dim3(kSelBlock), kargs, 0, s));
  count_launch();
}

}  // namespace rrgpu
