// graph_dev.cu -- on-device graph preparation.
//
// A caller holding an edge list uploads it once and the device builds what
// rrg_graph_create takes, instead of the host-side detail::build_graph
// (graph.hpp:69-115) and normalize_lt_weights (graph.hpp:207-235):
//   * transpose: the reference's in-list of v holds v's in-edges ordered by
//     source id, parallel edges in input order (a stable counting sort by
//     source, then one by target). That is a STABLE sort of the edges by the
//     64-bit key (dst << 32 | src): one radix sort of (key, edge index) pairs,
//     then a gather of the weights; offsets by a lower_bound per vertex over the
//     sorted keys (no atomics on hub counters, no serial fill of empty runs);
//   * normalize_lt_weights, restated per in-list with the same sequential fp64
//     sums, the same float roundings and the same 64-attempt deflation, so the
//     weights are bit-identical (the library builds with --fmad=false).
#include <cub/device/device_radix_sort.cuh>

#include "internal.hpp"

namespace rrgpu {

namespace {

__global__ void k_edge_keys(const uint32_t* src, const uint32_t* dst, uint64_t m, uint32_t n,
                            unsigned long long* keys, uint32_t* idx, uint32_t* bad) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = src[i], d = dst[i];
    if (s >= n || d >= n) atomicOr(bad, 1u);
    keys[i] = (static_cast<unsigned long long>(d) << 32) | s;
    idx[i] = static_cast<uint32_t>(i);
  }
}

// Sorted keys -> transpose sources and weights (edge i of the sorted order).
__global__ void k_scatter_transpose(const unsigned long long* keys, const uint32_t* idx,
                                    const float* w_in, uint64_t m, uint32_t* rsrc, float* rw) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    rsrc[i] = static_cast<uint32_t>(keys[i]);
    rw[i] = w_in[idx[i]];
  }
}

// off[v] = index of the first sorted key whose target is >= v (v in [0, n]), one
// thread per vertex with a lower_bound over the sorted keys: no serial fill of
// zero-in-degree runs, whatever the gaps between targets.
__global__ void k_transpose_offsets(const unsigned long long* keys, uint64_t m, uint32_t n,
                                    uint32_t* off) {
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v <= n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long key = static_cast<unsigned long long>(v) << 32;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    off[v] = static_cast<uint32_t>(lo);
  }
}

// normalize_lt_weights (graph.hpp:207-235) for in-list v, sequential like the
// reference: sum of the float weights in fp64; if above 1, scale = 1/sum,
// deflated by (1 - 2^-20) until the fp64 sum of the float-rounded scaled
// weights is <= 1 (at most 64 attempts), then the weights are rescaled.
__device__ void normalize_list(float* w, uint32_t b, uint32_t e, uint32_t v, uint32_t* bad) {
  double sum = 0.0;
  for (uint32_t j = b; j < e; ++j) {
    const float x = w[j];
    if (x < 0.0f) {
      atomicMin(bad, v);  // the reference throws at the first such vertex
      return;
    }
    sum = __dadd_rn(sum, static_cast<double>(x));
  }
  if (sum <= 1.0) return;
  double scale = __ddiv_rn(1.0, sum);
  for (int attempt = 0; attempt < 64; ++attempt) {
    double scaled = 0.0;
    for (uint32_t j = b; j < e; ++j)
      scaled = __dadd_rn(scaled, static_cast<double>(__double2float_rn(
                                     __dmul_rn(static_cast<double>(w[j]), scale))));
    if (scaled <= 1.0) break;
    scale = __dmul_rn(scale, 1.0 - 0x1.0p-20);
  }
  for (uint32_t j = b; j < e; ++j)
    w[j] = __double2float_rn(__dmul_rn(static_cast<double>(w[j]), scale));
}

// Lists of at least kNormWarpMin in-edges (hubs: cfg4's largest has 543K) go to
// a warp each, so the sequential fp64 chain is not also a chain of dependent
// global loads: the lanes load and convert a chunk of kNormChunk addends into
// shared memory (the next chunk's loads in flight meanwhile) and lane 0 adds
// them in list order -- the same additions, in the same order, as above.
constexpr uint32_t kNormWarpMin = 256;
constexpr uint32_t kNormChunk = 256;
constexpr int kNormWarps = 8;

__global__ void k_normalize_lt(const uint32_t* off, uint32_t n, float* w, uint32_t* bad) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t b = off[v], e = off[v + 1];
    if (e - b < kNormWarpMin) normalize_list(w, b, e, v, bad);
  }
}

// s = fl(a + b); err |= (a + b != s): Knuth's TwoSum, no ordering assumption.
__device__ __forceinline__ double norm_add_checked(double a, double b, bool& err) {
  const double s = __dadd_rn(a, b);
  const double bb = __dadd_rn(s, -a);
  const double e = __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb));
  err |= e != 0.0;
  return s;
}

// Sum over w[b, e) in list order of x (scale == 0) or of float(x * scale),
// both widened to fp64; returns the sum in every lane. *neg is set when an
// addend is negative (first pass only, like the reference's check).
// The reference's running sum is a serial fp64 chain, but almost all of its adds
// are exact (float addends, a sum of order 1), and exact adds are associative: a
// chunk of 256 addends is scanned in parallel -- eight consecutive addends per
// lane, a warp scan of the lane totals, the running sum added last -- with every
// add checked by TwoSum. When all error terms are zero EVERY prefix of the chunk
// came out exact, hence representable, hence what the serial chain holds at that
// point (by induction from the running sum): the chunk's last prefix is the
// chain's value. Checking only a reduction tree would not do -- a prefix can
// need rounding while the total does not. A chunk with a nonzero error term is
// added by lane 0 in list order (the plain chain).
__device__ double warp_list_sum(const float* w, uint32_t b, uint32_t e, double scale,
                                double* sm, bool* neg) {
  const uint32_t lane = threadIdx.x & 31;
  float r[kNormChunk / 32];
  auto load = [&](uint32_t c) {  // lane l: addends [8 l, 8 l + 8) of the chunk
#pragma unroll
    for (uint32_t k = 0; k < kNormChunk / 32; ++k) {
      const uint32_t i = c + 8 * lane + k;
      r[k] = i < e ? w[i] : 0.0f;
    }
  };
  double sum = 0.0;
  bool anyneg = false;
  load(b);
  for (uint32_t c = b; c < e; c += kNormChunk) {
    bool mine = false, err = false;
    double x[kNormChunk / 32], run = 0.0;
#pragma unroll
    for (uint32_t k = 0; k < kNormChunk / 32; ++k) {
      mine |= r[k] < 0.0f;
      x[k] = scale == 0.0
          ? static_cast<double>(r[k])
          : static_cast<double>(__double2float_rn(__dmul_rn(static_cast<double>(r[k]), scale)));
      run = k == 0 ? x[0] : norm_add_checked(run, x[k], err);  // prefixes inside the lane
    }
    if (__any_sync(0xffffffffu, mine)) {
      anyneg = true;
      break;
    }
    if (c + kNormChunk < e) load(c + kNormChunk);
    double incl = run;  // inclusive scan of the lane totals: the prefixes at lane ends
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl = norm_add_checked(y, incl, err);
    }
    double base = __shfl_up_sync(0xffffffffu, incl, 1);
    base = lane == 0 ? sum : norm_add_checked(sum, base, err);
    // every prefix of the chunk: running sum + lanes before + inside the lane
    double pre = base;
#pragma unroll
    for (uint32_t k = 0; k < kNormChunk / 32; ++k) pre = norm_add_checked(pre, x[k], err);
    // (pre re-adds the lane's addends onto base one by one: each step IS a prefix)
    if (!__any_sync(0xffffffffu, err)) {
      sum = __shfl_sync(0xffffffffu, pre, 31);
    } else {  // some add rounded: the plain chain over this chunk
#pragma unroll
      for (uint32_t k = 0; k < kNormChunk / 32; ++k) sm[8 * lane + k] = x[k];
      __syncwarp();
      if (lane == 0) {
        const uint32_t cnt = e - c < kNormChunk ? e - c : kNormChunk;
#pragma unroll 8
        for (uint32_t i = 0; i < cnt; ++i) sum = __dadd_rn(sum, sm[i]);
      }
      sum = __shfl_sync(0xffffffffu, sum, 0);
      __syncwarp();
    }
  }
  *neg = anyneg;
  return sum;
}

__global__ void __launch_bounds__(kNormWarps * 32)
    k_normalize_lt_hubs(const uint32_t* off, uint32_t n, float* w, uint32_t* bad) {
  __shared__ double smem[kNormWarps][kNormChunk];
  double* sm = smem[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = warp * 32; base < n; base += nwarps * 32) {
    const uint32_t mv = base + lane;
    const bool hub = mv < n && off[mv + 1] - off[mv] >= kNormWarpMin;
    uint32_t hubs = __ballot_sync(0xffffffffu, hub);
    while (hubs) {
      const uint32_t v = base + __ffs(hubs) - 1;
      hubs &= hubs - 1;
      const uint32_t b = off[v], e = off[v + 1];
      bool neg = false;
      const double sum = warp_list_sum(w, b, e, 0.0, sm, &neg);
      if (neg) {
        if (lane == 0) atomicMin(bad, v);
        continue;
      }
      if (sum <= 1.0) continue;
      double scale = __ddiv_rn(1.0, sum);
      for (int attempt = 0; attempt < 64; ++attempt) {
        // scale > 0 here (sum is finite > 1, or +inf/NaN giving 0/NaN: then
        // the scaled pass below uses the sequential form instead).
        double scaled;
        if (scale > 0.0) {
          scaled = warp_list_sum(w, b, e, scale, sm, &neg);
        } else {
          scaled = 0.0;
          if (lane == 0)
            for (uint32_t j = b; j < e; ++j)
              scaled = __dadd_rn(scaled, static_cast<double>(__double2float_rn(
                                             __dmul_rn(static_cast<double>(w[j]), scale))));
          scaled = __shfl_sync(0xffffffffu, scaled, 0);
        }
        if (scaled <= 1.0) break;
        scale = __dmul_rn(scale, 1.0 - 0x1.0p-20);
      }
      for (uint32_t j = b + lane; j < e; j += 32)
        w[j] = __double2float_rn(__dmul_rn(static_cast<double>(w[j]), scale));
      __syncwarp();
    }
  }
}

}  // namespace

// Builds g->off/src/w from an edge list already on the device (d_src, d_dst, d_w).
// Returns 0, or 1 for an out-of-range vertex id, or 2 + v for a negative weight
// on vertex v (normalize only).
uint64_t build_transpose_device(rrg_graph* g, const uint32_t* d_src, const uint32_t* d_dst,
                                const float* d_w, bool normalize, cudaEvent_t w_ready) {
  const uint32_t n = g->n;
  const uint64_t m = g->m;
  const cudaStream_t st = g->stream;
  g->off.reserve_discard(static_cast<size_t>(n) + 1);
  g->src.reserve_discard(m ? m : 1);
  g->w.reserve_discard(m ? m : 1);
  DevBuf<uint32_t> bad;
  bad.reserve_discard(2);
  const uint32_t init[2] = {0u, 0xffffffffu};
  RRG_CUDA(cudaMemcpyAsync(bad.ptr, init, 8, cudaMemcpyHostToDevice, st));
  if (m == 0) {
    if (w_ready) RRG_CUDA(cudaStreamWaitEvent(st, w_ready, 0));
    RRG_CUDA(cudaMemsetAsync(g->off.ptr, 0, (static_cast<size_t>(n) + 1) * 4, st));
  } else {
    DevBuf<unsigned long long> keys, keys2;
    DevBuf<uint32_t> idx, idx2;
    keys.reserve_discard(m);
    keys2.reserve_discard(m);
    idx.reserve_discard(m);
    idx2.reserve_discard(m);
    const int grid = g->num_sms * 8;
    k_edge_keys<<<grid, 256, 0, st>>>(d_src, d_dst, m, n, keys.ptr, idx.ptr, bad.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    // Out-of-range ids are rejected before the sort: the keys only carry
    // 32 + vbits bits, and the offsets below assume every target is < n.
    uint32_t hbad = 0;
    RRG_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, 4, cudaMemcpyDeviceToHost, st));
    host_sync((st));
    if (hbad) return 1;
    int vbits = 1;
    while (vbits < 32 && (1ull << vbits) < n) ++vbits;
    size_t temp_bytes = 0;
    RRG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys.ptr, keys2.ptr, idx.ptr,
                                             idx2.ptr, static_cast<int64_t>(m), 0, 32 + vbits,
                                             st));
    DevBuf<uint8_t> temp;
    temp.reserve_discard(temp_bytes ? temp_bytes : 1);
    RRG_CUDA(cub::DeviceRadixSort::SortPairs(temp.ptr, temp_bytes, keys.ptr, keys2.ptr, idx.ptr,
                                             idx2.ptr, static_cast<int64_t>(m), 0, 32 + vbits,
                                             st));
    count_launch();
    if (w_ready) RRG_CUDA(cudaStreamWaitEvent(st, w_ready, 0));
    k_scatter_transpose<<<grid, 256, 0, st>>>(keys2.ptr, idx2.ptr, d_w, m, g->src.ptr,
                                              g->w.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    k_transpose_offsets<<<(n + 256) / 256, 256, 0, st>>>(keys2.ptr, m, n, g->off.ptr);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    host_sync((st));  // temporaries are released at scope end
  }
  uint32_t hb[2] = {0, 0};
  RRG_CUDA(cudaMemcpyAsync(hb, bad.ptr, 8, cudaMemcpyDeviceToHost, st));
  host_sync((st));
  if (hb[0]) return 1;
  if (normalize && n) {
    k_normalize_lt<<<(n + 127) / 128, 128, 0, st>>>(g->off.ptr, n, g->w.ptr, bad.ptr + 1);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    k_normalize_lt_hubs<<<g->num_sms * 4, kNormWarps * 32, 0, st>>>(g->off.ptr, n, g->w.ptr,
                                                                    bad.ptr + 1);
    RRG_CUDA(cudaGetLastError());
    count_launch();
    RRG_CUDA(cudaMemcpyAsync(hb, bad.ptr, 8, cudaMemcpyDeviceToHost, st));
    host_sync((st));
    if (hb[1] != 0xffffffffu) return 2ull + hb[1];
  }
  return 0;
}

}  // namespace rrgpu
