// dense.cu -- the dense arm of the RRR store.
//
// The reference keeps a sketch of >= n / density_divisor members as an n-bit
// map instead of a sorted id list (make_repr, rrr_set.hpp:73-90; pack_sketch
// snapshots the visited words, sampling.hpp:68-84). On the device a dense set
// is a row of a pool of n-bit maps (u32 words, rows 16-byte aligned) and an
// EMPTY range of the flat list buffer; the row carries the member count and
// the root. The kernels here:
//   * convert staged lists of long sets into rows at commit (the block / warp /
//     lane schedules emit lists; the big-set path writes rows itself from its
//     visited map, sample.cu);
//   * column sums over rows: counter[v] +/-= #rows holding v -- thread per
//     (word, 32-row chunk), each row's word loaded coalesced across the warp and
//     added into six bit-sliced planes, so a row costs one load and ~18 logic
//     ops per 32 vertices instead of one atomic per member. This is the recount
//     of rebuild_update (selection.hpp:161-203), the decrement of covered rows
//     and build_counter (:79-95) over rows;
//   * export: lengths, then rows decoded root first, ascending after it;
//   * fraction_covered over rows; row gathers for store-to-store appends.
#include "internal.hpp"

#include <cmath>

namespace rrgpu {

namespace {

constexpr uint32_t kChunkRows = 32;  // rows per column-sum work item (counts < 64: 6 planes)

__global__ void k_dense_mark(const uint32_t* slot_len, uint64_t count, uint32_t thr,
                             uint32_t* dreq, unsigned long long* dctl) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t len = slot_len[i];
    if (len && len >= thr) dreq[atomicAdd(dctl, 1ull)] = static_cast<uint32_t>(i);
  }
}

__global__ void k_densify(const uint32_t* dreq, uint64_t nreq, const uint32_t* stage,
                          const uint64_t* slot_start, uint32_t* slot_len, uint32_t* bdix,
                          uint64_t row0, uint64_t set_base, uint32_t* dbits, uint32_t dwords,
                          uint32_t* dlen, uint32_t* droot, uint32_t* dslot,
                          unsigned long long* dctl) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  for (uint64_t j = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; j < nreq;
       j += warps) {
    const uint32_t i = dreq[j];
    const uint64_t row = row0 + j;
    uint32_t* dst = dbits + row * dwords;
    for (uint32_t w = lane; w < dwords; w += 32) dst[w] = 0u;
    __syncwarp();
    const uint32_t len = slot_len[i];
    const uint32_t* from = stage + slot_start[i];
    for (uint32_t t = lane; t < len; t += 32) {
      const uint32_t v = from[t];
      RRG_DCHECK(v < dwords * 32u, 9);
      atomicOr(dst + (v >> 5), 1u << (v & 31));
    }
    __syncwarp();
    if (lane == 0) {
      dlen[row] = len;
      droot[row] = from[0];  // visit order: the root first
      dslot[row] = static_cast<uint32_t>(set_base + i);
      bdix[i] = static_cast<uint32_t>(row);
      slot_len[i] = 0;  // empty list range
      atomicAdd(dctl + 1, static_cast<unsigned long long>(len));
      atomicMax(dctl + 2, static_cast<unsigned long long>(len));
    }
  }
}

// x added into the bit-sliced counters p[0..5] (lane b of p[i] = bit i of the
// count of vertex 32 w + b).
__device__ __forceinline__ void slice_add(uint32_t (&p)[6], uint32_t x) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t c = p[i] & x;
    p[i] ^= x;
    x = c;
  }
}

__global__ void k_dense_colsum(const uint32_t* dbits, uint32_t dwords, uint32_t n,
                               const uint32_t* rows, uint64_t row0, uint64_t nrows,
                               uint32_t* counter, int sign) {
  const uint64_t nchunks = (nrows + kChunkRows - 1) / kChunkRows;
  const uint64_t items = nchunks * dwords;
  for (uint64_t it = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; it < items;
       it += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = it / dwords;
    const uint32_t w = static_cast<uint32_t>(it - c * dwords);
    if (static_cast<uint64_t>(w) * 32 >= n) continue;
    uint32_t p[6] = {0, 0, 0, 0, 0, 0};
    const uint64_t d0 = c * kChunkRows;
    const uint64_t d1 = d0 + kChunkRows < nrows ? d0 + kChunkRows : nrows;
    for (uint64_t d = d0; d < d1; ++d) {
      const uint64_t row = rows ? rows[d] : row0 + d;
      slice_add(p, __ldg(dbits + row * dwords + w));
    }
    uint32_t any = p[0] | p[1] | p[2] | p[3] | p[4] | p[5];
    while (any) {
      const int b = __ffs(any) - 1;
      any &= any - 1;
      uint32_t cnt = 0;
#pragma unroll
      for (int i = 0; i < 6; ++i) cnt |= ((p[i] >> b) & 1u) << i;
      uint32_t* dst = counter + static_cast<uint64_t>(w) * 32 + b;
      if (sign > 0) atomicAdd(dst, cnt);
      else atomicSub(dst, cnt);
    }
  }
}

__global__ void k_set_lengths(const uint64_t* off, const uint32_t* dix, const uint32_t* dlen,
                              uint64_t first, uint64_t count, uint32_t* xlen) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = first + i;
    const uint32_t r = dix[s];
    xlen[i] = r == kNoRow ? static_cast<uint32_t>(off[s + 1] - off[s]) : dlen[r];
  }
}

__global__ void k_materialize(const uint64_t* off, const uint32_t* mem, const uint32_t* dix,
                              const uint32_t* dbits, uint32_t dwords, const uint32_t* droot,
                              uint64_t first, uint64_t count, const uint64_t* xoff,
                              uint32_t* xmem) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < count;
       i += warps) {
    const uint64_t s = first + i;
    const uint32_t r = dix[s];
    const uint64_t o = xoff[i];
    if (r == kNoRow) {
      const uint64_t b = off[s], e = off[s + 1];
      for (uint64_t t = b + lane; t < e; t += 32) xmem[o + (t - b)] = mem[t];
      continue;
    }
    const uint32_t root = droot[r];
    const uint32_t* row = dbits + static_cast<uint64_t>(r) * dwords;
    if (lane == 0) xmem[o] = root;
    uint64_t pos = o + 1;
    for (uint32_t w0 = 0; w0 < dwords; w0 += 32) {
      const uint32_t w = w0 + lane;
      uint32_t x = w < dwords ? row[w] : 0u;
      if (w == (root >> 5)) x &= ~(1u << (root & 31));
      const uint32_t c = __popc(x);
      uint32_t incl = c;
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
      }
      uint64_t at = pos + incl - c;
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        RRG_DCHECK(at < xoff[i + 1], 10);
        xmem[at++] = w * 32 + b;
      }
      pos += __shfl_sync(kFull, incl, 31);
    }
  }
}

__global__ void k_dense_fraction(const uint32_t* dbits, uint32_t dwords, uint64_t nrows,
                                 const uint32_t* seeds, uint32_t nseeds,
                                 unsigned long long* hits) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * blockDim.x / 32;
  unsigned long long local = 0;
  for (uint64_t r = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; r < nrows;
       r += warps) {
    const uint32_t* row = dbits + r * dwords;
    bool hit = false;
    for (uint32_t i = lane; i < nseeds && !hit; i += 32) {
      const uint32_t v = seeds[i];
      hit = (row[v >> 5] >> (v & 31)) & 1u;
    }
    if (__any_sync(kFull, hit) && lane == 0) ++local;
  }
  if (lane == 0 && local) atomicAdd(hits, local);
}

__global__ void k_gather_rows(const uint32_t* src, uint32_t dwords, const uint32_t* src_rows,
                              uint64_t nrows, uint32_t* dst, uint64_t dst_row0) {
  const uint32_t q = dwords / 4;  // rows are 16-byte aligned, dwords % 4 == 0
  for (uint64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const uint4* a = reinterpret_cast<const uint4*>(src + static_cast<uint64_t>(src_rows[r]) * dwords);
    uint4* b = reinterpret_cast<uint4*>(dst + (dst_row0 + r) * dwords);
    for (uint32_t t = threadIdx.x; t < q; t += blockDim.x) b[t] = a[t];
  }
}

__global__ void k_live_flags(const uint64_t* off, const uint32_t* dix, const uint32_t* wmem,
                             const uint32_t* covered, const uint32_t* dcov, bool scan,
                             uint64_t first, uint64_t count, uint8_t* out) {
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = first + i;
    const uint32_t r = dix[s];
    bool live;
    if (r != kNoRow) live = dcov[r] == 0u;
    else if (scan) live = wmem[off[s]] != 0xffffffffu;  // covered sets are blanked
    else live = covered[s] == 0u;
    out[i] = live ? 1 : 0;
  }
}

int grid_items(uint64_t items, int block) {
  const uint64_t b = (items + block - 1) / block;
  return static_cast<int>(b < 1 ? 1 : (b > 65535 ? 65535 : b));
}

}  // namespace

uint32_t dense_threshold(uint32_t n, uint32_t divisor) {
  if (divisor == 0) return kNoDense;
  const double t = std::ceil(static_cast<double>(n) / static_cast<double>(divisor));
  if (!(t < 4294967295.0)) return kNoDense;
  return t < 1.0 ? 1u : static_cast<uint32_t>(t);
}

void launch_dense_mark(const uint32_t* slot_len, uint64_t count, uint32_t thr, uint32_t* dreq,
                       unsigned long long* dctl, cudaStream_t s) {
  if (!count) return;
  k_dense_mark<<<grid_items(count, 256), 256, 0, s>>>(slot_len, count, thr, dreq, dctl);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_densify(const uint32_t* dreq, uint64_t nreq, const uint32_t* stage,
                    const uint64_t* slot_start, uint32_t* slot_len, uint32_t* bdix, uint64_t row0,
                    uint64_t set_base, uint32_t* dbits, uint32_t dwords, uint32_t* dlen,
                    uint32_t* droot, uint32_t* dslot, unsigned long long* dctl, cudaStream_t s) {
  if (!nreq) return;
  k_densify<<<grid_items(nreq * 32, 256), 256, 0, s>>>(dreq, nreq, stage, slot_start, slot_len,
                                                       bdix, row0, set_base, dbits, dwords, dlen,
                                                       droot, dslot, dctl);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_dense_colsum(const uint32_t* dbits, uint32_t dwords, uint32_t n, const uint32_t* rows,
                         uint64_t row0, uint64_t nrows, uint32_t* counter, int sign,
                         cudaStream_t s) {
  if (!nrows || !dwords) return;
  const uint64_t items = (nrows + kChunkRows - 1) / kChunkRows * dwords;
  k_dense_colsum<<<grid_items(items, 256), 256, 0, s>>>(dbits, dwords, n, rows, row0, nrows,
                                                        counter, sign);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_set_lengths(const uint64_t* off, const uint32_t* dix, const uint32_t* dlen,
                        uint64_t first, uint64_t count, uint32_t* xlen, cudaStream_t s) {
  if (!count) return;
  k_set_lengths<<<grid_items(count, 256), 256, 0, s>>>(off, dix, dlen, first, count, xlen);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_materialize(const uint64_t* off, const uint32_t* mem, const uint32_t* dix,
                        const uint32_t* dbits, uint32_t dwords, const uint32_t* droot,
                        uint64_t first, uint64_t count, const uint64_t* xoff, uint32_t* xmem,
                        cudaStream_t s) {
  if (!count) return;
  k_materialize<<<grid_items(count * 32, 256), 256, 0, s>>>(off, mem, dix, dbits, dwords, droot,
                                                           first, count, xoff, xmem);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_live_flags(const uint64_t* off, const uint32_t* dix, const uint32_t* wmem,
                       const uint32_t* covered, const uint32_t* dcov, bool scan, uint64_t first,
                       uint64_t count, uint8_t* out, cudaStream_t s) {
  k_live_flags<<<grid_items(count, 256), 256, 0, s>>>(off, dix, wmem, covered, dcov, scan, first,
                                                      count, out);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_dense_fraction(const uint32_t* dbits, uint32_t dwords, uint64_t nrows,
                           const uint32_t* seeds, uint32_t nseeds, unsigned long long* hits,
                           cudaStream_t s) {
  if (!nrows || !nseeds) return;
  k_dense_fraction<<<grid_items(nrows * 32, 256), 256, 0, s>>>(dbits, dwords, nrows, seeds, nseeds,
                                                              hits);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

void launch_gather_rows(const uint32_t* src, uint32_t dwords, const uint32_t* src_rows,
                        uint64_t nrows, uint32_t* dst, uint64_t dst_row0, cudaStream_t s) {
  if (!nrows) return;
  k_gather_rows<<<static_cast<unsigned>(nrows < 4096 ? nrows : 4096), 256, 0, s>>>(
      src, dwords, src_rows, nrows, dst, dst_row0);
  RRG_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace rrgpu
