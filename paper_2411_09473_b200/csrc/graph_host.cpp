// graph_host.cpp -- host-side graph preparation: the reference's transpose
// construction and LT normalization (restated; the device builds the same
// arrays in graph_dev.cu). The synthetic BASELINE generators live in
// graph_gen.cpp, a separate executable (rrgen), so a process that only needs
// the inputs -- bench.py's reference arm -- never maps librrgpu.so.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/rrgpu.h"

namespace rrgpu {
void set_error(const std::string& msg);
}

extern "C" {

rrg_status rrg_build_transpose(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                               const float* w, uint64_t* roff, uint32_t* rsrc, float* rw) {
  // detail::build_graph (graph.hpp:69-115): forward slots by a stable counting
  // sort on the source; the transpose then walks sources ascending and forward
  // slots in order, so each in-list is ordered by (source, input position).
  if (!roff || (m && (!src || !dst || !w || !rsrc || !rw))) {
    rrgpu::set_error("rrg_build_transpose: null argument");
    return RRG_EINVAL;
  }
  for (uint64_t e = 0; e < m; ++e) {
    if (src[e] >= n || dst[e] >= n) {
      rrgpu::set_error("rrg_build_transpose: vertex id out of range");
      return RRG_EINVAL;
    }
  }
  try {
    std::vector<uint64_t> fo(static_cast<size_t>(n) + 1, 0);
    for (uint64_t e = 0; e < m; ++e) fo[src[e] + 1]++;
    for (uint32_t v = 0; v < n; ++v) fo[v + 1] += fo[v];
    std::vector<uint64_t> order(m);  // forward slot -> input edge
    {
      std::vector<uint64_t> cur(fo.begin(), fo.end() - 1);
      for (uint64_t e = 0; e < m; ++e) order[cur[src[e]]++] = e;
    }
    std::fill(roff, roff + n + 1, 0);
    for (uint64_t e = 0; e < m; ++e) roff[dst[e] + 1]++;
    for (uint32_t v = 0; v < n; ++v) roff[v + 1] += roff[v];
    std::vector<uint64_t> cur(roff, roff + n);
    for (uint64_t slot = 0; slot < m; ++slot) {
      const uint64_t e = order[slot];
      const uint64_t p = cur[dst[e]]++;
      rsrc[p] = src[e];
      rw[p] = w[e];
    }
    return RRG_OK;
  } catch (const std::bad_alloc&) {
    rrgpu::set_error("rrg_build_transpose: out of host memory");
    return RRG_ENOMEM;
  }
}

rrg_status rrg_normalize_lt_weights(uint32_t n, const uint64_t* roff, float* rw) {
  // normalize_lt_weights (graph.hpp:207-235): in-lists whose double sum exceeds
  // one are rescaled, the scale deflated by (1 - 2^-20) until the float-rounded
  // sum stays <= 1; feasible in-lists are untouched. Negative weights rejected.
  if (!roff || (roff[n] && !rw)) {
    rrgpu::set_error("rrg_normalize_lt_weights: null argument");
    return RRG_EINVAL;
  }
  for (uint32_t v = 0; v < n; ++v) {
    const uint64_t b = roff[v], e = roff[v + 1];
    double sum = 0.0;
    for (uint64_t j = b; j < e; ++j) {
      if (rw[j] < 0.0f) {
        rrgpu::set_error("negative edge weight on vertex " + std::to_string(v));
        return RRG_EINVAL;
      }
      sum += rw[j];
    }
    if (sum <= 1.0) continue;
    double scale = 1.0 / sum;
    for (int attempt = 0; attempt < 64; ++attempt) {
      double check = 0.0;
      for (uint64_t j = b; j < e; ++j) check += static_cast<float>(rw[j] * scale);
      if (check <= 1.0) break;
      scale *= 1.0 - 0x1.0p-20;
    }
    for (uint64_t j = b; j < e; ++j) rw[j] = static_cast<float>(rw[j] * scale);
  }
  return RRG_OK;
}

}  // extern "C"
