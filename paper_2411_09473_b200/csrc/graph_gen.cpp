// graph_gen.cpp -- rrgen: the pinned synthetic inputs of the BASELINE configs
// (SURVEY.md Appendix B), as a standalone executable.
//
//   rrgen KIND N M P0 P1 P2 P3 FLAGS GRAPH_SEED WEIGHTS WEIGHT_SCALE WEIGHT_SEED THREADS
//
// writes to stdout: u32 n, u32 0, u64 arcs, then the transpose arrays
// reverse_offsets u64[n+1], reverse_sources u32[arcs], reverse_weights f32[arcs]
// (the reverse arrays of rrflow::Graph, in detail::build_graph's in-list order,
// graph.hpp:69-115). Exit status 2 + a message on stderr for a bad spec.
//
// It is plumbing, not product: a separate process so that both bench arms get
// byte-identical graphs while the reference arm maps only oracle/_ref, and the
// product library (librrgpu.so) carries no generator.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
static std::string g_error;
void set_error(const std::string& msg) { g_error = msg; }
}  // namespace rrgpu

namespace {

enum GenKind {
  kGenRmat = 0,          // p0 = scale, p1..p3 = a, b, c; edges = m (unique, no loops)
  kGenChungLu = 1,       // directed; p0 = gamma; flags bit 0: correlated in/out
  kGenChungLuUndir = 2,  // undirected, m unique pairs -> 2m arcs
};
enum WeightKind {
  kWWc = 0,         // f32(1/indeg(v))
  kWUniform = 1,    // U(0, scale) f32
  kWLtUniform = 2,  // U(0,1) / per-vertex double sum, then normalize_lt_weights
};
struct GenSpec {
  int kind;
  uint32_t n;
  uint64_t m;  // edges (directed) or unique pairs (undirected)
  double p0, p1, p2, p3;
  uint32_t flags;
  uint64_t graph_seed;
  int weights;
  double weight_scale;
  uint64_t weight_seed;
  uint32_t threads;  // 0 = hardware concurrency
};

}  // namespace

namespace {

unsigned pick_threads(uint32_t req) {
  unsigned t = req ? req : std::thread::hardware_concurrency();
  return t ? t : 1;
}

// Runs fn(t, begin, end) over `threads` contiguous slices of [0, total).
void parallel_slices(uint64_t total, unsigned threads,
                     const std::function<void(unsigned, uint64_t, uint64_t)>& fn) {
  if (threads <= 1 || total < 4096) {
    fn(0, 0, total);
    return;
  }
  std::vector<std::thread> pool;
  const uint64_t chunk = (total + threads - 1) / threads;
  for (unsigned t = 0; t < threads; ++t) {
    const uint64_t b = std::min<uint64_t>(total, t * chunk);
    const uint64_t e = std::min<uint64_t>(total, b + chunk);
    pool.emplace_back([&fn, t, b, e] { fn(t, b, e); });
  }
  for (auto& th : pool) th.join();
}

inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Counter-based uniform in [0,1) for item i of stream `seed`.
inline double hash_u01(uint64_t seed, uint64_t i) {
  const uint64_t x = mix64(seed ^ mix64(i * 0xd1b54a32d192ed03ULL + 0x632be59bd9b4e019ULL));
  return static_cast<double>(x >> 11) * 0x1.0p-53;
}

struct Rng {  // xoshiro256** seeded per candidate (generators only)
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    for (auto& w : s) {
      seed = mix64(seed);
      w = seed;
    }
  }
  static uint64_t rol(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t out = rol(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rol(s[3], 45);
    return out;
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

// Parallel LSD radix sort of 64-bit keys on their low `bits` bits.
void radix_sort(std::vector<uint64_t>& keys, unsigned bits, unsigned threads) {
  std::vector<uint64_t> tmp(keys.size());
  const uint64_t total = keys.size();
  for (unsigned shift = 0; shift < bits; shift += 8) {
    std::vector<std::vector<uint64_t>> hist(threads, std::vector<uint64_t>(256, 0));
    parallel_slices(total, threads, [&](unsigned t, uint64_t b, uint64_t e) {
      auto& h = hist[t];
      for (uint64_t i = b; i < e; ++i) h[(keys[i] >> shift) & 255]++;
    });
    // the slices used above must match the scatter slices: recompute them
    uint64_t run = 0;
    const bool single = threads <= 1 || total < 4096;
    const unsigned used = single ? 1 : threads;
    std::vector<std::vector<uint64_t>> pos(used, std::vector<uint64_t>(256, 0));
    for (unsigned d = 0; d < 256; ++d)
      for (unsigned t = 0; t < used; ++t) {
        pos[t][d] = run;
        run += hist[t][d];
      }
    parallel_slices(total, threads, [&](unsigned t, uint64_t b, uint64_t e) {
      auto& p = pos[t];
      for (uint64_t i = b; i < e; ++i) tmp[p[(keys[i] >> shift) & 255]++] = keys[i];
    });
    keys.swap(tmp);
  }
}

struct KeyIdx {
  uint64_t key;
  uint64_t idx;
};

// Stable parallel LSD radix sort of (key, idx) records on the key's low `bits`.
void radix_sort_pairs(std::vector<KeyIdx>& a, unsigned bits, unsigned threads) {
  std::vector<KeyIdx> tmp(a.size());
  const uint64_t total = a.size();
  const bool single = threads <= 1 || total < 4096;
  const unsigned used = single ? 1 : threads;
  for (unsigned shift = 0; shift < bits; shift += 8) {
    std::vector<std::vector<uint64_t>> hist(used, std::vector<uint64_t>(256, 0));
    parallel_slices(total, threads, [&](unsigned t, uint64_t b, uint64_t e) {
      auto& h = hist[t];
      for (uint64_t i = b; i < e; ++i) h[(a[i].key >> shift) & 255]++;
    });
    uint64_t run = 0;
    for (unsigned d = 0; d < 256; ++d)
      for (unsigned t = 0; t < used; ++t) {
        const uint64_t c = hist[t][d];
        hist[t][d] = run;
        run += c;
      }
    parallel_slices(total, threads, [&](unsigned t, uint64_t b, uint64_t e) {
      auto& p = hist[t];
      for (uint64_t i = b; i < e; ++i) tmp[p[(a[i].key >> shift) & 255]++] = a[i];
    });
    a.swap(tmp);
  }
}

// Deduplicated, loop-free edge keys (src << 32 | dst): the first `m` distinct
// candidates in candidate-index order, returned sorted ascending. `draw(i)`
// yields candidate i as a key or UINT64_MAX (self-loop). The candidate pool
// grows by 1.25x until it holds m distinct keys. Deterministic for any thread
// count (every step is a function of the candidate sequence only).
std::vector<uint64_t> unique_edges(uint64_t m, unsigned bits, unsigned threads,
                                   const std::function<uint64_t(uint64_t)>& draw) {
  uint64_t pool = m + m / 4 + 1024;
  for (int attempt = 0; attempt < 64; ++attempt, pool += pool / 4) {
    std::vector<KeyIdx> a(pool);
    parallel_slices(pool, threads, [&](unsigned, uint64_t b, uint64_t e) {
      for (uint64_t i = b; i < e; ++i) a[i] = {draw(i), i};
    });
    radix_sort_pairs(a, bits, threads);  // loops (all ones) sort last; idx ascending per key
    std::vector<uint8_t> first(pool, 0);
    parallel_slices(pool, threads, [&](unsigned, uint64_t b, uint64_t e) {
      for (uint64_t j = b; j < e; ++j) {
        if (a[j].key == UINT64_MAX) continue;
        if (j == 0 || a[j - 1].key != a[j].key) first[a[j].idx] = 1;
      }
    });
    uint64_t distinct = 0;
    for (uint64_t i = 0; i < pool; ++i) distinct += first[i];
    if (distinct < m) continue;
    // the m distinct keys whose first occurrence comes earliest
    uint64_t cutoff = 0, seen = 0;
    while (seen < m) seen += first[cutoff++];
    std::vector<uint64_t> keys;
    keys.reserve(m);
    for (uint64_t j = 0; j < pool; ++j) {
      const KeyIdx& r = a[j];
      if (r.key == UINT64_MAX) break;
      if ((j == 0 || a[j - 1].key != r.key) && r.idx < cutoff) keys.push_back(r.key);
    }
    return keys;  // already ascending
  }
  throw std::runtime_error("generator cannot reach the edge count");
}

// Transpose of sorted (src, dst) keys: in-lists ordered by source ascending,
// which is the order detail::build_graph produces (graph.hpp:96-113).
void keys_to_transpose(uint32_t n, const std::vector<uint64_t>& keys, unsigned threads,
                       uint64_t* roff, uint32_t* rsrc) {
  const uint64_t m = keys.size();
  const bool single = threads <= 1 || m < 4096;
  const unsigned used = single ? 1 : threads;
  std::vector<std::vector<uint32_t>> cnt(used);
  parallel_slices(m, threads, [&](unsigned t, uint64_t b, uint64_t e) {
    auto& c = cnt[t];
    c.assign(n, 0);
    for (uint64_t i = b; i < e; ++i) c[static_cast<uint32_t>(keys[i])]++;
  });
  uint64_t run = 0;
  std::vector<std::vector<uint64_t>> pos(used, std::vector<uint64_t>(n));
  for (uint32_t v = 0; v < n; ++v) {
    roff[v] = run;
    for (unsigned t = 0; t < used; ++t) {
      pos[t][v] = run;
      run += cnt[t][v];
    }
  }
  roff[n] = run;
  cnt.clear();
  parallel_slices(m, threads, [&](unsigned t, uint64_t b, uint64_t e) {
    auto& p = pos[t];
    for (uint64_t i = b; i < e; ++i) {
      const uint32_t d = static_cast<uint32_t>(keys[i]);
      rsrc[p[d]++] = static_cast<uint32_t>(keys[i] >> 32);
    }
  });
}

unsigned key_bits(uint32_t n) {
  unsigned b = 1;
  while ((1ull << b) < n) ++b;
  return 32 + b;  // src occupies bits [32, 32+b)
}

// Chung-Lu sampler: rank i has weight (i+1)^(-1/(gamma-1)), drawn in O(1) with
// a Vose alias table; ranks map to ids through a seeded permutation.
struct ChungLu {
  std::vector<double> prob;
  std::vector<uint32_t> alias;
  std::vector<uint32_t> perm_out, perm_in;
  ChungLu(uint32_t n, double gamma, bool correlated, uint64_t seed) {
    const double ex = -1.0 / (gamma - 1.0);
    std::vector<double> w(n);
    double total = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
      w[i] = std::pow(static_cast<double>(i + 1), ex);
      total += w[i];
    }
    prob.assign(n, 1.0);
    alias.resize(n);
    std::vector<uint32_t> small, large;
    for (uint32_t i = 0; i < n; ++i) {
      w[i] = w[i] * n / total;
      alias[i] = i;
      (w[i] < 1.0 ? small : large).push_back(i);
    }
    while (!small.empty() && !large.empty()) {
      const uint32_t s = small.back(), l = large.back();
      small.pop_back();
      prob[s] = w[s];
      alias[s] = l;
      w[l] = (w[l] + w[s]) - 1.0;
      if (w[l] < 1.0) {
        large.pop_back();
        small.push_back(l);
      }
    }
    auto shuffle = [n](uint64_t s) {
      std::vector<uint32_t> p(n);
      for (uint32_t i = 0; i < n; ++i) p[i] = i;
      Rng r(s);
      for (uint32_t i = n; i > 1; --i) {
        const uint32_t j = static_cast<uint32_t>((static_cast<unsigned __int128>(r.next()) * i) >> 64);
        std::swap(p[i - 1], p[j]);
      }
      return p;
    };
    perm_out = shuffle(mix64(seed ^ 0x0badc0deULL));
    perm_in = correlated ? perm_out : shuffle(mix64(seed ^ 0x5eedf00dULL));
  }
  uint32_t rank(double u) const {
    const double x = u * static_cast<double>(prob.size());
    uint32_t i = static_cast<uint32_t>(x);
    if (i >= prob.size()) i = static_cast<uint32_t>(prob.size() - 1);
    return (x - i) < prob[i] ? i : alias[i];
  }
};


rrg_status generate_graph(const GenSpec* spec, uint32_t* n_out, uint64_t* m_out, uint64_t* roff,
                          uint32_t* rsrc, float* rw) {
  if (!spec || !n_out || !m_out) {
    rrgpu::set_error("generate_graph: null argument");
    return RRG_EINVAL;
  }
  uint32_t n = spec->n;
  uint64_t arcs = spec->m;
  if (spec->kind == kGenRmat) {
    const int scale = static_cast<int>(spec->p0);
    if (scale < 1 || scale > 31) {
      rrgpu::set_error("rmat: scale out of range");
      return RRG_EINVAL;
    }
    n = 1u << scale;
  } else if (spec->kind == kGenChungLuUndir) {
    arcs = 2 * spec->m;
  } else if (spec->kind != kGenChungLu) {
    rrgpu::set_error("unknown generator");
    return RRG_EINVAL;
  }
  if (n < 2 || arcs >= (1ull << 32)) {
    rrgpu::set_error("generator: n must be >= 2 and arcs < 2^32");
    return RRG_EINVAL;
  }
  const double pairs = static_cast<double>(n) * (n - 1) / (spec->kind == kGenChungLuUndir ? 2 : 1);
  if (static_cast<double>(spec->m) > 0.5 * pairs) {
    rrgpu::set_error("generator: too dense");
    return RRG_EINVAL;
  }
  *n_out = n;
  *m_out = arcs;
  if (!roff) return RRG_OK;
  if (!rsrc || !rw) {
    rrgpu::set_error("generate_graph: null arrays");
    return RRG_EINVAL;
  }
  try {
    const unsigned threads = pick_threads(spec->threads);
    const unsigned bits = key_bits(n);
    const uint64_t gseed = spec->graph_seed;
    std::vector<uint64_t> keys;
    if (spec->kind == kGenRmat) {
      // R-MAT: per level pick a quadrant with probabilities a, b, c, d=1-a-b-c
      const int scale = static_cast<int>(spec->p0);
      const double a = spec->p1, ab = spec->p1 + spec->p2, abc = spec->p1 + spec->p2 + spec->p3;
      keys = unique_edges(spec->m, bits, threads, [&](uint64_t i) -> uint64_t {
        Rng r(gseed * 0x9e3779b97f4a7c15ULL + i);
        uint32_t s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
          const double u = r.u01();
          const uint32_t sb = u >= ab ? 1u : 0u;
          const uint32_t db = (u >= a && u < ab) || u >= abc ? 1u : 0u;
          s = (s << 1) | sb;
          d = (d << 1) | db;
        }
        if (s == d) return UINT64_MAX;
        return (static_cast<uint64_t>(s) << 32) | d;
      });
    } else {
      const bool correlated = spec->flags & 1u;
      const bool undirected = spec->kind == kGenChungLuUndir;
      ChungLu cl(n, spec->p0, correlated || undirected, gseed);
      keys = unique_edges(spec->m, bits, threads, [&](uint64_t i) -> uint64_t {
        const uint32_t s = cl.perm_out[cl.rank(hash_u01(gseed, 2 * i))];
        const uint32_t d = cl.perm_in[cl.rank(hash_u01(gseed, 2 * i + 1))];
        if (s == d) return UINT64_MAX;
        if (undirected) {
          const uint32_t lo = std::min(s, d), hi = std::max(s, d);
          return (static_cast<uint64_t>(lo) << 32) | hi;
        }
        return (static_cast<uint64_t>(s) << 32) | d;
      });
      if (undirected) {
        const uint64_t pairs_n = keys.size();
        keys.resize(2 * pairs_n);
        for (uint64_t i = 0; i < pairs_n; ++i) {
          const uint64_t k = keys[i];
          keys[pairs_n + i] = (k << 32) | (k >> 32);
        }
        radix_sort(keys, bits, threads);
      }
    }
    keys_to_transpose(n, keys, threads, roff, rsrc);
    keys.clear();
    keys.shrink_to_fit();
    // weights, keyed by transpose position j (deterministic for any thread count)
    const uint64_t wseed = spec->weight_seed;
    if (spec->weights == kWWc) {
      parallel_slices(n, threads, [&](unsigned, uint64_t b, uint64_t e) {
        for (uint64_t v = b; v < e; ++v) {
          const uint64_t deg = roff[v + 1] - roff[v];
          if (!deg) continue;
          const float p = static_cast<float>(1.0 / static_cast<double>(deg));
          for (uint64_t j = roff[v]; j < roff[v + 1]; ++j) rw[j] = p;
        }
      });
    } else if (spec->weights == kWUniform) {
      const double sc = spec->weight_scale;
      parallel_slices(arcs, threads, [&](unsigned, uint64_t b, uint64_t e) {
        for (uint64_t j = b; j < e; ++j) rw[j] = static_cast<float>(hash_u01(wseed, j) * sc);
      });
    } else if (spec->weights == kWLtUniform) {
      parallel_slices(n, threads, [&](unsigned, uint64_t b, uint64_t e) {
        for (uint64_t v = b; v < e; ++v) {
          double sum = 0.0;
          for (uint64_t j = roff[v]; j < roff[v + 1]; ++j) sum += hash_u01(wseed, j);
          for (uint64_t j = roff[v]; j < roff[v + 1]; ++j)
            rw[j] = static_cast<float>(hash_u01(wseed, j) / sum);
        }
      });
      const rrg_status st = rrg_normalize_lt_weights(n, roff, rw);
      if (st != RRG_OK) return st;
    } else {
      rrgpu::set_error("unknown weight model");
      return RRG_EINVAL;
    }
    return RRG_OK;
  } catch (const std::bad_alloc&) {
    rrgpu::set_error("generate_graph: out of host memory");
    return RRG_ENOMEM;
  } catch (const std::exception& e) {
    rrgpu::set_error(e.what());
    return RRG_EINVAL;
  }
}

}  // namespace

namespace {

bool write_all(const void* p, size_t bytes) {
  const char* c = static_cast<const char*>(p);
  while (bytes) {
    const size_t w = std::fwrite(c, 1, std::min<size_t>(bytes, 1u << 26), stdout);
    if (!w) return false;
    c += w;
    bytes -= w;
  }
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 14) {
    std::fprintf(stderr, "usage: rrgen KIND N M P0 P1 P2 P3 FLAGS GRAPH_SEED WEIGHTS "
                         "WEIGHT_SCALE WEIGHT_SEED THREADS\n");
    return 2;
  }
  GenSpec s{};
  s.kind = std::atoi(argv[1]);
  s.n = static_cast<uint32_t>(std::strtoul(argv[2], nullptr, 10));
  s.m = std::strtoull(argv[3], nullptr, 10);
  s.p0 = std::strtod(argv[4], nullptr);
  s.p1 = std::strtod(argv[5], nullptr);
  s.p2 = std::strtod(argv[6], nullptr);
  s.p3 = std::strtod(argv[7], nullptr);
  s.flags = static_cast<uint32_t>(std::strtoul(argv[8], nullptr, 10));
  s.graph_seed = std::strtoull(argv[9], nullptr, 10);
  s.weights = std::atoi(argv[10]);
  s.weight_scale = std::strtod(argv[11], nullptr);
  s.weight_seed = std::strtoull(argv[12], nullptr, 10);
  s.threads = static_cast<uint32_t>(std::strtoul(argv[13], nullptr, 10));
  uint32_t n = 0;
  uint64_t m = 0;
  if (generate_graph(&s, &n, &m, nullptr, nullptr, nullptr) != RRG_OK) {
    std::fprintf(stderr, "%s\n", rrgpu::g_error.c_str());
    return 2;
  }
  std::vector<uint64_t> roff(static_cast<size_t>(n) + 1);
  std::vector<uint32_t> rsrc(m ? m : 1);
  std::vector<float> rw(m ? m : 1);
  if (generate_graph(&s, &n, &m, roff.data(), rsrc.data(), rw.data()) != RRG_OK) {
    std::fprintf(stderr, "%s\n", rrgpu::g_error.c_str());
    return 2;
  }
  const uint32_t hdr32[2] = {n, 0u};
  if (!write_all(hdr32, 8) || !write_all(&m, 8) || !write_all(roff.data(), roff.size() * 8) ||
      !write_all(rsrc.data(), m * 4) || !write_all(rw.data(), m * 4) || std::fflush(stdout)) {
    std::fprintf(stderr, "rrgen: write failed\n");
    return 3;
  }
  return 0;
}
