// jump.cpp -- GF(2) jump-ahead for the per-slot xoshiro256** stream.
//
// The xoshiro256** state update (prng.hpp:33-43, without the output scrambler)
// is linear over GF(2)^256: s' = T s. Column c of T is the update applied to
// the unit state e_c; T^(2^i) follows by repeated squaring. Advancing a state
// by k draws is then the product of the T^(2^i) for the set bits of k -- the
// same stream position the reference reaches by calling next_u64() k times.
// The IC hub expansion (sample.cu) uses these matrices to give each lane of a
// warp its own exact segment of one slot's draw sequence.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/rrgpu.h"

namespace rrgpu {

namespace {

void state_step(uint64_t s[4]) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

void apply(const uint64_t* m, const uint64_t s[4], uint64_t out[4]) {
  uint64_t o[4] = {0, 0, 0, 0};
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = s[w];
    while (bits) {
      const int b = __builtin_ctzll(bits);
      bits &= bits - 1;
      const uint64_t* col = m + (static_cast<size_t>(w * 64 + b) * 4);
      o[0] ^= col[0];
      o[1] ^= col[1];
      o[2] ^= col[2];
      o[3] ^= col[3];
    }
  }
  std::memcpy(out, o, sizeof(o));
}

}  // namespace

// matrices[i] = T^(2^i), i in [0, count); each 256 columns x 4 words, column-major.
std::vector<uint64_t> jump_matrices(int count) {
  std::vector<uint64_t> mats(static_cast<size_t>(count) * 256 * 4);
  uint64_t* t0 = mats.data();
  for (int c = 0; c < 256; ++c) {
    uint64_t s[4] = {0, 0, 0, 0};
    s[c / 64] = 1ull << (c % 64);
    state_step(s);
    std::memcpy(t0 + c * 4, s, sizeof(s));
  }
  for (int i = 1; i < count; ++i) {
    const uint64_t* prev = mats.data() + static_cast<size_t>(i - 1) * 1024;
    uint64_t* cur = mats.data() + static_cast<size_t>(i) * 1024;
    for (int c = 0; c < 256; ++c) apply(prev, prev + c * 4, cur + c * 4);
  }
  return mats;
}

void jump_host(const std::vector<uint64_t>& mats, uint64_t s[4], uint64_t k) {
  for (int i = 0; k; ++i, k >>= 1)
    if (k & 1) apply(mats.data() + static_cast<size_t>(i) * 1024, s, s);
}

// M_l = T^(seg * l) for l = 1..count, column-major like jump_matrices(): lane l of
// a warp starts its segment of a window seg*l draws into the stream.
std::vector<uint64_t> segment_matrices(uint64_t seg, int count) {
  static const std::vector<uint64_t> pow2 = jump_matrices(64);
  std::vector<uint64_t> out(static_cast<size_t>(count) * 1024);
  for (int l = 1; l <= count; ++l) {
    uint64_t* m = out.data() + static_cast<size_t>(l - 1) * 1024;
    for (int c = 0; c < 256; ++c) {
      uint64_t s[4] = {0, 0, 0, 0};
      s[c / 64] = 1ull << (c % 64);
      jump_host(pow2, s, seg * static_cast<uint64_t>(l));
      std::memcpy(m + c * 4, s, sizeof(s));
    }
  }
  return out;
}

// Byte tables of the same matrices ("four Russians"): for byte position p of
// the state and byte value x, tab[p][x] = XOR of the columns 8p+i with bit i of x
// set. A jump is then 32 independent 32-byte loads XORed together instead of a
// data-dependent walk over up to 256 columns. Layout per matrix: [32][256][4].
std::vector<uint64_t> segment_tables(uint64_t seg, int count) {
  const std::vector<uint64_t> mats = segment_matrices(seg, count);
  std::vector<uint64_t> out(static_cast<size_t>(count) * 32 * 256 * 4);
  for (int l = 0; l < count; ++l) {
    const uint64_t* m = mats.data() + static_cast<size_t>(l) * 1024;
    uint64_t* t = out.data() + static_cast<size_t>(l) * 32 * 256 * 4;
    for (int p = 0; p < 32; ++p) {
      for (int x = 0; x < 256; ++x) {
        uint64_t acc[4] = {0, 0, 0, 0};
        for (int i = 0; i < 8; ++i) {
          if (!((x >> i) & 1)) continue;
          const uint64_t* col = m + static_cast<size_t>(8 * p + i) * 4;
          for (int w = 0; w < 4; ++w) acc[w] ^= col[w];
        }
        std::memcpy(t + (static_cast<size_t>(p) * 256 + x) * 4, acc, sizeof(acc));
      }
    }
  }
  return out;
}

}  // namespace rrgpu

extern "C" void rrg_debug_jump(const uint64_t* state_in, uint64_t k, uint64_t* state_out) {
  static const std::vector<uint64_t> mats = rrgpu::jump_matrices(64);
  uint64_t s[4];
  std::memcpy(s, state_in, sizeof(s));
  rrgpu::jump_host(mats, s, k);
  std::memcpy(state_out, s, sizeof(s));
}
