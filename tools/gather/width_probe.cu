// width_probe.cu -- DRAM bytes per random dependent gather as a function of the
// load width (8 / 16 / 32 B at 32-B-aligned addresses; 64 B at 64-B-aligned) and
// of the L2 prefetch-size hint. Run under ncu (dram__bytes_read.sum per kernel).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o width_probe width_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill(uint2* t, uint64_t n8, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n8;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9e3779b97f4a7c15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    t[i] = make_uint2((uint32_t)z, (uint32_t)(z >> 32));
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) chase(const char* t, uint64_t n, int steps,
                                             unsigned long long* sink) {
  // n = number of 32-B entries (MODE 4: 64-B entries, n / 2 of them)
  uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull % n;
  uint32_t acc = 0;
  for (int s = 0; s < steps; ++s) {
    uint32_t x, y;
    if (MODE == 0) {  // 8 B
      asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "l"(t + 32 * i));
    } else if (MODE == 1) {  // 16 B
      uint32_t a, b;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(a), "=r"(b) : "l"(t + 32 * i));
      acc += a ^ b;
    } else if (MODE == 2) {  // 32 B
      uint32_t a, b, c, d, e, f;
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(x), "=r"(y), "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f) : "l"(t + 32 * i));
      acc += a ^ b ^ c ^ d ^ e ^ f;
    } else if (MODE == 3) {  // 32 B, plain ld.global (L1 allocate)
      uint32_t a, b, c, d, e, f;
      asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(x), "=r"(y), "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f) : "l"(t + 32 * i));
      acc += a ^ b ^ c ^ d ^ e ^ f;
    } else if (MODE == 4) {  // 64 B at 64-B alignment (two 32-B loads)
      uint32_t a, b, c, d, e, f, x2, y2;
      const char* q = t + 64 * (i >> 1);
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(x), "=r"(y), "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f) : "l"(q));
      acc += a ^ b ^ c ^ d ^ e ^ f;
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(x2), "=r"(y2), "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f) : "l"(q + 32));
      acc += a ^ b ^ c ^ d ^ e ^ f ^ x2 ^ y2;
    } else if (MODE == 5) {  // 32 B with evict-first policy
      uint32_t a, b, c, d, e, f;
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                   : "=r"(x), "=r"(y), "=r"(a), "=r"(b), "=r"(c), "=r"(d), "=r"(e), "=r"(f) : "l"(t + 32 * i), "l"(pol));
      acc += a ^ b ^ c ^ d ^ e ^ f;
    } else {  // 6: 4 B scalar
      asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(x) : "l"(t + 32 * i));
      asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(y) : "l"(t + 32 * i + 4));
    }
    const uint64_t z = ((uint64_t)y << 32) | x;
    acc += x;
    i = z % n;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 8.0;
  const int steps = argc > 2 ? atoi(argv[2]) : 64;
  const uint64_t n = (uint64_t)(gb * (1ull << 30)) / 32;
  char* t;
  unsigned long long* sink;
  cudaMalloc(&t, n * 32);
  cudaMalloc(&sink, 8);
  fill<<<148 * 16, 256>>>((uint2*)t, n * 4, 7);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8;
  const char* names[] = {"8B", "16B", "32B nc", "32B plain", "64B", "32B evict_first", "2x4B"};
  for (int mode = 0; mode < 7; ++mode) {
    cudaEventRecord(e0);
    switch (mode) {
      case 0: chase<0><<<grid, 256>>>(t, n, steps, sink); break;
      case 1: chase<1><<<grid, 256>>>(t, n, steps, sink); break;
      case 2: chase<2><<<grid, 256>>>(t, n, steps, sink); break;
      case 3: chase<3><<<grid, 256>>>(t, n, steps, sink); break;
      case 4: chase<4><<<grid, 256>>>(t, n, steps, sink); break;
      case 5: chase<5><<<grid, 256>>>(t, n, steps, sink); break;
      case 6: chase<6><<<grid, 256>>>(t, n, steps, sink); break;
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double loads = (double)grid * 256 * steps;
    printf("{\"mode\": \"%s\", \"gathers\": %.0f, \"ms\": %.3f, \"ggathers_per_s\": %.3f}\n", names[mode],
           loads, ms, loads / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
