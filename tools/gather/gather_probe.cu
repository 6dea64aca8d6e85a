// gather_probe.cu -- B200 ceiling for the guide-mode LT walk: random 32-byte
// gathers from a table far larger than L2, issued as DEPENDENT chains (each
// load's address comes from the previous load's payload, like a walk step) by
// `lanes` concurrent chains. Prints loads/s and the 32-B-sector bandwidth; run
// under ncu to read the DRAM bytes per load (fetch granularity).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -DGATHER_MAIN -o gather_probe gather_probe.cu
//   ./gather_probe [table_GB=8] [steps=256]
// Built as libgather_probe.so (Makefile) for bench.py, which measures the
// ceiling live on the box it benchmarks on: gather_ceiling().
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const uint4* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                 "=r"(b.w)
               : "l"(p));
}

__global__ void fill(uint4* t, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + 1) * 0x9e3779b97f4a7c15ull ^ seed;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    t[2 * i] = make_uint4((uint32_t)z, (uint32_t)(z >> 32), 0, 0);
    t[2 * i + 1] = make_uint4(0, 0, 0, 0);
  }
}

// chains: every thread follows `steps` dependent 32-B loads
__global__ void __launch_bounds__(256) chase(const uint4* t, uint64_t n, int steps,
                                             unsigned long long* sink) {
  uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull % n;
  uint32_t acc = 0;
  for (int s = 0; s < steps; ++s) {
    uint4 a, b;
    ld256(t + 2 * i, a, b);
    const uint64_t z = ((uint64_t)a.y << 32) | a.x;
    acc += a.x;
    i = z % n;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// Best dependent random 32-B gathers per second over 1..8 blocks of 256 chains
// per SM from a table of `gb` GB (0 on a CUDA error). The table is freed.
extern "C" double gather_ceiling(double gb, int steps) {
  const uint64_t n = (uint64_t)(gb * (1ull << 30)) / 32;
  uint4* t = nullptr;
  unsigned long long* sink = nullptr;
  if (cudaMalloc(&t, n * 32) != cudaSuccess) return 0.0;
  if (cudaMalloc(&sink, 8) != cudaSuccess) {
    cudaFree(t);
    return 0.0;
  }
  fill<<<148 * 16, 256>>>(t, n, 7);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int bps : {1, 2, 4, 8}) {
    const int grid = sms * bps;
    chase<<<grid, 256>>>(t, n, 8, sink);  // warm
    cudaEventRecord(e0);
    chase<<<grid, 256>>>(t, n, steps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double rate = (double)grid * 256 * steps / (ms * 1e-3);
    if (rate > best) best = rate;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(t);
  return cudaGetLastError() == cudaSuccess ? best : 0.0;
}

#ifdef GATHER_MAIN
int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 8.0;
  const int steps = argc > 2 ? atoi(argv[2]) : 256;
  const uint64_t n = (uint64_t)(gb * (1ull << 30)) / 32;
  if (argc > 3) {  // L2 fetch granularity hint in bytes (32 / 64 / 128)
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[3]));
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("{\"l2_fetch_granularity\": %zu}\n", got);
  }
  uint4* t;
  unsigned long long* sink;
  cudaMalloc(&t, n * 32);
  cudaMalloc(&sink, 8);
  fill<<<148 * 16, 256>>>(t, n, 7);
  cudaDeviceSynchronize();
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {1, 2, 4, 8}) {
    const int grid = sms * bps;
    chase<<<grid, 256>>>(t, n, 8, sink);  // warm
    cudaEventRecord(e0);
    chase<<<grid, 256>>>(t, n, steps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double loads = (double)grid * 256 * steps;
    printf("{\"chains\": %d, \"steps\": %d, \"ms\": %.3f, \"gloads_per_s\": %.3f, "
           "\"sector_GBps\": %.1f, \"ns_per_step\": %.1f}\n",
           grid * 256, steps, ms, loads / ms / 1e6, loads * 32 / ms / 1e6, ms * 1e6 / steps);
  }
  return 0;
}
#endif
