// gridsync_probe.cu -- cost of one cooperative-groups grid barrier on this GPU
// (the selection loop pays two per round). nvcc -O3 -arch=sm_100a -o gs gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x ^ i;
    g.sync();
  }
  if (acc == 0xdeadbeef) atomicAdd(sink, 1u);
}
int main() {
  unsigned* sink;
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bps : {1, 2}) for (int th : {256, 512, 1024}) {
    if (bps * th > 1024) continue;
    int grid = sms * bps, iters = 2000;
    void* args[] = {&iters, &sink};
    int it0 = 10;
    void* a0[] = {&it0, &sink};
    cudaLaunchCooperativeKernel((void*)k, grid, th, a0, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, grid, th, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid %d x %d: %.3f us per grid.sync (%s)\n", grid, th, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
}
