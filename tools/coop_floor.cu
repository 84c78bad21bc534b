// latency floor of a cooperative launch with N grid syncs (DESIGN.md adv-norm table):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o coop_floor tools/coop_floor.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int n, int* out) { cg::grid_group g = cg::this_grid(); for (int i = 0; i < n; ++i) g.sync(); if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = n; }
__global__ void kn(int* out) { if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = 1; }
int main() {
  int* d; cudaMalloc(&d, 4); cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {33, 148, 296}) for (int n : {0, 1, 2, 4, 8}) {
    void* args[] = {&n, &d};
    float best = 1e9;
    for (int it = 0; it < 30; ++it) {
      cudaEventRecord(a, s);
      cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, s);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (it > 3 && ms < best) best = ms;
    }
    printf("coop grid %d syncs %d: %.2f us\n", grid, n, best * 1e3);
  }
  float best = 1e9;
  for (int it = 0; it < 30; ++it) { cudaEventRecord(a, s); kn<<<33, 256, 0, s>>>(d); cudaEventRecord(b, s); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (it > 3 && ms < best) best = ms; }
  printf("plain launch: %.2f us\n", best * 1e3);
}
