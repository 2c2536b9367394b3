// Probe: does a tail launch wait for the parent's fire-and-forget children?
#include <cstdio>
#include <cuda_runtime.h>
__device__ volatile int g_flag;
__device__ int g_seen[4];
__device__ long long g_t[8];
__device__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void slow_k() {
  if (threadIdx.x == 0 && blockIdx.x == 0) { g_t[1] = gt(); long long t0 = clock64(); while (clock64() - t0 < 400000) {} g_flag = 1; __threadfence(); g_t[2] = gt(); }
}
__global__ void check_k(int i) { if (threadIdx.x == 0 && blockIdx.x == 0) { g_seen[i] = g_flag; g_t[3 + i] = gt(); } }
__global__ void planner() {
  if (threadIdx.x) return;
  g_t[0] = gt();
  slow_k<<<148, 128, 0, cudaStreamFireAndForget>>>();
  for (int i = 0; i < 3; ++i) check_k<<<1, 32, 0, cudaStreamTailLaunch>>>(i);
  g_t[7] = gt();
}
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int r = 0; r < 3; ++r) {
    int z = 0; cudaMemcpyToSymbol(g_flag, &z, 4);
    planner<<<1, 32, 0, st>>>(); cudaStreamSynchronize(st);
    int s[4]; long long t[8]; cudaMemcpyFromSymbol(s, g_seen, 16); cudaMemcpyFromSymbol(t, g_t, 64);
    printf("tail saw flag: %d %d %d | slow start %+lld end %+lld, planner end %+lld, checks %+lld %+lld %+lld (ns from planner start)\n", s[0], s[1], s[2],
           t[1]-t[0], t[2]-t[0], t[7]-t[0], t[3]-t[0], t[4]-t[0], t[5]-t[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
