// Probe: CDP2 tail launches (ordering, chains, big dynamic smem, stream capture, latency).
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_log[64];
__device__ unsigned g_pos;
__device__ long long g_t[8];
__global__ void stamp(int id) {
  if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned p = atomicAdd(&g_pos, 1); if (p < 64) g_log[p] = id; }
}
__global__ void bigsmem(int id) {
  extern __shared__ int s[];
  s[threadIdx.x] = id; __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned p = atomicAdd(&g_pos, 1); if (p < 64) g_log[p] = 1000 + s[0]; }
}
__global__ void planner(int level, int maxl) {
  if (threadIdx.x) return;
  stamp<<<100, 64, 0, cudaStreamTailLaunch>>>(level * 10 + 1);
  bigsmem<<<10, 128, 200 * 1024, cudaStreamTailLaunch>>>(level * 10 + 2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("device launch error %d at level %d\n", (int)e, level);
  stamp<<<3, 32, 0, cudaStreamTailLaunch>>>(level * 10 + 3);
  if (level + 1 < maxl) planner<<<1, 32, 0, cudaStreamTailLaunch>>>(level + 1, maxl);
}
__global__ void chain(int left) {
  if (threadIdx.x) return;
  if (left > 0) chain<<<1, 32, 0, cudaStreamTailLaunch>>>(left - 1);
}
__global__ void manytail(int n) {
  if (threadIdx.x) return;
  for (int i = 0; i < n; ++i) stamp<<<1, 32, 0, cudaStreamTailLaunch>>>(500 + i);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("manytail error %d\n", (int)e);
}
__global__ void after() { unsigned p = atomicAdd(&g_pos, 1); if (p < 64) g_log[p] = 9999; }
int main() {
  cudaFuncSetAttribute(bigsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  unsigned z = 0;
  cudaMemcpyToSymbol(g_pos, &z, 4);
  planner<<<1, 32, 0, st>>>(0, 3);
  after<<<1, 1, 0, st>>>();
  cudaError_t q = cudaStreamQuery(st);
  printf("query right after launch: %s\n", cudaGetErrorString(q));
  cudaStreamSynchronize(st);
  printf("sync: %s\n", cudaGetErrorString(cudaGetLastError()));
  unsigned long long lg[64]; unsigned pos;
  cudaMemcpyFromSymbol(lg, g_log, sizeof lg); cudaMemcpyFromSymbol(&pos, g_pos, 4);
  printf("order (%u):", pos); for (unsigned i = 0; i < pos && i < 64; ++i) printf(" %llu", lg[i]); printf("\n");
  // many tail launches from one grid
  cudaMemcpyToSymbol(g_pos, &z, 4);
  manytail<<<1, 32, 0, st>>>(40);
  cudaStreamSynchronize(st);
  cudaMemcpyFromSymbol(&pos, g_pos, 4);
  printf("manytail(40) ran %u: %s\n", pos, cudaGetErrorString(cudaGetLastError()));
  // latency of a chain of tail launches
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a, st); chain<<<1, 32, 0, st>>>(1000); cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("chain of 1000 tail launches: %.3f ms (%s)\n", ms, cudaGetErrorString(cudaGetLastError()));
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a, st); for (int i = 0; i < 1000; ++i) stamp<<<1, 32, 0, st>>>(0); cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("1000 host launches: %.3f ms\n", ms);
  }
  // stream capture
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaMemcpyToSymbol(g_pos, &z, 4);
  cudaError_t e1 = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  planner<<<1, 32, 0, st>>>(0, 2);
  after<<<1, 1, 0, st>>>();
  cudaError_t e2 = cudaStreamEndCapture(st, &g);
  cudaError_t e3 = cudaGraphInstantiate(&ge, g, 0);
  printf("capture: %s %s %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3));
  if (e3 == cudaSuccess) {
    for (int r = 0; r < 2; ++r) { cudaError_t e4 = cudaGraphLaunch(ge, st); printf("graph launch: %s\n", cudaGetErrorString(e4)); }
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(lg, g_log, sizeof lg); cudaMemcpyFromSymbol(&pos, g_pos, 4);
    printf("graph order (%u):", pos); for (unsigned i = 0; i < pos && i < 64; ++i) printf(" %llu", lg[i]); printf("  err %s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
