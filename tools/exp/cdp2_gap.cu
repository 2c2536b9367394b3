// Probe: per-kernel gap of queued tail launches vs host launches (grids of 888 CTAs x 256 thr).
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned g_sink;
__global__ void work(int id) { if (threadIdx.x == 0 && blockIdx.x == 9999999) g_sink = id; }
__global__ void planner(int nk, int levels) {
  if (threadIdx.x) return;
  for (int i = 0; i < nk; ++i) work<<<888, 256, 0, cudaStreamTailLaunch>>>(i);
  if (levels > 1) planner<<<1, 32, 0, cudaStreamTailLaunch>>>(nk, levels - 1);
}
__global__ void planner_ff(int nk) {  // fire-and-forget into a device stream is unordered; here: one child per level via NULL stream
  if (threadIdx.x) return;
  for (int i = 0; i < nk; ++i) work<<<888, 256>>>(i);
}
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a, st); planner<<<1, 32, 0, st>>>(10, 3); cudaEventRecord(b, st); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("tail: 3 levels x 10 kernels: %.1f us (%s)\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    cudaEventRecord(a, st); for (int i = 0; i < 30; ++i) work<<<888, 256, 0, st>>>(i); cudaEventRecord(b, st); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("host: 30 kernels: %.1f us\n", ms * 1e3);
    cudaEventRecord(a, st); planner_ff<<<1, 32, 0, st>>>(30); cudaEventRecord(b, st); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("device NULL-stream: 30 kernels: %.1f us (%s)\n", ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
