// Probe: cost split of a device launch: parameter buffer (parallel, many threads) vs the launch call.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned g_sink;
__device__ long long g_t[64];
__global__ void stamp_k(int i) { if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_t[i] = t; } }
__global__ void launcher2(int k) {
  __shared__ void *bufs[32];
  __shared__ long long tget[32];
  long long t0 = clock64();
  if (threadIdx.x < k) {
    long long a = clock64();
    void *b = cudaGetParameterBufferV2((void *)stamp_k, dim3(888), dim3(256), 0);
    *(int *)b = threadIdx.x;
    bufs[threadIdx.x] = b;
    tget[threadIdx.x] = clock64() - a;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < k; ++i) cudaLaunchDeviceV2(bufs[i], cudaStreamTailLaunch);
    long long t2 = clock64();
    printf("k=%d: get (parallel) %lld cycles (thread0 %lld), launch calls %lld cycles (%lld each)\n", k, t1 - t0, tget[0], t2 - t1, (t2 - t1) / k);
  }
}
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int r = 0; r < 3; ++r) {
    launcher2<<<1, 32, 0, st>>>(12); cudaStreamSynchronize(st);
    long long t[64]; cudaMemcpyFromSymbol(t, g_t, sizeof t);
    printf("order/gaps (ns):"); for (int i = 1; i < 12; ++i) printf(" %lld", t[i] - t[i-1]); printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
