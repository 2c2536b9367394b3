// Probe: device-side launch call cost vs parameter size, and gap between tail-launched kernels.
#include <cstdio>
#include <cuda_runtime.h>
struct Big { unsigned long long w[42]; };  // 336 B like LevelArgs
__device__ unsigned g_sink;
__device__ long long g_t[64];
__global__ void small_k(unsigned long long x) { if (threadIdx.x == 0 && blockIdx.x == 99999) g_sink = (unsigned)x; }
__global__ void big_k(Big b) { if (threadIdx.x == 0 && blockIdx.x == 99999) g_sink = (unsigned)b.w[3]; }
__global__ void stamp_k(int i) { if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_t[i] = t; } }
__global__ void launcher(int mode, int k) {
  if (threadIdx.x) return;
  long long t0 = clock64();
  Big b; for (int i = 0; i < 42; ++i) b.w[i] = i;
  for (int i = 0; i < k; ++i) {
    if (mode == 0) small_k<<<888, 256, 0, cudaStreamTailLaunch>>>(i);
    else if (mode == 1) big_k<<<888, 256, 0, cudaStreamTailLaunch>>>(b);
    else stamp_k<<<888, 256, 0, cudaStreamTailLaunch>>>(i);
  }
  long long t1 = clock64();
  printf("mode %d: %d launches %lld cycles (%lld per launch)\n", mode, k, t1 - t0, (t1 - t0) / k);
}
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int r = 0; r < 2; ++r) {
    launcher<<<1, 32, 0, st>>>(0, 10); cudaStreamSynchronize(st);
    launcher<<<1, 32, 0, st>>>(1, 10); cudaStreamSynchronize(st);
    launcher<<<1, 32, 0, st>>>(2, 20); cudaStreamSynchronize(st);
    long long t[64]; cudaMemcpyFromSymbol(t, g_t, sizeof t);
    printf("gaps between tail-launched kernels (ns):"); for (int i = 1; i < 20; ++i) printf(" %lld", t[i] - t[i-1]); printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
