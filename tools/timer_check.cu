// timer_check.cu -- do %clock64 and %globaltimer agree with CUDA events?
#include <cstdio>
__global__ void spin(long long cycles, unsigned long long* out) {
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long c0 = clock64();
  while (clock64() - c0 < cycles) {}
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = c1 - c0; out[1] = g1 - g0; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (long long cyc : {1000000LL, 10000000LL}) {
    spin<<<148, 32>>>(cyc, d);
    cudaEventRecord(a); spin<<<148, 32>>>(cyc, d); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"cycles\":%llu,\"globaltimer_ns\":%llu,\"event_ms\":%.4f,\"clock_ghz\":%.3f,\"gt_vs_event\":%.3f}\n", h[0], h[1], ms, h[0] / (h[1] * 1.0), h[1] / (ms * 1e6));
  }
  return 0;
}
