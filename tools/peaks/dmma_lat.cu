// DMMA issue/latency microbenchmark: one CTA per SM, W warps per CTA, C independent
// accumulator chains per warp.  Reports TFLOP/s per (W, C) to expose the DMMA
// latency (C needed per warp) and the warps per SMSP needed to saturate the pipe.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void dmma_chain(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < C; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; i++) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int C>
double run(int sms, int warps, int iters) {
  double* out; cudaMalloc(&out, 8192);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_chain<C><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e0);
  dmma_chain<C><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  double flops = (double)sms * warps * iters * C * 512.0;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int ws[] = {1, 2, 3, 4, 5, 8, 16};
  printf("warps/CTA(1 CTA/SM) x chains/warp -> TFLOP/s\n");
  for (int w : ws) {
    printf("W=%2d: C1 %.1f  C2 %.1f  C4 %.1f  C8 %.1f  C16 %.1f\n", w, run<1>(sms, w, 20000), run<2>(sms, w, 10000),
           run<4>(sms, w, 5000), run<8>(sms, w, 2500), run<16>(sms, w, 1250));
  }
  return 0;
}
