// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Measures burst (short) and sustained (~3 s) throughput; prints one JSON line.
// Used to fix the roofline denominator (B200_PROFILING.md: no FP64 entry in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += c[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, double flops_per_thread_iter, double secs_target, float* ms_out) {
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters, 1e-3);  // warm
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int reps = 1;
  if (secs_target > 0) {
    reps = std::max(1, (int)(secs_target * 1e3 / ms));
    cudaEventRecord(e0);
    for (int r = 0; r < reps; r++) kern<<<blocks, threads>>>(out, iters, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  *ms_out = ms;
  cudaFree(out);
  return (double)blocks * threads * iters * flops_per_thread_iter * reps / (ms * 1e-3) / 1e12;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  float ms;
  // DMMA: 8x8x4 = 256 MAC = 512 flop per warp-instruction -> 16 flop per thread
  const int C = 8;
  double best_dmma = 0, best_dfma = 0; int best_occ_m = 0, best_occ_f = 0;
  for (int occ : {1, 2, 4, 8}) {
    double t = run(dmma_loop<C>, sms * occ, 256, 4096, 16.0 * C, 0, &ms);
    if (t > best_dmma) { best_dmma = t; best_occ_m = occ; }
    double f = run(dfma_loop<C>, sms * occ, 256, 4096, 2.0 * C, 0, &ms);
    if (f > best_dfma) { best_dfma = f; best_occ_f = occ; }
  }
  double sus_dmma = run(dmma_loop<C>, sms * best_occ_m, 256, 4096, 16.0 * C, 3.0, &ms);
  double sus_dfma = run(dfma_loop<C>, sms * best_occ_f, 256, 4096, 2.0 * C, 3.0, &ms);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, "
         "\"dfma_tflops_burst\": %.3f, \"dfma_tflops_sustained\": %.3f, \"occ_dmma\": %d, \"occ_dfma\": %d}\n",
         p.name, sms, best_dmma, sus_dmma, best_dfma, sus_dfma, best_occ_m, best_occ_f);
  return 0;
}
