// FP64 pipe sharing: cost of DADDs interleaved with DMMAs.  One CTA per SM,
// W warps, 4 independent DMMA chains per warp, K independent DADD chains
// issued per group of 4 DMMAs.  Prints ns per group and the marginal cost of
// one DADD in DMMA units ((t_K - t_0) / K / (t_0 / 4)).
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void mix(double *out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[4][2];
  double d[K > 0 ? K : 1];
#pragma unroll
  for (int i = 0; i < 4; i++) c[i][0] = c[i][1] = 0;
#pragma unroll
  for (int i = 0; i < (K > 0 ? K : 1); i++) d[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int k = i; k < K; k += 4) asm volatile("add.f64 %0, %0, %1;" : "+d"(d[k]) : "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (K > 0 ? K : 1); i++) s += d[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int K>
double run(int sms, int warps, int iters) {
  double *out;
  cudaMalloc(&out, 8192);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<K><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e0);
  mix<K><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return ms * 1e6 / iters;   // ns per group (all warps)
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int w : {4, 8, 12}) {
    const double t0 = run<0>(sms, w, iters);
    const double tf = (double)sms * w * 4 * 512.0 / (t0 * 1e-9) / 1e12;
    printf("W=%2d: 4 DMMA/group %.3f ns (%.1f TFLOP/s)\n", w, t0, tf);
    const double t[] = {run<1>(sms, w, iters), run<2>(sms, w, iters), run<4>(sms, w, iters), run<8>(sms, w, iters),
                        run<16>(sms, w, iters)};
    const int ks[] = {1, 2, 4, 8, 16};
    for (int i = 0; i < 5; i++)
      printf("   +%2d DADD: %.3f ns  -> one DADD = %.3f DMMA\n", ks[i], t[i], (t[i] - t0) / ks[i] / (t0 / 4));
  }
  return 0;
}
