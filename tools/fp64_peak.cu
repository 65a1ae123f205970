// FP64 peak microbenchmark (B200): DMMA m8n8k4 (FP64 tensor cores) and DFMA.
// Prints one JSON line {"dmma_tflops": .., "dfma_tflops": ..}.  The roofline
// denominator for the sweep's FP64 kernels (MEASURED_PEAKS.json has no FP64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double c[8][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double c[8];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  double best_mma = 0, best_fma = 0;
  for (int rep = 0; rep < 5; ++rep) {
    const int it = 20000;
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(out, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 256.0 * 8 * it * (double)blocks * (threads / 32);  // 256 FMA per DMMA.8x8x4
    if (rep) best_mma = fmax(best_mma, fl / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ff = 2.0 * 8 * it * (double)blocks * threads;
    if (rep) best_fma = fmax(best_fma, ff / (ms * 1e-3) / 1e12);
  }
  printf("{\"dmma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"sms\": %d}\n", best_mma, best_fma, sms);
  return 0;
}
