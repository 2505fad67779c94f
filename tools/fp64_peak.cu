// fp64_peak.cu — measures the B200 FP64 roofline denominators that
// MEASURED_PEAKS.json lacks: DFMA (SIMT) and DMMA (mma.sync m8n8k4 f64) peak
// TFLOP/s, burst (one 0.2 s launch) and sustained (back-to-back for ~3 s).
// Prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// Mixed: even warps issue DMMA, odd warps DFMA, in the same CTA — does the
// FP64 tensor path add throughput on top of the DFMA pipe, or share it?
__global__ void mixed_kernel(double* out, int iters_mma, int iters_fma, double a0, double b0) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a0, b0);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
  } else {
    double a = threadIdx.x * 1e-3, b = 0.999;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  float ms;
  // DFMA: flops per launch = blocks*threads*iters*16*8*2
  int it = 2000;
  dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, it, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = (double)blocks * threads * it * 16 * 8 * 2;
  double dfma_burst = fl / (ms * 1e-3) / 1e12;
  cudaEventRecord(e0);
  int reps = 0;
  float tot = 0;
  while (tot < 3000.f) {
    for (int r = 0; r < 10; ++r) dfma_kernel<<<blocks, threads>>>(out, it, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&tot, e0, e1);
    reps += 10;
  }
  double dfma_sust = fl * reps / (tot * 1e-3) / 1e12;
  // DMMA: flops per mma = 512 per warp
  it = 1000;
  dmma_kernel<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  dmma_kernel<<<blocks, threads>>>(out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double flm = (double)blocks * (threads / 32) * it * 8 * 4 * 512;
  double dmma_burst = flm / (ms * 1e-3) / 1e12;
  cudaEventRecord(e0);
  reps = 0;
  tot = 0;
  while (tot < 3000.f) {
    for (int r = 0; r < 10; ++r) dmma_kernel<<<blocks, threads>>>(out, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&tot, e0, e1);
    reps += 10;
  }
  double dmma_sust = flm * reps / (tot * 1e-3) / 1e12;
  // mixed: half the warps each; per-warp work sized so that both halves take
  // about the same time if the two paths were independent
  const int im = 500, iff = 1000;
  mixed_kernel<<<blocks, threads>>>(out, 10, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  for (int r = 0; r < 10; ++r) mixed_kernel<<<blocks, threads>>>(out, im, iff, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double flmix = 10.0 * blocks * ((threads / 64) * (double)im * 8 * 4 * 512 +
                                  (threads / 2) * (double)iff * 16 * 8 * 2);
  double mixed = flmix / (ms * 1e-3) / 1e12;
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\": %d, \"dfma_tflops_burst\": %.3f, \"dfma_tflops_sustained\": %.3f, "
         "\"dmma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, \"mixed_half_warps_tflops\": %.3f, "
         "\"err\": \"%s\"}\n",
         sms, dfma_burst, dfma_sust, dmma_burst, dmma_sust, mixed, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
