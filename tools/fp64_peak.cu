// fp64_peak.cu -- FP64 pipe microbenchmark (B200, sm_100a): the denominator of
// bench.py's roofline.fp64_frac.  Every thread runs 8 independent dependency
// chains of DFMA / DMUL / DADD (enough ILP to hide the pipe latency) over a
// grid of 148 x 8 CTAs x 256 threads; throughput = thread-instructions / s,
// timed with CUDA events after a warm-up, best of 5.  The division and
// square root (MUFU.RCP64H / RSQ64H + DFMA Newton steps) are reported as
// calls / s for reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak > profiles/r02_fp64_peak.json
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_fp64(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = fma(x[k], a, b);
      if (OP == 1) x[k] = x[k] * a;
      if (OP == 2) x[k] = x[k] + b;
      if (OP == 3) x[k] = b / x[k];
      if (OP == 4) x[k] = sqrt(x[k] + b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

template <int OP>
double rate(int grid, int block, int iters, double a, double b) {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64<OP><<<grid, block>>>(out, iters, a, b);  // warm-up (clocks)
  k_fp64<OP><<<grid, block>>>(out, iters, a, b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fp64<OP><<<grid, block>>>(out, iters, a, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  return (double)grid * block * iters * 8 / (best * 1e-3);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = sms * 8, block = 256;
  const double fma_r = rate<0>(grid, block, 4096, 0.999999, 1e-7);
  const double mul_r = rate<1>(grid, block, 4096, 0.999999, 1e-7);
  const double add_r = rate<2>(grid, block, 4096, 0.999999, 1e-7);
  const double div_r = rate<3>(grid, block, 256, 0.999999, 1.0000001);
  const double sqrt_r = rate<4>(grid, block, 256, 0.999999, 1e-7);
  const double per_sm_clk = fma_r / sms / (clk * 1e3);
  std::printf(
      "{\"what\": \"FP64 pipe throughput, thread-instructions per second (8 independent chains per "
      "thread, %d CTAs x %d threads, best of 5, CUDA events)\",\n"
      " \"sms\": %d, \"clock_mhz_attr\": %.0f,\n"
      " \"dfma_per_s\": %.6e, \"dmul_per_s\": %.6e, \"dadd_per_s\": %.6e,\n"
      " \"ddiv_calls_per_s\": %.6e, \"dsqrt_calls_per_s\": %.6e,\n"
      " \"dfma_per_sm_per_clk_at_attr_clock\": %.2f,\n"
      " \"fp64_tflops_fma\": %.3f}\n",
      grid, block, sms, clk / 1e3, fma_r, mul_r, add_r, div_r, sqrt_r, per_sm_clk,
      2 * fma_r / 1e12);
  return 0;
}
