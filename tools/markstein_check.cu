// Exhaustive-ish check of the shared-reciprocal division used by vel()
// (csrc/swe_phys.cuh mk_div): for random (a, b) with b in the solver's depth
// range and a over a wide range of magnitudes and both signs, plus b with
// all-ones / all-zeros significands, RN(q0 + r y) must equal div.rn(a, b).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/markstein_check.cu -o /tmp/mk && /tmp/mk
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_rn(double a, double b) {
  double q;
  asm("div.rn.f64 %0, %1, %2;" : "=d"(q) : "d"(a), "d"(b));
  return q;
}
__device__ __forceinline__ double mk(double a, double b, double y) {
  if (!(fabs(a) >= 0x1p-900)) return a == 0.0 ? a : div_rn(a, b);
  const double q0 = a * y;
  const double r = fma(-b, q0, a);
  return fma(r, y, q0);
}
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
__global__ void k(uint64_t seed, long long n, unsigned long long* bad, double* ex) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t r1 = mix(seed ^ (2 * i + 1)), r2 = mix(seed + 0x9e3779b97f4a7c15ULL * (i + 7));
    // b: exponent in [2^-20, 2^14], significand random or extreme
    const int be = (int)(r1 % 35) - 20;
    uint64_t bm = r2 & 0xFFFFFFFFFFFFFULL;
    const int kind = (int)((r1 >> 40) % 8);
    if (kind == 0) bm = 0xFFFFFFFFFFFFFULL;
    if (kind == 1) bm = 0;
    if (kind == 2) bm = 0xFFFFFFFFFFFFFULL ^ ((r2 >> 20) & 0xFF);
    const double b = __longlong_as_double((long long)(((uint64_t)(1023 + be) << 52) | bm));
    // a: exponent in [2^-60, 2^20], random significand, random sign
    const int ae = (int)((r2 >> 52) % 81) - 60;
    const uint64_t am = mix(r1 ^ r2) & 0xFFFFFFFFFFFFFULL;
    const uint64_t sign = (r1 >> 63) << 63;
    const double a = __longlong_as_double((long long)(sign | ((uint64_t)(1023 + ae) << 52) | am));
    const double y = div_rn(1.0, b);
    const double q1 = div_rn(a, b), q2 = mk(a, b, y);
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) {
      const unsigned long long k2 = atomicAdd(bad, 1ULL);
      if (k2 < 4) { ex[2 * k2] = a; ex[2 * k2 + 1] = b; }
    }
  }
}
int main() {
  unsigned long long* bad; double* ex;
  cudaMallocManaged(&bad, sizeof(*bad)); cudaMallocManaged(&ex, 8 * sizeof(double));
  *bad = 0;
  const long long n = 1LL << 32;  // 4.3e9 pairs
  k<<<148 * 16, 256>>>(12345, n, bad, ex);
  cudaDeviceSynchronize();
  printf("{\"pairs\": %lld, \"mismatches\": %llu", n, *bad);
  for (unsigned long long i = 0; i < *bad && i < 4; ++i) printf(", \"ex%llu\": [%.17g, %.17g]", i, ex[2 * i], ex[2 * i + 1]);
  printf("}\n");
  return *bad ? 1 : 0;
}
