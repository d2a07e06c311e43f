// Accuracy of the force kernels' reciprocal and reciprocal square root (csrc/kernels.cuh rcp_nr,
// rsqrt_nr) against IEEE division / square root:
// max relative error over 2^24 inputs spread over [2^-4, 2^8) (r^2 of pairs inside a cutoff).
// nvcc -gencode arch=compute_100a,code=sm_100a -o rcp_check tools/rcp_check.cu && ./rcp_check
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double rcp3(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double rsq3(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y, e * fma(0.375, e, 0.5), y);
}
__device__ __forceinline__ double seed(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__global__ void k(double* out) {
  const unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  // log-uniform over 12 octaves, 2^24 samples, irrational stride inside the octave
  const double x = exp2(-4.0 + 12.0 * (double(t) + 0.5) / 16777216.0) * (1.0 + 1e-9 * double(t % 977));
  const double ref = 1.0 / x;
  const double rs = 1.0 / sqrt(x);
  const double e3 = fabs(rcp3(x) - ref) / ref, es = fabs(rsq3(x) - rs) / rs;
  __shared__ double m3[256], ms[256];
  m3[threadIdx.x] = e3;
  ms[threadIdx.x] = es;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (threadIdx.x < s) {
      m3[threadIdx.x] = fmax(m3[threadIdx.x], m3[threadIdx.x + s]);
      ms[threadIdx.x] = fmax(ms[threadIdx.x], ms[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[2 * blockIdx.x] = m3[0], out[2 * blockIdx.x + 1] = ms[0];
}
int main() {
  const int nb = 65536;
  double* d;
  cudaMalloc(&d, sizeof(double) * 2 * nb);
  k<<<nb, 256>>>(d);
  double* h = new double[2 * nb];
  cudaMemcpy(h, d, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost);
  double a = 0, b = 0;
  for (int i = 0; i < nb; ++i) a = fmax(a, h[2 * i]), b = fmax(b, h[2 * i + 1]);
  printf("max rel error: rcp third-order step %.3e (%.2f ulp), rsqrt third-order step %.3e (%.2f ulp)\n", a,
         a / 1.11e-16, b, b / 1.11e-16);
  return cudaGetLastError() != cudaSuccess;
}
