// FP64 latency / throughput microbenchmark (measurement only, not part of the library):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/fp64_latency.cu && /tmp/lat
// B200 (round 2): DFMA and DADD dependent latency 8.06 cycles; one dependent chain per warp
// reaches 17.7 / 34.9 / 36.3 TFLOP/s at 8 / 16 / 32 warps per SM (8 chains per warp: 30.3 TFLOP/s
// at 4 warps per SM) -- 4 independent DFMA in flight per scheduler saturate the fp64 pipe.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, double a, double b, int iters, long long* cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void dadd_chain(double* out, double a, int iters, long long* cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __dadd_rn(x, a);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
// throughput: ILP 8 independent chains per thread, many warps
__global__ void dfma_tput(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}
// issue rate with N warps per SM, each a single dependent DFMA chain
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
  long long h;
  int iters = 4096;
  dfma_chain<<<1, 32>>>(out, 1.0000001, 1e-9, iters, cyc); cudaDeviceSynchronize();
  dfma_chain<<<1, 32>>>(out, 1.0000001, 1e-9, iters, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", double(h) / (iters * 16));
  dadd_chain<<<1, 32>>>(out, 1e-9, iters, cyc); cudaDeviceSynchronize();
  dadd_chain<<<1, 32>>>(out, 1e-9, iters, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", double(h) / (iters * 16));
  // warps per SMSP sweep with one dependent chain each: cycles per DFMA per SMSP
  for (int w : {1, 2, 4, 8, 16, 32}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148;
    dfma_chain<<<blocks, 32 * w>>>(out, 1.0000001, 1e-9, iters, cyc);
    cudaEventRecord(e0);
    dfma_chain<<<blocks, 32 * w>>>(out, 1.0000001, 1e-9, iters, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * 32 * w * double(iters) * 16;
    printf("warps/SM %2d (1 chain each): %.2f TFLOP/s\n", w, flops / ms / 1e9);
  }
  for (int w : {4, 8, 16, 32}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148;
    dfma_tput<<<blocks, 32 * w>>>(out, 1.0000001, 1e-9, iters);
    cudaEventRecord(e0);
    dfma_tput<<<blocks, 32 * w>>>(out, 1.0000001, 1e-9, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * 32 * w * double(iters) * 8;
    printf("warps/SM %2d (8 chains each): %.2f TFLOP/s\n", w, flops / ms / 1e9);
  }
  return 0;
}
