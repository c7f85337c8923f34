// Microbenchmark: latency of a dependent fp64 add chain (the serial part of
// K3's bit-exact row sums) in registers and fed from shared memory, per
// element, in SM cycles. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_reg(double* out, long long* cyc, int n, double x) {
  double acc = 0.0, a = x, b = x * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, (k & 1) ? a : b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  cyc[threadIdx.x] = t1 - t0;
}

__global__ void chain_smem(double* out, long long* cyc, int n) {
  __shared__ double v[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) v[i] = 1e-9 * (i + 1);
  __syncthreads();
  if (threadIdx.x) return;
  double acc = 0.0;
  long long t0 = clock64();
  double x[8], y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = v[k];
  for (int i = 0; i + 16 <= n; i += 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = v[(i + 8 + k) & 4095];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = __dadd_rn(acc, x[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = y[k];
  }
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 1024 * 8);
  const int n = 1 << 20;
  for (int rep = 0; rep < 2; ++rep) {
    chain_reg<<<1, 1>>>(out, cyc, n, 1e-9);
    cudaDeviceSynchronize();
    printf("reg chain, 1 thread : %.2f cycles/DADD\n", (double)cyc[0] / n);
    chain_reg<<<1, 32>>>(out, cyc, n, 1e-9);
    cudaDeviceSynchronize();
    printf("reg chain, 1 warp   : %.2f cycles/DADD\n", (double)cyc[0] / n);
    chain_reg<<<1, 128>>>(out, cyc, n, 1e-9);
    cudaDeviceSynchronize();
    printf("reg chain, 4 warps  : %.2f cycles/DADD (per thread chain)\n", (double)cyc[0] / n);
    chain_smem<<<1, 256>>>(out, cyc, n);
    cudaDeviceSynchronize();
    printf("smem-fed chain      : %.2f cycles/element\n", (double)cyc[0] / n);
  }
  return 0;
}
