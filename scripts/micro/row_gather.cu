// Microbenchmark: random 512 B row reads (one warp per row, 16 B per lane)
// from a region of S bytes in HBM or in pinned mapped host memory — does the
// gather rate fall with the region size (GPU TLB reach)? Rows read: 115k per
// launch (a C3 minibatch), into a contiguous HBM output.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o row_gather row_gather.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void gather_rows(const uint4* __restrict__ src, const uint64_t* __restrict__ rows,
                            uint64_t n, uint4* __restrict__ dst) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w; i < n; i += nw) dst[i * 32 + lane] = __ldcs(src + rows[i] * 32 + lane);
}

int main() {
  const uint64_t n = 115000;
  uint64_t* rows_d; uint4* dst;
  cudaMalloc(&rows_d, 8 * n); cudaMalloc(&dst, 512 * n);
  uint64_t* rows = (uint64_t*)malloc(8 * n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double sizes_gb[] = {0.25, 1, 4, 11.4, 32};
  for (int host = 0; host < 2; ++host) {
    for (double gb : sizes_gb) {
      const uint64_t bytes = (uint64_t)(gb * (1ull << 30)) / 512 * 512, nrows = bytes / 512;
      void* buf = nullptr; const uint4* src = nullptr;
      if (host) {
        if (cudaHostAlloc(&buf, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) { printf("host alloc %.1f GB failed\n", gb); continue; }
        void* dp; cudaHostGetDevicePointer(&dp, buf, 0); src = (const uint4*)dp;
      } else {
        if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("dev alloc failed\n"); continue; }
        cudaMemset(buf, 1, bytes); src = (const uint4*)buf;
      }
      uint64_t s = 88172645463325252ull ^ (uint64_t)(gb * 1000);
      for (uint64_t i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; rows[i] = s % nrows; }
      cudaMemcpy(rows_d, rows, 8 * n, cudaMemcpyHostToDevice);
      float best = 1e9;
      for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a);
        gather_rows<<<148 * 16, 256>>>(src, rows_d, n, dst);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
      }
      printf("%s region %6.2f GB: %8.1f us for %llu random 512 B rows -> %7.1f GB/s\n",
             host ? "host-mapped" : "HBM        ", gb, best * 1e3, (unsigned long long)n,
             n * 512.0 / (best * 1e-3) / 1e9);
      if (host) cudaFreeHost(buf); else cudaFree(buf);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
