// Microbenchmark: the memory-system floor of K3's pull — E random 8-byte
// gathers from an N-double vector (L2-resident at C2: 19.6 MB) driven by a
// streamed u32 index array, summed per thread (no serial-order constraint).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather l2_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gather_sum(const uint32_t* __restrict__ idx, uint64_t e, const double* __restrict__ x,
                           double* __restrict__ out) {
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < e; i += 4 * stride) {
    const uint32_t a = idx[i], b = idx[i + stride], c = idx[i + 2 * stride], d = idx[i + 3 * stride];
    acc += __ldg(x + a) + __ldg(x + b) + __ldg(x + c) + __ldg(x + d);
  }
  for (; i < e; i += stride) acc += __ldg(x + idx[i]);
  if (acc == 1234.5) out[0] = acc;
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? atoll(argv[1]) : 2450000ull, e = argc > 2 ? atoll(argv[2]) : 47262823ull;
  uint32_t* idx; double* x; double* out;
  cudaMalloc(&idx, 4 * e); cudaMalloc(&x, 8 * n); cudaMalloc(&out, 8);
  uint32_t* h = (uint32_t*)malloc(4 * e);
  uint64_t s = 88172645463325252ull;
  for (uint64_t i = 0; i < e; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)(s % n); }
  cudaMemcpy(idx, h, 4 * e, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, 8 * n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks_per_sm : {4, 8, 16}) {
    const int grid = sms * blocks_per_sm;
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(a);
      gather_sum<<<grid, 256>>>(idx, e, x, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r && ms < best) best = ms;
    }
    printf("n=%llu e=%llu grid=%d: %.1f us  -> %.2f G gathers/s, %.0f GB/s of 32B sectors, %.0f GB/s algorithmic (4+8 B/edge)\n",
           (unsigned long long)n, (unsigned long long)e, grid, best * 1e3, e / (best * 1e-3) / 1e9,
           e * 32.0 / (best * 1e-3) / 1e9, e * 12.0 / (best * 1e-3) / 1e9);
  }
  return 0;
}
