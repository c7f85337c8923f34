// Reference point for the selection sort (K5): cub::DeviceRadixSort::SortPairs
// of (u64 key, u32 id) at the selection's sizes, on keys shaped like
// ~bits(PageRank score) (log-normal scores over ~20 binades). Not product
// code: it only says what a tuned library LSD sort reaches on this box, so
// K5's per-pass time has a yardstick.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sort_probe sort_probe.cu
// Run:   ./sort_probe [n=111000000]
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__global__ void make_keys(uint64_t* k, uint32_t* v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = i * 0x9E3779B97F4A7C15ull + 12345;
    s ^= s >> 31; s *= 0xBF58476D1CE4E5B9ull; s ^= s >> 27; s *= 0x94D049BB133111EBull; s ^= s >> 31;
    const double u1 = ((s >> 11) + 1) * (1.0 / 9007199254740993.0);
    const double u2 = (((s * 0x2545F4914F6CDD1Dull) >> 11)) * (1.0 / 9007199254740992.0);
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    const double score = 1e-8 * exp(2.5 * z);
    k[i] = ~static_cast<uint64_t>(__double_as_longlong(score));
    v[i] = static_cast<uint32_t>(i);
  }
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 111000000ull;
  uint64_t *k0, *k1;
  uint32_t *v0, *v1;
  cudaMalloc(&k0, 8 * n); cudaMalloc(&k1, 8 * n); cudaMalloc(&v0, 4 * n); cudaMalloc(&v1, 4 * n);
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DoubleBuffer<uint64_t> kb(k0, k1);
  cub::DoubleBuffer<uint32_t> vb(v0, v1);
  cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int)n);
  cudaMalloc(&tmp, tb);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bits : {64, 56, 48}) {
    float best = 1e9, sum = 0;
    for (int r = 0; r < 6; ++r) {
      make_keys<<<148 * 8, 256>>>(k0, v0, n);
      kb = cub::DoubleBuffer<uint64_t>(k0, k1);
      vb = cub::DoubleBuffer<uint32_t>(v0, v1);
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, (int)n, 64 - bits, 64);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r) { sum += ms; best = ms < best ? ms : best; }
    }
    const double gb = (double)n * 24 * ((bits + 7) / 8) / 1e9;
    printf("cub SortPairs u64/u32 n=%llu bits=%d: %.3f ms (best %.3f), %.1f GB/s over %d passes\n",
           (unsigned long long)n, bits, sum / 5, best, gb / (best * 1e-3), (bits + 7) / 8);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
