// Microbenchmark: zero-copy random 512 B row reads from a large pinned host
// region (57 GB ~ the C3 feature matrix), 3,400 NEW rows per launch (the
// cold share of a C3 minibatch) — how host memory is pinned decides the GPU's
// address-translation cost:
//   A cudaHostAlloc(Mapped|Portable)
//   B mmap + madvise(MADV_HUGEPAGE) (THP, 2 MB host pages) + cudaHostRegister
//   C mmap(MAP_HUGETLB) (hugetlbfs 2 MB) + cudaHostRegister, if pages exist
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_pages host_pages.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <cuda_runtime.h>

__global__ void gather_rows(const uint4* __restrict__ src, const uint64_t* __restrict__ rows,
                            uint64_t n, uint4* __restrict__ dst) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w; i < n; i += nw) dst[i * 32 + lane] = __ldcs(src + rows[i] * 32 + lane);
}

static void run(const char* name, void* host, uint64_t bytes) {
  void* dp = nullptr;
  if (cudaHostGetDevicePointer(&dp, host, 0) != cudaSuccess) { printf("%s: no device pointer\n", name); return; }
  const uint64_t nrows = bytes / 512, per = 3400, launches = 40;
  uint64_t* rows_d; uint4* dst;
  cudaMalloc(&rows_d, 8 * per * launches); cudaMalloc(&dst, 512 * per);
  uint64_t* rows = (uint64_t*)malloc(8 * per * launches);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (uint64_t i = 0; i < per * launches; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; rows[i] = s % nrows; }
  cudaMemcpy(rows_d, rows, 8 * per * launches, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double tot = 0, mn = 1e9;
  for (uint64_t l = 0; l < launches; ++l) {
    cudaEventRecord(a);
    gather_rows<<<148 * 8, 256>>>((const uint4*)dp, rows_d + l * per, per, dst);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (l) { tot += ms; if (ms < mn) mn = ms; }
  }
  // the same rows again: translations now warm
  double warm = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    gather_rows<<<148 * 8, 256>>>((const uint4*)dp, rows_d + per, per, dst);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < warm) warm = ms;
  }
  printf("%-34s new rows: avg %7.1f us (min %6.1f)  -> %5.1f GB/s | same rows again %6.1f us\n", name,
         tot / (launches - 1) * 1e3, mn * 1e3, per * 512.0 / (tot / (launches - 1) * 1e-3) / 1e9, warm * 1e3);
  cudaFree(rows_d); cudaFree(dst); free(rows);
}

int main(int argc, char** argv) {
  const uint64_t bytes = (uint64_t)(argc > 1 ? atof(argv[1]) : 57.0) * (1ull << 30) / 4096 * 4096;
  {
    void* h = nullptr;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
      run("A cudaHostAlloc", h, bytes); cudaFreeHost(h);
    } else printf("A alloc failed\n");
  }
  {
    void* h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h != MAP_FAILED) {
      madvise(h, bytes, MADV_HUGEPAGE);
      memset(h, 1, bytes);
      if (cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        run("B mmap+THP+cudaHostRegister", h, bytes); cudaHostUnregister(h);
      } else printf("B register failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      munmap(h, bytes);
    }
  }
  {
    void* h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB, -1, 0);
    if (h != MAP_FAILED) {
      memset(h, 1, bytes);
      if (cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        run("C hugetlb+cudaHostRegister", h, bytes); cudaHostUnregister(h);
      } else printf("C register failed\n");
      munmap(h, bytes);
    } else printf("C: no hugetlb pages reserved\n");
  }
  return 0;
}
