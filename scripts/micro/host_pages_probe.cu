// Does the HOST page size of the cold tier change its translation cost?
//
// cold_probe.cu (profiles/r02a) showed that a zero-copy read of random 512 B
// rows over a 45 GB pinned region costs per distinct 4 KB page and grows with
// the region size, whatever the GPU-side mapping granularity; the box's guest
// kernel runs its IOMMU in "Translated" mode (dmesg). If the IOMMU maps a
// physically contiguous huge page with one large IOTLB entry, a cold tier on
// 2 MB or 1 GB host pages would escape the per-4 KB-page cost. Modes:
//   A   cudaHostAlloc(Mapped|Portable)                  (the store's default)
//   T   mmap + MADV_HUGEPAGE (THP) + cudaHostRegister
//   H2  mmap(MAP_HUGETLB, 2 MB pages) + cudaHostRegister (reserves pages)
//   H1  mmap(MAP_HUGETLB | 1 GB pages) + cudaHostRegister (reserves pages)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_pages_probe host_pages_probe.cu
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#ifndef MAP_HUGE_SHIFT
#define MAP_HUGE_SHIFT 26
#endif

__global__ void zc_rows(const uint4* __restrict__ src, const uint64_t* __restrict__ rows, uint64_t n,
                        uint4* __restrict__ dst) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w; i < n; i += nw) dst[i * 32 + lane] = __ldcs(src + rows[i] * 32 + lane);
}

static void meminfo() {
  FILE* f = fopen("/proc/meminfo", "r");
  char line[256];
  while (f && fgets(line, sizeof line, f))
    if (!strncmp(line, "AnonHugePages", 13) || !strncmp(line, "HugePages_", 10) ||
        !strncmp(line, "Hugetlb", 7))
      printf("   %s", line);
  if (f) fclose(f);
}

static void sysw(const char* path, long v) {
  FILE* f = fopen(path, "w");
  if (!f) {
    printf("   cannot open %s\n", path);
    return;
  }
  fprintf(f, "%ld\n", v);
  fclose(f);
  f = fopen(path, "r");
  long got = -1;
  if (f && fscanf(f, "%ld", &got) == 1) printf("   %s = %ld (asked %ld)\n", path, got, v);
  if (f) fclose(f);
}

static void run(const char* name, uint8_t* h, uint64_t bytes, bool registered) {
  if (!h) {
    printf("%-4s allocation failed\n", name);
    return;
  }
  for (uint64_t o = 0; o < bytes; o += 4096) h[o] = static_cast<uint8_t>(o >> 12);
  if (registered) {
    cudaError_t e = cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      printf("%-4s cudaHostRegister failed: %s\n", name, cudaGetErrorString(e));
      cudaGetLastError();
      return;
    }
  }
  uint8_t* hd = nullptr;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd), h, 0);
  meminfo();
  const uint64_t nrows = bytes / 512, per = 3400, launches = 30;
  uint64_t *rows_d;
  uint4* dst;
  void* flush;
  cudaMalloc(&rows_d, 8 * per * launches);
  cudaMalloc(&dst, 512 * per);
  cudaMalloc(&flush, 256u << 20);
  std::vector<uint64_t> rows(per * launches);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (auto& r : rows) {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    r = s % nrows;
  }
  cudaMemcpy(rows_d, rows.data(), 8 * rows.size(), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double tot = 0;
  for (uint64_t l = 0; l < launches; ++l) {
    cudaMemsetAsync(flush, l & 0xff, 256u << 20);
    cudaEventRecord(a);
    zc_rows<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(hd), rows_d + l * per, per, dst);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (l) tot += ms;
  }
  const double us = tot / (launches - 1) * 1e3;
  printf("%-4s %5.1f GB region, %lu random 512 B rows per launch: %7.1f us -> %5.1f GB/s, %5.1f rows/us [%s]\n",
         name, bytes / double(1ull << 30), (unsigned long)per, us, per * 512.0 / (us * 1e-6) / 1e9,
         per / us, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaFree(rows_d);
  cudaFree(dst);
  cudaFree(flush);
  if (registered) cudaHostUnregister(h);
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 45.0;
  const uint64_t bytes = static_cast<uint64_t>(gb * (1ull << 30)) & ~((1ull << 30) - 1);
  cudaSetDevice(0);
  {
    uint8_t* h = nullptr;
    cudaHostAlloc(reinterpret_cast<void**>(&h), bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    run("A", h, bytes, false);
    cudaFreeHost(h);
  }
  {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p != MAP_FAILED) madvise(p, bytes, MADV_HUGEPAGE);
    run("T", p == MAP_FAILED ? nullptr : static_cast<uint8_t*>(p), bytes, true);
    if (p != MAP_FAILED) munmap(p, bytes);
  }
  {
    sysw("/proc/sys/vm/nr_hugepages", static_cast<long>(bytes >> 21));
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE,
                   MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB | MAP_POPULATE, -1, 0);
    if (p == MAP_FAILED) perror("   mmap 2MB hugetlb");
    run("H2", p == MAP_FAILED ? nullptr : static_cast<uint8_t*>(p), bytes, true);
    if (p != MAP_FAILED) munmap(p, bytes);
    sysw("/proc/sys/vm/nr_hugepages", 0);
  }
  {
    sysw("/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages", static_cast<long>(bytes >> 30));
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE,
                   MAP_PRIVATE | MAP_ANONYMOUS | MAP_HUGETLB | (30 << MAP_HUGE_SHIFT) | MAP_POPULATE,
                   -1, 0);
    if (p == MAP_FAILED) perror("   mmap 1GB hugetlb");
    run("H1", p == MAP_FAILED ? nullptr : static_cast<uint8_t*>(p), bytes, true);
    if (p != MAP_FAILED) munmap(p, bytes);
    sysw("/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages", 0);
  }
  return 0;
}
