// Microbenchmark: does the way the cold tier is pinned change the GPU's
// address-translation cost for random 512 B zero-copy row reads over a 57 GB
// host region (the C3 cold tier)? 3,400 NEW rows per launch (the cold share
// of one C3 minibatch), L2 flushed between launches like the bench.
//   A  cudaHostAlloc(Mapped|Portable)                    (4 KB host pages)
//   B  mmap + MADV_HUGEPAGE + cudaHostRegister           (THP, if it engages)
//   V  cuMemCreate(HOST_NUMA) + cuMemMap + cuMemSetAccess (VMM host allocation,
//      granularity-sized physically contiguous chunks)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o host_vmm host_vmm.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void gather_rows(const uint4* __restrict__ src, const uint64_t* __restrict__ rows,
                            uint64_t n, uint4* __restrict__ dst) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = w; i < n; i += nw) dst[i * 32 + lane] = __ldcs(src + rows[i] * 32 + lane);
}

static void* g_flush;

static void run(const char* name, const void* dp, uint64_t bytes, uint64_t per) {
  const uint64_t nrows = bytes / 512, launches = 40;
  uint64_t* rows_d; uint4* dst;
  cudaMalloc(&rows_d, 8 * per * launches); cudaMalloc(&dst, 512 * per);
  uint64_t* rows = (uint64_t*)malloc(8 * per * launches);
  uint64_t s = 0x9E3779B97F4A7C15ull;
  for (uint64_t i = 0; i < per * launches; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; rows[i] = s % nrows; }
  cudaMemcpy(rows_d, rows, 8 * per * launches, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double tot = 0, mn = 1e9;
  for (uint64_t l = 0; l < launches; ++l) {
    cudaMemsetAsync(g_flush, l & 0xff, 256u << 20);
    cudaEventRecord(a);
    gather_rows<<<148 * 8, 256>>>((const uint4*)dp, rows_d + l * per, per, dst);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (l) { tot += ms; if (ms < mn) mn = ms; }
  }
  double warm = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaMemsetAsync(g_flush, r, 256u << 20);
    cudaEventRecord(a);
    gather_rows<<<148 * 8, 256>>>((const uint4*)dp, rows_d + per, per, dst);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < warm) warm = ms;
  }
  printf("%-30s %6lu rows/launch: new rows avg %7.1f us (min %6.1f) -> %5.1f GB/s | same rows again %6.1f us  [%s]\n",
         name, (unsigned long)per, tot / (launches - 1) * 1e3, mn * 1e3,
         per * 512.0 / (tot / (launches - 1) * 1e-3) / 1e9, warm * 1e3,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
  cudaFree(rows_d); cudaFree(dst); free(rows);
}

static void anon_huge() {
  FILE* f = fopen("/proc/meminfo", "r");
  char line[256];
  while (f && fgets(line, sizeof line, f))
    if (!strncmp(line, "AnonHugePages", 13) || !strncmp(line, "HugePages_T", 11)) printf("   %s", line);
  if (f) fclose(f);
}

#define CU(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* m; cuGetErrorString(r_, &m); printf("%s failed: %s\n", #x, m); return; } } while (0)

static void vmm(uint64_t bytes, bool recommended) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  p.location.id = 0;
  size_t gmin = 0, grec = 0;
  CU(cuMemGetAllocationGranularity(&gmin, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CU(cuMemGetAllocationGranularity(&grec, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = recommended ? grec : gmin;
  printf("V granularity: minimum %zu, recommended %zu\n", gmin, grec);
  bytes = (bytes + g - 1) / g * g;
  CUmemGenericAllocationHandle h;
  CU(cuMemCreate(&h, bytes, &p, 0));
  CUdeviceptr va;
  CU(cuMemAddressReserve(&va, bytes, 1ull << 30, 0, 0));
  CU(cuMemMap(va, bytes, 0, h, 0));
  CUmemAccessDesc d[2]{};
  d[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d[0].location.id = 0;
  d[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  d[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  d[1].location.id = 0;
  d[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(va, bytes, d, 2));
  // the host writes through the same address (the feature fill)
  memset(reinterpret_cast<void*>(va), 1, 1 << 20);
  printf("V host write ok\n");
  run("V cuMemCreate(HOST_NUMA)", reinterpret_cast<void*>(va), bytes, 3400);
  run("V cuMemCreate(HOST_NUMA)", reinterpret_cast<void*>(va), bytes, 115000);
  cuMemUnmap(va, bytes);
  cuMemAddressFree(va, bytes);
  cuMemRelease(h);
}

int main(int argc, char** argv) {
  const uint64_t bytes = (uint64_t)(argc > 1 ? atof(argv[1]) : 57.0) * (1ull << 30) / 4096 * 4096;
  const char* which = argc > 2 ? argv[2] : "AVB";
  cudaFree(0);
  cudaMalloc(&g_flush, 256u << 20);
  if (strchr(which, 'V')) vmm(bytes, false);
  if (strchr(which, 'A')) {
    void* h = nullptr;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
      void* dp; cudaHostGetDevicePointer(&dp, h, 0);
      run("A cudaHostAlloc", dp, bytes, 3400);
      run("A cudaHostAlloc", dp, bytes, 115000);
      cudaFreeHost(h);
    } else printf("A alloc failed\n");
  }
  if (strchr(which, 'B')) {
    void* h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (h != MAP_FAILED) {
      madvise(h, bytes, MADV_HUGEPAGE);
      memset(h, 1, bytes);
      anon_huge();
      if (cudaHostRegister(h, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        void* dp; cudaHostGetDevicePointer(&dp, h, 0);
        run("B mmap+THP+cudaHostRegister", dp, bytes, 3400);
        cudaHostUnregister(h);
      } else printf("B register failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      munmap(h, bytes);
    }
  }
  return 0;
}
