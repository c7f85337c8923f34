// Where does the C3 cold-tier floor live?  (VERDICT r01 "do this" #3)
//
// The C3 cold tier is ~45 GB of pinned host memory; K8 reads ~3,400 random
// 512 B rows of it per minibatch at ~22 GB/s against a ~55 GB/s link. This
// probe separates the candidates:
//   * the access GRANULARITY the translation cost follows (rows per 4 KB
//     page, rows per 2 MB page): tells 4 KB (host IOMMU / 4 KB PTE) from
//     2 MB translation;
//   * the ENGINE: SM zero-copy loads vs the copy engines
//     (one cudaMemcpyAsync per row; r02b used a batched-copy call that this
//     pool has since closed), which share the
//     GPU page tables and the host IOMMU but not the SM-side TLBs;
//   * the REGION size (1 GB control vs the C3-sized region).
// Every launch reads FRESH random units (no translation reuse across
// launches), L2 flushed between launches, CUDA events on the stream.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cold_probe cold_probe.cu
// Run:   ./cold_probe [region_gb=45] [units=3400]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

// one warp per unit of `ubytes` (multiple of 512), 16 B streaming loads
__global__ void zc_gather(const uint4* __restrict__ src, const uint64_t* __restrict__ off,
                          uint64_t n, uint32_t ubytes, uint4* __restrict__ dst) {
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t v = ubytes / 16;
  for (uint64_t i = w; i < n; i += nw) {
    const uint4* s = src + off[i] / 16;
    uint4* d = dst + i * v;
    for (uint32_t k = lane; k < v; k += 32) d[k] = __ldcs(s + k);
  }
}

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t rnd() {
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 7;
  rng_state ^= rng_state << 17;
  return rng_state;
}

enum Pattern { kRow512, kPair4K, kPage4K, kSame2M, kSeq };
static const char* pname[] = {"random 512 B rows", "2 rows / random 4 KB page",
                              "8 rows = whole random 4 KB page", "8 rows / random 2 MB page",
                              "sequential 512 B rows"};

// unit byte offsets for one launch; every unit is 512 B (kPage4K: 4 KB)
static void make_units(Pattern p, uint64_t region, uint64_t units, std::vector<uint64_t>& off,
                       uint32_t* ubytes) {
  off.clear();
  *ubytes = p == kPage4K ? 4096 : 512;
  static uint64_t seq = 0;
  while (off.size() < units) {
    switch (p) {
      case kRow512: off.push_back((rnd() % (region / 512)) * 512); break;
      case kPair4K: {
        const uint64_t pg = (rnd() % (region / 4096)) * 4096;
        off.push_back(pg);
        off.push_back(pg + 2048);
        break;
      }
      case kPage4K: off.push_back((rnd() % (region / 4096)) * 4096); break;
      case kSame2M: {
        const uint64_t big = (rnd() % (region >> 21)) << 21;
        for (int k = 0; k < 8; ++k) off.push_back(big + (rnd() % 512) * 4096);
        break;
      }
      case kSeq: off.push_back(seq); seq = (seq + 512) % region; break;
    }
  }
  off.resize(units);
}

struct Res {
  double us, gbps;
};

static Res run(Pattern p, bool ce, const uint8_t* host_dev, const uint8_t* host_ptr, uint64_t region,
               uint64_t units, void* flush, uint8_t* dst, uint64_t* off_d, cudaStream_t st) {
  const int launches = 24;
  double tot = 0;
  uint64_t bytes = 0;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::vector<uint64_t> off;
  std::vector<void*> dsts(units), srcs(units);
  std::vector<size_t> sizes(units);
  for (int l = 0; l < launches + 1; ++l) {
    uint32_t ub;
    make_units(p, region, units, off, &ub);
    CK(cudaMemcpyAsync(off_d, off.data(), 8 * units, cudaMemcpyHostToDevice, st));
    if (ce)
      for (uint64_t i = 0; i < units; ++i) {
        dsts[i] = dst + i * ub;
        srcs[i] = const_cast<uint8_t*>(host_ptr + off[i]);
        sizes[i] = ub;
      }
    CK(cudaMemsetAsync(flush, l & 0xff, 256u << 20, st));
    CK(cudaEventRecord(a, st));
    if (ce) {
      for (uint64_t i = 0; i < units; ++i)
        CK(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyHostToDevice, st));
    } else {
      zc_gather<<<148 * 8, 256, 0, st>>>(reinterpret_cast<const uint4*>(host_dev), off_d, units, ub,
                                         reinterpret_cast<uint4*>(dst));
    }
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (l) {
      tot += ms;
      bytes += units * ub;
    }
  }
  CK(cudaGetLastError());
  Res r;
  r.us = tot / launches * 1e3;
  r.gbps = bytes / (tot * 1e-3) / 1e9;
  return r;
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 45.0;
  const uint64_t units = argc > 2 ? strtoull(argv[2], nullptr, 10) : 3400;
  CK(cudaSetDevice(0));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const uint64_t big = static_cast<uint64_t>(gb * (1ull << 30)) & ~((1ull << 21) - 1);
  uint8_t* h = nullptr;
  CK(cudaHostAlloc(reinterpret_cast<void**>(&h), big, cudaHostAllocMapped | cudaHostAllocPortable));
  // touch every page (first-touch) in parallel-ish chunks
  for (uint64_t o = 0; o < big; o += 4096) h[o] = static_cast<uint8_t>(o >> 12);
  uint8_t* hd = nullptr;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd), h, 0));
  void* flush;
  CK(cudaMalloc(&flush, 256u << 20));
  uint8_t* dst;
  CK(cudaMalloc(&dst, units * 4096));
  uint64_t* off_d;
  CK(cudaMalloc(&off_d, units * 8));
  // link reference: one contiguous DMA of the same bytes
  {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(a, st));
      CK(cudaMemcpyAsync(dst, h + (r + 1) * (64ull << 20), units * 4096, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    printf("link: contiguous DMA H2D of %.1f MB: %.1f GB/s\n", units * 4096 / 1e6,
           units * 4096 / (best * 1e-3) / 1e9);
  }
  const uint64_t regions[2] = {1ull << 30, big};
  for (uint64_t region : regions) {
    printf("--- region %.1f GB, %lu units per launch\n", region / double(1ull << 30),
           (unsigned long)units);
    for (int p = 0; p < 5; ++p)
      for (int ce = 0; ce < 2; ++ce) {
        Res r = run(static_cast<Pattern>(p), ce, hd, h, region, units, flush, dst, off_d, st);
        printf("  %-34s %-4s %8.1f us/launch  %6.1f GB/s  %6.1f units/us\n", pname[p],
               ce ? "CE" : "SM", r.us, r.gbps, units / r.us);
        fflush(stdout);
      }
  }
  return 0;
}
