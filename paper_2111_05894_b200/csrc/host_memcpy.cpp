// Multi-threaded memcpy between pageable and pinned host memory, the host leg
// of the pipelined host<->device copies (internal.cuh: copy_h2d / copy_d2h).
// A single thread moves ~5-10 GB/s (and takes the first-touch page faults of
// a fresh destination alone); the host cores together keep up with the DMA.
#include <omp.h>

#include <cstdint>
#include <cstring>

namespace tgb {

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kSlice = 1u << 20;
  if (bytes <= 4 * kSlice) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const long long ns = static_cast<long long>((bytes + kSlice - 1) / kSlice);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < ns; ++i) {
    const size_t off = static_cast<size_t>(i) * kSlice;
    const size_t len = bytes - off < kSlice ? bytes - off : kSlice;
    std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, len);
  }
}

// dst[i] = (u32) src[i] for i < count with all cores (the host leg of
// copy_h2d_narrow: half the pinned-buffer writes and half the PCIe bytes of a
// u64 copy). Returns the first i with src[i] >= limit, or ~0 when none is:
// the vectorisable pass only flags each slice, a flagged slice is rescanned.
uint64_t parallel_narrow_u64(uint32_t* dst, const uint64_t* src, size_t count, uint64_t limit) {
  constexpr size_t kSlice = 1u << 18;  // elements per work item
  const long long ns = static_cast<long long>((count + kSlice - 1) / kSlice);
  uint64_t first = ~0ull;
#pragma omp parallel for schedule(static) reduction(min : first) if (ns > 4)
  for (long long i = 0; i < ns; ++i) {
    const size_t b = static_cast<size_t>(i) * kSlice;
    const size_t e = count - b < kSlice ? count : b + kSlice;
    bool over = false;
    for (size_t j = b; j < e; ++j) {
      const uint64_t v = src[j];
      over |= v >= limit;
      dst[j] = static_cast<uint32_t>(v);
    }
    if (over)
      for (size_t j = b; j < e; ++j)
        if (src[j] >= limit) {
          if (j < first) first = j;
          break;
        }
  }
  return first;
}

}  // namespace tgb
