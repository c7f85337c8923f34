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

}  // namespace tgb
