// Host<->HBM copy rates of pageable memory: the library's pinned ring
// (mdgemm::h2d_copy / d2h_copy) vs the driver's pageable cudaMemcpyAsync vs
// a pinned buffer.  tools/copy_probe [MB ...]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

namespace mdgemm {
void h2d_copy(void* dst, const void* src, size_t n, cudaStream_t st);
void d2h_copy(void* dst, const void* src, size_t n, cudaStream_t st);
}

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char** argv) {
  std::vector<size_t> sizes;
  for (int i = 1; i < argc; ++i) sizes.push_back(std::strtoull(argv[i], nullptr, 10) << 20);
  if (sizes.empty()) sizes = {size_t(1) << 20, size_t(4) << 20, size_t(16) << 20, size_t(64) << 20, size_t(256) << 20};
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (size_t n : sizes) {
    std::vector<char> h(n, 1), h2(n, 0);
    void* d = nullptr;
    void* pin = nullptr;
    cudaMalloc(&d, n);
    cudaHostAlloc(&pin, n, 0);
    const int reps = n < (size_t(16) << 20) ? 20 : 5;
    auto rate = [&](auto fn) {
      fn();
      cudaStreamSynchronize(st);
      const double t0 = now();
      for (int r = 0; r < reps; ++r) fn();
      cudaStreamSynchronize(st);
      return n * reps / (now() - t0) / 1e9;
    };
    const double ring_in = rate([&] { mdgemm::h2d_copy(d, h.data(), n, st); });
    const double ring_out = rate([&] { mdgemm::d2h_copy(h2.data(), d, n, st); });
    const double drv_in = rate([&] { cudaMemcpyAsync(d, h.data(), n, cudaMemcpyHostToDevice, st); });
    const double drv_out = rate([&] { cudaMemcpyAsync(h2.data(), d, n, cudaMemcpyDeviceToHost, st); });
    const double pin_in = rate([&] { cudaMemcpyAsync(d, pin, n, cudaMemcpyHostToDevice, st); });
    const double pin_out = rate([&] { cudaMemcpyAsync(pin, d, n, cudaMemcpyDeviceToHost, st); });
    const double t0 = now();
    for (int r = 0; r < reps; ++r) std::memcpy(h2.data(), h.data(), n);
    const double mc = n * reps / (now() - t0) / 1e9;
    std::printf("%6zu MB  ring H2D %6.1f D2H %6.1f | driver pageable H2D %6.1f D2H %6.1f | pinned H2D %6.1f D2H %6.1f | "
                "1-thread memcpy %5.1f GB/s\n",
                n >> 20, ring_in, ring_out, drv_in, drv_out, pin_in, pin_out, mc);
    cudaFree(d);
    cudaFreeHost(pin);
  }
  return 0;
}
