// Micro-benchmark: a fresh 320 MB std::vector<Point2> filled from a buffer
// (what chainhull::convex_hull returns for 20M hull vertices) vs prefaulting
// its capacity with NT threads first. g++ -O2 -pthread -DNT=8 vecfault.cpp
#include <vector>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <sys/mman.h>
#include <cstdint>
struct P { double x, y; };
int main() {
  size_t n = 20000000;
  std::vector<P> src(n);
  for (size_t i = 0; i < n; ++i) src[i] = {double(i), double(i)};
  for (int it = 0; it < 3; ++it) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<P> v(src.data(), src.data() + n);
    auto t1 = std::chrono::steady_clock::now();
    std::vector<P> w; w.reserve(n);
    // parallel prefault of the capacity
    const size_t bytes = n * sizeof(P); char* b = reinterpret_cast<char*>(w.data());
#ifdef HUGE
    { uintptr_t a0 = (reinterpret_cast<uintptr_t>(b) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
      uintptr_t a1 = (reinterpret_cast<uintptr_t>(b) + bytes) & ~uintptr_t((2u << 20) - 1);
      if (a1 > a0) madvise(reinterpret_cast<void*>(a0), a1 - a0, MADV_HUGEPAGE); }
#endif
    std::vector<std::thread> th;
    for (int t = 0; t < NT; ++t) th.emplace_back([=] { for (size_t o = bytes * t / NT; o < bytes * (t + 1) / NT; o += 4096) b[o] = 0; });
    for (auto& x : th) x.join();
    auto t2 = std::chrono::steady_clock::now();
    w.assign(src.data(), src.data() + n);
    auto t3 = std::chrono::steady_clock::now();
    printf("vector(ptr,ptr+n) %.1f ms | prefault8 %.1f + assign %.1f ms\n",
      std::chrono::duration<double, std::milli>(t1 - t0).count(), std::chrono::duration<double, std::milli>(t2 - t1).count(), std::chrono::duration<double, std::milli>(t3 - t2).count());
  }
}
