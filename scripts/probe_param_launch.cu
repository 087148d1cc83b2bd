// Dev probe: host cost of launching a kernel with a large __grid_constant__
// parameter block (the fused marker kernel takes ~8 KB: SkinParamsN<2>)
// against a small one, and the synchronous round trip of each.
#include <chrono>
#include <cstdio>
#include <algorithm>
#include <vector>
template <int N>
struct Blob { double v[N]; };
template <int N>
__global__ void k_blob(const __grid_constant__ Blob<N> b, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = b.v[N - 1];
}
template <int N>
void run(const char* name, double* d) {
  Blob<N> b{};
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  std::vector<double> tl, tr;
  for (int k = 0; k < 2000; ++k) {
    b.v[N - 1] = k;
    const auto t0 = std::chrono::steady_clock::now();
    k_blob<N><<<444, 128, 0, s>>>(b, d);
    const auto t1 = std::chrono::steady_clock::now();
    while (cudaStreamQuery(s) == cudaErrorNotReady) {}
    const auto t2 = std::chrono::steady_clock::now();
    if (k >= 100) {
      tl.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      tr.push_back(std::chrono::duration<double, std::micro>(t2 - t0).count());
    }
  }
  std::sort(tl.begin(), tl.end());
  std::sort(tr.begin(), tr.end());
  std::printf("%s (%zu B params): launch %.2f us, launch+complete %.2f us (medians)\n", name, sizeof(Blob<N>),
              tl[tl.size() / 2], tr[tr.size() / 2]);
  cudaStreamDestroy(s);
}
int main() {
  double* d;
  cudaMalloc(&d, 8);
  run<16>("128 B", d);
  run<128>("1 KB", d);
  run<512>("4 KB", d);
  run<900>("7.2 KB", d);
  run<1800>("14.4 KB", d);
  return 0;
}
