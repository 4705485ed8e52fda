// L2-hit load latency (pointer chase over a buffer larger than L1, smaller
// than L2) and the latency of a volatile load and of an ld.global.cg load.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>

__global__ void chase(const unsigned* __restrict__ next, int steps, unsigned* out, long long* cyc) {
  unsigned p = 0;
  // warm: one pass
  for (int i = 0; i < steps; ++i) p = next[p];
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = (t1 - t0) / steps;
}

int main() {
  const int n = 4 << 20;  // 16 MiB of u32, 128-B strided permutation
  const int stride = 32;
  std::vector<unsigned> h(n, 0);
  std::vector<unsigned> idx(n / stride);
  for (unsigned i = 0; i < idx.size(); ++i) idx[i] = i * stride;
  std::shuffle(idx.begin() + 1, idx.end(), std::mt19937(1));
  for (size_t i = 0; i < idx.size(); ++i) h[idx[i]] = idx[(i + 1) % idx.size()];
  unsigned *d, *out; long long* cyc;
  cudaMalloc(&d, n * 4); cudaMalloc(&out, 4); cudaMallocManaged(&cyc, 8);
  cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) {
    chase<<<1, 1>>>(d, 20000, out, cyc);
    cudaDeviceSynchronize();
    printf("L2 hit (ld.global.cg) pointer-chase latency: %lld cycles\n", cyc[0]);
  }
  return 0;
}
