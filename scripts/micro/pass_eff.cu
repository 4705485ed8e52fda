// FP64 efficiency of the field kernel's register pass (16 points, 4 radix-2
// stages, twiddles from shared memory) for 1 or 2 row-groups (256 threads
// each) per SM, without exchanges: cycles per pass vs the FP64 issue bound.
#include <cstdio>
#include "afd_fft.cuh"
using namespace afd;

template <int PASS>
__global__ void __launch_bounds__(512, 1) passes(double* out, int reps) {
  constexpr int K = 12;
  __shared__ double2 tw[2600];
  for (int i = threadIdx.x; i < 2600; i += blockDim.x) tw[i] = make_double2(0.7 + 1e-4 * i, 0.3 - 1e-4 * i);
  __syncthreads();
  const SmemTw<K, 4> T{tw};
  const int tp = threadIdx.x % 256;
  double2 v[16];
  for (int i = 0; i < 16; ++i) v[i] = make_double2(1.0 + i + tp, 0.5 * i);
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    fft_pass<K, 4, PASS, true>(v, tp, T);
    asm volatile("" ::: "memory");
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += v[i].x + v[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[100000 + blockIdx.x] = (double)(t1 - t0) / reps;
}

int main() {
  double* out;
  cudaMalloc(&out, 8 << 20);
  for (int pass = 1; pass <= 2; ++pass) {
    for (int thr = 256; thr <= 512; thr += 256) {
      if (pass == 1) passes<1><<<148, thr>>>(out, 200);
      else passes<2><<<148, thr>>>(out, 200);
      cudaDeviceSynchronize();
      double cyc;
      cudaMemcpy(&cyc, out + 100000, 8, cudaMemcpyDeviceToHost);
      // FP64 instr per pass per thread: 4 stages x 8 butterflies x 8 = 256
      const double bound = (thr / 32.0) * 256 * 2 / 4;  // warps x instr x 2 cyc / 4 SMSPs
      printf("pass %d, %d threads/SM: %.0f cycles per pass, FP64 issue bound %.0f -> %.0f%%\n",
             pass, thr, cyc, bound, 100 * bound / cyc);
    }
  }
  return 0;
}
