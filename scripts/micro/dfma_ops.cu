// dfma_ops.cu — DFMA issue rate vs the number of distinct register operands per instruction
// (operand fetch / reuse cache), W warps per SM (W/4 per scheduler).
//   MODE 0: a[i] = fma(a[i], b, c)            one varying register operand (b, c shared)
//   MODE 1: a[i] = fma(x[i], b, a[i])         two varying
//   MODE 2: a[i] = fma(x[i], y[i], a[i])      three distinct register operands, no reuse
//   MODE 3: butterfly pairs  p = fma(-c, u[i], l[i]); q = fma(c, u[i], l[i])  (reuse-friendly)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double* out, double s, int iters, long long* cyc) {
  constexpr int CH = 16;
  double a[CH], x[CH], y[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = s + threadIdx.x * 1e-9 + i;
    x[i] = 1.0 + 1e-9 * (i + threadIdx.x);
    y[i] = 1.0 - 1e-9 * (i + 2 * threadIdx.x);
  }
  // runtime per-thread values: register operands, not constant-bank or immediates
  const double b = out[1 + (threadIdx.x & 1)], c = out[3 + (threadIdx.x & 1)];
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) a[i] = fma(a[i], b, c);
      else if (MODE == 1) a[i] = fma(x[i], b, a[i]);
      else if (MODE == 2) a[i] = fma(x[i], y[i], a[i]);
      else {
        const double p = fma(-b, x[i], a[i]), q = fma(b, x[i], a[i]);
        a[i] = p;
        x[i] = q;
      }
    }
  }
  const long long t1 = clock64();
  double t = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) t += a[i] + x[i] + y[i];
  if (t == 1.2345) out[0] = t;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run(int warps, double* out, long long* cyc) {
  const int iters = 1 << 13;
  k<MODE><<<148, warps * 32>>>(out, 1.0, 16, cyc);
  k<MODE><<<148, warps * 32>>>(out, 1.0, iters, cyc);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double n = (double)iters * 16 * (MODE == 3 ? 2 : 1);  // DFMAs per warp
  printf("mode %d warps/SM %2d: %.2f cycles per DFMA per warp, %.2f cycles per DFMA per scheduler\n",
         MODE, warps, h / n, h / n / (warps / 4.0));
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64);
  {
    const double h[8] = {0, 0.999999, 0.999999, 1e-7, 1e-7, 0, 0, 0};
    cudaMemcpy(out, h, 64, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 16}) {
    run<0>(w, out, cyc);
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<3>(w, out, cyc);
  }
  return 0;
}
