// FP64 pipe probe: throughput vs independent chains per thread and warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, int OP>
__global__ void k(double* out, double s, int iters) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = s + threadIdx.x * 1e-9 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (OP == 0) a[i] = fma(a[i], b, c);
      else if (OP == 1) a[i] = a[i] * b;
      else a[i] = a[i] + c;
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) t += a[i];
  if (t == 1.2345) out[0] = t;
}
template <int CH, int OP>
void run(int warps_per_sm, double* out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  int blocks = sms * (warps_per_sm * 32 / threads);
  int iters = 1 << 14;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH, OP><<<blocks, threads>>>(out, 1.0, iters);
  cudaEventRecord(e0);
  k<CH, OP><<<blocks, threads>>>(out, 1.0, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * CH;
  double flops = ops * (OP == 0 ? 2 : 1);
  // per-SM cycles per warp-instruction at ~1.9 GHz
  printf("op=%s chains=%2d warps/SM=%2d  %.2f Tops/s  (%.1f TF/s)\n", OP == 0 ? "DFMA" : OP == 1 ? "DMUL" : "DADD",
         CH, warps_per_sm, ops / (ms * 1e-3) / 1e12, flops / (ms * 1e-3) / 1e12);
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 16, 32, 64}) { run<1, 0>(w, out); run<2, 0>(w, out); run<4, 0>(w, out); run<6, 0>(w, out); run<8, 0>(w, out); run<12, 0>(w, out); run<16, 0>(w, out); }
  run<8, 1>(32, out); run<8, 2>(32, out); run<8, 1>(64, out); run<8, 2>(64, out);
  return 0;
}
