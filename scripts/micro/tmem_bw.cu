// tmem_bw.cu — tcgen05.ld (LDTM) read throughput per SM: W warps of one CTA per SM loop over
// .32x32b.xN loads of their lane quadrant (N = 8, 16, 32), optionally beside FP64 work.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NW>
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t (&r)[NW]);
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t a, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(a));
}
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t a, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(a));
}
template <>
__device__ __forceinline__ void tm_ld<32>(uint32_t a, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(a));
}

// FMA > 0: that many dependent-free DFMAs per load per thread (8 accumulators)
template <int NW, int FMA>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned* sink, double* dsink, long long* cyc) {
  __shared__ uint32_t tm_base;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tm_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  const uint32_t base = tm_base + ((uint32_t)((warp & 3) * 32) << 16);
  unsigned acc = 0;
  double d[8];
  for (int i = 0; i < 8; ++i) d[i] = 1.0 + threadIdx.x * 1e-9 + i;
  const double m = 1.0000000001, c = 1e-12;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t r[NW];
      tm_ld<NW>(base + ((it * 4 + u) * NW) % (512 - NW + 1) / NW * NW, r);
#pragma unroll
      for (int f = 0; f < FMA; ++f) d[f & 7] = fma(d[f & 7], m, c);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < NW; ++i) acc ^= r[i];
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i];
  if (s == 0.123) dsink[0] = s;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base) : "memory");
}

template <int NW, int FMA>
void run(int warps, int sms) {
  unsigned* sink;
  double* dsink;
  long long* cyc;
  cudaMalloc(&sink, 4);
  cudaMalloc(&dsink, 8);
  cudaMalloc(&cyc, 8 * sms);
  const int iters = 2000;
  k<NW, FMA><<<sms, warps * 32>>>(10, sink, dsink, cyc);
  k<NW, FMA><<<sms, warps * 32>>>(iters, sink, dsink, cyc);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaDeviceSynchronize();
  const double bytes = (double)iters * 4 * NW * 4 * 32 * warps;
  printf("x%-2d fma/ld %3d warps %2d: %8lld cycles, %6.1f B/clk/SM TMEM read, %5.1f DFMA/clk/SM  %s\n",
         NW, FMA, warps, h, bytes / h, (double)iters * 4 * FMA * 32 * warps / h,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(sink);
  cudaFree(dsink);
  cudaFree(cyc);
}

int main() {
  int sms = 148;
  for (int w : {1, 4, 8, 16}) {
    run<8, 0>(w, sms);
    run<16, 0>(w, sms);
    run<32, 0>(w, sms);
  }
  for (int w : {8, 16}) {
    run<32, 16>(w, sms);
    run<32, 32>(w, sms);
    run<32, 64>(w, sms);
    run<16, 32>(w, sms);
  }
  return 0;
}
