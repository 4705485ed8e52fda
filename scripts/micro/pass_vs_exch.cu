// Does one row-group's shared-memory exchange slow the other group's FP64
// pass?  Group 0 runs register passes (twiddles from smem, or constant);
// group 1 runs STS/LDS exchanges of its 16 values per thread.
#include <cstdio>
#include "afd_fft.cuh"
using namespace afd;

struct ConstTw {
  __device__ __forceinline__ double2 operator()(int b, int k) const {
    return make_double2(0.7 + 1e-3 * b, 0.3 - 1e-4 * k);
  }
};

template <bool SMEM_TW, bool EXCH>
__global__ void __launch_bounds__(512, 1) k(double* out, int reps) {
  constexpr int K = 12;
  extern __shared__ double2 sm[];
  double2* tw = sm;                 // 2600 twiddles
  double2* buf = sm + 2600;         // exchange buffer of group 1 (4608 slots)
  for (int i = threadIdx.x; i < 2600; i += blockDim.x) tw[i] = make_double2(0.7 + 1e-4 * i, 0.3 - 1e-4 * i);
  __syncthreads();
  const int g = threadIdx.x / 256, tp = threadIdx.x % 256;
  double2 v[16];
  for (int i = 0; i < 16; ++i) v[i] = make_double2(1.0 + i + tp, 0.5 * i);
  long long t0 = clock64();
  if (g == 0) {
    for (int r = 0; r < reps; ++r) {
      if (SMEM_TW) fft_pass<K, 4, 1, true>(v, tp, SmemTw<K, 4>{tw});
      else fft_pass<K, 4, 1, true>(v, tp, ConstTw{});
      asm volatile("" ::: "memory");
    }
  } else if (EXCH) {
    for (int r = 0; r < reps; ++r) {
      pass_store<K, 4, 0>(v, tp, buf);
      asm volatile("bar.sync 2, 256;" ::: "memory");
      pass_load<K, 4, 1>(v, tp, buf);
      asm volatile("bar.sync 2, 256;" ::: "memory");
      v[0].x += 1e-9;
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 16; ++i) s += v[i].x + v[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (tp == 0) out[100000 + blockIdx.x * 2 + g] = (double)(t1 - t0) / reps;
}

template <bool A, bool B>
void run(double* out, const char* name) {
  const int smem = (2600 + 4608) * 16;
  cudaFuncSetAttribute(k<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<A, B><<<148, 512, smem>>>(out, 400);
  cudaDeviceSynchronize();
  double c[2];
  cudaMemcpy(c, out + 100000, 16, cudaMemcpyDeviceToHost);
  printf("%-40s pass %.0f cyc (alone ~1100), exchange %.0f cyc/iter  [%s]\n", name, c[0], c[1],
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  cudaMalloc(&out, 8 << 20);
  run<true, false>(out, "smem twiddles, no exchange");
  run<true, true>(out, "smem twiddles, concurrent exchange");
  run<false, false>(out, "const twiddles, no exchange");
  run<false, true>(out, "const twiddles, concurrent exchange");
  return 0;
}
