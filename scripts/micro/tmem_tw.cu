// Twiddles from TMEM (tcgen05.ld) vs shared memory for the field pass while
// the other row-group runs its shared-memory exchange.
#include <cstdio>
#include "afd_fft.cuh"
using namespace afd;

__device__ __forceinline__ void tm_ld4(uint32_t taddr, double2& a) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  a.x = __hiloint2double(r1, r0);
  a.y = __hiloint2double(r3, r2);
}

// stage-wise TMEM twiddle source for pass 1 (K=12): slot (1<<q)-1+kk, 4 words each
struct TmemTw {
  uint32_t base;  // taddr of this thread's lane, column 0 of its set
  __device__ __forceinline__ double2 operator()(int b, int k) const {
    const int q = b - 4, kk = k >> 4;
    double2 w;
    tm_ld4(base + 4 * ((1 << q) - 1 + kk), w);
    return w;
  }
};

template <int MODE, bool EXCH>  // MODE 0 smem twiddles, 1 TMEM twiddles
__global__ void __launch_bounds__(512, 1) k(double* out, int reps) {
  constexpr int K = 12;
  using G = Geo<K, 4>;
  extern __shared__ double2 sm[];
  double2* tw = sm;                       // SmemTw image (2544 entries)
  double2* buf = sm + 2560;               // group 1 exchange buffer (4608 slots)
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 2560; i += blockDim.x) tw[i] = make_double2(0.7 + 1e-4 * i, 0.3 - 1e-4 * i);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((unsigned)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int g = threadIdx.x / 256, tp = threadIdx.x % 256;
  const uint32_t my = tbase + ((uint32_t)((warp % 4) * 32) << 16) + (uint32_t)(((warp % 8) / 4) * 120);
  if (g == 0) {  // fill: pass-1 twiddles of logical thread tp, 15 slots
    const SmemTw<K, 4> T{tw};
    for (int q = 0; q < 4; ++q)
      for (int kk = 0; kk < (1 << q); ++kk) {
        const double2 w = T(4 + q, (tp & 15) | (kk << 4));
        const uint32_t c = my + 4 * ((1 << q) - 1 + kk);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(c),
                     "r"(__double2loint(w.x)), "r"(__double2hiint(w.x)), "r"(__double2loint(w.y)),
                     "r"(__double2hiint(w.y)));
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  double2 v[16];
  for (int i = 0; i < 16; ++i) v[i] = make_double2(1.0 + i + tp, 0.5 * i);
  long long t0 = clock64();
  if (g == 0) {
    for (int r = 0; r < reps; ++r) {
      if (MODE == 0) fft_pass<K, 4, 1, true>(v, tp, SmemTw<K, 4>{tw});
      else fft_pass<K, 4, 1, true>(v, tp, TmemTw{my});
      asm volatile("" ::: "memory");
    }
  } else if (EXCH) {
    const int t0r = brev_bits(tp, G::TB);
    for (int r = 0; r < reps; ++r) {
      pass_store<K, 4, 0>(v, t0r, buf);
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
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

template <int A, bool B>
void run(double* out, const char* name) {
  const int smem = (2560 + 4608) * 16;
  cudaFuncSetAttribute(k<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<A, B><<<148, 512, smem>>>(out, 400);
  cudaError_t e = cudaDeviceSynchronize();
  double c[2];
  cudaMemcpy(c, out + 100000, 16, cudaMemcpyDeviceToHost);
  printf("%-42s pass %.0f cyc, exchange %.0f cyc/iter  [%s]\n", name, c[0], c[1], cudaGetErrorString(e));
}

int main() {
  double* out;
  cudaMalloc(&out, 8 << 20);
  run<0, false>(out, "smem twiddles, alone");
  run<0, true>(out, "smem twiddles, concurrent exchange");
  run<1, false>(out, "TMEM twiddles, alone");
  run<1, true>(out, "TMEM twiddles, concurrent exchange");
  return 0;
}
