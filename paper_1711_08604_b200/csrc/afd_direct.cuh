// afd_direct.cuh — the reference's "direct" engine (oracle.field_direct,
// oracle.py:51-73; core.py:381) on the device: every grid inner product by
// literal O(N) summation, O(M N^2) per field,
//     F[s][j] = sum_m G[m] * K_s[(j - m) mod N],
//     K_s[d]  = (sqrt(1 - r_s^2) / N) / (1 - r_s exp(2 pi i d / N)),
// i.e. the circular correlation np.correlate evaluates (oracle.py:69-72).
// The reference sums through np.correlate (a BLAS-style dot), whose order is
// not reproducible, so this engine matches the reference to its own engine
// agreement tolerance (test_core.py:313-326: indices identical, 1e-9
// relative), not bit for bit.  The fft engine is the bit-exact one.
//
// One CTA per (radius row, signal).  K_s is built in shared memory (padded
// so a lane-stride of 8 slots is conflict-free); each thread owns JT = 8
// consecutive outputs j0..j0+7 and slides a register window of K values
// over m: per m one shared load, one broadcast load of G[m], 8 complex FMAs.
#pragma once

#include "afd_kernels.cuh"

namespace afd {

constexpr int kDirectJT = 8;
constexpr int kDirectThreads = 256;

__host__ __device__ __forceinline__ int dpad(int x) { return x + (x >> 3); }

template <bool MATERIALIZE>
__global__ void __launch_bounds__(kDirectThreads)
direct_field_kernel(int n, const double2* __restrict__ g,   // [batch][n] remainder G_k
                    const double* __restrict__ radii, const double2* __restrict__ circle,
                    long long row0, long long row1, Cand* __restrict__ cand_out,
                    double2* __restrict__ field_out, const State* __restrict__ state) {
  extern __shared__ double2 ks[];  // dpad(n) slots
  const int sig = blockIdx.y;
  const long long s = row0 + blockIdx.x;
  pdl_wait();
  if ((state != nullptr && state[sig].stopped) || s >= row1) return;
  pdl_trigger();
  const double r = radii[s];
  const double sc = sqrt(1.0 - r * r) / (double)n;
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    const double2 z = circle[d];
    ks[dpad(d)] = np_cdiv(make_double2(sc, 0.0), make_double2(1.0 - r * z.x, 0.0 - r * z.y));
  }
  __syncthreads();
  const double2* __restrict__ gs = g + (size_t)sig * n;
  const int mask = n - 1;
  double best_mag = -1.0, best_re = 0.0, best_im = 0.0;
  int best_j = 0x7fffffff;
  for (int j0 = threadIdx.x * kDirectJT; j0 < n; j0 += blockDim.x * kDirectJT) {
    double2 acc[kDirectJT], win[kDirectJT];
#pragma unroll
    for (int t = 0; t < kDirectJT; ++t) {
      acc[t] = make_double2(0.0, 0.0);
      win[t] = ks[dpad((j0 + t) & mask)];  // K[(j0 + t - 0) mod n]
    }
    for (int m = 0; m < n; ++m) {
      const double2 gm = __ldg(gs + m);
#pragma unroll
      for (int t = 0; t < kDirectJT; ++t) {
        acc[t].x = fma(gm.x, win[t].x, fma(-gm.y, win[t].y, acc[t].x));
        acc[t].y = fma(gm.x, win[t].y, fma(gm.y, win[t].x, acc[t].y));
      }
      // slide: K[(j0 + t - (m+1))] = previous window shifted by one
#pragma unroll
      for (int t = kDirectJT - 1; t > 0; --t) win[t] = win[t - 1];
      win[0] = ks[dpad((j0 - m - 1) & mask)];
    }
#pragma unroll
    for (int t = 0; t < kDirectJT; ++t) {
      const int j = j0 + t;
      if (MATERIALIZE) {
        field_out[(size_t)(s - row0) * n + j] = acc[t];
      } else {
        const double mg = np_mag2(acc[t]);
        if (mg > best_mag) {  // j increases within and across chunks of a thread
          best_mag = mg;
          best_re = acc[t].x;
          best_im = acc[t].y;
          best_j = j;
        }
      }
    }
  }
  if (MATERIALIZE) return;
  Cand best;
  best.mag = best_mag;
  best.flat = best_mag >= 0.0 ? s * (long long)n + best_j : 0x7fffffffffffffffLL;
  best.re = best_re;
  best.im = best_im;
  __shared__ Cand red[32];
  best = warp_argmax(best);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = best;
  __syncthreads();
  if (wid == 0) {
    Cand c = lane < (int)(blockDim.x >> 5) ? red[lane] : best;
    c = warp_argmax(c);
    if (lane == 0) cand_out[(size_t)sig * gridDim.x + blockIdx.x] = c;
  }
}

}  // namespace afd
