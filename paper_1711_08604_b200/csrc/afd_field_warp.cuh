// afd_field_warp.cuh — fast-engine field + argmax for 1024-point rows, one
// warp per row (weighted_inverse_grid + maximal_selection, transform.py:185-201,
// core.py:285-300; the arithmetic of the fast engine, afd_fft.cuh "Fast mode").
//
// A 1024-point row is 32 threads x 32 points: two register passes of five
// stages each (32 x 32 = 1024) and ONE exchange through shared memory, and a
// row-group that is exactly one warp synchronises with __syncwarp — no named
// barriers.  The 16-point form (field_kernel<10, 4>: 64 threads x 16 points,
// three passes, two exchanges, bar.sync per exchange) moves 64 B per grid
// evaluation through shared memory against ~34 FP64 instructions: at 128 B
// per clock and 64 FP64 lanes per clock and SM the two pipes are loaded
// about equally and do not overlap perfectly (ncu: FP64 pipe 66% busy).
// Here the exchange traffic is 32 B per evaluation.
//
// Per CTA: 8 warps = 8 rows in flight, 128 registers of row data per thread.
// Tensor memory holds what depends on the lane only and is shared by the
// warps of a lane quadrant: the lane's 31 (c, t) twiddles of pass 1 (stage
// b = 5..9, register pair kk: S_b[lane | kk << 5], 124 columns) and the
// lane's 32 spectrum values (l = rev5(i) << 5 | lane, 128 columns) — both
// off the shared-memory path (tcgen05.ld).  Pass 0's twiddles are the 32nd
// roots of unity, compile-time constants.  The row's weights scale r^l =
// fw[lane] * fw[32 + rev5(i)] come from a 64-entry factor row; the next row's
// two factors per lane are fetched one row ahead and the second factor is
// broadcast through a 32-double shared-memory line per warp.
#pragma once

#include "afd_kernels.cuh"

namespace afd {

constexpr int kFwK = 10, kFwRB = 5, kFwWarps = 8;
using GeoW = Geo<kFwK, kFwRB>;        // N = 1024, P = 32, T = 32, two passes
constexpr int kFwStride = 64;         // factor row: scale r^t (t < 32), r^(32 m) (m < 32)
constexpr int kFwGhCol = 128;         // spectrum columns (after 124 twiddle columns)
constexpr int kFwTmCols = 256;
constexpr int kFwOrder = 8;           // interleaved sweeps over a warp's rows (see the kernel)
constexpr size_t kFwSmem = sizeof(double2) * GeoW::SMEM * kFwWarps;
static_assert(GeoW::P == 32 && GeoW::T == 32 && GeoW::NPASS == 2, "warp-per-row geometry");

// (c, t) of exp(+i pi a / 16), a = 1..15 (correctly rounded); a = 0 and
// a = 8 are the exact W = 1, W = +i butterflies.
__device__ __forceinline__ constexpr double ct_c16(int a) {
  constexpr double c[16] = {1.0,
                            0x1.f6297cff75cb0p-1,
                            0x1.d906bcf328d46p-1,
                            0x1.a9b66290ea1a3p-1,
                            0x1.6a09e667f3bcdp-1,
                            0x1.1c73b39ae68c8p-1,
                            0x1.87de2a6aea963p-2,
                            0x1.8f8b83c69a60bp-3,
                            0.0,
                            -0x1.8f8b83c69a60bp-3,
                            -0x1.87de2a6aea963p-2,
                            -0x1.1c73b39ae68c8p-1,
                            -0x1.6a09e667f3bcdp-1,
                            -0x1.a9b66290ea1a3p-1,
                            -0x1.d906bcf328d46p-1,
                            -0x1.f6297cff75cb0p-1};
  return c[a];
}
__device__ __forceinline__ constexpr double ct_t16(int a) {
  constexpr double t[16] = {0.0,
                            0x1.975f5e0553158p-3,
                            0x1.a827999fcef32p-2,
                            0x1.561b82ab7f990p-1,
                            1.0,
                            0x1.7f218e25a7461p+0,
                            0x1.3504f333f9de6p+1,
                            0x1.41bfee2424771p+2,
                            0.0,
                            -0x1.41bfee2424771p+2,
                            -0x1.3504f333f9de6p+1,
                            -0x1.7f218e25a7461p+0,
                            -1.0,
                            -0x1.561b82ab7f990p-1,
                            -0x1.a827999fcef32p-2,
                            -0x1.975f5e0553158p-3};
  return t[a];
}
template <int A>
__device__ __forceinline__ void bfly_root32(double2& lo, double2& hi) {
  if constexpr (A == 0) bfly1(lo, hi);
  else if constexpr (A == 8) bfly_pi(lo, hi);
  else bfly_ct(lo, hi, ct_c16(A), ct_t16(A));
}
// butterflies of register pair kk at stage B of pass 0: twiddle exp(+i pi kk / 2^B)
template <int B, int KK>
__device__ __forceinline__ void warp_pass0_pair(double2 (&v)[32]) {
#pragma unroll
  for (int h = 0; h < (32 >> (B + 1)); ++h) {
    const int i = KK | (h << (B + 1));
    bfly_root32<(KK << (4 - B))>(v[i], v[i | (1 << B)]);
  }
}
template <int B, int KK = 0>
__device__ __forceinline__ void warp_pass0_stage(double2 (&v)[32]) {
  if constexpr (KK < (1 << B)) {
    warp_pass0_pair<B, KK>(v);
    warp_pass0_stage<B, KK + 1>(v);
  }
}

// Registers produced by a tcgen05.ld are valid after tcgen05.wait::ld; the
// empty asm ties their later uses to a point after the wait.
template <int NW>
__device__ __forceinline__ void tm_dep(uint32_t (&r)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) asm volatile("" : "+r"(r[i]));
}
__device__ __forceinline__ double tm_dbl(const uint32_t* r) { return __hiloint2double(r[1], r[0]); }

// stage Q (b = 5 + Q) of pass 1, register pairs kk in [KK0, KK0 + NK), their
// (c, t) pairs in r (4 words each)
template <int Q, int KK0, int NK>
__device__ __forceinline__ void warp_pass1_stage(double2 (&v)[32], const uint32_t* r) {
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int kk = KK0 + k;
    const double cc = tm_dbl(r + 4 * k), tt = tm_dbl(r + 4 * k + 2);
#pragma unroll
    for (int h = 0; h < (32 >> (Q + 1)); ++h) {
      const int i = kk | (h << (Q + 1));
      bfly_ct(v[i], v[i | (1 << Q)], cc, tt);
    }
  }
}

// BATCH (batches of on-chip fields, afd_capi.cu pruned_small): blockIdx.y =
// sig * Q + q over the signals' Q = N / 1024 pre-twiddled spectra; limits,
// hint and candidate row are the signal's (SubMap lim_stride / cand_stride /
// cand_off: slot cand_off + q * gridDim.x + blockIdx.x).
template <bool MARG, bool BATCH = false>
__global__ void __launch_bounds__(32 * kFwWarps, 1)
field_warp_kernel(const double2* __restrict__ ghat,   // [batch][1024]
                  const double* __restrict__ fw,      // [rows of plan][64] factor rows
                  const double2* __restrict__ twct,   // (c, t) stage tables S_b at 2^b - 1
                  long long row0, long long row1,     // global rows to evaluate
                  long long pw_row0,                  // global row of fw[0]
                  Cand* __restrict__ cand_out,        // [batch][gridDim.x]
                  SubMap sub) {
  constexpr int N = GeoW::N, P = GeoW::P;
  extern __shared__ double2 smem[];
  __shared__ uint32_t tm_base;
  __shared__ double wsm[kFwWarps][32];
  const int sig = blockIdx.y;  // spectrum of the launch
  const int sig_b = BATCH ? (int)blockIdx.y / sub.q_mul : 0;  // signal of the batch
  const int q_b = BATCH ? (int)blockIdx.y % sub.q_mul : (int)blockIdx.y;
  const size_t slot = BATCH ? (size_t)sig_b * sub.cand_stride + sub.cand_off +
                                  (size_t)q_b * gridDim.x + blockIdx.x
                            : (size_t)sig * gridDim.x + blockIdx.x;
  if constexpr (BATCH) {
    if (sub.hint) sub.hint += sig_b;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (sub.lim_lo != nullptr) {
    const long long l = sub.lim_lo[(size_t)sig_b * sub.lim_stride];
    if (l > row0) row0 = l < row1 ? l : row1;
  }
  if (sub.lim != nullptr) {
    const long long l = sub.lim[(size_t)sig_b * sub.lim_stride];
    if (l < row1) row1 = l > row0 ? l : row0;
  }
  if (row1 <= row0) {  // no rows for this kernel this step: a neutral candidate
    if (threadIdx.x == 0) {
      Cand c;
      c.mag = -1.0;
      c.flat = 0x7fffffffffffffffLL;
      c.re = c.im = 0.0;
      cand_out[slot] = c;
      if constexpr (MARG) sub.cand2[slot] = -1.0;
    }
    return;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tm_base)),
                 "n"(kFwTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // the warp's lane quadrant; warps w and w + 4 share it
  const uint32_t tmw = tm_base + ((uint32_t)((warp & 3) * 32) << 16);
  const double2* __restrict__ gh = ghat + (size_t)sig * N;
  if (warp < 4) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
#pragma unroll
      for (int kk = 0; kk < (1 << q); ++kk) {
        const double2 w = __ldg(twct + ((1 << (5 + q)) - 1) + (lane | (kk << 5)));
        tm_st4(tmw + 4 * ((1 << q) - 1 + kk), w);
      }
    }
#pragma unroll
    for (int i0 = 0; i0 < P; i0 += 8) {
      double2 g[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) g[i] = __ldg(gh + GeoW::l0(lane, i0 + i));
#pragma unroll
      for (int i = 0; i < 8; ++i) tm_st4(tmw + kFwGhCol + 4 * (i0 + i), g[i]);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  const int rows = (int)(row1 - row0);
  const int per_round = (int)gridDim.x * kFwWarps;
  double2* sm = smem + warp * GeoW::SMEM;
  double* wrow = wsm[warp];
  const int tl = brev_bits(lane, 5);  // logical thread of pass 0

  // Running first maximum.  Along a radius sweep |F|^2 rises steadily towards
  // the best pole's radius, so rows visited in increasing order set a new
  // maximum almost every row (measured: the update path ran on ~100% of the
  // rows).  A warp therefore visits its rows in kFwOrder interleaved sweeps
  // (rows k = o, o + kFwOrder, ... of its list, o = 0..kFwOrder-1: the first
  // sweep already comes close to the maximum) and screens each row against
  // `thr`, a warp-uniform lower bound of the warp's final maximum (MARG: of
  // its final runner-up): only a row with a point >= thr runs the update
  // path, where each thread keeps its own first maximum under the full
  // (magnitude, lowest flat index) order — within a row j = lane | i << 5
  // increases with i.
  double best_mag = -1.0, best_re = 0.0, best_im = 0.0;
  int best_sl = -1, best_i = 0;
  [[maybe_unused]] double sec_mag = -1.0;
  // the screen starts from the largest |F|^2 (margins: runner-up) of the
  // tiers launched before (a lower bound of the step's; afd_field_reg.cuh)
  double thr = sub.hint ? __longlong_as_double((long long)*(volatile unsigned long long*)sub.hint) : 0.0;
  if (!(thr > 0.0)) thr = -1.0;

  const int sl0 = (int)blockIdx.x * kFwWarps + warp;
  const int nk = sl0 < rows ? (rows - sl0 + per_round - 1) / per_round : 0;
  double a_nx = 0.0, b_nx = 0.0;
  if (nk > 0) {
    const double* __restrict__ fr = fw + (size_t)(row0 + sl0 - pw_row0) * kFwStride;
    a_nx = __ldg(fr + lane);
    b_nx = __ldg(fr + 32 + lane);
  }
  int k = 0, sweep = 0;
  for (bool more = nk > 0; more;) {
    const int sl = sl0 + k * per_round;
    const double a = a_nx;
    wrow[lane] = b_nx;
    // also orders the previous row's exchange loads before this row's stores
    __syncwarp();
    k += kFwOrder;
    if (k >= nk) k = ++sweep;
    more = sweep < kFwOrder && k < nk;
    if (more) {  // next row's factors, one row ahead
      const double* __restrict__ fr =
          fw + (size_t)(row0 + sl0 + (long long)k * per_round - pw_row0) * kFwStride;
      a_nx = __ldg(fr + lane);
      b_nx = __ldg(fr + 32 + lane);
    }
    double2 v[P];
    {
      // y_i = scale r^l G^_l and the stage-0 butterflies (register pairs
      // 2h, 2h + 1), eight registers per TMEM load, the next load in flight
      uint32_t r[2][32];
      tm_ld<32>(tmw + kFwGhCol, r[0]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tm_wait_ld();
        tm_dep(r[c & 1]);
        if (c + 1 < 4) tm_ld<32>(tmw + kFwGhCol + 32 * (c + 1), r[(c + 1) & 1]);
        const uint32_t* rc = r[c & 1];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int i0 = 8 * c + 2 * h, i1 = i0 + 1;
          const double w0 = a * wrow[brev_bits(i0, 5)], w1 = a * wrow[brev_bits(i1, 5)];
          const double2 x0 = make_double2(tm_dbl(rc + 8 * h), tm_dbl(rc + 8 * h + 2));
          const double2 x1 = make_double2(tm_dbl(rc + 8 * h + 4), tm_dbl(rc + 8 * h + 6));
          const double zr = w1 * x1.x, zi = w1 * x1.y;
          v[i0] = make_double2(fma(w0, x0.x, zr), fma(w0, x0.y, zi));
          v[i1] = make_double2(fma(w0, x0.x, -zr), fma(w0, x0.y, -zi));
        }
      }
    }
    // pass 0, stages 1..4
    warp_pass0_stage<1>(v);
    warp_pass0_stage<2>(v);
    warp_pass0_stage<3>(v);
    warp_pass0_stage<4>(v);
    // the exchange; the twiddles of stages 5..8 load while the row is in
    // shared memory (v is dead between the stores and the loads)
    pass_store<kFwK, kFwRB, 0>(v, tl, sm);
    uint32_t t5[4], t6[8], t7[16], ta[16];
    tm_ld<4>(tmw + 0, t5);
    tm_ld<8>(tmw + 4, t6);
    tm_ld<16>(tmw + 12, t7);
    tm_ld<16>(tmw + 28, ta);  // stage 8, pairs 0..3
    __syncwarp();
    pass_load<kFwK, kFwRB, 1>(v, lane, sm);
    tm_wait_ld();
    tm_dep(t5);
    tm_dep(t6);
    tm_dep(t7);
    tm_dep(ta);
    uint32_t tb[16];
    tm_ld<16>(tmw + 44, tb);  // stage 8, pairs 4..7
    warp_pass1_stage<0, 0, 1>(v, t5);
    warp_pass1_stage<1, 0, 2>(v, t6);
    warp_pass1_stage<2, 0, 4>(v, t7);
    warp_pass1_stage<3, 0, 4>(v, ta);
    // 16-word twiddle chunks (four register pairs), the next in flight
    tm_wait_ld();
    tm_dep(tb);
    uint32_t tc[16];
    tm_ld<16>(tmw + 60, tc);
    warp_pass1_stage<3, 4, 4>(v, tb);
    tm_wait_ld();
    tm_dep(tc);
    uint32_t td[16];
    tm_ld<16>(tmw + 76, td);
    warp_pass1_stage<4, 0, 4>(v, tc);
    tm_wait_ld();
    tm_dep(td);
    uint32_t te[16];
    tm_ld<16>(tmw + 92, te);
    warp_pass1_stage<4, 4, 4>(v, td);
    tm_wait_ld();
    tm_dep(te);
    uint32_t tf[16];
    tm_ld<16>(tmw + 108, tf);
    warp_pass1_stage<4, 8, 4>(v, te);
    tm_wait_ld();
    tm_dep(tf);
    warp_pass1_stage<4, 12, 4>(v, tf);

    // the screen: one predicate-accumulating compare per point
    unsigned up = 0;
#pragma unroll
    for (int i0 = 0; i0 < P; i0 += 4) {
      double mg[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mg[i] = fast_mag2(v[i0 + i]);
      up = any_ge4(up, mg, thr);
    }
    if (__builtin_expect(__any_sync(0xffffffffu, up != 0), 0)) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        // recompute (do not keep P magnitudes live across the screen)
        double2 f = v[i];
        asm volatile("" : "+d"(f.x), "+d"(f.y));
        const double mg = fast_mag2(f);
        const bool better = mg > best_mag || (mg == best_mag && sl < best_sl);
        if (better) {
          if constexpr (MARG) sec_mag = best_mag;
          best_mag = mg;
          best_re = f.x;
          best_im = f.y;
          best_sl = sl;
          best_i = i;
        } else if constexpr (MARG) {
          if (mg > sec_mag) sec_mag = mg;
        }
      }
      double m = best_mag;
      [[maybe_unused]] double r = sec_mag;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
        if constexpr (MARG) {
          const double r2 = __shfl_xor_sync(0xffffffffu, r, o);
          r = runner_merge(r, m, r2, m2);
        }
        m = fmax(m, m2);
      }
      thr = fmax(thr, MARG ? r : m);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base),
                 "n"(kFwTmCols)
                 : "memory");
  Cand best;
  best.mag = best_mag;
  if (best_sl >= 0) {
    const long long j = (long long)(lane | (best_i << 5));
    best.flat = (row0 + best_sl) * (sub.row_stride ? sub.row_stride : (long long)N) +
                (sub.q_mul ? (long long)q_b + (long long)sub.q_mul * j : j);
  } else {
    best.flat = 0x7fffffffffffffffLL;
  }
  best.re = best_re;
  best.im = best_im;
  [[maybe_unused]] const double own_mag = best.mag;
  [[maybe_unused]] const long long own_flat = best.flat;
  __shared__ Cand red[kFwWarps];
  __shared__ long long win_flat;
  best = warp_argmax(best);
  if (lane == 0) red[warp] = best;
  __syncthreads();
  if (warp == 0) {
    Cand c = lane < kFwWarps ? red[lane] : best;
    c = warp_argmax(c);
    if (lane == 0) {
      cand_out[slot] = c;
      if constexpr (MARG) win_flat = c.flat;
      // non-negative doubles order like their bit patterns
      if (!MARG && sub.hint && c.mag > 0.0)
        atomicMax(sub.hint, (unsigned long long)__double_as_longlong(c.mag));
    }
  }
  if constexpr (MARG) {
    __shared__ double red2[32];
    __syncthreads();
    const double r2 = cta_runner_up(sec_mag, own_mag, own_flat, win_flat, red2);
    if (threadIdx.x == 0) {
      sub.cand2[slot] = r2;
      if (sub.hint && r2 > 0.0) atomicMax(sub.hint, (unsigned long long)__double_as_longlong(r2));
    }
  }
}

}  // namespace afd
