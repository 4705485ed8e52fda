// afd_field_sub.cuh — fast-engine field + argmax for rows that need at most
// L = 256 or 512 spectrum terms: the warp-per-row kernel's structure
// (afd_field_warp.cuh) with T = L / 32 = 8 or 16 threads per L-point
// sub-transform, so a warp runs S = 32 / T sub-transforms of ONE row side by
// side — the row's N / L pre-twiddled spectra q = S blockIdx.y + lane / T
// (afd_pruned.cuh) — and pass 1 has 3 or 4 butterfly stages instead of 5
// (weighted_inverse_grid + maximal_selection, transform.py:185-201,
// core.py:285-300; the arithmetic of the fast engine).
//
// Thread t = lane mod T holds 32 points: pass 0 (five register stages, the
// compile-time 32nd roots of unity) over l = rev5(i) << C | t, C = log2 T,
// one exchange through the warp's shared-memory rows (__syncwarp only), then
// stages b = 5 .. log2 L - 1 on register bit b - C with the twiddles
// S_b[t | kk << C] from tensor memory (28 or 30 (c, t) pairs per lane; the
// lane's 32 spectrum values beside them).  The row's weights scale r^l =
// fw[t] * fw[T + rev5(i)] come from a (T + 32)-entry factor row.  ~25 / ~28
// FP64 instructions per grid evaluation against ~31 for 1024 points.
// Row order, screening and hints as in the warp kernel.
#pragma once

#include "afd_field_warp.cuh"

namespace afd {

template <int KL>
struct SubGeo {
  static constexpr int C = KL - 5;        // thread bits of a sub-transform
  static constexpr int T = 1 << C;        // threads per sub-transform
  static constexpr int S = 32 / T;        // sub-transforms per warp
  static constexpr int L = 1 << KL;
  static constexpr int kStride = T + 32;  // factor row: scale r^t (t < T), r^(T m) (m < 32)
  static constexpr int kPairs = 32 - (32 >> C);  // twiddle pairs per lane (stages 5 .. KL-1)
  using G = Geo<KL, 5>;
  static constexpr size_t kSmem = sizeof(double2) * G::SMEM * S * kFwWarps;
  // first twiddle column (4 words per pair) of stage b
  __host__ __device__ static constexpr int col(int b) { return 4 * ((1 << (b - C)) - (32 >> C)); }
  static_assert(KL == 8 || KL == 9, "256- and 512-point sub-transforms");
  static_assert(G::P == 32 && G::T == T && G::NPASS == 2, "two passes of 32 points per thread");
};

template <int KL, bool MARG, bool BATCH = false>
__global__ void __launch_bounds__(32 * kFwWarps, 1)
field_sub_kernel(const double2* __restrict__ ghat,   // [spectra][L]
                 const double* __restrict__ fw,      // [rows of plan][T + 32] factor rows
                 const double2* __restrict__ twct,   // (c, t) stage tables S_b at 2^b - 1
                 long long row0, long long row1,     // global rows to evaluate
                 long long pw_row0,                  // global row of fw[0]
                 Cand* __restrict__ cand_out, SubMap sub) {
  using SG = SubGeo<KL>;
  using G = typename SG::G;
  constexpr int C = SG::C, T = SG::T, S = SG::S, L = SG::L, P = 32;
  extern __shared__ double2 smem[];
  __shared__ uint32_t tm_base;
  __shared__ double wsm[kFwWarps][32];
  // blockIdx.y: block of S consecutive spectra (BATCH: of one signal)
  const int qblocks = sub.q_mul / S;  // per signal
  const int sig_b = BATCH ? (int)blockIdx.y / qblocks : 0;
  const int qblk = BATCH ? (int)blockIdx.y % qblocks : (int)blockIdx.y;
  const size_t slot = BATCH ? (size_t)sig_b * sub.cand_stride + sub.cand_off +
                                  (size_t)qblk * gridDim.x + blockIdx.x
                            : (size_t)blockIdx.y * gridDim.x + blockIdx.x;
  if constexpr (BATCH) {
    if (sub.hint) sub.hint += sig_b;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> C, t = lane & (T - 1);
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
  // the warp's lane quadrant; warps w and w + 4 share it (same lane: same
  // thread t, same spectrum q)
  const uint32_t tmw = tm_base + ((uint32_t)((warp & 3) * 32) << 16);
  const int q = qblk * S + grp;  // the lane's spectrum within the signal
  const double2* __restrict__ gh =
      ghat + ((size_t)(BATCH ? sig_b : 0) * sub.q_mul + (size_t)q) * L;
  if (warp < 4) {
#pragma unroll
    for (int b = 5; b < KL; ++b) {
#pragma unroll
      for (int kk = 0; kk < (1 << (b - C)); ++kk) {
        const double2 w = __ldg(twct + ((1 << b) - 1) + (t | (kk << C)));
        tm_st4(tmw + SG::col(b) + 4 * kk, w);
      }
    }
#pragma unroll
    for (int i0 = 0; i0 < P; i0 += 8) {
      double2 g[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) g[i] = __ldg(gh + G::l0(t, i0 + i));
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
  double2* sm = smem + (size_t)(warp * S + grp) * G::SMEM;
  double* wrow = wsm[warp];
  const int tl = brev_bits(t, C);  // logical thread of pass 0

  double best_mag = -1.0, best_re = 0.0, best_im = 0.0;
  int best_sl = -1, best_i = 0;
  [[maybe_unused]] double sec_mag = -1.0;
  double thr = sub.hint ? __longlong_as_double((long long)*(volatile unsigned long long*)sub.hint) : 0.0;
  if (!(thr > 0.0)) thr = -1.0;

  const int sl0 = (int)blockIdx.x * kFwWarps + warp;
  const int nk = sl0 < rows ? (rows - sl0 + per_round - 1) / per_round : 0;
  double a_nx = 0.0, b_nx = 0.0;
  if (nk > 0) {
    const double* __restrict__ fr = fw + (size_t)(row0 + sl0 - pw_row0) * SG::kStride;
    a_nx = __ldg(fr + t);
    b_nx = __ldg(fr + T + lane);
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
          fw + (size_t)(row0 + sl0 + (long long)k * per_round - pw_row0) * SG::kStride;
      a_nx = __ldg(fr + t);
      b_nx = __ldg(fr + T + lane);
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
    // the exchange; the first twiddles load while the sub-transform is in
    // shared memory (v is dead between the stores and the loads)
    pass_store<KL, 5, 0>(v, tl, sm);
    if constexpr (KL == 8) {
      // stages 5, 6, 7 on register bits 2, 3, 4: 4, 8, 16 pairs at columns 0, 16, 48
      uint32_t t5[16], t6a[16], t6b[16];
      tm_ld<16>(tmw + 0, t5);
      tm_ld<16>(tmw + 16, t6a);
      tm_ld<16>(tmw + 32, t6b);
      __syncwarp();
      pass_load<KL, 5, 1>(v, t, sm);
      tm_wait_ld();
      tm_dep(t5);
      tm_dep(t6a);
      tm_dep(t6b);
      uint32_t ta[16];
      tm_ld<16>(tmw + 48, ta);
      warp_pass1_stage<2, 0, 4>(v, t5);
      warp_pass1_stage<3, 0, 4>(v, t6a);
      warp_pass1_stage<3, 4, 4>(v, t6b);
      tm_wait_ld();
      tm_dep(ta);
      uint32_t tb[16];
      tm_ld<16>(tmw + 64, tb);
      warp_pass1_stage<4, 0, 4>(v, ta);
      tm_wait_ld();
      tm_dep(tb);
      uint32_t tc[16];
      tm_ld<16>(tmw + 80, tc);
      warp_pass1_stage<4, 4, 4>(v, tb);
      tm_wait_ld();
      tm_dep(tc);
      uint32_t td[16];
      tm_ld<16>(tmw + 96, td);
      warp_pass1_stage<4, 8, 4>(v, tc);
      tm_wait_ld();
      tm_dep(td);
      warp_pass1_stage<4, 12, 4>(v, td);
    } else {
      // stages 5..8 on register bits 1..4: 2, 4, 8, 16 pairs at columns 0, 8, 24, 56
      uint32_t t5[8], t6[16], t7a[16];
      tm_ld<8>(tmw + 0, t5);
      tm_ld<16>(tmw + 8, t6);
      tm_ld<16>(tmw + 24, t7a);
      __syncwarp();
      pass_load<KL, 5, 1>(v, t, sm);
      tm_wait_ld();
      tm_dep(t5);
      tm_dep(t6);
      tm_dep(t7a);
      uint32_t t7b[16];
      tm_ld<16>(tmw + 40, t7b);
      warp_pass1_stage<1, 0, 2>(v, t5);
      warp_pass1_stage<2, 0, 4>(v, t6);
      warp_pass1_stage<3, 0, 4>(v, t7a);
      tm_wait_ld();
      tm_dep(t7b);
      uint32_t ta[16];
      tm_ld<16>(tmw + 56, ta);
      warp_pass1_stage<3, 4, 4>(v, t7b);
      tm_wait_ld();
      tm_dep(ta);
      uint32_t tb[16];
      tm_ld<16>(tmw + 72, tb);
      warp_pass1_stage<4, 0, 4>(v, ta);
      tm_wait_ld();
      tm_dep(tb);
      uint32_t tc[16];
      tm_ld<16>(tmw + 88, tc);
      warp_pass1_stage<4, 4, 4>(v, tb);
      tm_wait_ld();
      tm_dep(tc);
      uint32_t td[16];
      tm_ld<16>(tmw + 104, td);
      warp_pass1_stage<4, 8, 4>(v, tc);
      tm_wait_ld();
      tm_dep(td);
      warp_pass1_stage<4, 12, 4>(v, td);
    }

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
    // output register i of thread t sits at position t | i << C of spectrum q
    const long long j = (long long)(t | (best_i << C));
    best.flat = (row0 + best_sl) * sub.row_stride + (long long)q + (long long)sub.q_mul * j;
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
