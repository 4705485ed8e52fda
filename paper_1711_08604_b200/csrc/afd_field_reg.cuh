// afd_field_reg.cuh — fast-engine field + argmax for rows that need at most
// L = 32 D spectrum terms (D = 1, 2, 4), entirely in registers: one thread per
// 32 outputs, no exchange, no barriers (weighted_inverse_grid +
// maximal_selection, transform.py:185-201, core.py:285-300; the arithmetic
// of the fast engine, afd_fft.cuh "Fast mode").
//
// Row s of the field is F_s(j) = sum_l w_l G^_l e^{2 pi i l j / N} with
// w_l = scale_s r_s^l.  When the terms l >= 32 D are negligible
// (prune_rows_kernel: below 2^-64 of a kept term, r <= 0.25 for D = 1,
// r <= 0.5 for D = 2, r <= 0.7 for D = 4), split j = q' + Q' i with
// Q' = N / 32 and l = l0 + 32 m:
//   F_s(q' + Q' i) = sum_{l0 < 32} e^{2 pi i l0 i / 32} w_{l0} sum_{m < D} rho^m h^(q')_{l0, m},
//   h^(q')_{l0, m} = G^_{l0 + 32 m} e^{2 pi i (l0 + 32 m) q' / N},  rho = r_s^32,
// a 32-point inverse transform (five register stages with compile-time
// 32nd roots of unity: warp_pass0_stage) of a polynomial in rho of degree
// D - 1.  Thread q' keeps its 32 D pre-twiddled values h (row-independent,
// pretwiddle_reg_kernel) in tensor memory and walks the rows: per grid
// evaluation 2 (D - 1) DFMA for the polynomial, 3 for the weights fused with
// stage 0, ~10 for stages 1-4, 3 for |F|^2 and the screen: ~16-22 FP64
// instructions against ~33 for the 1024-point warp kernel, and no shared
// memory traffic beyond the row's 32 weights (a broadcast line per warp).
//
// Rows are visited in decreasing order (|F|^2 grows with r at small radii, so
// the first rows set the maximum and the rest only pass the screen), and the
// screen starts from `hint`: the largest |F|^2 (margins: runner-up) the
// tiers launched before have already found — a lower bound of the step's
// maximum, so no candidate is lost; ties (>=) still reach the update path.
#pragma once

#include "afd_field_warp.cuh"

namespace afd {

// Warps per CTA (one CTA per SM): tensor memory has room for 512 / (128 D)
// warps per lane quadrant, registers for 8 warps at 255.  D = 4 fills tensor
// memory with four warps (one per scheduler: FP64 pipe 73% busy).
// -DAFD_FR_SMWARPS4=3 adds three warps that keep their spectra in shared
// memory instead (64 KiB each, [value][lane]: conflict-free 16-byte loads,
// a chunk ahead) — measured slower (c4 5.95e11 -> 5.70e11 evals/s, c3
// 5.10e11 -> 4.92e11), so it is off.
#ifndef AFD_FR_WARPS1
#define AFD_FR_WARPS1 8
#endif
#ifndef AFD_FR_SMWARPS4
#define AFD_FR_SMWARPS4 0
#endif
// D = 4: tensor memory holds the spectra of only 128 values of q' per SM (four
// warps, one per scheduler: FP64 pipe 73% busy).  Warps w and w + 4 read the
// same lane quadrant, so a second set of four warps serves the SAME 128 q'
// from the same columns and takes every other row of the CTA's rows
// (AFD_FR_SHARE4 = 2 row sets): eight warps per SM without more storage.
#ifndef AFD_FR_SHARE4
#define AFD_FR_SHARE4 2
#endif
__host__ __device__ constexpr int fr_smem_warps(int D) { return D == 4 ? AFD_FR_SMWARPS4 : 0; }
__host__ __device__ constexpr int fr_share(int D) {
  return D == 4 && AFD_FR_SMWARPS4 == 0 ? AFD_FR_SHARE4 : 1;
}
__host__ __device__ constexpr int fr_warps(int D) {
  return D == 1 ? AFD_FR_WARPS1 : D == 2 ? 8 : 4 * fr_share(D) + fr_smem_warps(D);
}
__host__ __device__ constexpr int fr_threads(int D) { return 32 * fr_warps(D); }
// threads of a CTA that serve distinct q' (the CTA's extent along q')
__host__ __device__ constexpr int fr_qthreads(int D) { return fr_threads(D) / fr_share(D); }
__host__ __device__ constexpr size_t fr_smem_bytes(int D) {
  return sizeof(double2) * 32 * D * 32 * fr_smem_warps(D);
}

// BATCH: many signals of an on-chip N (afd_capi.cu pruned_small, BASELINE
// c3): thread g of the launch serves signal g >> kq and q' = g mod Q' (a warp
// never straddles signals: Q' >= 32), its spectra at h + sig * 128 Q' (four
// blocks per signal whatever D), its row limits and hint are the signal's
// (sub.lim_stride), and every warp writes its own candidate to the signal's
// candidate row: slot cand_off + (blockIdx.x * fr_share(D) + row set) * (Q' / 32)
// + (q' >> 5).
struct RegBatch {
  int kq;                   // log2 Q'
  long long threads_total;  // batch * Q'
  int cand_off;             // first slot of this tier in a signal's candidate row
};

template <int D, bool MARG, bool BATCH = false>
__global__ void __launch_bounds__(fr_threads(D), 1)
field_reg_kernel(const double2* __restrict__ h,      // [32 D][Q'] pre-twiddled spectra
                 const double* __restrict__ fw,      // [rows of plan][64] factor rows (kFwStride)
                 long long row0, long long row1,     // global rows to evaluate
                 long long pw_row0,                  // global row of fw[0]
                 long long qp_total,                 // Q' = N / 32
                 Cand* __restrict__ cand_out,        // [gridDim.y][gridDim.x]
                 const unsigned long long* __restrict__ hint, SubMap sub, RegBatch rb) {
  static_assert(D == 1 || D == 2 || D == 4, "chunks of 8 / D registers per 32-word TMEM load");
#ifndef AFD_FR_LDW4
#define AFD_FR_LDW4 32
#endif
  // words per TMEM load (-DAFD_FR_LDW4=64: twice as long for D = 4; measured
  // 1% slower)
  constexpr int W = D == 4 ? AFD_FR_LDW4 : 32;
  constexpr int CV = W / 4;          // complex values per load
  constexpr int GI = CV / D;         // registers i per load
  constexpr int NCH = 32 / GI;       // loads per row
  constexpr int kFrWarps = fr_warps(D), kFrThreads = fr_threads(D);
  constexpr int kCols = 128 * D;     // columns per warp
  constexpr int kShare = fr_share(D), kQThreads = fr_qthreads(D);
  constexpr int kSmWarps = fr_smem_warps(D), kTmWarps = (kFrWarps - kSmWarps) / kShare;
  constexpr int kTmCols = kCols * (kTmWarps / 4) <= 256 ? 256 : 512;
  static_assert(kTmWarps % 4 == 0 && kCols * (kTmWarps / 4) <= 512, "TMEM columns");
  extern __shared__ double2 hs_all[];  // [kSmWarps][32 D][32 lanes]
  __shared__ uint32_t tm_base;
  __shared__ __align__(16) double wsm[kFrWarps][2][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.y * gridDim.x + blockIdx.x;
  const int rset = (int)threadIdx.x / kQThreads;  // row set of the thread (kShare > 1)
  const long long gthread = (long long)blockIdx.y * kQThreads + (int)threadIdx.x % kQThreads;
  // warp-uniform (Q' is a multiple of 32)
  const bool active = gthread < (BATCH ? rb.threads_total : qp_total);
  const int sig = BATCH && active ? (int)(gthread >> rb.kq) : 0;
  const long long qp = BATCH ? gthread & (qp_total - 1) : gthread;
  if constexpr (BATCH) {
    h += (size_t)sig * 128 * (size_t)qp_total;
    if (hint) hint += sig;
  }
  if (sub.lim_lo != nullptr) {
    const long long l = sub.lim_lo[(size_t)sig * sub.lim_stride];
    if (l > row0) row0 = l < row1 ? l : row1;
  }
  if (sub.lim != nullptr) {
    const long long l = sub.lim[(size_t)sig * sub.lim_stride];
    if (l < row1) row1 = l > row0 ? l : row0;
  }
  const int rows = (int)(row1 - row0);
  if (!BATCH && rows <= (int)blockIdx.x) {  // no rows for this CTA this step: a neutral candidate
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
                 "n"(kTmCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // the warp's lane quadrant; warps w and w + 4 share it, side by side
  const int tw = kShare > 1 ? warp % kTmWarps : warp;  // the warp whose columns this one reads
  const uint32_t tmw = tm_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((tw >> 2) * kCols);
  const bool smem_fed = kSmWarps > 0 && warp >= kTmWarps;  // warp-uniform
  double2* __restrict__ hs = hs_all + (size_t)(smem_fed ? warp - kTmWarps : 0) * (32 * D * 32) + lane;
  // chunk c holds registers i = GI c .. GI c + GI - 1, block m at word 4 GI m
#pragma unroll
  for (int c = 0; c < NCH && active && rset == 0; ++c) {
    double2 g[CV];
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
      for (int u = 0; u < GI; ++u)
        g[m * GI + u] = __ldg(h + (size_t)(m * 32 + c * GI + u) * (size_t)qp_total + qp);
    if (smem_fed) {
#pragma unroll
      for (int x = 0; x < CV; ++x) hs[(CV * c + x) * 32] = g[x];
    } else {
#pragma unroll
      for (int x = 0; x < CV; ++x) tm_st4(tmw + W * c + 4 * x, g[x]);
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  if constexpr (kShare > 1) {  // the other row sets read what row set 0 stored
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }

  double best_mag = -1.0, best_re = 0.0, best_im = 0.0;
  int best_sl = 0x7fffffff, best_i = 0;
  [[maybe_unused]] double sec_mag = -1.0;
  double thr = hint ? __longlong_as_double((long long)*hint) : 0.0;
  if (!(thr > 0.0)) thr = -1.0;

  // rows sl = blockIdx.x + k gridDim.x, k = nk - 1 .. 0 (row set s: every
  // kShare-th of them from nk - 1 - s down)
  const int nk = active && rows > (int)blockIdx.x
                     ? (rows - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                     : 0;
  const double* __restrict__ fr0 = fw + (size_t)(row0 + blockIdx.x - pw_row0) * kFwStride;
  const size_t fstep = (size_t)gridDim.x * kFwStride;
  const int k0 = nk - 1 - rset;
  double a_nx = k0 >= 0 ? __ldg(fr0 + (size_t)k0 * fstep + lane) : 0.0;
  [[maybe_unused]] double rho_nx = D > 1 && k0 >= 0 ? __ldg(fr0 + (size_t)k0 * fstep + 33) : 0.0;
  const int wpos = brev_bits(lane, 5);  // weight of l0 = lane sits at register index rev5(l0)
  int it = 0;
  for (int k = k0; k >= 0; k -= kShare, ++it) {
    const int sl = (int)blockIdx.x + k * (int)gridDim.x;
    double* wrow = wsm[warp][it & 1];
    wrow[wpos] = a_nx;
    [[maybe_unused]] const double rho = rho_nx;
    __syncwarp();
    if (k >= kShare) {  // next row's factors, one row ahead
      a_nx = __ldg(fr0 + (size_t)(k - kShare) * fstep + lane);
      if constexpr (D > 1) rho_nx = __ldg(fr0 + (size_t)(k - kShare) * fstep + 33);
    }
    double2 v[32];
    {
      // y_i = w_l0 sum_m rho^m h_(l0, m) and the stage-0 butterflies (register
      // pairs 2 u, 2 u + 1), GI registers per TMEM load, the next load in flight
      // (shared-memory warps: the same 32-word chunks by eight 16-byte loads)
      uint32_t r[2][W];
      auto fetch = [&](int c, uint32_t (&buf)[W]) {
        if (smem_fed) {
#pragma unroll
          for (int x = 0; x < CV; ++x) {
            const uint4 t = *reinterpret_cast<const uint4*>(hs + (CV * c + x) * 32);
            buf[4 * x] = t.x;
            buf[4 * x + 1] = t.y;
            buf[4 * x + 2] = t.z;
            buf[4 * x + 3] = t.w;
          }
        } else {
          tm_ld<W>(tmw + W * c, buf);
        }
      };
      fetch(0, r[0]);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (!smem_fed) tm_wait_ld();
        tm_dep(r[c & 1]);
        if (c + 1 < NCH) fetch(c + 1, r[(c + 1) & 1]);
        const uint32_t* rc = r[c & 1];
#pragma unroll
        for (int u = 0; u < GI; u += 2) {
          const int i0 = GI * c + u, i1 = i0 + 1;
          const double2 w = *reinterpret_cast<const double2*>(wrow + i0);
          double2 x0 = make_double2(tm_dbl(rc + 4 * ((D - 1) * GI + u)),
                                    tm_dbl(rc + 4 * ((D - 1) * GI + u) + 2));
          double2 x1 = make_double2(tm_dbl(rc + 4 * ((D - 1) * GI + u + 1)),
                                    tm_dbl(rc + 4 * ((D - 1) * GI + u + 1) + 2));
#pragma unroll
          for (int m = D - 2; m >= 0; --m) {
            x0.x = fma(rho, x0.x, tm_dbl(rc + 4 * (m * GI + u)));
            x0.y = fma(rho, x0.y, tm_dbl(rc + 4 * (m * GI + u) + 2));
            x1.x = fma(rho, x1.x, tm_dbl(rc + 4 * (m * GI + u + 1)));
            x1.y = fma(rho, x1.y, tm_dbl(rc + 4 * (m * GI + u + 1) + 2));
          }
          const double zr = w.y * x1.x, zi = w.y * x1.y;
          v[i0] = make_double2(fma(w.x, x0.x, zr), fma(w.x, x0.y, zi));
          v[i1] = make_double2(fma(w.x, x0.x, -zr), fma(w.x, x0.y, -zi));
        }
      }
    }
    warp_pass0_stage<1>(v);
    warp_pass0_stage<2>(v);
    warp_pass0_stage<3>(v);
    warp_pass0_stage<4>(v);

    // the screen: one predicate-accumulating compare per point
    unsigned up = 0;
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 4) {
      double mg[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mg[i] = fast_mag2(v[i0 + i]);
      up = any_ge4(up, mg, thr);
    }
    if (__builtin_expect(__any_sync(0xffffffffu, up != 0), 0)) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        double2 f = v[i];
        asm volatile("" : "+d"(f.x), "+d"(f.y));
        const double mg = fast_mag2(f);
        // rows descend: an equal magnitude in a lower row wins; within a row
        // j = q' + Q' i increases with i
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
                 "n"(kTmCols)
                 : "memory");
  Cand best;
  best.mag = best_mag;
  if (best_mag >= 0.0) {
    best.flat = (row0 + best_sl) * sub.row_stride + qp + qp_total * (long long)best_i;
  } else {
    best.flat = 0x7fffffffffffffffLL;
  }
  best.re = best_re;
  best.im = best_im;
  [[maybe_unused]] const double own_mag = best.mag;
  [[maybe_unused]] const long long own_flat = best.flat;
  if constexpr (BATCH) {  // one candidate per warp, in the signal's candidate row
    best = warp_argmax(best);
    const size_t ws = (size_t)sig * sub.cand_stride + rb.cand_off +
                      ((size_t)blockIdx.x * kShare + rset) * (size_t)(qp_total >> 5) +
                      (size_t)(qp >> 5);
    if (active && lane == 0) cand_out[ws] = best;
    if constexpr (MARG) {
      const long long wf = __shfl_sync(0xffffffffu, best.flat, 0);
      double x = fmax(sec_mag, own_flat != wf ? own_mag : -1.0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (active && lane == 0) sub.cand2[ws] = x;
    }
    return;
  }
  __shared__ Cand red[kFrWarps];
  __shared__ long long win_flat;
  best = warp_argmax(best);
  if (lane == 0) red[warp] = best;
  __syncthreads();
  if (warp == 0) {
    Cand c = lane < kFrWarps ? red[lane] : best;
    c = warp_argmax(c);
    if (lane == 0) {
      cand_out[slot] = c;
      if constexpr (MARG) win_flat = c.flat;
    }
  }
  if constexpr (MARG) {
    __shared__ double red2[32];
    __syncthreads();
    const double r2 = cta_runner_up(sec_mag, own_mag, own_flat, win_flat, red2);
    if (threadIdx.x == 0) sub.cand2[slot] = r2;
  }
}

}  // namespace afd
