// afd_kernels.cuh — the sm_100a kernels of the AFD selection hot path for
// on-chip transform lengths N = 2^K <= 8192.
//
//   field_kernel   ★ K2 of SURVEY.md §2.2: per (signal, radius row) the
//                  prologue r^l * Ghat[l], the inverse butterflies, the
//                  sqrt(1-r^2)/(N(1-r^N)) scale, |.|^2 and the running
//                  first-maximum; one 32-byte candidate per CTA (or the
//                  materialised rows, for parity tests).
//                  Reference: transform.weighted_inverse_grid + maximal_selection
//                  (transform.py:185-201, core.py:285-300).
//   step_kernel    K3+K4+K1: reduce the candidates (first max), form the
//                  pole a = r_s z_j, update the remainder
//                  (core.py:303-314), its energy (core.py:195-198), record
//                  the step, test the stop rules (core.py:386-389) and
//                  forward-transform the new remainder for the next step
//                  (core.py:248-250).  One CTA per signal.
//   fft_kernel     dft_forward / dft_inverse (transform.py:106-134) and the
//                  analytic projection (core.py:201-231).
//
// All kernels reproduce the reference's arithmetic bit for bit (see
// afd_common.cuh); the library is compiled with -fmad=false.
#pragma once

#include <type_traits>

#include "afd_fft.cuh"

namespace afd {

struct State {
  int stopped;   // no further steps for this signal
  int nsteps;    // recorded steps
  int flags;     // OR of step flags
  int pad;
  double initial;
};

// Must match afd_step in include/afd_capi.h.
struct Step {
  long long s, j;
  double radius, a_re, a_im, c_re, c_im, residual;
  int flags;
  float margin;  // fast engine: top-2 relative margin of |F|^2; NaN if not tracked
};

enum : int { kStepPowAmbiguous = 1 };

#ifdef AFD_FIELD_TIMING
// %globaltimer stamps (ns) of each row-group leader: [cta][group][row][slot]
//   0 start, 1 after the PDL wait, per row: 2 prologue done, 3/5/7 pass
//   ends, 4/6 exchange ends, 14 epilogue done; 15 = SM id (row 0 only)
__device__ long long g_field_stamps[512][2][4][16];
__device__ __forceinline__ long long ftime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FSTAMP(r, i)                                                                      \
  do {                                                                                    \
    if (tp == 0 && blockIdx.x < 512 && g < 2 && (r) < 4) g_field_stamps[blockIdx.x][g][r][i] = \
        ftime();                                                                          \
  } while (0)
#else
#define FSTAMP(r, i) \
  do {               \
  } while (0)
#endif

// Phase offset between the two row-groups of a field CTA.  The butterfly
// passes are FP64-bound and the exchanges / prologue / epilogue shared-memory
// or L1 bound; started together the groups run in lock step and the FP64
// pipe idles through every exchange.  Group 1 therefore starts its first
// pass only when group 0 has finished its own first pass (named barrier 3:
// group 0 arrives, group 1 syncs), after which the groups run free, one
// phase apart (AFD_FIELD_PP=0 disables it; measured 8.8e10 -> 9.3e10 c1).
struct FieldHook {
  bool arrive;     // group 0, first row: release group 1 after pass 0
  int count;       // threads of both groups
  long long* st;   // timing stamps of this row (timing builds) or null
  bool tm_fence;   // TMEM written before the release (gh spectrum, TM variant)
  // dynamic rows: the group leader publishes its claim of the next row after
  // the first exchange (the atomic has long returned; the second exchange's
  // barriers make the slot visible to the group)
  int* claim_slot;           // null: not the leader / static rows
  const unsigned* claim;     // the leader's atomicAdd result
  int claim_base;
  __device__ __forceinline__ void before(int) const {}
  __device__ __forceinline__ void after(int pass) const {
    if (pass == 0 && arrive) {
      if (tm_fence) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("bar.arrive 3, %0;" ::"r"(count) : "memory");
    }
#ifdef AFD_FIELD_TIMING
    if (st) st[3 + 2 * pass] = ftime();
#endif
  }
  __device__ __forceinline__ void exch(int pass) const {
    if (pass == 0 && claim_slot != nullptr) *claim_slot = claim_base + (int)*claim;
#ifdef AFD_FIELD_TIMING
    if (st) st[4 + 2 * pass] = ftime();
#endif
  }
};

// ---------------------------------------------------------------------------
// Field + argmax (or materialised field).  Block = G row-groups of T threads;
// each group evaluates one radius row per round; rows are strided over the
// CTAs of a signal (blockIdx.y).
// ---------------------------------------------------------------------------
// Fast weights (AFD_PLAN_FAST): row s of `pw` is then the factor table
// fw[s] = { scale_s r_s^t (t < T), r_s^(T m) (m < P) }, so register i of
// thread t (natural l = (rev(i) << TB) | t) is weighted by
// w = fw[t] * fw[T + rev(i)] = scale r^l, formed on chip (1 DMUL) instead of
// read from the M x N cumprod table, and the weighting is fused into
// stage 0: z = w_b y_b, lo/hi = fma(w_a, y_a, +-z).
template <int K, int RB>
struct FastW {
  static constexpr int T = Geo<K, RB>::T, P = Geo<K, RB>::P;
  static constexpr int STRIDE = T + P;
  // weights of thread tp's P registers for table row `fr`
  __device__ __forceinline__ static void load(const double* __restrict__ fr, int tp,
                                              double (&w)[P]) {
    const double a = __ldg(fr + tp);
    double b[P];
#pragma unroll
    for (int m = 0; m < P; ++m) b[m] = __ldg(fr + T + m);
#pragma unroll
    for (int i = 0; i < P; ++i) w[i] = a * b[brev_bits(i, Geo<K, RB>::RB)];
  }
};
// y_i = w_i x_i followed by the stage-0 butterflies (pairs 2h, 2h+1; W = 1)
template <int P>
__device__ __forceinline__ void fast_prologue(double2 (&v)[P], const double (&w)[P]) {
#pragma unroll
  for (int h = 0; h < P / 2; ++h) {
    const double2 a = v[2 * h], b = v[2 * h + 1];
    const double zr = w[2 * h + 1] * b.x, zi = w[2 * h + 1] * b.y;
    v[2 * h] = make_double2(fma(w[2 * h], a.x, zr), fma(w[2 * h], a.y, zi));
    v[2 * h + 1] = make_double2(fma(w[2 * h], a.x, -zr), fma(w[2 * h], a.y, -zi));
  }
}
__device__ __forceinline__ double fast_mag2(double2 f) { return fma(f.x, f.x, f.y * f.y); }

// flag | (any of m[0..3] > best): one predicate-accumulating compare per value
// (setp.gt.or), instead of the max/select chain the compiler makes of `|=`.
__device__ __forceinline__ unsigned any_gt2(unsigned flag, const double (&m)[2], double best) {
  unsigned out;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "setp.gt.or.f64 p, %2, %4, p;\n\t"
      "setp.gt.or.f64 p, %3, %4, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(out)
      : "r"(flag), "d"(m[0]), "d"(m[1]), "d"(best));
  return out;
}
__device__ __forceinline__ unsigned any_ge4(unsigned flag, const double (&m)[4], double best) {
  unsigned out;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "setp.ge.or.f64 p, %2, %6, p;\n\t"
      "setp.ge.or.f64 p, %3, %6, p;\n\t"
      "setp.ge.or.f64 p, %4, %6, p;\n\t"
      "setp.ge.or.f64 p, %5, %6, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(out)
      : "r"(flag), "d"(m[0]), "d"(m[1]), "d"(m[2]), "d"(m[3]), "d"(best));
  return out;
}
__device__ __forceinline__ unsigned any_gt4(unsigned flag, const double (&m)[4], double best) {
  unsigned out;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "setp.gt.or.f64 p, %2, %6, p;\n\t"
      "setp.gt.or.f64 p, %3, %6, p;\n\t"
      "setp.gt.or.f64 p, %4, %6, p;\n\t"
      "setp.gt.or.f64 p, %5, %6, p;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(out)
      : "r"(flag), "d"(m[0]), "d"(m[1]), "d"(m[2]), "d"(m[3]), "d"(best));
  return out;
}

// Field launch extensions.
// Sub-transform mapping of a pruned large-N field (afd_pruned.cuh): the
// kernel's "signals" are the Q = N_big / N pre-twiddled spectra of one
// N_big-point row set, so signal q's output p is the big field's position
// j = q + Q p of row s (flat s N_big + j), and rows at or above *lim (the
// first row whose weight tail is not negligible, prune_rows_kernel) are
// left to the two-pass path.  Default: identity (flat s N + j, no limit).
// cand2 (fast mode): per CTA slot, the largest |F|^2 of the CTA's grid
// points other than its candidate's — the runner-up, from which the step
// kernels report the step's top-2 relative margin.
struct SubMap {
  long long row_stride;  // flat index row stride (0: N)
  int q_mul;             // 0: j = p; else j = blockIdx.y + q_mul * p
  const int* lim;        // device row limit (rows >= *lim skipped) or null
  double* cand2;         // [batch][gridDim.x] runner-up magnitudes or null
  const int* lim_lo;     // device lower row limit (rows < *lim_lo skipped) or null
  unsigned long long* hint;  // max-reduced bits of the launch's largest |F|^2 (margins: runner-up)
                             // for the screens of later tiers (afd_field_reg.cuh), or null
  // batches of on-chip fields with register tiers (pruned_small): the limits
  // and the hint are per signal (lim[sig * lim_stride], hint[sig]) and the
  // candidates of signal `sig` go to cand_out[sig * cand_stride + slot]
  int lim_stride;            // 0: one limit / hint for the launch
  int cand_stride;           // 0: gridDim.x
  int cand_off;              // first slot of the launch in a signal's candidate row
};
__device__ __forceinline__ size_t cand_slot(const SubMap& sub, int sig) {
  return (size_t)sig * (sub.cand_stride ? (unsigned)sub.cand_stride : gridDim.x) + blockIdx.x;
}

// First maximum of a CTA's candidates and the runner-up: the largest of
// the threads' runner-ups and of their maxima other than the winner.
__device__ __forceinline__ double cta_runner_up(double sec, double mag, long long flat,
                                                long long win_flat, double* red2) {
  double x = fmax(sec, flat != win_flat ? mag : -1.0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red2[wid] = x;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double y = -1.0;
  for (int w = 0; w < nw; ++w) y = fmax(y, red2[w]);
  return y;
}

// MARG (with FAST): track the runner-up into sub.cand2 (AFD_PLAN_MARGINS).
template <int K, int RB, int G, bool MATERIALIZE, bool TM = false, bool FAST = false,
          bool MARG = false>
__global__ void __launch_bounds__(Geo<K, RB>::T * G, (RB <= 3 && Geo<K, RB>::T * G <= 512) ? 2 : 1)
field_kernel(const double2* __restrict__ ghat,     // [batch][N]
             const double* __restrict__ pw,        // [rows of plan][N], r^l natural l (FAST: fw)
             const double* __restrict__ scales,    // [M] (global radius index)
             const double2* __restrict__ twst,     // stage twiddle tables (N-1)
             long long row0, long long row1,       // global rows to evaluate
             long long pw_row0,                    // global row of pw[0]
             Cand* __restrict__ cand_out,          // [batch][gridDim.x]
             double2* __restrict__ field_out,      // [row1-row0][N] (MATERIALIZE)
             const State* __restrict__ state,      // per-signal stop flags or null
             const double2* __restrict__ tw_img,   // SmemTw<K,RB> image (one bulk copy)
             int pp,                               // 1: offset the row-groups (FieldHook)
             unsigned* __restrict__ row_ctr,       // dynamic rows: [batch][2] counters or null
             int launch_id,                        // selects / resets the counter pair
             SubMap sub) {                         // pruned large-N mapping (launched without PDL)
  using Gm = Geo<K, RB>;
  constexpr int N = Gm::N, T = Gm::T, P = Gm::P;
  extern __shared__ double2 smem[];
  const int sig = blockIdx.y;
  const int g = threadIdx.x / T;
  const int tp = threadIdx.x % T;
  const int Gr = blockDim.x / T;  // row-groups actually launched (<= G)
  using TwT = SmemTw<K, RB>;
  if (sub.lim_lo != nullptr) {  // pruned tier: rows below *lim_lo belong to a shorter tier
    const long long l = sub.lim_lo[(size_t)sig * sub.lim_stride];
    if (l > row0) row0 = l < row1 ? l : row1;
  }
  if (sub.lim != nullptr && sub.lim[(size_t)sig * sub.lim_stride] <= row0) {
    // pruned launch with no on-chip rows this step (all rows long, or the
    // signal stopped): a neutral candidate, no TMEM or twiddle setup
    if (!MATERIALIZE && threadIdx.x == 0) {
      Cand c;
      c.mag = -1.0;
      c.flat = 0x7fffffffffffffffLL;
      c.re = c.im = 0.0;
      cand_out[cand_slot(sub, sig)] = c;
      if constexpr (MARG) sub.cand2[cand_slot(sub, sig)] = -1.0;
    }
    return;
  }
  FSTAMP(0, 0);
#ifdef AFD_FIELD_TIMING
  if (tp == 0 && blockIdx.x < 512 && g < 2) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_field_stamps[blockIdx.x][g][0][15] = smid;
  }
#endif
  // Twiddle image: one TMA bulk copy (issued by thread 0, completes on an
  // mbarrier) overlapping the first row's prologue loads.
  __shared__ unsigned long long tw_bar;
  __shared__ uint32_t tm_base;  // TMEM twiddle store (TM)
  if (threadIdx.x == 0) mbar_init(&tw_bar, 1);
  if constexpr (TM) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&tm_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if constexpr (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    constexpr unsigned bytes = sizeof(double2) * TwT::ENTRIES;
    const unsigned m = (unsigned)__cvta_generic_to_shared(&tw_bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
                 : "memory");
    constexpr unsigned chunk = 16384;
    for (unsigned off = 0; off < bytes; off += chunk) {
      const unsigned nb = bytes - off < chunk ? bytes - off : chunk;
      const unsigned d = (unsigned)__cvta_generic_to_shared((char*)smem + off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(d), "l"((const char*)tw_img + off), "r"(nb), "r"(m)
          : "memory");
    }
  }
  bool tw_ready = false;
  using TwSrc = std::conditional_t<TM, std::conditional_t<FAST, TmemTwCT, TmemTw>,
                                   std::conditional_t<FAST, SmemTwCT<K, RB>, TwT>>;
  TwSrc tw;
  // TMEM lanes follow the warp's quadrant (warp & 3): with T >= 128 every
  // group's warps cover all four quadrants in thread order, with T = 64 two
  // groups do, so the first kTmFill groups write the twiddles and spectrum
  [[maybe_unused]] constexpr int kTmFill = T >= 128 ? 1 : 128 / T;
  if constexpr (TM) {
    const int warp = threadIdx.x >> 5;
    // lane quadrant of the warp; one column set per 128 threads of a row
    // (tp >> 7): two sets at N = 4096 (T = 256), one for N = 1024, 2048
    // (shared by all groups)
    tw.base = tm_base + ((uint32_t)((warp & 3) * 32) << 16) +
              (uint32_t)((tp >> 7) * TmemTw::kSetCols);
  } else {
    tw.sm = smem;
  }
  double2* sm = smem + TwT::ENTRIES + g * Gm::SMEM;
  const double2* __restrict__ gh = ghat + (size_t)sig * N;
  // TM variant: rows after the first take the spectrum from TMEM (written by
  // group 0 during the first prologue) instead of re-reading it from L2
  // (measured c1 1.09e11 -> 1.12e11 evals/s; staging r^l in shared memory by
  // TMA as well was slower: the extra 32 KiB of shared memory costs L1)
  uint32_t gh_tm = 0;
  if constexpr (TM) {
    static_assert(TmemTw::kGhCol + 2 * 4 * P <= 512, "TMEM columns");
    const int warp = threadIdx.x >> 5;
    gh_tm = tm_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)TmemTw::kGhCol +
            (uint32_t)((tp >> 7) * (4 * P));
  }

  // Running first maximum.  Rows are visited in increasing s and, within a
  // row, a thread's outputs j = out_pos(tp, i) increase with i, so a strict
  // '>' keeps the lowest flat index among equal magnitudes; the flat index is
  // formed once at the end.
  double best_mag = -1.0, best_re = 0.0, best_im = 0.0;
  int best_sl = -1, best_i = 0;
  // fast mode with a runner-up slot: the screen lets through every value
  // above the runner-up (a value above it may become either of the two)
  constexpr bool track2 = FAST && MARG;
  [[maybe_unused]] double sec_mag = -1.0;

  // row counts fit 32 bits (M <= 2^31); 32-bit loop state keeps registers
  // for the butterflies
  if (sub.lim != nullptr) {
    const long long l = sub.lim[(size_t)sig * sub.lim_stride];
    if (l < row1) row1 = l > row0 ? l : row0;
  }
  const int rows = (int)(row1 - row0);
  const int per_round = (int)gridDim.x * Gr;
  // Row-groups of >= 32 threads synchronise on their own named barrier and
  // loop over their own rows independently, so the G rows of a CTA drift out
  // of phase (one group's loads overlap another's FP64 passes); smaller
  // groups share warps and step together with the whole block.
  constexpr bool kGroupSync = (T % 32 == 0) && G > 1;
  static_assert(!kGroupSync || T == 32 || G <= 15, "named barriers 1 + g must be < 16");
  const int rounds = kGroupSync ? (rows - ((int)blockIdx.x * Gr + g) + per_round - 1) / per_round
                                : (rows + per_round - 1) / per_round;
  // phase offset of group 1 (FieldHook): only when both groups have rows
  // (always for TM: group 1 reads the spectrum group 0 put in TMEM)
  const bool offset = kGroupSync && Gr == 2 && (pp > 0 || TM) &&
                      (int)blockIdx.x * Gr + 1 < rows;
  // Dynamic rows (row_ctr): each group's first row is static, later rows are
  // claimed from a per-launch counter (atomicAdd one row ahead), so groups
  // that start late or run slow take fewer rows.  Rows of a group still
  // increase, which the first-maximum tracking below relies on.
  const bool dyn = kGroupSync && row_ctr != nullptr;
  unsigned* ctr = dyn ? row_ctr + 2 * sig + (launch_id & 1) : nullptr;
  __shared__ int next_sl[2][2];  // [group][row parity]
  // First row: its r^l values are step-independent and are loaded before the
  // PDL wait; the spectrum and the stop flags come from the previous kernel.
  double2 v[P];
  constexpr int PWS = FAST ? FastW<K, RB>::STRIDE : N;  // table row stride
  {
    const long long s0 = row0 + (long long)blockIdx.x * Gr + g;
    const bool act0 = rounds > 0 && s0 < row1;
    double pv[P];
    if (act0) {
      const double* __restrict__ pr = pw + (size_t)(s0 - pw_row0) * PWS;
      if constexpr (FAST) {
        FastW<K, RB>::load(pr, tp, pv);
      } else {
#pragma unroll
        for (int i = 0; i < P; ++i) pv[i] = __ldg(pr + Gm::l0(tp, i));
      }
    }
    if constexpr (TM) {  // step-independent: fill TMEM before the PDL wait
      mbar_wait(&tw_bar, 0);
      tw_ready = true;
      if (g < kTmFill) {
        tw.template fill<K, RB, !FAST>(tp, TwT{smem});
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    pdl_wait();
    // the stop flag's load overlaps the spectrum loads (both are L2 round
    // trips on the critical path); the flag is tested once v is formed
    const int stopped = state != nullptr ? __ldcg(&state[sig].stopped) : 0;
    if (act0) {
      // all sixteen spectrum loads in flight before the first TMEM store (a
      // tcgen05.st is a memory barrier to the compiler: loads after one are
      // not hoisted above it)
#pragma unroll
      for (int i = 0; i < P; ++i) v[i] = __ldg(gh + Gm::l0(tp, i));
      if constexpr (TM) {
        if (g < kTmFill) {
#pragma unroll
          for (int i = 0; i < P; ++i) tm_st4(gh_tm + 4 * i, v[i]);
        }
      }
      if constexpr (FAST) {
        fast_prologue(v, pv);
      } else {
#pragma unroll
        for (int i = 0; i < P; ++i) v[i] = make_double2(pv[i] * v[i].x, pv[i] * v[i].y);  // transform.py:198
      }
#pragma unroll
      for (int i = 0; i < P; ++i) asm volatile("" ::"d"(v[i].x), "d"(v[i].y));  // formed before the test
      if constexpr (TM) {
        if (g < kTmFill) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
    if (stopped) {
      mbar_wait(&tw_bar, 0);  // no bulk copy may target an exited CTA
      if constexpr (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32)
          asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base)
                       : "memory");
      }
      return;
    }
    pdl_trigger();
    FSTAMP(0, 1);
    // the previous launch is complete: clear the next launch's counter
    if (dyn && threadIdx.x == 0 && blockIdx.x == 0) row_ctr[2 * sig + ((launch_id + 1) & 1)] = 0;
  }
  // TMEM variant with more than two groups (N = 2048): no one-pass offset
  // orders group 0's spectrum store before the others read it at their
  // second row, so the CTA synchronises once here
  if constexpr (TM && G > 2) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // row within [row0, row1); groups that share warps (no kGroupSync) step
  // through `rounds` together with inactive tails masked
  int sl = (int)blockIdx.x * Gr + g;
  for (int rd = 0; kGroupSync ? sl < rows : rd < rounds; ++rd) {
    const long long s = row0 + sl;
    const bool active = kGroupSync || sl < rows;
    unsigned claim = 0;
    if (dyn && tp == 0) claim = atomicAdd(ctr, 1u);
    if (rd > 0 && active) {
      // prologue: y = powers * c[rev] (transform.py:198), per component
      if constexpr (TM) {
        const double* __restrict__ pr = pw + (size_t)(s - pw_row0) * PWS;
        // all r^l loads issued before the TMEM reads (tcgen05.wait::ld is a
        // memory barrier to the compiler: loads placed after one cannot be
        // hoisted above it)
        double pv[P];
        if constexpr (FAST) {
          FastW<K, RB>::load(pr, tp, pv);
        } else {
#pragma unroll
          for (int i = 0; i < P; ++i) pv[i] = __ldg(pr + Gm::l0(tp, i));
        }
#pragma unroll
        for (int i0 = 0; i0 < P; i0 += 4) {
          uint32_t r[16];
          tm_ld<16>(gh_tm + 4 * i0, r);
          tm_wait_ld();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double2 c = make_double2(__hiloint2double(r[4 * j + 1], r[4 * j]),
                                           __hiloint2double(r[4 * j + 3], r[4 * j + 2]));
            if constexpr (FAST) {
              v[i0 + j] = c;
            } else {
              const double p = pv[i0 + j];
              v[i0 + j] = make_double2(p * c.x, p * c.y);
            }
          }
        }
        if constexpr (FAST) fast_prologue(v, pv);
      } else {
        const double* __restrict__ pr = pw + (size_t)(s - pw_row0) * PWS;
        if constexpr (FAST) {
          double pv[P];
          FastW<K, RB>::load(pr, tp, pv);
#pragma unroll
          for (int i = 0; i < P; ++i) v[i] = __ldg(gh + Gm::l0(tp, i));
          fast_prologue(v, pv);
        } else {
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const int l = Gm::l0(tp, i);
            const double p = __ldg(pr + l);
            const double2 c = __ldg(gh + l);
            v[i] = make_double2(p * c.x, p * c.y);
          }
        }
      }
    }
    if (!tw_ready) {  // twiddle image landed (pass 0 reads it)
      mbar_wait(&tw_bar, 0);
      tw_ready = true;
    }
    FSTAMP(rd, 2);
    if constexpr (kGroupSync) {
      long long* st = nullptr;
#ifdef AFD_FIELD_TIMING
      if (tp == 0 && blockIdx.x < 512 && g < 2 && rd < 4) st = &g_field_stamps[blockIdx.x][g][rd][0];
#endif
      if (offset && rd == 0 && g == 1) {
        asm volatile("bar.sync 3, %0;" ::"r"(2 * T) : "memory");
        if constexpr (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const FieldHook hook{offset && rd == 0 && g == 0, 2 * T, st, TM,
                           (dyn && tp == 0) ? &next_sl[g][rd & 1] : nullptr, &claim, per_round};
      if constexpr (T == 32)
        fft_passes<K, true, RB>(v, tp, active, sm, tw, WarpSync{}, hook);
      else
        fft_passes<K, true, RB>(v, tp, active, sm, tw, GroupSync{1 + g, T}, hook);
    } else {
      fft_passes<K, true, RB>(v, tp, active, sm, tw);
    }
    const int sl_next = dyn ? next_sl[g][rd & 1] : sl + per_round;
    if (active) {
      const double sc = FAST ? 1.0 : __ldg(scales + s);  // FAST: scale is in the weights
      if (MATERIALIZE) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
          // y *= scales[:, None] (transform.py:200)
          const double2 f = FAST ? v[i] : make_double2(v[i].x * sc, v[i].y * sc);
          field_out[(size_t)(s - row0) * N + out_pos<K, RB>(tp, i)] = f;
        }
      } else if constexpr (FAST) {
        // Running first maximum.  A thread's maximum rarely improves after
        // the first rows, so the row is screened with one compare per point
        // (predicate-accumulating setp) and only a row with a new maximum
        // pays for the selects, recomputing |F|^2 (the same operations).
        // (Exact mode keeps the per-point selects: the screen spills there.)
        unsigned up = 0;
#pragma unroll
        for (int i0 = 0; i0 < P; i0 += 4) {
          double mg[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) mg[i] = fast_mag2(v[i0 + i]);
          up = any_gt4(up, mg, track2 ? sec_mag : best_mag);
        }
        if (__builtin_expect(up != 0, 0)) {
#pragma unroll
          for (int i = 0; i < P; ++i) {
            // recompute (do not keep P magnitudes live across the screen)
            double2 f = v[i];
            asm volatile("" : "+d"(f.x), "+d"(f.y));
            const double mg = fast_mag2(f);
            if constexpr (track2) {
              if (mg > best_mag) {
                sec_mag = best_mag;
                best_mag = mg;
                best_re = f.x;
                best_im = f.y;
                best_sl = sl;
                best_i = i;
              } else if (mg > sec_mag) {
                sec_mag = mg;
              }
            } else if (mg > best_mag) {
              best_mag = mg;
              best_re = f.x;
              best_im = f.y;
              best_sl = sl;
              best_i = i;
            }
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < P; ++i) {
          // y *= scales[:, None] (transform.py:200)
          const double2 f = make_double2(v[i].x * sc, v[i].y * sc);
          const double mg = np_mag2(f);  // core.py:298
          if (__builtin_expect(mg > best_mag, 0)) {
            best_mag = mg;
            best_re = f.x;
            best_im = f.y;
            best_sl = sl;
            best_i = i;
          }
        }
      }
    }
    FSTAMP(rd, 14);
    sl = sl_next;
  }
  if constexpr (TM) {  // all TMEM reads done: release the columns
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base)
                   : "memory");
  }
  if (MATERIALIZE) return;
  __syncthreads();  // all groups done before the block-wide reduction
  Cand best;
  best.mag = best_mag;
  if (best_sl >= 0) {
    const long long j = out_pos<K, RB>(tp, best_i);
    best.flat = (row0 + best_sl) * (sub.row_stride ? sub.row_stride : (long long)N) +
                (sub.q_mul ? (long long)sig + (long long)sub.q_mul * j : j);
  } else {
    best.flat = 0x7fffffffffffffffLL;
  }
  best.re = best_re;
  best.im = best_im;
  [[maybe_unused]] const double own_mag = best.mag;
  [[maybe_unused]] const long long own_flat = best.flat;
  // CTA reduction of the candidates (first maximum).
  __shared__ Cand red[32];
  __shared__ long long win_flat;
  best = warp_argmax(best);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = best;
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    Cand c = lane < nw ? red[lane] : best;
    c = warp_argmax(c);
    if (lane == 0) {
      cand_out[cand_slot(sub, sig)] = c;
      if constexpr (track2) win_flat = c.flat;
      // non-negative doubles order like their bit patterns
      if (!track2 && sub.hint && c.mag > 0.0)
        atomicMax(sub.hint + (sub.lim_stride ? sig : 0),
                  (unsigned long long)__double_as_longlong(c.mag));
    }
  }
  if constexpr (track2) {
    __shared__ double red2[32];
    __syncthreads();
    const double r2 = cta_runner_up(sec_mag, own_mag, own_flat, win_flat, red2);
    if (threadIdx.x == 0) {
      sub.cand2[cand_slot(sub, sig)] = r2;
      if (sub.hint && r2 > 0.0)
        atomicMax(sub.hint + (sub.lim_stride ? sig : 0),
                  (unsigned long long)__double_as_longlong(r2));
    }
  }
}

// ---------------------------------------------------------------------------
// Shared helpers for the one-CTA-per-signal kernels.
// ---------------------------------------------------------------------------

// Forward (INV=false) or inverse transform of the row held in `buf`
// (natural order, swizzled), result written to `out` (natural order,
// global).  For the inverse, SCALE_N applies `y /= n` (transform.py:133).
template <int K, bool INV, bool SCALE_N, class Tw>
__device__ void row_transform(double2* buf, const Tw& tw, double2* __restrict__ out) {
  using Gm = Geo<K>;
  constexpr int T = Gm::T, P = Gm::P;
  const int tp = threadIdx.x;
  const bool active = tp < T;
  double2 v[P];
  if (active) {
#pragma unroll
    for (int i = 0; i < P; ++i) v[i] = buf[Gm::sw(Gm::l0(tp, i))];
  }
  __syncthreads();
  fft_passes<K, INV>(v, tp, active, buf, tw);
  if (active) {
    const double2 dn = make_double2((double)Gm::N, 0.0);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      double2 y = v[i];
      if (SCALE_N) y = np_cdiv(y, dn);
      out[out_pos<K>(tp, i)] = y;
    }
  }
  __syncthreads();
}

template <int K, bool SMEM>
__device__ __forceinline__ auto make_tw(double2* sm, const double2* __restrict__ st) {
  if constexpr (SMEM) {
    return SmemTw<K>{sm};
  } else {
    return GlobalTw{st};
  }
}

template <int K>
struct SwIdx {
  __device__ __forceinline__ int operator()(int i) const { return Geo<K>::sw(i); }
};
struct PlainIdx {
  __device__ __forceinline__ int operator()(int i) const { return i; }
};

// Shared-memory layout of the one-CTA-per-signal kernels.
// Twiddles go to shared memory when they fit beside the row buffers
// (all N <= 4096); N = 8192 reads the global stage tables.
template <int K>
struct RowSmemBase {
  static constexpr int N = 1 << K;
  static constexpr size_t rest = sizeof(double2) * Geo<K>::SMEM + sizeof(double) * N +
                                 sizeof(double) * 2 * (N / 8 + 16);
  static constexpr bool smem_tw = sizeof(double2) * SmemTw<K>::ENTRIES + rest <= 200 * 1024;
};

template <int K>
struct RowSmem {
  static constexpr int N = 1 << K;
  static constexpr bool smem_tw = RowSmemBase<K>::smem_tw;
  static constexpr size_t tw = 0;                                   // SmemTw<K> (if smem_tw)
  static constexpr size_t buf = smem_tw ? sizeof(double2) * SmemTw<K>::ENTRIES : 0;  // N double2
  static constexpr size_t mag = buf + sizeof(double2) * Geo<K>::SMEM;  // N double
  static constexpr size_t scratch = mag + sizeof(double) * N;       // 2*(N/8+16) double
  static constexpr size_t bytes = scratch + sizeof(double) * 2 * (N / 8 + 16);
};

// ---------------------------------------------------------------------------
// step_kernel: one CTA per signal.
//   k < 0  : initialise (copy g0, initial energy, forward transform)
//   k >= 0 : select / update / energy / record / stop / forward transform
// ---------------------------------------------------------------------------
template <int K, bool MARG = false>
__global__ void __launch_bounds__(Geo<K>::T < 64 ? 64 : Geo<K>::T)
step_kernel(int k, int max_terms, double threshold, int dc_first,
            const double2* __restrict__ g0,       // [batch][N] (init only)
            double2* __restrict__ rem,            // [batch][N] remainder G_k
            double2* __restrict__ ghat,           // [batch][N] DFT(G_k)
            const Cand* __restrict__ cand,        // [batch][ncand]
            int ncand,
            const double* __restrict__ radii,     // [M] global
            const double2* __restrict__ circle,   // [N] z_m
            const double2* __restrict__ twst,
            State* __restrict__ state,            // [batch]
            Step* __restrict__ steps,             // [batch][max_terms]
            const double* __restrict__ pow2,      // [M][kPowRow] (kernel_norm_grid)
            const double* __restrict__ cand2) {   // [batch][ncand] runner-ups or null
  constexpr int N = 1 << K;
  using L = RowSmem<K>;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* buf = reinterpret_cast<double2*>(smraw + L::buf);
  double* mag = reinterpret_cast<double*>(smraw + L::mag);
  double* scratch = reinterpret_cast<double*>(smraw + L::scratch);
  double2* twsm = reinterpret_cast<double2*>(smraw + L::tw);
  __shared__ Cand red[32];
  __shared__ int s_stop;
  using TwT = typename std::conditional<L::smem_tw, SmemTw<K>, GlobalTw>::type;
  const TwT tw = make_tw<K, L::smem_tw>(twsm, twst);
  const SwIdx<K> SW;
  const int sig = blockIdx.x;
  State& st = state[sig];
  double2* __restrict__ r = rem + (size_t)sig * N;
  double2* __restrict__ gh = ghat + (size_t)sig * N;

  if (L::smem_tw) SmemTw<K>::load(twsm, twst);  // visible after the next barrier
  pdl_wait();  // candidates, state and the remainder come from earlier kernels
  pdl_trigger();
  if (k < 0) {
    const double2* __restrict__ x = g0 + (size_t)sig * N;
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
      const double2 v = x[m];
      r[m] = v;
      buf[SW(m)] = v;
      mag[m] = np_mag2(v);
    }
    __syncthreads();
    // discrete_energy (core.py:195-198): np.mean(re**2 + im**2)
    const double e0 = pairwise_sum_block(mag, N, scratch, PlainIdx()) / (double)N;
    if (threadIdx.x == 0) {
      st.initial = e0;
      st.nsteps = 0;
      st.flags = 0;
      st.stopped = (e0 == 0.0) ? 1 : 0;  // core.py:366-368
      s_stop = st.stopped;
    }
    __syncthreads();
    if (!s_stop) row_transform<K, false, false>(buf, tw, gh);
    return;
  }

  if (st.stopped) return;  // block-uniform
  long long s = 0, j = 0;
  double radius = 0.0;
  double2 a = make_double2(0.0, 0.0), coeff;
  double runner = -2.0;  // -2: not tracked
  if (k == 0 && dc_first) {
    // core.py:373-375: a = 0, coeff = complex(np.mean(remainder))
    for (int m = threadIdx.x; m < N; m += blockDim.x) buf[SW(m)] = r[m];
    __syncthreads();
    const double2 sum = cpairwise_sum_block(buf, N, scratch, SW);
    coeff = np_cdiv(sum, make_double2((double)N, 0.0));
  } else {
    // first maximum over the candidates (np.argmax, core.py:299)
    Cand b;
    b.mag = -1.0;
    b.flat = 0x7fffffffffffffffLL;
    b.re = b.im = 0.0;
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) cand_merge(b, cand[(size_t)sig * ncand + i]);
    b = warp_argmax(b);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = b;
    __syncthreads();
    if (wid == 0) {
      Cand c = lane < (int)(blockDim.x >> 5) ? red[lane] : b;
      c = warp_argmax(c);
      if (lane == 0) red[0] = c;
    }
    __syncthreads();
    b = red[0];
    if constexpr (MARG) {  // the step's runner-up (AFD_PLAN_MARGINS)
      double r = -1.0;
      for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
        const Cand x = cand[(size_t)sig * ncand + i];
        r = fmax(r, cand2[(size_t)sig * ncand + i]);
        if (x.flat != b.flat) r = fmax(r, x.mag);
      }
      runner = block_max(r);
    }
    s = b.flat / N;
    j = b.flat % N;
    radius = radii[s];
    // grid.point (core.py:163-167): r * exp(2 pi i j / N) == (r Re z_j, r Im z_j)
    const double2 zj = circle[j];
    a = make_double2(radius * zj.x, radius * zj.y);
    coeff = make_double2(b.re, b.im);
  }

  // remainder_update (core.py:303-314) + kernel_samples (core.py:234-238)
  int amb = 0;
  const double kn = kernel_norm_grid(a, radius, pow2 ? pow2 + (size_t)s * kPowRow : nullptr, &amb);
  const double2 sc = make_double2(kn, 0.0);
  constexpr bool elide = (size_t)N * 16 >= 256 * 1024;  // numpy temporary elision
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    const double2 z = circle[m];
    const double2 d = one_minus_conja_z(a, z);
    const double2 e = np_cdiv(sc, d);
    const double2 ce = elide ? np_cmul(e, coeff) : np_cmul(coeff, e);
    const double2 g = r[m];
    const double2 stp = make_double2(g.x - ce.x, g.y - ce.y);
    const double2 num = elide ? np_cmul(d, stp) : np_cmul(stp, d);
    const double2 den = make_double2(z.x - a.x, z.y - a.y);
    const double2 out = np_cdiv(num, den);
    r[m] = out;
    buf[SW(m)] = out;
    mag[m] = np_mag2(out);
  }
  __syncthreads();
  const double residual = pairwise_sum_block(mag, N, scratch, PlainIdx()) / (double)N;
  if (threadIdx.x == 0) {
    Step rec;
    rec.s = s;
    rec.j = j;
    rec.radius = radius;
    rec.a_re = a.x;
    rec.a_im = a.y;
    rec.c_re = coeff.x;
    rec.c_im = coeff.y;
    rec.residual = residual;
    rec.flags = amb ? kStepPowAmbiguous : 0;
    rec.margin = runner >= -1.0 ? top2_margin(coeff_mag2(coeff), runner) : __int_as_float(0x7fc00000);
    steps[(size_t)sig * max_terms + k] = rec;
    st.nsteps = k + 1;
    st.flags |= rec.flags;
    int stop = 0;
    if (threshold > 0.0 && residual <= threshold * st.initial) stop = 1;  // core.py:386-387
    if (residual == 0.0) stop = 1;                                         // core.py:388-389
    if (k + 1 >= max_terms) stop = 1;
    st.stopped = stop;
    s_stop = stop;
  }
  __syncthreads();
  if (!s_stop) row_transform<K, false, false>(buf, tw, gh);
}

// ---------------------------------------------------------------------------
// Standalone transforms, one CTA per signal.
//   mode 0: dft_forward   mode 1: dft_inverse   mode 2: analytic projection
//   (real input given as complex with zero imaginary part)
// ---------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(Geo<K>::T < 64 ? 64 : Geo<K>::T)
fft_kernel(int mode, const double2* __restrict__ x, double2* __restrict__ y,
           const double2* __restrict__ twst) {
  constexpr int N = 1 << K;
  using L = RowSmem<K>;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* buf = reinterpret_cast<double2*>(smraw + L::buf);
  double2* twsm = reinterpret_cast<double2*>(smraw + L::tw);
  if (L::smem_tw) SmemTw<K>::load(twsm, twst);
  using TwT = typename std::conditional<L::smem_tw, SmemTw<K>, GlobalTw>::type;
  const TwT tw = make_tw<K, L::smem_tw>(twsm, twst);
  const SwIdx<K> SW;
  const double2* __restrict__ xs = x + (size_t)blockIdx.x * N;
  double2* __restrict__ ys = y + (size_t)blockIdx.x * N;
  for (int m = threadIdx.x; m < N; m += blockDim.x) buf[SW(m)] = xs[m];
  __syncthreads();
  if (mode == 0) {
    row_transform<K, false, false>(buf, tw, ys);
  } else if (mode == 1) {
    row_transform<K, true, true>(buf, tw, ys);
  } else {
    // core.py:224-231: spectrum = dft_forward(x); spectrum[1:half] *= 2;
    // spectrum[half+1:] = 0; dft_inverse(spectrum)
    row_transform<K, false, false>(buf, tw, ys);
    constexpr int half = N / 2;
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
      double2 v = ys[m];
      if (m >= 1 && m < half) v = make_double2(v.x * 2.0, v.y * 2.0);
      if (m > half) v = make_double2(0.0, 0.0);
      buf[SW(m)] = v;
    }
    __syncthreads();
    row_transform<K, true, true>(buf, tw, ys);
  }
}

}  // namespace afd
