// afd_pruned.cuh — the fast large-N field as on-chip 4096-point transforms
// (AFD_PLAN_FAST, N = 2^K > 8192; BASELINE c2, c4).
//
// The field of row s is F_s(j) = scale_s sum_l r_s^l G^_l e^{+2 pi i l j / N}
// (transform.py:185-201).  Its weights decay geometrically, so for all but
// the radii closest to 1 the terms l >= L = 4096 are far below the
// transform's own rounding: with T = max_l |G^_l| and
// B_s = max_{l < L} r_s^l |G^_l| (the largest kept term),
//     |sum_{l >= L} r^l G^_l e^{..}| <= T r^L / (1 - r) <= 2^-64 B_s
// is ~2^-11 of the FP64 rounding error of any N-point transform of the row
// (>= 2^-53 B_s per stage).  For such a row, split j = q + Q p (Q = N / L):
//     F_s(q + Q p) = scale_s sum_{l < L} r_s^l (G^_l e^{2 pi i l q / N}) e^{2 pi i l p / L},
// an L-point inverse transform of the pre-twiddled spectrum
// g^(q)_l = G^_l e^{2 pi i l q / N}, which does not depend on the row.  So
// the field over the prunable rows is the N = 4096 field kernel run on a
// batch of Q spectra g^(q) with the big plan's radii and scales: on chip,
// no row-batch intermediate in HBM, 12 butterfly stages instead of 20.
// Rows whose tail beyond L = 1024 is already negligible (~96% of r_m = m/M
// at c4) run as N/1024 1024-point fields instead (prune_k).
// Rows that fail the test (the last ~1% of r_m = m/M at c4) keep the
// two-pass path (pass A + TMA column pass), limited on the device to rows
// at or above the first failing row, so the loop stays free of host syncs
// and graph-capturable.  The fast engine's contract (identical grid
// indices, 1e-9 relative) is unchanged; exact mode never prunes.
#pragma once

#include "afd_big.cuh"

namespace afd {

// On-chip sub-transform tiers, by the number of spectrum terms L a row needs
// (its tail beyond l = L negligible): L = 32, 64 and 128 run in registers,
// one thread per 32 outputs and no exchange at all (afd_field_reg.cuh: 70%
// of r_m = m/M), L = 256 and 512 as N/L L-point fields on 8 or 16 threads
// each (afd_field_sub.cuh), L = 1024 as N/1024 1024-point fields (one warp
// per row, afd_field_warp.cuh), L = 4096 as N/4096 4096-point fields, the
// rest two-pass.  mstar[t] = first row failing tier t's test; tiers are nested
// (a row failing a longer tier fails every shorter one), so mstar[] is
// non-decreasing and tier t takes rows [mstar[t-1], mstar[t]).
constexpr int kPruneTiers = 7;
constexpr int kRegTiers = 3;  // tiers 0..2: the register kernels (D = 1, 2, 4 blocks of 32 terms)
constexpr int kTierSub = 3;   // tiers 3, 4: 256- and 512-point sub-warp fields
constexpr int kTier1k = 5, kTier4k = 6;
__host__ __device__ constexpr int prune_k(int t) {
  return t < kRegTiers ? 5 + t : t == 3 ? 8 : t == 4 ? 9 : t == kTier1k ? 10 : 12;
}
constexpr int kPruneK = 12;  // the longest tier (the spectrum head staged by prune_rows)

// mstar[t] = m1 (tiers below `first`: m0, switched off), *tmax = 0 (the tail
// maximum is max-reduced on its bits), *hint = 0 (the screening hint of the
// register tiers, afd_field_reg.cuh)
__global__ void prune_init_kernel(int* mstar, long long m0, long long m1, int first,
                                  unsigned long long* tmax, unsigned long long* hint) {
  for (int t = 0; t < kPruneTiers; ++t) mstar[t] = (int)(t < first ? m0 : m1);
  *tmax = 0ull;
  *hint = 0ull;
}

// T^2 = max_l |G^_l|^2 over the whole spectrum (an upper bound of the tail's)
__global__ void prune_tail_kernel(const double2* __restrict__ ghat, long long n,
                                  unsigned long long* tmax) {
  double m = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldg(ghat + i);
    m = fmax(m, fma(v.x, v.x, v.y * v.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(tmax, (unsigned long long)__double_as_longlong(m));
}

// G^_l of a large-N plan's field spectrum (pass-A layout, big_pass_col
// out_mode 4: position rev(l) permuted by perm_of_pos)
__device__ __forceinline__ double2 spectrum_at(const double2* __restrict__ ghat_perm, int l,
                                               int K, int ka) {
  return __ldg(ghat_perm + perm_of_pos(brev_rt(l, K), ka));
}

// First row s in [m0, m1) whose tail is not negligible, per tier t:
//   log2 T + L_t log2 r - log2(1 - r) > log2 B_s(L_t) - 64 -> atomicMin(mstar[t], s),
// B_s(L) = max_{l < L} r^l |G^_l|.  One warp per row; the CTA stages
// log2 |G^_l| (l < 4096, natural order from the permuted spectrum) in
// shared memory.  A stopped signal pins every mstar[t] to m0 (and the field
// kernels then do nothing).
__global__ void __launch_bounds__(256) prune_rows_kernel(
    int K, int ka, const double2* __restrict__ ghat_rev, const double* __restrict__ radii, long long m0,
    long long m1, const unsigned long long* __restrict__ tmax, const int* __restrict__ stopped,
    int* mstar) {
  constexpr int L = 1 << kPruneK;
  __shared__ double lg[L];
  if (stopped && *stopped) {
    if (blockIdx.x == 0 && threadIdx.x < kPruneTiers) atomicMin(mstar + threadIdx.x, (int)m0);
    return;
  }
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    const double2 v = spectrum_at(ghat_rev, l, K, ka);
    const double a2 = fma(v.x, v.x, v.y * v.y);
    lg[l] = a2 > 0.0 ? 0.5 * log2(a2) : -INFINITY;
  }
  __syncthreads();
  const double t2 = __longlong_as_double((long long)*tmax);
  const double lt = t2 > 0.0 ? 0.5 * log2(t2) : -INFINITY;
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long s = m0 + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < m1;
       s += warps) {
    const double r = radii[s];
    if (r == 0.0 || lt == -INFINITY) continue;  // no tail at all
    const double lr = log2(r), l1r = log2(1.0 - r);
    double b = -INFINITY;
    int lo = 0;
#pragma unroll
    for (int t = 0; t < kPruneTiers; ++t) {
      const int L_t = 1 << prune_k(t);
      for (int l = lo + lane; l < L_t; l += 32) b = fmax(b, fma((double)l, lr, lg[l]));
      lo = L_t;
      double bt = b;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bt = fmax(bt, __shfl_xor_sync(0xffffffffu, bt, o));
      const double tail = lt + (double)L_t * lr - l1r;
      // (warp-uniform) a row that passes a tier passes every longer one: the
      // tail bound falls and the kept maximum grows with L
      if (tail <= bt - 64.0) break;
      if (lane == 0) atomicMin(mstar + t, (int)s);
    }
  }
}

// g^(q)_l = G^_l e^{+2 pi i l q / N}, q < N / L, l < L = 2^kl (q-major,
// natural l); the root is the plan's circle table exp(2 pi i m / N)
// (core.py:87).
__global__ void pretwiddle_kernel(int K, int ka, int kl, const double2* __restrict__ ghat_rev,
                                  const double2* __restrict__ circle, double2* __restrict__ out,
                                  const int* __restrict__ stopped) {
  if (stopped && *stopped) return;
  const int L = 1 << kl;
  const long long n = 1LL << K, total = n;  // (N / L) * L entries
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const long long q = x >> kl;
    const int l = (int)(x & (L - 1));
    const double2 g = spectrum_at(ghat_rev, l, K, ka);
    const double2 w = __ldg(circle + (((long long)l * q) & (n - 1)));
    out[x] = make_double2(fma(g.x, w.x, -(g.y * w.y)), fma(g.x, w.y, g.y * w.x));
  }
}

// The register tiers' spectra (afd_field_reg.cuh): for q' < Q' = N / 32,
// register i < 32 and block m < D,
//   h[(m 32 + i) Q' + q'] = G^_l e^{+2 pi i l q' / N},  l = rev5(i) + 32 m
// (q' fastest: thread q' of the field kernel reads its 32 D values coalesced).
__global__ void pretwiddle_reg_kernel(int K, int ka, int D, const double2* __restrict__ ghat_rev,
                                      const double2* __restrict__ circle,
                                      double2* __restrict__ out, const int* __restrict__ stopped) {
  if (stopped && *stopped) return;
  const int kq = K - 5;
  const long long n = 1LL << K, qmask = (1LL << kq) - 1, total = (long long)D << K;
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const long long q = x & qmask;
    const int im = (int)(x >> kq);
    const int l = (int)(__brev((unsigned)(im & 31)) >> 27) + 32 * (im >> 5);
    const double2 g = spectrum_at(ghat_rev, l, K, ka);
    const double2 w = __ldg(circle + (((long long)l * q) & (n - 1)));
    out[x] = make_double2(fma(g.x, w.x, -(g.y * w.y)), fma(g.x, w.y, g.y * w.x));
  }
}

// Batches of on-chip fields (N <= 8192, many signals: BASELINE c3) with the
// register tiers and (N >= 4096: gl.g[] != null) the 256-, 512- and
// 1024-point tiers: one CTA per signal decides the signal's tier limits
// mstar[sig][t], t < kSmallTiers (the same tail test as prune_rows_kernel;
// without the longer tiers their limits repeat the last register tier's; a
// stopped signal: every limit m0, and the field kernels then do nothing),
// clears its hint and writes its pre-twiddled spectra
//   h[sig][(m 32 + i) Q' + q'] = G^_l e^{+2 pi i l q' / N},  l = rev5(i) + 32 m,  m < 4,
//   gl.g[u][sig][q][l] = G^_l e^{+2 pi i l q / N},  q < N / L_u,  l < L_u = 256 << u
// (natural-order spectrum, [batch][N]).  Rows from the last limit on stay
// with the N-point field kernel (SubMap::lim_lo).  One thread per row;
// rlog[s - m0] = {log2 r_s, log2(1 - r_s)} is tabulated at plan time (-inf
// for r = 0: no tail at all).
constexpr int kSmallTiers = kTier1k + 1;  // limits per signal: tiers 0 .. kTier1k
struct SmallSpectra {
  double2* g[3];  // L = 256, 512, 1024 (null: tier not used)
};
__global__ void __launch_bounds__(256) prune_small_kernel(
    int K, const double2* __restrict__ ghat, const double2* __restrict__ rlog, long long m0,
    long long m1, const double2* __restrict__ circle, const State* __restrict__ state,
    int* __restrict__ mstar, unsigned long long* __restrict__ hint, double2* __restrict__ h,
    SmallSpectra gl) {
  constexpr int L = 128;  // terms of the longest register tier
  constexpr int LG = 1 << prune_k(kTier1k);  // 1024: the longest tier tested here
  static_assert(LG == 1024 && kTier1k == kRegTiers + 2, "tiers 256, 512, 1024 follow the register tiers");
  __shared__ double lg[LG];
  __shared__ double wmax[8];
  __shared__ int ms[kSmallTiers];
  const int ntier = gl.g[2] ? kSmallTiers : kRegTiers;
  const int sig = blockIdx.x;
  const int n = 1 << K, kq = K - 5, qn = 1 << kq;
  const double2* __restrict__ gh = ghat + (size_t)sig * n;
  if (threadIdx.x == 0) hint[sig] = 0ull;
  if (state && state[sig].stopped) {
    if (threadIdx.x < kSmallTiers) mstar[sig * kSmallTiers + threadIdx.x] = (int)m0;
    return;
  }
  if (threadIdx.x < kSmallTiers) ms[threadIdx.x] = (int)m1;
  double m = 0.0;
  for (int l = threadIdx.x; l < n; l += blockDim.x) {
    const double2 v = __ldg(gh + l);
    const double a2 = fma(v.x, v.x, v.y * v.y);
    m = fmax(m, a2);
    if (l < LG) lg[l] = a2 > 0.0 ? 0.5 * log2(a2) : -INFINITY;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  double t2 = 0.0;
  for (int w = 0; w < 8; ++w) t2 = fmax(t2, wmax[w]);
  const double lt = t2 > 0.0 ? 0.5 * log2(t2) : -INFINITY;
  for (long long s = m0 + threadIdx.x; s < m1 && lt != -INFINITY; s += blockDim.x) {
    const double2 rl = __ldg(rlog + (s - m0));
    if (rl.x == -INFINITY) continue;  // r = 0: no tail at all
    double b = -INFINITY;
    int lo = 0;
    for (int t = 0; t < ntier; ++t) {
      const int L_t = 1 << prune_k(t);
      // four independent maxima (the loop is a latency chain otherwise)
      double b0 = b, b1 = b, b2 = b, b3 = b;
      for (int l = lo; l < L_t; l += 4) {
        b0 = fmax(b0, fma((double)l, rl.x, lg[l]));
        b1 = fmax(b1, fma((double)(l + 1), rl.x, lg[l + 1]));
        b2 = fmax(b2, fma((double)(l + 2), rl.x, lg[l + 2]));
        b3 = fmax(b3, fma((double)(l + 3), rl.x, lg[l + 3]));
      }
      b = fmax(fmax(b0, b1), fmax(b2, b3));
      lo = L_t;
      const double tail = lt + (double)L_t * rl.x - rl.y;
      if (tail <= b - 64.0) break;  // passes: it passes every longer tier as well
      atomicMin(ms + t, (int)s);
    }
  }
  __syncthreads();
  if (threadIdx.x < kSmallTiers) {
    // a row failing tier t fails every shorter one: limits are non-decreasing
    int v = ms[threadIdx.x < ntier ? threadIdx.x : ntier - 1];
    for (int t = threadIdx.x + 1; t < ntier; ++t) v = min(v, ms[t]);
    mstar[sig * kSmallTiers + threadIdx.x] = v;
  }
  double2* __restrict__ out = h + (size_t)sig * L * qn;
  for (int x = threadIdx.x; x < L * qn; x += blockDim.x) {
    const int q = x & (qn - 1), im = x >> kq;
    const int l = (int)(__brev((unsigned)(im & 31)) >> 27) + 32 * (im >> 5);
    const double2 g = __ldg(gh + l);
    const double2 w = __ldg(circle + ((l * q) & (n - 1)));
    out[x] = make_double2(fma(g.x, w.x, -(g.y * w.y)), fma(g.x, w.y, g.y * w.x));
  }
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    if (!gl.g[u]) continue;
    const int kl = 8 + u;
    double2* __restrict__ o1 = gl.g[u] + (size_t)sig * n;
    for (int x = threadIdx.x; x < n; x += blockDim.x) {
      const int q = x >> kl, l = x & ((1 << kl) - 1);
      const double2 g = __ldg(gh + l);
      const double2 w = __ldg(circle + ((l * q) & (n - 1)));
      o1[x] = make_double2(fma(g.x, w.x, -(g.y * w.y)), fma(g.x, w.y, g.y * w.x));
    }
  }
}

}  // namespace afd
