// afd_fft.cuh — the reference's radix-2 decimation-in-time transform
// (transform.py:73-93), executed on-chip for N = 2^K <= 8192.
//
// Exactness.  The reference runs log2(N) butterfly stages over a
// bit-reversed buffer; stage b (span 2^(b+1)) pairs positions p and
// p + 2^b (bit b of p clear) with twiddle w[(p mod 2^b) << (K-1-b)] of the
// numpy table w = exp(-2 pi i k/N), conjugated for the inverse direction:
//     t = hi * tw;  hi = lo - t;  lo = lo + t.
// The DAG of those butterflies fixes every rounding, but not who computes
// them or in which order independent butterflies run.  Here each thread
// holds 16 points in registers and executes 4 consecutive stages on them
// (a "pass"), exchanging through shared memory between passes.  Every
// butterfly is the same operation on the same operands with the same
// twiddle bits as in the reference, so outputs are bit-identical.
//
// Layout.  Pass j covers stage bits [4j, min(4j+4, K)); the thread's
// register index i supplies position bits [c, c+4) with c = b1 - 4, the
// thread index the rest:
//     pos(c, t, i) = (t & (2^c - 1)) | (i << c) | ((t >> c) << (c + 4)).
// In pass 0 (c = 0) physical thread t' plays logical thread rev(t'), so the
// bit-reversed input position (rev(t') << 4 | i) holds natural index
// l = (rev4(i) << (K-4)) | t': loads of G / Ghat / r^l are coalesced and
// no bit-reversal gather is needed.  Shared memory is addressed through
// SW(p) = p ^ ((p >> (K-3)) & 7), which makes every 16-byte exchange access
// of every pass conflict-free (each quarter-warp hits 8 distinct 16-B bank
// groups).  Twiddles come from per-stage tables S_b[k] = w[k << (K-1-b)]
// (offset 2^b - 1, N-1 entries total): warp-uniform in pass 0, consecutive
// across lanes later.
#pragma once

#include "afd_common.cuh"

namespace afd {

__host__ __device__ constexpr int brev_bits(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

template <int K>
struct Geo {
  static constexpr int N = 1 << K;
  static constexpr int RB = K >= 4 ? 4 : K;  // register (stage) bits per pass
  static constexpr int P = 1 << RB;          // points per thread
  static constexpr int T = N / P;            // threads per row
  static constexpr int TB = K - RB;          // thread-index bits
  static constexpr int NPASS = (K + 3) / 4;

  __device__ __forceinline__ static int sw(int p) {
    if constexpr (K >= 6) {
      return p ^ ((p >> (K - 3)) & 7);
    } else {
      return p;
    }
  }
  __host__ __device__ static constexpr int c_of(int pass) {
    return ((4 * pass + 4) < K ? (4 * pass + 4) : K) - RB;
  }
  __device__ __forceinline__ static int pos(int c, int t, int i) {
    return (t & ((1 << c) - 1)) | (i << c) | ((t >> c) << (c + RB));
  }
  // natural index of register i of physical thread t in pass 0
  __device__ __forceinline__ static int l0(int t, int i) {
    return (brev_bits(i, RB) << TB) | t;
  }
};

// Twiddle used by the butterfly: numpy's table value, conjugated for the
// inverse direction (np.conj(w), transform.py:132,199).
template <bool INV>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tb, int k) {
  double2 w = __ldg(tb + k);
  if (INV) w.y = -w.y;
  return w;
}

// One butterfly exactly as transform.py:89-91 evaluates it.
__device__ __forceinline__ void bfly(double2& lo, double2& hi, double2 w) {
  const double2 t = np_cmul(hi, w);
  hi = make_double2(lo.x - t.x, lo.y - t.y);
  lo = make_double2(lo.x + t.x, lo.y + t.y);
}

// Stage b = 0 has the single twiddle w[0] = exp(0) = (1, +-0): the product
// hi * w equals hi up to the sign of a zero, so the multiply is skipped.
__device__ __forceinline__ void bfly1(double2& lo, double2& hi) {
  const double2 t = hi;
  hi = make_double2(lo.x - t.x, lo.y - t.y);
  lo = make_double2(lo.x + t.x, lo.y + t.y);
}

// Butterflies of pass PASS on the 16 registers of logical thread t.
template <int K, int PASS, bool INV>
__device__ __forceinline__ void fft_pass(double2 (&v)[Geo<K>::P], int t,
                                         const double2* __restrict__ twst) {
  using G = Geo<K>;
  constexpr int b0 = 4 * PASS;
  constexpr int b1 = (4 * PASS + 4) < K ? (4 * PASS + 4) : K;
  constexpr int c = G::c_of(PASS);
  const int tlow = t & ((1 << c) - 1);
#pragma unroll
  for (int b = b0; b < b1; ++b) {
    const int q = b - c;  // register bit paired by this stage
    if (b == 0) {
#pragma unroll
      for (int h = 0; h < G::P / 2; ++h) bfly1(v[2 * h], v[2 * h + 1]);
      continue;
    }
    const double2* __restrict__ tb = twst + ((1 << b) - 1);
#pragma unroll
    for (int kk = 0; kk < (1 << q); ++kk) {
      const double2 w = twiddle<INV>(tb, tlow | (kk << c));
#pragma unroll
      for (int h = 0; h < (G::P >> (q + 1)); ++h) {
        const int i = kk | (h << (q + 1));
        bfly(v[i], v[i | (1 << q)], w);
      }
    }
  }
}

// Store the registers of pass PASS to shared memory (swizzled positions).
template <int K, int PASS>
__device__ __forceinline__ void pass_store(const double2 (&v)[Geo<K>::P], int t, double2* sm) {
  using G = Geo<K>;
  constexpr int c = G::c_of(PASS);
#pragma unroll
  for (int i = 0; i < G::P; ++i) sm[G::sw(G::pos(c, t, i))] = v[i];
}

template <int K, int PASS>
__device__ __forceinline__ void pass_load(double2 (&v)[Geo<K>::P], int t, const double2* sm) {
  using G = Geo<K>;
  constexpr int c = G::c_of(PASS);
#pragma unroll
  for (int i = 0; i < G::P; ++i) v[i] = sm[G::sw(G::pos(c, t, i))];
}

// Passes PASS..NPASS-1 of a row whose pass-0 input is already in v
// (physical thread tp; pass 0 uses logical thread rev(tp)).  Between passes
// the row goes through `sm` (N double2, swizzled); every thread of the block
// calls this (block-uniform __syncthreads), `active` masks threads that own
// no row this round.  On return v holds pass NPASS-1's outputs at natural
// positions pos(c_last, tp, i).
template <int K, bool INV, int PASS = 0>
__device__ __forceinline__ void fft_passes(double2 (&v)[Geo<K>::P], int tp, bool active,
                                           double2* sm, const double2* __restrict__ twst) {
  using G = Geo<K>;
  const int t = PASS == 0 ? brev_bits(tp, G::TB) : tp;
  if (active) fft_pass<K, PASS, INV>(v, t, twst);
  if constexpr (PASS + 1 < G::NPASS) {
    if (active) pass_store<K, PASS>(v, t, sm);
    __syncthreads();
    if (active) pass_load<K, PASS + 1>(v, tp, sm);
    __syncthreads();
    fft_passes<K, INV, PASS + 1>(v, tp, active, sm, twst);
  }
}

// Natural output position of register i after the last pass.
template <int K>
__device__ __forceinline__ int out_pos(int tp, int i) {
  using G = Geo<K>;
  return G::pos(G::c_of(G::NPASS - 1), tp, i);
}

}  // namespace afd
