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
// across lanes later.  (Shared-memory slots are padded, see Geo::sw.)
#pragma once

#include <type_traits>

#include "afd_common.cuh"

namespace afd {

__host__ __device__ constexpr int brev_bits(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

template <int K, int RBITS = 4>
struct Geo {
  static constexpr int N = 1 << K;
  static constexpr int RB = K >= RBITS ? RBITS : K;  // register (stage) bits per pass
  static constexpr int P = 1 << RB;                  // points per thread
  static constexpr int T = N / P;                    // threads per row
  static constexpr int TB = K - RB;                  // thread-index bits
  static constexpr int NPASS = (K + RB - 1) / RB;

  // Shared-memory slot of position p: one pad slot per 2^(K-3) positions.
  // pos() is an OR of disjoint bit fields of the thread index and of the
  // register index, so SW(pos) = base(thread) + const(register): every
  // exchange access is a register base plus an immediate offset.
  __host__ __device__ __forceinline__ static constexpr int sw(int p) {
    return K >= 6 ? p + (p >> (K - 3)) : p;
  }
  static constexpr int SMEM = K >= 6 ? N + (N >> (K - 3)) : N;  // slots per row
  __host__ __device__ static constexpr int c_of(int pass) {
    return ((RB * pass + RB) < K ? (RB * pass + RB) : K) - RB;
  }
  __device__ __forceinline__ static int pos(int c, int t, int i) {
    return (t & ((1 << c) - 1)) | (i << c) | ((t >> c) << (c + RB));
  }
  // natural index of register i of physical thread t in pass 0
  __device__ __forceinline__ static int l0(int t, int i) {
    return (brev_bits(i, RB) << TB) | t;
  }
};

// TMA bulk copy global -> shared completing on an mbarrier (one thread
// issues; every thread waits with mbar_wait).  16-byte aligned, size % 16 == 0.
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, unsigned bytes,
                                          unsigned long long* mbar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const unsigned m = (unsigned)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(d), "l"(gsrc), "r"(bytes), "r"(m)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, unsigned parity) {
  const unsigned m = (unsigned)__cvta_generic_to_shared(mbar);
  unsigned done = 0;
  unsigned spins = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(m), "r"(parity)
        : "memory");
    if (++spins == (1u << 28)) __trap();  // a lost transfer fails the launch, never hangs
  }
}

// Twiddle sources.  tw(b, k) returns numpy's w[k << (K-1-b)] for stage b.
//
// GlobalTw: per-stage tables S_b (offset 2^b - 1) in global memory, read
// through the read-only path.
struct GlobalTw {
  const double2* __restrict__ st;
  __device__ __forceinline__ double2 operator()(int b, int k) const {
    return __ldg(st + ((1 << b) - 1) + k);
  }
};

// SmemTw<K>: shared-memory copy laid out so every warp access is
// conflict-free.  Stages b < 4 (pass 0) are warp-uniform and stages
// b >= K-4 read the half table w[0..N/2) at lane stride 2^(K-1-b) <= 8,
// stored XOR-swizzled (i ^ ((i >> 3) & 7)) so strides 1, 2, 4 and 8 all hit
// 8 distinct 16-byte bank groups per quarter-warp.  The middle stages
// 4 <= b < K-4 (lane stride >= 16) use compact per-stage tables.
template <int K, int RB = 4>
struct SmemTw {
  static constexpr int HALF = 1 << (K - 1);
  static constexpr int HALF_SLOTS = HALF + HALF / 8;  // padded half table
  static constexpr int LO = RB;      // first thread-dependent stage
  static constexpr int HI = K - 4;   // stages >= HI read the half table
  static constexpr int MID = (HI > LO) ? (1 << HI) - (1 << LO) : 0;  // S_LO..S_{HI-1}
  static constexpr int ENTRIES = HALF_SLOTS + MID;
  const double2* sm;
  // padded slot: strides 1, 2, 4, 8 over a quarter-warp hit 8 distinct
  // 16-byte bank groups, and slot(a | b) = slot(a) + slot(b) for disjoint
  // bit fields (base + immediate addressing)
  __device__ __forceinline__ static int swz(int i) { return i + (i >> 3); }
  __device__ __forceinline__ double2 operator()(int b, int k) const {
    if (b >= LO && b < HI) return sm[HALF_SLOTS + (1 << b) - (1 << LO) + k];
    return sm[swz(k << (K - 1 - b))];
  }
  // Build the shared-memory image (ENTRIES double2, this layout) in global
  // memory once per plan, so kernels can fetch it with one bulk copy.
  __device__ static void build_image(double2* img, const double2* __restrict__ st) {
    const double2* half = st + (1 << (K - 1)) - 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ENTRIES;
         i += gridDim.x * blockDim.x) {
      double2 v = make_double2(0.0, 0.0);
      if (i >= HALF_SLOTS) {
        v = st[(1 << LO) - 1 + (i - HALF_SLOTS)];
      } else {
        // slot i holds half[k] with swz(k) == i (pad slots stay zero)
        const int k = i - i / 9;  // inverse of k + k/8 on non-pad slots
        if (swz(k) == i) v = half[k];
      }
      img[i] = v;
    }
  }
  // Fill from the global stage tables (all threads of the block).
  __device__ static void load(double2* dst, const double2* __restrict__ st) {
    // half table = stage K-1 table S_{K-1}[k] = w[k]
    const double2* half = st + (1 << (K - 1)) - 1;
    for (int i = threadIdx.x; i < HALF; i += blockDim.x) dst[swz(i)] = __ldg(half + i);
    for (int i = threadIdx.x; i < MID; i += blockDim.x)
      dst[HALF_SLOTS + i] = __ldg(st + (1 << LO) - 1 + i);
  }
};

// One butterfly exactly as transform.py:89-91 evaluates it.
__device__ __forceinline__ void bfly(double2& lo, double2& hi, double2 w) {
  const double2 t = np_cmul(hi, w);
  hi = make_double2(lo.x - t.x, lo.y - t.y);
  lo = make_double2(lo.x + t.x, lo.y + t.y);
}

// Stage b = 0 has the single twiddle w[0] = exp(0) = (1, +-0): the product
// hi * w equals hi up to the sign of a zero, so the multiply is skipped.  The
// same holds for every butterfly of a later stage whose twiddle index is 0:
// in pass 0 (thread bits above the stage) those are the kk = 0 register
// pairs, known at compile time (stages 1-3: 1.75 of 54 FP64 instructions
// per point saved).  A sign-of-zero difference can only reach an output
// that is itself exactly zero.
__device__ __forceinline__ void bfly1(double2& lo, double2& hi) {
  const double2 t = hi;
  hi = make_double2(lo.x - t.x, lo.y - t.y);
  lo = make_double2(lo.x + t.x, lo.y + t.y);
}

// Butterflies of pass PASS on the 16 registers of logical thread t.
template <int K, int RB, int PASS, bool INV, class Tw>
__device__ __forceinline__ void fft_pass(double2 (&v)[Geo<K, RB>::P], int t, const Tw& tw) {
  using G = Geo<K, RB>;
  constexpr int b0 = G::RB * PASS;
  constexpr int b1 = (G::RB * PASS + G::RB) < K ? (G::RB * PASS + G::RB) : K;
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
#pragma unroll
    for (int kk = 0; kk < (1 << q); ++kk) {
      if (c == 0 && kk == 0) {  // pass 0: twiddle index 0 is w[0] (see bfly1)
#pragma unroll
        for (int h = 0; h < (G::P >> (q + 1)); ++h) {
          const int i = h << (q + 1);
          bfly1(v[i], v[i | (1 << q)]);
        }
        continue;
      }
      double2 w = tw(b, tlow | (kk << c));
      if (INV) w.y = -w.y;  // np.conj(w), transform.py:132,199
#pragma unroll
      for (int h = 0; h < (G::P >> (q + 1)); ++h) {
        const int i = kk | (h << (q + 1));
        bfly(v[i], v[i | (1 << q)], w);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Twiddles in tensor memory (TMEM).  The field kernel's two row-groups
// alternate FP64-bound passes with shared-memory exchanges; twiddles read
// from shared memory queue behind the other group's exchange traffic (a
// pass measured 1.1k cycles alone, 1.9k beside an exchange).  TMEM has its
// own data path (tcgen05.ld), so each thread keeps its per-pass twiddles
// there: 3 passes x 15 slots x 4 words (conjugated for the inverse), lane =
// the thread's TMEM lane in its warp's quadrant, one column set per pair of
// warps sharing a quadrant (the two row-groups share the sets).  Filled once
// per CTA before the PDL wait.  Used for N = 4096 (RB = 4, 3 passes).
// ---------------------------------------------------------------------------
template <int NW>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t (&r)[NW]);
template <>
__device__ __forceinline__ void tm_ld<4>(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
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
template <>
__device__ __forceinline__ void tm_ld<64>(uint32_t a, uint32_t (&r)[64]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
               : "r"(a));
}
__device__ __forceinline__ void tm_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_st4(uint32_t a, double2 w) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
               "r"(__double2loint(w.x)), "r"(__double2hiint(w.x)), "r"(__double2loint(w.y)),
               "r"(__double2hiint(w.y))
               : "memory");
}

struct TmemTw {
  static constexpr bool kTmem = true;
  static constexpr int kSetCols = 180;  // 3 passes x 15 slots x 4 words
  static constexpr int kGhCol = 2 * kSetCols;  // field spectrum: 2 sets x 16 values x 4 words
  uint32_t base;  // warp-uniform: lane quadrant of this warp, column 0 of its set
  __device__ __forceinline__ static uint32_t col(int pass, int slot) {
    return (uint32_t)(pass * 60 + slot * 4);
  }
  // Fill this thread's lane (all threads of the warp call it, same slot).
  template <int K, int RB, bool INV, class Src>
  __device__ __forceinline__ void fill(int tp, const Src& src) const {
    using G = Geo<K, RB>;
    static_assert(G::NPASS <= 3 && G::RB == 4, "TMEM twiddle layout: <= 3 passes of 4 stages");
#pragma unroll
    for (int pass = 0; pass < G::NPASS; ++pass) {
      const int c = G::c_of(pass);
      const int t = pass == 0 ? brev_bits(tp, G::TB) : tp;
      const int tlow = t & ((1 << c) - 1);
      const int b0 = G::RB * pass;
      const int b1 = (b0 + G::RB) < K ? (b0 + G::RB) : K;
#pragma unroll
      for (int b = b0; b < b1; ++b) {
        if (b == 0) continue;
        const int q = b - c;
#pragma unroll
        for (int kk = 0; kk < (1 << q); ++kk) {
          double2 w = src(b, tlow | (kk << c));
          if (INV) w.y = -w.y;  // np.conj(w), transform.py:132,199
          tm_st4(base + col(pass, (1 << q) - 1 + kk), w);
        }
      }
    }
  }
};

template <class Tw>
struct IsTmemTw {
  static constexpr bool value = false;
};
template <>
struct IsTmemTw<TmemTw> {
  static constexpr bool value = true;
};

// fft_pass with per-stage twiddles from TMEM (already conjugated): one
// tcgen05.ld of the stage's 2^q twiddles, then its butterflies.
template <int K, int RB, int PASS, int B>
__device__ __forceinline__ void fft_stage_tm(double2 (&v)[Geo<K, RB>::P], const TmemTw& tw) {
  using G = Geo<K, RB>;
  constexpr int c = G::c_of(PASS);
  constexpr int q = B - c;
  if constexpr (B == 0) {
#pragma unroll
    for (int h = 0; h < G::P / 2; ++h) bfly1(v[2 * h], v[2 * h + 1]);
  } else {
    uint32_t r[4 << q];
    tm_ld<(4 << q)>(tw.base + TmemTw::col(PASS, (1 << q) - 1), r);
    tm_wait_ld();
#pragma unroll
    for (int kk = 0; kk < (1 << q); ++kk) {
      if (c == 0 && kk == 0) {  // pass 0: twiddle index 0 is w[0] (see bfly1)
#pragma unroll
        for (int h = 0; h < (G::P >> (q + 1)); ++h) {
          const int i = h << (q + 1);
          bfly1(v[i], v[i | (1 << q)]);
        }
        continue;
      }
      const double2 w = make_double2(__hiloint2double(r[4 * kk + 1], r[4 * kk]),
                                     __hiloint2double(r[4 * kk + 3], r[4 * kk + 2]));
#pragma unroll
      for (int h = 0; h < (G::P >> (q + 1)); ++h) {
        const int i = kk | (h << (q + 1));
        bfly(v[i], v[i | (1 << q)], w);
      }
    }
  }
}

template <int K, int RB, int PASS, int B = Geo<K, RB>::RB * PASS>
__device__ __forceinline__ void fft_pass_tm(double2 (&v)[Geo<K, RB>::P], const TmemTw& tw) {
  using G = Geo<K, RB>;
  constexpr int b1 = (G::RB * PASS + G::RB) < K ? (G::RB * PASS + G::RB) : K;
  if constexpr (B < b1) {
    fft_stage_tm<K, RB, PASS, B>(v, tw);
    fft_pass_tm<K, RB, PASS, B + 1>(v, tw);
  }
}

// ---------------------------------------------------------------------------
// Fast mode (AFD_PLAN_FAST).  The same DIT dataflow, but each butterfly is
// FMA-fused: a twiddle is held as (c, t) with W = c (1 + i t) (c = cos,
// t = tan of the conjugated numpy twiddle, built once per plan), so
//     u  = hi (1 + i t)          2 DFMA
//     lo, hi = lo +- c u         4 DFMA
// is 6 FP64 instructions instead of the reference's 2 DMUL + 2 DFMA + 4 DADD,
// and is exact to a few ulp for every angle (t is large only where c is
// small; numpy's W_4 = 6.12e-17 - 1j keeps t finite).  Pass 0's twiddles
// are the 16th roots of unity, applied as compile-time constants: W = 1 and
// W = +i are exact add/sub butterflies (no multiply at all).  The weighting
// r^l and the scale are formed on chip and fused into stage 0 (see
// fast_prologue), so stage 0 is skipped here.  Results agree with the
// reference to ~1e-14 relative, not bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bfly_ct(double2& lo, double2& hi, double c, double t) {
  const double ur = fma(-t, hi.y, hi.x);
  const double ui = fma(t, hi.x, hi.y);
  hi = make_double2(fma(-c, ur, lo.x), fma(-c, ui, lo.y));
  lo = make_double2(fma(c, ur, lo.x), fma(c, ui, lo.y));
}
// W = +i (inverse transform, quarter turn): lo +- (-hi.y, hi.x)
__device__ __forceinline__ void bfly_pi(double2& lo, double2& hi) {
  const double2 l = lo;
  lo = make_double2(l.x - hi.y, l.y + hi.x);
  hi = make_double2(l.x + hi.y, l.y - hi.x);
}
// exact (re, im) twiddle or (c, t) twiddle, by mode
template <bool FAST>
__device__ __forceinline__ void bfly_any(double2& lo, double2& hi, double2 w) {
  if constexpr (FAST) bfly_ct(lo, hi, w.x, w.y);
  else bfly(lo, hi, w);
}

// (c, t) of exp(+i pi a / 8), a = 0..7 (correctly rounded); a = 0, 4 are the
// exact W = 1, W = +i butterflies.
__device__ __forceinline__ constexpr double ct_c8(int a) {
  return a == 1 ? 0x1.d906bcf328d46p-1 : a == 2 ? 0x1.6a09e667f3bcdp-1 :
         a == 3 ? 0x1.87de2a6aea963p-2 : a == 5 ? -0x1.87de2a6aea963p-2 :
         a == 6 ? -0x1.6a09e667f3bcdp-1 : a == 7 ? -0x1.d906bcf328d46p-1 : 1.0;
}
__device__ __forceinline__ constexpr double ct_t8(int a) {
  return a == 1 ? 0x1.a827999fcef32p-2 : a == 2 ? 1.0 : a == 3 ? 0x1.3504f333f9de6p+1 :
         a == 5 ? -0x1.3504f333f9de6p+1 : a == 6 ? -1.0 : a == 7 ? -0x1.a827999fcef32p-2 : 0.0;
}
template <int A>
__device__ __forceinline__ void bfly_root16(double2& lo, double2& hi) {
  if constexpr (A == 0) bfly1(lo, hi);
  else if constexpr (A == 4) bfly_pi(lo, hi);
  else bfly_ct(lo, hi, ct_c8(A), ct_t8(A));
}

// Fast twiddle sources: the (c, t) stage tables in the SmemTw layout
// (shared memory) or in the TmemTw layout (tensor memory).
template <int K, int RB = 4>
struct SmemTwCT : SmemTw<K, RB> {};
struct TmemTwCT : TmemTw {};
template <class Tw>
struct IsFastTw {
  static constexpr bool value = false;
};
template <int K, int RB>
struct IsFastTw<SmemTwCT<K, RB>> {
  static constexpr bool value = true;
};
template <>
struct IsFastTw<TmemTwCT> {
  static constexpr bool value = true;
};

// Pass 0, stages 1..RB-1 (stage 0 is fused into the prologue): the
// twiddle of register pair kk at stage b is exp(+i pi kk / 2^b).
template <int RB, int B = 1>
__device__ __forceinline__ void fast_pass0(double2 (&v)[1 << RB]) {
  if constexpr (B < RB) {
    constexpr int P = 1 << RB;
#pragma unroll
    for (int kk = 0; kk < (1 << B); ++kk) {
#pragma unroll
      for (int h = 0; h < (P >> (B + 1)); ++h) {
        const int i = kk | (h << (B + 1));
        // angle kk / 2^B of pi, in eighths
        switch (kk << (3 - B)) {
          case 0: bfly_root16<0>(v[i], v[i | (1 << B)]); break;
          case 1: bfly_root16<1>(v[i], v[i | (1 << B)]); break;
          case 2: bfly_root16<2>(v[i], v[i | (1 << B)]); break;
          case 3: bfly_root16<3>(v[i], v[i | (1 << B)]); break;
          case 4: bfly_root16<4>(v[i], v[i | (1 << B)]); break;
          case 5: bfly_root16<5>(v[i], v[i | (1 << B)]); break;
          case 6: bfly_root16<6>(v[i], v[i | (1 << B)]); break;
          default: bfly_root16<7>(v[i], v[i | (1 << B)]); break;
        }
      }
    }
    fast_pass0<RB, B + 1>(v);
  }
}

// Passes >= 1 with (c, t) twiddles of logical thread t.
template <int K, int RB, int PASS, int B, class Tw>
__device__ __forceinline__ void fast_stage(double2 (&v)[Geo<K, RB>::P], int t, const Tw& tw) {
  using G = Geo<K, RB>;
  constexpr int c = G::c_of(PASS);
  constexpr int q = B - c;
  if constexpr (std::is_same<Tw, TmemTwCT>::value) {
    // one tcgen05.ld of the stage's 2^q (c, t) pairs (stored by fill<.., false>)
    uint32_t r[4 << q];
    tm_ld<(4 << q)>(tw.base + TmemTw::col(PASS, (1 << q) - 1), r);
    tm_wait_ld();
#pragma unroll
    for (int kk = 0; kk < (1 << q); ++kk) {
      const double cc = __hiloint2double(r[4 * kk + 1], r[4 * kk]);
      const double tt = __hiloint2double(r[4 * kk + 3], r[4 * kk + 2]);
#pragma unroll
      for (int h = 0; h < (G::P >> (q + 1)); ++h) {
        const int i = kk | (h << (q + 1));
        bfly_ct(v[i], v[i | (1 << q)], cc, tt);
      }
    }
  } else {
    const int tlow = t & ((1 << c) - 1);
#pragma unroll
    for (int kk = 0; kk < (1 << q); ++kk) {
      const double2 w = tw(B, tlow | (kk << c));
#pragma unroll
      for (int h = 0; h < (G::P >> (q + 1)); ++h) {
        const int i = kk | (h << (q + 1));
        bfly_ct(v[i], v[i | (1 << q)], w.x, w.y);
      }
    }
  }
}

template <int K, int RB, int PASS, class Tw, int B = Geo<K, RB>::RB * PASS>
__device__ __forceinline__ void fast_pass(double2 (&v)[Geo<K, RB>::P], int t, const Tw& tw) {
  using G = Geo<K, RB>;
  static_assert(PASS > 0, "pass 0 is fast_pass0");
  constexpr int b1 = (G::RB * PASS + G::RB) < K ? (G::RB * PASS + G::RB) : K;
  if constexpr (B < b1) {
    fast_stage<K, RB, PASS, B>(v, t, tw);
    fast_pass<K, RB, PASS, Tw, B + 1>(v, t, tw);
  }
}

// Store the registers of pass PASS to shared memory (swizzled positions).
template <int K, int RB, int PASS>
__device__ __forceinline__ void pass_store(const double2 (&v)[Geo<K, RB>::P], int t, double2* sm) {
  using G = Geo<K, RB>;
  constexpr int c = G::c_of(PASS);
#pragma unroll
  for (int i = 0; i < G::P; ++i) sm[G::sw(G::pos(c, t, i))] = v[i];
}

template <int K, int RB, int PASS>
__device__ __forceinline__ void pass_load(double2 (&v)[Geo<K, RB>::P], int t, const double2* sm) {
  using G = Geo<K, RB>;
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
// Barrier between passes: the whole block (default) or only the row-group
// that shares `sm` (named barrier `id` over `count` threads), so several rows
// of one CTA can run out of phase.
struct BlockSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct GroupSync {
  int id, count;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
};
// A group that is exactly one warp (N = 512: sixteen 32-thread groups, more
// than the 15 named barriers 1..15 a CTA has) synchronises as a warp.
struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};

// Optional per-pass hook: before(PASS) / after(PASS) around a pass's
// butterflies, exch(PASS) after the exchange that follows it (timing
// probes, inter-group scheduling).
struct NoHook {
  __device__ __forceinline__ void before(int) const {}
  __device__ __forceinline__ void after(int) const {}
  __device__ __forceinline__ void exch(int) const {}
};

template <int K, bool INV, int RB = 4, int PASS = 0, class Tw, class Sync = BlockSync,
          class Hook = NoHook>
__device__ __forceinline__ void fft_passes(double2 (&v)[Geo<K, RB>::P], int tp, bool active,
                                           double2* sm, const Tw& tw, Sync sync = Sync(),
                                           const Hook& hook = Hook()) {
  using G = Geo<K, RB>;
  const int t = PASS == 0 ? brev_bits(tp, G::TB) : tp;
  hook.before(PASS);
  if constexpr (IsFastTw<Tw>::value) {
    if (active) {
      if constexpr (PASS == 0) fast_pass0<G::RB>(v);
      else fast_pass<K, RB, PASS, Tw>(v, t, tw);
    }
  } else if constexpr (IsTmemTw<Tw>::value) {
    static_assert(INV, "TMEM twiddles are stored conjugated (inverse transform)");
    if (active) fft_pass_tm<K, RB, PASS>(v, tw);
  } else {
    if (active) fft_pass<K, RB, PASS, INV>(v, t, tw);
  }
  hook.after(PASS);
  if constexpr (PASS + 1 < G::NPASS) {
    if (active) pass_store<K, RB, PASS>(v, t, sm);
    sync();
    if (active) pass_load<K, RB, PASS + 1>(v, tp, sm);
    sync();
    hook.exch(PASS);
    fft_passes<K, INV, RB, PASS + 1>(v, tp, active, sm, tw, sync, hook);
  }
}

// Natural output position of register i after the last pass.
template <int K, int RB = 4>
__device__ __forceinline__ int out_pos(int tp, int i) {
  using G = Geo<K, RB>;
  return G::pos(G::c_of(G::NPASS - 1), tp, i);
}

}  // namespace afd
