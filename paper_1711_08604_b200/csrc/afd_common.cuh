// afd_common.cuh — device arithmetic that reproduces the reference's
// numpy/CPython operations bit for bit (see oracle/afd_oracle.c for the CPU
// statement of the same forms and SURVEY.md Appendix A for the probes).
//
// The whole library is compiled with -fmad=false: nvcc never contracts
// a*b+c on its own, and every fused multiply-add below is an explicit fma().
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace afd {

// numpy complex128 multiply, AVX-512 loop form (transform.py:89,
// core.py:238,313-314): re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br).
__device__ __forceinline__ double2 np_cmul(double2 a, double2 b) {
  double2 o;
  o.x = fma(a.x, b.x, -(a.y * b.y));
  o.y = fma(a.x, b.y, a.y * b.x);
  return o;
}

// numpy complex128 true_divide: Smith's algorithm, unfused.
__device__ __forceinline__ double2 np_cdiv(double2 a, double2 b) {
  double2 o;
  if (fabs(b.x) >= fabs(b.y)) {
    const double rat = b.y / b.x;
    const double scl = 1.0 / (b.x + b.y * rat);
    o.x = (a.x + a.y * rat) * scl;
    o.y = (a.y - a.x * rat) * scl;
  } else {
    const double rat = b.x / b.y;
    const double scl = 1.0 / (b.y + b.x * rat);
    o.x = (a.x * rat + a.y) * scl;
    o.y = (a.y * rat - a.x) * scl;
  }
  return o;
}

// np_cdiv split in two: the divisor-only part (branch, ratio, reciprocal —
// both divisions) and the numerator part; np_cdiv_fin(a, np_cdiv_pre(b)) is
// np_cdiv(a, b) operation for operation.  Lets a caller issue the divisions
// before the numerator is known.
struct CdivPre {
  double rat, scl;
  bool xbig;
};
__device__ __forceinline__ CdivPre np_cdiv_pre(double2 b) {
  CdivPre p;
  p.xbig = fabs(b.x) >= fabs(b.y);
  if (p.xbig) {
    p.rat = b.y / b.x;
    p.scl = 1.0 / (b.x + b.y * p.rat);
  } else {
    p.rat = b.x / b.y;
    p.scl = 1.0 / (b.y + b.x * p.rat);
  }
  return p;
}
__device__ __forceinline__ double2 np_cdiv_fin(double2 a, const CdivPre& p) {
  double2 o;
  if (p.xbig) {
    o.x = (a.x + a.y * p.rat) * p.scl;
    o.y = (a.y - a.x * p.rat) * p.scl;
  } else {
    o.x = (a.x * p.rat + a.y) * p.scl;
    o.y = (a.y * p.rat - a.x) * p.scl;
  }
  return o;
}

// |z|^2 as core.py:298 evaluates it: re**2 + im**2, two roundings + add.
__device__ __forceinline__ double np_mag2(double2 v) { return v.x * v.x + v.y * v.y; }

// CPython abs(complex) -> glibc 2.39 hypot (no-FMA build of the Borges
// "MyHypot3" correction, glibc sysdeps/ieee754/dbl-64/e_hypot.c).  Verified
// bit-identical to the host libm on 6e7 random pairs (tests/test_oracle.py
// re-checks the CPU copy of this routine against libm hypot).  Inputs here
// are finite with |a| < 1, so the overflow / subnormal scaling branches of
// the library routine are never needed.
__device__ __forceinline__ double glibc_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x;
  const double ay = x < y ? x : y;
  if (ay <= ax * 0x1p-54) return ax + ay;
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

// sqrt(1.0 - abs(a) ** 2) (core.py:238).  CPython's float ** 2 calls libm
// pow(h, 2.0), which (0.52 ulp) can differ from the correctly rounded h*h
// only when h*h's low part is within 0.008 ulp of a rounding midpoint
// (measured: every mismatch had |lo| >= 0.492 ulp).  We return the h*h
// form and raise *ambiguous when |lo| > 0.49 ulp, so callers can report
// the step as "not provably bit-identical".
__device__ __forceinline__ double kernel_norm(double2 a, int* ambiguous) {
  const double h = glibc_hypot(a.x, a.y);
  const double hh = h * h;
  const double lo = fma(h, h, -hh);
  if (hh != 0.0) {
    // ulp(hh) for a normal positive double: 2^(exponent - 52)
    const long long bits = __double_as_longlong(hh);
    const int e = (int)((bits >> 52) & 0x7ff);
    const double ulp = __longlong_as_double((long long)(e > 52 ? e - 52 : 1) << 52);
    if (fabs(lo) > 0.49 * ulp) *ambiguous = 1;
  }
  return sqrt(1.0 - hh);
}

// sqrt(1.0 - abs(a) ** 2) bit for bit for a grid pole a = r_s z_j.  The
// plan tabulates, per radius r_s, CPython's float ** 2 — libm pow(h, 2.0)
// called on the host — for the kPowWin ulps either side of r_s:
// h = hypot(a) lies within 1 ulp of r_s for every grid pole (|z_j| = 1 to
// an ulp; measured over N = 2^10..2^20).  The lookup makes the step kernels'
// norms identical to the reference's; a pole outside the window (never for
// grid poles) falls back to kernel_norm and its ambiguity flag.
constexpr int kPowWin = 4;
constexpr int kPowRow = 2 * kPowWin + 1;
__device__ __forceinline__ double kernel_norm_grid(double2 a, double r,
                                                   const double* __restrict__ pow_row,
                                                   int* ambiguous) {
  if (pow_row != nullptr) {
    const double h = glibc_hypot(a.x, a.y);
    const long long d = __double_as_longlong(h) - __double_as_longlong(r) + kPowWin;
    if (d >= 0 && d < kPowRow) return sqrt(1.0 - __ldg(pow_row + d));
  }
  return kernel_norm(a, ambiguous);
}

// The per-point factors shared by kernel_samples, blaschke_samples and
// remainder_update (core.py:234-245, 303-314):
//   d = 1.0 - conj(a) * z          (numpy: (1 - pr, 0 - pi))
__device__ __forceinline__ double2 one_minus_conja_z(double2 a, double2 z) {
  const double2 ca = make_double2(a.x, -a.y);
  const double2 p = np_cmul(ca, z);
  return make_double2(1.0 - p.x, 0.0 - p.y);
}

// Opaque register copy: the compiler can neither fold the value nor
// rematerialise it from the constant bank later.  Kernels copy the
// parameters they need after griddepcontrol.wait through opq() before the
// wait: constant-bank reads issued after the wait were measured to cost up
// to ~0.7 us each on the critical path of the per-step kernel.
__device__ __forceinline__ int opq(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ long long opq(long long v) {
  long long r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(v));
  return r;
}
__device__ __forceinline__ double opq(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}
template <class T>
__device__ __forceinline__ T* opq(T* p) {
  return reinterpret_cast<T*>(opq(reinterpret_cast<long long>(p)));
}

// Programmatic dependent launch (PDL): kernels launched with programmatic
// stream serialization may start while their predecessor drains; everything
// before pdl_wait() must not read the predecessor's outputs.  Both are
// no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Candidate of the grid argmax: first maximum in row-major (s, j) order.
struct __align__(16) Cand {
  double mag;
  long long flat;
  double re, im;
};

__device__ __forceinline__ bool cand_better(double m1, long long f1, double m2, long long f2) {
  return m1 > m2 || (m1 == m2 && f1 < f2);
}

__device__ __forceinline__ void cand_merge(Cand& a, const Cand& b) {
  if (cand_better(b.mag, b.flat, a.mag, a.flat)) a = b;
}

// Runner-up bookkeeping (fast engine): a candidate set
// carries, beside its first maximum, the largest |F|^2 of its other grid
// points.  Merging two sets, the loser's maximum competes for runner-up.
__device__ __forceinline__ double runner_merge(double r1, double m1, double r2, double m2) {
  return fmax(fmax(r1, r2), fmin(m1, m2));
}
// Block-wide maximum of a double; result valid in every thread.
__device__ double block_max(double x) {
  __shared__ double redm[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) redm[wid] = x;
  __syncthreads();
  double y = -1.0;
  for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) y = fmax(y, redm[w]);
  __syncthreads();
  return y;
}

// |F|^2 of a selected value as the fast epilogues form it
__device__ __forceinline__ double coeff_mag2(double2 c) { return fma(c.x, c.x, c.y * c.y); }
// Top-2 relative margin (best - runner-up) / best of the step's |F|^2.
__device__ __forceinline__ float top2_margin(double best, double runner) {
  if (!(best > 0.0)) return 0.0f;
  return (float)((best - fmax(runner, 0.0)) / best);
}

__device__ __forceinline__ Cand cand_shfl_down(const Cand& c, int off) {
  Cand o;
  o.mag = __shfl_down_sync(0xffffffffu, c.mag, off);
  o.flat = __shfl_down_sync(0xffffffffu, c.flat, off);
  o.re = __shfl_down_sync(0xffffffffu, c.re, off);
  o.im = __shfl_down_sync(0xffffffffu, c.im, off);
  return o;
}

__device__ __forceinline__ Cand warp_argmax(Cand c) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cand_merge(c, cand_shfl_down(c, off));
  return c;
}

// numpy pairwise summation (np.sum / np.mean over float64) of n = 2^K >= 8
// doubles held in shared memory at `buf[SW(i)]`; executed by the whole
// block, result returned to every thread.  Recursion (numpy
// loops_utils.h pairwise_sum): blocks of <= 128 with 8 strided
// accumulators, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), halves added
// left + right.  `scratch` needs max(n/16, 8) doubles.
template <class Idx>
__device__ double pairwise_sum_block(const double* buf, int n, double* scratch, Idx SW,
                                     int nthreads = -1) {
  const int nt = nthreads > 0 ? nthreads : (int)blockDim.x;
  const int nblk = n >= 128 ? n / 128 : 1;
  const int bl = n >= 128 ? 128 : n;
  // phase 1: accumulator k of block b sums elements b*bl + k + 8 i
  for (int a = threadIdx.x; a < nblk * 8; a += nt) {
    const int b = a >> 3, k = a & 7;
    const int base = b * bl;
    double r = buf[SW(base + k)];
    for (int i = 8; i < bl; i += 8) r += buf[SW(base + i + k)];
    scratch[a] = r;
  }
  __syncthreads();
  // phase 2: per block ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
  double* sums = scratch + nblk * 8;
  for (int b = threadIdx.x; b < nblk; b += nt) {
    const double* r = scratch + b * 8;
    sums[b] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  }
  __syncthreads();
  // phase 3: binary tree over blocks, left + right
  for (int w = nblk; w > 1; w >>= 1) {
    for (int b = threadIdx.x; b < w / 2; b += nt) sums[b] = sums[2 * b] + sums[2 * b + 1];
    __syncthreads();
  }
  const double res = sums[0];
  __syncthreads();
  return res;
}

// numpy pairwise summation of complex128 (np.mean on complex, core.py:375):
// n complex values (2n doubles); blocks of <= 64 complex with 4 strided
// complex accumulators, rr = (r0+r2)+(r4+r6), ri = (r1+r3)+(r5+r7).
// `scratch` needs max(n/8, 8) * 2 doubles.
template <class Idx>
__device__ double2 cpairwise_sum_block(const double2* buf, int n, double* scratch, Idx SW,
                                       int nthreads = -1) {
  const int nt = nthreads > 0 ? nthreads : (int)blockDim.x;
  const int nblk = n >= 64 ? n / 64 : 1;
  const int bl = n >= 64 ? 64 : n;
  for (int a = threadIdx.x; a < nblk * 4; a += nt) {
    const int b = a >> 2, q = a & 3;
    const int base = b * bl;
    double2 v = buf[SW(base + q)];
    double rr = v.x, ri = v.y;
    for (int i = 4; i < bl; i += 4) {
      const double2 u = buf[SW(base + i + q)];
      rr += u.x;
      ri += u.y;
    }
    scratch[2 * a] = rr;
    scratch[2 * a + 1] = ri;
  }
  __syncthreads();
  double* sums = scratch + nblk * 8;
  for (int b = threadIdx.x; b < nblk; b += nt) {
    const double* r = scratch + b * 8;
    sums[2 * b] = (r[0] + r[2]) + (r[4] + r[6]);
    sums[2 * b + 1] = (r[1] + r[3]) + (r[5] + r[7]);
  }
  __syncthreads();
  for (int w = nblk; w > 1; w >>= 1) {
    for (int b = threadIdx.x; b < w / 2; b += nt) {
      sums[2 * b] = sums[4 * b] + sums[4 * b + 2];
      sums[2 * b + 1] = sums[4 * b + 1] + sums[4 * b + 3];
    }
    __syncthreads();
  }
  const double2 res = make_double2(sums[0], sums[1]);
  __syncthreads();
  return res;
}

}  // namespace afd
