// afd_aux.cuh — plan setup, candidate reduction and bookkeeping kernels.
//   power_table_kernel    np.cumprod radius powers (transform.py:147-150)
//   cand_reduce_kernel    first-maximum reduction of per-CTA candidates
//   argmax_kernel         core.maximal_selection on a materialised field
//   atom_kernel           kernel_samples / blaschke_samples / remainder_update
//   energy_kernel         core.discrete_energy
//   error_trace_kernel    core.error_trace + core.reconstruct (core.py:411-460)
//   gather_outputs_kernel copy the device-resident loop's results out
#pragma once

#include "afd_kernels.cuh"

namespace afd {

// Rows [m0, m1) of r^l, l < n, as the sequential left fold of numpy's
// cumprod over [1, r, r, ...].  One warp = 32 radii; each lane runs its
// radius' chain, a 32x32 shared tile turns the lane-per-row values into
// coalesced row writes.
// pw_len[row] = the first l with r^l == 0 (the fold has underflowed and stays
// +0 from there on), or n: the large-N prologue skips loading the zero tail.
__global__ void power_table_kernel(const double* __restrict__ radii, long long m0, long long m1,
                                   long long n, double* __restrict__ pw, int* __restrict__ pw_len) {
  __shared__ double tile[32][33];
  const int lane = threadIdx.x;
  const long long row = m0 + (long long)blockIdx.x * 32 + lane;
  const double r = row < m1 ? radii[row] : 0.0;
  double v = 1.0;
  long long len = n;
  for (long long c0 = 0; c0 < n; c0 += 32) {
#pragma unroll 8
    for (int i = 0; i < 32; ++i) {
      if (c0 + i > 0) v = v * r;
      if (v == 0.0 && len == n) len = c0 + i;
      tile[lane][i] = v;
    }
    __syncwarp();
    for (int rr = 0; rr < 32; ++rr) {
      const long long row2 = m0 + (long long)blockIdx.x * 32 + rr;
      if (row2 < m1 && c0 + lane < n) pw[(size_t)(row2 - m0) * n + c0 + lane] = tile[rr][lane];
    }
    __syncwarp();
  }
  if (pw_len != nullptr && row < m1) pw_len[row - m0] = (int)len;
}

// Fast-mode weight factor tables (AFD_PLAN_FAST), one row per plan radius:
// section j (j = 0, 1, 2; n_j entries, exponent step 2^e_j, e_0 = 0) holds
// r^(k 2^e_j), section 0 times the row's scale sqrt(1-r^2)/(N(1-r^N)) (the
// reference's own scales, transform.py:153).  The kernels weight position l
// by the product of one entry per section (its bit fields), so r^l is never
// tabulated: ~2 ulp per pow, a few ulp per product, against the reference's
// cumprod (transform.py:147-150), which itself drifts by up to 6e-14.
__global__ void fast_weight_kernel(const double* __restrict__ radii,
                                   const double* __restrict__ scales, long long m0,
                                   long long rows, int stride, int n0, int n1, int e1, int n2,
                                   int e2, double* __restrict__ fw) {
  const long long total = rows * stride;
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const long long row = x / stride;
    const int k = (int)(x % stride);
    const double r = radii[m0 + row];
    double v;
    if (k < n0) v = scales[m0 + row] * pow(r, (double)k);
    else if (k < n0 + n1) v = pow(r, ldexp((double)(k - n0), e1));
    else v = pow(r, ldexp((double)(k - n0 - n1), e2));
    (void)n2;
    fw[x] = v;
  }
}

__device__ __forceinline__ Cand cand_none() {
  Cand c;
  c.mag = -1.0;
  c.flat = 0x7fffffffffffffffLL;
  c.re = c.im = 0.0;
  return c;
}

// Block-wide first-maximum; result valid in every thread.
__device__ Cand block_argmax(Cand c) {
  __shared__ Cand red[32];
  c = warp_argmax(c);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = c;
  __syncthreads();
  if (wid == 0) {
    Cand d = lane < (int)((blockDim.x + 31) >> 5) ? red[lane] : cand_none();
    d = warp_argmax(d);
    if (lane == 0) red[0] = d;
  }
  __syncthreads();
  const Cand r = red[0];
  __syncthreads();
  return r;
}

__global__ void cand_reduce_kernel(const Cand* __restrict__ in, int n_per, Cand* __restrict__ out) {
  Cand b = cand_none();
  for (int i = threadIdx.x; i < n_per; i += blockDim.x) cand_merge(b, in[(size_t)blockIdx.x * n_per + i]);
  b = block_argmax(b);
  if (threadIdx.x == 0) out[blockIdx.x] = b;
}

// First stage of a large candidate reduction: CTA b reduces in[b*per ..
// min((b+1)*per, n)) -> out[b] (loads issued 4 at a time; the first-maximum
// merge is order-free, so any split gives the same result).
// With runner-up slots (in2/out2 non-null): out2[b] = the largest of the
// range's runner-ups and of its candidates other than the winner.
__global__ void cand_partial_kernel(const Cand* __restrict__ in, int n, int per,
                                    Cand* __restrict__ out, const double* __restrict__ in2 = nullptr,
                                    double* __restrict__ out2 = nullptr) {
  Cand b = cand_none();
  const int lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int i = lo + threadIdx.x; i < hi; i += 4 * blockDim.x) {
    Cand c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = i + u * blockDim.x;
      c[u] = k < hi ? in[k] : cand_none();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) cand_merge(b, c[u]);
  }
  b = block_argmax(b);
  if (threadIdx.x == 0) out[blockIdx.x] = b;
  if (in2 != nullptr) {
    double r = -1.0;
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      r = fmax(r, in2[i]);
      const Cand c = in[i];
      if (c.flat != b.flat) r = fmax(r, c.mag);
    }
    r = block_max(r);
    if (threadIdx.x == 0) out2[blockIdx.x] = r;
  }
}

__global__ void neutral_cand_kernel(Cand* out, int batch) {
  for (int i = threadIdx.x; i < batch; i += blockDim.x) out[i] = cand_none();
}

// magnitude = f.real**2 + f.imag**2; np.argmax (core.py:298-299)
__global__ void argmax_kernel(const double2* __restrict__ f, long long total, Cand* __restrict__ out) {
  Cand b = cand_none();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = f[i];
    const double mg = np_mag2(v);
    if (cand_better(mg, i, b.mag, b.flat)) {
      b.mag = mg;
      b.flat = i;
      b.re = v.x;
      b.im = v.y;
    }
  }
  b = block_argmax(b);
  if (threadIdx.x == 0) out[blockIdx.x] = b;
}

// kind 0: kernel_samples(a) (core.py:234-238)
// kind 1: blaschke_samples(a) (core.py:241-245)
// kind 2: remainder_update(g, a, c) (core.py:303-314)
// kind 3: g * blaschke_samples(a) (core.py:406-407; the samples are the
//         temporary, so numpy's elision evaluates `bs *= b` for n >= 16384)
// norm: sqrt(1 - abs(a) ** 2) as the caller computed it (the reference's own
// CPython/libm scalar, core.py:237), or NaN to form it on the device.
__global__ void atom_kernel(int kind, int n, const double2* __restrict__ g, double2 a, double2 c,
                            const double2* __restrict__ circle, double2* __restrict__ out,
                            double norm) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  int amb = 0;
  const double kn = norm == norm ? norm : kernel_norm(a, &amb);
  const bool elide = (size_t)n * 16 >= 256 * 1024;
  const double2 z = circle[m];
  const double2 d = one_minus_conja_z(a, z);
  if (kind == 0) {
    out[m] = np_cdiv(make_double2(kn, 0.0), d);
  } else if (kind == 1) {
    out[m] = np_cdiv(make_double2(z.x - a.x, z.y - a.y), d);
  } else if (kind == 3) {
    const double2 bs = np_cdiv(make_double2(z.x - a.x, z.y - a.y), d);
    out[m] = elide ? np_cmul(bs, g[m]) : np_cmul(g[m], bs);
  } else {
    const double2 e = np_cdiv(make_double2(kn, 0.0), d);
    const double2 ce = elide ? np_cmul(e, c) : np_cmul(c, e);
    const double2 gm = g[m];
    const double2 stp = make_double2(gm.x - ce.x, gm.y - ce.y);
    const double2 num = elide ? np_cmul(d, stp) : np_cmul(stp, d);
    out[m] = np_cdiv(num, make_double2(z.x - a.x, z.y - a.y));
  }
}

// core.discrete_energy for one signal per block (of g - s when s != null);
// scratch per signal: n (mags) + 2*(n/8+16) doubles.
__global__ void energy_kernel(int n, const double2* __restrict__ g, const double2* __restrict__ s,
                              double* __restrict__ scratch, double* __restrict__ energies) {
  const size_t per = (size_t)n + 2 * ((size_t)n / 8 + 16);
  double* mag = scratch + per * blockIdx.x;
  double* acc = mag + n;
  const double2* gs = g + (size_t)blockIdx.x * n;
  const double2* ss = s ? s + (size_t)blockIdx.x * n : nullptr;
  for (int m = threadIdx.x; m < n; m += blockDim.x) {
    double2 v = gs[m];
    if (ss) v = make_double2(v.x - ss[m].x, v.y - ss[m].y);
    mag[m] = np_mag2(v);
  }
  __syncthreads();
  const double sum = pairwise_sum_block(mag, n, acc, PlainIdx());
  if (threadIdx.x == 0) energies[blockIdx.x] = sum / (double)n;
}

// core.error_trace (core.py:442-460): partial sums accumulated once,
//   total = total + c * kernel_samples(a) * blaschke_prod
//   blaschke_prod = blaschke_prod * blaschke_samples(a)
//   errors[k] = discrete_energy(g - total) / discrete_energy(g)
// numpy's temporary elision swaps `c * ks` and `bp * bs` for n >= 16384.
__global__ void error_trace_kernel(int n, const double2* __restrict__ g,
                                   const Step* __restrict__ steps, int max_terms,
                                   const int* __restrict__ n_steps,
                                   const double2* __restrict__ circle, double* __restrict__ scratch,
                                   double* __restrict__ errors, double2* __restrict__ recon,
                                   const double* __restrict__ norms) {
  const int sig = blockIdx.x;
  const size_t per = 2 * (size_t)n * 2 + n + 2 * ((size_t)n / 8 + 16);
  double2* total = reinterpret_cast<double2*>(scratch + per * sig);
  double2* bp = total + n;
  double* mag = reinterpret_cast<double*>(bp + n);
  double* acc = mag + n;
  const double2* gs = g + (size_t)sig * n;
  const bool elide = (size_t)n * 16 >= 256 * 1024;
  for (int m = threadIdx.x; m < n; m += blockDim.x) {
    total[m] = make_double2(0.0, 0.0);
    bp[m] = make_double2(1.0, 0.0);
    mag[m] = np_mag2(gs[m]);
  }
  __syncthreads();
  const double eg = pairwise_sum_block(mag, n, acc, PlainIdx()) / (double)n;
  const int ns = n_steps[sig];
  for (int k = 0; k < ns; ++k) {
    const Step s = steps[(size_t)sig * max_terms + k];
    const double2 a = make_double2(s.a_re, s.a_im);
    const double2 c = make_double2(s.c_re, s.c_im);
    int amb = 0;
    const double kn = norms ? norms[(size_t)sig * max_terms + k] : kernel_norm(a, &amb);
    for (int m = threadIdx.x; m < n; m += blockDim.x) {
      const double2 z = circle[m];
      const double2 d = one_minus_conja_z(a, z);
      const double2 ks = np_cdiv(make_double2(kn, 0.0), d);
      const double2 bs = np_cdiv(make_double2(z.x - a.x, z.y - a.y), d);
      const double2 cks = elide ? np_cmul(ks, c) : np_cmul(c, ks);
      const double2 t = np_cmul(cks, bp[m]);
      const double2 tt = make_double2(total[m].x + t.x, total[m].y + t.y);
      total[m] = tt;
      bp[m] = elide ? np_cmul(bs, bp[m]) : np_cmul(bp[m], bs);
      mag[m] = np_mag2(make_double2(gs[m].x - tt.x, gs[m].y - tt.y));
    }
    __syncthreads();
    const double e = pairwise_sum_block(mag, n, acc, PlainIdx()) / (double)n;
    if (threadIdx.x == 0) errors[(size_t)sig * max_terms + k] = e / eg;
    __syncthreads();
  }
  if (recon) {
    for (int m = threadIdx.x; m < n; m += blockDim.x) recon[(size_t)sig * n + m] = total[m];
  }
}

__global__ void gather_outputs_kernel(int n, int max_terms, const Step* __restrict__ src,
                                      const State* __restrict__ state,
                                      const double2* __restrict__ rem, Step* __restrict__ dst,
                                      int* __restrict__ n_steps, double* __restrict__ initial,
                                      double2* __restrict__ remainder, int* __restrict__ stopped) {
  const int sig = blockIdx.x;
  if (threadIdx.x == 0) {
    n_steps[sig] = state[sig].nsteps;
    initial[sig] = state[sig].initial;
    if (stopped) stopped[sig] = state[sig].stopped;
  }
  if (src && dst) {
    for (int k = threadIdx.x; k < max_terms; k += blockDim.x)
      dst[(size_t)sig * max_terms + k] = src[(size_t)sig * max_terms + k];
  }
  for (int m = threadIdx.x; m < n; m += blockDim.x)
    remainder[(size_t)sig * n + m] = rem[(size_t)sig * n + m];
}

}  // namespace afd

namespace afd {

// DFMA throughput probe: 8 independent chains per thread, ITERS rounds.
template <int ITERS>
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace afd
