/*
 * afd_oracle.c — CPU restatement of the reference FFT-AFD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file: it is the checker that tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg compare the CUDA path
 * against.  It restates /root/reference/pkg/src/fastafd/{transform,core}.py
 * operation for operation, reproducing numpy 2.3 (AVX-512 dispatch) and
 * CPython/glibc arithmetic bit for bit:
 *
 *   complex*complex   re = fma(ar,br,-(ai*bi)), im = fma(ar,bi,ai*br)
 *                     (numpy AVX-512 loop; first operand = left operand)
 *   complex/complex   Smith's algorithm, unfused (numpy CDOUBLE_divide)
 *   float*complex     per component (numpy promotes to (s,0) and the fma
 *                     form collapses to one rounding per component)
 *   np.sum / np.mean  numpy pairwise summation (8 accumulators, 128 block)
 *   abs(complex)      libm hypot (CPython _Py_c_abs)
 *   float ** 2        libm pow(x, 2.0) (CPython float_pow; NOT x*x)
 *   `x * tmp`         numpy temporary elision: when `tmp` is a fresh array
 *                     of >= 256 KiB (complex128: N >= 16384) and the op is
 *                     commutative, numpy evaluates `tmp *= x`, i.e. the
 *                     multiply runs with its operands swapped -- which
 *                     changes the bits of the fma form.  ELIDE(n) below.
 *
 * Build with -ffp-contract=off so the C compiler never fuses a*b+c on its
 * own; every fma below is explicit.  Pinned against the reference itself
 * by tests/golden/ (fixtures produced by running /root/reference in the
 * build container, script tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef struct { double re, im; } cplx;

/* numpy temp_elide.c: NPY_MIN_ELIDE_BYTES = 256 KiB. */
#define ELIDE(n) ((n) * 16 >= 256 * 1024)

typedef struct {
  int64_t s, j;          /* radius index, angle index (grid.point(s, j)) */
  double radius;
  double a_re, a_im;     /* selected pole value                          */
  double c_re, c_im;     /* coefficient <G_k, e_a>                        */
  double residual;       /* discrete_energy(G_{k+1})                      */
} afdo_step;

/* ---- numpy / CPython arithmetic primitives ------------------------------ */

/* numpy complex128 multiply (transform.py:89 `blocks[:, half:] * tw`,
 * core.py:238, core.py:313-314). */
static inline cplx np_cmul(cplx a, cplx b) {
  cplx o;
  o.re = fma(a.re, b.re, -(a.im * b.im));
  o.im = fma(a.re, b.im, a.im * b.re);
  return o;
}

/* numpy complex128 true_divide (core.py:238, core.py:313-314): Smith. */
static inline cplx np_cdiv(cplx a, cplx b) {
  cplx o;
  if (fabs(b.re) >= fabs(b.im)) {
    double rat = b.im / b.re;
    double scl = 1.0 / (b.re + b.im * rat);
    o.re = (a.re + a.im * rat) * scl;
    o.im = (a.im - a.re * rat) * scl;
  } else {
    double rat = b.re / b.im;
    double scl = 1.0 / (b.im + b.re * rat);
    o.re = (a.re * rat + a.im) * scl;
    o.im = (a.im * rat - a.re) * scl;
  }
  return o;
}

/* numpy pairwise summation of n doubles (np.sum / np.mean on float64). */
static double np_pairwise(const double *a, int64_t n) {
  if (n < 8) {
    double r = 0.;
    for (int64_t i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; k++) r[k] = a[k];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

/* numpy pairwise summation of complex128 (n counts doubles). */
static void np_cpairwise(double *rr, double *ri, const double *a, int64_t n) {
  if (n < 8) {
    *rr = 0.; *ri = 0.;
    for (int64_t i = 0; i < n; i += 2) { *rr += a[i]; *ri += a[i + 1]; }
    return;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; k++) r[k] = a[k];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += a[i + k];
    *rr = ((r[0] + r[2]) + (r[4] + r[6]));
    *ri = ((r[1] + r[3]) + (r[5] + r[7]));
    for (; i < n; i += 2) { *rr += a[i]; *ri += a[i + 1]; }
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  double r1, i1, r2, i2;
  np_cpairwise(&r1, &i1, a, n2);
  np_cpairwise(&r2, &i2, a + n2, n - n2);
  *rr = r1 + r2;
  *ri = i1 + i2;
}

/* ---- transform.py ------------------------------------------------------- */

/* transform.py:48-53 _bit_reversal_indices */
void afdo_bitrev(int64_t n, int64_t *rev) {
  int64_t len = 1;
  rev[0] = 0;
  while (len < n) {
    for (int64_t i = 0; i < len; i++) {
      rev[len + i] = 2 * rev[i] + 1;
      rev[i] = 2 * rev[i];
    }
    len *= 2;
  }
}

/* transform.py:73-93 _butterflies on one row, twiddles w = half table
 * exp(-2 pi i k/N) (transform.py:65), conjugated for the inverse direction
 * (transform.py:132,199: np.conj(w) negates the imaginary part). */
static void butterflies_row(cplx *y, int64_t n, const cplx *w, int conj) {
  for (int64_t span = 2; span <= n; span *= 2) {
    int64_t half = span / 2, stride = n / span;
    for (int64_t b = 0; b < n; b += span) {
      for (int64_t k = 0; k < half; k++) {
        cplx tw = w[k * stride];
        if (conj) tw.im = -tw.im;
        cplx lo = y[b + k], hi = y[b + half + k];
        cplx t = np_cmul(hi, tw);
        y[b + half + k].re = lo.re - t.re;
        y[b + half + k].im = lo.im - t.im;
        y[b + k].re = lo.re + t.re;
        y[b + k].im = lo.im + t.im;
      }
    }
  }
}

/* transform.py:106-124 dft_forward (x complex; bit-reversed gather first). */
void afdo_dft_forward(const cplx *x, int64_t n, const cplx *w, cplx *out) {
  int64_t *rev = malloc(sizeof(int64_t) * n);
  afdo_bitrev(n, rev);
  for (int64_t i = 0; i < n; i++) out[i] = x[rev[i]];
  butterflies_row(out, n, w, 0);
  free(rev);
}

/* transform.py:127-134 dft_inverse: conj twiddles then `y /= n`
 * (numpy complex/int: Smith with (n,0) -> each part times 1/n). */
void afdo_dft_inverse(const cplx *c, int64_t n, const cplx *w, cplx *out) {
  int64_t *rev = malloc(sizeof(int64_t) * n);
  afdo_bitrev(n, rev);
  for (int64_t i = 0; i < n; i++) out[i] = c[rev[i]];
  butterflies_row(out, n, w, 1);
  cplx d = {(double)n, 0.0};
  for (int64_t i = 0; i < n; i++) out[i] = np_cdiv(out[i], d);
  free(rev);
}

/* One field row, transform.py:185-201 restricted to radius r:
 *   powers = cumprod([1, r, r, ...]) then columns bit-reversed (137-151)
 *   y = powers * c[rev]                                         (198)
 *   inverse butterflies with conj(w)                            (199)
 *   y *= scale                                                  (200)  */
static void field_row(const cplx *ghat, int64_t n, double r, double scale,
                      const cplx *w, const int64_t *rev, double *pw, cplx *y) {
  pw[0] = 1.0;
  for (int64_t l = 1; l < n; l++) pw[l] = pw[l - 1] * r;   /* np.cumprod */
  for (int64_t p = 0; p < n; p++) {
    int64_t l = rev[p];
    y[p].re = pw[l] * ghat[l].re;
    y[p].im = pw[l] * ghat[l].im;
  }
  butterflies_row(y, n, w, 1);
  for (int64_t p = 0; p < n; p++) { y[p].re *= scale; y[p].im *= scale; }
}

static int resolve_threads(int nthreads) {
  if (nthreads > 0) return nthreads;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

typedef struct { double mag; int64_t flat; double re, im; } afdo_cand;

/* Work shared by the row workers: rows [m0, m1) of one field, handed out
 * one at a time through an atomic counter. */
typedef struct {
  const cplx *ghat; int64_t n; const double *radii; const double *scales;
  int64_t m0, m1; const cplx *w; const int64_t *rev;
  cplx *out;            /* materialised rows (afdo_field) or NULL       */
  afdo_cand *per;       /* per-row best (afdo_field_argmax) or NULL     */
  int64_t next;         /* atomic row counter                           */
} row_job;

static void *row_worker(void *arg) {
  row_job *jb = (row_job *)arg;
  int64_t n = jb->n;
  double *pw = malloc(sizeof(double) * n);
  cplx *tmp = jb->out ? NULL : malloc(sizeof(cplx) * n);
  for (;;) {
    int64_t s = __atomic_fetch_add(&jb->next, 1, __ATOMIC_RELAXED);
    if (s >= jb->m1) break;
    cplx *y = jb->out ? jb->out + (s - jb->m0) * n : tmp;
    field_row(jb->ghat, n, jb->radii[s], jb->scales[s], jb->w, jb->rev, pw, y);
    if (jb->per) {
      /* core.py:298-299: magnitude = re**2 + im**2; np.argmax = first max */
      afdo_cand c = {-1.0, -1, 0.0, 0.0};
      for (int64_t j = 0; j < n; j++) {
        double mg = y[j].re * y[j].re + y[j].im * y[j].im;
        if (mg > c.mag) { c.mag = mg; c.flat = s * n + j; c.re = y[j].re; c.im = y[j].im; }
      }
      jb->per[s - jb->m0] = c;
    }
  }
  free(pw);
  free(tmp);
  return NULL;
}

static void run_rows(row_job *jb, int nthreads) {
  int nt = resolve_threads(nthreads);
  int64_t rows = jb->m1 - jb->m0;
  if (nt > rows) nt = (int)(rows > 0 ? rows : 1);
  jb->next = jb->m0;
  if (nt <= 1) { row_worker(jb); return; }
  pthread_t *th = malloc(sizeof(pthread_t) * nt);
  for (int t = 0; t < nt; t++) pthread_create(&th[t], NULL, row_worker, jb);
  for (int t = 0; t < nt; t++) pthread_join(th[t], NULL);
  free(th);
}

/* Materialised field rows m0..m1-1 (core.inner_product_field, core.py:259-282). */
void afdo_field(const cplx *ghat, int64_t n, const double *radii, const double *scales,
                int64_t m0, int64_t m1, const cplx *w, cplx *out, int nthreads) {
  int64_t *rev = malloc(sizeof(int64_t) * n);
  afdo_bitrev(n, rev);
  row_job jb = {ghat, n, radii, scales, m0, m1, w, rev, out, NULL, 0};
  run_rows(&jb, nthreads);
  free(rev);
}

/* core.maximal_selection (core.py:285-300) fused with the field: rows are
 * evaluated in parallel and merged in row order with a strict '>' so the
 * earliest row wins ties (np.argmax first-maximum, row-major). */
void afdo_field_argmax(const cplx *ghat, int64_t n, const double *radii, const double *scales,
                       int64_t m0, int64_t m1, const cplx *w, afdo_cand *best, int nthreads) {
  int64_t rows = m1 - m0;
  int64_t *rev = malloc(sizeof(int64_t) * n);
  afdo_bitrev(n, rev);
  afdo_cand *per = malloc(sizeof(afdo_cand) * (rows > 0 ? rows : 1));
  row_job jb = {ghat, n, radii, scales, m0, m1, w, rev, NULL, per, 0};
  run_rows(&jb, nthreads);
  afdo_cand b = {-1.0, -1, 0.0, 0.0};
  for (int64_t i = 0; i < rows; i++)
    if (per[i].mag > b.mag) b = per[i];
  *best = b;
  free(per);
  free(rev);
}

/* ---- core.py ------------------------------------------------------------ */

/* core.py:195-198 discrete_energy: np.mean(g.real**2 + g.imag**2). */
double afdo_energy(const cplx *g, int64_t n) {
  double *e = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; i++) e[i] = g[i].re * g[i].re + g[i].im * g[i].im;
  double s = np_pairwise(e, n);
  free(e);
  return s / (double)n;
}

/* core.py:375 complex(np.mean(remainder)) */
void afdo_cmean(const cplx *g, int64_t n, cplx *out) {
  double rr, ri;
  np_cpairwise(&rr, &ri, (const double *)g, 2 * n);
  cplx s = {rr, ri}, d = {(double)n, 0.0};
  *out = np_cdiv(s, d);
}

/* sqrt(1.0 - abs(value) ** 2) as CPython + numpy evaluate it (core.py:238):
 * abs(complex) is libm hypot, float ** 2 is libm pow. */
double afdo_kernel_norm(double a_re, double a_im) {
  volatile double two = 2.0;  /* keep gcc from folding pow(x, 2) into x*x */
  double h = hypot(a_re, a_im);
  return sqrt(1.0 - pow(h, two));
}

/* core.py:234-238 kernel_samples */
void afdo_kernel_samples(double a_re, double a_im, int64_t n, const cplx *z, cplx *out) {
  double s = afdo_kernel_norm(a_re, a_im);
  cplx ca = {a_re, -a_im}, sc = {s, 0.0};
  for (int64_t m = 0; m < n; m++) {
    cplx p = np_cmul(ca, z[m]);
    cplx d = {1.0 - p.re, 0.0 - p.im};
    out[m] = np_cdiv(sc, d);
  }
}

/* core.py:241-245 blaschke_samples: (z - a)/(1 - conj(a) z) */
void afdo_blaschke_samples(double a_re, double a_im, int64_t n, const cplx *z, cplx *out) {
  cplx ca = {a_re, -a_im};
  for (int64_t m = 0; m < n; m++) {
    cplx p = np_cmul(ca, z[m]);
    cplx d = {1.0 - p.re, 0.0 - p.im};
    cplx num = {z[m].re - a_re, z[m].im - a_im};
    out[m] = np_cdiv(num, d);
  }
}

/* core.py:303-314 remainder_update:
 *   stripped = g - c * kernel_samples(a)
 *   out = stripped * (1.0 - conj(a) z) / (z - a)                        */
void afdo_remainder_update(const cplx *g, int64_t n, double a_re, double a_im,
                           double c_re, double c_im, const cplx *z, cplx *out) {
  double s = afdo_kernel_norm(a_re, a_im);
  cplx ca = {a_re, -a_im}, sc = {s, 0.0}, c = {c_re, c_im};
  const int el = ELIDE(n);
  for (int64_t m = 0; m < n; m++) {
    cplx p = np_cmul(ca, z[m]);
    cplx d = {1.0 - p.re, 0.0 - p.im};
    cplx e = np_cdiv(sc, d);
    /* core.py:313 `c * kernel_samples(...)`: the kernel samples are a fresh
     * temporary -> elided to `ks *= c` for large N. */
    cplx ce = el ? np_cmul(e, c) : np_cmul(c, e);
    cplx st = {g[m].re - ce.re, g[m].im - ce.im};
    /* core.py:314 `stripped * (1.0 - conj(a) z)`: right operand temporary. */
    cplx num = el ? np_cmul(d, st) : np_cmul(st, d);
    cplx den = {z[m].re - a_re, z[m].im - a_im};
    out[m] = np_cdiv(num, den);
  }
}

/* core.py:317-391 decompose, engine="fft".  threshold <= 0 means None.
 * Returns the number of recorded steps; *initial receives the initial
 * energy; remainder receives the final G_{n+1} (a copy of g when the
 * input has zero energy, core.py:366-368). */
int afdo_decompose(const cplx *g, int64_t n, const double *radii, int64_t m,
                   const double *scales, const cplx *w, const cplx *z,
                   int max_terms, double threshold, int dc_first, int nthreads,
                   afdo_step *steps, cplx *remainder, double *initial) {
  double e0 = afdo_energy(g, n);
  *initial = e0;
  memcpy(remainder, g, sizeof(cplx) * n);
  if (e0 == 0.0) return 0;
  cplx *ghat = malloc(sizeof(cplx) * n);
  cplx *next = malloc(sizeof(cplx) * n);
  int count = 0;
  for (int k = 0; k < max_terms; k++) {
    afdo_step st;
    if (k == 0 && dc_first) {
      cplx mean;
      afdo_cmean(remainder, n, &mean);
      st.s = 0; st.j = 0; st.radius = 0.0; st.a_re = 0.0; st.a_im = 0.0;
      st.c_re = mean.re; st.c_im = mean.im;
    } else {
      afdo_cand b;
      afdo_dft_forward(remainder, n, w, ghat);
      afdo_field_argmax(ghat, n, radii, scales, 0, m, w, &b, nthreads);
      st.s = b.flat / n; st.j = b.flat % n; st.radius = radii[st.s];
      /* grid.point (core.py:163-167): r * exp(2 pi i j / N) == r * z[j] */
      st.a_re = st.radius * z[st.j].re;
      st.a_im = st.radius * z[st.j].im;
      st.c_re = b.re; st.c_im = b.im;
    }
    afdo_remainder_update(remainder, n, st.a_re, st.a_im, st.c_re, st.c_im, z, next);
    memcpy(remainder, next, sizeof(cplx) * n);
    st.residual = afdo_energy(remainder, n);
    steps[count++] = st;
    if (threshold > 0.0 && st.residual <= threshold * e0) break;
    if (st.residual == 0.0) break;
  }
  free(ghat);
  free(next);
  return count;
}

/* core.py:442-460 error_trace (and core.py:411-427 reconstruct for the
 * final partial sum, written to total_out when non-NULL). */
void afdo_error_trace(const cplx *g, int64_t n, const afdo_step *steps, int nsteps,
                      const cplx *z, double *errors, cplx *total_out) {
  cplx *total = calloc(n, sizeof(cplx));
  cplx *bp = malloc(sizeof(cplx) * n);
  cplx *ks = malloc(sizeof(cplx) * n);
  cplx *bs = malloc(sizeof(cplx) * n);
  cplx *diff = malloc(sizeof(cplx) * n);
  for (int64_t i = 0; i < n; i++) { bp[i].re = 1.0; bp[i].im = 0.0; }
  double eg = afdo_energy(g, n);
  const int el = ELIDE(n);
  for (int k = 0; k < nsteps; k++) {
    cplx c = {steps[k].c_re, steps[k].c_im};
    afdo_kernel_samples(steps[k].a_re, steps[k].a_im, n, z, ks);
    afdo_blaschke_samples(steps[k].a_re, steps[k].a_im, n, z, bs);
    for (int64_t i = 0; i < n; i++) {
      /* core.py:458-459; elision swaps `c * ks` and `bp * bs` for large N */
      cplx cks = el ? np_cmul(ks[i], c) : np_cmul(c, ks[i]);
      cplx t = np_cmul(cks, bp[i]);
      total[i].re = total[i].re + t.re;
      total[i].im = total[i].im + t.im;
      bp[i] = el ? np_cmul(bs[i], bp[i]) : np_cmul(bp[i], bs[i]);
    }
    if (errors) {
      for (int64_t i = 0; i < n; i++) {
        diff[i].re = g[i].re - total[i].re;
        diff[i].im = g[i].im - total[i].im;
      }
      errors[k] = afdo_energy(diff, n) / eg;
    }
  }
  if (total_out) memcpy(total_out, total, sizeof(cplx) * n);
  free(total); free(bp); free(ks); free(bs); free(diff);
}

/* core.py:201-231 analytic_projection (x real, length n). */
void afdo_analytic_projection(const double *x, int64_t n, const cplx *w, cplx *out) {
  cplx *xc = calloc(n, sizeof(cplx));
  cplx *sp = malloc(sizeof(cplx) * n);
  for (int64_t i = 0; i < n; i++) { xc[i].re = x[i]; xc[i].im = 0.0; }
  afdo_dft_forward(xc, n, w, sp);
  int64_t half = n / 2;
  for (int64_t i = 1; i < half; i++) { sp[i].re *= 2.0; sp[i].im *= 2.0; }
  for (int64_t i = half + 1; i < n; i++) { sp[i].re = 0.0; sp[i].im = 0.0; }
  afdo_dft_inverse(sp, n, w, out);
  free(xc);
  free(sp);
}

int afdo_max_threads(void) { return resolve_threads(0); }
