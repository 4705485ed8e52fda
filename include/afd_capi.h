/*
 * afd_capi.h — C ABI of the B200-native FFT-AFD selection hot path.
 *
 * The reference (arXiv 1711.08604, package `fastafd`) is pure Python/numpy
 * with no FFI; its seam is the Python API.  Each entry point below replaces
 * one reference function (file:line under /root/reference/pkg/src/fastafd)
 * and reproduces its results bit for bit (numpy/CPython arithmetic is
 * emulated on the device; see paper_1711_08604_b200/csrc/afd_common.cuh).
 * The Python package `paper_1711_08604_b200` binds these with ctypes
 * (paper_1711_08604_b200/_capi.py); INTEGRATION.md shows the binding a
 * `fastafd` maintainer would add.
 *
 * Conventions
 *  - Every function returns 0 on success or a negative AFD_E* code; the
 *    message is available from afd_last_error() (thread-local).  Nothing
 *    throws across the ABI.
 *  - Complex numbers are interleaved (re, im) doubles (numpy complex128).
 *  - Pointers are DEVICE pointers owned by the caller unless named *_host.
 *    All work is stream-ordered on the caller's `stream` (a cudaStream_t;
 *    NULL = legacy default stream).
 *  - A plan binds one device, one transform length N = 2^K (8 <= N), the
 *    radius grid (M radii, of which this plan evaluates rows [m0, m1)) and
 *    a maximum batch of independent signals.  A plan's buffers are shared by
 *    its calls: calls on one plan must not overlap (the Python layer holds a
 *    per-plan lock); use one plan per concurrent caller.
 *  - Host tables are taken from the caller so both sides start from the
 *    same bits: twiddles exp(-2 pi i k/N), k < N/2 (transform.py:65),
 *    circle exp(2 pi i m/N) (core.py:87), scales
 *    sqrt(1-r^2)/(N(1-r^N)) (transform.py:153).
 */
#ifndef AFD_CAPI_H
#define AFD_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFD_OK 0
#define AFD_E_INVALID -1     /* bad argument (the reference raises ValueError)  */
#define AFD_E_CUDA -2        /* CUDA runtime error                              */
#define AFD_E_UNSUPPORTED -3 /* size not supported by this build                */
#define AFD_E_NOMEM -4       /* device allocation failed                        */

/* Step record of one AFD step (core.DecompositionStep, core.py:170-175).
 * s, j: grid indices of the selected pole a = r_s exp(2 pi i j/N)
 * (core.ParameterGrid.point, core.py:163-167); coefficient <G_k, e_a>;
 * residual = discrete_energy(G_{k+1}).  flags bit 0: the pole's
 * sqrt(1 - abs(a) ** 2) could not be taken from the plan's table of libm
 * pow(h, 2.0) values (never for grid poles: kernel_norm_grid) and the
 * device's h*h is not provably CPython's pow.  margin (fast engine with
 * AFD_PLAN_MARGINS): the step's top-2 relative margin (|F|^2_max -
 * |F|^2_runner-up) / |F|^2_max over the whole grid, the runner-up being the
 * largest |F|^2 at any other grid point; a fast pick is provably the
 * reference's when the margin exceeds the fast field's error (~1e-14).  NaN
 * when not tracked (exact engine, fast plans without AFD_PLAN_MARGINS,
 * dc_first step, radius-sharded runs).
 * 72 bytes. */
typedef struct afd_step {
  int64_t s, j;
  double radius, a_re, a_im, c_re, c_im, residual;
  int32_t flags;
  float margin;
} afd_step;

/* Grid candidate: |F|^2, flat index s*N + j (global s), F.  32 bytes.
 * Ordering: larger mag2 wins, ties go to the lower flat index (np.argmax
 * first-maximum, core.py:299). */
typedef struct afd_candidate {
  double mag2;
  int64_t flat;
  double re, im;
} afd_candidate;

typedef struct afd_plan afd_plan;

const char *afd_last_error(void);
int afd_version(void);

/* Plan flags.
 * AFD_PLAN_FAST: the field (the M x N grid of weighted inverse transforms,
 *   transform.py:185-201) is computed with FMA-fused FP64 butterflies,
 *   exact trivial rotations and r^l generated on chip from per-radius
 *   factor tables instead of the reference's radix-2 numpy arithmetic and
 *   M x N cumprod table: the selected indices are identical to the
 *   reference's and coefficients, remainders and errors agree to ~1e-14
 *   relative (the parity contract is 1e-9), not bit for bit.  Everything
 *   after the argmax (update, energy, forward transform, records) stays
 *   bit-exact arithmetic.  Default (0): bit-identical to the reference. */
#define AFD_PLAN_FAST 1
/* AFD_PLAN_MARGINS (with AFD_PLAN_FAST): the field kernels also track each
 * step's runner-up |F|^2 and the records carry the top-2 margin
 * (afd_step.margin); costs ~10-15% of the field (every value above a
 * thread's runner-up takes the slow path of the screened epilogue). */
#define AFD_PLAN_MARGINS 2

/* Create a plan.  radii_host/scales_host hold all M radii/scales
 * (core.ParameterGrid.radii, core.py:115-145); the plan evaluates global
 * rows [m0, m1) (radius sharding across GPUs).
 * Replaces transform._plan + transform._radius_tables
 * (transform.py:56-70, 137-156). */
int afd_plan_create(afd_plan **out, int device, int64_t n, int64_t m, int64_t m0, int64_t m1,
                    int64_t max_batch, const double *radii_host, const double *scales_host,
                    const double *twiddle_host /* N/2 complex */,
                    const double *circle_host /* N complex */, int flags /* AFD_PLAN_* */);
int afd_plan_destroy(afd_plan *plan);

/* transform.dft_forward / dft_inverse (transform.py:106-134), batch rows. */
int afd_dft_forward(afd_plan *plan, const double *x, double *out, int64_t batch, void *stream);
int afd_dft_inverse(afd_plan *plan, const double *c, double *out, int64_t batch, void *stream);

/* core.analytic_projection (core.py:201-231) of `batch` real rows given as
 * complex with zero imaginary part. */
int afd_analytic_projection(afd_plan *plan, const double *x, double *out, int64_t batch,
                            void *stream);

/* core.inner_product_field restricted to global rows [r0, r1) of ONE
 * signal's spectrum (transform.weighted_inverse_grid, transform.py:185-201):
 * field is (r1-r0) x N complex. */
int afd_field(afd_plan *plan, const double *ghat, double *field, int64_t r0, int64_t r1,
              void *stream);

/* Engine of the plan's decompositions (core.py:357-358, 377-381):
 * 0 = "fft" (default; transform engine, bit-identical to the reference),
 * 1 = "direct" (oracle.field_direct, O(M N^2) literal sums of the signal;
 *     matches the reference to its engine-agreement tolerance, N <= 8192). */
int afd_plan_set_engine(afd_plan *plan, int engine);

/* oracle.field_direct (oracle.py:51-73) rows [r0, r1) of ONE signal g (not
 * its spectrum): (r1-r0) x N complex. */
int afd_field_direct(afd_plan *plan, const double *g, double *field, int64_t r0, int64_t r1,
                     void *stream);

/* Fused field + maximal_selection over the plan's rows for `batch` spectra
 * (core.inner_product_field + core.maximal_selection, core.py:259-300):
 * writes one candidate per signal to out[batch]. */
int afd_field_argmax(afd_plan *plan, const double *ghat, afd_candidate *out, int64_t batch,
                     void *stream);

/* core.maximal_selection on a materialised (rows x N) field (core.py:285-300):
 * out receives the first maximum, flat index relative to the field. */
int afd_argmax(afd_plan *plan, const double *field, int64_t rows, afd_candidate *out,
               void *stream);

/* Pointwise atoms over the circle (core.py:234-245, 303-314), N points:
 *   kind 0 kernel_samples(a)      kind 1 blaschke_samples(a)
 *   kind 2 remainder_update(g, a, c)
 *   kind 3 g * blaschke_samples(a)  (core.tm_basis_samples step, core.py:406-407)
 * g is used by kinds 2 and 3 only.  norm = sqrt(1 - abs(a) ** 2) as the
 * caller's scalar arithmetic gives it (the reference evaluates it in CPython,
 * core.py:237: libm hypot and pow), or NaN to form it on the device. */
int afd_atom(afd_plan *plan, int kind, const double *g, double a_re, double a_im, double c_re,
             double c_im, double norm, double *out, void *stream);

/* core.discrete_energy (core.py:195-198) of `batch` signals -> energies[batch].
 * With s != NULL the energy of g - s (core.relative_error, core.py:430-439). */
int afd_energy(afd_plan *plan, const double *g, double *energies, int64_t batch, void *stream);
int afd_energy_diff(afd_plan *plan, const double *g, const double *s, double *energies,
                    int64_t batch, void *stream);

/* core.decompose (core.py:317-391), engine "fft", for `batch` independent
 * signals g0 (batch x N).  threshold <= 0 means None.  Outputs (device):
 * steps[batch][max_terms], n_steps[batch], initial[batch] (initial energy),
 * remainder[batch][N] (final G_{n+1}; a copy of g0 for zero-energy input).
 * The loop runs device-resident (captured once into a CUDA graph per
 * (max_terms, threshold, dc_first, batch)).  Requires m0 == 0 && m1 == M
 * (single-shard plan); sharded plans use afd_select_local/afd_apply_step. */
int afd_decompose(afd_plan *plan, const double *g0, int64_t batch, int max_terms,
                  double threshold, int dc_first, afd_step *steps, int32_t *n_steps,
                  double *initial, double *remainder, void *stream);

/* afd_decompose with HOST buffers (pageable or pinned): the library stages
 * the input through its own pinned buffer, copies it to the device, replays
 * the decomposition graph, gathers all outputs into one packed device buffer,
 * copies that back with a single transfer and synchronises `stream` once.
 * This is the reference-facing call (core.decompose on host numpy arrays).
 * *h2d_bytes / *d2h_bytes (may be NULL) receive the bytes moved. */
int afd_decompose_host(afd_plan *plan, const double *g0_host, int64_t batch, int max_terms,
                       double threshold, int dc_first, afd_step *steps_host,
                       int32_t *n_steps_host, double *initial_host, double *remainder_host,
                       int64_t *h2d_bytes, int64_t *d2h_bytes, void *stream);

/* Radius-sharded decomposition, one step at a time:
 *   afd_sharded_begin        copy g0, initial energy, first spectrum
 *   afd_select_local         field + argmax over the plan's rows -> cand[batch]
 *   (caller all-gathers the candidates of all ranks, rank-major)
 *   afd_apply_step           reduce cands[batch][ncand], update, energy, record,
 *                            next spectrum; identical on every rank
 *   afd_sharded_state        n_steps / stopped flags / initial energies   */
int afd_sharded_begin(afd_plan *plan, const double *g0, int64_t batch, void *stream);
int afd_select_local(afd_plan *plan, int k, int dc_first, afd_candidate *cand, int64_t batch,
                     void *stream);
int afd_apply_step(afd_plan *plan, int k, int max_terms, double threshold, int dc_first,
                   const afd_candidate *cands, int ncand, int64_t batch, afd_step *steps,
                   void *stream);
int afd_sharded_finish(afd_plan *plan, int64_t batch, int32_t *n_steps, double *initial,
                       double *remainder, int32_t *stopped, void *stream);

/* Device-resident radius-sharded decomposition (SURVEY.md §8(b)'s
 * afd_decompose(..., nccl_comm)).  A communicator is an NCCL communicator
 * over the ranks that share the radius grid (one process per GPU); the
 * library loads libnccl.so.2 at run time (the copy already in the process,
 * e.g. torch's, else the system's).  Rank 0 calls afd_comm_unique_id and
 * the caller distributes the 128 bytes to every rank (any side channel:
 * torch.distributed, MPI, a file), then each rank calls afd_comm_init.
 *
 * afd_decompose_sharded: every rank passes the same g0 and a plan over its
 * own rows [m0, m1); the whole loop — local field + argmax, an ncclAllGather
 * of one 32-byte candidate per rank and signal, the replicated update,
 * energy and next spectrum — is captured once into a CUDA graph (per comm,
 * max_terms, threshold, dc_first, batch, stream) and replayed, so no step
 * returns to the host.  Outputs as afd_decompose, identical on every rank
 * and identical to the unsharded result.  Replaces the reference's only
 * parallelism, the radius-row thread pool (core.py:253-282). */
typedef struct afd_comm afd_comm;
int afd_comm_unique_id(void *id_out /* 128 bytes */);
int afd_comm_init(afd_comm **out, const void *id /* 128 bytes */, int world, int rank,
                  int device);
int afd_comm_destroy(afd_comm *comm);
int afd_decompose_sharded(afd_plan *plan, afd_comm *comm, const double *g0, int64_t batch,
                          int max_terms, double threshold, int dc_first, afd_step *steps,
                          int32_t *n_steps, double *initial, double *remainder, void *stream);

/* core.error_trace + core.reconstruct (core.py:411-460) for `batch` signals:
 * errors[batch][max_terms] (entry k = relative error of the (k+1)-term
 * partial sum), recon[batch][N] = S_{n_steps} (may be NULL).  norms
 * [batch][max_terms] (may be NULL: formed on the device) are the poles'
 * sqrt(1 - abs(a) ** 2), as for afd_atom. */
int afd_error_trace(afd_plan *plan, const double *g, const afd_step *steps, int max_terms,
                    const int32_t *n_steps, int64_t batch, const double *norms, double *errors,
                    double *recon, void *stream);

/* Number of this library's kernels launched since plan creation (counts
 * launches issued, including those replayed inside CUDA graphs). */
int64_t afd_launch_count(afd_plan *plan);

/* Diagnostics (not reference functions).
 * afd_time_field: `reps` back-to-back launches of the fused field+argmax
 * kernel over the plan's rows for `batch` spectra, each bracketed by CUDA
 * events on `stream`; *avg_ms = mean event time per launch.
 * afd_fp64_peak: DFMA throughput microbenchmark on `device` (independent
 * FMA chains on every SM), *tflops counts 2 flops per DFMA. */
int afd_time_field(afd_plan *plan, const double *ghat, int64_t batch, int reps, double *avg_ms,
                   void *stream);
/* afd_field_split: how the last large-N fast field evaluation on `stream`
 * (synchronised here) split the plan's rows: *onchip rows went through the
 * pruned on-chip 4096-point transforms (their weight tail r^l, l >= 4096,
 * is below 2^-64 of the largest kept term), *twopass rows through pass A +
 * the TMA column pass.  Exact plans and N <= 8192: *onchip = 0 and every
 * row is counted as *twopass (large N) or *onchip = rows (on-chip N). */
int afd_field_split(afd_plan *plan, int64_t *onchip, int64_t *twopass, void *stream);
/* afd_field_tiers: the same split by on-chip tier: rows3[0] rows as
 * at most 1024-point transforms (tail beyond l = 1024 negligible), rows3[1] as
 * 4096-point transforms, rows3[2] two-pass (zeros for on-chip N). */
int afd_field_tiers(afd_plan *plan, int64_t *rows3, void *stream);
/* afd_field_tier_rows: the split by every tier, in row order: terms[t] =
 * spectrum terms a row of tier t is evaluated from (32, 64, 128: in
 * registers, one thread per 32 outputs; 256, 512 (when in use), 1024, 4096:
 * on-chip transforms; N: two-pass — for batches of on-chip N: the N-point
 * field kernel, rows summed over the signals — the last entry), rows[t] =
 * its rows in the last evaluation.
 * Writes *count <= cap entries (cap >= 8 always suffices; one entry
 * {N, all rows} for unpruned plans). */
int afd_field_tier_rows(afd_plan *plan, int64_t *terms, int64_t *rows, int cap, int *count,
                        void *stream);
int afd_fp64_peak(int device, double *tflops, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* AFD_CAPI_H */
