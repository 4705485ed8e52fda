// afd_step_cluster.cuh — the per-step select / update / energy / forward
// transform of one signal spread over a thread-block cluster of C CTAs
// (C SMs; C = 8 for N = 1024, 16 - a non-portable cluster size - for
// 2048 <= N <= 8192) with distributed shared memory.
//
// Same arithmetic, same results as step_kernel (afd_kernels.cuh); only the
// work distribution differs:
//   * CTA c owns natural samples m in [c*NC, (c+1)*NC), NC = N/C: it
//     updates them (core.py:303-314) and sums their |G|^2 - with NC >= 128 a
//     power of two, that slice is exactly one node of numpy's pairwise-sum
//     tree, so the C node sums combined as a left+right binary tree
//     reproduce np.mean bit for bit (core.py:195-198).  dc_first's complex
//     mean (core.py:375) is combined the same way.
//   * The forward DIT (transform.py:106-124): stages 0..K-CB-1 (CB = log2 C)
//     pair positions inside aligned blocks of NC bit-reversed positions, so
//     CTA c runs them on positions [c*NC, (c+1)*NC) (inputs gathered over
//     DSMEM: natural index l = C*rev(q) + rev_CB(c)); stages K-CB..K-1 pair
//     positions that differ in the top CB bits, so after a cluster barrier
//     CTA c runs them as radix-C butterflies on NC/C position groups
//     q + NC*u, u < C, gathered from all C CTAs over DSMEM.  Every butterfly
//     uses numpy's N-point table value, as in the reference.
#pragma once

#include <cooperative_groups.h>

#include "afd_kernels.cuh"

namespace afd {

namespace cg = cooperative_groups;

// cluster size used for a transform length 2^K (the slice must stay >= 128)
__host__ __device__ constexpr int cluster_ctas(int K) { return K >= 11 ? 16 : 8; }

#ifdef AFD_STEP_TIMING
__device__ unsigned long long g_step_stamps[64][24];
__device__ unsigned long long g_step_cta_start[64][16];  // per-CTA start, signal 0
// stamp row of this step, resolved once (opaque register) so that a stamp
// never waits on a constant-bank load
#define STAMP(i)                                                                       \
  do {                                                                                 \
    if (stamp_row != nullptr) {                                                        \
      unsigned long long t_;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
      stamp_row[i] = t_;                                                               \
    }                                                                                  \
  } while (0)
#else
#define STAMP(i) \
  do {           \
  } while (0)
#endif

template <int K>
struct ClusterGeo {
  static constexpr int C = cluster_ctas(K);         // CTAs per cluster
  static constexpr int CB = C == 16 ? 4 : 3;        // log2 C
  static constexpr int N = 1 << K;
  static constexpr int NC = N / C;                  // samples / positions per CTA
  static constexpr int KL = K - CB;                 // bits of the CTA-local transform
  static constexpr int RB = 2;                      // local pass register bits
  using GL = Geo<KL, RB>;                           // local transform geometry
  static constexpr int LOCAL_THREADS = GL::T;       // threads of the local transform
  static constexpr int GROUPS = NC / C;             // radix-C groups per CTA in phase 2
  static constexpr int H = C / 4;                   // phase-2 threads per group (4 points each)
  static constexpr int LH = H == 4 ? 2 : 1;         // log2 H
  static constexpr int P2_THREADS = GROUPS * H;     // = NC / 4
  static constexpr int THREADS = 256;
  static_assert(NC >= 128, "slice must be a pairwise-sum tree node");
  static_assert(LOCAL_THREADS < THREADS && P2_THREADS <= THREADS, "block too small");
  static_assert(P2_THREADS % 32 == 0, "phase-2 groups must not straddle warps");
};

template <int K>
struct ClusterSmem {
  using CG = ClusterGeo<K>;
  static constexpr size_t slice = 0;                                   // NC double2
  static constexpr size_t part = slice + sizeof(double2) * CG::NC;     // GL::SMEM double2
  static constexpr size_t emag = part + sizeof(double2) * CG::GL::SMEM;  // NC double
  static constexpr size_t twl = emag + sizeof(double) * CG::NC;          // NC-1 double2
  static constexpr size_t scratch = twl + sizeof(double2) * (CG::NC - 1);  // 2*(NC/8+16)
  static constexpr size_t circ = scratch + sizeof(double) * 2 * (CG::NC / 8 + 16);  // N double2
  static constexpr size_t rad = circ + sizeof(double2) * CG::N;  // up to kRadSmem radii
  static constexpr int kRadSmem = K >= 13 ? 1024 : 4096;  // N = 8192: smem is nearly full
  static constexpr size_t bytes = rad + sizeof(double) * kRadSmem;
  static_assert(circ % 16 == 0, "bulk-copy destination must be 16-byte aligned");
  static_assert(bytes + 1024 <= 232448, "cluster step kernel exceeds shared memory");
};

// left+right binary tree over C values (numpy pairwise halves)
template <int C>
__device__ __forceinline__ double tree_combine(const double* v) {
  if constexpr (C == 1) {
    return v[0];
  } else {
    return tree_combine<C / 2>(v) + tree_combine<C / 2>(v + C / 2);
  }
}

// Local stage tables S_0..S_{K-4} copied to shared memory.
struct LocalTw {
  const double2* sm;
  __device__ __forceinline__ double2 operator()(int b, int k) const { return sm[(1 << b) - 1 + k]; }
};

// Launched with a runtime cluster dimension of ClusterGeo<K>::C.
template <int K, bool MARG = false>
__global__ void __launch_bounds__(256)
step_cluster_kernel(int k, int max_terms, double threshold, int dc_first,
                    const double2* __restrict__ g0, double2* __restrict__ rem,
                    double2* __restrict__ ghat, const Cand* __restrict__ cand, int ncand,
                    const double* __restrict__ radii, int nrad,
                    const double2* __restrict__ circle, const double2* __restrict__ twst,
                    State* __restrict__ state, Step* __restrict__ steps,
                    const double* __restrict__ pow2, const double* __restrict__ cand2) {
  using CG = ClusterGeo<K>;
  using L = ClusterSmem<K>;
  using GL = typename CG::GL;
  constexpr int N = CG::N, NC = CG::NC, C = CG::C, CB = CG::CB;
  // parameters used after the PDL wait live in registers (see opq)
  k = opq(k);
  max_terms = opq(max_terms);
  threshold = opq(threshold);
  dc_first = opq(dc_first);
  ncand = opq(ncand);
  nrad = opq(nrad);
  cand = opq(cand);
  radii = opq(radii);
  steps = opq(steps);
  state = opq(state);
  rem = opq(rem);
  ghat = opq(ghat);
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  const int sig = blockIdx.x / C;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* slice = reinterpret_cast<double2*>(smraw + L::slice);
  double2* part = reinterpret_cast<double2*>(smraw + L::part);
  double* emag = reinterpret_cast<double*>(smraw + L::emag);  // |G_{k+1}|^2, my natural slice
  double2* twl = reinterpret_cast<double2*>(smraw + L::twl);
  double* scratch = reinterpret_cast<double*>(smraw + L::scratch);
  double2* circ = reinterpret_cast<double2*>(smraw + L::circ);  // z_m, all N
  double* rad = reinterpret_cast<double*>(smraw + L::rad);    // radii (if <= kRadSmem)
  __shared__ double s_node[2];   // this CTA's pairwise-tree node sums
  __shared__ double s_nodes[16];  // CTA 0: every CTA's energy node sum
  State& st = state[sig];
  double2* __restrict__ r = rem + (size_t)sig * N;
  double2* __restrict__ gh = ghat + (size_t)sig * N;
  const int tid = threadIdx.x;
  const int m0 = c * NC;
#ifdef AFD_STEP_TIMING
  unsigned long long* stamp_row = nullptr;
  if (threadIdx.x == 0 && blockIdx.x == 0 && k >= 0 && k < 64) {
    unsigned long long* p_ = &g_step_stamps[k][0];
    asm volatile("mov.b64 %0, %1;" : "=l"(stamp_row) : "l"(p_));
  }
#endif
  STAMP(0);
#ifdef AFD_STEP_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 16 && k >= 0 && k < 64) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_step_cta_start[k][blockIdx.x] = t_;
  }
#endif

  // The whole circle z_m (step-independent) lands in shared memory by bulk
  // copy: the pole lookup circle[j] and this CTA's update slice read it there.
  __shared__ unsigned long long circ_bar;
  if (tid == 0) {
    mbar_init(&circ_bar, 1);
    const unsigned m = (unsigned)__cvta_generic_to_shared(&circ_bar);
    constexpr unsigned bytes = sizeof(double2) * N;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
                 : "memory");
    constexpr unsigned chunk = 32768;
    for (unsigned off = 0; off < bytes; off += chunk) {
      const unsigned nb = bytes - off < chunk ? bytes - off : chunk;
      const unsigned d = (unsigned)__cvta_generic_to_shared((char*)circ + off);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(d), "l"((const char*)circle + off), "r"(nb), "r"(m)
          : "memory");
    }
  }
  // local stage tables S_0..S_{K-CB-1} (== twst[0 .. NC-1))
  for (int i = tid; i < NC - 1; i += CG::THREADS) twl[i] = __ldg(twst + i);
  // Phase-2 twiddles of this thread (radix-C group q, sub-thread h; stage
  // b = K-CB+e uses w[(q + NC*(u mod 2^e)) << (CB-1-e)]), prefetched:
  //   layout A (u = 4h + i, e = 0, 1): u mod 2^e = i mod 2^e
  //   layout B (u = h + H i, e >= 2): u mod 2^e = h + H (i mod 2^(e-LH))
  constexpr int H = CG::H, LH = CG::LH;
  const int gq = tid / H, hh = tid % H;
  const int q = c * CG::GROUPS + gq;
  double2 wa[3], wb[4];
  if (tid < CG::P2_THREADS) {
    const double2* half = twst + (N / 2) - 1;  // S_{K-1}[k] = w[k]
    wa[0] = __ldg(half + (q << (CB - 1)));
    wa[1] = __ldg(half + (q << (CB - 2)));
    wa[2] = __ldg(half + ((q + NC) << (CB - 2)));
#pragma unroll
    for (int e = 2; e < CB; ++e)
#pragma unroll
      for (int mm = 0; mm < (1 << (e - LH)); ++mm)
        wb[(1 << (e - LH)) - 1 + mm] = __ldg(half + ((q + NC * (hh + H * mm)) << (CB - 1 - e)));
  }
  // this CTA's slice of the remainder: G_k was written by the previous step
  // kernel, which completed before our PDL predecessor (the field kernel)
  // passed its own pdl_wait and triggered us, so it is final here (except
  // for the dc_first step 0, loaded after the wait)
  // CTA c owns the samples l = C*m + rc (m < NC, rc = bitrev(c)): exactly
  // the inputs of its CTA-local DIT, so the update feeds the transform
  // without a cluster exchange (only |G|^2 goes to CTA 0 for the energy)
  constexpr int PER = (NC + CG::THREADS - 1) / CG::THREADS;
  const int rc = brev_bits(c, CB);
  double2 gs[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = tid + u * CG::THREADS;
    const int l = C * i + rc;
    if (i < NC && !(k == 0 && dc_first)) gs[u] = k >= 0 ? r[l] : g0[(size_t)sig * N + l];
  }
  // radii for grid.point: staged in shared memory when they fit
  const bool rad_smem = nrad <= L::kRadSmem;
  if (rad_smem)
    for (int i = tid; i < nrad; i += CG::THREADS) rad[i] = radii[i];
  __syncthreads();  // rad / twl / barrier init visible
  // every CTA of the cluster is running before anyone touches distributed
  // shared memory (waited right after the PDL wait)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  STAMP(1);

  pdl_wait();
  STAMP(2);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  STAMP(18);
  if (k == 0 && dc_first) {
    // this kernel's PDL predecessor is the init step kernel itself (no field
    // launch in between), so G_0 is only final after the wait
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = tid + u * CG::THREADS;
      if (i < NC) gs[u] = r[C * i + rc];
    }
  }
  // the stop flag's load overlaps the candidate loads below; it is tested
  // once the candidates are in (cluster-uniform)
  const int stopped = k >= 0 ? __ldcg(&st.stopped) : 0;

  // ---- select ---------------------------------------------------------------
  long long s = 0, j = 0;
  double radius = 0.0;
  double runner = -2.0;  // step's runner-up |F|^2 (fast engine, CTA 0 warp 0); -2: none
  double2 a = make_double2(0.0, 0.0), coeff = make_double2(0.0, 0.0);
  if (!(k >= 0 && !(k == 0 && dc_first))) {  // select-free paths
    if (stopped) {
      mbar_wait(&circ_bar, 0);
      return;
    }
    pdl_trigger();
  }
  if (k == 0 && dc_first) {
    // core.py:373-375: coeff = complex(np.mean(remainder)), pairwise over N
    for (int i = tid; i < NC; i += CG::THREADS) slice[i] = r[m0 + i];
    __syncthreads();
    const double2 node = cpairwise_sum_block(slice, NC, scratch, PlainIdx(), CG::THREADS);
    if (tid == 0) {
      s_node[0] = node.x;
      s_node[1] = node.y;
    }
    cluster.sync();
    double re[C], im[C];
#pragma unroll
    for (int u = 0; u < C; ++u) {
      const double* rn = cluster.map_shared_rank(s_node, u);
      re[u] = rn[0];
      im[u] = rn[1];
    }
    const double2 sum = make_double2(tree_combine<C>(re), tree_combine<C>(im));
    coeff = np_cdiv(sum, make_double2((double)N, 0.0));
    cluster.sync();  // everyone has read s_node before it is reused
  } else if (k >= 0) {
    // every warp reduces all candidates itself (first maximum): no block
    // barrier on the critical path
    Cand b;
    b.mag = -1.0;
    b.flat = 0x7fffffffffffffffLL;
    b.re = b.im = 0.0;
    const int lane = tid & 31;
    // up to 4 candidates per lane loaded before any is merged: one L2 round
    // trip (a plain loop issued each lane's loads one merge apart)
    const Cand* cs = cand + (size_t)sig * ncand;
    auto load_cand = [&](int i) {
      Cand x;
      const double2 lo = __ldcg(reinterpret_cast<const double2*>(cs + i));
      const double2 hi = __ldcg(reinterpret_cast<const double2*>(cs + i) + 1);
      x.mag = lo.x;
      x.flat = __double_as_longlong(lo.y);
      x.re = hi.x;
      x.im = hi.y;
      return x;
    };
    // the record's runner-up (fast engine): warp 0 of CTA 0 loads the
    // runner-up slots in the same round trip and keeps its candidates
    const bool want2 = MARG && c == 0 && tid < 32;
    Cand xs[4];
    double xs2[4] = {-1.0, -1.0, -1.0, -1.0};
    {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = lane + 32 * u;
        if (i < ncand) xs[u] = load_cand(i);
        if (want2 && i < ncand) xs2[u] = __ldcg(cand2 + (size_t)sig * ncand + i);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lane + 32 * u < ncand) cand_merge(b, xs[u]);
    }
    for (int i = lane + 128; i < ncand; i += 32) cand_merge(b, load_cand(i));
    STAMP(16);
    if (stopped) {
      mbar_wait(&circ_bar, 0);  // no bulk copy may target an exited CTA
      return;
    }
    pdl_trigger();  // (releasing the next field launch later measured slower)
    STAMP(17);
    b = warp_argmax(b);
    b.mag = __shfl_sync(0xffffffffu, b.mag, 0);
    b.flat = __shfl_sync(0xffffffffu, b.flat, 0);
    b.re = __shfl_sync(0xffffffffu, b.re, 0);
    b.im = __shfl_sync(0xffffffffu, b.im, 0);
    if (MARG && want2) {
      double r = -1.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (lane + 32 * u < ncand) {
          r = fmax(r, xs2[u]);
          if (xs[u].flat != b.flat) r = fmax(r, xs[u].mag);
        }
      }
      for (int i = lane + 128; i < ncand; i += 32) {
        const Cand x = load_cand(i);
        r = fmax(r, __ldcg(cand2 + (size_t)sig * ncand + i));
        if (x.flat != b.flat) r = fmax(r, x.mag);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
      runner = r;
    }
    STAMP(13);
    s = b.flat / N;
    j = b.flat % N;
    radius = rad_smem ? rad[s] : radii[s];
    mbar_wait(&circ_bar, 0);
    const double2 zj = circ[j];
    a = make_double2(radius * zj.x, radius * zj.y);  // grid.point, core.py:163-167
    coeff = make_double2(b.re, b.im);
    STAMP(14);
  }
  mbar_wait(&circ_bar, 0);  // (no-op when already passed) circle slice for the update

  STAMP(3);
  // ---- update this CTA's samples (or copy g0 at init) -------------------------
  int amb = 0;
  {
    // the divisions of both complex quotients depend only on a and z: they
    // are issued first and run under kernel_norm's dependency chain
    double2 dd[PER];
    CdivPre q1[PER], q2[PER];
    if (k >= 0) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int i = tid + u * CG::THREADS;
        const int l = C * (i < NC ? i : 0) + rc;
        const double2 z = circ[l];
        dd[u] = one_minus_conja_z(a, z);
        q1[u] = np_cdiv_pre(dd[u]);
        q2[u] = np_cdiv_pre(make_double2(z.x - a.x, z.y - a.y));
      }
    }
    double kn = 0.0;
    if (k >= 0) kn = kernel_norm_grid(a, radius, pow2 ? pow2 + (size_t)s * kPowRow : nullptr, &amb);
    const double2 sc = make_double2(kn, 0.0);
    STAMP(15);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = tid + u * CG::THREADS;
      if (i < NC) {
        const int l = C * i + rc;
        double2 out = gs[u];
        if (k >= 0) {
          const double2 d = dd[u];
          const double2 e = np_cdiv_fin(sc, q1[u]);  // np_cdiv(sc, d)
          const double2 ce = np_cmul(coeff, e);  // N <= 8192: no numpy elision
          const double2 g = gs[u];
          const double2 stp = make_double2(g.x - ce.x, g.y - ce.y);
          const double2 num = np_cmul(stp, d);
          out = np_cdiv_fin(num, q2[u]);  // np_cdiv(num, z - a)
        }
        slice[i] = out;
        // |G|^2 to the CTA whose natural slice holds l (a pairwise-sum node)
        cluster.map_shared_rank(emag, l / NC)[l % NC] = np_mag2(out);
        r[l] = out;  // completes under the local DIT, before the next cluster barrier
      }
    }
  }
  __syncthreads();
  STAMP(4);
  STAMP(5);
  STAMP(6);
  constexpr int kFftWarps = (CG::LOCAL_THREADS + 31) / 32;
  static_assert(kFftWarps * 32 < CG::THREADS, "need a spare warp for the energy");
  const int warp = tid >> 5;
  if (warp < kFftWarps) {
    // ---- forward transform, stages 0..K-CB-1 on positions [c*NC, (c+1)*NC) ----
    // (computed even on the last step: harmless)
    STAMP(7);
    const int tp = tid;
    const bool active = tp < CG::LOCAL_THREADS;
    double2 v[GL::P];
    if (active) {
#pragma unroll
      for (int i = 0; i < GL::P; ++i) v[i] = slice[GL::l0(tp, i)];  // l = C*l0 + rc
    }
    STAMP(8);
    fft_passes<CG::KL, false, CG::RB>(v, tp, active, part, LocalTw{twl},
                                      GroupSync{1, kFftWarps * 32});
    STAMP(9);
    if (active) {
#pragma unroll
      for (int i = 0; i < GL::P; ++i) part[GL::sw(out_pos<CG::KL, CG::RB>(tp, i))] = v[i];
    }
  }
  cluster.sync();  // DIT outputs and the |G|^2 pushes visible cluster-wide
  STAMP(10);

  // ---- stages K-CB..K-1: radix-C over the top CB position bits ----------------
  // Group q (positions q + NC*u, u < C) is held by H threads, 4 points each:
  // stages e = 0, 1 in layout A (thread h holds u = 4h + i), then a 4x4
  // transpose through shared memory (the group's H threads share a warp),
  // then stages e >= 2 in layout B (u = h + H i).
  // Meanwhile the last warp sums this CTA's |G|^2 node (numpy pairwise
  // blocks of 128 over the natural slice) and hands it to CTA 0.
  if (tid < CG::P2_THREADS) {
    double2 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = cluster.map_shared_rank(part, 4 * hh + i)[GL::sw(q)];
    // my remote reads are done: let the other CTAs go (split cluster barrier)
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
    bfly(v[0], v[1], wa[0]);  // e = 0
    bfly(v[2], v[3], wa[0]);
    bfly(v[0], v[2], wa[1]);  // e = 1: u mod 2 = i mod 2
    bfly(v[1], v[3], wa[2]);
    double2* x = slice + gq * C;  // slice is free after the cluster barrier
#pragma unroll
    for (int i = 0; i < 4; ++i) x[4 * hh + i] = v[i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = x[hh + H * i];
#pragma unroll
    for (int e = 2; e < CB; ++e) {
      const int ib = e - LH;  // bit of i paired by stage e
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i & (1 << ib)) continue;
        const double2 w = wb[(1 << ib) - 1 + (i & ((1 << ib) - 1))];
        bfly(v[i], v[i | (1 << ib)], w);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) gh[q + NC * (hh + H * i)] = v[i];
  } else if (tid >= CG::THREADS - 32) {
    // node sum: accumulator a (lane) of block a/8 sums emag[128 (a/8) + a%8 + 8 i]
    const int lane = tid & 31;
    constexpr int NB = NC / 128;  // blocks in the slice (1..4)
    double acc = 0.0;
    if (lane < 8 * NB) {
      const double* xb = emag + 128 * (lane >> 3) + (lane & 7);
      acc = xb[0];
#pragma unroll
      for (int i = 8; i < 128; i += 8) acc += xb[i];
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) per block, then blocks left+right
#pragma unroll
    for (int off = 1; off < 8 * NB; off <<= 1) {
      const double o = __shfl_down_sync(0xffffffffu, acc, off);
      if ((lane & (2 * off - 1)) == 0) acc = acc + o;
    }
    if (lane == 0) cluster.map_shared_rank(s_nodes, 0)[c] = acc;
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
  } else {
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
  }
  STAMP(11);
  // no CTA leaves while another may still read its shared memory
  asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
  STAMP(12);
  if (c == 0 && tid == 0) {
    // energy = np.mean(|G|^2) (core.py:195-198): the C node sums combined as
    // numpy's left+right tree, then / N; record, stop rules (core.py:366-389)
    const double energy = tree_combine<C>(s_nodes) / (double)N;
    if (k < 0) {
      st.initial = energy;
      st.nsteps = 0;
      st.flags = 0;
      st.stopped = (energy == 0.0) ? 1 : 0;  // core.py:366-368
    } else {
      int stop = 0;
      if (threshold > 0.0 && energy <= threshold * st.initial) stop = 1;  // core.py:386-387
      if (energy == 0.0) stop = 1;                                         // core.py:388-389
      if (k + 1 >= max_terms) stop = 1;
      Step rec;
      rec.s = s;
      rec.j = j;
      rec.radius = radius;
      rec.a_re = a.x;
      rec.a_im = a.y;
      rec.c_re = coeff.x;
      rec.c_im = coeff.y;
      rec.residual = energy;
      rec.flags = amb ? kStepPowAmbiguous : 0;
      rec.margin = runner >= -1.0 ? top2_margin(coeff_mag2(coeff), runner) : __int_as_float(0x7fc00000);
      steps[(size_t)sig * max_terms + k] = rec;
      st.nsteps = k + 1;
      st.flags |= rec.flags;
      st.stopped = stop;
    }
  }
}

}  // namespace afd
