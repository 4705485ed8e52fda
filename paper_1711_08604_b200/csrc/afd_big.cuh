// afd_big.cuh — transform lengths N = 2^K > 8192 (BASELINE c2: 2^16,
// c4: 2^20), where one row no longer fits in shared memory.
//
// The reference's radix-2 DIT (transform.py:73-93) is split by stage bits:
//   pass A  stages 0..11: they pair positions inside aligned blocks of 4096
//           bit-reversed positions, so one CTA runs them on-chip exactly as
//           afd_fft.cuh does (the N-table stage twiddles S_b, b < 12, are the
//           same per-stage tables; SmemTw<12> reads them from the N plan);
//   pass C  stages b0..b0+3 (b0 = 12, 16): they pair positions that differ
//           in bits b0..b0+3 only, so each thread owns one "column"
//           q + 2^b0 u, u < 16, and runs 4 stages in registers; lanes own
//           consecutive q, so every load/store is coalesced.
// Intermediates live in a row-batch buffer sized to stay L2-resident.  The
// input of pass A is the bit-reversed gather of transform.py:151,198, stored
// directly in pass A's register layout: inside each 2^KA block, position
// (rev(t) << 4) | i (what register i of thread t holds in pass 0) lives at
// index i*T + t, so pass A loads straight into registers, coalesced.  The
// plan keeps the r^l table that way (pw_perm) and the step kernels write the
// field spectrum that way (ghat_perm).
// Every butterfly is the reference's, so results stay bit-identical.
//
// Per-step bookkeeping for large N is split over grid kernels: the numpy
// pairwise sum over N (core.py:195-198) is reproduced from per-CTA node sums
// over aligned 2048-sample slices (nodes of numpy's halving tree) combined
// left+right by a single CTA.
#pragma once

#include "afd_kernels.cuh"

namespace afd {

constexpr int kNodeLen = 2048;             // samples per energy node
constexpr int kMaxNodes = (1 << 22) / kNodeLen;  // node sums at the largest N (2^22)
constexpr int kColThreads = 256;

// Pass-A bits: K = KA + 4 c with 9 <= KA <= 12 (K = 14..22).
__host__ __device__ constexpr int big_ka(int K) { return K - 4 * ((K - 9) / 4); }

template <int KA>
__host__ __device__ constexpr size_t big_a_smem() {
  return sizeof(double2) * (SmemTw<KA, 4>::ENTRIES + Geo<KA, 4>::SMEM);
}

__device__ __forceinline__ int brev_rt(int x, int bits) { return (int)(__brev((unsigned)x) >> (32 - bits)); }

// index of bit-reversed-array position p in the pass-A register layout
__device__ __forceinline__ long long perm_of_pos(long long p, int ka) {
  const int T = 1 << (ka - 4);
  const int q = (int)(p & ((1LL << ka) - 1));
  const int tp = brev_rt(q >> 4, ka - 4);
  return (p & ~((1LL << ka) - 1)) + (long long)(q & 15) * T + tp;
}

// ---------------------------------------------------------------------------
// Pass A.  mode 0: field prologue y[p] = pw_rev[row][p] * ghat_rev[p]
//          mode 1: transform of one signal, input gathered x[rev(p)] (natural x)
// blockIdx.x = 4096-block, blockIdx.y = row within the batch.
// ---------------------------------------------------------------------------
// Persistent over work items (row, block): 2 row-groups of T threads per
// CTA, each with its own buffer and named barrier, so one group's loads
// overlap the other's butterflies; twiddles are loaded once per CTA.
constexpr int kBigGroups = 2;

template <int KA>
__host__ __device__ constexpr size_t big_a_smem_g() {
  return sizeof(double2) * (SmemTw<KA, 4>::ENTRIES + kBigGroups * Geo<KA, 4>::SMEM);
}

// TM (KA = 12, field mode): the field kernel's N = 4096 machinery —
// per-thread twiddles in TMEM (TmemTw) and the one-pass offset between the
// two row-groups (FieldHook) — on pass A's 4096-point blocks.
template <int KA, bool INV, bool TM = false>
__global__ void __launch_bounds__(Geo<KA, 4>::T * kBigGroups, 1)
big_pass_a(int K, int mode, const double* __restrict__ pw_rev, long long pw_row0,
           const double2* __restrict__ ghat_rev, const double2* __restrict__ x,
           const double2* __restrict__ twst, long long row0, long long row1,
           double2* __restrict__ Y, const int* __restrict__ stopped,
           const int* __restrict__ pw_len) {
  using GA = Geo<KA, 4>;
  using TwA = SmemTw<KA, 4>;
  constexpr int BLK = 1 << KA, T = GA::T;
  static_assert(!TM || (KA == 12 && INV), "TMEM pass A: field blocks of 4096");
  extern __shared__ double2 smem[];
  if (stopped && *stopped) return;
  const long long N = 1LL << K;
  const long long nblk = N >> KA;
  const long long items = (row1 - row0) * nblk;
  __shared__ uint32_t tm_base;
  if constexpr (TM) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&tm_base))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  TwA::load(smem, twst);  // N-table stage twiddles S_b, b < KA
  if constexpr (TM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (TM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  using TwSrc = std::conditional_t<TM, TmemTw, TwA>;
  TwSrc tw;
  if constexpr (TM) {
    const int warp = threadIdx.x >> 5;
    tw.base = tm_base + ((uint32_t)((warp & 3) * 32) << 16) +
              (uint32_t)(((warp & 7) >> 2) * TmemTw::kSetCols);
    if (g == 0) {
      tw.template fill<KA, 4, true>(tid, TwA{smem});
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  } else {
    tw.sm = smem;
  }
  double2* buf = smem + TwA::ENTRIES + g * GA::SMEM;
  const GroupSync sync{1 + g, T};
  const int t0 = brev_bits(tid, GA::TB);
  const bool offset = TM && (long long)blockIdx.x * kBigGroups + 1 < items;
  bool first = true;
#ifndef AFD_PASSA_NO_BULK
  constexpr bool kBulkOut = TM;  // field mode (TM is only instantiated for it)
#else
  constexpr bool kBulkOut = false;
#endif
  bool bulk_pending = false;
  for (long long it = (long long)blockIdx.x * kBigGroups + g; it < items;
       it += (long long)gridDim.x * kBigGroups) {
    const long long rl = it / nblk;               // row within the batch
    const long long base = (it % nblk) * BLK;
    double2 v[GA::P];
    if (mode == 0) {
      // prologue y = powers * c[rev] (transform.py:198) straight from the
      // register-layout tables (coalesced over t)
      // r^l is exactly +0 from pw_len on (underflow): those entries are not
      // loaded (only radii <= 0.5 reach zero — larger ones stick at a
      // subnormal — so about half of the c2/c4 table), the product with the
      // spectrum still forms the same signed zeros
      const double* __restrict__ pr = pw_rev + (size_t)(row0 + rl - pw_row0) * N + base;
      const double2* __restrict__ gr = ghat_rev + base;
      const int L = pw_len[row0 + rl - pw_row0];
#pragma unroll
      for (int i = 0; i < GA::P; ++i) {
        const int l = brev_rt((int)(base + ((t0 << 4) | i)), K);  // natural index
        // a predicated load in PTX: the compiler must not turn it into an
        // unconditional load + select (the address is valid either way)
        double p = 0.0;
        asm volatile("{ .reg .pred q; setp.lt.s32 q, %1, %2; @q ld.global.nc.f64 %0, [%3]; }"
                     : "+d"(p)
                     : "r"(l), "r"(L), "l"(pr + i * T + tid));
        const double2 c = __ldg(gr + i * T + tid);
        v[i] = make_double2(p * c.x, p * c.y);
      }
    } else {
      // transform of one natural-order signal: gather x[rev(p)] via smem
      for (int q = tid; q < BLK; q += T) buf[GA::sw(q)] = x[brev_rt((int)(base + q), K)];
      sync();
#pragma unroll
      for (int i = 0; i < GA::P; ++i) v[i] = buf[GA::sw(GA::pos(0, t0, i))];
      sync();
    }
    if constexpr (kBulkOut) {
      // the previous item's bulk store has read the buffer out
      if (bulk_pending) {
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        sync();
        bulk_pending = false;
      }
    }
    if constexpr (TM) {
      if (offset && first && g == 1) asm volatile("bar.sync 3, %0;" ::"r"(2 * T) : "memory");
      const FieldHook hook{offset && first && g == 0, 2 * T, nullptr, false};
      fft_passes<KA, INV, 4>(v, tid, true, buf, tw, sync, hook);
      first = false;
    } else {
      fft_passes<KA, INV, 4>(v, tid, true, buf, tw, sync);
    }
    double2* __restrict__ y = Y + (size_t)rl * N + base;
    if constexpr (kBulkOut) {
      // field blocks: staged in natural order in the group's buffer and
      // written by one bulk copy (TMA) — off the load/store pipe the next
      // item's prologue loads need
#pragma unroll
      for (int i = 0; i < GA::P; ++i) buf[out_pos<KA, 4>(tid, i)] = v[i];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sync();
      if (tid == 0) {
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(y),
            "r"((unsigned)__cvta_generic_to_shared(buf)), "r"((unsigned)(sizeof(double2) * BLK))
            : "memory");
      }
      bulk_pending = true;
    } else {
#pragma unroll
      for (int i = 0; i < GA::P; ++i) y[out_pos<KA, 4>(tid, i)] = v[i];
      sync();  // buffer reuse by the next item
    }
  }
  if constexpr (kBulkOut) {
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if constexpr (TM) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base)
                   : "memory");
  }
}

// FieldHook plus: the previous item's bulk store must have read the group's
// buffer before the first exchange overwrites it — waited for after pass 0
// (not before it: the store is still draining when the prologue ends).
struct BulkWaitHook {
  FieldHook fh;
  bool pending, leader;
  GroupSync sync;
  __device__ __forceinline__ void before(int pass) const { fh.before(pass); }
  __device__ __forceinline__ void after(int pass) const {
    if (pass == 0 && pending) {
      if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      sync();
    }
    fh.after(pass);
  }
  __device__ __forceinline__ void exch(int pass) const { fh.exch(pass); }
};

// ---------------------------------------------------------------------------
// Field pass A for 4096-point blocks (N = 2^16, 2^20: KA = 12), block-major.
// The two row-groups of a CTA always work on the same block index of two
// rows (a "pair"), and each CTA walks a contiguous range of pairs in
// block-major order, so the block's 64 KiB of spectrum is loaded into tensor
// memory once per block change (a few per CTA and launch) instead of from L2
// for every item — the field kernel's spectrum-in-TMEM, with its TMEM
// twiddles, one-pass row-group offset and the bulk-stored outputs of
// big_pass_a.  Same butterflies, same bits.
// ---------------------------------------------------------------------------
// FAST (AFD_PLAN_FAST): pw_rev is the weight factor table fw (row stride
// 2^(K-12) + 256 + 16; fast_weight_kernel) and twst the (c, t) stage table.
// Register i of thread t in block blk holds natural index
//   l = rev_{K-12}(blk) + (t << (K-12)) + (rev4(i) << (K-4)),
// so its weight scale r^l = fw[rev(blk)] * fw[2^(K-12) + t] * fw[2^(K-12) + 256 + rev4(i)].
template <bool FAST = false>
__global__ void __launch_bounds__(Geo<12, 4>::T * kBigGroups, 1)
big_field_a(int K, const double* __restrict__ pw_rev, long long pw_row0,
            const double2* __restrict__ ghat_rev, const double2* __restrict__ twst,
            long long row0, long long row1, double2* __restrict__ Y,
            const int* __restrict__ stopped, const int* __restrict__ pw_len,
            int direct_out, const int* __restrict__ lim = nullptr) {
  constexpr int KA = 12;
  using GA = Geo<KA, 4>;
  using TwA = SmemTw<KA, 4>;
  constexpr int BLK = 1 << KA, T = GA::T, P = GA::P;
  extern __shared__ double2 smem[];
  if (stopped && *stopped) return;
  if (lim != nullptr) {  // pruned field: rows below *lim are done on chip (afd_pruned.cuh)
    const long long l = *lim;
    if (l > row0) row0 = l < row1 ? l : row1;
    if (row0 >= row1) return;
  }
  const long long N = 1LL << K;
  const int nblk = (int)(N >> KA);
  const int rows = (int)(row1 - row0);
  const int rpairs = (rows + 1) / 2;
  const long long pairs = (long long)nblk * rpairs;
  const long long p0 = pairs * blockIdx.x / gridDim.x, p1 = pairs * (blockIdx.x + 1) / gridDim.x;
  __shared__ uint32_t tm_base;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tm_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  TwA::load(smem, twst);  // N-table stage twiddles S_b, b < 12 (for the TMEM fill)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int g = threadIdx.x / T, tid = threadIdx.x % T;
  const int warp = threadIdx.x >> 5;
  std::conditional_t<FAST, TmemTwCT, TmemTw> tw;
  tw.base = tm_base + ((uint32_t)((warp & 3) * 32) << 16) +
            (uint32_t)(((warp & 7) >> 2) * TmemTw::kSetCols);
  // spectrum of the current block: 16 values per thread, shared by the two
  // groups (same thread index, same values), as in field_kernel
  const uint32_t gh_tm = tm_base + ((uint32_t)((warp & 3) * 32) << 16) +
                         (uint32_t)TmemTw::kGhCol + (uint32_t)(((warp & 7) >> 2) * (4 * P));
  const int kb = K - KA;                 // FAST: bits of the block index
  const int fws = (1 << kb) + 256 + 16;  // FAST: weight table row stride
  if (g == 0) {
    tw.template fill<KA, 4, !FAST>(tid, TwA{smem});
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  double2* buf = smem + TwA::ENTRIES + g * GA::SMEM;
  const GroupSync sync{1 + g, T};
  const int t0 = brev_bits(tid, GA::TB);
  int cur_blk = -1;
  bool first = true, bulk_pending = false;
  for (long long ip = p0; ip < p1; ++ip) {
    const int blk = (int)(ip / rpairs);
    const int rl = 2 * (int)(ip % rpairs) + g;  // row within the batch
    const bool live = rl < rows;               // odd row count: last pair half empty
    const int base = blk * BLK;
    if (blk != cur_blk) {
      // block change: both groups done with the old spectrum (and, the
      // first time, the twiddle fill visible), group 0 loads the new one
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (g == 0) {
        // all loads before the first TMEM store (a tcgen05.st is a memory
        // barrier to the compiler: loads after one are not hoisted)
        const double2* __restrict__ gr = ghat_rev + base;
        double2 gv[P];
#pragma unroll
        for (int i = 0; i < P; ++i) gv[i] = __ldg(gr + i * T + tid);
#pragma unroll
        for (int i = 0; i < P; ++i) tm_st4(gh_tm + 4 * i, gv[i]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      cur_blk = blk;
      first = true;  // re-establish the one-pass group offset
    }
    double2 v[P];
    if (live && FAST) {
      const double* __restrict__ fr = pw_rev + (size_t)(row0 + rl - pw_row0) * fws;
      const double a = __ldg(fr + brev_rt(blk, kb)) * __ldg(fr + (1 << kb) + tid);
      double w[P];
#pragma unroll
      for (int m = 0; m < P; ++m) w[m] = __ldg(fr + (1 << kb) + 256 + m);
#pragma unroll
      for (int i = 0; i < P; ++i) w[i] = a * w[i];  // now indexed by rev4(i) below
      double wi[P];
#pragma unroll
      for (int i = 0; i < P; ++i) wi[i] = w[brev_bits(i, 4)];
#pragma unroll
      for (int i0 = 0; i0 < P; i0 += 4) {
        uint32_t r[16];
        tm_ld<16>(gh_tm + 4 * i0, r);
        tm_wait_ld();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[i0 + j] = make_double2(__hiloint2double(r[4 * j + 1], r[4 * j]),
                                   __hiloint2double(r[4 * j + 3], r[4 * j + 2]));
      }
      fast_prologue(v, wi);
    } else if (live) {
      // prologue y = powers * c[rev] (transform.py:198); r^l from the
      // register-layout table (predicated past the underflow, see big_pass_a)
      const double* __restrict__ pr = pw_rev + (size_t)(row0 + rl - pw_row0) * N + base;
      const int L = pw_len[row0 + rl - pw_row0];
      // all sixteen HBM loads in flight before the first use (the volatile
      // loads keep program order, so interleaving them with the TMEM reads
      // below serialised four round trips)
      double pv[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int l = brev_rt(base + ((t0 << 4) | i), K);  // natural index
        pv[i] = 0.0;
        asm volatile("{ .reg .pred q; setp.lt.s32 q, %1, %2; @q ld.global.nc.f64 %0, [%3]; }"
                     : "+d"(pv[i])
                     : "r"(l), "r"(L), "l"(pr + i * T + tid));
      }
#pragma unroll
      for (int i0 = 0; i0 < P; i0 += 4) {
        uint32_t r[16];
        tm_ld<16>(gh_tm + 4 * i0, r);
        tm_wait_ld();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = i0 + j;
          const double p = pv[i];
          const double2 c = make_double2(__hiloint2double(r[4 * j + 1], r[4 * j]),
                                         __hiloint2double(r[4 * j + 3], r[4 * j + 2]));
          v[i] = make_double2(p * c.x, p * c.y);
        }
      }
    }
    if (first && g == 1) asm volatile("bar.sync 3, %0;" ::"r"(2 * T) : "memory");
    if (live) {
      const BulkWaitHook hook{{first && g == 0, 2 * T, nullptr, false}, bulk_pending, tid == 0,
                              sync};
      fft_passes<KA, true, 4>(v, tid, true, buf, tw, sync, hook);
      bulk_pending = false;
      double2* __restrict__ y = Y + (size_t)rl * N + base;
      if (direct_out) {
        // straight from registers (lanes hold consecutive positions: every
        // store is a coalesced 512-B warp write), no shared-memory staging
#pragma unroll
        for (int i = 0; i < P; ++i) __stcs(y + out_pos<KA, 4>(tid, i), v[i]);
        first = false;
        continue;
      }
#pragma unroll
      for (int i = 0; i < P; ++i) buf[out_pos<KA, 4>(tid, i)] = v[i];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sync();
      if (tid == 0) {
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(y),
            "r"((unsigned)__cvta_generic_to_shared(buf)), "r"((unsigned)(sizeof(double2) * BLK))
            : "memory");
      }
      bulk_pending = true;
    } else {
      if (first && g == 0) asm volatile("bar.arrive 3, %0;" ::"r"(2 * T) : "memory");  // (never)
      if (bulk_pending) {  // a dead item: drain the pending store here
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        sync();
        bulk_pending = false;
      }
    }
    first = false;
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm_base)
                 : "memory");
}

// ---------------------------------------------------------------------------
// Column pass over stage bits [b0, b0+4).  Thread = column q (bits b0..b0+3
// of q clear); blockIdx.y = row within the batch.
//   out_mode 0: write back to Y in place
//   out_mode 1: field epilogue: scale, |.|^2, running first maximum -> cand
//   out_mode 2: field epilogue, materialise rows into fout[row - row0][j]
//   out_mode 3: transform output in natural order fout[j] (optionally / N)
//   out_mode 4: field spectrum: position rev(j) in pass-A layout (ghat_perm)
// ---------------------------------------------------------------------------
// MODE >= 0 fixes out_mode at compile time (the field pass, MODE = 1: fewer
// live registers than the all-modes kernel, no spills); MODE = -1 dispatches
// on out_mode at run time.
// FAST (field modes 0-2 only): (c, t) twiddles, no scale (see col_tma_kernel).
template <bool INV, int MODE = -1, bool FAST = false>
__global__ void __launch_bounds__(kColThreads, 2)
big_pass_col(int K, int ka, int b0, int out_mode_rt, int scale_n, double2* __restrict__ Y,
             const double2* __restrict__ twst, const double* __restrict__ scales,
             long long row0, long long row1, Cand* __restrict__ cand,
             double2* __restrict__ fout, const int* __restrict__ stopped) {
  const int out_mode = MODE >= 0 ? MODE : out_mode_rt;
  if (stopped && *stopped) return;
  const long long N = 1LL << K;
  const long long row = row0 + blockIdx.y;
  const long long x = (long long)blockIdx.x * kColThreads + threadIdx.x;  // column index
  Cand best;
  best.mag = -1.0;
  best.flat = 0x7fffffffffffffffLL;
  best.re = best.im = 0.0;
  if (row < row1 && x < (N >> 4)) {
    const long long lowmask = (1LL << b0) - 1;
    const long long q = (x & lowmask) | ((x >> b0) << (b0 + 4));
    double2* __restrict__ y = Y + (size_t)blockIdx.y * N;
    double2 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = y[q + ((long long)u << b0)];
    const long long qlow = q & lowmask;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int b = b0 + e;
      // per-stage table S_b[k] = w[k << (K-1-b)]: lanes read consecutive entries
      const double2* __restrict__ sb = twst + ((1LL << b) - 1);
#pragma unroll
      for (int kk = 0; kk < (1 << e); ++kk) {
        double2 w = __ldg(sb + qlow + ((long long)kk << b0));
        if (INV && !FAST) w.y = -w.y;
#pragma unroll
        for (int h = 0; h < (16 >> (e + 1)); ++h) {
          const int i = kk | (h << (e + 1));
          bfly_any<FAST>(v[i], v[i | (1 << e)], w);
        }
      }
    }
    if (out_mode == 0) {
#pragma unroll
      for (int u = 0; u < 16; ++u) y[q + ((long long)u << b0)] = v[u];
    } else if (out_mode == 1 || out_mode == 2) {
      const double sc = FAST ? 1.0 : __ldg(scales + row);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const long long j = q + ((long long)u << b0);
        const double2 f = FAST ? v[u] : make_double2(v[u].x * sc, v[u].y * sc);  // transform.py:200
        if (out_mode == 2) {
          fout[(size_t)(row - row0) * N + j] = f;
        } else {
          const double mg = FAST ? fast_mag2(f) : np_mag2(f);
          if (mg > best.mag) {  // j increases with u: first maximum
            best.mag = mg;
            best.flat = row * N + j;
            best.re = f.x;
            best.im = f.y;
          }
        }
      }
    } else {
      const double2 dn = make_double2((double)N, 0.0);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const long long j = q + ((long long)u << b0);
        double2 o = v[u];
        if (scale_n) o = np_cdiv(o, dn);  // `y /= n`, transform.py:133
        if (out_mode == 3) fout[j] = o;
        else fout[perm_of_pos(brev_rt((int)j, K), ka)] = o;
      }
    }
  }
  if (out_mode != 1) return;
  // merge this CTA's first maximum into its slot (slots persist over the
  // row batches of one step; the (mag, flat) order makes merging order-free)
  __shared__ Cand red[32];
  best = warp_argmax(best);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = best;
  __syncthreads();
  if (wid == 0) {
    Cand c = lane < (kColThreads >> 5) ? red[lane] : best;
    c = warp_argmax(c);
    if (lane == 0) {
      Cand& slot = cand[(size_t)blockIdx.y * gridDim.x + blockIdx.x];
      Cand o = slot;
      cand_merge(o, c);
      slot = o;
    }
  }
}

// ---------------------------------------------------------------------------
// Two column passes in one: stage bits [b0, b0+8) (N = 2^17..2^20: everything
// after pass A).  A column is 256 positions q + 2^b0 u, u < 256, held by 16
// threads; stages b0..b0+3 (u bits 0-3) in layout A (thread h holds
// u = 16h + i), a transpose through shared memory, stages b0+4..b0+7 (u bits
// 4-7) in layout B (thread h holds u = h + 16i).  One read of the row batch
// intermediate instead of read + write + read (HBM-bound at N = 2^20).
// CTA = 16 consecutive columns; slots as big_pass_col (N/4096 CTAs per row).
//   MODE 1: field epilogue -> cand;  MODE 0: write back to Y in place.
// ---------------------------------------------------------------------------
constexpr int kCol8Pad = 257;  // smem slots per column (256 + 1: conflict-free)

template <int MODE>
__global__ void __launch_bounds__(256, 2)
big_pass_col8(int K, int b0, double2* __restrict__ Y, const double2* __restrict__ twst,
              const double* __restrict__ scales, long long row0, long long row1,
              Cand* __restrict__ cand, const int* __restrict__ stopped) {
  extern __shared__ double2 col_sm[];  // [16][kCol8Pad]
  if (stopped && *stopped) return;
  const long long N = 1LL << K;
  const long long row = row0 + blockIdx.y;
  const int c = threadIdx.x & 15, h = threadIdx.x >> 4;
  const long long x = (long long)blockIdx.x * 16 + c;  // column
  const long long lowmask = (1LL << b0) - 1;
  const long long q = (x & lowmask) | ((x >> b0) << (b0 + 8));
  const long long qlow = q & lowmask;
  double2* __restrict__ y = Y + (size_t)blockIdx.y * N;
  double2* sm = col_sm + c * kCol8Pad;
  Cand best;
  best.mag = -1.0;
  best.flat = 0x7fffffffffffffffLL;
  best.re = best.im = 0.0;
  const bool live = row < row1;
  double2 v[16];
  if (live) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[q + ((long long)(16 * h + i) << b0)];
    // stages b0..b0+3: u mod 2^e = i mod 2^e
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double2* __restrict__ sb = twst + ((1LL << (b0 + e)) - 1);  // S_b[k] = w[k << (K-1-b)]
#pragma unroll
      for (int kk = 0; kk < (1 << e); ++kk) {
        double2 w = __ldg(sb + qlow + ((long long)kk << b0));
        w.y = -w.y;  // np.conj(w), transform.py:199
#pragma unroll
        for (int hh = 0; hh < (16 >> (e + 1)); ++hh) {
          const int i = kk | (hh << (e + 1));
          bfly(v[i], v[i | (1 << e)], w);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) sm[16 * h + i] = v[i];
  }
  __syncthreads();
  if (live) {
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = sm[h + 16 * i];
    // stages b0+4..b0+7: u mod 2^e = h + 16 (i mod 2^(e-4))
#pragma unroll
    for (int e = 4; e < 8; ++e) {
      const double2* __restrict__ sb = twst + ((1LL << (b0 + e)) - 1);
      const int ib = e - 4;
#pragma unroll
      for (int kk = 0; kk < (1 << ib); ++kk) {
        double2 w = __ldg(sb + qlow + ((long long)(h + 16 * kk) << b0));
        w.y = -w.y;
#pragma unroll
        for (int hh = 0; hh < (16 >> (ib + 1)); ++hh) {
          const int i = kk | (hh << (ib + 1));
          bfly(v[i], v[i | (1 << ib)], w);
        }
      }
    }
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) y[q + ((long long)(h + 16 * i) << b0)] = v[i];
    } else {
      const double sc = __ldg(scales + row);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const long long j = q + ((long long)(h + 16 * i) << b0);
        const double2 f = make_double2(v[i].x * sc, v[i].y * sc);  // transform.py:200
        const double mg = np_mag2(f);                              // core.py:298
        if (mg > best.mag) {  // j increases with i: first maximum
          best.mag = mg;
          best.flat = row * N + j;
          best.re = f.x;
          best.im = f.y;
        }
      }
    }
  }
  if (MODE == 0) return;
  __shared__ Cand red[8];
  best = warp_argmax(best);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = best;
  __syncthreads();
  if (wid == 0) {
    Cand cc = lane < 8 ? red[lane] : best;
    cc = warp_argmax(cc);
    if (lane == 0) {
      Cand& slot = cand[(size_t)blockIdx.y * gridDim.x + blockIdx.x];
      Cand o = slot;
      cand_merge(o, cc);
      slot = o;
    }
  }
}

__global__ void cand_init_kernel(Cand* c, int n, double* c2 = nullptr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    c[i].mag = -1.0;
    c[i].flat = 0x7fffffffffffffffLL;
    c[i].re = c[i].im = 0.0;
    if (c2 != nullptr) c2[i] = -1.0;
  }
}

// ---------------------------------------------------------------------------
// Per-step bookkeeping for one signal, large N.
// ---------------------------------------------------------------------------
struct BigSel {
  long long s, j;
  double radius;
  double2 a, coeff;
  int valid;
  float margin;  // top-2 relative margin (fast engine) or NaN
};

// numpy pairwise node sums over aligned kNodeLen slices:
// kind 0: |x|^2 of a complex signal, kind 1: complex sum of the signal
// (one CTA per slice, 256 threads).
__global__ void __launch_bounds__(256)
node_sums_kernel(int kind, const double2* __restrict__ x, double* __restrict__ nodes) {
  __shared__ double buf[kNodeLen * 2];
  __shared__ double scratch[2 * (kNodeLen / 8 + 16)];
  const double2* xs = x + (size_t)blockIdx.x * kNodeLen;
  if (kind == 0) {
    for (int i = threadIdx.x; i < kNodeLen; i += blockDim.x) buf[i] = np_mag2(xs[i]);
    __syncthreads();
    const double s = pairwise_sum_block(buf, kNodeLen, scratch, PlainIdx());
    if (threadIdx.x == 0) nodes[blockIdx.x] = s;
  } else {
    double2* b2 = reinterpret_cast<double2*>(buf);
    for (int i = threadIdx.x; i < kNodeLen; i += blockDim.x) b2[i] = xs[i];
    __syncthreads();
    const double2 s = cpairwise_sum_block(b2, kNodeLen, scratch, PlainIdx());
    if (threadIdx.x == 0) {
      nodes[2 * blockIdx.x] = s.x;
      nodes[2 * blockIdx.x + 1] = s.y;
    }
  }
}

// Left+right tree over `n` (power of two) node values held in shared memory.
__device__ double tree_sum(double* v, int n) {
  for (int w = n; w > 1; w >>= 1) {
    for (int b = threadIdx.x; b < w / 2; b += blockDim.x) v[b] = v[2 * b] + v[2 * b + 1];
    __syncthreads();
  }
  return v[0];
}

// Select: candidates -> pole + coefficient (or the dc_first mean atom).
__global__ void __launch_bounds__(256)
big_select_kernel(int k, int dc_first, int K, const Cand* __restrict__ cand, int ncand,
                  const double* __restrict__ nodes, int nnodes,
                  const double* __restrict__ radii, const double2* __restrict__ circle,
                  const State* __restrict__ state, BigSel* __restrict__ sel,
                  const double* __restrict__ cand2 = nullptr) {
  __shared__ double re[kMaxNodes], im[kMaxNodes];
  if (state->stopped) return;
  const long long N = 1LL << K;
  BigSel out;
  out.valid = 1;
  out.margin = __int_as_float(0x7fc00000);
  if (k == 0 && dc_first) {
    for (int i = threadIdx.x; i < nnodes; i += blockDim.x) {
      re[i] = nodes[2 * i];
      im[i] = nodes[2 * i + 1];
    }
    __syncthreads();
    const double sr = tree_sum(re, nnodes);
    const double si = tree_sum(im, nnodes);
    out.s = out.j = 0;
    out.radius = 0.0;
    out.a = make_double2(0.0, 0.0);
    out.coeff = np_cdiv(make_double2(sr, si), make_double2((double)N, 0.0));  // core.py:375
  } else {
    Cand b;
    b.mag = -1.0;
    b.flat = 0x7fffffffffffffffLL;
    b.re = b.im = 0.0;
    for (int i = threadIdx.x; i < ncand; i += blockDim.x) cand_merge(b, cand[i]);
    __shared__ Cand red[32];
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
    if (cand2 != nullptr) {  // runner-up of the step (fast engine)
      double r = -1.0;
      for (int i = threadIdx.x; i < ncand; i += blockDim.x) {
        r = fmax(r, cand2[i]);
        if (cand[i].flat != b.flat) r = fmax(r, cand[i].mag);
      }
      r = block_max(r);
      out.margin = top2_margin(b.mag, r);
    }
    out.s = b.flat / N;
    out.j = b.flat % N;
    out.radius = radii[out.s];
    const double2 zj = circle[out.j];
    out.a = make_double2(out.radius * zj.x, out.radius * zj.y);  // core.py:163-167
    out.coeff = make_double2(b.re, b.im);
  }
  if (threadIdx.x == 0) *sel = out;
}

// Update (core.py:303-314; numpy's temporary elision applies for N >= 16384)
// or, at init (sel == null), copy g0.  Writes the remainder and the |.|^2
// node sums of each kNodeLen slice.
__global__ void __launch_bounds__(256)
big_update_kernel(int K, const BigSel* __restrict__ sel, const double2* __restrict__ g0,
                  double2* __restrict__ rem, const double2* __restrict__ circle,
                  const State* __restrict__ state, double* __restrict__ nodes,
                  int* __restrict__ amb_out, const double* __restrict__ pow2) {
  __shared__ double buf[kNodeLen];
  __shared__ double scratch[2 * (kNodeLen / 8 + 16)];
  if (sel && state->stopped) return;
  const long long N = 1LL << K;
  const bool elide = (size_t)N * 16 >= 256 * 1024;
  const long long m0 = (long long)blockIdx.x * kNodeLen;
  int amb = 0;
  if (!sel) {
    for (int i = threadIdx.x; i < kNodeLen; i += blockDim.x) {
      const double2 v = g0[m0 + i];
      rem[m0 + i] = v;
      buf[i] = np_mag2(v);
    }
  } else {
    const BigSel s = *sel;
    const double kn = kernel_norm_grid(s.a, s.radius, pow2 ? pow2 + (size_t)s.s * kPowRow : nullptr,
                                       &amb);
    const double2 sc = make_double2(kn, 0.0);
    for (int i = threadIdx.x; i < kNodeLen; i += blockDim.x) {
      const long long m = m0 + i;
      const double2 z = circle[m];
      const double2 d = one_minus_conja_z(s.a, z);
      const double2 e = np_cdiv(sc, d);
      const double2 ce = elide ? np_cmul(e, s.coeff) : np_cmul(s.coeff, e);
      const double2 g = rem[m];
      const double2 stp = make_double2(g.x - ce.x, g.y - ce.y);
      const double2 num = elide ? np_cmul(d, stp) : np_cmul(stp, d);
      const double2 out = np_cdiv(num, make_double2(z.x - s.a.x, z.y - s.a.y));
      rem[m] = out;
      buf[i] = np_mag2(out);
    }
  }
  __syncthreads();
  const double ns = pairwise_sum_block(buf, kNodeLen, scratch, PlainIdx());
  if (threadIdx.x == 0) {
    nodes[blockIdx.x] = ns;
    if (blockIdx.x == 0 && amb_out) *amb_out = amb;
  }
}

// Energy + record + stop rules (k < 0: initial energy).
__global__ void __launch_bounds__(256)
big_finalize_kernel(int k, int K, int max_terms, double threshold, const double* __restrict__ nodes,
                    int nnodes, const BigSel* __restrict__ sel, const int* __restrict__ amb,
                    State* __restrict__ state, Step* __restrict__ steps) {
  __shared__ double v[kMaxNodes];
  if (k >= 0 && state->stopped) return;
  const double N = (double)(1LL << K);
  for (int i = threadIdx.x; i < nnodes; i += blockDim.x) v[i] = nodes[i];
  __syncthreads();
  const double energy = tree_sum(v, nnodes) / N;
  if (threadIdx.x != 0) return;
  if (k < 0) {
    state->initial = energy;
    state->nsteps = 0;
    state->flags = 0;
    state->stopped = energy == 0.0 ? 1 : 0;  // core.py:366-368
    return;
  }
  const BigSel s = *sel;
  Step rec;
  rec.s = s.s;
  rec.j = s.j;
  rec.radius = s.radius;
  rec.a_re = s.a.x;
  rec.a_im = s.a.y;
  rec.c_re = s.coeff.x;
  rec.c_im = s.coeff.y;
  rec.residual = energy;
  rec.flags = *amb ? kStepPowAmbiguous : 0;
  rec.margin = s.margin;
  steps[k] = rec;
  state->nsteps = k + 1;
  state->flags |= rec.flags;
  int stop = 0;
  if (threshold > 0.0 && energy <= threshold * state->initial) stop = 1;  // core.py:386-387
  if (energy == 0.0) stop = 1;                                            // core.py:388-389
  if (k + 1 >= max_terms) stop = 1;
  state->stopped = stop;
}

// In-place bit reversal of rows of length 2^K (K >= 10), used to turn the
// natural-order r^l table into pw_rev.  Index l = (hi, mid, lo) with 5, K-10
// and 5 bits; rev(l) = (rev5(lo), rev(mid), rev5(hi)), so the 32x32 tile of
// (hi, lo) at `mid` and the tile at rev(mid) swap through shared memory with
// coalesced loads and stores.  blockIdx.x = mid, blockIdx.y = row.
__global__ void __launch_bounds__(1024) bitrev_rows_kernel(double* __restrict__ pw, int K) {
  __shared__ double A[32][33], B[32][33];
  const int mb = K - 10;
  const int mid = blockIdx.x;
  const int mid2 = mb > 0 ? brev_rt(mid, mb) : 0;
  if (mid2 < mid) return;
  double* row = pw + ((size_t)blockIdx.y << K);
  const int hi = threadIdx.y, lo = threadIdx.x;
  const size_t la = ((size_t)hi << (K - 5)) | ((size_t)mid << 5) | lo;
  const size_t lb = ((size_t)hi << (K - 5)) | ((size_t)mid2 << 5) | lo;
  A[hi][lo] = row[la];
  B[hi][lo] = row[lb];
  __syncthreads();
  const int rh = brev_rt(hi, 5), rl = brev_rt(lo, 5);
  // element (h, m, l) moves to (rev5(l), rev(m), rev5(h))
  row[lb] = A[rl][rh];
  if (mid2 != mid) row[la] = B[rl][rh];
}

// natural spectrum -> field input order: dst[perm(p)] = src[rev(p)]
__global__ void bitrev_copy_kernel(int K, int ka, const double2* __restrict__ src,
                                   double2* __restrict__ dst) {
  const long long N = 1LL << K;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N;
       p += (long long)gridDim.x * blockDim.x)
    dst[perm_of_pos(p, ka)] = src[brev_rt((int)p, K)];
}

// In-place reorder of each 2^ka block of position-ordered rows into the
// pass-A register layout (pw_rev -> pw_perm).  blockIdx.x = block, y = row.
__global__ void __launch_bounds__(256) perm_blocks_kernel(double* __restrict__ pw, int K, int ka) {
  extern __shared__ double blk[];
  const int BLK = 1 << ka, T = 1 << (ka - 4);
  double* row = pw + ((size_t)blockIdx.y << K) + ((size_t)blockIdx.x << ka);
  for (int q = threadIdx.x; q < BLK; q += blockDim.x) blk[q] = row[q];
  __syncthreads();
  for (int e = threadIdx.x; e < BLK; e += blockDim.x) {
    const int i = e / T, tp = e % T;
    row[e] = blk[(brev_rt(tp, ka - 4) << 4) | i];
  }
}

// natural-order spectrum mask of the analytic projection (core.py:229-230)
__global__ void analytic_mask_kernel(int K, double2* __restrict__ s) {
  const long long N = 1LL << K, half = N / 2;
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < N;
       m += (long long)gridDim.x * blockDim.x) {
    if (m >= 1 && m < half) s[m] = make_double2(s[m].x * 2.0, s[m].y * 2.0);
    else if (m > half) s[m] = make_double2(0.0, 0.0);
  }
}

}  // namespace afd
