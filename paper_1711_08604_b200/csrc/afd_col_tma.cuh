// afd_col_tma.cuh — the field's last column stages for large N as a
// persistent, TMA-pipelined kernel (replaces big_pass_col<..,1> and
// big_pass_col8<1> in the field, transform.py:199-200 + core.py:298-299).
//
// The column pass streams the row-batch intermediate from HBM once.  The
// one-tile-per-CTA kernels issue their 16 loads per thread, then compute,
// with two CTAs per SM: the SM alternates between waiting and computing
// (c4: 3.0 TB/s, FP64 39% busy).  Here one CTA per SM walks a contiguous
// range of tiles; while it computes tile n, tile n+1 is already in flight
// into shared memory by bulk copies (cp.async.bulk, completion on an
// mbarrier), so HBM streams continuously.
//
// Tile = 4096 evaluations of one row.  KC = 8 (the last eight stages,
// N = 2^17..2^20): 16 columns q0..q0+15 x 256 positions q + (u << b0), landed
// as smem[u][c] by one tensor copy (a 3-d tensor map over the row batch:
// 256-B inner box x 256 positions x 1 row); thread (c, h) runs stages b0..b0+3
// on u = 16h + i, writes back in place, and stages b0+4..b0+7 on u = h + 16i
// (the transpose is the change of index, conflict-free both ways).  KC = 4
// (N = 2^14..2^16): 256 columns x 16 positions (16 copies of 4 KiB), one
// column per thread.  Tiles run column-chunk-major, so a CTA's tiles share
// their columns and the stage twiddles (they depend on the column only) stay
// in shared memory, conjugated once.  Butterflies, scale and |.|^2 are the
// reference's own operations, so the field and its first maximum are
// bit-identical to the two-kernel form.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "afd_big.cuh"

namespace afd {

// GROUPS = 2: two 256-thread groups per CTA take alternate tiles from a
// ring of three stages (tile n: group n & 1, stage n % 3), so 16 warps
// compute while a tile is in flight.  The one-group form keeps 8 warps per
// SM, and its column stages were latency-bound (FP64 pipe ~42% busy, 2
// warps per scheduler) rather than HBM-bound.
template <int KC, int GROUPS = 1>
struct ColTma {
  static constexpr int COLS = KC == 8 ? 16 : 256;     // columns per tile
  static constexpr int U = 1 << KC;                    // positions per column
  static constexpr int TILE = COLS * U;                // double2 per tile (4096)
  static constexpr int STAGES = GROUPS == 2 ? 3 : 2;
  static constexpr int THREADS = 256 * GROUPS;
  // twiddles live in tensor memory, per thread: 15 slots per 4-stage group
  // (slot 2^e - 1 + kk), 4 words each; one column set per pair of warps
  // sharing a lane quadrant (2 sets per group)
  static constexpr int NSLOT = KC == 8 ? 30 : 15;
  static constexpr int SET_COLS = 4 * NSLOT;                       // 120 / 60
  static constexpr unsigned TM_COLS =
      GROUPS == 2 ? (KC == 8 ? 512 : 256) : (KC == 8 ? 256 : 128);  // >= sets, power of 2
  static constexpr size_t SMEM = sizeof(double2) * (STAGES * TILE);
};

__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, unsigned bytes,
                                         unsigned long long* mbar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const unsigned m = (unsigned)__cvta_generic_to_shared(mbar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(d), "l"(gsrc), "r"(bytes), "r"(m)
      : "memory");
}

// FAST (AFD_PLAN_FAST): twst is the (c, t) table (already conjugated), the
// butterflies are bfly_ct and the scale is already in pass A's weights.
// Four radix-2 stages on the thread's 16 registers (stage e pairs bit e)
// with the twiddles of slots SLOT0 + 2^e - 1 + kk from tensor memory: one
// tcgen05.ld per stage (a separate data path from the shared-memory traffic
// of the tile and the transpose).
template <bool FAST, int SLOT0, int E = 0>
__device__ __forceinline__ void col_stages4(double2 (&v)[16], uint32_t twm) {
  if constexpr (E < 4) {
    uint32_t r[4 << E];
    tm_ld<(4 << E)>(twm + 4 * (SLOT0 + (1 << E) - 1), r);
    tm_wait_ld();
#pragma unroll
    for (int kk = 0; kk < (1 << E); ++kk) {
      const double2 w = make_double2(__hiloint2double(r[4 * kk + 1], r[4 * kk]),
                                     __hiloint2double(r[4 * kk + 3], r[4 * kk + 2]));
#pragma unroll
      for (int hh = 0; hh < (16 >> (E + 1)); ++hh) {
        const int i = kk | (hh << (E + 1));
        bfly_any<FAST>(v[i], v[i | (1 << E)], w);
      }
    }
    col_stages4<FAST, SLOT0, E + 1>(v, twm);
  }
}

template <int KC, bool FAST = false, int GROUPS = 1, bool MARG = false>
__global__ void __launch_bounds__(256 * GROUPS, 1)
col_tma_kernel(int K, int b0, const double2* __restrict__ Y, const double2* __restrict__ twst,
               const double* __restrict__ scales, long long row0, long long row1,
               Cand* __restrict__ cand, const int* __restrict__ stopped,
               const int* __restrict__ lim, double* __restrict__ cand2,
               const __grid_constant__ CUtensorMap ymap) {
  using C = ColTma<KC, GROUPS>;
  constexpr int COLS = C::COLS, U = C::U, TILE = C::TILE;
  extern __shared__ __align__(128) double2 csm[];
  __shared__ __align__(8) unsigned long long full[C::STAGES];
  // GROUPS = 2: rel[s] completes a phase when the group that consumed a
  // tile of stage s has issued the stage's next copy.  A group waits on it
  // before its full[s] wait, because the other group may still be on the
  // stage's previous tile (a parity wait alone would alias to that phase).
  __shared__ __align__(8) unsigned long long rel[C::STAGES];
  if (stopped && *stopped) return;
  if (lim != nullptr) {  // pruned field: the rows below *lim were done on chip
    const long long l = *lim;
    if (l > row0) row0 = l < row1 ? l : row1;
    if (row0 >= row1) return;
  }
  __shared__ uint32_t tm_base_s;
  const long long N = 1LL << K;
  const int rows = (int)(row1 - row0);
  const int chunks = (1 << b0) / COLS;
  const long long tiles = (long long)rows * chunks;
  // contiguous tile range of this CTA, tile = chunk * rows + row
  const long long t0 = tiles * blockIdx.x / gridDim.x;
  const long long t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  const int ntile = (int)(t1 - t0);
  const int lane = threadIdx.x & 31;
  const int grp = GROUPS == 2 ? (int)(threadIdx.x >> 8) : 0;
  const int tid = threadIdx.x & 255;  // thread within its group
  // group-local barrier (named barrier 1 + group; the whole CTA if one group)
  auto gsync = [&]() {
    if constexpr (GROUPS == 2) asm volatile("bar.sync %0, 256;" ::"r"(1 + grp) : "memory");
    else __syncthreads();
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&rel[s], 1);
    }
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&tm_base_s)),
                 "r"(C::TM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this thread's twiddle cells: its lane of the warp's quadrant, its set
  const uint32_t twm = tm_base_s + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16) +
                       (uint32_t)((threadIdx.x >> 7) * C::SET_COLS);
  // one warp issues the copies of local tile n into stage n % STAGES
  auto issue = [&](int n) {
    const long long t = t0 + n;
    const int chunk = (int)(t / rows), row = (int)(t % rows);
    const double2* src = Y + (size_t)row * N + (size_t)chunk * COLS;
    double2* dst = csm + (n % C::STAGES) * TILE;
    unsigned long long* mb = &full[n % C::STAGES];
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(mb)),
                   "r"((unsigned)(sizeof(double2) * TILE))
                   : "memory");
    __syncwarp();
    if constexpr (KC == 8) {
      // box {32 doubles, 256 positions, 1 row} at (2 q0, 0, row)
      if (lane == 0)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
            "l"(reinterpret_cast<unsigned long long>(&ymap)), "r"(2 * chunk * COLS), "r"(0),
            "r"(row), "r"((unsigned)__cvta_generic_to_shared(mb))
            : "memory");
    } else {
      for (int u = lane; u < U; u += 32)
        bulk_g2s(dst + u * COLS, src + ((size_t)u << b0), sizeof(double2) * COLS, mb);
    }
  };
  if (threadIdx.x < 32) {
    for (int n = 0; n < C::STAGES && n < ntile; ++n) issue(n);
  }

  Cand best;
  best.mag = -1.0;
  best.flat = 0x7fffffffffffffffLL;
  best.re = best.im = 0.0;
  // runner-up slots (fast engine): the screen passes every value above the
  // thread's runner-up, which may become either of its top two
  constexpr bool track2 = FAST && MARG;
  [[maybe_unused]] double sec = -1.0;
  int tw_chunk = -1;
  const int c = KC == 8 ? (tid & 15) : tid;
  const int h = KC == 8 ? (tid >> 4) : 0;
  for (int n = grp; n < ntile; n += GROUPS) {
    const long long t = t0 + n;
    const int chunk = (int)(t / rows), rl = (int)(t % rows);
    const long long row = row0 + rl;
    const int q0 = chunk * COLS;
    if (chunk != tw_chunk) {
      // this thread's stage twiddles for the chunk's column q0 + c, straight
      // from the stage tables into its tensor-memory cells (no other thread
      // reads them: no barrier), conjugated (transform.py:199) unless FAST
      // (already the (c, t) form): S_b[q + (k << b0)], b = b0 + e
#pragma unroll
      for (int e = 0; e < 4; ++e) {
#pragma unroll
        for (int kk = 0; kk < (1 << e); ++kk) {
          double2 w = __ldg(twst + ((1LL << (b0 + e)) - 1) + q0 + c + ((long long)kk << b0));
          if (!FAST) w.y = -w.y;
          tm_st4(twm + 4 * ((1 << e) - 1 + kk), w);
        }
      }
      if constexpr (KC == 8) {
#pragma unroll
        for (int ib = 0; ib < 4; ++ib) {
#pragma unroll
          for (int kk = 0; kk < (1 << ib); ++kk) {
            double2 w = __ldg(twst + ((1LL << (b0 + 4 + ib)) - 1) + q0 + c +
                              ((long long)(h + 16 * kk) << b0));
            if (!FAST) w.y = -w.y;
            tm_st4(twm + 4 * (15 + (1 << ib) - 1 + kk), w);
          }
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tw_chunk = chunk;
    }
    const int s = n % C::STAGES;
    double2* tile = csm + s * TILE;
    if (GROUPS == 2 && n >= C::STAGES)
      mbar_wait(&rel[s], (unsigned)(((n - C::STAGES) / C::STAGES) & 1));
    mbar_wait(&full[s], (unsigned)((n / C::STAGES) & 1));
    const double sc = FAST ? 1.0 : __ldg(scales + row);
    const int q = q0 + c;
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = tile[(16 * h + i) * COLS + c];
    col_stages4<FAST, 0>(v, twm);
    if constexpr (KC == 8) {
#pragma unroll
      for (int i = 0; i < 16; ++i) tile[(16 * h + i) * COLS + c] = v[i];
      gsync();
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = tile[(h + 16 * i) * COLS + c];
      col_stages4<FAST, 15>(v, twm);
    }
    // this tile's stage is free once every thread has read it: refill it
    // with tile n + STAGES (generic-proxy writes above precede the async
    // proxy's overwrite)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    gsync();
    if (tid < 32 && n + C::STAGES < ntile) {
      issue(n + C::STAGES);
      if (GROUPS == 2 && lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&rel[s]))
                     : "memory");
    }
    // FAST: screen the tile with one predicate-accumulating compare per
    // point; the (rare) tile holding a candidate at least as large as the
    // thread's best runs the full first-maximum update
    unsigned up = 1;
    if constexpr (FAST) {
      up = 0;
#pragma unroll
      for (int i0 = 0; i0 < 16; i0 += 4) {
        double mg[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) mg[i] = fast_mag2(v[i0 + i]);
        up = any_ge4(up, mg, track2 ? sec : best.mag);
      }
    }
    if (!FAST || __builtin_expect(up != 0, 0)) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const long long j = q + ((long long)(KC == 8 ? h + 16 * i : i) << b0);
        const double2 f = FAST ? v[i] : make_double2(v[i].x * sc, v[i].y * sc);  // transform.py:200
        const double mg = FAST ? fast_mag2(f) : np_mag2(f);                     // core.py:298
        const long long flat = row * N + j;
        if (mg >= best.mag && cand_better(mg, flat, best.mag, best.flat)) {
          if constexpr (track2) sec = fmax(sec, best.mag);
          best.mag = mg;
          best.flat = flat;
          best.re = f.x;
          best.im = f.y;
        } else if constexpr (track2) {
          sec = fmax(sec, mg);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base_s),
                 "r"(C::TM_COLS)
                 : "memory");
  // merge this CTA's first maximum into its slot (slots persist over the
  // row batches of one step; the (mag, flat) order makes merging order-free)
  __shared__ Cand red[8 * GROUPS];
  __shared__ Cand win;
  [[maybe_unused]] const double own_mag = best.mag;
  [[maybe_unused]] const long long own_flat = best.flat;
  best = warp_argmax(best);
  const int wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = best;
  __syncthreads();
  if (wid == 0) {
    Cand cc = lane < 8 * GROUPS ? red[lane] : best;
    cc = warp_argmax(cc);
    if (lane == 0) win = cc;
  }
  __syncthreads();
  [[maybe_unused]] double r2 = -1.0;
  if constexpr (track2) {
    __shared__ double red2[8 * GROUPS];
    r2 = cta_runner_up(sec, own_mag, own_flat, win.flat, red2);
  }
  if (threadIdx.x == 0) {
    const Cand cc = win;
    Cand& slot = cand[blockIdx.x];
    Cand o = slot;
    if constexpr (track2) cand2[blockIdx.x] = runner_merge(cand2[blockIdx.x], o.mag, r2, cc.mag);
    cand_merge(o, cc);
    slot = o;
  }
}

}  // namespace afd
