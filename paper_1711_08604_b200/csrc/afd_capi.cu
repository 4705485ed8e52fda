// afd_capi.cu — host runtime behind include/afd_capi.h: plans (device
// tables), kernel dispatch by transform length, the device-resident
// decomposition loop captured as a CUDA graph, and the sharded step API.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is loaded at run time (nccl())

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/afd_capi.h"
#include "afd_kernels.cuh"
#include "afd_aux.cuh"
#include "afd_col_tma.cuh"
#include "afd_step_cluster.cuh"
#include "afd_big.cuh"
#include "afd_pruned.cuh"
#include "afd_field_warp.cuh"
#include "afd_field_reg.cuh"
#include "afd_field_sub.cuh"
#include "afd_direct.cuh"

using namespace afd;

static_assert(sizeof(afd_step) == sizeof(Step), "afd_step layout");
static_assert(sizeof(afd_candidate) == sizeof(Cand), "afd_candidate layout");

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(AFD_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                            \
  } while (0)

constexpr int kMinK = 3;
constexpr int kMaxOnChipK = 13;
constexpr int kMaxK = 22;
// Row-batch intermediate for large N.  Larger batches measured faster all the
// way up (fewer launches and launch tails; L2 residency matters less): c2
// field 3.34 ms at 148 rows -> 2.59 ms with all 4096 rows (4 GiB).
constexpr size_t kBigBatchBytes = 4ull << 30;
constexpr int kBigParts = 256;  // first-stage candidate partials (large N)

}  // namespace

struct afd_plan {
  int device = 0;
  int K = 0;
  int64_t n = 0, m = 0, m0 = 0, m1 = 0, max_batch = 0;
  int sms = 148;
  // device tables
  double* radii = nullptr;    // [M]
  double* pow2 = nullptr;     // [M][kPowRow] libm pow(h, 2.0) around each radius
  double* scales = nullptr;   // [M]
  double2* twst = nullptr;    // stage tables [N-1]
  double2* circle = nullptr;  // [N]
  double* pw = nullptr;       // [m1-m0][N] cumprod r^l (exact mode)
  double2* tw_img = nullptr;  // field kernel's shared-memory twiddle image
  // fast mode (AFD_PLAN_FAST): (c, t) stage tables, their shared-memory
  // image, and per-row weight factor tables instead of pw
  bool fast = false;
  double2* twct = nullptr;     // [N-1] (cos, tan) of the conjugated stage twiddles
  double2* tw_img_ct = nullptr;
  double* fw = nullptr;        // [m1-m0][fw_stride]
  int fw_stride = 0;
  // per-signal working buffers
  double2* ghat = nullptr;    // [max_batch][N]
  double2* rem = nullptr;     // [max_batch][N]
  double2* gin = nullptr;     // [max_batch][N] staged input
  State* state = nullptr;     // [max_batch]
  Cand* cand = nullptr;       // [max_batch][ncand_cap]
  double* cand2 = nullptr;    // [max_batch][ncand_cap] runner-ups (AFD_PLAN_MARGINS)
  bool margins = false;
  int ncand_cap = 0;
  Step* steps = nullptr;      // [max_batch][steps_cap]
  int steps_cap = 0;
  double* scratch = nullptr;  // generic scratch (bookkeeping kernels)
  size_t scratch_bytes = 0;
  // field launch geometry
  int field_occ = 1;
  int field_block = 1;
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  int g_max_terms = -1, g_dc_first = -1;
  double g_threshold = -2;
  int64_t g_batch = -1;
  cudaStream_t g_stream = nullptr;
  int64_t launches = 0;
  int64_t graph_launches_per_replay = 0;
  // 0 = fft engine (bit-exact), 1 = direct engine (O(M N^2) quadrature)
  int engine = 0;
  // large N (K > 13): pw holds pw_rev, ghat holds ghat_rev
  bool big = false;
  int ka = 0;
  int64_t big_rows = 0;        // rows per batch
  double2* Y = nullptr;        // [big_rows][N]
  Cand* big_cand = nullptr;    // [big_rows][N/16/256]
  Cand* big_part = nullptr;    // [kBigParts] first-stage reduction of big_cand
  double* big_cand2 = nullptr; // runner-ups of big_cand / big_part (fast engine)
  double* big_part2 = nullptr;
  unsigned* row_ctr = nullptr; // [max_batch][2] field row counters (dynamic rows)
  int* pw_len = nullptr;       // [m1-m0] first l with r^l == 0 (or N)
  CUtensorMap ymap;            // Y as [big_rows][256][2^ka complex] (8-stage TMA column pass)
  bool ymap_ok = false;
  // pruned fast field (afd_pruned.cuh): rows with a negligible weight tail
  // as batches of Q = N / L on-chip L-point fields, per tier (prune_k)
  bool pruned = false;
  struct PruneTier {
    double* fw = nullptr;       // [m1-m0][FastW<k,4>::STRIDE] weights (this plan's scales)
    double2* ghq = nullptr;     // [Q][L] pre-twiddled spectra
    double2* tw_img = nullptr;  // SmemTw<k,4> (c, t) image
    Cand* cand = nullptr;       // [Q][ncta]
    double* cand2 = nullptr;
    int ncta = 0;
    bool warp = false;          // 1024-point tier: one warp per row (afd_field_warp.cuh)
    int qblocks = 0;            // register tiers: CTAs along q' (afd_field_reg.cuh)
  } tier[kPruneTiers];
  int64_t est_rows[kPruneTiers] = {};  // rows per tier expected from the radii alone
  int first_tier = 0;          // tiers below are switched off (AFD_REG_TIERS=0: kRegTiers)
  bool tier_on[kPruneTiers] = {};  // tiers in use: an unused tier's rows go to the next one
  unsigned long long* hint = nullptr;  // screening hint of the register tiers
  // register tiers for batches of on-chip fields (pruned_small: fast engine,
  // 1024 <= N <= 8192, many signals; afd_field_reg.cuh BATCH)
  bool sp = false;
  double* sp_fw = nullptr;               // [m1-m0][kFwStride] factor rows
  int* sp_mstar = nullptr;               // [max_batch][kSmallTiers] tier limits per signal
  double2* sp_g1k = nullptr;             // [max_batch][N/1024][1024] spectra of the warp tier (N >= 4096)
  double2* sp_gsub[2] = {nullptr, nullptr};  // [max_batch][N/L][L], L = 256, 512 (N >= 4096)
  double* sp_fwsub[2] = {nullptr, nullptr};  // [m1-m0][L/32 + 32] factor rows of the sub tiers
  unsigned long long* sp_hint = nullptr; // [max_batch]
  double2* sp_h = nullptr;               // [max_batch][128 N/32] pre-twiddled spectra
  double2* sp_rlog = nullptr;            // [m1-m0] {log2 r, log2(1 - r)}
  int64_t sp_last_batch = 0;
  int* mstar = nullptr;        // [kPruneTiers] first row failing each tier's test
  unsigned long long* tmax = nullptr;
  // the step's two-pass limit read back by the host (one pinned int, an event
  // right after the pruning test) so that the row batches wholly below it —
  // 63 of 64 at c4 — are not launched at all; not under stream capture
  int* lim_host = nullptr;
  cudaEvent_t lim_ev = nullptr;
  double* nodes = nullptr;     // [2 * N / kNodeLen]
  BigSel* sel = nullptr;
  int* amb = nullptr;
  double2* tmp = nullptr;      // [N] projection spectrum
  // radius-sharded decomposition graph (afd_decompose_sharded)
  Cand* loc_cand = nullptr;    // [max_batch] this rank's candidates
  Cand* gath_cand = nullptr;   // [world][max_batch] all-gathered
  Cand* gath_t = nullptr;      // [max_batch][world] transposed
  int gath_world = 0;
  cudaGraphExec_t sgexec = nullptr;
  const void* sg_comm = nullptr;
  int sg_max_terms = -1, sg_dc_first = -1;
  double sg_threshold = -2;
  int64_t sg_batch = -1;
  cudaStream_t sg_stream = nullptr;
  int64_t sgraph_launches = 0;
  // host-buffer entry point: pinned staging + packed device output
  void* pin = nullptr;
  size_t pin_bytes = 0;
  unsigned char* packed = nullptr;
  size_t packed_bytes = 0;
};

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor in the stream drains (it calls pdl_wait() before
// touching the predecessor's outputs).  Captured graphs keep the edges.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t st, int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  int n = 1;
  if (cluster > 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    n = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  return launch_pdl_cluster(kern, grid, block, smem, st, 1, args...);
}

// ---------------------------------------------------------------------------
// Templated launchers, dispatched on K.
// ---------------------------------------------------------------------------
// Runner-up slots (fast engine, on-chip N) beside the plan's own field
// candidates; null for exact plans, the direct engine and foreign
// candidate arrays (e.g. all-gathered shards), whose records carry NaN.
const double* runner_ups_for(const afd_plan* p, const Cand* cand) {
  return (p->margins && p->engine == 0 && cand != nullptr && cand == p->cand) ? p->cand2 : nullptr;
}

namespace {

// Field kernel geometry: 8 points per thread (radix-8 register passes,
// ~64 registers) so two 512-thread CTAs share an SM; rows of N <= 2048
// are grouped to fill 512 threads.
#ifndef AFD_FIELD_RB
#define AFD_FIELD_RB 4
#endif
constexpr int kFieldRB = AFD_FIELD_RB;
#ifndef AFD_GE_FACTOR
#define AFD_GE_FACTOR 1
#endif

template <int K>
constexpr int groups_for() {
  return Geo<K, kFieldRB>::T >= 512 ? 1 : 512 / Geo<K, kFieldRB>::T;
}

template <int K>
int field_block() {
  return Geo<K, kFieldRB>::T * groups_for<K>();
}

template <int K>
size_t field_smem() {
  return sizeof(double2) *
         (Geo<K, kFieldRB>::SMEM * groups_for<K>() + SmemTw<K, kFieldRB>::ENTRIES);
}

// Single-signal steps spread over an 8-CTA cluster for 1024 <= N <= 8192
// (afd_step_cluster.cuh); smaller N use one CTA per signal.
template <int K>
constexpr bool use_cluster_step() {
  return K >= 10 && K <= 13;
}

// Phase offset between the two row-groups of a field CTA (FieldHook);
// AFD_FIELD_PP=0 turns it off (experiments).
static int field_pp() {
  static int v = [] {
    const char* e = getenv("AFD_FIELD_PP");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int K>
int row_block() {
  return Geo<K>::T < 64 ? 64 : Geo<K>::T;
}

// Field launches with two full row-groups at N = 4096 (four at N = 2048)
// keep their twiddles in TMEM (TmemTw, afd_fft.cuh); AFD_FIELD_TMEM=0 turns
// it off (experiments).
#ifndef AFD_FIELD_TMEM11
#define AFD_FIELD_TMEM11 1
#endif
constexpr bool kFieldTmem11 = AFD_FIELD_TMEM11 != 0;
#ifndef AFD_FIELD_TMEM10
#define AFD_FIELD_TMEM10 1
#endif
constexpr bool kFieldTmem10 = AFD_FIELD_TMEM10 != 0;
#ifndef AFD_FIELD_TMEM9
#define AFD_FIELD_TMEM9 0
#endif
constexpr bool kFieldTmem9 = AFD_FIELD_TMEM9 != 0;
template <int K>
constexpr bool field_tmem_capable() {
  return kFieldRB == 4 && ((K == 12 && groups_for<K>() == 2) ||
                           (K == 11 && groups_for<K>() == 4 && kFieldTmem11) ||
                           (K == 10 && groups_for<K>() == 8 && kFieldTmem10) ||
                           (K == 9 && groups_for<K>() == 16 && kFieldTmem9));
}
static bool field_tmem_enabled() {
  static int v = [] {
    const char* e = getenv("AFD_FIELD_TMEM");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

template <int K, bool MAT>
int setup_field_kernel(int* occ) {
  auto kern = field_kernel<K, kFieldRB, groups_for<K>(), MAT>;
  CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem<K>()));
  CU(cudaFuncSetAttribute(field_kernel<K, kFieldRB, groups_for<K>(), MAT, false, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem<K>()));
  if constexpr (field_tmem_capable<K>()) {
    CU(cudaFuncSetAttribute(field_kernel<K, kFieldRB, groups_for<K>(), MAT, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)field_smem<K>()));
    CU(cudaFuncSetAttribute(field_kernel<K, kFieldRB, groups_for<K>(), MAT, true, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)field_smem<K>()));
    if constexpr (!MAT)
      CU(cudaFuncSetAttribute(field_kernel<K, kFieldRB, groups_for<K>(), MAT, true, true, true>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)field_smem<K>()));
  }
  if constexpr (!MAT)
    CU(cudaFuncSetAttribute(field_kernel<K, kFieldRB, groups_for<K>(), MAT, false, true, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem<K>()));
  if (occ) CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, field_block<K>(), field_smem<K>()));
  return 0;
}

template <int K>
__global__ void build_tw_image_kernel(double2* img, const double2* st) {
  SmemTw<K, kFieldRB>::build_image(img, st);
}

template <int K>
int setup_kernels(afd_plan* p) {
  int rc;
  {
    const int smem = (int)(sizeof(double2) * dpad(1 << K));
    CU(cudaFuncSetAttribute(direct_field_kernel<false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CU(cudaFuncSetAttribute(direct_field_kernel<true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  CU(cudaMalloc(&p->tw_img, sizeof(double2) * SmemTw<K, kFieldRB>::ENTRIES));
  build_tw_image_kernel<K><<<32, 256>>>(p->tw_img, p->twst);
  p->launches++;
  if (p->fast) {
    CU(cudaMalloc(&p->tw_img_ct, sizeof(double2) * SmemTw<K, kFieldRB>::ENTRIES));
    build_tw_image_kernel<K><<<32, 256>>>(p->tw_img_ct, p->twct);
    p->launches++;
  }
  CU(cudaGetLastError());
  p->field_block = field_block<K>();
  if ((rc = setup_field_kernel<K, false>(&p->field_occ))) return rc;
  if ((rc = setup_field_kernel<K, true>(nullptr))) return rc;
  CU(cudaFuncSetAttribute(step_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)RowSmem<K>::bytes));
  CU(cudaFuncSetAttribute(step_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)RowSmem<K>::bytes));
  if constexpr (use_cluster_step<K>()) {
    CU(cudaFuncSetAttribute(step_cluster_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ClusterSmem<K>::bytes));
    CU(cudaFuncSetAttribute(step_cluster_kernel<K>,
                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CU(cudaFuncSetAttribute(step_cluster_kernel<K, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ClusterSmem<K>::bytes));
    CU(cudaFuncSetAttribute(step_cluster_kernel<K, true>,
                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  CU(cudaFuncSetAttribute(fft_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)RowSmem<K>::bytes));
  if (p->field_occ < 1) p->field_occ = 1;
  return 0;
}

// Number of CTAs per signal for `rows` rows: minimise waves x (units per CTA
// + one unit of per-CTA setup: TMEM allocation and twiddle fill, first-row
// loads, the closing reduction — measured ~1 row-pair; c3 with 16-row CTAs
// ran 10% slower than with whole-signal CTAs, 128 signals with 2-row CTAs 1.9x).
int field_ctas(const afd_plan* p, int64_t rows, int G, int64_t batch, int block = 0) {
  const int64_t units = (rows + G - 1) / G;
  // a reduced block (fewer row-groups) fits proportionally more CTAs per SM
  const int occ = block > 0 ? std::max(1, std::min(32, (int)(p->field_occ * (int64_t)p->field_block / block)))
                            : p->field_occ;
  const int64_t slots = (int64_t)p->sms * occ;
  int64_t best_x = 1;
  double best_t = 1e300;
  for (int64_t x = 1; x <= units && x <= 65535; ++x) {
    const int64_t per = (units + x - 1) / x;
    if (x > 1 && (units + x - 2) / (x - 1) == per) continue;  // same per-CTA load, more CTAs
    const int64_t ctas = x * batch;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double t = (double)waves * (double)(per + 1) + 1e-3 * (double)ctas / (double)slots;
    if (t < best_t) {
      best_t = t;
      best_x = x;
    }
  }
  return (int)best_x;
}

// Row-groups per CTA actually launched: fewer than G when the launch is too
// small to fill the GPU with full CTAs (small M, e.g. BASELINE c0).
template <int K>
int groups_eff(const afd_plan* p, int64_t rows, int64_t batch) {
  constexpr int G = groups_for<K>();
  constexpr int gmin = Geo<K, kFieldRB>::T >= 32 ? 1 : 32 / Geo<K, kFieldRB>::T;  // >= 1 warp
  int g = G;
  while (g > gmin && ((rows + g - 1) / g) * batch < AFD_GE_FACTOR * p->sms) g >>= 1;
  return g;
}

template <int K>
int launch_field(afd_plan* p, const double2* ghat, int64_t r0, int64_t r1, int64_t batch,
                 Cand* cand, int ncta, double2* field_out, const State* state, cudaStream_t st,
                 unsigned* row_ctr = nullptr, int launch_id = 0, const SubMap* subp = nullptr) {
  constexpr int G = groups_for<K>();
  const int ge = groups_eff<K>(p, r1 - r0, batch);  // ncta from field_ctas_for
  dim3 grid(ncta, (unsigned)batch);
  const int block = Geo<K, kFieldRB>::T * ge;
  const size_t smem = sizeof(double2) *
                      (Geo<K, kFieldRB>::SMEM * ge + SmemTw<K, kFieldRB>::ENTRIES);
  // TMEM twiddles need the whole TMEM of the SM: only for one full-size CTA
  // (both row-groups) per SM
  const bool tm = field_tmem_capable<K>() && ge == G && field_tmem_enabled();
  constexpr bool TMC = field_tmem_capable<K>();
  // exact: the cumprod table and the numpy twiddle image; fast: the weight
  // factor tables and the (c, t) image
  const double* tab = p->fast ? p->fw : p->pw;
  const double2* img = p->fast ? p->tw_img_ct : p->tw_img;
  if (field_out) {
    auto kern = p->fast ? (tm ? field_kernel<K, kFieldRB, G, true, TMC, true>
                              : field_kernel<K, kFieldRB, G, true, false, true>)
                        : (tm ? field_kernel<K, kFieldRB, G, true, TMC>
                              : field_kernel<K, kFieldRB, G, true>);
    kern<<<grid, block, smem, st>>>(ghat, tab, p->scales, p->twst, r0, r1, p->m0, nullptr,
                                    field_out, nullptr, img, field_pp(), (unsigned*)nullptr, 0,
                                    SubMap{0, 0, nullptr, nullptr});
  } else {
    const bool mg = runner_ups_for(p, cand) != nullptr;
    auto kern = p->fast ? (mg ? (tm ? field_kernel<K, kFieldRB, G, false, TMC, true, true>
                                    : field_kernel<K, kFieldRB, G, false, false, true, true>)
                              : (tm ? field_kernel<K, kFieldRB, G, false, TMC, true>
                                    : field_kernel<K, kFieldRB, G, false, false, true>))
                        : (tm ? field_kernel<K, kFieldRB, G, false, TMC>
                              : field_kernel<K, kFieldRB, G, false>);
    if (subp)  // pruned_small: the launch reads its row limits at its top, so no PDL
      kern<<<grid, block, smem, st>>>(ghat, tab, (const double*)p->scales,
                                      (const double2*)p->twst, (long long)r0, (long long)r1,
                                      (long long)p->m0, cand, (double2*)nullptr, state, img,
                                      field_pp(), row_ctr, launch_id, *subp);
    else
    CU(launch_pdl(kern, grid, dim3(block), smem, st, ghat, tab,
                  (const double*)p->scales, (const double2*)p->twst, (long long)r0,
                  (long long)r1, (long long)p->m0, cand, (double2*)nullptr, state,
                  img, field_pp(), row_ctr, launch_id,
                  SubMap{0, 0, nullptr, const_cast<double*>(runner_ups_for(p, cand))}));
  }
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

// Batches of at least this many signals (default: one per SM) take one CTA
// per signal for the step instead of a cluster (c3, 1024 signals: +3%);
// AFD_STEP_CTA_BATCH overrides (experiments).
static const int64_t kStepCtaBatchEnv =
    getenv("AFD_STEP_CTA_BATCH") ? atoll(getenv("AFD_STEP_CTA_BATCH")) : 0;

template <int K>
int launch_step(afd_plan* p, int k, int max_terms, double thr, int dc_first, const double2* g0,
                const Cand* cand, int ncand, int64_t batch, Step* steps, cudaStream_t st) {
  // the fast field's runner-ups travel beside its own candidates
  const double* c2 = runner_ups_for(p, cand);
  // A single signal's step is latency-bound: a cluster of CTAs shares it.
  // Many signals fill the GPU with one CTA each.
  const int64_t cta_batch = kStepCtaBatchEnv > 0 ? kStepCtaBatchEnv : (int64_t)p->sms;
  if (use_cluster_step<K>() && batch < cta_batch) {
    if constexpr (use_cluster_step<K>())
    CU(launch_pdl_cluster(c2 ? step_cluster_kernel<K, true> : step_cluster_kernel<K, false>,
                  dim3((unsigned)(batch * ClusterGeo<K>::C)),
                  dim3(ClusterGeo<K>::THREADS), ClusterSmem<K>::bytes, st, ClusterGeo<K>::C, k,
                  max_terms, thr, dc_first, g0, p->rem, p->ghat, cand, ncand,
                  (const double*)p->radii, (int)p->m, (const double2*)p->circle,
                  (const double2*)p->twst, p->state, steps, (const double*)p->pow2, c2));
  } else {
    CU(launch_pdl(c2 ? step_kernel<K, true> : step_kernel<K, false>, dim3((unsigned)batch),
                  dim3(row_block<K>()),
                  RowSmem<K>::bytes, st, k, max_terms, thr, dc_first, g0, p->rem, p->ghat, cand,
                  ncand, (const double*)p->radii, (const double2*)p->circle,
                  (const double2*)p->twst, p->state, steps, (const double*)p->pow2, c2));
  }
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

template <int K>
int launch_fft(afd_plan* p, int mode, const double2* x, double2* y, int64_t batch,
               cudaStream_t st) {
  fft_kernel<K><<<(unsigned)batch, row_block<K>(), RowSmem<K>::bytes, st>>>(mode, x, y, p->twst);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

// Dispatch helper: calls F<K>::run(args...) for the plan's K.
#define AFD_DISPATCH(KV, ...)                 \
  switch (KV) {                                \
    case 3: { constexpr int KK = 3; __VA_ARGS__; }    \
    case 4: { constexpr int KK = 4; __VA_ARGS__; }    \
    case 5: { constexpr int KK = 5; __VA_ARGS__; }    \
    case 6: { constexpr int KK = 6; __VA_ARGS__; }    \
    case 7: { constexpr int KK = 7; __VA_ARGS__; }    \
    case 8: { constexpr int KK = 8; __VA_ARGS__; }    \
    case 9: { constexpr int KK = 9; __VA_ARGS__; }    \
    case 10: { constexpr int KK = 10; __VA_ARGS__; }  \
    case 11: { constexpr int KK = 11; __VA_ARGS__; }  \
    case 12: { constexpr int KK = 12; __VA_ARGS__; }  \
    case 13: { constexpr int KK = 13; __VA_ARGS__; }  \
    default:                                   \
      return fail(AFD_E_UNSUPPORTED, "transform length 2^%d not supported yet", KV); \
  }

int groups_of(int K) {
  AFD_DISPATCH(K, return groups_for<KK>());
}

// Direct engine: one CTA per (row, signal) reading the remainder G_k.
int launch_direct(afd_plan* p, const double2* g, int64_t r0, int64_t r1, int64_t batch,
                  Cand* cand, double2* field_out, const State* state, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (size_t)dpad((int)p->n);
  dim3 grid((unsigned)(r1 - r0), (unsigned)batch);
  if (field_out) {
    direct_field_kernel<true><<<grid, kDirectThreads, smem, st>>>(
        (int)p->n, g, p->radii, p->circle, r0, r1, nullptr, field_out, nullptr);
  } else {
    CU(launch_pdl(direct_field_kernel<false>, grid, dim3(kDirectThreads), smem, st, (int)p->n,
                  g, (const double*)p->radii, (const double2*)p->circle, (long long)r0,
                  (long long)r1, cand, (double2*)nullptr, state));
  }
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

// CTAs per signal of a field launch over `rows` rows (what launch_field uses).
int field_ctas_for(const afd_plan* p, int64_t rows, int64_t batch) {
  if (p->engine == 1) return (int)rows;
  if (const char* e = getenv("AFD_FIELD_CTAS")) {  // experiments
    const int x = atoi(e);
    if (x > 0) return (int)std::min<int64_t>(x, rows);
  }
  AFD_DISPATCH(p->K, {
    constexpr int G = groups_for<KK>();
    const int ge = groups_eff<KK>(p, rows, batch);
    return ge == G ? field_ctas(p, rows, G, batch)
                   : field_ctas(p, rows, ge, batch, Geo<KK, kFieldRB>::T * ge);
  });
}


// Dynamic field rows (field_kernel row_ctr): a single signal whose rows fill
// both row-groups of every CTA runs on every SM, later rows claimed at run
// time.  Off by default (AFD_FIELD_DYN=1 turns it on): on c1 the 148-CTA
// launch with run-time rows measured slower (1.095e11 vs 1.163e11 evals/s)
// than the static 128-CTA schedule.  0 = not used.
static bool field_dyn_enabled() {
  static int v = [] {
    const char* e = getenv("AFD_FIELD_DYN");
    return e ? atoi(e) : 0;
  }();
  return v != 0;
}
int field_dyn_ctas(const afd_plan* p, int64_t rows, int64_t batch) {
  if (!field_dyn_enabled() || p->big || p->engine != 0 || batch != 1) return 0;
  AFD_DISPATCH(p->K, {
    constexpr int G = groups_for<KK>();
    if (G < 2 || Geo<KK, kFieldRB>::T % 32 != 0 || groups_eff<KK>(p, rows, batch) != G) return 0;
    const int64_t slots = (int64_t)p->sms * p->field_occ;
    if ((rows + G - 1) / G <= slots) return 0;  // one row per group already: nothing to balance
    return (int)slots;
  });
}

// CTAs per signal of the decomposition's field launches
int decomp_field_ctas(const afd_plan* p, int64_t batch) {
  const int64_t rows = p->m1 - p->m0;
  const int d = field_dyn_ctas(p, rows, batch);
  return d ? d : field_ctas_for(p, rows, batch);
}

// The decomposition graph bakes in the addresses of the plan's buffers:
// any reallocation must drop it (it is re-captured on the next call).
void invalidate_graph(afd_plan* p) {
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  p->gexec = nullptr;
  if (p->sgexec) cudaGraphExecDestroy(p->sgexec);
  p->sgexec = nullptr;
  p->sg_comm = nullptr;
  p->g_max_terms = -1;
  p->g_dc_first = -1;
  p->g_threshold = -2;
  p->g_batch = -1;
  p->g_stream = nullptr;
}

int ensure_cand(afd_plan* p, int64_t batch, int ncta) {
  if (ncta > p->ncand_cap) {
    invalidate_graph(p);
    if (p->cand) cudaFree(p->cand);
    if (p->cand2) cudaFree(p->cand2);
    p->cand = nullptr;
    p->cand2 = nullptr;
    p->ncand_cap = 0;
    CU(cudaMalloc(&p->cand, sizeof(Cand) * (size_t)p->max_batch * ncta));
    if (p->margins) CU(cudaMalloc(&p->cand2, sizeof(double) * (size_t)p->max_batch * ncta));
    p->ncand_cap = ncta;
  }
  (void)batch;
  return 0;
}

int ensure_steps(afd_plan* p, int max_terms) {
  if (max_terms > p->steps_cap) {
    invalidate_graph(p);
    if (p->steps) cudaFree(p->steps);
    p->steps = nullptr;
    p->steps_cap = 0;
    CU(cudaMalloc(&p->steps, sizeof(Step) * (size_t)p->max_batch * max_terms));
    p->steps_cap = max_terms;
  }
  return 0;
}

int ensure_scratch(afd_plan* p, size_t bytes) {
  if (bytes > p->scratch_bytes) {
    if (p->scratch) cudaFree(p->scratch);
    p->scratch = nullptr;
    p->scratch_bytes = 0;
    CU(cudaMalloc(&p->scratch, bytes));
    p->scratch_bytes = bytes;
  }
  return 0;
}

int check_batch(const afd_plan* p, int64_t batch) {
  if (batch < 1 || batch > p->max_batch)
    return fail(AFD_E_INVALID, "batch %lld outside 1..%lld", (long long)batch,
                (long long)p->max_batch);
  return 0;
}

int set_device(const afd_plan* p) {
  CU(cudaSetDevice(p->device));
  return 0;
}

// Batches of on-chip fields with the register tiers (pruned_small).  Per
// step: prune_small_kernel (per-signal tier limits, hints, pre-twiddled
// spectra), the N-point field kernel over each signal's rows from its last
// limit on (it publishes the signal's hint), then the register kernels over
// the rows below — all into one candidate row per signal: [ncta N-point
// slots | per tier nc[t] * Q'/32 warp slots].
static const bool kSmallPrunedOn = !(getenv("AFD_SMALL_PRUNED") && atoi(getenv("AFD_SMALL_PRUNED")) == 0);
// AFD_SMALL_WARP_TIER=0: no 1024-point warp tier in batches (A/B switch)
static const bool kSmallWarpTier = !(getenv("AFD_SMALL_WARP_TIER") && atoi(getenv("AFD_SMALL_WARP_TIER")) == 0);
constexpr int64_t kSmallPrunedMinEvals = 1LL << 28;  // per field launch (c3: 2^32)

int tier_ncta(const afd_plan* p, int64_t q, int64_t est, int rpc, double prologue);

// the register kernels whose extra warps keep their spectra in shared memory
int reg_kernel_attrs() {
  if (fr_smem_bytes(4) > 0) {
    const int b = (int)fr_smem_bytes(4);
    CU(cudaFuncSetAttribute(field_reg_kernel<4, false, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CU(cudaFuncSetAttribute(field_reg_kernel<4, true, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CU(cudaFuncSetAttribute(field_reg_kernel<4, false, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, b));
    CU(cudaFuncSetAttribute(field_reg_kernel<4, true, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, b));
  }
  return 0;
}

struct SmallGrid {
  bool pruned;
  int ncta;            // CTAs per signal of the N-point field
  int nc[kRegTiers];   // row splits per register tier
  int off[kRegTiers];  // first candidate slot per tier
  int nc1k, off1k;     // the 1024-point warp tier (N >= 4096; nc1k = 0: none)
  int ncs[2], offs[2]; // the 256- and 512-point tiers (ncs = 0: none)
  int ncand;           // candidates per signal
};

SmallGrid small_grid(const afd_plan* p, int64_t batch, int ncta) {
  SmallGrid g{};
  g.ncta = ncta;
  g.ncand = ncta;
  const int64_t rows = p->m1 - p->m0;
  g.pruned = p->sp && batch >= 8 && batch * rows * p->n >= kSmallPrunedMinEvals;
  if (!g.pruned) return g;
  const int64_t qn = p->n >> 5;
  for (int t = 0; t < kRegTiers; ++t) {
    const int qt = fr_qthreads(1 << t), share = fr_share(1 << t);
    const int64_t yb = (batch * qn + qt - 1) / qt;
    g.nc[t] = (int)std::min<int64_t>(tier_ncta(p, yb, p->est_rows[t], share, 1.0), rows);
    g.off[t] = g.ncand;
    g.ncand += g.nc[t] * share * (int)(qn >> 5);
  }
  if (p->sp_g1k) {
    const int64_t q1k = p->n >> kFwK;
    g.nc1k = (int)std::max<int64_t>(
        1, std::min<int64_t>(tier_ncta(p, batch * q1k, p->est_rows[kRegTiers], kFwWarps, 1.6),
                             (rows + kFwWarps - 1) / kFwWarps));
    g.off1k = g.ncand;
    g.ncand += g.nc1k * (int)q1k;
  }
  for (int u = 0; u < 2; ++u) {
    if (!p->sp_gsub[u]) continue;
    const int kl = 8 + u, S = 32 >> (kl - 5);
    const int64_t qb = (p->n >> kl) / S;  // CTAs along y per signal
    g.ncs[u] = (int)std::max<int64_t>(
        1, std::min<int64_t>(tier_ncta(p, batch * qb, p->est_rows[kTierSub + u], kFwWarps, 1.6),
                             (rows + kFwWarps - 1) / kFwWarps));
    g.offs[u] = g.ncand;
    g.ncand += g.ncs[u] * (int)qb;
  }
  return g;
}

// lower limit of tier t: the limit of the last tier in use below it
const int* tier_lo(const afd_plan* p, const int* mstar, int t) {
  for (int u = t - 1; u >= 0; --u)
    if (p->tier_on[u]) return mstar + u;
  return nullptr;
}

template <int D>
int launch_reg_small(afd_plan* p, int t, int64_t batch, Cand* cand, const SmallGrid& sg,
                     cudaStream_t st) {
  const int64_t qn = p->n >> 5;
  const int threads = fr_threads(D);
  const unsigned yb = (unsigned)((batch * qn + fr_qthreads(D) - 1) / fr_qthreads(D));
  double* c2 = const_cast<double*>(runner_ups_for(p, cand));
  auto rk = c2 ? field_reg_kernel<D, true, true> : field_reg_kernel<D, false, true>;
  rk<<<dim3((unsigned)sg.nc[t], yb), threads, fr_smem_bytes(D), st>>>(
      p->sp_h, p->sp_fw, (long long)p->m0, (long long)p->m1, (long long)p->m0, (long long)qn, cand,
      p->sp_hint,
      SubMap{(long long)p->n, 0, p->sp_mstar + t, c2, tier_lo(p, p->sp_mstar, t), nullptr,
             kSmallTiers, sg.ncand, 0},
      RegBatch{p->K - 5, batch * qn, sg.off[t]});
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

template <int KL>
int launch_sub_small(afd_plan* p, int u, int64_t batch, Cand* cand, const SmallGrid& sg,
                     cudaStream_t st) {
  using SG = SubGeo<KL>;
  const int ql = (int)(p->n >> KL);
  double* c2 = const_cast<double*>(runner_ups_for(p, cand));
  auto sk = c2 ? field_sub_kernel<KL, true, true> : field_sub_kernel<KL, false, true>;
  sk<<<dim3((unsigned)sg.ncs[u], (unsigned)(batch * (ql / SG::S))), 32 * kFwWarps, SG::kSmem, st>>>(
      p->sp_gsub[u], p->sp_fwsub[u], p->twct, (long long)p->m0, (long long)p->m1, (long long)p->m0,
      cand,
      SubMap{(long long)p->n, ql, p->sp_mstar + kTierSub + u, c2,
             tier_lo(p, p->sp_mstar, kTierSub + u), p->sp_hint, kSmallTiers, sg.ncand,
             sg.offs[u]});
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

template <int K>
int launch_field_small_pruned(afd_plan* p, const double2* ghat, int64_t batch, Cand* cand,
                              const SmallGrid& sg, const State* state, cudaStream_t st) {
  int rc;
  prune_small_kernel<<<(unsigned)batch, 256, 0, st>>>(K, ghat, p->sp_rlog, p->m0, p->m1, p->circle,
                                                      state, p->sp_mstar, p->sp_hint, p->sp_h,
                                                      SmallSpectra{{p->sp_gsub[0], p->sp_gsub[1],
                                                                    p->sp_g1k}});
  p->launches++;
  CU(cudaGetLastError());
  p->sp_last_batch = batch;
  double* c2 = const_cast<double*>(runner_ups_for(p, cand));
  // (without the longer tiers their limits repeat the last register tier's)
  const SubMap sub{0, 0, nullptr, c2, p->sp_mstar + kSmallTiers - 1, p->sp_hint, kSmallTiers,
                   sg.ncand, 0};
  if ((rc = launch_field<K>(p, ghat, p->m0, p->m1, batch, cand, sg.ncta, nullptr, state, st,
                            nullptr, 0, &sub)))
    return rc;
  if (sg.nc1k > 0) {  // rows up to the 1024-term limit as N / 1024 1024-point fields, one warp per row
    const int q1k = (int)(p->n >> kFwK);
    auto wk = c2 ? field_warp_kernel<true, true> : field_warp_kernel<false, true>;
    wk<<<dim3((unsigned)sg.nc1k, (unsigned)(batch * q1k)), 32 * kFwWarps, kFwSmem, st>>>(
        p->sp_g1k, p->sp_fw, p->twct, (long long)p->m0, (long long)p->m1, (long long)p->m0, cand,
        SubMap{(long long)p->n, q1k, p->sp_mstar + kTier1k, c2, tier_lo(p, p->sp_mstar, kTier1k),
               p->sp_hint, kSmallTiers, sg.ncand, sg.off1k});
    p->launches++;
    CU(cudaGetLastError());
  }
  if (sg.ncs[1] > 0 && (rc = launch_sub_small<9>(p, 1, batch, cand, sg, st))) return rc;
  if (sg.ncs[0] > 0 && (rc = launch_sub_small<8>(p, 0, batch, cand, sg, st))) return rc;
  if ((rc = launch_reg_small<1>(p, 0, batch, cand, sg, st))) return rc;
  if ((rc = launch_reg_small<2>(p, 1, batch, cand, sg, st))) return rc;
  return launch_reg_small<4>(p, 2, batch, cand, sg, st);
}

// Enqueue the whole decomposition (init + max_terms steps) on `st`.
int enqueue_decompose(afd_plan* p, int64_t batch, int max_terms, double thr, int dc_first,
                      cudaStream_t st) {
  const int64_t rows = p->m1 - p->m0;
  const int G = groups_of(p->K);
  const int ncta = decomp_field_ctas(p, batch);
  const bool dyn = field_dyn_ctas(p, rows, batch) > 0;
  const SmallGrid sg = small_grid(p, batch, ncta);
  int rc;
  if ((rc = ensure_cand(p, batch, sg.ncand))) return rc;
  if (dyn) CU(cudaMemsetAsync(p->row_ctr, 0, sizeof(unsigned) * 2 * (size_t)batch, st));
  AFD_DISPATCH(p->K, {
    if ((rc = launch_step<KK>(p, -1, max_terms, thr, dc_first, p->gin, nullptr, 0, batch,
                              p->steps, st)))
      return rc;
    for (int k = 0; k < max_terms; ++k) {
      if (!(k == 0 && dc_first)) {
        if (p->engine == 1)
          rc = launch_direct(p, p->rem, p->m0, p->m1, batch, p->cand, nullptr, p->state, st);
        else if (sg.pruned)
          rc = launch_field_small_pruned<KK>(p, p->ghat, batch, p->cand, sg, p->state, st);
        else
          rc = launch_field<KK>(p, p->ghat, p->m0, p->m1, batch, p->cand, ncta, nullptr,
                                p->state, st, dyn ? p->row_ctr : nullptr, k);
        if (rc) return rc;
      }
      if ((rc = launch_step<KK>(p, k, max_terms, thr, dc_first, nullptr, p->cand, sg.ncand, batch,
                                p->steps, st)))
        return rc;
    }
    return 0;
  });
}

// ---------------------------------------------------------------------------
// Large N (K > 13): row-batched two-level DIT (afd_big.cuh).
// ---------------------------------------------------------------------------
#define AFD_KA_DISPATCH(KAV, ...)             \
  switch (KAV) {                               \
    case 9: { constexpr int KA = 9; __VA_ARGS__; }    \
    case 10: { constexpr int KA = 10; __VA_ARGS__; }  \
    case 11: { constexpr int KA = 11; __VA_ARGS__; }  \
    case 12: { constexpr int KA = 12; __VA_ARGS__; }  \
    default:                                   \
      return fail(AFD_E_UNSUPPORTED, "bad pass-A size %d", KAV); \
  }

int big_col_ctas(const afd_plan* p) { return (int)((p->n / 16 + kColThreads - 1) / kColThreads); }

int big_setup(afd_plan* p) {
  AFD_KA_DISPATCH(p->ka, {
    CU(cudaFuncSetAttribute(big_pass_a<KA, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)big_a_smem_g<KA>()));
    CU(cudaFuncSetAttribute(big_pass_a<KA, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)big_a_smem_g<KA>()));
    CU(cudaFuncSetAttribute(big_pass_a<KA, true, KA == 12>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big_a_smem_g<KA>()));
    CU(cudaFuncSetAttribute(big_field_a<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)big_a_smem_g<12>()));
    CU(cudaFuncSetAttribute(big_field_a<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)big_a_smem_g<12>()));
    CU(cudaFuncSetAttribute(col_tma_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ColTma<4>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ColTma<8>::SMEM));
    CU(cudaFuncSetAttribute(big_pass_col8<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double2) * 16 * kCol8Pad)));
    CU(cudaFuncSetAttribute(big_pass_col8<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double2) * 16 * kCol8Pad)));
    CU(cudaFuncSetAttribute(col_tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ColTma<4>::SMEM));
    if (p->K - p->ka == 8) {
      // Y as float64 [big_rows][256 positions u][2 * 2^ka] (position u of
      // column q at q + (u << ka)), boxes of 16 columns x 256 positions
      using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult qr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) ==
              cudaSuccess &&
          qr == cudaDriverEntryPointSuccess && fn) {
        const cuuint64_t dims[3] = {2ull << p->ka, 256, (cuuint64_t)p->big_rows};
        const cuuint64_t strides[2] = {16ull << p->ka, 16ull * (cuuint64_t)p->n};
        const cuuint32_t box[3] = {32, 256, 1}, estr[3] = {1, 1, 1};
        p->ymap_ok = ((EncodeFn)fn)(&p->ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, p->Y, dims,
                                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      }
    }
    CU(cudaFuncSetAttribute(col_tma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ColTma<8>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<8, true, 2>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColTma<8, 2>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<8, false, 2>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColTma<8, 2>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<4, true, 2>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColTma<4, 2>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<4, false, 2>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColTma<4, 2>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<8, true, 2, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColTma<8, 2>::SMEM));
    CU(cudaFuncSetAttribute(col_tma_kernel<4, true, 2, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ColTma<4, 2>::SMEM));
    return 0;
  });
}

// Block-major field pass A with the spectrum in TMEM (big_field_a);
// AFD_FIELD_A=0 keeps big_pass_a's item order (experiments).
static const bool kFieldAEnabled = !(getenv("AFD_FIELD_A") && atoi(getenv("AFD_FIELD_A")) == 0);

// Field pass A writes its blocks straight from registers (1) or stages them
// in shared memory for one TMA bulk store (0); AFD_PASSA_DIRECT selects.
static const int kPassADirect = getenv("AFD_PASSA_DIRECT") ? atoi(getenv("AFD_PASSA_DIRECT")) : 0;

// Pass A over rows [r0, r0+rows) (mode 0: field prologue) or one signal (mode 1).
int big_launch_a(afd_plan* p, bool inv, int mode, const double2* ghat_rev, const double2* x,
                 int64_t r0, int64_t rows, const int* stopped, cudaStream_t st,
                 const int* lim = nullptr) {
  const int64_t items = (p->n >> p->ka) * rows;
  AFD_KA_DISPATCH(p->ka, {
    // persistent: one CTA per SM (2 row-groups each), work items strided
    const unsigned grid = (unsigned)std::min<int64_t>(p->sms, (items + kBigGroups - 1) / kBigGroups);
    const int block = Geo<KA, 4>::T * kBigGroups;
    if (p->fast && inv && mode == 0) {
      // fast field: weights from the factor tables, (c, t) twiddles
      if (KA != 12) return fail(AFD_E_UNSUPPORTED, "fast pass A needs 4096-point blocks");
      big_field_a<true><<<grid, block, big_a_smem_g<KA>(), st>>>(
          p->K, p->fw, p->m0, ghat_rev, p->twct, r0, r0 + rows, p->Y, stopped, nullptr,
          kPassADirect, lim);
    } else if (inv && mode == 0 && KA == 12 && field_tmem_enabled() && kFieldAEnabled)
      big_field_a<false><<<grid, block, big_a_smem_g<KA>(), st>>>(
          p->K, p->pw, p->m0, ghat_rev, p->twst, r0, r0 + rows, p->Y, stopped, p->pw_len,
          kPassADirect);
    else if (inv && mode == 0 && KA == 12 && field_tmem_enabled())
      big_pass_a<KA, true, KA == 12><<<grid, block, big_a_smem_g<KA>(), st>>>(
          p->K, mode, p->pw, p->m0, ghat_rev, x, p->twst, r0, r0 + rows, p->Y, stopped,
          p->pw_len);
    else if (inv)
      big_pass_a<KA, true><<<grid, block, big_a_smem_g<KA>(), st>>>(
          p->K, mode, p->pw, p->m0, ghat_rev, x, p->twst, r0, r0 + rows, p->Y, stopped,
          p->pw_len);
    else
      big_pass_a<KA, false><<<grid, block, big_a_smem_g<KA>(), st>>>(
          p->K, mode, p->pw, p->m0, ghat_rev, x, p->twst, r0, r0 + rows, p->Y, stopped,
          p->pw_len);
    p->launches++;
    CU(cudaGetLastError());
    return 0;
  });
}

static const bool kCol8Enabled = !(getenv("AFD_COL8") && atoi(getenv("AFD_COL8")) == 0);

// The field's last column stages as the persistent TMA-pipelined kernel
// (afd_col_tma.cuh); AFD_COL_TMA=0 keeps the one-tile-per-CTA kernels.
static const bool kColTmaEnabled = !(getenv("AFD_COL_TMA") && atoi(getenv("AFD_COL_TMA")) == 0);

// Thread groups of the TMA column pass (ColTma): 2 = two 256-thread groups
// on a three-stage ring; AFD_COL_GROUPS selects (experiments).
static const int kColGroups = getenv("AFD_COL_GROUPS") ? atoi(getenv("AFD_COL_GROUPS")) : 2;

// Pruned fast field (afd_pruned.cuh); AFD_PRUNED=0 keeps the two-pass path
// for every row (experiments).  It needs the TMA column pass for the rows it
// leaves to the two-pass path (that kernel honours the device row limit).
static const bool kPrunedEnabled = !(getenv("AFD_PRUNED") && atoi(getenv("AFD_PRUNED")) == 0);
bool pruned_col_ok(const afd_plan* p) {
  const int left = p->K - p->ka;
  return kColTmaEnabled && (left == 4 || (left == 8 && kCol8Enabled && p->ymap_ok));
}

int big_launch_cols(afd_plan* p, bool inv, int last_mode, int scale_n, int64_t r0, int64_t rows,
                    double2* fout, const int* stopped, cudaStream_t st, const int* lim = nullptr) {
  dim3 grid((unsigned)big_col_ctas(p), (unsigned)rows);
  // fast arithmetic for the field's column stages only (the transforms of
  // the step bookkeeping stay exact)
  const bool fastf = p->fast && inv && (last_mode == 1 || last_mode == 2);
  for (int b0 = p->ka; b0 < p->K; b0 += 4) {
    const int left = p->K - b0;
    if (inv && last_mode == 1 && kColTmaEnabled &&
        (left == 4 || (left == 8 && kCol8Enabled && p->ymap_ok))) {
      const int64_t tiles = rows * ((int64_t)1 << b0) / (left == 8 ? 16 : 256);
      const unsigned g = (unsigned)std::min<int64_t>(p->sms, tiles);
      const double2* tws = fastf ? p->twct : p->twst;
      if (kColGroups == 2 || p->margins) {  // (runner-ups: two-group kernels only)
        const bool mg = fastf && p->margins;
        auto k8 = mg ? col_tma_kernel<8, true, 2, true>
                     : fastf ? col_tma_kernel<8, true, 2> : col_tma_kernel<8, false, 2>;
        auto k4 = mg ? col_tma_kernel<4, true, 2, true>
                     : fastf ? col_tma_kernel<4, true, 2> : col_tma_kernel<4, false, 2>;
        if (left == 8)
          k8<<<g, 512, ColTma<8, 2>::SMEM, st>>>(p->K, b0, p->Y, tws, p->scales, r0, r0 + rows,
                                                 p->big_cand, stopped, lim, p->big_cand2, p->ymap);
        else
          k4<<<g, 512, ColTma<4, 2>::SMEM, st>>>(p->K, b0, p->Y, tws, p->scales, r0, r0 + rows,
                                                 p->big_cand, stopped, lim, p->big_cand2, p->ymap);
      } else {
        auto k8 = fastf ? col_tma_kernel<8, true> : col_tma_kernel<8>;
        auto k4 = fastf ? col_tma_kernel<4, true> : col_tma_kernel<4>;
        if (left == 8)
          k8<<<g, 256, ColTma<8>::SMEM, st>>>(p->K, b0, p->Y, tws, p->scales, r0, r0 + rows,
                                              p->big_cand, stopped, lim, p->big_cand2, p->ymap);
        else
          k4<<<g, 256, ColTma<4>::SMEM, st>>>(p->K, b0, p->Y, tws, p->scales, r0, r0 + rows,
                                              p->big_cand, stopped, lim, p->big_cand2, p->ymap);
      }
      p->launches++;
      CU(cudaGetLastError());
      break;
    }
    if (fastf) {
      // materialised fast field rows / fallback: one 4-stage pass at a time
      const int mode = (b0 + 4 >= p->K) ? last_mode : 0;
      if (mode == 0)
        big_pass_col<true, 0, true><<<grid, kColThreads, 0, st>>>(
            p->K, p->ka, b0, mode, scale_n, p->Y, p->twct, p->scales, r0, r0 + rows,
            p->big_cand, fout, stopped);
      else if (mode == 1)
        big_pass_col<true, 1, true><<<grid, kColThreads, 0, st>>>(
            p->K, p->ka, b0, mode, scale_n, p->Y, p->twct, p->scales, r0, r0 + rows,
            p->big_cand, fout, stopped);
      else
        big_pass_col<true, -1, true><<<grid, kColThreads, 0, st>>>(
            p->K, p->ka, b0, mode, scale_n, p->Y, p->twct, p->scales, r0, r0 + rows,
            p->big_cand, fout, stopped);
      p->launches++;
      CU(cudaGetLastError());
      continue;
    }
    // 8 stages at once (big_pass_col8) where they are the field's last eight
    // or are followed by more column stages (in-place)
    if (inv && b0 + 8 <= p->K && (last_mode == 1 || b0 + 8 < p->K) && kCol8Enabled) {
      const int mode8 = (b0 + 8 >= p->K) ? 1 : 0;
      const size_t sm8 = sizeof(double2) * 16 * kCol8Pad;
      if (mode8 == 1)
        big_pass_col8<1><<<grid, 256, sm8, st>>>(p->K, b0, p->Y, p->twst, p->scales, r0,
                                                 r0 + rows, p->big_cand, stopped);
      else
        big_pass_col8<0><<<grid, 256, sm8, st>>>(p->K, b0, p->Y, p->twst, p->scales, r0,
                                                 r0 + rows, p->big_cand, stopped);
      p->launches++;
      CU(cudaGetLastError());
      b0 += 4;
      continue;
    }
    const int mode = (b0 + 4 >= p->K) ? last_mode : 0;
    if (inv && mode == 1)
      big_pass_col<true, 1><<<grid, kColThreads, 0, st>>>(p->K, p->ka, b0, mode, scale_n, p->Y,
                                                          p->twst, p->scales, r0, r0 + rows,
                                                          p->big_cand, fout, stopped);
    else if (inv && mode == 0)
      big_pass_col<true, 0><<<grid, kColThreads, 0, st>>>(p->K, p->ka, b0, mode, scale_n, p->Y,
                                                          p->twst, p->scales, r0, r0 + rows,
                                                          p->big_cand, fout, stopped);
    else if (inv)
      big_pass_col<true><<<grid, kColThreads, 0, st>>>(p->K, p->ka, b0, mode, scale_n, p->Y, p->twst,
                                                       p->scales, r0, r0 + rows, p->big_cand,
                                                       fout, stopped);
    else
      big_pass_col<false><<<grid, kColThreads, 0, st>>>(p->K, p->ka, b0, mode, scale_n, p->Y, p->twst,
                                                        p->scales, r0, r0 + rows, p->big_cand,
                                                        fout, stopped);
    p->launches++;
    CU(cudaGetLastError());
  }
  return 0;
}

// The field's per-CTA candidates (big_rows x col CTAs, up to 65536) reduced
// in two stages: kBigParts CTAs, then one (a single CTA over all of them was
// 147 us per c2 step).  Returns the partials and their count for big_select.
int big_reduce_cands(afd_plan* p, cudaStream_t st, const Cand** parts, int* nparts) {
  const int n = (int)(p->big_rows * big_col_ctas(p));
  const int np = std::min(kBigParts, (n + 255) / 256);
  const int per = (n + np - 1) / np;
  cand_partial_kernel<<<np, 256, 0, st>>>(p->big_cand, n, per, p->big_part, p->big_cand2,
                                          p->big_part2);
  p->launches++;
  CU(cudaGetLastError());
  *parts = p->big_part;
  *nparts = np;
  return 0;
}

// AFD_WARP_FIELD=0: the 1024-point tier on field_kernel<10> (16 points per
// thread, two exchanges) instead of the warp-per-row kernel (A/B switch).
static const int kWarpField = getenv("AFD_WARP_FIELD") ? atoi(getenv("AFD_WARP_FIELD")) : 1;

// AFD_TIER_NCTA=n: row splits of every on-chip tier (default: tier_ncta).
static const int kTierNcta = getenv("AFD_TIER_NCTA") ? atoi(getenv("AFD_TIER_NCTA")) : 0;

// Rows per tier from the radii alone (a flat spectrum: T = B_s): the tier of
// r is the first L with r^L / (1 - r) <= 2^-64.  The device decides per step
// (prune_rows_kernel); this only sizes the grids.
void estimate_tier_rows(afd_plan* p, const double* radii_host) {
  for (auto& e : p->est_rows) e = 0;
  for (int64_t s = p->m0; s < p->m1; ++s) {
    const double r = radii_host[s];
    int t = 0;
    if (r > 0.0)
      while (t < kPruneTiers &&
             (double)(1 << prune_k(t)) * std::log2(r) - std::log2(1.0 - r) > -64.0)
        ++t;
    while (t < kPruneTiers && !p->tier_on[t]) ++t;
    if (t < kPruneTiers) p->est_rows[t]++;
  }
}

// Row splits of a tier's grid (nc x q CTAs, one CTA per SM at a time, each
// running its share of the tier's rows `rpc` at a time after a prologue
// worth `prologue` row-times: TMEM allocation, twiddles, the spectrum): the
// nc that minimises waves x (prologue + row rounds) for the expected rows.
int tier_ncta(const afd_plan* p, int64_t q, int64_t est, int rpc, double prologue) {
  if (kTierNcta > 0) return kTierNcta;
  est = std::max<int64_t>(est, rpc);
  int best = 1;
  double best_cost = 1e300;
  for (int nc = 1; nc <= p->sms; ++nc) {
    const double waves = std::ceil((double)nc * q / p->sms);
    const double rounds = std::ceil((double)est / ((double)nc * rpc));
    const double cost = waves * (prologue + rounds);
    if (cost < best_cost) {
      best_cost = cost;
      best = nc;
    }
  }
  return best;
}

// One tier of the pruned fast field (afd_pruned.cuh): tables at plan time.
template <int KT>
int setup_pruned_tier(afd_plan* p, int t) {
  static_assert(field_tmem_capable<KT>(), "pruned tiers use the TMEM field kernel");
  constexpr int G = groups_for<KT>();
  auto& T = p->tier[t];
  T.warp = KT == kFwK && kWarpField;
  const int STR = T.warp ? kFwStride : FastW<KT, kFieldRB>::STRIDE;
  const int rows_per_cta = T.warp ? kFwWarps : G;
  const int64_t rows = p->m1 - p->m0, Q = p->n >> KT;
  CU(cudaMalloc(&T.fw, sizeof(double) * STR * (size_t)rows));
  CU(cudaMalloc(&T.ghq, sizeof(double2) * (size_t)p->n));
  CU(cudaMalloc(&T.tw_img, sizeof(double2) * (SmemTw<KT, kFieldRB>::ENTRIES)));
  // row splits of the grid (ncta x Q): tier_ncta
  const int nc = tier_ncta(p, Q, p->est_rows[t], rows_per_cta, 1.6);
  T.ncta = (int)std::max<int64_t>(1, std::min<int64_t>(nc, (rows + rows_per_cta - 1) / rows_per_cta));
  CU(cudaMalloc(&T.cand, sizeof(Cand) * (size_t)Q * T.ncta));
  if (p->margins) CU(cudaMalloc(&T.cand2, sizeof(double) * (size_t)Q * T.ncta));
  const int64_t total = rows * STR;
  if (T.warp)  // scale r^t (t < 32), r^(32 m) (m < 32): afd_field_warp.cuh
    fast_weight_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256>>>(
        p->radii, p->scales, p->m0, rows, STR, 32, 32, 5, 0, 0, T.fw);
  else
    fast_weight_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256>>>(
        p->radii, p->scales, p->m0, rows, STR, 1 << (KT - 4), 16, KT - 4, 0, 0, T.fw);
  build_tw_image_kernel<KT><<<32, 256>>>(T.tw_img, p->twct);
  p->launches += 2;
  CU(cudaGetLastError());
  CU(cudaFuncSetAttribute(field_kernel<KT, kFieldRB, G, false, true, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem<KT>()));
  CU(cudaFuncSetAttribute(field_kernel<KT, kFieldRB, G, false, true, true, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem<KT>()));
  if (T.warp) {
    CU(cudaFuncSetAttribute(field_warp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kFwSmem));
    CU(cudaFuncSetAttribute(field_warp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kFwSmem));
  }
  return 0;
}

// AFD_LIM_READBACK=0: launch every two-pass row batch (they exit on the
// device limit) instead of reading the limit back (A/B switch).
static const int kLimReadback = getenv("AFD_LIM_READBACK") ? atoi(getenv("AFD_LIM_READBACK")) : 1;

// AFD_SUB_TIERS=0: no 256- / 512-point tiers (their rows stay on the
// 1024-point tier; A/B switch).  A sub tier is used when the rows the radii
// predict for it make at least AFD_SUB_MIN_EVALS grid evaluations per field
// (default 2^30: c4 — field 28.0 -> 26.7 ms; below that the extra launches and
// CTA prologues cost what the shorter transforms save: c2 +2%, c3 +0.3%
// slower when forced on).  The GPU tests run with AFD_SUB_MIN_EVALS=0.
static const int kSubTiersOn = getenv("AFD_SUB_TIERS") ? atoi(getenv("AFD_SUB_TIERS")) : 1;
static const double kSubMinEvals =
    getenv("AFD_SUB_MIN_EVALS") ? atof(getenv("AFD_SUB_MIN_EVALS")) : (double)(1LL << 30);
void estimate_tier_rows(afd_plan* p, const double* radii_host);
// tier_on[] of the sub tiers (the others set by the caller) and est_rows[]
void choose_sub_tiers(afd_plan* p, const double* radii_host, int64_t fields) {
  for (int t = kTierSub; t < kTier1k; ++t) p->tier_on[t] = kSubTiersOn != 0 && p->tier_on[kTier1k];
  estimate_tier_rows(p, radii_host);
  bool changed = false;
  for (int t = kTierSub; t < kTier1k; ++t)
    if (p->tier_on[t] && (double)p->est_rows[t] * (double)p->n * (double)fields < kSubMinEvals) {
      p->tier_on[t] = false;
      changed = true;
    }
  if (changed) estimate_tier_rows(p, radii_host);
}

// A sub-warp tier (afd_field_sub.cuh, L = 2^KL = 256 or 512): factor rows
// {scale r^t, t < L/32; r^(L/32 m), m < 32}, the N/L pre-twiddled spectra,
// per-CTA candidates.
template <int KL>
int setup_sub_tier(afd_plan* p, int t) {
  using SG = SubGeo<KL>;
  auto& T = p->tier[t];
  const int64_t rows = p->m1 - p->m0, Q = p->n >> KL;
  CU(cudaMalloc(&T.fw, sizeof(double) * SG::kStride * (size_t)rows));
  CU(cudaMalloc(&T.ghq, sizeof(double2) * (size_t)p->n));
  T.qblocks = (int)(Q / SG::S);
  const int nc = tier_ncta(p, T.qblocks, p->est_rows[t], kFwWarps, 1.6);
  T.ncta = (int)std::max<int64_t>(1, std::min<int64_t>(nc, (rows + kFwWarps - 1) / kFwWarps));
  CU(cudaMalloc(&T.cand, sizeof(Cand) * (size_t)T.qblocks * T.ncta));
  if (p->margins) CU(cudaMalloc(&T.cand2, sizeof(double) * (size_t)T.qblocks * T.ncta));
  const int64_t total = rows * SG::kStride;
  fast_weight_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256>>>(
      p->radii, p->scales, p->m0, rows, SG::kStride, SG::T, 32, SG::C, 0, 0, T.fw);
  p->launches++;
  CU(cudaGetLastError());
  CU(cudaFuncSetAttribute(field_sub_kernel<KL, false, false>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SG::kSmem));
  CU(cudaFuncSetAttribute(field_sub_kernel<KL, true, false>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SG::kSmem));
  return 0;
}

template <int KL>
int launch_sub_tier(afd_plan* p, int t, const double2* ghat_rev, int64_t r0, int64_t r1,
                    const int* lo, const int* hi, const int* stopped, int* slot, cudaStream_t st) {
  using SG = SubGeo<KL>;
  auto& T = p->tier[t];
  const int Q = (int)(p->n >> KL);
  pretwiddle_kernel<<<4 * p->sms, 256, 0, st>>>(p->K, p->ka, KL, ghat_rev, p->circle, T.ghq,
                                                stopped);
  auto sk = p->margins ? field_sub_kernel<KL, true> : field_sub_kernel<KL, false>;
  sk<<<dim3((unsigned)T.ncta, (unsigned)T.qblocks), 32 * kFwWarps, SG::kSmem, st>>>(
      T.ghq, T.fw, p->twct, (long long)r0, (long long)r1, (long long)p->m0, T.cand,
      SubMap{(long long)p->n, Q, hi, T.cand2, lo, p->hint});
  const int n = T.qblocks * T.ncta;
  const int slots = (int)(p->big_rows * big_col_ctas(p));
  const int np = std::max(1, std::min(std::min(kBigParts, (n + 255) / 256), (slots - *slot) / 2));
  cand_partial_kernel<<<np, 256, 0, st>>>(T.cand, n, (n + np - 1) / np, p->big_cand + *slot,
                                          T.cand2, p->big_cand2 ? p->big_cand2 + *slot : nullptr);
  *slot += np;
  p->launches += 3;
  CU(cudaGetLastError());
  return 0;
}

// AFD_REG_TIERS=0: no register tiers (rows of r <= 0.5 stay on the 1024-point
// tier; A/B switch).
static const int kRegTiersOn = getenv("AFD_REG_TIERS") ? atoi(getenv("AFD_REG_TIERS")) : 1;

// A register tier (afd_field_reg.cuh, D = 2^t blocks of 32 terms): the
// factor rows {scale r^t, t < 32; r^(32 m), m < 32} (tier 0's are shared),
// the [32 D][N / 32] pre-twiddled spectra, per-CTA candidates.
int setup_reg_tier(afd_plan* p, int t) {
  auto& T = p->tier[t];
  const int D = 1 << t;
  const int64_t rows = p->m1 - p->m0, Qp = p->n >> 5;
  T.qblocks = (int)((Qp + fr_qthreads(D) - 1) / fr_qthreads(D));
  if (t == 0) {
    CU(cudaMalloc(&T.fw, sizeof(double) * kFwStride * (size_t)rows));
    const int64_t total = rows * kFwStride;
    fast_weight_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256>>>(
        p->radii, p->scales, p->m0, rows, kFwStride, 32, 32, 5, 0, 0, T.fw);
    p->launches++;
    CU(cudaGetLastError());
  }
  // one buffer of pre-twiddled spectra for the three tiers: block m of
  // register i sits at row m 32 + i whatever D, so the D = 4 layout holds the
  // other two as prefixes (tier[kRegTiers - 1].ghq, one pretwiddle launch)
  if (t == kRegTiers - 1) CU(cudaMalloc(&T.ghq, sizeof(double2) * (size_t)p->n * D));
  const int nc = tier_ncta(p, T.qblocks, p->est_rows[t], fr_share(D), 1.0);
  T.ncta = (int)std::max<int64_t>(1, std::min<int64_t>(nc, rows));
  CU(cudaMalloc(&T.cand, sizeof(Cand) * (size_t)T.qblocks * T.ncta));
  if (p->margins) CU(cudaMalloc(&T.cand2, sizeof(double) * (size_t)T.qblocks * T.ncta));
  return 0;
}

template <int D>
int launch_reg_tier(afd_plan* p, int t, const double2* ghat_rev, int64_t r0, int64_t r1,
                    const int* lo, const int* hi, const int* stopped, int* slot, cudaStream_t st) {
  auto& T = p->tier[t];
  double2* hq = p->tier[kRegTiers - 1].ghq;
  if (t == 0) {  // the register tiers launch in order 0, 1, 2: one pre-twiddle for all
    pretwiddle_reg_kernel<<<4 * p->sms, 256, 0, st>>>(p->K, p->ka, 1 << (kRegTiers - 1), ghat_rev,
                                                      p->circle, hq, stopped);
    p->launches++;
  }
  auto rk = p->margins ? field_reg_kernel<D, true> : field_reg_kernel<D, false>;
  rk<<<dim3((unsigned)T.ncta, (unsigned)T.qblocks), fr_threads(D), fr_smem_bytes(D), st>>>(
      hq, p->tier[0].fw, (long long)r0, (long long)r1, (long long)p->m0,
      (long long)(p->n >> 5), T.cand, p->hint,
      SubMap{(long long)p->n, 0, hi, T.cand2, lo, nullptr}, RegBatch{});
  const int n = T.qblocks * T.ncta;
  const int slots = (int)(p->big_rows * big_col_ctas(p));
  const int np = std::max(1, std::min(std::min(kBigParts, (n + 255) / 256), (slots - *slot) / 2));
  cand_partial_kernel<<<np, 256, 0, st>>>(T.cand, n, (n + np - 1) / np, p->big_cand + *slot,
                                          T.cand2, p->big_cand2 ? p->big_cand2 + *slot : nullptr);
  *slot += np;
  p->launches += 2;
  CU(cudaGetLastError());
  return 0;
}

// One tier per step: pre-twiddled spectra, the on-chip field over rows
// [max(r0, *lo), min(r1, *hi)) (device limits), candidate partials into
// big_cand slots from *slot on.
template <int KT>
int launch_pruned_tier(afd_plan* p, int t, const double2* ghat_rev, int64_t r0, int64_t r1,
                       const int* lo, const int* hi, const int* stopped, int* slot,
                       cudaStream_t st) {
  constexpr int G = groups_for<KT>();
  const int Q = (int)(p->n >> KT);
  auto& T = p->tier[t];
  pretwiddle_kernel<<<4 * p->sms, 256, 0, st>>>(p->K, p->ka, KT, ghat_rev, p->circle, T.ghq,
                                                stopped);
  if (T.warp) {  // 1024-point rows, one warp per row (afd_field_warp.cuh)
    auto wk = p->margins ? field_warp_kernel<true> : field_warp_kernel<false>;
    wk<<<dim3((unsigned)T.ncta, (unsigned)Q), 32 * kFwWarps, kFwSmem, st>>>(
        T.ghq, T.fw, p->twct, (long long)r0, (long long)r1, (long long)p->m0, T.cand,
        SubMap{(long long)p->n, Q, hi, T.cand2, lo, p->hint});
  } else {
    auto pk = p->margins ? field_kernel<KT, kFieldRB, G, false, true, true, true>
                         : field_kernel<KT, kFieldRB, G, false, true, true>;
    pk<<<dim3((unsigned)T.ncta, (unsigned)Q), Geo<KT, kFieldRB>::T * G, field_smem<KT>(), st>>>(
        T.ghq, T.fw, p->scales, p->twct, (long long)r0, (long long)r1, (long long)p->m0, T.cand,
        nullptr, nullptr, T.tw_img, field_pp(), (unsigned*)nullptr, 0,
        SubMap{(long long)p->n, Q, hi, T.cand2, lo, p->hint});
  }
  const int n = Q * T.ncta;
  const int slots = (int)(p->big_rows * big_col_ctas(p));
  const int np = std::max(1, std::min(std::min(kBigParts, (n + 255) / 256), (slots - *slot) / 2));
  cand_partial_kernel<<<np, 256, 0, st>>>(T.cand, n, (n + np - 1) / np, p->big_cand + *slot,
                                          T.cand2, p->big_cand2 ? p->big_cand2 + *slot : nullptr);
  *slot += np;
  p->launches += 3;
  CU(cudaGetLastError());
  return 0;
}

// Timing experiments only (wrong results): AFD_BIG_SKIP=1 skips pass A of
// the field, 2 its column pass.
static const int kBigSkip = getenv("AFD_BIG_SKIP") ? atoi(getenv("AFD_BIG_SKIP")) : 0;

// Field rows [r0, r1) of one spectrum: argmax into big_cand (fout == null,
// slots initialised here) or materialised rows into fout.
int big_field(afd_plan* p, const double2* ghat_rev, int64_t r0, int64_t r1, double2* fout,
              const int* stopped, cudaStream_t st) {
  int rc;
  if (!fout) {
    const int n = (int)(p->big_rows * big_col_ctas(p));
    cand_init_kernel<<<(n + 255) / 256, 256, 0, st>>>(p->big_cand, n, p->big_cand2);
    p->launches++;
  }
  const int* lim = nullptr;
  bool read_lim = false;
  if (!fout && p->pruned) {
    // tier t takes rows [mstar[t-1], mstar[t]) (of the tiers in use): tiers
    // 0..2 in registers (32, 64 and 128 terms), 3 and 4 as N/256 256-point and
    // N/512 512-point fields on 8 / 16 threads each, 5 as N/1024 1024-point
    // fields, 6 as N/4096 4096-point fields, rows [mstar[6], r1) through the
    // batches below (all limits read on the device).  Longest tiers first (the largest |F|^2
    // sit at the radii closest to the poles): each tier's maxima start the
    // next tiers' screens (hint).
    prune_init_kernel<<<1, 1, 0, st>>>(p->mstar, r0, r1, p->first_tier, p->tmax, p->hint);
    prune_tail_kernel<<<2 * p->sms, 256, 0, st>>>(ghat_rev, p->n, p->tmax);
    prune_rows_kernel<<<2 * p->sms, 256, 0, st>>>(p->K, p->ka, ghat_rev, p->radii, r0, r1,
                                                  p->tmax, stopped, p->mstar);
    p->launches += 3;
    CU(cudaGetLastError());
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(st, &cap));
    // (worth a host wait only when there are several batches to skip: c2's
    // rows fit one batch and the wait cost it 1.5%)
    read_lim = kLimReadback && p->lim_host && cap == cudaStreamCaptureStatusNone &&
               (r1 - r0 + p->big_rows - 1) / p->big_rows >= 4;
    if (read_lim) {
      CU(cudaMemcpyAsync(p->lim_host, p->mstar + kPruneTiers - 1, sizeof(int),
                         cudaMemcpyDeviceToHost, st));
      CU(cudaEventRecord(p->lim_ev, st));
    }
    int slot = 0, rc2;
    constexpr int t1k = kTier1k, t4k = kTier4k;
    const int* ms = p->mstar;
    if ((rc2 = launch_pruned_tier<prune_k(t4k)>(p, t4k, ghat_rev, r0, r1, tier_lo(p, ms, t4k),
                                                 ms + t4k, stopped, &slot, st)))
      return rc2;
    if ((rc2 = launch_pruned_tier<prune_k(t1k)>(p, t1k, ghat_rev, r0, r1, tier_lo(p, ms, t1k),
                                                 ms + t1k, stopped, &slot, st)))
      return rc2;
    if (p->tier_on[kTierSub + 1] &&
        (rc2 = launch_sub_tier<9>(p, kTierSub + 1, ghat_rev, r0, r1, tier_lo(p, ms, kTierSub + 1),
                                  ms + kTierSub + 1, stopped, &slot, st)))
      return rc2;
    if (p->tier_on[kTierSub] &&
        (rc2 = launch_sub_tier<8>(p, kTierSub, ghat_rev, r0, r1, tier_lo(p, ms, kTierSub),
                                  ms + kTierSub, stopped, &slot, st)))
      return rc2;
    if (p->tier_on[0]) {
      if ((rc2 = launch_reg_tier<1>(p, 0, ghat_rev, r0, r1, nullptr, ms, stopped, &slot, st)))
        return rc2;
      if ((rc2 = launch_reg_tier<2>(p, 1, ghat_rev, r0, r1, ms, ms + 1, stopped, &slot, st)))
        return rc2;
      if ((rc2 = launch_reg_tier<4>(p, 2, ghat_rev, r0, r1, ms + 1, ms + 2, stopped, &slot, st)))
        return rc2;
    }
    lim = p->mstar + kPruneTiers - 1;
  }
  int64_t first_row = r0;
  if (read_lim) {
    // the tier kernels are already queued: the device stays busy while the
    // host waits for the pruning test only
    CU(cudaEventSynchronize(p->lim_ev));
    first_row = std::max<int64_t>(r0, std::min<int64_t>(r1, *p->lim_host));
  }
  for (int64_t b = r0; b < r1; b += p->big_rows) {
    const int64_t rows = std::min<int64_t>(p->big_rows, r1 - b);
    if (b + rows <= first_row) continue;  // every row of the batch is on chip
    if (!(kBigSkip & 1) &&
        (rc = big_launch_a(p, true, 0, ghat_rev, nullptr, b, rows, stopped, st, lim)))
      return rc;
    if (kBigSkip & 2) continue;
    if ((rc = big_launch_cols(p, true, fout ? 2 : 1, 0, b, rows,
                              fout ? fout + (size_t)(b - r0) * p->n : nullptr, stopped, st, lim)))
      return rc;
  }
  return 0;
}

// One signal's transform: out_mode 3 (natural) or 4 (bit-reversed).
int big_fft(afd_plan* p, const double2* x, double2* out, bool inv, int scale_n, int out_mode,
            const int* stopped, cudaStream_t st) {
  int rc;
  if ((rc = big_launch_a(p, inv, 1, nullptr, x, 0, 1, stopped, st))) return rc;
  return big_launch_cols(p, inv, out_mode, scale_n, 0, 1, out, stopped, st);
}

int big_nnodes(const afd_plan* p) { return (int)(p->n / kNodeLen); }

// init (k < 0) or one step of signal `sig`; cands == null uses the local field.
int big_step(afd_plan* p, int sig, int k, int max_terms, double thr, int dc_first,
             const double2* g0, const Cand* cands, int ncand, Step* steps, cudaStream_t st) {
  int rc;
  const size_t N = (size_t)p->n;
  double2* rem = p->rem + sig * N;
  double2* ghat_rev = p->ghat + sig * N;
  State* state = p->state + sig;
  const int* stopped = &state->stopped;
  const int nn = big_nnodes(p);
  if (k < 0) {
    big_update_kernel<<<nn, 256, 0, st>>>(p->K, nullptr, g0, rem, p->circle, state, p->nodes,
                                          nullptr, nullptr);
    big_finalize_kernel<<<1, 256, 0, st>>>(-1, p->K, max_terms, thr, p->nodes, nn, nullptr,
                                           nullptr, state, nullptr);
    p->launches += 2;
    CU(cudaGetLastError());
    return big_fft(p, rem, ghat_rev, false, 0, 4, stopped, st);
  }
  if (k == 0 && dc_first) {
    node_sums_kernel<<<nn, 256, 0, st>>>(1, rem, p->nodes);
    big_select_kernel<<<1, 256, 0, st>>>(k, dc_first, p->K, nullptr, 0, p->nodes, nn, p->radii,
                                         p->circle, state, p->sel);
    p->launches += 2;
  } else {
    if (!cands) {
      if ((rc = big_field(p, ghat_rev, p->m0, p->m1, nullptr, stopped, st))) return rc;
      if ((rc = big_reduce_cands(p, st, &cands, &ncand))) return rc;
    }
    // runner-ups only for the plan's own field (not all-gathered shards)
    big_select_kernel<<<1, 256, 0, st>>>(k, dc_first, p->K, cands, ncand, nullptr, 0, p->radii,
                                         p->circle, state, p->sel,
                                         cands == p->big_part ? p->big_part2 : nullptr);
    p->launches++;
  }
  big_update_kernel<<<nn, 256, 0, st>>>(p->K, p->sel, nullptr, rem, p->circle, state, p->nodes,
                                        p->amb, p->pow2);
  big_finalize_kernel<<<1, 256, 0, st>>>(k, p->K, max_terms, thr, p->nodes, nn, p->sel, p->amb,
                                         state, steps + (size_t)sig * max_terms);
  p->launches += 2;
  CU(cudaGetLastError());
  return big_fft(p, rem, ghat_rev, false, 0, 4, stopped, st);
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the single-GPU library has no NCCL dependency):
// the process's already-loaded libnccl.so.2 (e.g. torch's) if there is one,
// else the system's.  Only the five entry points the sharded loop needs.
// ---------------------------------------------------------------------------
struct Nccl {
  bool ok = false;
  std::string err;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.err = std::string("libnccl.so.2 not found: ") + dlerror();
      return x;
    }
    x.getUniqueId = (decltype(x.getUniqueId))dlsym(h, "ncclGetUniqueId");
    x.commInitRank = (decltype(x.commInitRank))dlsym(h, "ncclCommInitRank");
    x.commDestroy = (decltype(x.commDestroy))dlsym(h, "ncclCommDestroy");
    x.allGather = (decltype(x.allGather))dlsym(h, "ncclAllGather");
    x.getErrorString = (decltype(x.getErrorString))dlsym(h, "ncclGetErrorString");
    x.ok = x.getUniqueId && x.commInitRank && x.commDestroy && x.allGather && x.getErrorString;
    if (!x.ok) x.err = "libnccl.so.2 lacks a required symbol";
    return x;
  }();
  return n;
}

#define NC(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return fail(AFD_E_CUDA, "%s: %s", #call, nccl().getErrorString(r_));              \
  } while (0)

// [world][batch] candidates (all-gather order) -> [batch][world] (rank-major
// per signal: the step kernels' merge keeps the lowest flat index on ties)
__global__ void cand_transpose_kernel(const Cand* __restrict__ in, int world, int batch,
                                      Cand* __restrict__ out) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < world * batch;
       x += gridDim.x * blockDim.x) {
    const int r = x / batch, b = x % batch;
    out[(size_t)b * world + r] = in[x];
  }
}

}  // namespace

struct afd_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
};

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* afd_last_error(void) { return g_err.c_str(); }

int afd_version(void) { return 1; }

int afd_plan_create(afd_plan** out, int device, int64_t n, int64_t m, int64_t m0, int64_t m1,
                    int64_t max_batch, const double* radii_host, const double* scales_host,
                    const double* twiddle_host, const double* circle_host, int flags) {
  if (!out) return fail(AFD_E_INVALID, "out is NULL");
  *out = nullptr;
  if (n < 8 || (n & (n - 1)))
    return fail(AFD_E_INVALID, "signal length must be a power of two >= 8, got %lld",
                (long long)n);
  int K = 0;
  while ((1LL << K) < n) ++K;
  if (K < kMinK || K > kMaxK)
    return fail(AFD_E_UNSUPPORTED, "transform length 2^%d not supported (max 2^%d)", K, kMaxK);
  if (m < 1) return fail(AFD_E_INVALID, "grid needs at least one radius");
  if (m0 < 0 || m1 > m || m0 >= m1) return fail(AFD_E_INVALID, "bad radius shard [%lld, %lld)",
                                                (long long)m0, (long long)m1);
  if (max_batch < 1) return fail(AFD_E_INVALID, "max_batch must be >= 1");
  if (!radii_host || !scales_host || !twiddle_host || !circle_host)
    return fail(AFD_E_INVALID, "NULL host table");
  if (flags & ~(AFD_PLAN_FAST | AFD_PLAN_MARGINS))
    return fail(AFD_E_INVALID, "unknown plan flags 0x%x", flags);
  if ((flags & AFD_PLAN_MARGINS) && !(flags & AFD_PLAN_FAST))
    return fail(AFD_E_INVALID, "AFD_PLAN_MARGINS needs AFD_PLAN_FAST");
  if ((flags & AFD_PLAN_FAST) && K > kMaxOnChipK && K != 16 && K != 20)
    return fail(AFD_E_UNSUPPORTED, "fast mode for N = 2^%d not built (2^3..2^13, 2^16, 2^20)", K);
  for (int64_t i = 0; i < m; ++i) {
    if (!(radii_host[i] >= 0.0 && radii_host[i] < 1.0))
      return fail(AFD_E_INVALID, "grid radii must lie in [0, 1), got %g", radii_host[i]);
  }
  afd_plan* p = new afd_plan();
  p->device = device;
  p->K = K;
  p->n = n;
  p->m = m;
  p->m0 = m0;
  p->m1 = m1;
  p->max_batch = max_batch;
  p->fast = (flags & AFD_PLAN_FAST) != 0;
  p->margins = (flags & AFD_PLAN_MARGINS) != 0;
  auto cleanup = [&](int rc) {
    afd_plan_destroy(p);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) return cleanup(fail(AFD_E_CUDA, "cudaSetDevice(%d)", device));
  cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
  const size_t N = (size_t)n;
  // stage twiddle tables S_b[k] = w[k << (K-1-b)], offset 2^b - 1
  std::vector<double2> st(N - 1);
  for (int b = 0; b < K; ++b)
    for (int64_t k = 0; k < (1LL << b); ++k) {
      const int64_t idx = k << (K - 1 - b);
      st[(1LL << b) - 1 + k] = make_double2(twiddle_host[2 * idx], twiddle_host[2 * idx + 1]);
    }
#define ALLOC(ptr, bytes)                                                          \
  do {                                                                             \
    if (cudaMalloc(&(ptr), (bytes)) != cudaSuccess)                                \
      return cleanup(fail(AFD_E_NOMEM, "cudaMalloc(%zu) failed", (size_t)(bytes))); \
  } while (0)
  ALLOC(p->radii, sizeof(double) * m);
  ALLOC(p->pow2, sizeof(double) * kPowRow * m);
  ALLOC(p->scales, sizeof(double) * m);
  ALLOC(p->twst, sizeof(double2) * (N - 1));
  ALLOC(p->circle, sizeof(double2) * N);
  // fast mode: per-row weight factor tables (fast_weight_kernel) instead of
  // the M x N cumprod table
  int fw_sec[3] = {0, 0, 0}, fw_exp[3] = {0, 0, 0};
  if (p->fast) {
    if (K <= kMaxOnChipK) {
      const int rb = K >= 4 ? 4 : K;  // Geo<K, kFieldRB>
      fw_sec[0] = 1 << (K - rb);      // scale r^t, t < T
      fw_sec[1] = 1 << rb;            // r^(T m), m < P
      fw_exp[1] = K - rb;
    } else {
      const int ka = big_ka(K);
      fw_sec[0] = 1 << (K - ka);  // scale r^c, c < N / 2^ka (the block's low bits)
      fw_sec[1] = 1 << (ka - 4);  // r^(t 2^(K-ka)), t < 2^(ka-4)
      fw_exp[1] = K - ka;
      fw_sec[2] = 16;             // r^(m 2^(K-4)), m < 16
      fw_exp[2] = K - 4;
    }
    p->fw_stride = fw_sec[0] + fw_sec[1] + fw_sec[2];
    ALLOC(p->fw, sizeof(double) * (size_t)p->fw_stride * (size_t)(m1 - m0));
    ALLOC(p->twct, sizeof(double2) * (N - 1));
  } else {
    ALLOC(p->pw, sizeof(double) * N * (size_t)(m1 - m0));
    ALLOC(p->pw_len, sizeof(int) * (size_t)(m1 - m0));
  }
  ALLOC(p->ghat, sizeof(double2) * N * max_batch);
  ALLOC(p->rem, sizeof(double2) * N * max_batch);
  ALLOC(p->gin, sizeof(double2) * N * max_batch);
  ALLOC(p->state, sizeof(State) * max_batch);
  ALLOC(p->row_ctr, sizeof(unsigned) * 2 * max_batch);
#undef ALLOC
#define ALLOC2(ptr, bytes)                                                         \
  do {                                                                             \
    if (cudaMalloc(&(ptr), (bytes)) != cudaSuccess)                                \
      return cleanup(fail(AFD_E_NOMEM, "cudaMalloc(%zu) failed", (size_t)(bytes))); \
  } while (0)
  {
    // CPython's abs(a) ** 2 (core.py:237) is libm pow(h, 2.0): tabulated here
    // with the host's own libm for the doubles h within kPowWin ulps of each
    // radius (kernel_norm_grid).  The exponent goes through a volatile so the
    // compiler cannot fold pow(h, 2.0) into h * h.
    volatile double two = 2.0;
    std::vector<double> pw2((size_t)kPowRow * m);
    for (int64_t i = 0; i < m; ++i) {
      const int64_t rb = (int64_t)__builtin_bit_cast(uint64_t, radii_host[i]);
      for (int d = 0; d < kPowRow; ++d) {
        const int64_t hb = rb + d - kPowWin;
        pw2[(size_t)i * kPowRow + d] =
            hb >= 0 ? std::pow(__builtin_bit_cast(double, (uint64_t)hb), (double)two) : 0.0;
      }
    }
    if (cudaMemcpy(p->pow2, pw2.data(), sizeof(double) * pw2.size(), cudaMemcpyHostToDevice) !=
        cudaSuccess)
      return cleanup(fail(AFD_E_CUDA, "table upload failed"));
  }
  if (cudaMemcpy(p->radii, radii_host, sizeof(double) * m, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->scales, scales_host, sizeof(double) * m, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->twst, st.data(), sizeof(double2) * (N - 1), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->circle, circle_host, sizeof(double2) * N, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(p->state, 0, sizeof(State) * max_batch) != cudaSuccess)
    return cleanup(fail(AFD_E_CUDA, "table upload failed"));
  if (p->fast) {
    // (c, t) of the conjugated stage twiddles W = conj(w) = c (1 + i t),
    // c = Re W, t = Im W / Re W (numpy's table never has Re W == 0 exactly:
    // W_4 = 6.12e-17 + 1j keeps t finite; guarded anyway)
    std::vector<double2> ct(N - 1);
    for (size_t i = 0; i < N - 1; ++i) {
      const double wr = st[i].x, wi = -st[i].y;
      const double c = wr != 0.0 ? wr : 0x1p-60;
      ct[i] = make_double2(c, wi / c);
    }
    if (cudaMemcpy(p->twct, ct.data(), sizeof(double2) * (N - 1), cudaMemcpyHostToDevice) !=
        cudaSuccess)
      return cleanup(fail(AFD_E_CUDA, "table upload failed"));
    const int64_t rows = m1 - m0;
    const int64_t total = rows * p->fw_stride;
    fast_weight_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256>>>(
        p->radii, p->scales, m0, rows, p->fw_stride, fw_sec[0], fw_sec[1], fw_exp[1], fw_sec[2],
        fw_exp[2], p->fw);
    p->launches++;
    if (cudaGetLastError() != cudaSuccess) return cleanup(fail(AFD_E_CUDA, "weight table launch"));
  } else {
    // r^l power rows (np.cumprod, transform.py:147-150), once per plan
    const int64_t rows = m1 - m0;
    power_table_kernel<<<(unsigned)((rows + 31) / 32), 32>>>(p->radii, m0, m1, n, p->pw,
                                                             p->pw_len);
    p->launches++;
    if (cudaGetLastError() != cudaSuccess) return cleanup(fail(AFD_E_CUDA, "power table launch"));
  }
  int rc = 0;
  if (K > kMaxOnChipK) {
    // large N: bit-reversed power rows (transform.py:151) and batch buffers
    p->big = true;
    p->ka = big_ka(K);
    if (!p->fast) {
      bitrev_rows_kernel<<<dim3(1u << (K - 10), (unsigned)(m1 - m0)), dim3(32, 32)>>>(p->pw, K);
      perm_blocks_kernel<<<dim3(1u << (K - p->ka), (unsigned)(m1 - m0)), 256,
                           sizeof(double) << p->ka>>>(p->pw, K, p->ka);
      p->launches += 2;
      if (cudaGetLastError() != cudaSuccess) return cleanup(fail(AFD_E_CUDA, "bitrev launch"));
    }
    {
      // Rows per batch: all of them if kBigBatchBytes allows, else as many as
      // it allows rounded down to a whole number of pass-A rounds.
      const int64_t cap = std::max<int64_t>(1, (int64_t)(kBigBatchBytes / (N * 16)));
      const int64_t nblk = N >> p->ka, slots = 2LL * p->sms;
      int64_t rows = cap;
      if (m1 - m0 <= cap) {
        rows = m1 - m0;  // one batch: no per-batch launch tails at all
      } else {
        for (int64_t r = cap; r >= std::max<int64_t>(1, cap / 2); --r)
          if ((r * nblk) % slots == 0) {
            rows = r;
            break;
          }
      }
      if (const char* e = getenv("AFD_BIG_ROWS")) rows = atoll(e);  // experiments
      p->big_rows = std::max<int64_t>(1, std::min<int64_t>(m1 - m0, rows));
    }
    ALLOC2(p->Y, sizeof(double2) * N * p->big_rows);
    ALLOC2(p->big_cand, sizeof(Cand) * p->big_rows * big_col_ctas(p));
    ALLOC2(p->big_part, sizeof(Cand) * kBigParts);
    if (p->margins) {
      ALLOC2(p->big_cand2, sizeof(double) * p->big_rows * big_col_ctas(p));
      ALLOC2(p->big_part2, sizeof(double) * kBigParts);
    }
    ALLOC2(p->nodes, sizeof(double) * 2 * (N / kNodeLen));
    ALLOC2(p->sel, sizeof(BigSel));
    ALLOC2(p->amb, sizeof(int));
    ALLOC2(p->tmp, sizeof(double2) * N);
    rc = big_setup(p);
    if (!rc && p->fast && kPrunedEnabled && K > kPruneK && pruned_col_ok(p)) {
      // pruned fast field, per tier: weights {scale r^t, t < L/16;
      // r^(L/16 m), m < 16} of this plan's radii and N-point scales, the
      // L-point (c, t) twiddle image (the stage tables S_b, b < log2 L, are
      // the first L - 1 entries of the N-point tables), per-CTA candidates
      ALLOC2(p->mstar, sizeof(int) * kPruneTiers);
      ALLOC2(p->tmax, sizeof(unsigned long long));
      if (cudaHostAlloc(&p->lim_host, sizeof(int), cudaHostAllocDefault) != cudaSuccess ||
          cudaEventCreateWithFlags(&p->lim_ev, cudaEventDisableTiming) != cudaSuccess)
        return cleanup(fail(AFD_E_CUDA, "plan init: limit readback"));
      ALLOC2(p->hint, sizeof(unsigned long long));
      for (int t = 0; t < kPruneTiers; ++t) p->tier_on[t] = t < kRegTiers ? kRegTiersOn != 0 : true;
      choose_sub_tiers(p, radii_host, 1);
      p->first_tier = 0;
      while (!p->tier_on[p->first_tier]) ++p->first_tier;
      rc = setup_pruned_tier<prune_k(kTier1k)>(p, kTier1k);
      if (!rc) rc = setup_pruned_tier<prune_k(kTier4k)>(p, kTier4k);
      if (!rc && p->tier_on[kTierSub]) rc = setup_sub_tier<8>(p, kTierSub);
      if (!rc && p->tier_on[kTierSub + 1]) rc = setup_sub_tier<9>(p, kTierSub + 1);
      for (int t = 0; t < kRegTiers && !rc && p->tier_on[t]; ++t) rc = setup_reg_tier(p, t);
      if (!rc) rc = reg_kernel_attrs();
      if (rc) return cleanup(rc);
      p->pruned = true;
    }
  } else {
    AFD_DISPATCH(K, { rc = setup_kernels<KK>(p); break; });
    const int64_t rows = m1 - m0;
    if (!rc && p->fast && p->engine == 0 && kSmallPrunedOn && K >= 10 && max_batch >= 8 &&
        max_batch * rows * N >= (size_t)kSmallPrunedMinEvals) {
      // register tiers for batches (pruned_small)
      ALLOC2(p->sp_fw, sizeof(double) * kFwStride * (size_t)rows);
      ALLOC2(p->sp_mstar, sizeof(int) * kSmallTiers * (size_t)max_batch);
      for (int t = 0; t < kPruneTiers; ++t)
        p->tier_on[t] = t < kRegTiers || (K >= 12 && kSmallWarpTier && t == kTier1k);
      choose_sub_tiers(p, radii_host, max_batch);
      {
        for (int u = 0; u < 2; ++u) {
          if (!p->tier_on[kTierSub + u]) continue;
          const int T = 8 << u, stride = T + 32;
          ALLOC2(p->sp_gsub[u], sizeof(double2) * N * (size_t)max_batch);
          ALLOC2(p->sp_fwsub[u], sizeof(double) * stride * (size_t)rows);
          const int64_t tot = rows * stride;
          fast_weight_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 65535), 256>>>(
              p->radii, p->scales, p->m0, rows, stride, T, 32, 3 + u, 0, 0, p->sp_fwsub[u]);
          p->launches++;
        }
        CU(cudaFuncSetAttribute(field_sub_kernel<8, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SubGeo<8>::kSmem));
        CU(cudaFuncSetAttribute(field_sub_kernel<8, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SubGeo<8>::kSmem));
        CU(cudaFuncSetAttribute(field_sub_kernel<9, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SubGeo<9>::kSmem));
        CU(cudaFuncSetAttribute(field_sub_kernel<9, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SubGeo<9>::kSmem));
      }
      if (K >= 12 && kSmallWarpTier) {
        ALLOC2(p->sp_g1k, sizeof(double2) * N * (size_t)max_batch);
        CU(cudaFuncSetAttribute(field_warp_kernel<false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwSmem));
        CU(cudaFuncSetAttribute(field_warp_kernel<true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFwSmem));
      }
      ALLOC2(p->sp_hint, sizeof(unsigned long long) * (size_t)max_batch);
      ALLOC2(p->sp_h, sizeof(double2) * 128 * (N >> 5) * (size_t)max_batch);
      ALLOC2(p->sp_rlog, sizeof(double2) * (size_t)rows);
      {
        std::vector<double2> rl((size_t)rows);
        for (int64_t s = 0; s < rows; ++s) {
          const double r = radii_host[m0 + s];
          rl[s] = make_double2(r > 0.0 ? std::log2(r) : -INFINITY, std::log2(1.0 - r));
        }
        if (cudaMemcpy(p->sp_rlog, rl.data(), sizeof(double2) * rl.size(),
                       cudaMemcpyHostToDevice) != cudaSuccess)
          return cleanup(fail(AFD_E_CUDA, "plan init: rlog upload"));
      }
      const int64_t total = rows * kFwStride;
      fast_weight_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256>>>(
          p->radii, p->scales, p->m0, rows, kFwStride, 32, 32, 5, 0, 0, p->sp_fw);
      p->launches++;
      p->first_tier = 0;
      if ((rc = reg_kernel_attrs())) return cleanup(rc);
      p->sp = true;
    }
  }
  if (rc) return cleanup(rc);
  if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(AFD_E_CUDA, "plan init: %s",
                                                                  cudaGetErrorString(cudaGetLastError())));
  *out = p;
  return AFD_OK;
}

int afd_plan_destroy(afd_plan* p) {
  if (!p) return AFD_OK;
  cudaSetDevice(p->device);
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  if (p->sgexec) cudaGraphExecDestroy(p->sgexec);
  cudaFree(p->loc_cand);
  cudaFree(p->gath_cand);
  cudaFree(p->gath_t);
  cudaFree(p->radii);
  cudaFree(p->pow2);
  cudaFree(p->scales);
  cudaFree(p->twst);
  cudaFree(p->circle);
  cudaFree(p->pw);
  cudaFree(p->tw_img);
  cudaFree(p->twct);
  cudaFree(p->tw_img_ct);
  cudaFree(p->fw);
  cudaFree(p->ghat);
  cudaFree(p->rem);
  cudaFree(p->gin);
  cudaFree(p->state);
  cudaFree(p->cand);
  cudaFree(p->steps);
  cudaFree(p->row_ctr);
  cudaFree(p->pw_len);
  cudaFree(p->scratch);
  cudaFree(p->Y);
  cudaFree(p->big_cand);
  for (auto& t : p->tier) {
    cudaFree(t.fw);
    cudaFree(t.ghq);
    cudaFree(t.tw_img);
    cudaFree(t.cand);
    cudaFree(t.cand2);
  }
  cudaFree(p->big_cand2);
  cudaFree(p->big_part2);
  cudaFree(p->cand2);
  cudaFree(p->mstar);
  cudaFree(p->tmax);
  if (p->lim_host) cudaFreeHost(p->lim_host);
  if (p->lim_ev) cudaEventDestroy(p->lim_ev);
  cudaFree(p->hint);
  cudaFree(p->sp_fw);
  cudaFree(p->sp_mstar);
  cudaFree(p->sp_hint);
  cudaFree(p->sp_h);
  cudaFree(p->sp_rlog);
  cudaFree(p->sp_g1k);
  for (int u = 0; u < 2; ++u) {
    cudaFree(p->sp_gsub[u]);
    cudaFree(p->sp_fwsub[u]);
  }
  cudaFree(p->big_part);
  cudaFree(p->nodes);
  cudaFree(p->sel);
  cudaFree(p->amb);
  cudaFree(p->tmp);
  cudaFree(p->packed);
  if (p->pin) cudaFreeHost(p->pin);
  delete p;
  return AFD_OK;
}

static int fft_entry(afd_plan* p, int mode, const double* x, double* out, int64_t batch,
                     void* stream) {
  if (!p || !x || !out) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->big) {
    const size_t N = (size_t)p->n;
    for (int64_t b = 0; b < batch; ++b) {
      const double2* xb = (const double2*)x + b * N;
      double2* ob = (double2*)out + b * N;
      if (mode == 0) {
        if ((rc = big_fft(p, xb, ob, false, 0, 3, nullptr, st))) return rc;
      } else if (mode == 1) {
        if ((rc = big_fft(p, xb, ob, true, 1, 3, nullptr, st))) return rc;
      } else {
        // core.py:224-231: forward, fold the spectrum one-sided, 1/N inverse
        if ((rc = big_fft(p, xb, p->tmp, false, 0, 3, nullptr, st))) return rc;
        analytic_mask_kernel<<<256, 256, 0, st>>>(p->K, p->tmp);
        p->launches++;
        if ((rc = big_fft(p, p->tmp, ob, true, 1, 3, nullptr, st))) return rc;
      }
    }
    return 0;
  }
  AFD_DISPATCH(p->K, return launch_fft<KK>(p, mode, (const double2*)x, (double2*)out, batch, st));
}

int afd_dft_forward(afd_plan* p, const double* x, double* out, int64_t batch, void* stream) {
  return fft_entry(p, 0, x, out, batch, stream);
}
int afd_dft_inverse(afd_plan* p, const double* c, double* out, int64_t batch, void* stream) {
  return fft_entry(p, 1, c, out, batch, stream);
}
int afd_analytic_projection(afd_plan* p, const double* x, double* out, int64_t batch,
                            void* stream) {
  return fft_entry(p, 2, x, out, batch, stream);
}

int afd_field(afd_plan* p, const double* ghat, double* field, int64_t r0, int64_t r1,
              void* stream) {
  if (!p || !ghat || !field) return fail(AFD_E_INVALID, "NULL argument");
  if (r0 < p->m0 || r1 > p->m1 || r0 >= r1)
    return fail(AFD_E_INVALID, "rows [%lld, %lld) outside the plan's [%lld, %lld)",
                (long long)r0, (long long)r1, (long long)p->m0, (long long)p->m1);
  int rc;
  if ((rc = set_device(p))) return rc;
  if (p->big) {
    // the large-N field kernels read the spectrum bit-reversed
    cudaStream_t st = (cudaStream_t)stream;
    bitrev_copy_kernel<<<256, 256, 0, st>>>(p->K, p->ka, (const double2*)ghat, p->tmp);
    p->launches++;
    return big_field(p, p->tmp, r0, r1, (double2*)field, nullptr, st);
  }
  const int ncta = field_ctas_for(p, r1 - r0, 1);
  AFD_DISPATCH(p->K, return launch_field<KK>(p, (const double2*)ghat, r0, r1, 1, nullptr, ncta,
                                             (double2*)field, nullptr, (cudaStream_t)stream));
}

int afd_field_direct(afd_plan* p, const double* g, double* field, int64_t r0, int64_t r1,
                     void* stream) {
  if (!p || !g || !field) return fail(AFD_E_INVALID, "NULL argument");
  if (p->big) return fail(AFD_E_UNSUPPORTED, "direct engine supports N <= 8192");
  if (r0 < p->m0 || r1 > p->m1 || r0 >= r1)
    return fail(AFD_E_INVALID, "rows [%lld, %lld) outside the plan's [%lld, %lld)",
                (long long)r0, (long long)r1, (long long)p->m0, (long long)p->m1);
  int rc;
  if ((rc = set_device(p))) return rc;
  return launch_direct(p, (const double2*)g, r0, r1, 1, nullptr, (double2*)field, nullptr,
                       (cudaStream_t)stream);
}

int afd_plan_set_engine(afd_plan* p, int engine) {
  if (!p) return fail(AFD_E_INVALID, "NULL plan");
  if (engine != 0 && engine != 1) return fail(AFD_E_INVALID, "engine must be 0 (fft) or 1 (direct)");
  if (engine == 1 && p->big) return fail(AFD_E_UNSUPPORTED, "direct engine supports N <= 8192");
  if (engine != p->engine) invalidate_graph(p);
  p->engine = engine;
  return 0;
}

int afd_field_argmax(afd_plan* p, const double* ghat, afd_candidate* out, int64_t batch,
                     void* stream) {
  if (!p || !ghat || !out) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->big) {
    for (int64_t b = 0; b < batch; ++b) {
      bitrev_copy_kernel<<<256, 256, 0, st>>>(p->K, p->ka, (const double2*)ghat + b * p->n,
                                              p->tmp);
      p->launches++;
      if ((rc = big_field(p, p->tmp, p->m0, p->m1, nullptr, nullptr, st))) return rc;
      const Cand* parts;
      int np;
      if ((rc = big_reduce_cands(p, st, &parts, &np))) return rc;
      cand_reduce_kernel<<<1, 256, 0, st>>>(parts, np, (Cand*)out + b);
      p->launches++;
    }
    CU(cudaGetLastError());
    return 0;
  }
  const int ncta = field_ctas_for(p, p->m1 - p->m0, batch);
  const SmallGrid sg = small_grid(p, batch, ncta);
  if ((rc = ensure_cand(p, batch, sg.ncand))) return rc;
  AFD_DISPATCH(p->K, {
    if (sg.pruned)
      rc = launch_field_small_pruned<KK>(p, (const double2*)ghat, batch, p->cand, sg, nullptr, st);
    else
      rc = launch_field<KK>(p, (const double2*)ghat, p->m0, p->m1, batch, p->cand, ncta, nullptr,
                            nullptr, st);
    if (rc) return rc;
    break;
  });
  cand_reduce_kernel<<<(unsigned)batch, 128, 0, st>>>(p->cand, sg.ncand, (Cand*)out);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

int afd_argmax(afd_plan* p, const double* field, int64_t rows, afd_candidate* out, void* stream) {
  if (!p || !field || !out) return fail(AFD_E_INVALID, "NULL argument");
  if (rows < 1) return fail(AFD_E_INVALID, "empty field");
  int rc;
  if ((rc = set_device(p))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const long long total = rows * p->n;
  int nblk = (int)std::min<long long>((total + 255) / 256, (long long)p->sms * 8);
  if ((rc = ensure_scratch(p, sizeof(Cand) * nblk))) return rc;
  argmax_kernel<<<nblk, 256, 0, st>>>((const double2*)field, total, (Cand*)p->scratch);
  cand_reduce_kernel<<<1, 256, 0, st>>>((const Cand*)p->scratch, nblk, (Cand*)out);
  p->launches += 2;
  CU(cudaGetLastError());
  return 0;
}

int afd_atom(afd_plan* p, int kind, const double* g, double a_re, double a_im, double c_re,
             double c_im, double norm, double* out, void* stream) {
  if (!p || !out || (kind == 2 && !g)) return fail(AFD_E_INVALID, "NULL argument");
  if (kind < 0 || kind > 3) return fail(AFD_E_INVALID, "bad atom kind %d", kind);
  if (kind == 3 && !g) return fail(AFD_E_INVALID, "NULL argument");
  if (!(a_re * a_re + a_im * a_im < 1.0))
    return fail(AFD_E_INVALID, "pole must lie strictly inside the unit disc");
  int rc;
  if ((rc = set_device(p))) return rc;
  const int n = (int)p->n;
  atom_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      kind, n, (const double2*)g, make_double2(a_re, a_im), make_double2(c_re, c_im), p->circle,
      (double2*)out, norm);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

int afd_energy(afd_plan* p, const double* g, double* energies, int64_t batch, void* stream) {
  return afd_energy_diff(p, g, nullptr, energies, batch, stream);
}

int afd_energy_diff(afd_plan* p, const double* g, const double* s, double* energies,
                    int64_t batch, void* stream) {
  if (!p || !g || !energies) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = set_device(p))) return rc;
  const size_t per = (size_t)p->n + 2 * ((size_t)p->n / 8 + 16);
  if ((rc = ensure_scratch(p, sizeof(double) * per * batch))) return rc;
  energy_kernel<<<(unsigned)batch, 256, 0, (cudaStream_t)stream>>>(
      (int)p->n, (const double2*)g, (const double2*)s, p->scratch, energies);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

int afd_decompose(afd_plan* p, const double* g0, int64_t batch, int max_terms, double threshold,
                  int dc_first, afd_step* steps, int32_t* n_steps, double* initial,
                  double* remainder, void* stream) {
  if (!p || !g0 || !steps || !n_steps || !initial || !remainder)
    return fail(AFD_E_INVALID, "NULL argument");
  if (max_terms < 1) return fail(AFD_E_INVALID, "max_terms must be >= 1");
  if (p->m0 != 0 || p->m1 != p->m)
    return fail(AFD_E_INVALID, "afd_decompose needs an unsharded plan (use the step API)");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  if ((rc = ensure_steps(p, max_terms))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const double thr = threshold > 0.0 ? threshold : 0.0;
  const size_t sig_bytes = sizeof(double2) * (size_t)p->n * batch;
  if ((const void*)g0 != (const void*)p->gin)
    CU(cudaMemcpyAsync(p->gin, g0, sig_bytes, cudaMemcpyDeviceToDevice, st));
  if (p->big) {
    // large N: host-driven loop (each step is dominated by ~M*N/4096-CTA
    // field launches; a graph would only add instantiation cost)
    for (int64_t b = 0; b < batch; ++b) {
      if ((rc = big_step(p, (int)b, -1, max_terms, thr, dc_first, p->gin + b * p->n, nullptr, 0,
                         p->steps, st)))
        return rc;
      for (int k = 0; k < max_terms; ++k)
        if ((rc = big_step(p, (int)b, k, max_terms, thr, dc_first, nullptr, nullptr, 0, p->steps,
                           st)))
          return rc;
    }
    gather_outputs_kernel<<<(unsigned)batch, 256, 0, st>>>(
        (int)p->n, max_terms, p->steps, p->state, p->rem, (Step*)steps, n_steps, initial,
        (double2*)remainder, nullptr);
    p->launches++;
    CU(cudaGetLastError());
    return 0;
  }
  const bool reuse = p->gexec && p->g_max_terms == max_terms && p->g_dc_first == dc_first &&
                     p->g_threshold == thr && p->g_batch == batch && p->g_stream == st;
  if (!reuse) {
    invalidate_graph(p);
    // make sure buffers exist before capture (allocation is not capturable)
    const int ncta = small_grid(p, batch, decomp_field_ctas(p, batch)).ncand;
    if ((rc = ensure_cand(p, batch, ncta))) return rc;
    cudaStream_t cap;
    CU(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t graph;
    const int64_t before = p->launches;
    CU(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_decompose(p, batch, max_terms, thr, dc_first, cap);
    cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    cudaStreamDestroy(cap);
    if (rc) return rc;
    if (ce != cudaSuccess) return fail(AFD_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    p->graph_launches_per_replay = p->launches - before;
    p->launches = before;
    ce = cudaGraphInstantiate(&p->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return fail(AFD_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    p->g_max_terms = max_terms;
    p->g_dc_first = dc_first;
    p->g_threshold = thr;
    p->g_batch = batch;
    p->g_stream = st;
  }
  CU(cudaGraphLaunch(p->gexec, st));
  p->launches += p->graph_launches_per_replay;
  // outputs
  gather_outputs_kernel<<<(unsigned)batch, 256, 0, st>>>(
      (int)p->n, max_terms, p->steps, p->state, p->rem, (Step*)steps, n_steps, initial,
      (double2*)remainder, nullptr);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

// Host memcpy on up to 8 threads for large buffers (the pinned staging copies
// of a batch run at one core's bandwidth otherwise: 64 MiB ~6 ms).
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kMin = (size_t)8 << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::min<size_t>(std::min(8u, hw), bytes / kMin);
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = ((bytes + nt - 1) / nt + 63) & ~(size_t)63;
  std::vector<std::thread> th;
  for (int i = 1; i < nt; ++i) {
    const size_t o = per * i;
    if (o >= bytes) break;
    th.emplace_back([=] { std::memcpy((char*)dst + o, (const char*)src + o, std::min(per, bytes - o)); });
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

int afd_decompose_host(afd_plan* p, const double* g0_host, int64_t batch, int max_terms,
                       double threshold, int dc_first, afd_step* steps_host,
                       int32_t* n_steps_host, double* initial_host, double* remainder_host,
                       int64_t* h2d_bytes, int64_t* d2h_bytes, void* stream) {
  if (!p || !g0_host || !steps_host || !n_steps_host || !initial_host || !remainder_host)
    return fail(AFD_E_INVALID, "NULL argument");
  if (max_terms < 1) return fail(AFD_E_INVALID, "max_terms must be >= 1");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t sig = sizeof(double2) * (size_t)p->n * batch;
  const size_t stp = sizeof(Step) * (size_t)max_terms * batch;
  // packed layout: steps | n_steps | initial | remainder, each part 16-byte
  // aligned (afd_step is 72 bytes; the remainder is read as double2)
  auto al16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t o_ns = al16(stp), o_in = al16(o_ns + sizeof(int32_t) * batch);
  const size_t o_rm = al16(o_in + sizeof(double) * batch);
  const size_t need_pack = o_rm + sig;
  if (need_pack > p->packed_bytes) {
    cudaFree(p->packed);
    p->packed = nullptr;
    p->packed_bytes = 0;
    CU(cudaMalloc(&p->packed, need_pack));
    p->packed_bytes = need_pack;
  }
  const size_t need_pin = std::max(sig, need_pack);
  if (need_pin > p->pin_bytes) {
    if (p->pin) cudaFreeHost(p->pin);
    p->pin = nullptr;
    p->pin_bytes = 0;
    CU(cudaHostAlloc(&p->pin, need_pin, cudaHostAllocDefault));
    p->pin_bytes = need_pin;
  }
  par_memcpy(p->pin, g0_host, sig);
  CU(cudaMemcpyAsync(p->gin, p->pin, sig, cudaMemcpyHostToDevice, st));
  unsigned char* d = p->packed;
  if ((rc = afd_decompose(p, (const double*)p->gin, batch, max_terms, threshold, dc_first,
                          (afd_step*)d, (int32_t*)(d + o_ns), (double*)(d + o_in),
                          (double*)(d + o_rm), stream)))
    return rc;
  CU(cudaMemcpyAsync(p->pin, d, need_pack, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  const unsigned char* hp = (const unsigned char*)p->pin;
  std::memcpy(steps_host, hp, stp);
  std::memcpy(n_steps_host, hp + o_ns, sizeof(int32_t) * batch);
  std::memcpy(initial_host, hp + o_in, sizeof(double) * batch);
  par_memcpy(remainder_host, hp + o_rm, sig);
  if (h2d_bytes) *h2d_bytes = (int64_t)sig;
  if (d2h_bytes) *d2h_bytes = (int64_t)need_pack;
  return 0;
}

static int enqueue_sharded_begin(afd_plan* p, const double* g0, int64_t batch, cudaStream_t st) {
  int rc;
  if ((const void*)g0 != (const void*)p->gin)
    CU(cudaMemcpyAsync(p->gin, g0, sizeof(double2) * (size_t)p->n * batch,
                       cudaMemcpyDeviceToDevice, st));
  if (p->big) {
    for (int64_t b = 0; b < batch; ++b)
      if ((rc = big_step(p, (int)b, -1, 1, 0.0, 0, p->gin + b * p->n, nullptr, 0, p->steps, st)))
        return rc;
    return 0;
  }
  AFD_DISPATCH(p->K, return launch_step<KK>(p, -1, 1, 0.0, 0, p->gin, nullptr, 0, batch, p->steps,
                                            st));
}

// Field + argmax over the plan's rows -> cand[batch] (neutral at a dc_first
// step 0).  ensure_cand must have run (capture cannot allocate).
static int enqueue_select_local(afd_plan* p, int k, int dc_first, Cand* cand, int64_t batch,
                                cudaStream_t st) {
  int rc;
  if (k == 0 && dc_first) {
    // the pinned mean atom needs no field; emit a neutral candidate
    neutral_cand_kernel<<<1, 128, 0, st>>>(cand, (int)batch);
    p->launches++;
    CU(cudaGetLastError());
    return 0;
  }
  if (p->big) {
    for (int64_t b = 0; b < batch; ++b) {
      if ((rc = big_field(p, p->ghat + b * p->n, p->m0, p->m1, nullptr, &p->state[b].stopped, st)))
        return rc;
      const Cand* parts;
      int np;
      if ((rc = big_reduce_cands(p, st, &parts, &np))) return rc;
      cand_reduce_kernel<<<1, 256, 0, st>>>(parts, np, cand + b);
      p->launches++;
    }
    CU(cudaGetLastError());
    return 0;
  }
  const int ncta = field_ctas_for(p, p->m1 - p->m0, batch);
  if (ncta > p->ncand_cap) return fail(AFD_E_INVALID, "candidate buffer not sized");
  if (p->engine == 1) {
    if ((rc = launch_direct(p, p->rem, p->m0, p->m1, batch, p->cand, nullptr, p->state, st)))
      return rc;
  } else {
    AFD_DISPATCH(p->K, {
      if ((rc = launch_field<KK>(p, p->ghat, p->m0, p->m1, batch, p->cand, ncta, nullptr,
                                 p->state, st)))
        return rc;
      break;
    });
  }
  cand_reduce_kernel<<<(unsigned)batch, 128, 0, st>>>(p->cand, ncta, cand);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

static int enqueue_apply_step(afd_plan* p, int k, int max_terms, double thr, int dc_first,
                              const Cand* cands, int ncand, int64_t batch, Step* steps,
                              cudaStream_t st) {
  int rc;
  if (p->big) {
    for (int64_t b = 0; b < batch; ++b)
      if ((rc = big_step(p, (int)b, k, max_terms, thr, dc_first, nullptr, cands + b * ncand,
                         ncand, steps, st)))
        return rc;
    return 0;
  }
  AFD_DISPATCH(p->K, return launch_step<KK>(p, k, max_terms, thr, dc_first, nullptr, cands,
                                            ncand, batch, steps, st));
}

int afd_sharded_begin(afd_plan* p, const double* g0, int64_t batch, void* stream) {
  if (!p || !g0) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  return enqueue_sharded_begin(p, g0, batch, (cudaStream_t)stream);
}

int afd_select_local(afd_plan* p, int k, int dc_first, afd_candidate* cand, int64_t batch,
                     void* stream) {
  if (!p || !cand) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  if (!p->big && !(k == 0 && dc_first) &&
      (rc = ensure_cand(p, batch, field_ctas_for(p, p->m1 - p->m0, batch))))
    return rc;
  return enqueue_select_local(p, k, dc_first, (Cand*)cand, batch, (cudaStream_t)stream);
}

int afd_apply_step(afd_plan* p, int k, int max_terms, double threshold, int dc_first,
                   const afd_candidate* cands, int ncand, int64_t batch, afd_step* steps,
                   void* stream) {
  if (!p || !cands || !steps) return fail(AFD_E_INVALID, "NULL argument");
  if (k < 0 || k >= max_terms) return fail(AFD_E_INVALID, "step %d outside 0..%d", k, max_terms - 1);
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  const double thr = threshold > 0.0 ? threshold : 0.0;
  return enqueue_apply_step(p, k, max_terms, thr, dc_first, (const Cand*)cands, ncand, batch,
                            (Step*)steps, (cudaStream_t)stream);
}

// The radius-sharded loop with its all-gathers: init + max_terms x (local
// field + argmax -> NCCL all-gather of the 32-byte candidates -> replicated
// update), all stream-ordered on st (captured into a graph by the caller).
static int enqueue_decompose_sharded(afd_plan* p, afd_comm* c, int64_t batch, int max_terms, double thr,
                              int dc_first, cudaStream_t st) {
  int rc;
  if ((rc = enqueue_sharded_begin(p, (const double*)p->gin, batch, st))) return rc;
  const size_t bytes = sizeof(Cand) * (size_t)batch;
  for (int k = 0; k < max_terms; ++k) {
    if ((rc = enqueue_select_local(p, k, dc_first, p->loc_cand, batch, st))) return rc;
    NC(nccl().allGather(p->loc_cand, p->gath_cand, bytes, ncclUint8, c->comm, st));
    const Cand* cands = p->gath_cand;
    if (batch > 1 && c->world > 1) {
      cand_transpose_kernel<<<1, 256, 0, st>>>(p->gath_cand, c->world, (int)batch, p->gath_t);
      p->launches++;
      cands = p->gath_t;
    }
    if ((rc = enqueue_apply_step(p, k, max_terms, thr, dc_first, cands, c->world, batch,
                                 p->steps, st)))
      return rc;
  }
  CU(cudaGetLastError());
  return 0;
}

int afd_comm_unique_id(void* id_out) {
  if (!id_out) return fail(AFD_E_INVALID, "NULL argument");
  if (!nccl().ok) return fail(AFD_E_UNSUPPORTED, "%s", nccl().err.c_str());
  ncclUniqueId id;
  NC(nccl().getUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
  return 0;
}

int afd_comm_init(afd_comm** out, const void* id, int world, int rank, int device) {
  if (!out || !id) return fail(AFD_E_INVALID, "NULL argument");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world)
    return fail(AFD_E_INVALID, "rank %d outside world of %d", rank, world);
  if (!nccl().ok) return fail(AFD_E_UNSUPPORTED, "%s", nccl().err.c_str());
  CU(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  afd_comm* c = new afd_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  const ncclResult_t r = nccl().commInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(AFD_E_CUDA, "ncclCommInitRank: %s", nccl().getErrorString(r));
  }
  *out = c;
  return 0;
}

int afd_comm_destroy(afd_comm* c) {
  if (!c) return 0;
  if (c->comm) nccl().commDestroy(c->comm);
  delete c;
  return 0;
}

int afd_decompose_sharded(afd_plan* p, afd_comm* c, const double* g0, int64_t batch,
                          int max_terms, double threshold, int dc_first, afd_step* steps,
                          int32_t* n_steps, double* initial, double* remainder, void* stream) {
  if (!p || !c || !g0 || !steps || !n_steps || !initial || !remainder)
    return fail(AFD_E_INVALID, "NULL argument");
  if (max_terms < 1) return fail(AFD_E_INVALID, "max_terms must be >= 1");
  if (c->device != p->device) return fail(AFD_E_INVALID, "communicator and plan on different devices");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  if ((rc = ensure_steps(p, max_terms))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const double thr = threshold > 0.0 ? threshold : 0.0;
  if (!p->big && (rc = ensure_cand(p, batch, field_ctas_for(p, p->m1 - p->m0, batch)))) return rc;
  if (p->gath_world < c->world) {
    invalidate_graph(p);
    cudaFree(p->loc_cand);
    cudaFree(p->gath_cand);
    cudaFree(p->gath_t);
    p->loc_cand = p->gath_cand = p->gath_t = nullptr;
    p->gath_world = 0;
    CU(cudaMalloc(&p->loc_cand, sizeof(Cand) * (size_t)p->max_batch));
    CU(cudaMalloc(&p->gath_cand, sizeof(Cand) * (size_t)p->max_batch * c->world));
    CU(cudaMalloc(&p->gath_t, sizeof(Cand) * (size_t)p->max_batch * c->world));
    p->gath_world = c->world;
  }
  CU(cudaMemcpyAsync(p->gin, g0, sizeof(double2) * (size_t)p->n * batch, cudaMemcpyDeviceToDevice,
                     st));
  const bool reuse = p->sgexec && p->sg_comm == (const void*)c && p->sg_max_terms == max_terms &&
                     p->sg_dc_first == dc_first && p->sg_threshold == thr &&
                     p->sg_batch == batch && p->sg_stream == st;
  if (!reuse) {
    if (p->sgexec) cudaGraphExecDestroy(p->sgexec);
    p->sgexec = nullptr;
    cudaStream_t cap;
    CU(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t graph;
    const int64_t before = p->launches;
    CU(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_decompose_sharded(p, c, batch, max_terms, thr, dc_first, cap);
    cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    cudaStreamDestroy(cap);
    if (rc) return rc;
    if (ce != cudaSuccess) return fail(AFD_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    p->sgraph_launches = p->launches - before;
    p->launches = before;
    ce = cudaGraphInstantiate(&p->sgexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return fail(AFD_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    p->sg_comm = c;
    p->sg_max_terms = max_terms;
    p->sg_dc_first = dc_first;
    p->sg_threshold = thr;
    p->sg_batch = batch;
    p->sg_stream = st;
  }
  CU(cudaGraphLaunch(p->sgexec, st));
  p->launches += p->sgraph_launches;
  gather_outputs_kernel<<<(unsigned)batch, 256, 0, st>>>(
      (int)p->n, max_terms, p->steps, p->state, p->rem, (Step*)steps, n_steps, initial,
      (double2*)remainder, nullptr);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

int afd_sharded_finish(afd_plan* p, int64_t batch, int32_t* n_steps, double* initial,
                       double* remainder, int32_t* stopped, void* stream) {
  if (!p || !n_steps || !initial || !remainder) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  gather_outputs_kernel<<<(unsigned)batch, 256, 0, (cudaStream_t)stream>>>(
      (int)p->n, 0, nullptr, p->state, p->rem, nullptr, n_steps, initial, (double2*)remainder,
      stopped);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

int afd_error_trace(afd_plan* p, const double* g, const afd_step* steps, int max_terms,
                    const int32_t* n_steps, int64_t batch, const double* norms, double* errors,
                    double* recon, void* stream) {
  if (!p || !g || !steps || !n_steps || !errors) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = set_device(p))) return rc;
  const size_t n = (size_t)p->n;
  const size_t per = 2 * n * 2 + n + 2 * (n / 8 + 16);  // total, bp (complex), mag, scratch
  if ((rc = ensure_scratch(p, sizeof(double) * per * batch))) return rc;
  error_trace_kernel<<<(unsigned)batch, 256, 0, (cudaStream_t)stream>>>(
      (int)n, (const double2*)g, (const Step*)steps, max_terms, n_steps, p->circle, p->scratch,
      errors, (double2*)recon, norms);
  p->launches++;
  CU(cudaGetLastError());
  return 0;
}

int64_t afd_launch_count(afd_plan* p) { return p ? p->launches : 0; }

int afd_time_field(afd_plan* p, const double* ghat, int64_t batch, int reps, double* avg_ms,
                   void* stream) {
  if (!p || !ghat || !avg_ms || reps < 1) return fail(AFD_E_INVALID, "bad argument");
  int rc;
  if ((rc = check_batch(p, batch)) || (rc = set_device(p))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (p->big) {
    // one whole large-N field evaluation (all row batches) per timed rep
    bitrev_copy_kernel<<<256, 256, 0, st>>>(p->K, p->ka, (const double2*)ghat, p->tmp);
    p->launches++;
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    CU(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r)
      if ((rc = big_field(p, p->tmp, p->m0, p->m1, nullptr, nullptr, st))) return rc;
    CU(cudaEventRecord(e1, st));
    CU(cudaEventSynchronize(e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *avg_ms = ms / reps;
    return 0;
  }
  // back-to-back launches (PDL-chained, as inside a decomposition) between
  // two events: the average launch duration in a stream of field launches
  // (the decomposition's launch configuration, dynamic rows included)
  const int ncta = decomp_field_ctas(p, batch);
  const bool dyn = field_dyn_ctas(p, p->m1 - p->m0, batch) > 0;
  const SmallGrid sg = small_grid(p, batch, ncta);
  if ((rc = ensure_cand(p, batch, sg.ncand))) return rc;
  if (dyn) CU(cudaMemsetAsync(p->row_ctr, 0, sizeof(unsigned) * 2 * (size_t)batch, st));
  int launch_id = 0;
  auto one = [&]() -> int {
    AFD_DISPATCH(p->K, {
      if (sg.pruned)
        return launch_field_small_pruned<KK>(p, (const double2*)ghat, batch, p->cand, sg, nullptr,
                                             st);
      return launch_field<KK>(p, (const double2*)ghat, p->m0, p->m1, batch, p->cand, ncta,
                              nullptr, nullptr, st, dyn ? p->row_ctr : nullptr, launch_id++);
    });
    return fail(AFD_E_UNSUPPORTED, "transform length");
  };
  if ((rc = one())) return rc;  // warm
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  CU(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r)
    if ((rc = one())) return rc;
  CU(cudaEventRecord(e1, st));
  CU(cudaEventSynchronize(e1));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *avg_ms = ms / reps;
  return 0;
}

int afd_field_split(afd_plan* p, int64_t* onchip, int64_t* twopass, void* stream) {
  if (!p || !onchip || !twopass) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = set_device(p))) return rc;
  const int64_t rows = p->m1 - p->m0;
  if (!p->big) {
    *onchip = rows;
    *twopass = 0;
    return 0;
  }
  if (!p->pruned) {
    *onchip = 0;
    *twopass = rows;
    return 0;
  }
  int64_t tiers[3];
  int rc2;
  if ((rc2 = afd_field_tiers(p, tiers, stream))) return rc2;
  *onchip = tiers[0] + tiers[1];
  *twopass = tiers[2];
  return 0;
}

int afd_field_tier_rows(afd_plan* p, int64_t* terms, int64_t* rows_out, int cap, int* count,
                        void* stream) {
  if (!p || !terms || !rows_out || !count) return fail(AFD_E_INVALID, "NULL argument");
  int rc;
  if ((rc = set_device(p))) return rc;
  const int64_t rows = p->m1 - p->m0;
  // tiers in use, in row order; an unused tier's rows belong to the next one
  int act[kPruneTiers], na = 0;
  const int tmax = p->big ? kPruneTiers : kSmallTiers;
  for (int t = 0; t < tmax; ++t)
    if (p->tier_on[t]) act[na++] = t;
  auto clampr = [&](int64_t x) { return std::max<int64_t>(0, std::min<int64_t>(rows, x - p->m0)); };
  if (!p->big && p->sp && p->sp_last_batch > 0) {
    // batches of on-chip fields with register tiers: rows summed over the
    // signals of the last evaluation
    if (cap < na + 1)
      return fail(AFD_E_INVALID, "afd_field_tier_rows: cap %d < %d", cap, na + 1);
    std::vector<int> ms((size_t)p->sp_last_batch * kSmallTiers);
    CU(cudaMemcpyAsync(ms.data(), p->sp_mstar, sizeof(int) * ms.size(), cudaMemcpyDeviceToHost,
                       (cudaStream_t)stream));
    CU(cudaStreamSynchronize((cudaStream_t)stream));
    for (int a = 0; a <= na; ++a) {
      terms[a] = a < na ? 1LL << prune_k(act[a]) : p->n;
      rows_out[a] = 0;
    }
    for (int64_t b = 0; b < p->sp_last_batch; ++b) {
      int64_t prev = 0;
      for (int a = 0; a < na; ++a) {
        const int64_t e = std::max(prev, clampr(ms[b * kSmallTiers + act[a]]));
        rows_out[a] += e - prev;
        prev = e;
      }
      rows_out[na] += rows - prev;
    }
    *count = na + 1;
    return 0;
  }
  if (!p->big || !p->pruned) {
    if (cap < 1) return fail(AFD_E_INVALID, "afd_field_tier_rows: cap %d < 1", cap);
    terms[0] = p->n;
    rows_out[0] = rows;
    *count = 1;
    return 0;
  }
  if (cap < na + 1)
    return fail(AFD_E_INVALID, "afd_field_tier_rows: cap %d < %d", cap, na + 1);
  int ms[kPruneTiers] = {};
  CU(cudaMemcpyAsync(ms, p->mstar, sizeof(ms), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  int64_t prev = 0;
  for (int a = 0; a < na; ++a) {
    const int64_t e = std::max(prev, clampr(ms[act[a]]));
    terms[a] = 1LL << prune_k(act[a]);
    rows_out[a] = e - prev;
    prev = e;
  }
  terms[na] = p->n;
  rows_out[na] = rows - prev;
  *count = na + 1;
  return 0;
}

int afd_field_tiers(afd_plan* p, int64_t* rows3, void* stream) {
  if (!p || !rows3) return fail(AFD_E_INVALID, "NULL argument");
  rows3[0] = rows3[1] = rows3[2] = 0;
  if (!p->big) return 0;
  int64_t terms[kPruneTiers + 1], r[kPruneTiers + 1];
  int rc, cnt = 0;
  if ((rc = afd_field_tier_rows(p, terms, r, kPruneTiers + 1, &cnt, stream))) return rc;
  for (int t = 0; t < cnt; ++t) rows3[t == cnt - 1 ? 2 : terms[t] <= 1024 ? 0 : 1] += r[t];
  return 0;
}

int afd_fp64_peak(int device, double* tflops, void* stream) {
  if (!tflops) return fail(AFD_E_INVALID, "NULL argument");
  CU(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out;
  CU(cudaMalloc(&out, sizeof(double)));
  constexpr int kIters = 1 << 14;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  fp64_peak_kernel<kIters><<<blocks, threads, 0, st>>>(out, 1.0);  // warm-up
  CU(cudaEventRecord(e0, st));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) fp64_peak_kernel<kIters><<<blocks, threads, 0, st>>>(out, 1.0);
  CU(cudaEventRecord(e1, st));
  CU(cudaEventSynchronize(e1));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * kIters * (double)blocks * threads * reps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return 0;
}

}  // extern "C"

#ifdef AFD_STEP_TIMING
// Debug builds only: globaltimer stamps of step_cluster_kernel phases.
extern "C" int afd_debug_step_stamps(unsigned long long* host_out) {
  CU(cudaMemcpyFromSymbol(host_out, afd::g_step_stamps, sizeof(afd::g_step_stamps)));
  return 0;
}
extern "C" int afd_debug_step_cta_start(unsigned long long* host_out) {
  CU(cudaMemcpyFromSymbol(host_out, afd::g_step_cta_start, sizeof(afd::g_step_cta_start)));
  return 0;
}
#endif

#ifdef AFD_FIELD_TIMING
// Debug builds only: clock64 stamps of field_kernel row phases.
extern "C" int afd_debug_field_stamps(long long* host_out) {
  CU(cudaMemcpyFromSymbol(host_out, afd::g_field_stamps, sizeof(afd::g_field_stamps)));
  return 0;
}
#endif
