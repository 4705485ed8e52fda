// HBM streaming ceilings on this B200 for the access shapes of the large-N
// field: pure reads, pure writes (st.global.cs 16 B per thread and 64 KiB
// TMA bulk stores from shared memory), copy, and the column pass's strided
// read shape (256-B pieces at 64 KiB stride, CTA-contiguous vs round-robin
// tile order).  GB/s over a 4 GiB buffer, best of 5.
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void rd(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i);
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
__global__ void wr(double2* __restrict__ a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(a + i, make_double2((double)i, 1.0));
}
__global__ void wr_plain(double2* __restrict__ a, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a[i] = make_double2((double)i, 1.0);
}
__global__ void cp(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
// 64 KiB blocks: fill shared memory, one bulk store per block, 2 in flight
__global__ void __launch_bounds__(256) bulk_wr(double2* __restrict__ a, size_t nblk) {
  extern __shared__ __align__(128) double2 sm[];
  for (int i = threadIdx.x; i < 8192; i += 256) sm[i] = make_double2(i, 1.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  int k = 0;
  for (size_t b = blockIdx.x; b < nblk; b += gridDim.x, ++k) {
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\tcp.async.bulk.commit_group;"
                   :: "l"(a + b * 4096), "r"((unsigned)__cvta_generic_to_shared(sm + (k & 1) * 4096)), "r"(65536u) : "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// strided tiles: tile = 256 pieces of 256 B at stride 64 KiB (16 columns of
// a 4096-column row), rows of 2^20 points; order 0 = CTA-contiguous
// chunk-major, 1 = round-robin row-major.  Warp w loads pieces w, w+8, ...
__global__ void __launch_bounds__(256) tiles_rd(const double2* __restrict__ y, int rows, int order, double* out) {
  const int chunks = 256;
  const long long tiles = (long long)rows * chunks;
  const long long t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  const long long nt = order ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : t1 - t0;
  double s = 0;
  const int lane = threadIdx.x & 15, u0 = threadIdx.x >> 4;
  for (long long n = 0; n < nt; ++n) {
    long long chunk, row;
    if (order) { long long t = n * gridDim.x + blockIdx.x; row = t / chunks; chunk = t % chunks; }
    else { long long t = t0 + n; chunk = t / rows; row = t % rows; }
    const double2* base = y + row * (1LL << 20) + chunk * 16 + lane;
#pragma unroll 4
    for (int u = u0; u < 256; u += 16) { double2 v = __ldcs(base + (long long)u * 4096); s += v.x + v.y; }
  }
  if (s == 1.2345) out[0] = s;
}

// strided bulk stores: a CTA-item writes 4096 points as 256 pieces of 256 B
// at 64 KiB stride (pass A writing a column-tile-contiguous layout:
// Y[row][chunk][block][16]); items in block-major order per CTA range
__global__ void __launch_bounds__(256) bulk_wr_strided(double2* __restrict__ y, int rows) {
  extern __shared__ __align__(128) double2 sm[];
  for (int i = threadIdx.x; i < 8192; i += 256) sm[i] = make_double2(i, 1.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const long long items = (long long)rows * 256;  // (block, row), block-major
  const long long i0 = items * blockIdx.x / gridDim.x, i1 = items * (blockIdx.x + 1) / gridDim.x;
  int k = 0;
  for (long long it = i0; it < i1; ++it, ++k) {
    const long long blk = it / rows, row = it % rows;
    // warp 0: lanes issue 8 pieces each
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
      __syncwarp();
      for (int c = threadIdx.x; c < 256; c += 32) {
        double2* dst = y + row * (1LL << 20) + (long long)c * 4096 + blk * 16;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(dst), "r"((unsigned)__cvta_generic_to_shared(sm + (k & 1) * 4096 + c * 16)), "r"(256u) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x < 32) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// contiguous tile reads: 64 KiB per tile (the col pass on that layout)
__global__ void __launch_bounds__(256) tiles_rd_contig(const double2* __restrict__ y, size_t n, double* out) {
  double s = 0;
  for (size_t t = blockIdx.x; t < n / 4096; t += gridDim.x) {
#pragma unroll 4
    for (int u = threadIdx.x; u < 4096; u += 256) { double2 v = __ldcs(y + t * 4096 + u); s += v.x + v.y; }
  }
  if (s == 1.2345) out[0] = s;
}

int main() {
  const size_t bytes = 4ULL << 30, n = bytes / 16;
  double2 *a, *b; double* out;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMalloc(&out, 8));
  CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaFuncSetAttribute(bulk_wr, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, double gb, auto f) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = ms < best ? ms : best;
    }
    printf("%-44s %8.3f ms  %7.0f GB/s\n", name, best, gb / (best * 1e-3));
  };
  const double G = bytes / 1e9;
  for (int blocks : {sms * 4, sms * 8, sms * 16}) {
    char nm[64];
    snprintf(nm, 64, "read 16B/thread (%d CTAs x 512)", blocks); run(nm, G, [&] { rd<<<blocks, 512>>>(a, n, out); });
    snprintf(nm, 64, "write st.cs 16B (%d CTAs x 512)", blocks); run(nm, G, [&] { wr<<<blocks, 512>>>(a, n); });
    snprintf(nm, 64, "write st 16B (%d CTAs x 512)", blocks); run(nm, G, [&] { wr_plain<<<blocks, 512>>>(a, n); });
    snprintf(nm, 64, "copy (%d CTAs x 512, r+w bytes)", blocks); run(nm, 2 * G, [&] { cp<<<blocks, 512>>>(a, b, n); });
  }
  run("bulk store 64 KiB (1 CTA/SM)", G, [&] { bulk_wr<<<sms, 256, 131072>>>(a, n / 4096); });
  run("tiles read, CTA-contiguous (1 CTA/SM x 256)", G, [&] { tiles_rd<<<sms, 256>>>(a, 256, 0, out); });
  run("tiles read, round-robin (1 CTA/SM x 256)", G, [&] { tiles_rd<<<sms, 256>>>(a, 256, 1, out); });
  run("tiles read, CTA-contiguous (4 CTA/SM x 256)", G, [&] { tiles_rd<<<sms * 4, 256>>>(a, 256, 0, out); });
  run("tiles read, round-robin (4 CTA/SM x 256)", G, [&] { tiles_rd<<<sms * 4, 256>>>(a, 256, 1, out); });
  return 0;
}

// ctypes entry for scripts/micro/power_patterns.py: run pattern `which` reps
// times on the current stream (buffers allocated on first call).
extern "C" int hbm_pattern(int which, int reps) {
  static double2 *a = nullptr, *b = nullptr; static double* out = nullptr;
  const size_t bytes = 4ULL << 30, n = bytes / 16;
  if (!a) {
    if (cudaMalloc(&a, bytes) || cudaMalloc(&b, bytes) || cudaMalloc(&out, 8)) return 1;
    cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
    cudaFuncSetAttribute(bulk_wr, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    cudaFuncSetAttribute(bulk_wr_strided, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int r = 0; r < reps; ++r) {
    switch (which) {
      case 0: rd<<<sms * 8, 512>>>(a, n, out); break;
      case 1: wr<<<sms * 8, 512>>>(a, n); break;
      case 2: bulk_wr<<<sms, 256, 131072>>>(a, n / 4096); break;
      case 3: tiles_rd<<<sms * 4, 256>>>(a, 256, 0, out); break;
      case 4: tiles_rd<<<sms * 4, 256>>>(a, 256, 1, out); break;
      case 5: bulk_wr_strided<<<sms, 256, 131072>>>(a, 256); break;
      case 6: tiles_rd_contig<<<sms * 4, 256>>>(a, n, out); break;
      default: return 2;
    }
  }
  return cudaGetLastError() != cudaSuccess;
}
