// Latency of the step kernel's serial FP64 chains on one warp (warm i-cache):
// kernel_norm, np_cdiv, and the full per-point remainder update.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I paper_1711_08604_b200/csrc
#include <cstdio>
#include "afd_common.cuh"
using namespace afd;

__global__ void lat(double* out, long long* cyc, double seed) {
  double2 a = make_double2(0.6 + seed, 0.7);
  int amb = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) {
    const double kn = kernel_norm(a, &amb);
    a.x = kn * 0.9;  // dependent
  }
  long long t1 = clock64();
  double2 x = make_double2(0.3, 0.2), y = make_double2(0.5 + seed, 0.25);
  for (int i = 0; i < 256; ++i) x = np_cdiv(y, make_double2(x.x + 1.0, x.y));
  long long t2 = clock64();
  double2 g = make_double2(0.1, 0.2), z = make_double2(0.8, 0.6), coeff = make_double2(0.3, -0.1);
  for (int i = 0; i < 256; ++i) {
    const double2 d = one_minus_conja_z(a, z);
    const double2 e = np_cdiv(make_double2(0.9, 0.0), d);
    const double2 ce = np_cmul(coeff, e);
    const double2 stp = make_double2(g.x - ce.x, g.y - ce.y);
    const double2 num = np_cmul(stp, d);
    g = np_cdiv(num, make_double2(z.x - a.x, z.y - a.y));
    g.x *= 0.5;
  }
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) acc = fma(acc, 0.999, 1e-3);
  long long t4 = clock64();
  for (int i = 0; i < 256; ++i) acc = sqrt(acc + 1.0);
  long long t5 = clock64();
  for (int i = 0; i < 256; ++i) acc = 1.0 / (acc + 1.0);
  long long t6 = clock64();
  out[threadIdx.x] = a.x + x.x + g.x + acc + amb;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256;
    cyc[3] = (t4 - t3) / 256; cyc[4] = (t5 - t4) / 256; cyc[5] = (t6 - t5) / 256;
  }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
  for (int threads = 32; threads <= 256; threads *= 2) {
  for (int rep = 0; rep < 3; ++rep) {
    lat<<<1, threads>>>(out, cyc, 0.01 * rep);
    cudaDeviceSynchronize();
  }
  printf("threads %d: ", threads);
  printf("cycles per call: kernel_norm %lld  np_cdiv %lld  update_point %lld  dfma %lld  sqrt %lld  rcp %lld\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
  }
  return 0;
}
