// Cold vs warm single call of kernel_norm inside a fresh kernel (clock64).
#include <cstdio>
#include "afd_common.cuh"
using namespace afd;

__global__ void cold(const double* in, double* out, long long* cyc) {
  double2 a = make_double2(in[0], in[1]);
  int amb = 0;
  long long t0 = clock64();
  double kn = kernel_norm(a, &amb);
  long long t1 = clock64();
  a.x = kn * 0.5;  // second (dependent) call of a second inlined copy
  double kn2 = kernel_norm(a, &amb);
  long long t2 = clock64();
  out[threadIdx.x] = kn + kn2 + amb;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

int main() {
  double *in, *out; long long* cyc;
  cudaMallocManaged(&in, 16); cudaMalloc(&out, 8192); cudaMallocManaged(&cyc, 16);
  in[0] = 0.61; in[1] = 0.52;
  for (int rep = 0; rep < 4; ++rep) {
    cold<<<1, 256>>>(in, out, cyc);
    cudaDeviceSynchronize();
    printf("launch %d: first call %lld cycles, second call %lld cycles\n", rep, cyc[0], cyc[1]);
  }
  return 0;
}
