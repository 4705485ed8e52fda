// Latency of constant-bank (kernel parameter) reads and of an L2 load in a
// PDL secondary kernel, before vs after griddepcontrol.wait.
#include <cstdio>

__global__ void primary(double* x, int iters) {
  double v = x[threadIdx.x];
  for (int i = 0; i < iters; ++i) v = fma(v, 0.999999, 1e-9);
  x[threadIdx.x] = v;
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void secondary(const int* __restrict__ flag, long long* out, int p0, int p1, int p2,
                          int p3, int p4, int p5, int p6, int p7) {
  long long t0 = clock64();
  int a = p0 + p1;  // touch the parameter bank before the wait
  asm volatile("" : "+r"(a));
  long long t1 = clock64();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  long long t2 = clock64();
  int b = p6 * 3 + p7;  // parameter read after the wait
  asm volatile("" : "+r"(b));
  long long t3 = clock64();
  int f = __ldcg(flag);
  asm volatile("" : "+r"(f));
  long long t4 = clock64();
  int g = *(volatile const int*)(flag + 64);
  asm volatile("" : "+r"(g));
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t4 - t3; out[3] = t5 - t4; out[4] = a + b + f + g;
  }
}

int main() {
  double* x; int* flag; long long* out;
  cudaMalloc(&x, 8192); cudaMalloc(&flag, 4096); cudaMallocManaged(&out, 64);
  cudaMemset(x, 0, 8192); cudaMemset(flag, 0, 4096);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int rep = 0; rep < 4; ++rep) {
      primary<<<148, 256, 0, st>>>(x, 20000);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1); cfg.blockDim = dim3(32); cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = pdl;
      cfg.attrs = attr; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, secondary, (const int*)flag, out, 1, 2, 3, 4, 5, 6, 7, 8);
      cudaStreamSynchronize(st);
      printf("pdl=%d: param before wait %lld cyc, param after wait %lld, ldcg after %lld, volatile %lld\n",
             pdl, out[0], out[1], out[2], out[3]);
    }
  }
  return 0;
}
