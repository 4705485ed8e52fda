// Primary -> secondary hand-off latency on B200: time from the last primary
// CTA's final store to (a) the secondary's griddepcontrol.wait returning and
// (b) a secondary that polls a release counter instead.
#include <cstdio>

__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void primary(double* x, int iters, unsigned long long* exit_t, unsigned* counter,
                        double* cand) {
  asm volatile("griddepcontrol.launch_dependents;");
  double v = x[threadIdx.x + blockIdx.x * blockDim.x];
  for (int i = 0; i < iters + (blockIdx.x * 37) % 200; ++i) v = fma(v, 0.999999, 1e-9);
  x[threadIdx.x + blockIdx.x * blockDim.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    cand[blockIdx.x * 4] = v;
    __threadfence();
    atomicAdd(counter, 1u);
    exit_t[blockIdx.x] = gt();
  }
}

__global__ void secondary_wait(const double* cand, int n, unsigned long long* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  unsigned long long t0 = gt();
  double s = 0;
  for (int i = threadIdx.x; i < n; i += 32) s += __ldcg(cand + 4 * i);
  asm volatile("" : "+d"(s));
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) { out[0] = t0; out[1] = t1; out[2] = (unsigned long long)s; }
}

__global__ void secondary_poll(const double* cand, int n, unsigned* counter, unsigned target,
                               unsigned long long* out) {
  unsigned c = 0;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(counter) : "memory");
  } while (c < target);
  unsigned long long t0 = gt();
  double s = 0;
  for (int i = threadIdx.x; i < n; i += 32) s += __ldcg(cand + 4 * i);
  asm volatile("" : "+d"(s));
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) { out[0] = t0; out[1] = t1; out[2] = (unsigned long long)s; }
}

int main() {
  const int P = 128;
  double *x, *cand; unsigned long long *ex, *out; unsigned* counter;
  cudaMalloc(&x, P * 256 * 8); cudaMalloc(&cand, P * 32);
  cudaMalloc(&ex, P * 8); cudaMalloc(&out, 64); cudaMalloc(&counter, 4);
  cudaMemset(x, 0, P * 256 * 8);
  cudaMemset(counter, 0, 4);
  unsigned long long hex[P], hout[8];
  cudaStream_t st; cudaStreamCreate(&st);
  unsigned target = 0;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 5; ++rep) {
      primary<<<P, 256, 0, st>>>(x, 20000, ex, counter, cand);
      target += P;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1); cfg.blockDim = dim3(32); cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      if (mode == 0)
        cudaLaunchKernelEx(&cfg, secondary_wait, (const double*)cand, P, out);
      else
        cudaLaunchKernelEx(&cfg, secondary_poll, (const double*)cand, P, counter, target, out);
      cudaStreamSynchronize(st);
      cudaMemcpy(hex, ex, sizeof(hex), cudaMemcpyDeviceToHost);
      cudaMemcpy(hout, out, sizeof(hout), cudaMemcpyDeviceToHost);
      unsigned long long last = 0;
      for (int i = 0; i < P; ++i) last = hex[i] > last ? hex[i] : last;
      printf("%s: last primary store -> secondary go %lld ns, cand loads %lld ns\n",
             mode ? "poll" : "wait", (long long)(hout[0] - last), (long long)(hout[1] - hout[0]));
    }
  }
  return 0;
}
