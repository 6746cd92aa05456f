// Throwaway-style microbenchmark kept in tools/: measures B200 fp64 pipe throughput
// (DADD, DMUL, DFMA, sqrt, div) and fp32 FFMA for the roofline denominator in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
template <int OP>
__global__ void kern(double* out, double a, double b, int iters) {
  double x0 = threadIdx.x * 1e-3 + 1.0, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#define STEP(x) \
    if (OP == 0) x = __dadd_rn(x, a); \
    else if (OP == 1) x = __dmul_rn(x, b); \
    else if (OP == 2) x = __fma_rn(x, b, a); \
    else if (OP == 3) x = __dsqrt_rn(x) + a; \
    else if (OP == 4) x = __ddiv_rn(a, x) + b;
    STEP(x0) STEP(x1) STEP(x2) STEP(x3) STEP(x4) STEP(x5) STEP(x6) STEP(x7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kernf(float* out, float a, float b, int iters) {
  float x0 = threadIdx.x * 1e-3f + 1.0f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#define STEPF(x) x = __fmaf_rn(x, b, a);
    STEPF(x0) STEPF(x1) STEPF(x2) STEPF(x3) STEPF(x4) STEPF(x5) STEPF(x6) STEPF(x7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock(kHz) %d\n", p.name, sms, p.clockRate);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"DADD", "DMUL", "DFMA", "DSQRT_rn(+add)", "DDIV_rn(+add)"};
  for (int op = 0; op < 5; ++op) {
    int iters = op >= 3 ? ITERS / 16 : ITERS;
    for (int rep = 0; rep < 2; ++rep) {
      dim3 grid(sms * 8), block(256);
      cudaEventRecord(e0);
      switch (op) {
        case 0: kern<0><<<grid, block>>>(out, 1e-9, 0.999999, iters); break;
        case 1: kern<1><<<grid, block>>>(out, 1e-9, 0.999999, iters); break;
        case 2: kern<2><<<grid, block>>>(out, 1e-9, 0.999999, iters); break;
        case 3: kern<3><<<grid, block>>>(out, 1e-9, 0.999999, iters); break;
        case 4: kern<4><<<grid, block>>>(out, 1.5, 0.5, iters); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = double(sms) * 8 * 256 * iters * 8;
      if (rep) printf("%-16s %.3f ms  %.3e ops/s  (%.1f per SM per cycle at %.0f MHz nominal)\n", names[op], ms,
                      ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1e3);
    }
  }
  float* outf; cudaMalloc(&outf, sizeof(float) * sms * 8 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    kernf<<<sms * 8, 256>>>(outf, 1e-9f, 0.999999f, ITERS);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = double(sms) * 8 * 256 * ITERS * 8;
    if (rep) printf("%-16s %.3f ms  %.3e ops/s  (%.1f per SM per cycle)\n", "FFMA", ms, ops / (ms * 1e-3),
                    ops / (ms * 1e-3) / sms / (p.clockRate * 1e3));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
