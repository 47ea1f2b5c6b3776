// Diagnostics: FP64 FMA / ADD / DIV issue rate per SM on this GPU
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_rate.cu)
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int n, double s) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = fma(a[j], s, 1e-9);
      if (OP == 1) a[j] = a[j] + s;
      if (OP == 2) a[j] = s / a[j];
      if (OP == 3) a[j] = (double)((float)a[j] + 1.0f);        // F2F both ways
      if (OP == 4) a[j] = floor(a[j] * s);                      // FRND.F64 (+ DMUL)
      if (OP == 5) a[j] = (double)((int)(a[j] * s) & 1023);     // F2I.F64 + I2F.F64 (+ DMUL)
      if (OP == 6) {
        double y;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a[j]));
        a[j] = y;
      }
    }
  double t = 0;
  for (int j = 0; j < 8; ++j) t += a[j];
  if (t == 12345.678) out[0] = t;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[7] = {"dfma", "dadd", "ddiv", "f2f f32<->f64 (2 ops)", "dmul+frnd.f64",
                          "dmul+f2i.f64+i2f.f64", "mufu.rcp64h"};
  void (*fns[7])(double*, int, double) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  for (int op = 0; op < 7; ++op) {
    int n = op == 2 ? 200 : 2000;
    auto f = fns[op];
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      f<<<sms * 4, 512>>>(o, n, 1.0000001);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 4 * 512 * n * 8;
    double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%s: %.3f ms, %.1f Gop/s, %.2f lane-ops per SM per clock (max clock %d MHz)\n",
           names[op], ms, ops / ms / 1e6, per_sm_clk, clk / 1000);
  }
  return 0;
}
