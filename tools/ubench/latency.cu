// Dependent-chain latency microbenchmark (one warp): cycles per dependent op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* outd, float* outf, long long* cyc, double xd, float xf, int n) {
  long long t0, t1;
  double d = xd; float f = xf;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) d = fma(d, 0.999999, 1e-9);
  t1 = clock64(); cyc[0] = t1 - t0;
  // FFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) f = __fmaf_rn(f, 0.999999f, 1e-9f);
  t1 = clock64(); cyc[1] = t1 - t0;
  // F2F f32->f64->f32 chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) { double q = (double)f; f = (float)(q * 1.0000001); }
  t1 = clock64(); cyc[2] = t1 - t0;
  // MUFU.RCP chain
  float g = xf;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(g)); g = r + 1.0f; }
  t1 = clock64(); cyc[3] = t1 - t0;
  // DMUL chain
  double m = xd;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) m = m * 1.0000001;
  t1 = clock64(); cyc[4] = t1 - t0;
  // IMAD.HI chain (philox-like)
  unsigned u = (unsigned)xf;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) u = __umulhi(u, 0xD2511F53u) ^ 0x1234u;
  t1 = clock64(); cyc[5] = t1 - t0;
  // libdevice exp(double) chain
  double ex = xd * 1e-3;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < n / 16; ++i) ex = exp(ex) * 1e-3;
  t1 = clock64(); cyc[6] = (t1 - t0) * 16;
  // SHFL chain (fp32)
  float sh = xf;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) sh = __shfl_sync(0xffffffffu, sh, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[7] = t1 - t0;
  // DADD chain
  double da = xd;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) da = da + 1e-9;
  t1 = clock64(); cyc[8] = t1 - t0;
  outd[0] = d + m + ex + da; outf[0] = f + g + (float)u + sh;
}
int main() {
  double* od; float* of; long long* c;
  cudaMalloc(&od, 8); cudaMalloc(&of, 4); cudaMalloc(&c, 128);
  int n = 4096;
  k<<<1, 32>>>(od, of, c, 1.0, 1.0f, n);
  k<<<1, 32>>>(od, of, c, 1.0, 1.0f, n);
  long long h[9]; cudaMemcpy(h, c, 72, cudaMemcpyDeviceToHost);
  const char* names[9] = {"DFMA", "FFMA", "F2F64+DMUL+F2F32 (3 ops)", "MUFU.RCP+FADD (2 ops)", "DMUL", "IMAD.HI+LOP (2 ops)",
                          "exp(double)+DMUL", "SHFL.IDX (fp32)", "DADD"};
  for (int i = 0; i < 9; ++i) printf("%-28s %.2f cycles per iteration\n", names[i], (double)h[i] / n);
  return 0;
}
