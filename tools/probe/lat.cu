// Latency microbenchmarks: dependent DADD / DFMA / SHFL(f64) / LDS.64 chains, one warp.
#include <cstdio>
__global__ void lat(double* out, long long* t, int n) {
  __shared__ double sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x * 0.5;
  __syncthreads();
  double a = out[0], b = out[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + b;            // DADD chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, b);     // DFMA chain
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + i) & 31);  // SHFL chain (2x32)
  long long t3 = clock64();
  int idx = threadIdx.x & 31;
  double s = 0;
  for (int i = 0; i < n; ++i) { s = sm[idx]; idx = ((int)s) & 31; }  // LDS chain
  long long t4 = clock64();
  float f = a;
  for (int i = 0; i < n; ++i) f = f + 1.5f;          // FADD chain
  long long t5 = clock64();
  double r = a;
  for (int i = 0; i < n; ++i) r = sqrt(r + 1.0);     // sqrt
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) r = 1.0 / (r + 1.0);   // div
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) r = rsqrt(r + 1.0);    // rsqrt
  long long t8 = clock64();
  for (int i = 0; i < n; ++i) r = __drcp_rn(r + 1.0);  // rcp
  long long t9 = clock64();
  if (threadIdx.x == 0) {
    t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4;
    t[5] = t6 - t5; t[6] = t7 - t6; t[7] = t8 - t7; t[8] = t9 - t8;
  }
  out[2] = a + s + f + r;
}
int main() {
  double* d; long long* t; cudaMalloc(&d, 64); cudaMalloc(&t, 128);
  double h[2] = {1.0, 1e-9}; cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
  int n = 1000; long long ht[9];
  lat<<<1, 32>>>(d, t, n); cudaDeviceSynchronize();
  lat<<<1, 32>>>(d, t, n); cudaDeviceSynchronize();
  cudaMemcpy(ht, t, sizeof(ht), cudaMemcpyDeviceToHost);
  const char* nm[9] = {"DADD", "DFMA", "SHFL.f64", "LDS.64", "FADD", "sqrt.f64(+add)", "div.f64(+add)", "rsqrt.f64(+add)", "rcp.f64(+add)"};
  for (int i = 0; i < 9; ++i) printf("%-16s %.1f cycles/op\n", nm[i], ht[i] / (double)n);
  return 0;
}
