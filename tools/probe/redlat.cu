// Latency probe for the leaf's per-step building blocks (one warp per SM
// sub-partition, dependent iterations): the shuffle transpose-reduction of 8
// slots + a norm, the same through DMMA (ones x partials), through shared
// memory, and the rsqrt / rcp scalar chain (library vs float-seeded Newton).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o redlat redlat.cu && ./redlat
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int RC>
__device__ __forceinline__ void warp_transpose_reduce(double (&v)[RC], int lane) {
  int n = RC;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      const bool up = (lane & o) != 0;
      const int h = n / 2;
#pragma unroll
      for (int q = 0; q < RC / 2; ++q)
        if (q < h) {
          const double send = up ? v[q] : v[q + h], keep = up ? v[q + h] : v[q];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      n = h;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// mode 0: shuffles; 1: DMMA; 2: shared memory
template <int MODE>
__global__ void red_kernel(double* out, long long* cyc, int iters) {
  __shared__ double sm[4][8][34];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s[8], nr = lane * 0.25;
  for (int c = 0; c < 8; ++c) s[c] = lane + c * 0.5;
  double acc = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = s[c] + acc;  // depends on the previous iteration
    double n2 = nr + acc, tot;
    if (MODE == 0) {
      n2 = warp_sum(n2);
      warp_transpose_reduce<8>(v, lane);
      tot = v[0];
    } else if (MODE == 1) {
      double u[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        double d0 = 0.0, d1 = 0.0;
        dmma884(d0, d1, 1.0, v[c]);
        u[c] = d0 + d1;
      }
      double e0 = 0.0, e1 = 0.0;
      dmma884(e0, e1, 1.0, n2);
      n2 = e0 + e1;
      const int g = lane >> 2;
      const double a0 = (g & 1) ? u[1] : u[0], a1 = (g & 1) ? u[3] : u[2], a2 = (g & 1) ? u[5] : u[4],
                   a3 = (g & 1) ? u[7] : u[6];
      const double b0 = (g & 2) ? a1 : a0, b1 = (g & 2) ? a3 : a2;
      const double sel = (g & 4) ? b1 : b0;
      double f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;
      dmma884(f0, f1, 1.0, sel);
      dmma884(g0, g1, 1.0, n2);
      n2 = g0;
      tot = f0 + f1 * 1e-3;  // both slot totals of this lane are live
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) sm[warp][c][lane] = v[c];
      __syncwarp();
      const int c = lane >> 2, q = lane & 3;
      double w[8];
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const double2 t = *reinterpret_cast<const double2*>(&sm[warp][c][8 * q + k]);
        w[k] = t.x;
        w[k + 1] = t.y;
      }
      __syncwarp();
      double t = ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      n2 = warp_sum(n2);
      tot = t;
    }
    acc = (tot + n2) * 1e-9;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  out[threadIdx.x] = acc;
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y = (double)rsqrtf((float)x);
  const double hx = 0.5 * x;
  double e = fma(-hx * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-hx * y, y, 0.5);
  return fma(y, e, y);
}
__device__ __forceinline__ double fast_rcp(double d) {
  double r = (double)__frcp_rn((float)d);
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
template <int MODE>
__global__ void scal_kernel(double* out, long long* cyc, int iters) {
  double nrm2 = 3.0 + threadIdx.x, x0 = 0.7;
  const long long t0 = clock64();
  double rinv = 0.0, rb = 0.0;
  for (int it = 0; it < iters; ++it) {
    double rs, beta;
    if (MODE == 0) {
      rs = rsqrt(nrm2);
      const double nrm = nrm2 * rs;
      beta = (x0 < 0.0) ? nrm : -nrm;
      rinv = __drcp_rn(x0 - beta);
    } else {
      rs = fast_rsqrt(nrm2);
      const double nrm = nrm2 * rs;
      beta = (x0 < 0.0) ? nrm : -nrm;
      rinv = fast_rcp(x0 - beta);
    }
    rb = rs;
    nrm2 = nrm2 + rinv * 1e-9 + rb * 1e-9;  // next iteration depends on this one
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  out[threadIdx.x] = rinv + rb;
}
int main() {
  double* out;
  long long *cyc, h;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8);
  const char* names[3] = {"shuffle transpose-reduce 8 + norm", "DMMA reduce 8 + norm", "smem transpose 8 + shuffle norm"};
  for (int rep = 0; rep < 2; ++rep) {
    red_kernel<0><<<1, 128>>>(out, cyc, 2000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", names[0], h);
    red_kernel<1><<<1, 128>>>(out, cyc, 2000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", names[1], h);
    red_kernel<2><<<1, 128>>>(out, cyc, 2000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%s: %lld cycles\n", names[2], h);
    scal_kernel<0><<<1, 128>>>(out, cyc, 2000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("rsqrt + rcp chain (library): %lld cycles\n", h);
    scal_kernel<1><<<1, 128>>>(out, cyc, 2000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("rsqrt + rcp chain (float seed + 2 Newton): %lld cycles\n", h);
  }
  // accuracy of the fast versions
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
