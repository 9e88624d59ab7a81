// Microbenchmarks used to pick the design: DMMA vs DFMA throughput,
// cluster-barrier and grid-barrier latency on B200 (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma16_loop(double* out, int iters) {
  double a[8], b[4], c[2][4];
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; i++) b[i] = 1.0 + i * 1e-4;
  for (int i = 0; i < 2; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 2; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),
                     "d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
  }
  double s = 0; for (int i = 0; i < 2; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-9;
  double c[16];
  for (int i = 0; i < 16; i++) c[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) c[i] = fma(c[i], b, a);
  }
  double s = 0; for (int i = 0; i < 16; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void cluster_bar(double* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = double(t1 - t0) / iters;
}
__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;
__global__ void grid_bar(double* out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned int gen = g_gen;
      __threadfence();
      unsigned int arrived = atomicAdd(&g_count, 1);
      if (arrived == gridDim.x - 1) { g_count = 0; __threadfence(); g_gen = gen + 1; }
      else { while (g_gen == gen) { } }
      __threadfence();
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = double(t1 - t0) / iters;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s SMs %d l2 %d MB smemOptin %zu clock(kHz) %d\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    int iters = 20000; float ms;
    dmma_loop<<<sms * 2, 32 * warps>>>(d, 100);
    cudaEventRecord(e0); dmma_loop<<<sms * 2, 32 * warps>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * sms * 2 * warps;
    printf("DMMA m8n8k4  warps/CTA %2d x2 CTA/SM: %.2f TFLOP/s (%.3f ms)\n", warps, fl / ms / 1e9, ms);
    cudaEventRecord(e0); dmma16_loop<<<sms * 2, 32 * warps>>>(d, iters / 4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 2048 * 2 * (double)(iters / 4) * sms * 2 * warps;
    printf("DMMA m16n8k16 warps/CTA %2d x2 CTA/SM: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    cudaEventRecord(e0); dfma_loop<<<sms * 2, 32 * warps>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * (double)iters * sms * 2 * warps * 32;
    printf("DFMA        warps/CTA %2d x2 CTA/SM: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  double h[4];
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 0;
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (cs > 8) CK(cudaFuncSetAttribute(cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaError_t e = cudaLaunchKernelEx(&cfg, cluster_bar, d, 10000);
    if (e != cudaSuccess) { printf("cluster %d launch fail %s\n", cs, cudaGetErrorString(e)); cudaGetLastError(); continue; }
    CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost));
    printf("cluster barrier size %2d: %.0f cycles\n", cs, h[1]);
  }
  for (int g : {4, 16, 64, 148}) {
    grid_bar<<<g, 256>>>(d, 2000); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost));
    printf("grid barrier %3d CTAs: %.0f cycles\n", g, h[2]);
  }
  return 0;
}
