// Feasibility probe: SM partitions (green contexts) for the panel stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -o green green.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s failed: %s\n", #x, s); return 1; } } while (0)
#define RK(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void smid_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}
__global__ void __cluster_dims__(16, 1, 1) cluster_kernel(int* out) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
}
__global__ void spin_kernel(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource sm;
  CK(cuDeviceGetDevResource(dev, &sm, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", sm.sm.smCount);
  for (unsigned flags : {0u, (unsigned)CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE}) {
    for (unsigned minc : {8u, 16u, 18u, 20u, 24u}) {
      unsigned n = 0;
      CUresult r = cuDevSmResourceSplitByCount(nullptr, &n, &sm, nullptr, flags, minc);
      printf("flags %u minCount %u -> groups %u (rc %d)\n", flags, minc, n, (int)r);
    }
  }
  CUdevResource part, rest;
  unsigned n = 1;
  CK(cuDevSmResourceSplitByCount(&part, &n, &sm, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, 16));
  printf("panel partition %u SMs, rest %u SMs\n", part.sm.smCount, rest.sm.smCount);
  CUdevResourceDesc dp, dr;
  CK(cuDevResourceGenerateDesc(&dp, &part, 1));
  CK(cuDevResourceGenerateDesc(&dr, &rest, 1));
  CUgreenCtx gp, gr;
  CK(cuGreenCtxCreate(&gp, dp, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sp, sr;
  CK(cuGreenCtxStreamCreate(&sp, gp, CU_STREAM_NON_BLOCKING, -5));
  CK(cuGreenCtxStreamCreate(&sr, gr, CU_STREAM_NON_BLOCKING, 0));
  int* buf;
  RK(cudaMalloc(&buf, 4096 * sizeof(int)));  // primary-context allocation
  smid_kernel<<<1024, 32, 0, (cudaStream_t)sr>>>(buf);
  RK(cudaGetLastError());
  RK(cudaStreamSynchronize((cudaStream_t)sr));
  std::vector<int> h(4096);
  RK(cudaMemcpy(h.data(), buf, 1024 * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> used(256, 0);
  for (int i = 0; i < 1024; ++i) used[h[i]]++;
  int cnt = 0;
  for (int i = 0; i < 256; ++i) cnt += used[i] > 0;
  printf("main partition kernel used %d distinct SMs\n", cnt);
  smid_kernel<<<1024, 32, 0, (cudaStream_t)sp>>>(buf);
  RK(cudaGetLastError());
  RK(cudaStreamSynchronize((cudaStream_t)sp));
  RK(cudaMemcpy(h.data(), buf, 1024 * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> usedp(256, 0);
  for (int i = 0; i < 1024; ++i) usedp[h[i]]++;
  cnt = 0;
  int overlap = 0;
  for (int i = 0; i < 256; ++i) { cnt += usedp[i] > 0; overlap += (usedp[i] > 0 && used[i] > 0); }
  printf("panel partition kernel used %d distinct SMs, overlap with main %d\n", cnt, overlap);
  cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cluster_kernel<<<16, 128, 0, (cudaStream_t)sp>>>(buf);
  cudaError_t e = cudaGetLastError();
  printf("cluster-16 launch in panel partition: %s\n", cudaGetErrorString(e));
  e = cudaStreamSynchronize((cudaStream_t)sp);
  printf("cluster-16 sync: %s\n", cudaGetErrorString(e));
  // concurrency: spin kernels on both partitions
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, (cudaStream_t)sr);
  spin_kernel<<<rest.sm.smCount, 32, 0, (cudaStream_t)sr>>>(2000000);
  spin_kernel<<<part.sm.smCount, 32, 0, (cudaStream_t)sp>>>(2000000);
  cudaEventRecord(b, (cudaStream_t)sr);
  RK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("concurrent spin (1 ms each): main stream %.3f ms\n", ms);
  return 0;
}
