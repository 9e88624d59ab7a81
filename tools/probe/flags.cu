// Probe: kernel <-> stream-memop handshake (cuStreamWaitValue32 / WriteValue32).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned ldacq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void strel(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

__global__ void persist(unsigned* f, unsigned ep, int* out) {
  if (threadIdx.x == 0) {
    strel(&f[0], ep);  // done[0]
    unsigned long long t0 = gt();
    while (ldacq(&f[64 + 1]) != ep) {
      __nanosleep(100);
      if (gt() - t0 > 2000000000ull) { out[0] = -1; return; }
    }
    out[0] = (int)((gt() - t0) / 1000);
  }
}
__global__ void work(int* out) { if (threadIdx.x == 0) out[1] = 42; }

typedef CUresult (*PW)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
int main() {
  cudaSetDevice(0);
  cudaFree(0);
  void *f1, *f2;
  cudaDriverEntryPointQueryResult q;
  printf("get wait: %d\n", (int)cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &f1, 12000, cudaEnableDefault, &q));
  printf("q=%d\n", (int)q);
  printf("get write: %d\n", (int)cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &f2, 12000, cudaEnableDefault, &q));
  printf("linked wait %p write %p\n", (void*)&cuStreamWaitValue32, (void*)&cuStreamWriteValue32);
  for (unsigned ver : {11070u, 12000u, 12090u}) {
    void *a = nullptr, *b = nullptr;
    cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &a, ver, cudaEnableDefault, &q);
    cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &b, ver, cudaEnableDefault, &q);
    printf("ver %u: wait %p write %p\n", ver, a, b);
  }
  { void *a = nullptr; cudaGetDriverEntryPoint("cuStreamWaitValue32", &a, cudaEnableDefault, &q); printf("unversioned wait %p\n", a); }
  CUdevice d; cuDeviceGet(&d, 0);
  int a1 = -1, a2 = -1;
  cuDeviceGetAttribute(&a1, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, d);
  cuDeviceGetAttribute(&a2, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, d);
  printf("attr nor %d 64bit %d\n", a1, a2);
  unsigned* f; int* out;
  cudaMalloc(&f, 128 * 4); cudaMemset(f, 0, 512);
  cudaMalloc(&out, 8); cudaMemset(out, 0, 8);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  persist<<<1, 32, 0, s1>>>(f, 7, out);
  CUresult r1 = ((PW)f1)((CUstream)s2, (CUdeviceptr)&f[0], 7, CU_STREAM_WAIT_VALUE_EQ);
  work<<<1, 32, 0, s2>>>(out);
  CUresult r2 = ((PW)f2)((CUstream)s2, (CUdeviceptr)&f[65], 7, CU_STREAM_WRITE_VALUE_DEFAULT);
  printf("memop rc %d %d\n", (int)r1, (int)r2);
  cudaError_t e = cudaDeviceSynchronize();
  int h[2]; cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
  printf("sync %s: persist waited %d us (-1 = timeout), work=%d\n", cudaGetErrorString(e), h[0], h[1]);
  // variant: direct driver symbol via cuGetProcAddress-free path using linked libcuda
  cudaMemset(f, 0, 512); cudaMemset(out, 0, 8);
  persist<<<1, 32, 0, s1>>>(f, 9, out);
  r1 = cuStreamWaitValue32((CUstream)s2, (CUdeviceptr)&f[0], 9, CU_STREAM_WAIT_VALUE_EQ);
  work<<<1, 32, 0, s2>>>(out);
  r2 = cuStreamWriteValue32((CUstream)s2, (CUdeviceptr)&f[65], 9, CU_STREAM_WRITE_VALUE_DEFAULT);
  e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
  printf("linked: rc %d %d sync %s: persist waited %d us, work=%d\n", (int)r1, (int)r2, cudaGetErrorString(e), h[0], h[1]);
  return 0;
}
