// Shared device/host helpers for the B200 (sm_100a) band-reduction library.
#pragma once
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace br {

// Thread-local last error text, surfaced through br_last_error().
void set_error(const char* fmt, ...);

#define BR_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      ::br::set_error("%s failed at %s:%d: %s", #call, __FILE__, __LINE__,         \
                      cudaGetErrorString(e_));                                     \
      return 1000 + (int)e_;                                                       \
    }                                                                              \
  } while (0)

#define BR_CHECK(call)                                                             \
  do {                                                                             \
    int s_ = (call);                                                               \
    if (s_ != 0) return s_;                                                        \
  } while (0)

// Column-major fp64 matrix view. Element (r, c) lives at
//   p[r + c*ld]  when !trans,   p[c + r*ld]  when trans
// so a transposed view of a column-major block is just a flag flip.
struct MatView {
  double* p = nullptr;
  int64_t ld = 0;
  int64_t rows = 0, cols = 0;
  bool trans = false;
  __host__ __device__ MatView() {}
  __host__ __device__ MatView(double* p_, int64_t ld_, int64_t r_, int64_t c_, bool t_ = false)
      : p(p_), ld(ld_), rows(r_), cols(c_), trans(t_) {}
  __host__ __device__ double* at(int64_t r, int64_t c) const {
    return trans ? p + c + r * ld : p + r + c * ld;
  }
  __host__ __device__ MatView sub(int64_t r0, int64_t c0, int64_t nr, int64_t nc) const {
    return MatView(at(r0, c0), ld, nr, nc, trans);
  }
  __host__ __device__ MatView T() const { return MatView(p, ld, cols, rows, !trans); }
};

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace br

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
namespace br {

// D = A*B + C, m8n8k4 fp64 tensor-core MMA (SASS DMMA.8x8x4 on sm_100a).
// Lane l: a = A[l/4][l%4], b = B[l%4][l/4], c/d = C[l/4][2*(l%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global->shared, zero-filling (16 - src_bytes) bytes.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_u32(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
// 8-byte async copy global->shared, zero-filling when src_bytes == 0.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its predecessor in the stream finishes; pdl_wait() blocks
// until the predecessor grid has completed and its writes are visible, and
// pdl_trigger() lets the successor start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Cluster-wide barrier with release/acquire semantics for shared::cluster.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}
// Map a local shared address to the same offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_cluster(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ double ld_cluster_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
// Remote (DSMEM) store; ordered for the cluster by the next
// barrier.cluster.arrive.release.
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Host: when set, the kernel launchers only load their kernel (lazy module
// loading would otherwise load it at first launch, which blocks while a
// persistent panel kernel waits for that very launch) and return.
extern thread_local bool g_preload_only;

// Host: launch `kern` with programmatic stream serialization (BR_PDL=0
// disables it). Every kernel of the library starts with pdl_wait().
bool pdl_enabled();
// The stream's priority, attached to every launch as a launch attribute so it
// survives CUDA-graph capture (graph kernel nodes do not inherit it).
int stream_priority(cudaStream_t st);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = stream_priority(st);
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (g_preload_only) {
    cudaFuncAttributes fa;
    return cudaFuncGetAttributes(&fa, kern);
  }
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace br
#endif
