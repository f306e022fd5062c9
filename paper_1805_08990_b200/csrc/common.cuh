// Shared device/host helpers for the DME (differential matrix equation) B200 path.
// sm_100a only: FP64 DMMA (mma.sync m8n8k4 f64), TMA (cp.async.bulk.tensor) + mbarrier pipelines.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

namespace dme {

// ------------------------------------------------------------------ errors
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define DME_CUDA(x)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw ::dme::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " @ " +  \
                             __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)
void note_launch();            // counts every kernel launch of the library
int64_t launch_count();
#define DME_KCHECK()                    \
  do {                                  \
    ::dme::note_launch();               \
    DME_CUDA(cudaGetLastError());       \
  } while (0)

// Run f (kernel attribute setup: cudaFuncSetAttribute applies per device) once per device ordinal;
// the mutex also makes concurrent first calls from several host threads safe.
template <class F>
inline void per_device_once(std::mutex& m, uint64_t& mask, F&& f) {
  int dev = 0;
  DME_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(m);
  if ((mask >> (dev & 63)) & 1) return;
  f();
  mask |= 1ull << (dev & 63);
}

// ------------------------------------------------------------------ programmatic dependent launch
// The latency-bound kernels of the step's critical stream are launched with programmatic stream
// serialisation: the next kernel is scheduled while its predecessor drains (after every CTA of the
// predecessor executed pdl_trigger() or exited) and waits in pdl_wait() -- its first statement --
// until the predecessor has completed and its memory is visible. Without the attribute both are
// no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DME_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// plain bulk copy global -> shared (no tensor map, no swizzle applied: the source must already
// hold the shared-memory image), completion counted on the mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same with an L2 eviction-priority hint (policy from createpolicy, e.g. evict_first for data
// streamed exactly once)
__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}
// FP64 tensor-core MMA: D(8x8) += A(8x4,row) * B(4x8,col). On sm_100a this is DMMA.8x8x4.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
// Fragment row g (0..7) of an m8n8k4 operand -> row of the 128B-swizzled tile, chosen so that each
// half-warp (g = 0..3 / 4..7) touches 8 distinct 16-byte chunks under SWIZZLE_128B (chunk ^ (row&7)).
__device__ __forceinline__ int frag_perm(int g) { return ((g & 3) << 1) | (g >> 2); }
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ host helpers
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms();                 // cached cudaDevAttrMultiProcessorCount of the current device
CUtensorMap make_tmap_2d(const double* base, uint64_t inner, uint64_t outer,
                         uint64_t outer_stride_elems, uint32_t box_inner, uint32_t box_outer,
                         bool swizzle128);
CUtensorMap make_tmap_3d(const double* base, uint64_t d0, uint64_t d1, uint64_t d2,
                         uint64_t s1_elems, uint64_t s2_elems, uint32_t b0, uint32_t b1,
                         uint32_t b2, bool swizzle128);
// 3D byte tensor (int8 digit slices), 128B swizzle; strides in bytes
CUtensorMap make_tmap_3d_u8(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
                            uint64_t s2_bytes, uint32_t b0, uint32_t b1, uint32_t b2);

}  // namespace dme
