// Scratch microbenchmark: cycles per tcgen05.mma (kind::i8 / kind::f16, M=128, SS operands in
// 128B-swizzled smem) as a function of N, issued back to back by one thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/mma_probe.cu -o /tmp/mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
template <bool I8>
__device__ __forceinline__ uint32_t idesc(int N) {
  if (I8) return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  // f16: D f32 (1), A bf16 (1), B bf16 (1)
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
}
template <bool I8>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (I8)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}

template <bool I8>
__global__ void __launch_bounds__(128, 1) probe(int N, int reps, int a_stride_mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t A = smem_u32(base), B = smem_u32(base + 32768);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t ad = sdesc(A + (a_stride_mode ? (r & 7) * 16384 : 0) + ks * 32);
        const uint64_t bd = sdesc(B + ks * 32);
        mma<I8>(tm + (uint32_t)((r & 1) * 0), ad, bd, idesc<I8>(N), 1u);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

// The Ozaki kc sequence: order 0 = for a { for ks { chunks } }, order 1 = for ks { for a { chunks } },
// order 2 = like 0 but every MMA to a disjoint D range (dependency-free reference)
__global__ void __launch_bounds__(128, 1) probe_seq(int NP, int order, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t A = smem_u32(base), B = smem_u32(base + 65536);
    long long t0 = clock64();
    int cnt = 0;
    for (int r = 0; r < reps; ++r) {
      if (order == 1) {
        for (int ks = 0; ks < 4; ++ks)
          for (int a = 0; a < 8; ++a) {
            const int rows = (8 - a) * NP;
            for (int r0 = 0; r0 < rows; r0 += 256) {
              const int nn = min(256, rows - r0);
              mma<true>(tm + a * NP + r0, sdesc(A + (a & 3) * 16384 + ks * 32), sdesc(B + r0 * 128 + ks * 32), idesc<true>(nn), 1u);
            }
          }
      } else {
        for (int a = 0; a < 8; ++a)
          for (int ks = 0; ks < 4; ++ks) {
            const int rows = (8 - a) * NP;
            for (int r0 = 0; r0 < rows; r0 += 256) {
              const int nn = min(256, rows - r0);
              const uint32_t d = order == 2 ? (uint32_t)((cnt++ & 1) * 256) : (uint32_t)(a * NP + r0);
              mma<true>(tm + d, sdesc(A + (a & 3) * 16384 + ks * 32), sdesc(B + r0 * 128 + ks * 32), idesc<true>(nn), 1u);
            }
          }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

// issue-overhead probe: 8 MMAs per iteration with loop-invariant descriptors
__global__ void __launch_bounds__(128, 1) probe_issue(int N, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x < 32) {
    const uint32_t A = smem_u32(base), B = smem_u32(base + 65536);
    const uint64_t a0 = sdesc(A), a1 = sdesc(A + 32), a2 = sdesc(A + 64), a3 = sdesc(A + 96);
    const uint64_t b0 = sdesc(B), b1 = sdesc(B + 32), b2 = sdesc(B + 64), b3 = sdesc(B + 96);
    const uint32_t id = idesc<true>(N);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (threadIdx.x == 0) {
        mma<true>(tm, a0, b0, id, 1u); mma<true>(tm, a1, b1, id, 1u);
        mma<true>(tm, a2, b2, id, 1u); mma<true>(tm, a3, b3, id, 1u);
        mma<true>(tm + 256, a0, b0, id, 1u); mma<true>(tm + 256, a1, b1, id, 1u);
        mma<true>(tm + 256, a2, b2, id, 1u); mma<true>(tm + 256, a3, b3, id, 1u);
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
      long long t1 = clock64();
      out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

__device__ __forceinline__ uint64_t mk(uint32_t lo) {
  return (uint64_t)lo | ((uint64_t)((1024 >> 4) | (1u << 14) | (2u << 29)) << 32);
}
// exact Ozaki kc sequence, fast descriptors, optional commit per slice
template <int NP>
__global__ void __launch_bounds__(128, 1) probe_oz(int reps, int commits, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 12345u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    ((uint32_t*)base)[i] = commits >= 2 ? (x & 0x3f3f3f3fu) ^ 0x80808080u * 0 : 0x01010101u * (i & 7);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x < 32) {
    const uint32_t loA = ((smem_u32(base) >> 4) & 0x3FFF) | (1u << 16);
    const uint32_t loB = ((smem_u32(base + 131072) >> 4) & 0x3FFF) | (1u << 16);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const uint32_t la = loA + (uint32_t)(((r * 8 + a) % 7) * 1024);
        if (threadIdx.x == 0) {
          const int rows = (8 - a) * NP;
          const int n0 = rows <= 256 ? rows : ((rows / 2 + 15) / 16) * 16;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            mma<true>(tm + a * NP, mk(la + ks * 2), mk(loB + ks * 2), idesc<true>(n0), 1u);
            if (rows > n0) mma<true>(tm + a * NP + n0, mk(la + ks * 2), mk(loB + ks * 2 + n0 * 8), idesc<true>(rows - n0), 1u);
          }
          if (commits) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)) : "memory");
        }
        __syncwarp();
      }
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
      long long t1 = clock64();
      out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}
template <int NP>
void run_oz(unsigned long long* d, unsigned long long* h, int smem) {
  cudaFuncSetAttribute(probe_oz<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int commits = 0; commits < 3; ++commits) {
    probe_oz<NP><<<148, 128, smem>>>(200, commits, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148 * 200.0;
    printf("oz NP=%d commits=%d: %7.0f cyc/kc (ideal %5.0f, %.2f)\n", NP, commits, avg, 72.0 * NP, 72.0 * NP / avg);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  for (int kind = 0; kind < 2; ++kind)
    for (int mode = 0; mode < 2; ++mode)
      for (int N : {16, 32, 48, 64, 96, 128, 192, 256}) {
        if (kind == 0) probe<true><<<148, 128, smem>>>(N, reps, mode, d);
        else probe<false><<<148, 128, smem>>>(N, reps, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double per = avg / (reps * 4.0);
        const double macs = 128.0 * N * (kind == 0 ? 32 : 16);
        printf("%s mode=%d N=%3d: %7.1f cyc/mma  %7.0f MAC/cyc\n", kind == 0 ? "i8 " : "f16", mode, N, per, macs / per);
      }
  run_oz<16>(d, h, smem); run_oz<32>(d, h, smem); run_oz<48>(d, h, smem); run_oz<64>(d, h, smem);
  cudaFuncSetAttribute(probe_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int N : {32, 64, 128, 192, 256}) {
    probe_issue<<<148, 128, smem>>>(N, 500, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148 * 500.0 * 8;
    printf("issue N=%d: %.1f cyc/mma\n", N, avg);
  }
  cudaFuncSetAttribute(probe_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int NP : {16, 32, 48, 64})
    for (int order = 0; order < 3; ++order) {
      probe_seq<<<148, 128, smem>>>(NP, order, 200, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148 * 200.0;
      const double ideal = 4 * 36 * NP / 2.0;
      printf("seq NP=%d order=%d: %8.0f cyc/kc (ideal %6.0f) -> %.2f of int8 peak\n", NP, order, avg, ideal, ideal / avg);
    }
  return 0;
}
