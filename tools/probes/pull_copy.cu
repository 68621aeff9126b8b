// Probe (verdict r1 item 3): an SM-driven pull copy of pinned host memory into HBM,
// as an alternative to the copy engine for re-streaming. Two forms:
//   pull_ld  -- every thread streams 16-byte loads of the host source (UVA) into
//               registers, U loads in flight, then streaming (evict-first) stores;
//   pull_tma -- one thread per CTA moves CH-byte chunks with cp.async.bulk
//               host -> shared (mbarrier complete_tx) and cp.async.bulk
//               shared -> global (bulk groups), NB chunks in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//        tools/probes/pull_copy.cu -o tools/probes/libpull.so
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint4 ld_nc_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs_v4(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

template <int U>
__global__ void __launch_bounds__(32) pull_ld(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t j = i + u * stride;
      if (j < n16) v[u] = ld_nc_v4(src + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t j = i + u * stride;
      if (j < n16) st_cs_v4(dst + j, v[u]);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// chunks [blockIdx.x, blockIdx.x + grid, ...] of CH bytes; NB in flight per CTA
template <int CH, int NB>
__global__ void __launch_bounds__(32) pull_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                size_t bytes) {
  extern __shared__ __align__(128) uint8_t buf[];
  __shared__ __align__(8) uint64_t bar[NB];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NB; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nch = (bytes + CH - 1) / CH;
  size_t mine = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto chunk_at = [&](size_t k) { return (size_t)blockIdx.x + k * gridDim.x; };
  auto issue = [&](size_t k) {
    const size_t c = chunk_at(k);
    const uint32_t n = (uint32_t)((c + 1) * CH <= bytes ? CH : bytes - c * CH);
    const int b = (int)(k % NB);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(n)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf + (size_t)b * CH)),
        "l"(src + c * CH), "r"(n), "r"(smem_u32(&bar[b]))
        : "memory");
  };
  for (size_t k = 0; k < mine && k < NB; ++k) issue(k);
  for (size_t k = 0; k < mine; ++k) {
    const int b = (int)(k % NB);
    const uint32_t ph = (uint32_t)((k / NB) & 1);
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            smem_u32(&bar[b])),
        "r"(ph)
        : "memory");
    const size_t c = chunk_at(k);
    const uint32_t n = (uint32_t)((c + 1) * CH <= bytes ? CH : bytes - c * CH);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CH),
                 "r"(smem_u32(buf + (size_t)b * CH)), "r"(n)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (k + NB < mine) {
      // buffer b is refilled next: its store must have read shared memory first
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(k + NB);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

extern "C" int pull_copy(int mode, const void* src, void* dst, size_t bytes, int grid, void* stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (mode == 0) {
    pull_ld<8><<<grid, 32, 0, s>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), bytes / 16);
  } else if (mode == 1) {
    pull_ld<16><<<grid, 32, 0, s>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), bytes / 16);
  } else if (mode == 2) {
    constexpr int CH = 4096, NB = 3;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(pull_tma<CH, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * NB);
      set = true;
    }
    pull_tma<CH, NB><<<grid, 32, CH * NB, s>>>(reinterpret_cast<const uint8_t*>(src),
                                              reinterpret_cast<uint8_t*>(dst), bytes);
  } else if (mode == 3) {
    constexpr int CH = 8192, NB = 4;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(pull_tma<CH, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * NB);
      set = true;
    }
    pull_tma<CH, NB><<<grid, 32, CH * NB, s>>>(reinterpret_cast<const uint8_t*>(src),
                                              reinterpret_cast<uint8_t*>(dst), bytes);
  } else {
    return -1;
  }
  return (int)cudaGetLastError();
}
