// Decode GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   Y[b][n] = sum_k X[b][k] * W[n][k]      (y = x W^T; W row-major [N][K] bf16, X [B][K] bf16)
//
// A decode step multiplies a skinny activation block (B rows, B <= 256) by the
// layer's weights, so the GEMM is weight-streaming bound (AI ~ B flop/B). It is
// computed swapped, Y^T = W X^T: the 128 weight rows of a tile are the MMA's M
// side and the batch is its N side (N = B rounded up to 16), so one
// tcgen05.mma.cta_group::1.kind::f16 M=128 x N=Bn x K=16 consumes 4 KB of weights
// straight from shared memory while the fp32 accumulator tile lives in TMEM
// (128 lanes x Bn columns).
//
// One CTA = one (128-row tile, K split). Warp roles: lane 0 of warp 0 issues the
// TMA loads (cp.async.bulk.tensor, 128B swizzle: 128 x 64 weight box + Bn x 64
// activation box per stage, an NS-deep full/empty mbarrier ring); lane 0 of warp
// 1 issues the MMAs (4 per stage, K = 16 each) and releases a stage with
// tcgen05.commit; warp 2 owns the TMEM allocation. After the last commit all 4
// warps drain TMEM (tcgen05.ld 32x32b: warp w reads lanes 32w..32w+31 = rows of
// the tile) and store the split's fp32 slice Y_s[b][n]. Split slices are summed
// in fixed order by the consumer (the residual kernel), so results are
// deterministic; with `peer` destinations the epilogue writes the slice straight
// into every tensor-parallel rank's exchange buffer (the fused all-reduce, a10).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.cuh"

namespace mirage {
namespace {

constexpr int kTileM = 128;  // weight rows per tile (MMA M)
constexpr int kTileK = 64;   // K per stage: one 128-byte swizzle row of bf16
constexpr int kMaxClusterSplits = 8;  // portable cluster size
constexpr int kSkMinUnits = 3;        // stream-K GEMM: K blocks per CTA at least
// ring depth: ~96-104 KB of stages per CTA, so two CTAs share an SM (two tiles
// streaming per SM: the grid of a decode GEMM is ~1-2 waves of small tiles)
template <int BN>
constexpr int stages() { return BN <= 32 ? 5 : (BN <= 64 ? 4 : (BN <= 128 ? 3 : 2)); }

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
// UMMA shared-memory descriptor, K-major operand in the 128B-swizzle canonical
// layout (rows of 128 bytes, 8-row groups 1024 bytes apart): start >> 4 in
// [0,14), LBO = 1 (unused for swizzled K-major) in [16,30), SBO = 1024 >> 4 in
// [32,46), version 1 (Blackwell) at 46, layout SWIZZLE_128B (2) in [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

// Instruction descriptor, kind::f16: D fp32 (bits 4-5 = 1), A and B bf16 (7-9 = 1,
// 10-12 = 1), both K-major (15, 16 = 0), N >> 3 in [17,23), M >> 4 in [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct GemmArgs {
  float* out;          // split s, row b, column n at out + s * slice + b * ldo + n
  long long slice;     // floats between split slices
  int ldo, N, K, B;
  int kb_per_split;    // 64-wide K blocks per split
  int n_kb;            // total K blocks
  // fused tensor-parallel epilogue: also store the slice into every rank's exchange
  // buffer (peer pointers); peer_slot = this rank's slot offset (floats) there
  float* const* peers;
  int n_peers;
  long long peer_slot;
  // arrival counters bumped (release, system scope) once the CTA's stores landed:
  // one per destination rank of a fused tensor-parallel GEMM
  unsigned long long* const* cnt;
  int n_cnt;
  // cluster split reduction: the grid's K splits of a tile form one thread-block
  // cluster (1 x S); each CTA parks its fp32 partial tile in its (now idle) stage
  // ring, and after a cluster barrier CTA r sums rows b in [r B / S, (r+1) B / S)
  // over the S partials through distributed shared memory, in split order, and
  // stores the final rows (one slice, no workspace)
  int creduce;
};

template <int BN>
__global__ void __launch_bounds__(128, 2)
decode_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, const GemmArgs g) {
  constexpr int A_BYTES = kTileM * kTileK * 2;  // 16 KB
  constexpr int B_BYTES = BN * kTileK * 2;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  constexpr int kStages = stages<BN>();
  extern __shared__ __align__(1024) uint8_t dsmem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[stages<BN>()], empty[stages<BN>()], done;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kTileM;
  const int split = blockIdx.y;
  const int zb = blockIdx.z * BN;  // column group: batch rows [zb, zb + BN) of this CTA
  const int kb0 = split * g.kb_per_split;
  const int kb1 = min(g.n_kb, kb0 + g.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mb_init(&full[i], 1);
      mb_init(&empty[i], 1);
    }
    mb_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
  }
  if (warp == 2) {  // TMEM accumulator: 128 lanes x TMEM_COLS fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_d = tmem_base;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int i = 0; i < nkb; ++i) {
      const int st = i % kStages;
      if (i >= kStages) mb_wait(&empty[st], ((i / kStages) - 1) & 1);
      uint8_t* a = smem + st * STAGE;
      mb_expect_tx(&full[st], STAGE);
      tma_2d(a, &tmW, (kb0 + i) * kTileK, n0, &full[st]);
      tma_2d(a + A_BYTES, &tmX, (kb0 + i) * kTileK, zb, &full[st]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (one thread) ----
    constexpr uint32_t idesc = idesc_bf16(kTileM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int st = i % kStages;
      mb_wait(&full[st], (i / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a = su32(smem + st * STAGE), b = a + A_BYTES;
#pragma unroll
      for (int k = 0; k < kTileK / 16; ++k)  // K = 16 per MMA: +32 bytes inside the swizzle row
        umma_f16(tmem_d, sw128_desc(a + 32 * k), sw128_desc(b + 32 * k), idesc, (i | k) != 0);
      umma_commit(&empty[st]);  // the stage is free once these MMAs have read it
    }
    umma_commit(&done);
  }
  __syncwarp();

  // ---- epilogue: TMEM -> registers -> global (all 4 warps; warp w owns lanes 32w..) ----
  mb_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int n = n0 + warp * 32 + lane;
  const uint32_t taddr = tmem_d + ((uint32_t)(warp * 32) << 16);
  float* dst = g.out + (long long)split * g.slice;
  if (g.creduce) {
    float* part = reinterpret_cast<float*>(smem);  // [b][128] fp32; the ring is idle after `done`
    const int row = warp * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < g.B) part[(c0 + j) * kTileM + row] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int S = gridDim.y;
    const int b0 = split * g.B / S, b1 = (split + 1) * g.B / S;
    uint32_t rbase[kMaxClusterSplits];
    const uint32_t mine = su32(part + row);
#pragma unroll
    for (int r = 0; r < kMaxClusterSplits; ++r)
      if (r < S) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbase[r]) : "r"(mine), "r"(r));
    if (n < g.N) {
#pragma unroll 1
      for (int b = b0; b < b1; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int r = 0; r < kMaxClusterSplits; ++r) {  // split order: deterministic
          if (r < S) {
            float x;
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(rbase[r] + (uint32_t)(b * kTileM * 4)));
            acc += x;
          }
        }
        g.out[(long long)b * g.ldo + n] = acc;
        for (int r = 0; r < g.n_peers; ++r) g.peers[r][g.peer_slot + (long long)b * g.ldo + n] = acc;
      }
    }
    // no CTA may leave (and release its shared memory) while the others still read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else
  // compact epilogue (one copy of the 16-column body: the unrolled form spent most
  // of its time fetching instructions)
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int nb = min(16, g.B - zb - c0);
    if (n < g.N && nb > 0) {
      const long long off = (long long)(zb + c0) * g.ldo + n;
#pragma unroll 1
      for (int r = -1; r < g.n_peers; ++r) {  // r = -1: the local slice; r >= 0: fused TP push to rank r
        float* d = (r < 0 ? dst : g.peers[r] + g.peer_slot + (long long)split * g.slice) + off;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < nb) d[(long long)j * g.ldo] = nkb > 0 ? __uint_as_float(v[j]) : 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(TMEM_COLS) : "memory");
  // fused all-reduce: the barrier above orders every thread's tile stores (local
  // and peer) before thread 0's system-scope release increments (cumulativity);
  // a consumer that acquires a counter value sees this tile in every slot.
  if (threadIdx.x == 0 && g.n_cnt) {
    __threadfence_system();
    for (int r = 0; r < g.n_cnt; ++r)
      asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(g.cnt[r]) : "memory");
  }
}

// ---- persistent stream-K decode GEMM ("SK") -----------------------------------
// The grid is one wave of G resident CTAs. The tiles x K-blocks of the GEMM are
// one stream of units (tile-major); CTA c takes the contiguous units
// [c U / G, (c+1) U / G), i.e. the tail of one tile, whole tiles, and the head of
// another. A tile cut between CTAs is finished by the CTA holding its K-block 0
// (the "owner", whose head piece is the LAST segment of its range): the others
// (whose piece is the FIRST segment of theirs, so they never wait) park their fp32
// partial in a per-CTA workspace slot and raise a flag; the owner adds the parked
// partials to its own in K order (deterministic) and stores the final tile once,
// with the epilogue (bias, ReLU, bf16) and the tensor-parallel push applied.
// Roles: warp 0 lane 0 issues the TMA loads of every segment through the stage
// ring; warp 1 lane 0 issues the MMAs into one of two TMEM accumulators (so the
// next segment's MMAs overlap the previous segment's epilogue); warps 2-5 drain
// TMEM (warp w reads lanes 32 (w % 4) ..) and run the epilogue.
struct SkArgs {
  float* out;                  // fp32 output (or null when out16 is set)
  __nv_bfloat16* out16;        // bf16 output
  int ldo, N, K, B, n_kb, tiles;
  long long U;                 // tiles * n_kb
  const __nv_bfloat16* bias;   // [N] or null
  int relu;
  float* ws;                   // [G][B][128] fp32 partials
  int* flags;                  // [G], zero between launches (the owner resets what it consumed)
  float* const* peers;         // fused TP push (fp32 output only)
  int n_peers;
  long long peer_slot;
  unsigned long long* const* cnt;
  int n_cnt;
};

__device__ __forceinline__ void tma_2d_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(su32(bar)), "l"(pol)
      : "memory");
}

template <int BN>
__global__ void __launch_bounds__(192, 2)
sk_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, const SkArgs g) {
  constexpr int A_BYTES = kTileM * kTileK * 2;
  constexpr int B_BYTES = BN * kTileK * 2;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int ACC_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  constexpr int NBUF = BN <= 128 ? 2 : 1;            // two CTAs per SM share 512 TMEM columns
  constexpr int TMEM_COLS = ACC_COLS * NBUF;
  constexpr int kStages = stages<BN>();
  extern __shared__ __align__(1024) uint8_t dsmem[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsmem) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[stages<BN>()], empty[stages<BN>()], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long G = gridDim.x;
  const long long u0 = (long long)blockIdx.x * g.U / G, u1 = (long long)(blockIdx.x + 1) * g.U / G;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mb_init(&full[i], 1);
      mb_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mb_init(&acc_full[i], 1);
      mb_init(&acc_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem0 = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer over every segment ----
      uint64_t w_pol;  // the weights are read once per GEMM: evict them first
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(w_pol));
      int i = 0;
      for (long long u = u0; u < u1;) {
        const int t = (int)(u / g.n_kb);
        const int kb_b = (int)(u - (long long)t * g.n_kb);
        const int kb_e = (int)min((long long)g.n_kb, u1 - (long long)t * g.n_kb);
        for (int kb = kb_b; kb < kb_e; ++kb, ++i) {
          const int st = i % kStages;
          if (i >= kStages) mb_wait(&empty[st], ((i / kStages) - 1) & 1);
          uint8_t* a = smem + st * STAGE;
          mb_expect_tx(&full[st], STAGE);
          tma_2d_hint(a, &tmW, kb * kTileK, t * kTileM, &full[st], w_pol);
          tma_2d(a + A_BYTES, &tmX, kb * kTileK, 0, &full[st]);
        }
        u = (long long)t * g.n_kb + kb_e;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = idesc_bf16(kTileM, BN);
      int i = 0, seg = 0;
      for (long long u = u0; u < u1; ++seg) {
        const int t = (int)(u / g.n_kb);
        const int kb_b = (int)(u - (long long)t * g.n_kb);
        const int kb_e = (int)min((long long)g.n_kb, u1 - (long long)t * g.n_kb);
        const int buf = seg % NBUF;
        if (seg >= NBUF) mb_wait(&acc_empty[buf], ((seg / NBUF) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tmem_d = tmem0 + (uint32_t)(buf * ACC_COLS);
        for (int kb = kb_b; kb < kb_e; ++kb, ++i) {
          const int st = i % kStages;
          mb_wait(&full[st], (i / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a = su32(smem + st * STAGE), b = a + A_BYTES;
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k)
            umma_f16(tmem_d, sw128_desc(a + 32 * k), sw128_desc(b + 32 * k), idesc, (kb != kb_b || k != 0));
          umma_commit(&empty[st]);
        }
        umma_commit(&acc_full[buf]);
        u = (long long)t * g.n_kb + kb_e;
      }
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lanes 32 (warp % 4) .. +31 = rows of the tile ----
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int etid = threadIdx.x - 64;  // 0..127
    auto ebar = [&]() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
    int seg = 0, finals = 0;
    for (long long u = u0; u < u1; ++seg) {
      const int t = (int)(u / g.n_kb);
      const int kb_b = (int)(u - (long long)t * g.n_kb);
      const int kb_e = (int)min((long long)g.n_kb, u1 - (long long)t * g.n_kb);
      u = (long long)t * g.n_kb + kb_e;
      const int buf = seg % NBUF;
      const bool part = kb_b > 0;                       // tail / middle piece: park it
      const bool owner = kb_b == 0 && kb_e < g.n_kb;    // head piece of a cut tile
      // the CTAs holding the rest of an owned tile: blockIdx+1 .. last (their first segments)
      int c_last = blockIdx.x;
      if (owner) {
        const long long tile_end = (long long)(t + 1) * g.n_kb;
        while (c_last + 1 < G && (long long)(c_last + 1) * g.U / G < tile_end) ++c_last;
        if (etid == 0) {
          for (int c2 = blockIdx.x + 1; c2 <= c_last; ++c2) {
            int f;
            do {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(g.flags + c2) : "memory");
            } while (f == 0);
            g.flags[c2] = 0;  // consumed: ready for the next launch (stream-ordered)
          }
        }
        ebar();  // the acquires (thread 0) order every epilogue thread's partial loads below
      }
      mb_wait(&acc_full[buf], (seg / NBUF) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem0 + (uint32_t)(buf * ACC_COLS) + ((uint32_t)(q * 32) << 16);
      const int n = t * kTileM + row;
      const float bv = (g.bias && n < g.N) ? __bfloat162float(g.bias[n]) : 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int nb = min(16, g.B - c0);
        if (nb <= 0) continue;
        if (part) {
          float* w = g.ws + (size_t)blockIdx.x * g.B * kTileM + (size_t)c0 * kTileM + row;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < nb) w[(size_t)j * kTileM] = __uint_as_float(v[j]);
          continue;
        }
        float acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(v[j]);
        for (int c2 = blockIdx.x + 1; owner && c2 <= c_last; ++c2) {  // K order: deterministic
          const float* w = g.ws + (size_t)c2 * g.B * kTileM + (size_t)c0 * kTileM + row;
          float pv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pv[j] = j < nb ? __ldcg(w + (size_t)j * kTileM) : 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += pv[j];
        }
        if (n < g.N) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j >= nb) break;
            float y = acc[j] + bv;
            if (g.relu) y = fmaxf(y, 0.f);
            const long long off = (long long)(c0 + j) * g.ldo + n;
            if (g.out16) g.out16[off] = __float2bfloat16_rn(y);
            else g.out[off] = y;
            for (int r = 0; r < g.n_peers; ++r) g.peers[r][g.peer_slot + off] = y;
          }
        }
      }
      // every tcgen05.ld of this buffer has completed (wait::ld): hand it back
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[buf])) : "memory");
      if (part) {  // publish the parked partial (at most one per CTA: its first segment)
        ebar();
        if (etid == 0) asm volatile("st.release.gpu.global.s32 [%0], 1;" ::"l"(g.flags + blockIdx.x), "r"(1) : "memory");
      } else {
        ++finals;
      }
    }
    if (g.n_cnt && finals) {  // fused TP all-reduce: one increment per finished tile per destination
      ebar();
      if (etid == 0) {
        __threadfence_system();
        for (int r = 0; r < g.n_cnt; ++r)
          asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(g.cnt[r]), "l"((unsigned long long)finals)
                       : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem0), "n"(TMEM_COLS) : "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map of a row-major [rows][cols] matrix (row pitch ld elements),
// box [box_rows][64] with 128-byte swizzle; cached by its arguments.
bool tensor_map(CUtensorMap* out, const void* base, int rows, int cols, int ld, int box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int, int>, CUtensorMap> cache;
  const auto key = std::make_tuple(base, rows, cols, ld, box_rows);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)kTileK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return true;
}

template <int BN>
constexpr int smem_of() { return stages<BN>() * (kTileM * kTileK * 2 + BN * kTileK * 2) + 1024; }

template <int BN>
cudaError_t launch_bn(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& g, int tiles, int splits,
                      int cgroups, cudaStream_t s) {
  constexpr int SMEM = smem_of<BN>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (!g.creduce) {
    decode_gemm_kernel<BN><<<dim3(tiles, splits, cgroups), 128, SMEM, s>>>(tw, tx, g);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tiles, splits);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = splits;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_gemm_kernel<BN>, tw, tx, g);
}

template <int BN>
cudaError_t launch_sk_bn(const CUtensorMap& tw, const CUtensorMap& tx, const SkArgs& g, cudaStream_t s) {
  constexpr int SMEM = smem_of<BN>();
  static int cap = 0;
  if (!cap) {
    cudaError_t e = cudaFuncSetAttribute(sk_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sk_gemm_kernel<BN>, 192, SMEM);
    if (e != cudaSuccess) return e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = std::max(1, std::min(per_sm, 2)) * sms;
  }
  // one wave (the owners wait on later CTAs, so every CTA must be resident), and
  // every CTA holds at least kSkMinUnits K blocks (>= 1, so none is empty)
  const long long G = std::max(1LL, std::min<long long>(cap, g.U / kSkMinUnits));
  sk_gemm_kernel<BN><<<(unsigned)G, 192, SMEM, s>>>(tw, tx, g);
  return cudaGetLastError();
}

}  // namespace

int decode_gemm_splits(int N, int K, int B, int sms) {
  // Per-SM load model of a one-tile-per-CTA grid at two resident CTAs per SM:
  // ceil(tiles * s / sms) CTAs per SM, each streaming ceil(kb / s) stages of
  // (weights + activations), plus the split slices every split writes and the
  // consumer reads back (2 * B * N * 4 bytes per split, spread over the SMs).
  const int tiles = (N + kTileM - 1) / kTileM;
  const int n_kb = (K + kTileK - 1) / kTileK;
  const int bn = B <= 32 ? 32 : (B <= 64 ? 64 : (B <= 128 ? 128 : 256));
  double best = 1e300;
  int best_s = 1;
  for (int s = 1; s <= kMaxGemmSplits && (s == 1 || n_kb / s >= 2); ++s) {
    const int per = (n_kb + s - 1) / s;
    const int used = (n_kb + per - 1) / per;  // splits that actually hold K blocks
    if (used != s) continue;
    // CTAs on the busiest SM; a CTA alone on an SM keeps only half the bytes in flight
    // (~0.6 of the SM's rate, measured by the split sweep of tools/gemm_bench.py)
    const int on_sm = (tiles * s + sms - 1) / sms;
    const double cost = (on_sm >= 2 ? on_sm : on_sm / 0.6) * per * (kTileM * kTileK * 2.0 + bn * kTileK * 2.0) +
                        (s > 1 ? 2.0 * s * B * N * 4.0 / sms : 0.0);
    if (cost < best * 0.995) {
      best = cost;
      best_s = s;
    }
  }
  return best_s;
}

cudaError_t launch_decode_gemm(const __nv_bfloat16* W, int N, int K, int ldw, const __nv_bfloat16* X, int B, int ldx,
                               float* out, int ldo, long long slice, int splits, float* const* peers, int n_peers,
                               long long peer_slot, cudaStream_t s, unsigned long long* const* cnt, int n_cnt,
                               bool reduce, int* slices_out, int cgroups) {
  if (B <= 0 || cgroups < 1 || cgroups > 8 || B > 256 * cgroups || N <= 0 || K <= 0 || splits < 1 ||
      splits > kMaxGemmSplits || (ldw % 8) || (ldx % 8))
    return cudaErrorInvalidValue;
  // column groups: the batch is cut into cgroups groups of bn rows, one CTA per
  // (tile, split, group); every group re-reads the tile's weights (from L2 when the
  // groups of a tile run side by side), so a GEMM with few tiles covers more SMs
  // without cutting K
  const int Bg = (B + cgroups - 1) / cgroups;
  const int BN = ((Bg + 15) / 16) * 16;
  const int bn = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  cgroups = (B + bn - 1) / bn;  // groups that actually hold rows
  CUtensorMap tw, tx;
  if (!tensor_map(&tw, W, N, K, ldw, kTileM) || !tensor_map(&tx, X, B, K, ldx, bn)) return cudaErrorInvalidValue;
  GemmArgs g{};
  g.out = out;
  g.slice = slice;
  g.ldo = ldo;
  g.N = N;
  g.K = K;
  g.B = B;
  g.n_kb = (K + kTileK - 1) / kTileK;
  g.kb_per_split = (g.n_kb + splits - 1) / splits;
  g.peers = peers;
  g.n_peers = peers ? n_peers : 0;
  g.peer_slot = peer_slot;
  g.cnt = cnt;
  g.n_cnt = cnt ? n_cnt : 0;
  // the partial tile parks in the stage ring: B x 128 fp32 must fit there (bn <= 128)
  g.creduce = reduce && cgroups == 1 && splits > 1 && splits <= kMaxClusterSplits && bn <= 128 &&
              B * kTileM * 4 <= smem_of<128>() - 1024;
  if (slices_out) *slices_out = g.creduce ? 1 : splits;
  const int tiles = (N + kTileM - 1) / kTileM;
  switch (bn) {
    case 32: return launch_bn<32>(tw, tx, g, tiles, splits, cgroups, s);
    case 64: return launch_bn<64>(tw, tx, g, tiles, splits, cgroups, s);
    case 128: return launch_bn<128>(tw, tx, g, tiles, splits, cgroups, s);
    default: return launch_bn<256>(tw, tx, g, tiles, splits, cgroups, s);
  }
}

int decode_gemm_cgroups(int N, int B, int sms) {
  // one K split (the fused tensor-parallel push): as many column groups of >= 32
  // rows as keep the grid within one wave of two CTAs per SM
  const int tiles = (N + kTileM - 1) / kTileM;
  int best = (B + 255) / 256;  // a group holds at most 256 rows (the MMA's N)
  for (int cg = 2 * best; cg <= 8; cg *= 2) {
    const int Bg = (B + cg - 1) / cg;
    if (Bg < 32 && cg > 1) break;
    if (tiles * cg > 2 * sms) break;
    best = cg;
  }
  return best;
}

int decode_gemm_ctas_per_split(int N, int B, int cgroups) {
  const int Bg = (B + cgroups - 1) / cgroups;
  const int BN = ((Bg + 15) / 16) * 16;
  const int bn = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  return ((N + kTileM - 1) / kTileM) * ((B + bn - 1) / bn);
}

int sk_gemm_max_ctas() { return 2 * 148 * 2; }

cudaError_t launch_sk_gemm(const __nv_bfloat16* W, int N, int K, int ldw, const __nv_bfloat16* X, int B, int ldx,
                           float* out, __nv_bfloat16* out16, int ldo, const __nv_bfloat16* bias, int relu, float* ws,
                           int* flags, float* const* peers, int n_peers, long long peer_slot, cudaStream_t s,
                           unsigned long long* const* cnt, int n_cnt) {
  if (B <= 0 || B > 256 || N <= 0 || K <= 0 || (ldw % 8) || (ldx % 8) || (!out && !out16) || !ws || !flags ||
      (out16 && peers))
    return cudaErrorInvalidValue;
  const int BN = ((B + 15) / 16) * 16;
  const int bn = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  CUtensorMap tw, tx;
  if (!tensor_map(&tw, W, N, K, ldw, kTileM) || !tensor_map(&tx, X, B, K, ldx, bn)) return cudaErrorInvalidValue;
  SkArgs g{};
  g.out = out;
  g.out16 = out16;
  g.ldo = ldo;
  g.N = N;
  g.K = K;
  g.B = B;
  g.n_kb = (K + kTileK - 1) / kTileK;
  g.tiles = (N + kTileM - 1) / kTileM;
  g.U = (long long)g.tiles * g.n_kb;
  g.bias = bias;
  g.relu = relu;
  g.ws = ws;
  g.flags = flags;
  g.peers = peers;
  g.n_peers = peers ? n_peers : 0;
  g.peer_slot = peer_slot;
  g.cnt = cnt;
  g.n_cnt = cnt ? n_cnt : 0;
  switch (bn) {
    case 32: return launch_sk_bn<32>(tw, tx, g, s);
    case 64: return launch_sk_bn<64>(tw, tx, g, s);
    case 128: return launch_sk_bn<128>(tw, tx, g, s);
    default: return launch_sk_bn<256>(tw, tx, g, s);
  }
}

}  // namespace mirage
