// Decode-shaped GEMM for small batches (supporting the
// decode step): y[M][N] = x[M][K] * W[N][K]^T (+ bias, ReLU), bf16 in, fp32
// accumulate, fp32 or bf16 out, for M <= 64 rows (the decode batch).
//
// At M <= 64 the product is bound by streaming W once from HBM (AI ~ M flop/B),
// so the kernel is built for bandwidth: W is the MMA's A operand (output
// features on the 16-row side, "swap AB"), the batch rows are the n8 columns,
// CTAs tile N by 128 features and split K so that about two CTAs per SM
// stream, and a 4-stage cp.async pipeline keeps 96 KB of W and x tiles in
// flight per CTA. The split-K partials are summed by the last-arriving CTA of
// each N tile in fixed split order (deterministic, like the attention combine),
// which also applies the epilogue.
#include <stdint.h>

#include <algorithm>

#include "kernels.cuh"

namespace mirage {
namespace {

constexpr int TN = 128;     // output features per CTA
constexpr int TK = 64;      // K per pipeline stage (128 bytes per row)
constexpr int STAGES = 4;
constexpr int MB = 64;      // batch rows staged per tile (M <= MB)
constexpr int THREADS = 128;
constexpr int STAGE_BYTES = (TN + MB) * TK * 2;  // 24 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// byte offset of 16-byte chunk `ch` of row `row` in a [rows][TK] bf16 tile (XOR swizzle)
__device__ __forceinline__ int sw(int row, int ch) { return row * (TK * 2) + ((ch ^ (row & 7)) << 4); }

template <int NB>  // n8 batch tiles: M <= 8 * NB
__global__ void __launch_bounds__(THREADS)
skinny_gemm_kernel(const SkinnyArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int am_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * TN;
  const int split = blockIdx.y;
  const int k0 = split * a.k_per_split;
  const int nsteps = (min(a.K, k0 + a.k_per_split) - k0) / TK;

  auto load_stage = [&](int t) {
    uint8_t* st = smem + (t % STAGES) * STAGE_BYTES;
    const int kk = k0 + t * TK;
#pragma unroll
    for (int i = 0; i < TN * 8 / THREADS; ++i) {  // W tile: 128 rows x 8 chunks
      const int c = tid + i * THREADS, row = c >> 3, ch = c & 7;
      const bool ok = n0 + row < a.N;
      cp_async16(st + sw(row, ch), a.W + (size_t)(ok ? n0 + row : 0) * a.K + kk + ch * 8, ok);
    }
#pragma unroll
    for (int i = 0; i < 8 * NB * 8 / THREADS + (8 * NB * 8 % THREADS ? 1 : 0); ++i) {  // x tile: 8*NB rows
      const int c = tid + i * THREADS, row = c >> 3, ch = c & 7;
      if (row < 8 * NB) {
        const bool ok = row < a.M;
        cp_async16(st + TN * TK * 2 + sw(row, ch), a.x + (size_t)(ok ? row : 0) * a.K + kk + ch * 8, ok);
      }
    }
  };

  float acc[2][NB][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NB; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[mt][nt][j] = 0.f;

#pragma unroll
  for (int t = 0; t < STAGES - 1; ++t) {
    if (t < nsteps) load_stage(t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int t = 0; t < nsteps; ++t) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();  // stage t landed for every thread; stage t-1 is no longer read
    if (t + STAGES - 1 < nsteps) load_stage(t + STAGES - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const uint8_t* Ws = smem + (t % STAGES) * STAGE_BYTES;
    const uint8_t* Xs = Ws + TN * TK * 2;
#pragma unroll
    for (int ks = 0; ks < TK / 16; ++ks) {
      uint32_t af[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)  // A: W rows warp*32 + mt*16 + (lane & 15), k chunk 2ks + (lane >> 4)
        ldsm_x4(af[mt], Ws + sw(warp * 32 + mt * 16 + (lane & 15), 2 * ks + (lane >> 4)));
#pragma unroll
      for (int np = 0; np < (NB + 1) / 2; ++np) {
        // B: x rows of n-tiles 2np (lanes 0-15) and 2np+1 (lanes 16-31), k chunks 2ks / 2ks+1
        uint32_t bf[4];
        const int row = np * 16 + ((lane >> 4) << 3) + (lane & 7);
        ldsm_x4(bf, Xs + sw(row < 8 * NB ? row : 0, 2 * ks + ((lane >> 3) & 1)));
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          mma_bf16(acc[mt][2 * np], af[mt], bf[0], bf[1]);
          if (2 * np + 1 < NB) mma_bf16(acc[mt][2 * np + 1], af[mt], bf[2], bf[3]);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // C fragment: acc[mt][nt][j] = y[m][n], n = n0 + warp*32 + mt*16 + gq (+8 for j >= 2),
  // m = nt*8 + 2tq + (j & 1)
  const int gq = lane >> 2, tq = lane & 3;
  auto epilogue_store = [&](int m, int n, float v) {
    if (a.bias) v += __bfloat162float(a.bias[n]);
    if (a.relu) v = fmaxf(v, 0.f);
    if (a.out_bf16) reinterpret_cast<__nv_bfloat16*>(a.y)[(size_t)m * a.N + n] = __float2bfloat16_rn(v);
    else reinterpret_cast<float*>(a.y)[(size_t)m * a.N + n] = v;
  };
  if (gridDim.y == 1) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NB; ++nt)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int n = n0 + warp * 32 + mt * 16 + gq + (j >= 2 ? 8 : 0), m = nt * 8 + 2 * tq + (j & 1);
          if (m < a.M && n < a.N) epilogue_store(m, n, acc[mt][nt][j]);
        }
    return;
  }
  // split-K: partials, then the last CTA of this N tile sums them in split order
  float* part = a.ws + (size_t)split * a.M * a.N;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NB; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + warp * 32 + mt * 16 + gq + (j >= 2 ? 8 : 0), m = nt * 8 + 2 * tq + (j & 1);
        if (m < a.M && n < a.N) part[(size_t)m * a.N + n] = acc[mt][nt][j];
      }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int prev = atomicAdd(a.tickets + blockIdx.x, 1);
    am_last = prev == (int)gridDim.y - 1;
    if (am_last) a.tickets[blockIdx.x] = 0;  // reset for the next launch
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const int nn = min(TN, a.N - n0);
  for (int e = tid; e < a.M * nn; e += THREADS) {
    const int m = e / nn, n = n0 + e % nn;
    float v = 0.f;
    for (int s = 0; s < (int)gridDim.y; ++s) v += __ldcg(a.ws + ((size_t)s * a.M + m) * a.N + n);
    epilogue_store(m, n, v);
  }
}

template <int NB>
cudaError_t launch_nb(const SkinnyArgs& a0, int splits, cudaStream_t s) {
  constexpr int SMEM = STAGES * STAGE_BYTES;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(skinny_gemm_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) !=
        cudaSuccess)
      return cudaErrorInvalidValue;
    attr = true;
  }
  SkinnyArgs a = a0;
  const int ksteps = a.K / TK;
  a.k_per_split = (ksteps + splits - 1) / splits * TK;
  const int used = (a.K + a.k_per_split - 1) / a.k_per_split;  // no empty split
  skinny_gemm_kernel<NB><<<dim3((a.N + TN - 1) / TN, used), THREADS, SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool skinny_gemm_ok(int M, int N, int K) { return M >= 1 && M <= MB && K % TK == 0 && N >= TN; }

int skinny_gemm_splits(int N, int K, int sms) {
  // about two CTAs per SM stream W (96 KB of stages each), at least 4 K-steps per split
  const int tiles = (N + TN - 1) / TN;
  int splits = std::max(1, (2 * sms + tiles - 1) / tiles);
  splits = std::min(splits, std::max(1, K / TK / 4));
  return std::min(splits, kSkinnyMaxSplits);
}

cudaError_t launch_skinny_gemm(const SkinnyArgs& a, int splits, cudaStream_t s) {
  if (!skinny_gemm_ok(a.M, a.N, a.K)) return cudaErrorInvalidValue;
  if (a.M <= 8) return launch_nb<1>(a, splits, s);
  if (a.M <= 16) return launch_nb<2>(a, splits, s);
  if (a.M <= 32) return launch_nb<4>(a, splits, s);
  return launch_nb<8>(a, splits, s);
}

}  // namespace mirage
