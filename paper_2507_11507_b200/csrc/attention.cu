// Paged-attention decode with fused split-K combine (a9)
// for sm_100a.
//
// Computes, for sequence s and query head h (KV head h' = h / G):
//   o = softmax(q K^T / sqrt(D)) V over the s's first ctx_len tokens,
// reading K/V through the block table and the block_base indirection, so a
// block may sit in the native pool or in reclaimed parameter memory
// (PAPER.md:161 PagedAttention; :558-564 reclaimed memory reused as KV).
//
// Design (HBM-bound gather, AI = G flop/B — CUDA cores, no tensor cores):
//   * grid = (units, H_kv); a unit is one (sequence, split) pair; CTA = 4 warps;
//     warp w handles blocks w, w+4, ... of the split (placement independent).
//   * one 16-token block of one (layer, kv-head) is a contiguous 2*16*D*2-byte
//     K|V tile, fetched whole by one cp.async.bulk (TMA engine) into shared
//     memory; every warp runs its own NS-deep ring (mbarrier complete_tx), so
//     NS tiles per warp are in flight while it computes; block addresses
//     (table -> block_base) are resolved 32 at a time, one per lane.
//   * lane owns 8 head dims (dims fixed per lane); QK partial dots are reduced
//     with a transpose-reduction (D/16 values across D/8 lanes in D/16 + 1
//     shuffles); online softmax in base 2; PV accumulates in registers.
//   * deterministic: fixed block->warp map, fixed warp merge order, fixed split
//     combine order by the last-arriving CTA (atomic ticket). Split sizes depend
//     only on logical lengths, so outputs are bit-identical under any physical
//     placement of the blocks (remap invariance).
#include <math_constants.h>
#include <stdlib.h>

#include "kernels.cuh"

namespace mirage {
namespace {


__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  f[0] = bf_lo(v.x); f[1] = bf_hi(v.x);
  f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
  f[4] = bf_lo(v.z); f[5] = bf_hi(v.z);
  f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
}

// ---- mbarrier / bulk-copy (TMA engine) helpers ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (cp.async.bulk).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}

constexpr int kMaxSplitsDev = 64;  // split-K partitions per (sequence, kv head)

template <int D, int W, int NS>
constexpr int smem_bytes() { return W * NS * 2 * (16 * D * 2); }

// W warps per CTA; every warp runs its own NS-deep ring of K|V tiles.
template <int D, int G, int W, int NS>
__global__ void __launch_bounds__(W * 32)
paged_attention_kernel(const AttnParams p) {
  constexpr int kWarps = W;
  constexpr int CPR = D / 8;        // 16-byte chunks per token row
  constexpr int TPI = 32 / CPR;     // token rows per warp-wide chunk sweep
  constexpr int ITERS = 16 / TPI;   // chunk sweeps per 16-token tile (== CPR / 2)
  constexpr int TILE = 16 * D * 2;  // bytes of K (or V) of one block/layer/head

  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarps][NS];

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const AttnUnit u = p.units[blockIdx.x];
  const int hk = blockIdx.y;
  const int s = u.seq;
  const int L = p.ctx_len[s];
  const int nblk = (L + 15) >> 4;
  const int b0 = u.split * p.split_blocks;
  const int b1 = min(b0 + p.split_blocks, nblk);
  const int dim0 = (lane % CPR) * 8;
  const int32_t* tbl = p.tables + (size_t)s * p.tbl_pitch;
  const uint64_t head_off = p.layer_off + (uint64_t)hk * (2 * TILE);
  uint8_t* ring = smem + (size_t)warp * NS * 2 * TILE;
  // this warp's blocks: b0 + warp + kWarps * it, it < n_it
  const int first = b0 + warp;
  const int n_it = first < b1 ? (b1 - first + kWarps - 1) / kWarps : 0;

  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NS; ++i) mbar_init(&bars[warp][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // block addresses of iterations [base, base + 32) live one per lane
  int addr_base = 0;
  uint64_t my_addr = 0;
  if (lane < n_it) my_addr = p.block_base[tbl[first + kWarps * lane]] + head_off;
  auto addr_of = [&](int it) -> uint64_t {  // warp-uniform it within [addr_base, addr_base+32)
    return __shfl_sync(0xffffffffu, my_addr, it - addr_base);
  };
  // prologue: fill the ring
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    if (i < n_it) {
      const uint64_t a = addr_of(i);
      if (lane == 0) {
        mbar_expect_tx(&bars[warp][i], 2 * TILE);
        bulk_g2s(ring + i * 2 * TILE, reinterpret_cast<const void*>(a), 2 * TILE, &bars[warp][i]);
      }
    }
  }

  float qr[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float* qp = p.q + ((size_t)s * p.H + hk * G + g) * D + dim0;
    float4 a = *reinterpret_cast<const float4*>(qp);
    float4 b = *reinterpret_cast<const float4*>(qp + 4);
    qr[g][0] = a.x * p.scale_log2; qr[g][1] = a.y * p.scale_log2;
    qr[g][2] = a.z * p.scale_log2; qr[g][3] = a.w * p.scale_log2;
    qr[g][4] = b.x * p.scale_log2; qr[g][5] = b.y * p.scale_log2;
    qr[g][6] = b.z * p.scale_log2; qr[g][7] = b.w * p.scale_log2;
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -CUDART_INF_F;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[g][j] = 0.f;
  }

  // token held (after the transpose-reduction) by this lane, and the lane that
  // holds the score of the token whose V row this lane owns in sweep i.
  const int my_i = (lane >> 1) & (ITERS - 1);
  const int my_tok = my_i * TPI + lane / CPR;
  const int src_base = (lane / CPR) * CPR;

  for (int it = 0; it < n_it; ++it) {
    const int st = it % NS;
    const uint32_t phase = (it / NS) & 1;
    const int blk = first + kWarps * it;
    mbar_wait(&bars[warp][st], phase);
    const uint8_t* tile = ring + st * 2 * TILE;
    const bool valid = blk * 16 + my_tok < L;
    const bool tail = blk * 16 + 16 > L;
    float part[G][ITERS];
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      float kf[8];
      unpack8(lds128(tile + (i * 32 + lane) * 16), kf);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) a = fmaf(qr[g][j], kf[j], a);
        part[g][i] = a;
      }
    }
    float pr[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float* v = part[g];
      // transpose-reduction over the CPR lanes sharing a token row
      int n = ITERS;
#pragma unroll
      for (int mask = CPR / 2; mask >= 1; mask >>= 1) {
        if (n > 1) {
          const bool up = lane & mask;
          const int half = n / 2;
#pragma unroll
          for (int j = 0; j < ITERS / 2; ++j) {
            if (j < half) {
              const float keep = up ? v[j + half] : v[j];
              const float send = up ? v[j] : v[j + half];
              v[j] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
            }
          }
          n = half;
        } else {
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], mask);
        }
      }
      const float sc = valid ? v[0] : -CUDART_INF_F;
      float bm = sc;
#pragma unroll
      for (int mask = 1; mask < 32; mask <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, mask));
      const float m_new = fmaxf(m[g], bm);
      const float alpha = exp2f(m[g] - m_new);
      pr[g] = valid ? exp2f(sc - m_new) : 0.f;
      float ps = pr[g];
#pragma unroll
      for (int mask = 2; mask < 32; mask <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, mask);
      l[g] = l[g] * alpha + ps;
      m[g] = m_new;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] *= alpha;
    }
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      float pi[G];
#pragma unroll
      for (int g = 0; g < G; ++g) pi[g] = __shfl_sync(0xffffffffu, pr[g], src_base + (i << 1));
      // rows past the context may hold any bytes (NaN/Inf): skip, don't multiply by 0
      if (tail && blk * 16 + i * TPI + lane / CPR >= L) continue;
      float vf[8];
      unpack8(lds128(tile + TILE + (i * 32 + lane) * 16), vf);
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[g][j] = fmaf(pi[g], vf[j], acc[g][j]);
    }
    // refill this stage with iteration it + NS (all lanes are done reading it)
    const int nx = it + NS;
    if (nx < n_it) {
      if (nx - addr_base >= 32) {  // next window of 32 block addresses
        addr_base += 32;
        const int j = addr_base + lane;
        my_addr = j < n_it ? p.block_base[tbl[first + kWarps * j]] + head_off : 0;
      }
      const uint64_t a = addr_of(nx);
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[warp][st], 2 * TILE);
        bulk_g2s(ring + st * 2 * TILE, reinterpret_cast<const void*>(a), 2 * TILE, &bars[warp][st]);
      }
    }
  }
  // lanes with equal lane % CPR hold the same dims for different token rows
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int mask = CPR; mask < 32; mask <<= 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], mask);

  __shared__ float sm_m[kWarps][G], sm_l[kWarps][G];
  __shared__ __align__(16) float sm_acc[kWarps][G][D];
  if (lane < CPR) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int j = 0; j < 8; ++j) sm_acc[warp][g][dim0 + j] = acc[g][j];
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      sm_m[warp][g] = m[g];
      sm_l[warp][g] = l[g];
    }
  }
  __syncthreads();

  // merge the warps in fixed order; thread t handles (g, d) pairs
  const bool split = u.nsplit > 1;
  for (int e = threadIdx.x; e < G * D; e += kWarps * 32) {
    const int g = e / D, d = e % D;
    float M = sm_m[0][g];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) M = fmaxf(M, sm_m[w][g]);
    float Ls = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float f = (sm_m[w][g] == -CUDART_INF_F) ? 0.f : exp2f(sm_m[w][g] - M);
      Ls += f * sm_l[w][g];
      o += f * sm_acc[w][g][d];
    }
    const int h = hk * G + g;
    if (!split) {
      const float r = o / Ls;
      const size_t oi = ((size_t)s * p.H + h) * D + d;
      if (p.out_fp32) reinterpret_cast<float*>(p.out)[oi] = r;
      else reinterpret_cast<__nv_bfloat16*>(p.out)[oi] = __float2bfloat16_rn(r);
    } else {
      float* rec = p.partial + ((size_t)(u.pbase + u.split) * p.H + h) * (D + 2);
      rec[d] = o;
      if (d == 0) {
        rec[D] = M;
        rec[D + 1] = Ls;
      }
    }
  }
  if (!split) return;

  // ---- split-K combine by the last-arriving CTA of this (seq, kv-head) ----
  __shared__ int am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* t = p.tickets + (size_t)s * p.H_kv + hk;
    const int prev = atomicAdd(t, 1);
    am_last = (prev == u.nsplit - 1);
    if (am_last) *t = 0;  // reset for the next launch
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // split weights w_i = 2^(m_i - M), Lambda = sum_i w_i l_i (fixed order i = 0..S-1)
  __shared__ float sw[kMaxSplitsDev][G];
  __shared__ float sL[G];
  const size_t stride = (size_t)p.H * (D + 2);
  const float* rec0 = p.partial + ((size_t)u.pbase * p.H + hk * G) * (D + 2);
  for (int e = threadIdx.x; e < u.nsplit * G; e += kWarps * 32) {
    const int i = e / G, g = e % G;
    sw[i][g] = __ldcg(rec0 + i * stride + g * (D + 2) + D);
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    float M = -CUDART_INF_F;
    for (int i = 0; i < u.nsplit; ++i) M = fmaxf(M, sw[i][g]);
    float Ls = 0.f;
    for (int i = 0; i < u.nsplit; ++i) {
      const float w = exp2f(sw[i][g] - M);
      Ls += w * __ldcg(rec0 + i * stride + g * (D + 2) + D + 1);
      sw[i][g] = w;
    }
    sL[g] = Ls;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * D; e += kWarps * 32) {
    const int g = e / D, d = e % D;
    const float* rec = rec0 + g * (D + 2) + d;
    float o = 0.f;
    int i = 0;
    for (; i + 4 <= u.nsplit; i += 4) {  // independent loads in flight
      const float a0 = __ldcg(rec + (i + 0) * stride), a1 = __ldcg(rec + (i + 1) * stride);
      const float a2 = __ldcg(rec + (i + 2) * stride), a3 = __ldcg(rec + (i + 3) * stride);
      o += sw[i][g] * a0;
      o += sw[i + 1][g] * a1;
      o += sw[i + 2][g] * a2;
      o += sw[i + 3][g] * a3;
    }
    for (; i < u.nsplit; ++i) o += sw[i][g] * __ldcg(rec + i * stride);
    const float r = o / sL[g];
    const size_t oi = ((size_t)s * p.H + hk * G + g) * D + d;
    if (p.out_fp32) reinterpret_cast<float*>(p.out)[oi] = r;
    else reinterpret_cast<__nv_bfloat16*>(p.out)[oi] = __float2bfloat16_rn(r);
  }
}

template <int D, int G, int W, int NS>
cudaError_t launch_v(const AttnParams& p, cudaStream_t s) {
  constexpr int SMEM = smem_bytes<D, W, NS>();
  static bool configured = false;  // opt in to > 48 KB dynamic shared memory once
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(paged_attention_kernel<D, G, W, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.n_units, p.H_kv);
  paged_attention_kernel<D, G, W, NS><<<grid, W * 32, SMEM, s>>>(p);
  return cudaGetLastError();
}

// tuning hook: MIRAGE_ATTN_VARIANT=0..3 selects (warps, stages) for D=128, G=1
int variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MIRAGE_ATTN_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int D, int G>
cudaError_t launch_dg(const AttnParams& p, cudaStream_t s) {
  if (D == 128 && G == 1) {
    switch (variant()) {
      case 1: return launch_v<D, G, 4, 3>(p, s);
      case 2: return launch_v<D, G, 8, 2>(p, s);
      case 3: return launch_v<D, G, 2, 4>(p, s);
      default: break;
    }
  }
  return launch_v<D, G, 4, D == 128 ? 2 : 4>(p, s);
}

template <int D>
cudaError_t launch_d(const AttnParams& p, cudaStream_t s) {
  switch (p.H / p.H_kv) {
    case 1: return launch_dg<D, 1>(p, s);
    case 2: return launch_dg<D, 2>(p, s);
    case 4: return launch_dg<D, 4>(p, s);
    case 8: return launch_dg<D, 8>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_paged_attention(const AttnParams& p, cudaStream_t s) {
  if (p.n_units == 0) return cudaSuccess;
  if (p.D == 128) return launch_d<128>(p, s);
  if (p.D == 64) return launch_d<64>(p, s);
  return cudaErrorInvalidValue;
}

}  // namespace mirage
