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
//     K|V tile; a warp fetches it with 16-byte coalesced ld.global.nc (512 B per
//     instruction), software-prefetching the next block.
//   * lane owns 8 head dims (dims fixed per lane); QK partial dots are reduced
//     with a transpose-reduction (D/16 values across D/8 lanes in D/16 + 1
//     shuffles); online softmax in base 2; PV accumulates in registers.
//   * deterministic: fixed block->warp map, fixed warp merge order, fixed split
//     combine order by the last-arriving CTA (atomic ticket). Split sizes depend
//     only on logical lengths, so outputs are bit-identical under any physical
//     placement of the blocks (remap invariance).
#include <math_constants.h>

#include "kernels.cuh"

namespace mirage {
namespace {

constexpr int kWarps = 4;

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  f[0] = bf_lo(v.x); f[1] = bf_hi(v.x);
  f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
  f[4] = bf_lo(v.z); f[5] = bf_hi(v.z);
  f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
}

template <int D, int G>
__global__ void __launch_bounds__(kWarps * 32)
paged_attention_kernel(const AttnParams p) {
  constexpr int CPR = D / 8;        // 16-byte chunks per token row
  constexpr int TPI = 32 / CPR;     // token rows per warp-wide load
  constexpr int ITERS = 16 / TPI;   // loads per 16-token tile (== CPR / 2)
  constexpr int TILE = 16 * D * 2;  // bytes of K (or V) of one block/layer/head

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
  // holds the score of the token whose V row this lane owns in load i.
  const int my_i = (lane >> 1) & (ITERS - 1);
  const int my_tok = my_i * TPI + lane / CPR;
  const int src_base = (lane / CPR) * CPR;

  uint4 kr[ITERS], vr[ITERS];
  int blk = b0 + warp;
  if (blk < b1) {
    const char* base = reinterpret_cast<const char*>(p.block_base[tbl[blk]] + head_off);
#pragma unroll
    for (int i = 0; i < ITERS; ++i) {
      kr[i] = ldg_stream(base + (size_t)(i * 32 + lane) * 16);
      vr[i] = ldg_stream(base + TILE + (size_t)(i * 32 + lane) * 16);
    }
  }
  for (; blk < b1; blk += kWarps) {
    // prefetch the next block of this warp
    uint4 nk[ITERS], nv[ITERS];
    const int nb = blk + kWarps;
    if (nb < b1) {
      const char* base = reinterpret_cast<const char*>(p.block_base[tbl[nb]] + head_off);
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        nk[i] = ldg_stream(base + (size_t)(i * 32 + lane) * 16);
        nv[i] = ldg_stream(base + TILE + (size_t)(i * 32 + lane) * 16);
      }
    }
    const bool valid = blk * 16 + my_tok < L;
    const bool tail = blk * 16 + 16 > L;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float v[ITERS];
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        float kf[8];
        unpack8(kr[i], kf);
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) a = fmaf(qr[g][j], kf[j], a);
        v[i] = a;
      }
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
      const float pr = valid ? exp2f(sc - m_new) : 0.f;
      float ps = pr;
#pragma unroll
      for (int mask = 2; mask < 32; mask <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, mask);
      l[g] = l[g] * alpha + ps;
      m[g] = m_new;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[g][j] *= alpha;
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        const float pi = __shfl_sync(0xffffffffu, pr, src_base + (i << 1));
        // rows past the context may hold any bytes (NaN/Inf): skip, don't multiply by 0
        if (tail && blk * 16 + i * TPI + lane / CPR >= L) continue;
        float vf[8];
        unpack8(vr[i], vf);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[g][j] = fmaf(pi, vf[j], acc[g][j]);
      }
    }
    if (nb < b1) {
#pragma unroll
      for (int i = 0; i < ITERS; ++i) {
        kr[i] = nk[i];
        vr[i] = nv[i];
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
  for (int e = threadIdx.x; e < G * D; e += kWarps * 32) {
    const int g = e / D, d = e % D;
    const int h = hk * G + g;
    const float* rec0 = p.partial + ((size_t)u.pbase * p.H + h) * (D + 2);
    const size_t stride = (size_t)p.H * (D + 2);
    float M = -CUDART_INF_F;
    for (int i = 0; i < u.nsplit; ++i) M = fmaxf(M, __ldcg(rec0 + i * stride + D));
    float Ls = 0.f, o = 0.f;
    for (int i = 0; i < u.nsplit; ++i) {
      const float* rec = rec0 + i * stride;
      const float f = exp2f(__ldcg(rec + D) - M);
      Ls += f * __ldcg(rec + D + 1);
      o += f * __ldcg(rec + d);
    }
    const float r = o / Ls;
    const size_t oi = ((size_t)s * p.H + h) * D + d;
    if (p.out_fp32) reinterpret_cast<float*>(p.out)[oi] = r;
    else reinterpret_cast<__nv_bfloat16*>(p.out)[oi] = __float2bfloat16_rn(r);
  }
}

template <int D>
cudaError_t launch_d(const AttnParams& p, cudaStream_t s) {
  dim3 grid(p.n_units, p.H_kv);
  const int G = p.H / p.H_kv;
  switch (G) {
    case 1: paged_attention_kernel<D, 1><<<grid, kWarps * 32, 0, s>>>(p); break;
    case 2: paged_attention_kernel<D, 2><<<grid, kWarps * 32, 0, s>>>(p); break;
    case 4: paged_attention_kernel<D, 4><<<grid, kWarps * 32, 0, s>>>(p); break;
    case 8: paged_attention_kernel<D, 8><<<grid, kWarps * 32, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_paged_attention(const AttnParams& p, cudaStream_t s) {
  if (p.n_units == 0) return cudaSuccess;
  if (p.D == 128) return launch_d<128>(p, s);
  if (p.D == 64) return launch_d<64>(p, s);
  return cudaErrorInvalidValue;
}

}  // namespace mirage
