// Dense-layer support kernels of the decode step:
// embedding + norm, residual + bias + norm, QKV post-processing fused with RoPE
// and the paged KV append, activations, argmax, and the KV fill/write hooks.
// These are not MIRAGE's contribution (the method leaves the
// model's kernels unchanged); they exist so that the whole step runs in this
// library's own kernels between cuBLAS GEMMs.
#include <math_constants.h>

#include "kernels.cuh"

namespace mirage {
namespace {

constexpr int kNormThreads = 256;
constexpr int kMaxPerThread = 32;  // d <= 8192

__device__ __forceinline__ float bf(const __nv_bfloat16* p, int i) { return __bfloat162float(p[i]); }

// KV tile row layout (include/mirage.h): element c of token row r sits in
// 16-byte chunk (c / 8) ^ (r & 7) -- the swizzle the attention kernel's
// ldmatrix reads are conflict-free under.
__device__ __forceinline__ int swz(int c, int r) { return (((c >> 3) ^ (r & 7)) << 3) | (c & 7); }

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];  // fixed order: deterministic
  return t;
}

// normalise the row held in v[] (fp32) and write bf16 x. family 0: LayerNorm
// (two-pass mean/var), 1: RMSNorm.
__device__ __forceinline__ void norm_row(int family, int d, float (&v)[kMaxPerThread], int cnt,
                                         const __nv_bfloat16* g, const __nv_bfloat16* bta,
                                         float eps, __nv_bfloat16* x, float* red) {
  const int tid = threadIdx.x;
  if (family == 0) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxPerThread; ++k)
      if (k < cnt) s += v[k];
    const float mean = block_sum<kNormThreads>(s, red) / d;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxPerThread; ++k) {
      if (k < cnt) {
        const float c = v[k] - mean;
        q += c * c;
      }
    }
    const float var = block_sum<kNormThreads>(q, red) / d;
    const float r = rsqrtf(var + eps);
#pragma unroll
    for (int k = 0; k < kMaxPerThread; ++k) {
      if (k < cnt) {
        const int i = tid + k * kNormThreads;
        x[i] = __float2bfloat16_rn((v[k] - mean) * r * bf(g, i) + bf(bta, i));
      }
    }
  } else {
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxPerThread; ++k)
      if (k < cnt) q += v[k] * v[k];
    const float ms = block_sum<kNormThreads>(q, red) / d;
    const float r = rsqrtf(ms + eps);
#pragma unroll
    for (int k = 0; k < kMaxPerThread; ++k) {
      if (k < cnt) {
        const int i = tid + k * kNormThreads;
        x[i] = __float2bfloat16_rn(v[k] * r * bf(g, i));
      }
    }
  }
}

__global__ void __launch_bounds__(kNormThreads)
embed_norm_kernel(int family, int d, const int32_t* tokens, const int32_t* positions,
                  const __nv_bfloat16* embed, const __nv_bfloat16* pos_embed,
                  const __nv_bfloat16* g, const __nv_bfloat16* bta, float eps, float* h,
                  __nv_bfloat16* x) {
  __shared__ float red[kNormThreads / 32];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const __nv_bfloat16* e = embed + (size_t)tokens[b] * d;
  const __nv_bfloat16* pe = family == 0 ? pos_embed + (size_t)(positions[b] + 2) * d : nullptr;
  float v[kMaxPerThread];
  const int cnt = (d - tid + kNormThreads - 1) / kNormThreads;
#pragma unroll
  for (int k = 0; k < kMaxPerThread; ++k) {
    if (k < cnt) {
      const int i = tid + k * kNormThreads;
      float t = bf(e, i);
      if (pe) t += bf(pe, i);
      v[k] = t;
      h[(size_t)b * d + i] = t;
    }
  }
  norm_row(family, d, v, cnt, g, bta, eps, x + (size_t)b * d, red);
}

__global__ void __launch_bounds__(kNormThreads)
residual_norm_kernel(int family, int d, const float* y, int ldy, const __nv_bfloat16* bias,
                     const __nv_bfloat16* g, const __nv_bfloat16* bta, float eps, float* h,
                     __nv_bfloat16* x) {
  __shared__ float red[kNormThreads / 32];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  float v[kMaxPerThread];
  const int cnt = (d - tid + kNormThreads - 1) / kNormThreads;
#pragma unroll
  for (int k = 0; k < kMaxPerThread; ++k) {
    if (k < cnt) {
      const int i = tid + k * kNormThreads;
      float t = h[(size_t)b * d + i];
      if (y) {  // y == nullptr: norm only
        t += y[(size_t)b * ldy + i];
        if (bias) t += bf(bias, i);
        h[(size_t)b * d + i] = t;
      }
      v[k] = t;
    }
  }
  if (g) norm_row(family, d, v, cnt, g, bta, eps, x + (size_t)b * d, red);  // g == nullptr: add only
}

// One CTA per sequence. Adds the bias, applies rotate-half RoPE (Llama) with the
// angle pos * theta^(-2i/D) evaluated in fp64, writes q (fp32) and appends k, v
// (bf16) into the paged cache row of position pos.
__global__ void qkv_post_kernel(int family, int H, int Hk, int D, const float* qkv,
                                const __nv_bfloat16* bias, const int32_t* positions,
                                const int32_t* tables, int tbl_pitch, const uint64_t* block_base,
                                uint64_t layer_off, float rope_theta, float* q) {
  extern __shared__ float cs[];  // [D/2] cos, [D/2] sin
  const int b = blockIdx.x;
  const int pos = positions[b];
  const int half = D / 2;
  const int W = (H + 2 * Hk) * D;
  const float* row = qkv + (size_t)b * W;
  if (family == 1) {
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
      const double inv = pow((double)rope_theta, -2.0 * i / D);
      double sn, cn;
      sincos((double)pos * inv, &sn, &cn);
      cs[i] = (float)cn;
      cs[half + i] = (float)sn;
    }
    __syncthreads();
  }
  const int32_t blk = tables[(size_t)b * tbl_pitch + (pos >> 4)];
  char* kvbase = reinterpret_cast<char*>(block_base[blk] + layer_off);
  const int r = pos & 15;
  // q and k heads: pairs (i, i + D/2)
  for (int e = threadIdx.x; e < (H + Hk) * half; e += blockDim.x) {
    const int hh = e / half, i = e % half;
    const int c0 = hh * D + i, c1 = c0 + half;
    float x0 = row[c0], x1 = row[c1];
    if (bias) {
      x0 += bf(bias, c0);
      x1 += bf(bias, c1);
    }
    float y0 = x0, y1 = x1;
    if (family == 1) {
      const float c = cs[i], s = cs[half + i];
      y0 = x0 * c - x1 * s;
      y1 = x1 * c + x0 * s;
    }
    if (hh < H) {
      q[((size_t)b * H + hh) * D + i] = y0;
      q[((size_t)b * H + hh) * D + i + half] = y1;
    } else {
      const int kh = hh - H;
      __nv_bfloat16* dst =
          reinterpret_cast<__nv_bfloat16*>(kvbase + ((size_t)(kh * 2 + 0) * 16 + r) * D * 2);
      dst[swz(i, r)] = __float2bfloat16_rn(y0);
      dst[swz(i + half, r)] = __float2bfloat16_rn(y1);
    }
  }
  for (int e = threadIdx.x; e < Hk * D; e += blockDim.x) {
    const int kh = e / D, i = e % D;
    const int c = (H + Hk) * D + e;
    float x0 = row[c];
    if (bias) x0 += bf(bias, c);
    __nv_bfloat16* dst =
        reinterpret_cast<__nv_bfloat16*>(kvbase + ((size_t)(kh * 2 + 1) * 16 + r) * D * 2);
    dst[swz(i, r)] = __float2bfloat16_rn(x0);
  }
}

__global__ void act_kernel(int family, int B, int f, const float* y, const __nv_bfloat16* bias,
                           __nv_bfloat16* out) {
  const size_t n = (size_t)B * f;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t b = e / f, i = e % f;
    float r;
    if (family == 0) {
      r = fmaxf(y[b * f + i] + bf(bias, (int)i), 0.f);
    } else {
      const float gt = y[b * 2 * f + i], up = y[b * 2 * f + f + i];
      r = gt / (1.f + expf(-gt)) * up;
    }
    out[e] = __float2bfloat16_rn(r);
  }
}

__global__ void __launch_bounds__(1024) argmax_kernel(int V, const float* logits, int32_t* out) {
  const int b = blockIdx.x;
  const float* row = logits + (size_t)b * V;
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = row[i];
    if (v > best) {  // i increases per thread: keeps the lowest index on ties
      best = v;
      bi = i;
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, m);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sv[k] > best || (sv[k] == best && si[k] < bi)) {
        best = sv[k];
        bi = si[k];
      }
    out[b] = bi;
  }
}

// ---- counter-based KV generator (spec: oracle/kvgen.py header; independent
// implementation) ----------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// one thread per (row, 8-element chunk); a row is one token of one
// (layer, kv head, K|V). Writes 16 bytes.
__global__ void fill_kv_kernel(uint64_t seed, int64_t seq_id, int L, int Hk, int D, int p0,
                               int n, const int32_t* table, const uint64_t* block_base) {
  const int cpr = D / 8;
  const size_t total = (size_t)L * Hk * 2 * n * cpr;
  const uint64_t key = seed * 0x9E3779B97F4A7C15ull;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const int ch = (int)(e % cpr);
    uint32_t r = (uint32_t)(e / cpr);
    const int t = (int)(r % (uint32_t)n);
    r /= (uint32_t)n;
    const int kv = (int)(r & 1);
    r >>= 1;
    const int hk = (int)(r % (uint32_t)Hk);
    const int layer = (int)(r / (uint32_t)Hk);
    const int pos = p0 + t;
    const uint64_t base = (((uint64_t)seq_id * L + layer) * Hk + hk) * 2 + kv;
    const uint64_t idx0 = (base * (1ull << 20) + (uint64_t)pos) * (uint64_t)D + (uint64_t)(ch * 8);
    uint32_t packed[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t hsh = splitmix64((idx0 + j) ^ key);
      const float u = (float)(uint32_t)(hsh >> 40) * 5.9604644775390625e-08f;  // 2^-24
      float x = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
      if (kv == 0) x = __fmul_rn(x, 1.7320508f);
      const uint32_t b = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
      if (j & 1) packed[j >> 1] |= b << 16;
      else packed[j >> 1] = b;
    }
    const int32_t blk = table[pos >> 4];
    uint4* dst = reinterpret_cast<uint4*>(block_base[blk] +
                                          ((((uint64_t)layer * Hk + hk) * 2 + kv) * 16 + (pos & 15)) * D * 2 +
                                          ((ch ^ (pos & 7)) * 16));
    *dst = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
}

__global__ void write_kv_kernel(int L, int Hk, int D, int p0, int n, const __nv_bfloat16* src,
                                const int32_t* table, const uint64_t* block_base) {
  const size_t total = (size_t)L * Hk * 2 * n * D;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    size_t r = e / D;
    const int t = (int)(r % n);
    r /= n;
    const int kv = (int)(r % 2);
    r /= 2;
    const int hk = (int)(r % Hk);
    const int layer = (int)(r / Hk);
    const int pos = p0 + t;
    const int32_t blk = table[pos >> 4];
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(
        block_base[blk] + ((((uint64_t)layer * Hk + hk) * 2 + kv) * 16 + (pos & 15)) * D * 2);
    dst[swz(d, pos & 15)] = src[e];
  }
}

int grid_for(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g ? g : 1);
}

}  // namespace

cudaError_t launch_embed_norm(int family, int B, int d, const int32_t* tokens,
                              const int32_t* positions, const __nv_bfloat16* embed,
                              const __nv_bfloat16* pos_embed, const __nv_bfloat16* g,
                              const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                              cudaStream_t s) {
  if (d > kNormThreads * kMaxPerThread) return cudaErrorInvalidValue;
  embed_norm_kernel<<<B, kNormThreads, 0, s>>>(family, d, tokens, positions, embed, pos_embed, g,
                                               bta, eps, h, x);
  return cudaGetLastError();
}

cudaError_t launch_residual_norm(int family, int B, int d, const float* y, int ldy,
                                 const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                 const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                 cudaStream_t s) {
  if (d > kNormThreads * kMaxPerThread) return cudaErrorInvalidValue;
  residual_norm_kernel<<<B, kNormThreads, 0, s>>>(family, d, y, ldy, bias, g, bta, eps, h, x);
  return cudaGetLastError();
}

cudaError_t launch_qkv_post(int family, int B, int H, int Hk, int D, const float* qkv,
                            const __nv_bfloat16* bias, const int32_t* positions,
                            const int32_t* tables, int tbl_pitch, const uint64_t* block_base,
                            uint64_t layer_off, float rope_theta, float* q, cudaStream_t s) {
  qkv_post_kernel<<<B, 256, D * sizeof(float), s>>>(family, H, Hk, D, qkv, bias, positions, tables,
                                                    tbl_pitch, block_base, layer_off, rope_theta,
                                                    q);
  return cudaGetLastError();
}

cudaError_t launch_act(int family, int B, int f, const float* y, const __nv_bfloat16* bias,
                       __nv_bfloat16* out, cudaStream_t s) {
  const size_t n = (size_t)B * f;
  act_kernel<<<grid_for(n, 256), 256, 0, s>>>(family, B, f, y, bias, out);
  return cudaGetLastError();
}

cudaError_t launch_argmax(int B, int V, const float* logits, int32_t* out, cudaStream_t s) {
  argmax_kernel<<<B, 1024, 0, s>>>(V, logits, out);
  return cudaGetLastError();
}

cudaError_t launch_fill_kv(uint64_t seed, int64_t seq_id, int L, int Hk, int D, int p0, int n,
                           const int32_t* table, const uint64_t* block_base, cudaStream_t s) {
  const size_t total = (size_t)L * Hk * 2 * n * (D / 8);
  if (!total) return cudaSuccess;
  fill_kv_kernel<<<grid_for(total, 256), 256, 0, s>>>(seed, seq_id, L, Hk, D, p0, n, table,
                                                     block_base);
  return cudaGetLastError();
}

cudaError_t launch_write_kv(int L, int Hk, int D, int p0, int n, const __nv_bfloat16* src,
                            const int32_t* table, const uint64_t* block_base, cudaStream_t s) {
  const size_t total = (size_t)L * Hk * 2 * n * D;
  if (!total) return cudaSuccess;
  write_kv_kernel<<<grid_for(total, 256), 256, 0, s>>>(L, Hk, D, p0, n, src, table, block_base);
  return cudaGetLastError();
}

}  // namespace mirage
