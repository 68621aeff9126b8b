// Dense-layer support kernels of the decode step:
// embedding + norm, residual + bias + norm, QKV post-processing fused with RoPE
// and the paged KV append, activations, argmax, and the KV fill/write hooks.
// These are not MIRAGE's contribution (the method leaves the
// model's kernels unchanged); they exist so that the whole step runs in this
// library's own kernels between cuBLAS GEMMs.
#include <math_constants.h>

#include <algorithm>

#include "kernels.cuh"

namespace mirage {
namespace {

// KV tile row layout (include/mirage.h): element c of token row r sits in
// 16-byte chunk (c / 8) ^ (r & 7) -- the swizzle the attention kernel's
// ldmatrix reads are conflict-free under.
__device__ __forceinline__ int swz(int c, int r) { return (((c >> 3) ^ (r & 7)) << 3) | (c & 7); }

__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
// 8 consecutive q elements (scaled) -> 4 words of part 0 (bf16 hi) at p and 4
// words of part 1 (lo = bf16(x - hi)) at p + D/2; word k packs elements 2k, 2k+1.
__device__ __forceinline__ void store_q_split(uint32_t* p, const float (&v)[8], float sc, int D) {
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float a = v[2 * k] * sc, b = v[2 * k + 1] * sc;
    const __nv_bfloat16 ah = __float2bfloat16_rn(a), bh = __float2bfloat16_rn(b);
    const __nv_bfloat16 al = __float2bfloat16_rn(a - __bfloat162float(ah));
    const __nv_bfloat16 bl = __float2bfloat16_rn(b - __bfloat162float(bh));
    hi[k] = (uint32_t)__bfloat16_as_ushort(ah) | ((uint32_t)__bfloat16_as_ushort(bh) << 16);
    lo[k] = (uint32_t)__bfloat16_as_ushort(al) | ((uint32_t)__bfloat16_as_ushort(bl) << 16);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(p + D / 2) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

__global__ void q_split_kernel(int64_t n8, int D, const float* q, float sc, uint32_t* out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the attention launch may start its prologue
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8, row = e / D;
    const int col = (int)(e % D);
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = q[e + k];
    uint32_t* dst = out + row * D + col / 2;  // word i of a part packs dims 2i, 2i+1
    store_q_split(dst, v, sc, D);
  }
}

__device__ __forceinline__ void load8bf(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[2 * k] = __uint_as_float(w[k] << 16);
    v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack8bf(const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    w[k] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * k])) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v[2 * k + 1])) << 16);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// block-wide sum, fixed order (deterministic); blockDim.x is a multiple of 32 and
// red is 16-byte aligned with room for 32 floats. The per-warp sums are read back
// as float4s (8 loads instead of up to 32) and added in warp order.
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  if (threadIdx.x < 32 && threadIdx.x >= nw) red[threadIdx.x] = 0.f;  // pad to whole float4s
  __syncthreads();
  float t = 0.f;
  const float4* r4 = reinterpret_cast<const float4*>(red);
  for (int i = 0; i < (nw + 3) / 4; ++i) {
    const float4 q = r4[i];
    t += q.x;
    t += q.y;
    t += q.z;
    t += q.w;
  }
  return t;
}

// A row of d fp32 elements is held CH float4 chunks per thread: thread t owns
// chunks t, t + T, ..., t + (CH - 1) T (T = blockDim.x), so each load instruction
// of a warp reads 512 consecutive bytes; chunks past d / 4 are not owned (zeros).
// CH = 4 for d >= 4096 keeps a block at <= 512 threads, so two or three rows
// are resident per SM at <= 64 registers and a decode batch runs in one wave.
__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void ld4cg(const float* p, float (&v)[4]) {  // L2 only (peer-written slots)
  const float4 a = __ldcg(reinterpret_cast<const float4*>(p));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
__device__ __forceinline__ void st4(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void unpack4bf(uint2 u, float (&v)[4]) {
  v[0] = __uint_as_float(u.x << 16);
  v[1] = __uint_as_float(u.x & 0xffff0000u);
  v[2] = __uint_as_float(u.y << 16);
  v[3] = __uint_as_float(u.y & 0xffff0000u);
}
__device__ __forceinline__ uint2 ld4bfw(const __nv_bfloat16* p) { return *reinterpret_cast<const uint2*>(p); }
__device__ __forceinline__ void ld4bf(const __nv_bfloat16* p, float (&v)[4]) { unpack4bf(ld4bfw(p), v); }
__device__ __forceinline__ uint2 pack4bf(const float (&v)[4]) {
  return make_uint2((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v[0])) |
                        ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v[1])) << 16),
                    (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v[2])) |
                        ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v[3])) << 16));
}
__host__ __device__ constexpr int row_chunks(int d) { return d >= 4096 ? 4 : 2; }
inline int row_threads(int d) { return ((d / 4 + row_chunks(d) - 1) / row_chunks(d) + 31) / 32 * 32; }

// Normalise the row and write bf16 x. family 0: LayerNorm (two-pass mean/var),
// 1: RMSNorm. Each thread sums its own elements in chunk order, then the block
// sums the per-thread values in fixed order (deterministic).
template <int CH>
__device__ __forceinline__ void norm_row(int family, int d, const float (&v)[CH][4], const __nv_bfloat16* g,
                                         const __nv_bfloat16* bta, float eps, __nv_bfloat16* x, float* red) {
  const int T = blockDim.x, nc = d >> 2;
  uint2 gw[CH], bw[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {  // issue the parameter loads before the reductions
    const int c = j * T + threadIdx.x;
    if (c < nc) {
      gw[j] = ld4bfw(g + 4 * c);
      if (family == 0) bw[j] = ld4bfw(bta + 4 * c);
    }
  }
  float mean = 0.f, q = 0.f;
  if (family == 0) {
    float sm = 0.f;
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) sm += v[j][k];  // unowned chunks are zero
    mean = block_sum(sm, red) / d;
  }
#pragma unroll
  for (int j = 0; j < CH; ++j)
    if (j * T + (int)threadIdx.x < nc)
#pragma unroll
      for (int k = 0; k < 4; ++k) q += (v[j][k] - mean) * (v[j][k] - mean);
  const float r = rsqrtf(block_sum(q, red) / d + eps);
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = j * T + threadIdx.x;
    if (c < nc) {
      float gv[4], out[4];
      unpack4bf(gw[j], gv);
      if (family == 0) {
        float bv[4];
        unpack4bf(bw[j], bv);
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = (v[j][k] - mean) * r * gv[k] + bv[k];
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = v[j][k] * r * gv[k];
      }
      *reinterpret_cast<uint2*>(x + 4 * c) = pack4bf(out);
    }
  }
}

template <int CH>
__global__ void __launch_bounds__(512, 2)
embed_norm_kernel(int family, int d, const int32_t* tokens, const int32_t* positions,
                  const __nv_bfloat16* embed, const __nv_bfloat16* pos_embed,
                  const __nv_bfloat16* g, const __nv_bfloat16* bta, float eps, float* h,
                  __nv_bfloat16* x) {
  __shared__ __align__(16) float red[32];
  const int b = blockIdx.x, T = blockDim.x, nc = d >> 2;
  float v[CH][4] = {};
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = j * T + threadIdx.x;
    if (c < nc) {
      ld4bf(embed + (size_t)tokens[b] * d + 4 * c, v[j]);
      if (family == 0) {
        float pv[4];
        ld4bf(pos_embed + (size_t)(positions[b] + 2) * d + 4 * c, pv);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[j][k] += pv[k];
      }
      st4(h + (size_t)b * d + 4 * c, v[j]);
    }
  }
  norm_row<CH>(family, d, v, g, bta, eps, x + (size_t)b * d, red);
}

// h[b] += y[b] (+ bias) if y != nullptr; then x[b] = bf16(norm(h[b])) if g != nullptr.
// y may hold nsplit split-K slices (the tcgen05 decode GEMM's output), `slice`
// floats apart: they are summed in slice order, then added.
template <int CH>
__global__ void __launch_bounds__(512, 2)
residual_norm_kernel(int family, int d, const float* y, int ldy, int nsplit, long long slice,
                     const __nv_bfloat16* bias, const __nv_bfloat16* g, const __nv_bfloat16* bta, float eps,
                     float* h, __nv_bfloat16* x) {
  __shared__ __align__(16) float red[32];
  const int b = blockIdx.x, T = blockDim.x, nc = d >> 2;
  float v[CH][4] = {};
  // under programmatic dependent launch the preceding kernel is the GEMM that
  // writes y: h (and the bias) may be read before waiting for it, y only after
  // (without y, the preceding kernel may have written h: wait first)
  if (!y) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = j * T + threadIdx.x;
    if (c < nc) ld4(h + (size_t)b * d + 4 * c, v[j]);
  }
  if (y) {
    // every load of the row is issued before the first store (a store to h between
    // them would serialise one DRAM round trip per chunk: the compiler cannot
    // prove h and y apart)
    uint2 bw[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (bias && j * T + (int)threadIdx.x < nc) bw[j] = ld4bfw(bias + 4 * (j * T + threadIdx.x));
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float yv[CH][4];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = j * T + threadIdx.x;
      if (c < nc) ld4(y + (size_t)b * ldy + 4 * c, yv[j]);
    }
    for (int s_ = 1; s_ < nsplit; ++s_)
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = j * T + threadIdx.x;
        if (c < nc) {
          float ys[4];
          ld4(y + s_ * slice + (size_t)b * ldy + 4 * c, ys);
#pragma unroll
          for (int k = 0; k < 4; ++k) yv[j][k] += ys[k];
        }
      }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = j * T + threadIdx.x;
      if (c < nc) {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[j][k] += yv[j][k];
        if (bias) {
          float bv[4];
          unpack4bf(bw[j], bv);
#pragma unroll
          for (int k = 0; k < 4; ++k) v[j][k] += bv[k];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = j * T + threadIdx.x;
      if (c < nc) st4(h + (size_t)b * d + 4 * c, v[j]);
    }
  }
  if (g) norm_row<CH>(family, d, v, g, bta, eps, x + (size_t)b * d, red);
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// h[b] += sum over ranks r (fixed order) of parts[r][b] (+ bias), then the norm
template <int CH>
__device__ __forceinline__ void tp_sum_norm(int family, int d, const float* const* parts, int tp, bool cg,
                                            const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                            const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                            float* red) {
  const int b = blockIdx.x, T = blockDim.x, nc = d >> 2;
  float v[CH][4] = {};
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = j * T + threadIdx.x;
    if (c < nc) ld4(h + (size_t)b * d + 4 * c, v[j]);
  }
  for (int r = 0; r < tp; ++r)  // fixed order: every rank computes the same sum
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = j * T + threadIdx.x;
      if (c < nc) {
        float pv[4];
        if (cg) ld4cg(parts[r] + (size_t)b * d + 4 * c, pv);
        else ld4(parts[r] + (size_t)b * d + 4 * c, pv);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[j][k] += pv[k];
      }
    }
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = j * T + threadIdx.x;
    if (c < nc) {
      if (bias) {
        float bv[4];
        ld4bf(bias + 4 * c, bv);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[j][k] += bv[k];
      }
      st4(h + (size_t)b * d + 4 * c, v[j]);
    }
  }
  if (g) norm_row<CH>(family, d, v, g, bta, eps, x + (size_t)b * d, red);
}

template <int CH>
__global__ void __launch_bounds__(512, 2)
tp_residual_norm_kernel(int family, int d, const float* const* parts, int tp, int rank,
                        unsigned long long* const* flags, unsigned long long epoch, unsigned int* err,
                        const __nv_bfloat16* bias, const __nv_bfloat16* g, const __nv_bfloat16* bta, float eps,
                        float* h, __nv_bfloat16* x) {
  __shared__ __align__(16) float red[32];
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    if (b == 0) {  // my partial (written by the preceding GEMM) is complete: publish
      __threadfence_system();
      st_release_sys(flags[rank], epoch);
    }
    for (int r = 0; r < tp; ++r) {  // bounded spin: a lost peer raises err instead of hanging
      if (r == rank) continue;
      long long n = 0;
      while (ld_acquire_sys(flags[r]) < epoch) {
        if (++n > (1ll << 26)) {
          atomicAdd(err, 1u);
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
  tp_sum_norm<CH>(family, d, parts, tp, false, bias, g, bta, eps, h, x, red);
}

template <int CH>
__global__ void __launch_bounds__(512, 2)
tp_push_residual_norm_kernel(int family, int d, const float* const* slots, int tp, const unsigned long long* cnt,
                             unsigned long long expect, unsigned int* err, const __nv_bfloat16* bias,
                             const __nv_bfloat16* g, const __nv_bfloat16* bta, float eps, float* h,
                             __nv_bfloat16* x) {
  __shared__ __align__(16) float red[32];
  if (threadIdx.x == 0) {
    for (int r = 0; r < tp; ++r) {  // every rank's tiles of this GEMM have landed here
      long long n = 0;
      while (ld_acquire_sys(cnt + r) < expect) {
        if (++n > (1ll << 26)) {
          atomicAdd(err, 1u);
          break;
        }
        __nanosleep(32);
      }
    }
  }
  __syncthreads();
  tp_sum_norm<CH>(family, d, slots, tp, true, bias, g, bta, eps, h, x, red);
}

// One CTA per sequence. Adds the bias, applies rotate-half RoPE (Llama) with the
// angle pos * theta^(-2i/D) evaluated in fp64, writes q (fp32) and appends k, v
// (bf16) into the paged cache row of position pos. Work items are 8-element
// chunks: (head, chunk pair c, c + D/16) for q/k, (kv head, chunk) for v.
__global__ void __launch_bounds__(256)
qkv_post_kernel(int family, int H, int Hk, int D, const float* qkv, const __nv_bfloat16* bias,
                const int32_t* positions, const int32_t* seq_off, const uint64_t* addrs,
                uint64_t layer_off, float rope_theta, float q_scale, uint32_t* q) {
  // the attention launch that follows may start its prologue (barriers, its first
  // work item's metadata) now; it waits (griddepcontrol.wait) before reading q / K / V
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ float cs[];  // [D/2] cos, [D/2] sin
  const int b = blockIdx.x;  // row; blockIdx.y = slice of the row's work items (one per thread)
  const int pos = positions[b];
  const int half = D / 2, hc = D / 16;  // chunks per half row
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
  char* kvbase = reinterpret_cast<char*>(addrs[seq_off[b] + (pos >> 4)] + layer_off);
  const int r = pos & 15;
  const int n_qk = (H + Hk) * hc, n_v = Hk * (D / 8);
  // the rotation angles and the cache address above need only this step's
  // metadata; the QKV GEMM's output is read from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < n_qk + n_v; e += gridDim.y * blockDim.x) {
    if (e < n_qk) {
      const int hh = e / hc, c = e % hc;
      const int c0 = hh * D + c * 8, c1 = c0 + half;
      float x0[8], x1[8];
      load8(row + c0, x0);
      load8(row + c1, x1);
      if (bias) {
        float b0[8], b1[8];
        load8bf(bias + c0, b0);
        load8bf(bias + c1, b1);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          x0[k] += b0[k];
          x1[k] += b1[k];
        }
      }
      if (family == 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float co = cs[c * 8 + k], si = cs[half + c * 8 + k];
          const float y0 = x0[k] * co - x1[k] * si, y1 = x1[k] * co + x0[k] * si;
          x0[k] = y0;
          x1[k] = y1;
        }
      }
      if (hh < H) {  // q * scale, split into bf16 hi | lo word pairs (AttnParams::q)
        uint32_t* qd = q + ((size_t)b * H + hh) * D + c * 4;
        store_q_split(qd, x0, q_scale, D);
        store_q_split(qd + half / 2, x1, q_scale, D);
      } else {
        char* dst = kvbase + ((size_t)((hh - H) * 2 + 0) * 16 + r) * D * 2;
        *reinterpret_cast<uint4*>(dst + ((c ^ (r & 7)) << 4)) = pack8bf(x0);
        *reinterpret_cast<uint4*>(dst + (((c + hc) ^ (r & 7)) << 4)) = pack8bf(x1);
      }
    } else {
      const int e2 = e - n_qk;
      const int kh = e2 / (D / 8), c = e2 % (D / 8);
      const int col = (H + Hk) * D + kh * D + c * 8;
      float x0[8];
      load8(row + col, x0);
      if (bias) {
        float b0[8];
        load8bf(bias + col, b0);
#pragma unroll
        for (int k = 0; k < 8; ++k) x0[k] += b0[k];
      }
      char* dst = kvbase + ((size_t)(kh * 2 + 1) * 16 + r) * D * 2;
      *reinterpret_cast<uint4*>(dst + ((c ^ (r & 7)) << 4)) = pack8bf(x0);
    }
  }
}

// 8 elements per thread. OPT: f = bf16(relu(y + b)); Llama: f = bf16(silu(g) * u),
// y = [gate | up] per row.
__global__ void act_kernel(int family, int B, int f, const float* y, const __nv_bfloat16* bias,
                           __nv_bfloat16* out) {
  const size_t n = (size_t)B * f / 8;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t b = e * 8 / f, i = e * 8 % f;
    float r[8];
    if (family == 0) {
      float bv[8];
      load8(y + b * f + i, r);
      load8bf(bias + i, bv);
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = fmaxf(r[k] + bv[k], 0.f);
    } else {
      float gt[8], up[8];
      load8(y + b * 2 * f + i, gt);
      load8(y + b * 2 * f + f + i, up);
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = gt[k] / (1.f + __expf(-gt[k])) * up[k];
    }
    *reinterpret_cast<uint4*>(out + e * 8) = pack8bf(r);
  }
}

__global__ void __launch_bounds__(1024) argmax_kernel(int V, const float* logits, int32_t* out) {
  const int b = blockIdx.x;
  const float* row = logits + (size_t)b * V;
  float best = -CUDART_INF_F;
  int bi = 0x7fffffff;
  // indices increase per thread, so a strict > keeps the lowest index on ties
  if ((V & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int V4 = V >> 2;
#pragma unroll 4
    for (int i = threadIdx.x; i < V4; i += blockDim.x) {
      const float4 q = __ldcs(r4 + i);  // read once: stream past L1/L2
      if (q.x > best) { best = q.x; bi = 4 * i; }
      if (q.y > best) { best = q.y; bi = 4 * i + 1; }
      if (q.z > best) { best = q.z; bi = 4 * i + 2; }
      if (q.w > best) { best = q.w; bi = 4 * i + 3; }
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      const float v = row[i];
      if (v > best) {
        best = v;
        bi = i;
      }
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

__global__ void tag_check_kernel(const uint32_t* tag, uint32_t expected, uint32_t* errors) {
  const uint32_t got = *reinterpret_cast<const volatile uint32_t*>(tag);
  if (got != expected) {
    atomicAdd(errors, 1u);
    errors[1] = got;
  }
}

__global__ void spin_kernel(uint64_t ns) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
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
  if (d % 8 || d > 8192) return cudaErrorInvalidValue;
  if (row_chunks(d) == 4)
    embed_norm_kernel<4><<<B, row_threads(d), 0, s>>>(family, d, tokens, positions, embed, pos_embed, g, bta, eps,
                                                      h, x);
  else
    embed_norm_kernel<2><<<B, row_threads(d), 0, s>>>(family, d, tokens, positions, embed, pos_embed, g, bta, eps,
                                                      h, x);
  return cudaGetLastError();
}

cudaError_t launch_residual_norm(int family, int B, int d, const float* y, int ldy,
                                 const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                 const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                 cudaStream_t s, int nsplit, long long slice, bool pdl) {
  if (d % 8 || d > 8192 || nsplit < 1) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(B);
  cfg.blockDim = dim3(row_threads(d));
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (row_chunks(d) == 4)
    return cudaLaunchKernelEx(&cfg, residual_norm_kernel<4>, family, d, y, ldy, nsplit, slice, bias, g, bta, eps, h,
                              x);
  return cudaLaunchKernelEx(&cfg, residual_norm_kernel<2>, family, d, y, ldy, nsplit, slice, bias, g, bta, eps, h, x);
}

cudaError_t launch_qkv_post(int family, int B, int H, int Hk, int D, const float* qkv,
                            const __nv_bfloat16* bias, const int32_t* positions,
                            const int32_t* seq_off, const uint64_t* addrs, uint64_t layer_off,
                            float rope_theta, float q_scale, uint32_t* q, cudaStream_t s, bool pdl) {
  // one thread per work item: all of a row's loads are in flight at once (the
  // kernel is latency-bound at decode batch sizes)
  const int items = (H + Hk) * (D / 16) + Hk * (D / 8);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(B, (items + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = D * sizeof(float);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qkv_post_kernel, family, H, Hk, D, qkv, bias, positions, seq_off, addrs, layer_off,
                            rope_theta, q_scale, q);
}

__global__ void block_copy_kernel(BlockMoves m, uint64_t n16) {
  const uint4* src = reinterpret_cast<const uint4*>(m.src[blockIdx.y]);
  uint4* dst = reinterpret_cast<uint4*>(m.dst[blockIdx.y]);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

cudaError_t launch_block_copy(const BlockMoves& m, uint64_t bytes, cudaStream_t s) {
  if (m.n <= 0) return cudaSuccess;
  if (bytes % 16 || m.n > 16) return cudaErrorInvalidValue;
  const uint64_t n16 = bytes / 16;
  const unsigned gx = (unsigned)std::min<uint64_t>((n16 + 255) / 256, 148 * 4 / (unsigned)m.n + 1);
  block_copy_kernel<<<dim3(gx, m.n), 256, 0, s>>>(m, n16);
  return cudaGetLastError();
}

cudaError_t launch_q_split(int64_t n, int D, const float* q, float q_scale, uint32_t* out, cudaStream_t s) {
  if (n % 8 || D % 16) return cudaErrorInvalidValue;
  const int64_t n8 = n / 8;
  q_split_kernel<<<(int)std::min<int64_t>((n8 + 255) / 256, 4096), 256, 0, s>>>(n8, D, q, q_scale, out);
  return cudaGetLastError();
}

cudaError_t launch_act(int family, int B, int f, const float* y, const __nv_bfloat16* bias,
                       __nv_bfloat16* out, cudaStream_t s) {
  const size_t n = (size_t)B * f / 8;
  act_kernel<<<grid_for(n, 256), 256, 0, s>>>(family, B, f, y, bias, out);
  return cudaGetLastError();
}

cudaError_t launch_argmax(int B, int V, const float* logits, int32_t* out, cudaStream_t s) {
  argmax_kernel<<<B, 1024, 0, s>>>(V, logits, out);
  return cudaGetLastError();
}

cudaError_t launch_tp_push_residual_norm(int family, int B, int d, const float* const* slots, int tp,
                                         const unsigned long long* cnt, unsigned long long expect, unsigned int* err,
                                         const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                         const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                         cudaStream_t s) {
  if (d % 8 || d > 8192) return cudaErrorInvalidValue;
  if (row_chunks(d) == 4)
    tp_push_residual_norm_kernel<4><<<B, row_threads(d), 0, s>>>(family, d, slots, tp, cnt, expect, err, bias, g,
                                                                 bta, eps, h, x);
  else
    tp_push_residual_norm_kernel<2><<<B, row_threads(d), 0, s>>>(family, d, slots, tp, cnt, expect, err, bias, g,
                                                                 bta, eps, h, x);
  return cudaGetLastError();
}

cudaError_t launch_tp_residual_norm(int family, int B, int d, const float* const* parts, int tp, int rank,
                                    unsigned long long* const* flags, unsigned long long epoch,
                                    unsigned int* err, const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                    const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                    cudaStream_t s) {
  if (d % 8 || d > 8192) return cudaErrorInvalidValue;
  if (row_chunks(d) == 4)
    tp_residual_norm_kernel<4><<<B, row_threads(d), 0, s>>>(family, d, parts, tp, rank, flags, epoch, err, bias, g,
                                                            bta, eps, h, x);
  else
    tp_residual_norm_kernel<2><<<B, row_threads(d), 0, s>>>(family, d, parts, tp, rank, flags, epoch, err, bias, g,
                                                            bta, eps, h, x);
  return cudaGetLastError();
}

cudaError_t launch_tag_check(const uint32_t* tag, uint32_t expected, uint32_t* errors, cudaStream_t s) {
  tag_check_kernel<<<1, 1, 0, s>>>(tag, expected, errors);
  return cudaGetLastError();
}

cudaError_t launch_spin(uint64_t ns, cudaStream_t s) {
  spin_kernel<<<1, 1, 0, s>>>(ns);
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
