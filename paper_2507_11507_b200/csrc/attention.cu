// Paged-attention decode with fused split-K combine (a9)
// for sm_100a.
//
// Computes, for sequence s and query head h (KV head h' = h / G):
//   o = softmax(q K^T / sqrt(D)) V over the s's first ctx_len tokens,
// reading K/V through the block table (resolved per step to block addresses), so a
// block may sit in the native pool or in reclaimed parameter memory
// (PAPER.md:161 PagedAttention; :558-564 reclaimed memory reused as KV).
//
// Design (HBM-bound gather; AI = G flop/B):
//   * a work item is (sequence, split, kv head); a CTA = 4 warps, warp w takes
//     blocks w, w+4, ... of the item (placement independent). The grid is
//     persistent (one wave of CTAs); CTAs claim items from a global counter in
//     the host's longest-first order (greedy LPT), and each warp's TMA ring
//     streams straight across item boundaries, so no CTA launch/prologue
//     bubbles remain. In a prefill step (QP > 1) an item carries up to QP
//     consecutive rows of one sequence as extra query columns, each with its
//     own causal length, so one K|V pass serves QP rows.
//   * q arrives scaled by log2(e)/sqrt(D) and split into bf16 hi|lo words in
//     the MMA fragment order (qkv_post_kernel), staged per item by one bulk copy.
//   * one 16-token block of one (layer, kv-head) is a contiguous 2*16*D*2-byte
//     K|V tile, fetched whole by one cp.async.bulk (TMA engine) into shared
//     memory; every consumer warp has its own NS-deep ring (full/empty mbarrier
//     pairs) that a fifth, producer warp keeps filled, so NS tiles per warp are
//     in flight while it computes; block addresses (table -> block_base) are
//     resolved 32 at a time, one per lane.
//   * QK^T and PV run on the tensor cores (mma.sync m16n8k16 bf16 -> fp32) with
//     q and p carried as bf16 hi+lo column pairs (near-fp32 accuracy); this cuts
//     the per-tile instruction count ~6x versus CUDA-core dot products so the
//     kernel stays memory-bound for every group size G in {1, 2, 4, 8}.
//     Online softmax in base 2 on the accumulator fragments.
//   * deterministic: fixed block->warp map, fixed warp merge order, fixed split
//     combine order by the last-arriving CTA (atomic ticket). Split sizes depend
//     only on logical lengths, so outputs are bit-identical under any physical
//     placement of the blocks (remap invariance).
#include <math_constants.h>
#include <stdlib.h>

#include <algorithm>

#include "kernels.cuh"

namespace mirage {
namespace {


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

// the same with an L2 cache policy (createpolicy), e.g. evict_first for K|V tiles
// that are read exactly once per launch
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_s(uint32_t (&r)[4], uint32_t saddr) {  // shared-window address
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
__device__ __forceinline__ void ldsm_x4_t_s(uint32_t (&r)[4], uint32_t saddr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
// D[16x8] += A[16x16] * B[16x8], bf16 in, fp32 accumulate (tensor cores)
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// x = hi + lo with hi = bf16(x), lo = bf16(x - hi): the pair carries ~16 mantissa bits
__device__ __forceinline__ float bf16_part(float x, int part) {
  const float hi = __bfloat162float(__float2bfloat16_rn(x));
  return part ? x - hi : hi;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
  const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(lo_elem));
  const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(hi_elem));
  return a | (b << 16);
}

constexpr int kMaxSplitsDev = 128;  // split-K partitions per (sequence, kv head); runtime agrees
// partial record: o[D], m, l, 2 pad floats (16-byte rows for float4 combine loads)

template <int D, int G, int QP, int W, int NS>
constexpr int smem_bytes() { return W * NS * 2 * (16 * D * 2) + (NS + 1) * G * QP * D * 4; }

// 2^x on the MUFU with flush-to-zero: the softmax arguments are <= 0 after the max
// subtraction, and a probability below 2^-126 adds nothing to l >= 1
__device__ __forceinline__ float exp2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace slots per CTA (16): 0 entry, 1 first tiles issued, 2 first tile landed
// (warp 0), 3 last tile consumed (warp 0), 4 last item's output / partial written,
// 5 last combine done, 6 exit, 7 items processed, 9 every consumer warp done with
// the last item (merge starts); combine phases of the last combine: 8 ticket
// taken, 10 weights computed; 12-15 SM cycles from the merge start to the ticket,
// M of head 0, the weights barrier and the end of the fold
#define ATTN_TRACE(slot, val)                                              \
  do {                                                                     \
    if (p.trace) p.trace[(size_t)blockIdx.x * 16 + (slot)] = (val);        \
  } while (0)

// Programmatic dependent launch: let the next kernel of the stream start its
// prologue now / wait until the previous kernel's results are visible (no-ops
// when the launch carries no programmatic dependency)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Tensor-core formulation per 16-token tile (one warp):
//   S[16 tok x 8 col] = K[16 x D] * Qc[D x 8]      (D/16 mma.m16n8k16 per n-tile)
//   O^T[D x 8]       += V^T[D x 16] * P[16 x 8]    (D/16 mma per n-tile)
// where column n = 2*head + part holds the bf16 hi (part 0) or lo (part 1) half
// of q (resp. p), so the fp32 accumulators see q and p to ~16 mantissa bits
// while K and V stay exact bf16. G <= 4 heads fill one n8 tile, G = 8 two.
// Prefill items (QP > 1) carry QP consecutive rows of one sequence: the columns
// are GV = G * QP virtual heads (row pp = v / G, head g = v % G), each with its
// own causal length len + pp, so one K|V tile serves QP query rows.
// The KV tile is stored XOR-swizzled in 16-byte chunks (chunk ^ (row & 7), see
// include/mirage.h), which makes every ldmatrix below bank-conflict free.
// WS (warp-specialized): one extra producer warp claims the items, stages q and
// issues every TMA tile for the W consumer warps (full/empty mbarrier pairs per
// ring stage); the consumers only compute. Otherwise each warp runs its own
// producer inline (pump).
// resident CTAs per SM the register budget must allow (the shared-memory rings
// decide the rest): 3 for MHA decode (G = 1), 2 otherwise
template <int G, int QP>
constexpr int min_ctas() { return (G == 1 && QP == 1) ? 3 : 2; }

template <int D, int G, int QP, int W, int NS, bool WS>
__global__ void __launch_bounds__((W + (WS ? 1 : 0)) * 32, min_ctas<G, QP>())
paged_attention_kernel(const AttnParams p) {
  constexpr int GV = G * QP;          // query column groups (virtual heads) per item
  constexpr int kWarps = W;
  constexpr int TILE = 16 * D * 2;    // bytes of K (or V) of one block/layer/head
  constexpr int ROW = 2 * D;          // bytes per token row
  constexpr int KS = D / 16;          // k-slices (QK) == dim tiles (PV)
  constexpr int NT = (2 * GV + 7) / 8; // n8 tiles of (head, part) columns

  constexpr int QB = NS + 1;           // q staging buffers per CTA (warp 0's producer runs ahead)
  // FA: G = 8 decode puts the query side on the MMA's M dimension (rows = 8 heads x
  // {hi, lo} bf16 parts of q, or of p): S[16 x tok] = Qc K^T leaves each lane the
  // scores of ONE head for 4 tokens, so the row max needs 2 shuffles and P feeds
  // the PV MMA as its A operand straight from the accumulator registers (no
  // transposing shuffles): ~100 instead of ~260 instructions per 16-token tile,
  // same HMMA count (16 + 16).
  constexpr bool FA = G == 8 && QP == 1 && WS;

  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kWarps][NS];
  __shared__ __align__(8) uint64_t qbars[QB];
  __shared__ __align__(8) uint64_t empty[WS ? kWarps : 1][NS];  // WS: consumer released the stage
  __shared__ __align__(8) uint64_t slot_free[WS ? QB : 1];      // WS: all consumers read the slot's q
  __shared__ int ptiles[WS ? kWarps : 1];                       // WS: tiles issued per consumer warp
  __shared__ float sm_m[kWarps][GV], sm_l[kWarps][GV];
  // per-warp O partials of an item; reused by the split combine for the weights
  constexpr int ACC_C = (kMaxSplitsDev + 1) * G;
  constexpr int ACC = kWarps * D * GV > ACC_C ? kWarps * D * GV : ACC_C;
  __shared__ __align__(16) float sm_accf[ACC];
  float(*sm_acc)[GV][D] = reinterpret_cast<float(*)[GV][D]>(sm_accf);
  __shared__ int am_last;
  // dynamic item queue: CTA item k (in claim order) lives in slot k % QB
  __shared__ int slot_claim[QB];
  __shared__ unsigned long long slot_word[QB];  // ((k + 1) << 32) | item, published atomically

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int gq = lane >> 2;  // mma group id (row / column index)
  const int tq = lane & 3;   // thread in group
  const int n_flat = (p.n_units_dev ? *p.n_units_dev : p.n_units) * p.H_kv;  // item f = unit * H_kv + kv head
  uint8_t* ring = smem + (size_t)(warp < kWarps ? warp : 0) * NS * 2 * TILE;
  // items past the static first ones come from the global counter; when the grid
  // covers every item (the small-batch regime) nobody claims, and the counter
  // needs no reset at exit
  // Balanced ranges (schedule 1, decode): CTA b runs the units of range b / H_kv,
  // in order, for kv head b % H_kv; no queue
  const bool rmode = p.hdr != nullptr && p.hdr[1] == 1;
  int r_first = 0, r_end = 0, r_kvh = 0;
  if (rmode) {
    r_first = p.rfirst[blockIdx.x / p.H_kv];
    r_end = p.rfirst[blockIdx.x / p.H_kv + 1];
    r_kvh = blockIdx.x % p.H_kv;
  }
  const bool dyn = !rmode && n_flat > (int)gridDim.x;
  auto claim = [&]() -> int { return dyn ? (int)gridDim.x + atomicAdd(p.sched, 1) : n_flat; };
  // the CTA's k-th work item (item f = unit * H_kv + kv head)
  auto item_at = [&](int k) -> int {
    if (rmode) return r_first + k < r_end ? (r_first + k) * p.H_kv + r_kvh : n_flat;
    return k == 0 ? (int)blockIdx.x : claim();
  };
  // q staging (dynamic smem after the rings): [QB][G][2][D/2] packed bf16 hi|lo words, one copy per CTA item
  uint32_t(*qbuf)[GV * D] = reinterpret_cast<uint32_t(*)[GV * D]>(smem + (size_t)kWarps * NS * 2 * TILE);

  pdl_trigger();  // every CTA is resident (one wave): the next launch may start its prologue
  if (threadIdx.x == 0) ATTN_TRACE(0, gtimer());
  if (lane == 0 && warp < kWarps) {
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bars[warp][i], 1);
      if (WS) mbar_init(&empty[WS ? warp : 0][i], 1);
    }
    if (WS) ptiles[WS ? warp : 0] = 0;
    if (warp == 0)
#pragma unroll
      for (int i = 0; i < QB; ++i) {
        mbar_init(&qbars[i], 1);
        if (WS) mbar_init(&slot_free[WS ? i : 0], kWarps);
        slot_word[i] = 0ull;
        slot_claim[i] = i - QB;
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // q barriers and item slots are shared by the CTA
  // consumer-only CTA barrier (named barrier 1) when a producer warp is present
  auto csync = [&]() {
    if (WS) asm volatile("bar.sync 1, %0;" ::"r"(kWarps * 32) : "memory");
    else __syncthreads();
  };

  // ---- work items are claimed dynamically from a global counter (items are in
  // longest-first order, so this is greedy LPT). The first warp of the CTA to
  // need the CTA's k-th item claims it, stages its q rows by bulk copy and
  // publishes it in slot k % QB; the other warps read the slot. ----
  auto get_item = [&](int k) -> int {
    const int sl = k % QB;
    int item = 0;
    if (lane == 0) {
      if (atomicCAS(&slot_claim[sl], k - QB, k) == k - QB) {
        item = item_at(k);
        if (item < n_flat) {
          const AttnUnit u = p.units[item / p.H_kv];
          const int nq = QP == 1 ? 1 : u.nq;  // rows u.seq .. u.seq + nq - 1, G heads each
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&qbars[sl], nq * G * D * 4);
          for (int pp = 0; pp < nq; ++pp)
            bulk_g2s(&qbuf[sl][pp * G * D], p.q + ((size_t)(u.seq + pp) * p.H + (item % p.H_kv) * G) * D,
                     G * D * 4, &qbars[sl]);
        }
        atomicExch(&slot_word[sl], ((unsigned long long)(k + 1) << 32) | (unsigned int)item);
      } else {
        unsigned long long w;
        while (((w = atomicAdd(&slot_word[sl], 0ull)) >> 32) != (unsigned long long)(k + 1)) __nanosleep(32);
        item = (int)(unsigned int)(w & 0xffffffffull);
      }
    }
    return __shfl_sync(0xffffffffu, item, 0);
  };

  // ---- producer: walks this warp's tile stream (blocks warp, warp+W, ... of each
  // of the CTA's items; tile t goes to stage t % NS) up to NS tiles ahead of the
  // consumer, across item boundaries, so the ring never drains between items.
  // It never claims an item more than QB-1 items ahead of its own consumer: by
  // then every warp has passed the merge of the item that last used the slot.
  int pk = -1, p_it = 0, p_n = 0, addr_base = 0;
  bool p_done = false;
  uint32_t pt = 0, rc = 0;  // tiles issued / consumed by this warp
  const uint64_t* p_tbl = nullptr;
  uint64_t p_off = 0, my_addr = 0;
  auto pump = [&](int ck) {
    if (WS) return;
    while (pt < rc + NS && !p_done) {
      if (p_it >= p_n) {
        if (pk + 1 > ck + QB - 1) return;  // slot window
        const int pf = get_item(++pk);
        if (pf >= n_flat) {
          p_done = true;
          return;
        }
        const AttnUnit u = p.units[pf / p.H_kv];
        const int first = u.b0 + warp;
        p_n = first < u.b1 ? (u.b1 - first + kWarps - 1) / kWarps : 0;
        p_it = 0;
        p_tbl = p.addrs + u.addr_off + first;
        p_off = p.layer_off + (uint64_t)(pf % p.H_kv) * (2 * TILE);
        addr_base = 0;
        my_addr = lane < p_n ? p_tbl[kWarps * lane] + p_off : 0;
        continue;
      }
      if (p_it - addr_base >= 32) {  // next window of 32 block addresses
        addr_base += 32;
        const int j = addr_base + lane;
        my_addr = j < p_n ? p_tbl[kWarps * j] + p_off : 0;
      }
      const uint64_t a = __shfl_sync(0xffffffffu, my_addr, p_it - addr_base);
      const int stage = pt % NS;
      ++p_it;
      ++pt;
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bars[warp][stage], 2 * TILE);
        bulk_g2s(ring + stage * 2 * TILE, reinterpret_cast<const void*>(a), 2 * TILE, &bars[warp][stage]);
      }
    }
  };
  if (WS && warp == kWarps) {
    // ---- producer warp: claim items in order, stage q, then issue every tile of
    // the item to its consumer warp's ring (block j -> warp (j - b0) % W), waiting
    // on that stage's empty barrier once the ring has wrapped ----
    // The static first item's unit record and first 32 block addresses depend only
    // on this step's metadata: fetch them before waiting for the previous kernel
    // (qkv_post writes q and the new token's K/V), so under programmatic dependent
    // launch these loads overlap that kernel's tail.
    AttnUnit u_first{};
    uint64_t a_first = 0;
    if (rmode ? r_first < r_end : (int)blockIdx.x < n_flat) {
      u_first = p.units[rmode ? r_first : blockIdx.x / p.H_kv];
      const int j = u_first.b0 + lane;
      a_first = j < u_first.b1 ? p.addrs[u_first.addr_off + j] : 0;
    }
    const uint64_t kv_pol = policy_evict_first();
    int my_t = 0;  // (per-lane producer) tiles issued to this lane's warp
    pdl_wait();
    for (int k = 0;; ++k) {
      const int sl_ = k % QB;
      int item = 0;
      if (lane == 0) {
        if (k >= QB) mbar_wait(&slot_free[WS ? sl_ : 0], ((k / QB) - 1) & 1);
        // the first item is static (CTA b takes item b: no atomic on the critical
        // path of the first tiles); later ones come from the counter, in order
        item = item_at(k);
        if (item < n_flat) {
          const AttnUnit u = k == 0 ? u_first : p.units[item / p.H_kv];
          const int nq = QP == 1 ? 1 : u.nq;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&qbars[sl_], nq * G * D * 4);
          for (int pp = 0; pp < nq; ++pp)
            bulk_g2s(&qbuf[sl_][pp * G * D], p.q + ((size_t)(u.seq + pp) * p.H + (item % p.H_kv) * G) * D,
                     G * D * 4, &qbars[sl_]);
        }
        atomicExch(&slot_word[sl_], ((unsigned long long)(k + 1) << 32) | (unsigned int)item);
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= n_flat) break;
      if (k == 0 && lane == 0) ATTN_TRACE(1, gtimer());
      const AttnUnit u = k == 0 ? u_first : p.units[item / p.H_kv];
      const uint64_t off = p.layer_off + (uint64_t)(item % p.H_kv) * (2 * TILE);
      const uint64_t* tbl = p.addrs + u.addr_off;
      const int Lmax_u = u.len + (QP > 1 ? u.nq - 1 : 0);
      if (p.prod_lanes) {
        // one producer lane per consumer warp: lane w issues blocks b0 + w, b0 + w + W, ...
        // into warp w's ring and waits only on warp w's stages (no head-of-line blocking
        // behind another warp's slow tile); addresses fetched 8 per lane at a time
        uint64_t pre[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) pre[q] = __shfl_sync(0xffffffffu, a_first, min(31, (lane % kWarps) + kWarps * q));
        if (lane < kWarps) {
          for (int j0 = u.b0 + lane, win = 0; j0 < u.b1; j0 += 8 * kWarps, ++win) {
            uint64_t ad[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int j = j0 + kWarps * q;
              ad[q] = j < u.b1 ? ((k == 0 && win == 0) ? pre[q] : tbl[j]) : 0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int j = j0 + kWarps * q;
              if (j >= u.b1) break;
              const int st = my_t % NS;
              if (my_t >= NS) mbar_wait(&empty[WS ? lane : 0][st], ((my_t / NS) - 1) & 1);
              ++my_t;
              uint8_t* dst = smem + (size_t)lane * NS * 2 * TILE + st * 2 * TILE;
              const int vr = min(16, Lmax_u - j * 16);
              const uint32_t part = vr < 16 ? (uint32_t)vr * ROW : 2u * TILE;
              mbar_expect_tx(&bars[lane][st], vr < 16 ? 2 * part : part);
              const char* src = reinterpret_cast<const char*>(ad[q] + off);
              if (p.kv_evict_first) {
                bulk_g2s_hint(dst, src, part, &bars[lane][st], kv_pol);
                if (vr < 16) bulk_g2s_hint(dst + TILE, src + TILE, part, &bars[lane][st], kv_pol);
              } else {
                bulk_g2s(dst, src, part, &bars[lane][st]);
                if (vr < 16) bulk_g2s(dst + TILE, src + TILE, part, &bars[lane][st]);
              }
            }
          }
        }
        __syncwarp();
        continue;
      }
      for (int base = u.b0; base < u.b1; base += 32) {
        const int j = base + lane;
        const uint64_t a = j < u.b1 ? ((k == 0 && base == u.b0) ? a_first : tbl[j]) + off : 0;
        const int cnt = min(32, u.b1 - base);
        for (int i = 0; i < cnt; ++i) {
          const uint64_t ai = __shfl_sync(0xffffffffu, a, i);
          if (lane == 0) {
            const int w = (base + i - u.b0) % kWarps;
            const int t = ptiles[WS ? w : 0]++;
            const int st = t % NS;
            if (t >= NS) mbar_wait(&empty[WS ? w : 0][st], ((t / NS) - 1) & 1);
            uint8_t* dst = smem + (size_t)w * NS * 2 * TILE + st * 2 * TILE;
            // the last, partly filled block of a sequence: fetch only its valid token
            // rows of K and of V (the consumer masks the scores of the other rows and
            // zeroes their V rows), so DRAM traffic equals the algorithmic bytes
            const int vr = min(16, Lmax_u - (base + i) * 16);
            const uint32_t part = vr < 16 ? (uint32_t)vr * ROW : 2u * TILE;
            mbar_expect_tx(&bars[w][st], vr < 16 ? 2 * part : part);
            const char* src = reinterpret_cast<const char*>(ai);
            if (p.kv_evict_first) {
              bulk_g2s_hint(dst, src, part, &bars[w][st], kv_pol);
              if (vr < 16) bulk_g2s_hint(dst + TILE, src + TILE, part, &bars[w][st], kv_pol);
            } else {
              bulk_g2s(dst, src, part, &bars[w][st]);
              if (vr < 16) bulk_g2s(dst + TILE, src + TILE, part, &bars[w][st]);
            }
          }
        }
      }
    }
  } else {
  pdl_wait();  // (inline-producer variants: no early prologue)
  pump(0);

  // ldmatrix lane addresses within a K|V tile (swizzled), computed once per warp
  const int k_row = (lane & 7) + ((lane >> 3) & 1) * 8, k_cadd = lane >> 4;
  const int v_row = (lane & 7) + (lane >> 4) * 8, v_cadd = (lane >> 3) & 1;
  const uint32_t ring_s = smem_u32(ring);
  uint32_t koff[KS], voff[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    koff[ks] = k_row * ROW + (((2 * ks + k_cadd) ^ (k_row & 7)) << 4);
    voff[ks] = TILE + v_row * ROW + (((2 * ks + v_cadd) ^ (v_row & 7)) << 4);
  }

  for (int ck = 0;; ++ck) {
    pump(ck);  // the producer has now visited item ck (or the stream has ended there)
    int f_ = 0;
    if (lane == 0) {
      unsigned long long w_;
      if (WS)  // the producer warp publishes item ck in slot ck % QB
        while (((w_ = atomicAdd(&slot_word[ck % QB], 0ull)) >> 32) != (unsigned long long)(ck + 1)) __nanosleep(32);
      else
        w_ = atomicAdd(&slot_word[ck % QB], 0ull);
      f_ = (int)(unsigned int)(w_ & 0xffffffffull);
    }
    const int f = __shfl_sync(0xffffffffu, f_, 0);
    if (f >= n_flat) break;
    const AttnUnit u = p.units[f / p.H_kv];
    const int hk = f % p.H_kv;
    const int s = u.seq;
    const int L = u.len;
    const int nq = QP == 1 ? 1 : u.nq;
    const int Lmax = L + nq - 1;  // tokens attended by the item's last row
    const int first = u.b0 + warp;
    const int n_it = first < u.b1 ? (u.b1 - first + kWarps - 1) / kWarps : 0;

    if constexpr (FA) {
      // ---- G = 8 decode, query heads as the M side (see the comment at FA) ----
      // A fragments of q: row gq = head gq's hi part, row gq + 8 = its lo part
      uint32_t qa[KS][4];
      const uint32_t* qs = &qbuf[ck % QB][0];
      if (n_it > 0) mbar_wait(&qbars[ck % QB], (ck / QB) & 1);
      {
        const uint32_t* qw = qs + gq * D + tq;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          qa[ks][0] = n_it > 0 ? qw[ks * 8] : 0u;                  // hi, dims 16ks + 2tq, +1
          qa[ks][1] = n_it > 0 ? qw[D / 2 + ks * 8] : 0u;          // lo
          qa[ks][2] = n_it > 0 ? qw[ks * 8 + 4] : 0u;              // hi, dims 16ks + 8 + 2tq, +1
          qa[ks][3] = n_it > 0 ? qw[D / 2 + ks * 8 + 4] : 0u;      // lo
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&slot_free[WS ? ck % QB : 0]);
      // per lane: softmax state of head gq; O rows gq (hi) and gq + 8 (lo), dims 8n + 2tq, +1
      float mh = -CUDART_INF_F, lh = 0.f;
      float oa[D / 8][4];
#pragma unroll
      for (int n = 0; n < D / 8; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j) oa[n][j] = 0.f;
      for (int it = 0; it < n_it; ++it) {
        const int st = rc % NS;
        const uint32_t phase = (rc / NS) & 1;
        const int blk = first + kWarps * it;
        mbar_wait(&bars[warp][st], phase);
        if (rc == 0 && warp == 0 && lane == 0) ATTN_TRACE(2, gtimer());
        uint8_t* tile = ring + st * 2 * TILE;
        const int valid_rows = min(16, Lmax - blk * 16);
        if (valid_rows < 16) {  // rows past the context may hold any bytes: zero V there
          for (int e = lane; e < (16 - valid_rows) * (ROW / 16); e += 32) {
            const int r = valid_rows + e / (ROW / 16), c = e % (ROW / 16);
            *reinterpret_cast<uint4*>(tile + TILE + r * ROW + c * 16) = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
        }
        const uint32_t tile_s = ring_s + st * 2 * TILE;
        // ---- S[16 x 16 tok] = Qc K^T: one accumulator chain per 8-token n-tile ----
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t bk[4];  // (tok 0-7, dims lo), (tok 0-7, hi), (tok 8-15, lo), (tok 8-15, hi)
          ldsm_x4_s(bk, tile_s + voff[ks] - TILE);
          const uint32_t b0[2] = {bk[0], bk[1]}, b1[2] = {bk[2], bk[3]};
          mma_bf16(s0, qa[ks], b0);
          mma_bf16(s1, qa[ks], b1);
        }
        // head gq's scores of tokens 2tq, 2tq + 1, 8 + 2tq, 9 + 2tq (hi row + lo row)
        float sc[4] = {s0[0] + s0[2], s0[1] + s0[3], s1[0] + s1[2], s1[1] + s1[3]};
        if (valid_rows < 16) {
          const int t0 = 2 * tq;
          if (t0 >= valid_rows) sc[0] = -CUDART_INF_F;
          if (t0 + 1 >= valid_rows) sc[1] = -CUDART_INF_F;
          if (t0 + 8 >= valid_rows) sc[2] = -CUDART_INF_F;
          if (t0 + 9 >= valid_rows) sc[3] = -CUDART_INF_F;
        }
        float bm = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
        const float m_new = fmaxf(mh, bm);
        float pv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) pv[j] = exp2_ftz(sc[j] - m_new);
        // rescale only when some head's running max moved (alpha == 1 otherwise:
        // skipping the multiply by exactly 1 leaves every bit unchanged)
        if (__any_sync(0xffffffffu, m_new != mh)) {
          const float alpha = exp2_ftz(mh - m_new);
          lh *= alpha;
#pragma unroll
          for (int n = 0; n < D / 8; ++n)
#pragma unroll
            for (int j = 0; j < 4; ++j) oa[n][j] *= alpha;
        }
        mh = m_new;
        lh += (pv[0] + pv[1]) + (pv[2] + pv[3]);
        // P as the A operand: rows gq = bf16 hi of p, gq + 8 = bf16(p - hi)
        uint32_t pa[4];
        {
          const __nv_bfloat162 h01 = __floats2bfloat162_rn(pv[0], pv[1]);
          const __nv_bfloat162 h89 = __floats2bfloat162_rn(pv[2], pv[3]);
          const float2 f01 = __bfloat1622float2(h01), f89 = __bfloat1622float2(h89);
          const __nv_bfloat162 l01 = __floats2bfloat162_rn(pv[0] - f01.x, pv[1] - f01.y);
          const __nv_bfloat162 l89 = __floats2bfloat162_rn(pv[2] - f89.x, pv[3] - f89.y);
          pa[0] = *reinterpret_cast<const uint32_t*>(&h01);
          pa[1] = *reinterpret_cast<const uint32_t*>(&l01);
          pa[2] = *reinterpret_cast<const uint32_t*>(&h89);
          pa[3] = *reinterpret_cast<const uint32_t*>(&l89);
        }
        // ---- O[16 x D] += P V: V^T fragments by ldmatrix.trans, two 8-dim n-tiles each ----
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t bv[4];  // (tok 0-7, dims 16ks..+7), (tok 8-15, same), (tok 0-7, +8..), (tok 8-15, +8..)
          ldsm_x4_t_s(bv, tile_s + koff[ks] + TILE);
          const uint32_t b0[2] = {bv[0], bv[1]}, b1[2] = {bv[2], bv[3]};
          mma_bf16(oa[2 * ks], pa, b0);
          mma_bf16(oa[2 * ks + 1], pa, b1);
        }
        ++rc;
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes (V zeroing) -> TMA
          mbar_arrive(&empty[WS ? warp : 0][st]);
        }
      }
      lh += __shfl_xor_sync(0xffffffffu, lh, 1);
      lh += __shfl_xor_sync(0xffffffffu, lh, 2);
      if (warp == 0 && lane == 0) {
        ATTN_TRACE(3, gtimer());
        ATTN_TRACE(7, ck + 1);
      }
      csync();  // the previous item's merge has finished reading sm_*
#pragma unroll
      for (int n = 0; n < D / 8; ++n)
        *reinterpret_cast<float2*>(&sm_acc[warp][gq][8 * n + 2 * tq]) =
            make_float2(oa[n][0] + oa[n][2], oa[n][1] + oa[n][3]);
      if (tq == 0) {
        sm_m[warp][gq] = mh;
        sm_l[warp][gq] = lh;
      }
      csync();
    } else {
    // B fragments of the query columns: column n = gq (+8 nt): head nt*4 + gq/2, part gq&1.
      // q arrives pre-scaled and pre-split (qkv_post): word i of (head, part) packs
      // elements 2i, 2i+1, so a fragment is two shared-memory words.
      uint32_t qb[NT][KS][2];
      const uint32_t* qs = &qbuf[ck % QB][0];
      if (n_it > 0) mbar_wait(&qbars[ck % QB], (ck / QB) & 1);
  #pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int hh = nt * 4 + (gq >> 1);
        const uint32_t* qw = qs + hh * D + (gq & 1) * (D / 2) + tq;
  #pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          if (hh < GV && hh / G < nq && n_it > 0) {
            qb[nt][ks][0] = qw[ks * 8];
            qb[nt][ks][1] = qw[ks * 8 + 4];
          } else {
            qb[nt][ks][0] = qb[nt][ks][1] = 0u;
          }
        }
      }
      if (WS) {  // this warp holds item ck's q in registers: its slot may be reused
        __syncwarp();
        if (lane == 0) mbar_arrive(&slot_free[WS ? ck % QB : 0]);
      }
      // per lane: softmax state of head nt*4 + tq; O^T accumulators (dims ks*16+gq,+8)
      float m[NT], l[NT], o[NT][KS][4];
      int Lv[NT];  // causal length of the lane's (virtual) head: row v / G of the item
  #pragma unroll
      for (int nt = 0; nt < NT; ++nt) Lv[nt] = L + min((nt * 4 + tq) / G, nq - 1);
  #pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        m[nt] = -CUDART_INF_F;
        l[nt] = 0.f;
  #pragma unroll
        for (int ks = 0; ks < KS; ++ks)
  #pragma unroll
          for (int j = 0; j < 4; ++j) o[nt][ks][j] = 0.f;
      }
  
      for (int it = 0; it < n_it; ++it) {
        const int st = rc % NS;
        const uint32_t phase = (rc / NS) & 1;
        const int blk = first + kWarps * it;
        mbar_wait(&bars[warp][st], phase);
        if (rc == 0 && warp == 0 && lane == 0) ATTN_TRACE(2, gtimer());
        uint8_t* tile = ring + st * 2 * TILE;
        const int valid_rows = min(16, Lmax - blk * 16);
        if (valid_rows < 16) {  // rows past the context may hold any bytes: zero V there
          for (int e = lane; e < (16 - valid_rows) * (ROW / 16); e += 32) {
            const int r = valid_rows + e / (ROW / 16), c = e % (ROW / 16);
            *reinterpret_cast<uint4*>(tile + TILE + r * ROW + c * 16) = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
        }
        // ---- S = K Qc (two independent accumulation chains: even / odd k-slices) ----
        float sacc[NT][4], sacc2[NT][4];
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt)
  #pragma unroll
          for (int j = 0; j < 4; ++j) sacc[nt][j] = sacc2[nt][j] = 0.f;
        const uint32_t tile_s = ring_s + st * 2 * TILE;
  #pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t a[4];
          ldsm_x4_s(a, tile_s + koff[ks]);
  #pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma_bf16((ks & 1) ? sacc2[nt] : sacc[nt], a, qb[nt][ks]);
        }
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt)
  #pragma unroll
          for (int j = 0; j < 4; ++j) sacc[nt][j] += sacc2[nt][j];
        // ---- online softmax (base 2) per head nt*4+tq; rows gq and gq+8 ----
        float pA[NT], pB[NT];
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int vr = QP == 1 ? valid_rows : Lv[nt] - blk * 16;  // rows of this tile the head sees
          const float s0 = (gq < vr) ? sacc[nt][0] + sacc[nt][1] : -CUDART_INF_F;
          const float s1 = (gq + 8 < vr) ? sacc[nt][2] + sacc[nt][3] : -CUDART_INF_F;
          float bm = fmaxf(s0, s1);
          bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
          bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
          bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
          const float m_new = fmaxf(m[nt], bm);
          pA[nt] = exp2_ftz(s0 - m_new);
          pB[nt] = exp2_ftz(s1 - m_new);
          if (QP > 1 && m_new == -CUDART_INF_F) pA[nt] = pB[nt] = 0.f;  // a row that sees none of this tile
          // rescale only when some head's running max moved (alpha == 1 otherwise:
          // skipping the multiply by exactly 1 leaves every bit unchanged)
          if (__any_sync(0xffffffffu, m_new != m[nt])) {
            // (a prefill row that has seen no token yet keeps m = -inf: alpha = 1, not NaN)
            const float alpha = (QP > 1 && m_new == -CUDART_INF_F) ? 1.f : exp2_ftz(m[nt] - m_new);
            l[nt] *= alpha;
  #pragma unroll
            for (int ks = 0; ks < KS; ++ks)
  #pragma unroll
              for (int j = 0; j < 4; ++j) o[nt][ks][j] *= alpha;
          }
          l[nt] = l[nt] + pA[nt] + pB[nt];
          m[nt] = m_new;
        }
        // ---- P as B fragments: lane needs P[2tq, 2tq+1, 2tq+8, 2tq+9][column gq] ----
        uint32_t pb[NT][2];
  #pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int src0 = 8 * tq + (gq >> 1), src1 = src0 + 4;
          const float a0 = __shfl_sync(0xffffffffu, pA[nt], src0);  // P[2tq]
          const float a8 = __shfl_sync(0xffffffffu, pB[nt], src0);  // P[2tq+8]
          const float c0 = __shfl_sync(0xffffffffu, pA[nt], src1);  // P[2tq+1]
          const float c8 = __shfl_sync(0xffffffffu, pB[nt], src1);  // P[2tq+9]
          const int part = gq & 1;
          if (nt * 4 + (gq >> 1) < GV) {
            pb[nt][0] = pack_bf16(bf16_part(a0, part), bf16_part(c0, part));
            pb[nt][1] = pack_bf16(bf16_part(a8, part), bf16_part(c8, part));
          } else {
            pb[nt][0] = pb[nt][1] = 0u;
          }
        }
        // ---- O^T += V^T P ----
  #pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          uint32_t a[4];
          ldsm_x4_t_s(a, tile_s + voff[ks]);
  #pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma_bf16(o[nt][ks], a, pb[nt]);
        }
        ++rc;
        if (WS) {  // hand the stage back to the producer warp
          __syncwarp();
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes (V zeroing) -> TMA
            mbar_arrive(&empty[WS ? warp : 0][st]);
          }
        }
        pump(ck);  // refill the freed stage with the tile NS ahead in the stream
      }
      if (warp == 0 && lane == 0) {
        ATTN_TRACE(3, gtimer());
        ATTN_TRACE(7, ck + 1);
      }
      // l: sum the lane partials over the 8 token groups
  #pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        l[nt] += __shfl_xor_sync(0xffffffffu, l[nt], 4);
        l[nt] += __shfl_xor_sync(0xffffffffu, l[nt], 8);
        l[nt] += __shfl_xor_sync(0xffffffffu, l[nt], 16);
      }
  
      csync();  // the previous item's merge has finished reading sm_*
  #pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int hh = nt * 4 + tq;
        if (hh < GV) {
  #pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            sm_acc[warp][hh][ks * 16 + gq] = o[nt][ks][0] + o[nt][ks][1];
            sm_acc[warp][hh][ks * 16 + gq + 8] = o[nt][ks][2] + o[nt][ks][3];
          }
          if (gq == 0) {
            sm_m[warp][hh] = m[nt];
            sm_l[warp][hh] = l[nt];
          }
        }
      }
      csync();
  
    }

    uint64_t c9 = 0;  // trace: SM clock at the merge start (fold phases below in cycles from here)
    if (threadIdx.x == 0 && p.trace) {
      ATTN_TRACE(9, gtimer());
      c9 = clock64();
    }
    // merge the warps in fixed order (w = 0..W-1); every thread derives its head's
    // weights itself: M = max_w m_w, fw_w = 2^(m_w - M) (0 for a warp that saw
    // nothing), Ls = sum_w fw_w l_w, then merges float4s of dims
    const bool split = u.nsplit > 1;
#pragma unroll 1
    for (int e = threadIdx.x; e < GV * D / 4; e += kWarps * 32) {
      const int g = e / (D / 4), d = (e % (D / 4)) * 4;
      if (QP > 1 && g / G >= nq) continue;
      float M = sm_m[0][g];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) M = fmaxf(M, sm_m[w][g]);
      float Ls = 0.f;
      float4 ov = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float fw = (sm_m[w][g] == -CUDART_INF_F) ? 0.f : exp2f(sm_m[w][g] - M);
        Ls += fw * sm_l[w][g];
        const float4 a = *reinterpret_cast<const float4*>(&sm_acc[w][g][d]);
        ov.x += fw * a.x;
        ov.y += fw * a.y;
        ov.z += fw * a.z;
        ov.w += fw * a.w;
      }
      const int h = hk * G + g % G;
      if (!split) {
        const size_t oi = ((size_t)(s + g / G) * p.H + h) * D + d;
        if (p.out_fp32) {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + oi) =
              make_float4(ov.x / Ls, ov.y / Ls, ov.z / Ls, ov.w / Ls);
        } else {
          const __nv_bfloat162 lo2 = __floats2bfloat162_rn(ov.x / Ls, ov.y / Ls);
          const __nv_bfloat162 hi2 = __floats2bfloat162_rn(ov.z / Ls, ov.w / Ls);
          uint2 pk;
          pk.x = *reinterpret_cast<const uint32_t*>(&lo2);
          pk.y = *reinterpret_cast<const uint32_t*>(&hi2);
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + oi) = pk;
        }
      } else {
        float* rec = p.partial + ((size_t)(u.pbase + u.split) * p.H + h) * (D + 4);
        *reinterpret_cast<float4*>(rec + d) = ov;
        if (d == 0) *reinterpret_cast<float2*>(rec + D) = make_float2(M, Ls);
      }
    }
    if (threadIdx.x == 0) ATTN_TRACE(4, gtimer());
    if (QP > 1 || !split) continue;  // prefill items are never split (host guarantees nsplit == 1)

    // ---- split-K combine: o = sum_i w_i o_i / sum_i w_i l_i over the splits i of
    // this (seq, kv head), w_i = 2^(m_i - M), M = max_i m_i; the reduction order
    // depends only on nsplit, so the result is deterministic and independent of
    // where the blocks live.
    // Publication: the barrier orders every consumer thread's partial stores before
    // thread 0's release-acquire ticket (cumulativity, as in CUTLASS's split-K
    // semaphore); the last arriver's barrier then orders its threads' loads after them.
    const int ns = u.nsplit;  // <= kMaxSplitsDev
    const size_t rstride = (size_t)p.H * (D + 4);
    const float* rec0 = p.partial + ((size_t)u.pbase * p.H + hk * G) * (D + 4);
    csync();
    // The last-arriving CTA of this (seq, kv head) folds everything. (A cooperative
    // variant in which the ns CTAs wait for each other and each fold a slice of the
    // columns measured slower on B200: 19.0 vs 16.8 us per 1 x 8k launch.)
    if (threadIdx.x == 0) {
      int* t = p.tickets + (size_t)s * p.H_kv + hk;
      int prev;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(t) : "memory");
      am_last = (prev == ns - 1);
      if (am_last) *t = 0;  // every split has arrived: reset for the next launch
    }
    csync();
    if (!am_last) continue;
    if (threadIdx.x == 0) {
      ATTN_TRACE(8, gtimer());
      ATTN_TRACE(12, clock64() - c9);
    }
    // Every load of the fold is issued ahead of its use, with nothing serial in
    // between: (0) each thread issues its first two batches of partial o loads
    // (they do not depend on the weights), (1) one warp per head loads (m_i, l_i)
    // and derives M, the w_i (zero past ns) and Lambda, (2) o = sum_i w_i o_i /
    // Lambda, one batch at a time, the batch after next loading meanwhile (double
    // buffer), with branch-free FMAs (o and w are zero past ns). Arithmetic and
    // order are those of reading #30 (per column: i = 0..ns-1).
    constexpr int NCOL = G * D / 4;                                // float4 columns of the G heads
    constexpr int CPT = (NCOL + kWarps * 32 - 1) / (kWarps * 32);  // columns per thread
    constexpr int NB = 8 / CPT;                                    // splits per load batch
    float4 ov0[CPT][NB], ov1[CPT][NB];
    auto load_batch = [&](float4 (&ov)[CPT][NB], int i0) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int e = threadIdx.x + c * kWarps * 32;
        const float* rg = rec0 + (e / (D / 4)) * (D + 4) + (e % (D / 4)) * 4;
#pragma unroll
        for (int k = 0; k < NB; ++k)
          ov[c][k] = (e < NCOL && i0 + k < ns) ? __ldcg(reinterpret_cast<const float4*>(rg + (i0 + k) * rstride))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    float* sw = sm_accf;                          // [G][kMaxSplitsDev], zero past ns
    float* sLam = sm_accf + kMaxSplitsDev * G;    // [G]
    constexpr int GI = (G + kWarps - 1) / kWarps;  // heads per warp
    float mv[GI][kMaxSplitsDev / 32], lv[GI][kMaxSplitsDev / 32];
#pragma unroll
    for (int gi = 0; gi < GI; ++gi) {  // the (m, l) loads first: they gate the weights
      const int g = warp + gi * kWarps;
#pragma unroll
      for (int k = 0; k < kMaxSplitsDev / 32; ++k) {
        const int i = lane + 32 * k;
        mv[gi][k] = -CUDART_INF_F;
        lv[gi][k] = 0.f;
        if (g < G && i < ns) {
          const float2 v = __ldcg(reinterpret_cast<const float2*>(rec0 + i * rstride + g * (D + 4) + D));
          mv[gi][k] = v.x;
          lv[gi][k] = v.y;
        }
      }
    }
    load_batch(ov0, 0);
    load_batch(ov1, NB);
#pragma unroll
    for (int gi = 0; gi < GI; ++gi) {
      const int g = warp + gi * kWarps;
      if (g >= G) break;
      float M = -CUDART_INF_F;
#pragma unroll
      for (int k = 0; k < kMaxSplitsDev / 32; ++k) M = fmaxf(M, mv[gi][k]);
#pragma unroll
      for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      if (threadIdx.x == 0 && gi == 0) ATTN_TRACE(13, clock64() - c9);
      float Ls = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxSplitsDev / 32; ++k) {
        const int i = lane + 32 * k;
        const float w = i < ns ? exp2f(mv[gi][k] - M) : 0.f;
        sw[g * kMaxSplitsDev + i] = w;
        Ls += w * lv[gi][k];
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) Ls += __shfl_xor_sync(0xffffffffu, Ls, o);
      if (lane == 0) sLam[g] = Ls;
    }
    if (threadIdx.x == 0) ATTN_TRACE(10, gtimer());
    csync();
    if (threadIdx.x == 0) ATTN_TRACE(14, clock64() - c9);
    float4 acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto fma_batch = [&](const float4 (&ov)[CPT][NB], int i0) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int g = min((int)(threadIdx.x + c * kWarps * 32) / (D / 4), G - 1);
#pragma unroll
        for (int k4 = 0; k4 < NB / 4; ++k4) {
          const float4 w4 = *reinterpret_cast<const float4*>(&sw[g * kMaxSplitsDev + i0 + 4 * k4]);
          const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4& o = ov[c][4 * k4 + j];
            acc[c].x += wk[j] * o.x;
            acc[c].y += wk[j] * o.y;
            acc[c].z += wk[j] * o.z;
            acc[c].w += wk[j] * o.w;
          }
        }
      }
    };
    for (int i0 = 0; i0 < ns; i0 += 2 * NB) {
      fma_batch(ov0, i0);
      if (i0 + 2 * NB < ns) load_batch(ov0, i0 + 2 * NB);
      if (i0 + NB >= ns) break;
      fma_batch(ov1, i0 + NB);
      if (i0 + 3 * NB < ns) load_batch(ov1, i0 + 3 * NB);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = threadIdx.x + c * kWarps * 32;
      if (e >= NCOL) continue;
      const int g = e / (D / 4), d = (e % (D / 4)) * 4;
      const float lam = sLam[g];
      const float4 r = make_float4(acc[c].x / lam, acc[c].y / lam, acc[c].z / lam, acc[c].w / lam);
      const size_t oi = ((size_t)s * p.H + hk * G + g) * D + d;
      if (p.out_fp32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + oi) = r;
      } else {
        const __nv_bfloat162 lo2 = __floats2bfloat162_rn(r.x, r.y);
        const __nv_bfloat162 hi2 = __floats2bfloat162_rn(r.z, r.w);
        uint2 pk;
        pk.x = *reinterpret_cast<const uint32_t*>(&lo2);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi2);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + oi) = pk;
      }
    }
    if (threadIdx.x == 0) {
      ATTN_TRACE(15, clock64() - c9);
      ATTN_TRACE(5, gtimer());
    }
  }
  }  // consumer warps
  // the last CTA to finish resets the work counter for the next launch
  __syncthreads();
  if (threadIdx.x == 0) ATTN_TRACE(6, gtimer());
  if (dyn && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
      atomicExch(p.sched, 0);
      atomicExch(p.sched + 1, 0);
    }
  }
}

template <int D, int G, int QP, int W, int NS, bool WS>
int grid_ctas() {  // persistent grid: as many CTAs as fit on the GPU at once
  constexpr int SMEM = smem_bytes<D, G, QP, W, NS>();
  constexpr int THREADS = (W + (WS ? 1 : 0)) * 32;
  static int ctas = 0;
  if (!ctas) {
    if (cudaFuncSetAttribute(paged_attention_kernel<D, G, QP, W, NS, WS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
      return -1;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, paged_attention_kernel<D, G, QP, W, NS, WS>,
                                                      THREADS, SMEM) != cudaSuccess)
      return -1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ctas = std::max(1, per_sm) * sms;
  }
  return ctas;
}

template <int D, int G, int QP, int W, int NS, bool WS = false>
cudaError_t launch_v(const AttnParams& p, cudaStream_t s, bool query, int* grid_out) {
  const int ctas = grid_ctas<D, G, QP, W, NS, WS>();
  if (ctas < 0) return cudaErrorInvalidValue;
  if (query) {
    *grid_out = ctas;
    return cudaSuccess;
  }
  const long items = (long)p.n_units * p.H_kv;
  const int grid = p.full_grid ? ctas : (int)std::min<long>(items, ctas);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3((W + (WS ? 1 : 0)) * 32);
  cfg.dynamicSmemBytes = smem_bytes<D, G, QP, W, NS>();
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, paged_attention_kernel<D, G, QP, W, NS, WS>, p);
}

// tuning hook: MIRAGE_ATTN_VARIANT selects alternatives (1: 3-deep rings, inline
// producers; 3: inline producers). Default: a producer warp per CTA for decode
// items (C2 in-step 6.02 vs 5.94 TB/s, alone 6.55 vs 6.49; two alternating runs)
int variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MIRAGE_ATTN_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int D, int G>
cudaError_t launch_dg(const AttnParams& p, cudaStream_t s, bool query, int* grid_out) {
  // the 4 warps of a CTA split the blocks of one work item, for any H_kv
  constexpr int NS = D == 128 ? 2 : 4;
  constexpr int QP = G < 8 ? 8 / G : 1;  // prefill rows per item: 8 virtual heads per kv head
  if (p.qp > 1 && QP > 1) return launch_v<D, G, QP, 4, NS>(p, s, query, grid_out);
  if (D == 128 && variant() == 1) return launch_v<D, G, 1, 4, 3>(p, s, query, grid_out);
  if (variant() == 3) return launch_v<D, G, 1, 4, NS>(p, s, query, grid_out);
  return launch_v<D, G, 1, 4, NS, true>(p, s, query, grid_out);
}

template <int D>
cudaError_t launch_d(const AttnParams& p, cudaStream_t s, bool query, int* grid_out) {
  switch (p.H / p.H_kv) {
    case 1: return launch_dg<D, 1>(p, s, query, grid_out);
    case 2: return launch_dg<D, 2>(p, s, query, grid_out);
    case 4: return launch_dg<D, 4>(p, s, query, grid_out);
    case 8: return launch_dg<D, 8>(p, s, query, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

cudaError_t launch_paged_attention(const AttnParams& p, cudaStream_t s) {
  if (p.n_units == 0) return cudaSuccess;
  if (p.D == 128) return launch_d<128>(p, s, false, nullptr);
  if (p.D == 64) return launch_d<64>(p, s, false, nullptr);
  return cudaErrorInvalidValue;
}

int attention_grid_ctas(int H, int H_kv, int D, int qp) {
  AttnParams p{};
  p.H = H;
  p.H_kv = H_kv;
  p.D = D;
  p.qp = qp;
  int g = -1;
  if (D == 128) launch_d<128>(p, nullptr, true, &g);
  if (D == 64) launch_d<64>(p, nullptr, true, &g);
  return g;
}

int attention_cta_warps(int) { return 4; }

int attention_prefill_rows(int H, int H_kv) {
  const int G = H / H_kv;
  return G < 8 ? 8 / G : 1;
}

}  // namespace mirage
