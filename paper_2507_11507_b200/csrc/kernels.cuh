// Internal kernel launch API of libmirage (not part of the C-ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mirage {

// One attention work unit: a (sequence, split) pair -- or, in a prefill step,
// nq consecutive rows of one sequence (positions len-1 .. len+nq-2); the kernel
// expands it over the kv heads. 32 bytes, everything the kernel needs without
// dependent loads.
struct AttnUnit {
  int32_t seq;       // (first) row in the step's batch
  int16_t split;     // split index within the sequence
  int16_t nsplit;    // number of splits of this sequence (1 when nq > 1)
  int32_t pbase;     // first partial record of this sequence (valid if nsplit > 1)
  int32_t len;       // tokens attended by the first row; row seq + i attends len + i
  int32_t b0, b1;    // this split's block range [b0, b1) (covers the last row)
  int32_t addr_off;  // index of the sequence's block 0 in AttnParams::addrs
  int32_t nq;        // rows in this unit (1 for decode)
};
static_assert(sizeof(AttnUnit) == 32, "AttnUnit is one 32-byte record");

struct AttnParams {
  const uint32_t* q;           // [B][H][2][D/2]: q * scale_log2 split into bf16 hi (part 0) and
                               // lo = bf16(x - hi) (part 1); word i packs elements 2i (low half), 2i+1
  const uint64_t* addrs;       // per-step block base addresses (host-resolved table -> block_base)
  uint64_t layer_off;          // layer * H_kv * 2 * 16 * D * 2 bytes
  const AttnUnit* units;       // [n_units], longest first
  int32_t n_units;             // host count (sizes the grid)
  const int32_t* n_units_dev;  // if set, the count is read here (CUDA-graph replays)
  const int32_t* hdr;          // step metadata header: [1] = schedule (0 = longest-first queue,
                               // 1 = balanced ranges: CTA b runs units rfirst[b / H_kv] ..
                               // rfirst[b / H_kv + 1] - 1 for kv head b % H_kv; grid = R * H_kv)
  const int32_t* rfirst;       // [R + 1] first unit of each range (schedule 1)
  int32_t H, H_kv, D;
  float scale_log2;            // log2(e) / sqrt(D) (already applied to q)
  float* partial;              // [(pbase + split) * H + h][D + 4]: o, m, l, pad
  int32_t* tickets;            // [B * H_kv], zero between launches
  int32_t* sched;              // [2] dynamic item counter + finished CTAs, zero between launches
  void* out;                   // [B][H][D] fp32 or bf16
  int32_t out_fp32;
  int32_t qp;                  // rows per unit the launch was planned for (1, or 8 / G for prefill)
  uint64_t* trace;             // optional [grid][16] %globaltimer stamps per CTA (MIRAGE_ATTN_TRACE), else null
  int32_t pdl;                 // launch with a programmatic dependency on the previous kernel (which
                               // must call griddepcontrol.launch_dependents early, as qkv_post does)
  int32_t full_grid;           // launch the whole persistent grid even if there are fewer items
                               // (schedule 1: CTA b serves range b / H_kv)
  int32_t prod_lanes;          // producer warp issues through one lane per consumer warp (else lane 0 issues all)
  int32_t kv_evict_first;      // K|V tiles are loaded with an L2 evict_first policy (they are read
                               // once per launch); MIRAGE_KV_EVICT_FIRST=0 turns it off
};

cudaError_t launch_paged_attention(const AttnParams& p, cudaStream_t s);
// CTAs of the persistent attention grid on this device (for split planning), and
// warps per CTA (blocks of one work item are spread over them).
int attention_grid_ctas(int H, int H_kv, int D, int qp = 1);
// rows per unit of the prefill variant (8 / G, 1 for G = 8)
int attention_prefill_rows(int H, int H_kv);
int attention_cta_warps(int H_kv);

// ---- decode GEMM on tcgen05 (decode_gemm.cu) ---------------------------------
// Y_s[b][n] = sum over split s's K range of X[b][k] W[n][k]: W [N][ldw] and X
// [B][ldx] bf16 row-major, 1 <= B <= 256; split slice s at out + s * slice, row b
// at + b * ldo. peers (device array of n_peers float*, or null): the slices are
// also stored at peers[r] + peer_slot + (same offsets) -- the fused TP all-reduce.
constexpr int kMaxGemmSplits = 16;
// cnt (device array of n_cnt counters, or null): each CTA increments every one of
// them (release, system scope) after its stores -- the arrival signal of the
// fused tensor-parallel all-reduce (one increment per tile per destination).
cudaError_t launch_decode_gemm(const __nv_bfloat16* W, int N, int K, int ldw, const __nv_bfloat16* X, int B, int ldx,
                               float* out, int ldo, long long slice, int splits, float* const* peers, int n_peers,
                               long long peer_slot, cudaStream_t s, unsigned long long* const* cnt = nullptr,
                               int n_cnt = 0, bool reduce = false, int* slices_out = nullptr, int cgroups = 1);
// reduce = true: up to 8 splits of a tile (batch <= 128) are summed inside the GEMM
// through a thread-block cluster's distributed shared memory, so `out` receives
// ONE slice (*slices_out = 1); otherwise *slices_out = splits.
// tiles (CTAs per split) of a decode GEMM with N output rows
inline int decode_gemm_tiles(int N) { return (N + 127) / 128; }
// cgroups > 1 cuts the batch into column groups of >= 32 rows, one CTA per (tile,
// split, group) (launch_decode_gemm rounds the group width up to 32/64/128/256 and
// drops empty groups): the column-group count the fused push GEMM uses, and the
// CTAs (= arrival-counter increments) per split for a given request
int decode_gemm_cgroups(int N, int B, int sms);
int decode_gemm_ctas_per_split(int N, int B, int cgroups);
// K splits for a B-row decode GEMM on `sms` SMs (per-SM load model, decode_gemm.cu)
int decode_gemm_splits(int N, int K, int B, int sms);
// Persistent stream-K form (decode_gemm.cu, "SK"): one wave of CTAs over the
// tiles x K-blocks stream, cut tiles finished in the GEMM (deterministic K-order
// fixup through ws [sk_gemm_max_ctas()][B][128] fp32 and flags [sk_gemm_max_ctas()]
// ints, zero before the first launch): ONE output, y = epilogue(x W^T) with
// optional bias[N], ReLU, and fp32 (out) or bf16 (out16) storage at row stride
// ldo; peers / cnt: the fused tensor-parallel push as in launch_decode_gemm
// (fp32 only; cnt gains one increment per tile per destination).
int sk_gemm_max_ctas();
cudaError_t launch_sk_gemm(const __nv_bfloat16* W, int N, int K, int ldw, const __nv_bfloat16* X, int B, int ldx,
                           float* out, __nv_bfloat16* out16, int ldo, const __nv_bfloat16* bias, int relu, float* ws,
                           int* flags, float* const* peers, int n_peers, long long peer_slot, cudaStream_t s,
                           unsigned long long* const* cnt = nullptr, int n_cnt = 0);

// ---- dense-layer support kernels -------------------------------------------
// h[b] = E[tok] (+ P[pos + 2] for OPT); x[b] = bf16(norm(h[b])).
cudaError_t launch_embed_norm(int family, int B, int d, const int32_t* tokens,
                              const int32_t* positions, const __nv_bfloat16* embed,
                              const __nv_bfloat16* pos_embed, const __nv_bfloat16* g,
                              const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                              cudaStream_t s);
// h[b] += y[b] (+ bias); x[b] = bf16(norm(h[b])). y row stride ldy; y may hold
// nsplit split-K slices `slice` floats apart (summed in slice order first).
cudaError_t launch_residual_norm(int family, int B, int d, const float* y, int ldy,
                                 const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                 const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                 cudaStream_t s, int nsplit = 1, long long slice = 0, bool pdl = false);
// qkv [B][(H+2Hk)D] fp32 (+bias, +RoPE) -> q in the attention kernel's split
// format (AttnParams::q, scaled by q_scale); K/V bf16 appended to the paged cache
// at positions[b] (block address addrs[seq_off[b] + pos / 16]).
cudaError_t launch_qkv_post(int family, int B, int H, int Hk, int D, const float* qkv,
                            const __nv_bfloat16* bias, const int32_t* positions,
                            const int32_t* seq_off, const uint64_t* addrs, uint64_t layer_off,
                            float rope_theta, float q_scale, uint32_t* q, cudaStream_t s, bool pdl = false);
// (pdl: launched with a programmatic dependency on the preceding kernel, the GEMM
// whose output it reads; the prologue that does not touch that output overlaps
// the GEMM's tail, griddepcontrol.wait guards the rest)
// Block migration (mirage_migrate_region): copy `bytes` from src[i] to dst[i]
// for i < n (device addresses, 16-byte aligned, bytes % 16 == 0).
struct BlockMoves {
  uint64_t src[16], dst[16];
  int n;
};
cudaError_t launch_block_copy(const BlockMoves& m, uint64_t bytes, cudaStream_t s);
// fp32 q [n_rows * D] (unscaled) -> the split format of AttnParams::q (test hook path)
cudaError_t launch_q_split(int64_t n, int D, const float* q, float q_scale, uint32_t* out, cudaStream_t s);
// OPT: f = bf16(relu(y + b)); Llama: f = bf16(silu(y[:, :f]) * y[:, f:]).
cudaError_t launch_act(int family, int B, int f, const float* y, const __nv_bfloat16* bias,
                       __nv_bfloat16* out, cudaStream_t s);
// argmax over each row of logits [B][V] (lowest index on ties).
cudaError_t launch_argmax(int B, int V, const float* logits, int32_t* out, cudaStream_t s);

// ---- tensor parallelism over peer memory (MIRAGE_FLAG_TP_IPC, a10 fused) ----
// One-shot all-reduce fused with the residual (+bias) and the next norm: rank r
// publishes `epoch` in its flag after its partial GEMM output is complete,
// waits for every peer's flag, sums the tp partial rows in fixed rank order
// (bit-identical on all ranks), then h += sum (+ bias); x = norm(h) if g.
// parts[r] / flags[r]: rank r's partial buffer / flag (peer pointers via IPC).
cudaError_t launch_tp_residual_norm(int family, int B, int d, const float* const* parts, int tp, int rank,
                                    unsigned long long* const* flags, unsigned long long epoch,
                                    unsigned int* err, const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                    const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                    cudaStream_t s);

// Fused variant (MIRAGE_FLAG_TC_GEMM + TP_IPC): every rank's decode GEMM pushed its
// partial rows into slot r of THIS rank's exchange buffer and bumped cnt[r]; wait
// until cnt[r] >= expect for every r (bounded spin: err++ on a lost peer), then
// h += sum_r slots[r] (fixed rank order) (+ bias); x = norm(h) if g. Local reads only.
cudaError_t launch_tp_push_residual_norm(int family, int B, int d, const float* const* slots, int tp,
                                         const unsigned long long* cnt, unsigned long long expect, unsigned int* err,
                                         const __nv_bfloat16* bias, const __nv_bfloat16* g,
                                         const __nv_bfloat16* bta, float eps, float* h, __nv_bfloat16* x,
                                         cudaStream_t s);

// ---- slot tags (MIRAGE_FLAG_SLOT_TAGS): race detector for the copy engine ----
// errors[0] += 1 and errors[1] = got if *tag != expected.
cudaError_t launch_tag_check(const uint32_t* tag, uint32_t expected, uint32_t* errors, cudaStream_t s);
// debug only: occupy the stream for ~ns nanoseconds (forces copy/compute races in tests)
cudaError_t launch_spin(uint64_t ns, cudaStream_t s);

// ---- KV hooks ----------------------------------------------------------------
cudaError_t launch_fill_kv(uint64_t seed, int64_t seq_id, int L, int Hk, int D, int p0, int n,
                           const int32_t* table, const uint64_t* block_base, cudaStream_t s);
// src: device bf16 [L][Hk][2][n][D] -> paged blocks at positions p0..p0+n-1.
cudaError_t launch_write_kv(int L, int Hk, int D, int p0, int n, const __nv_bfloat16* src,
                            const int32_t* table, const uint64_t* block_base, cudaStream_t s);

}  // namespace mirage
