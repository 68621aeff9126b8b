// libmirage host runtime: context, arena carving, block allocator with remap
// (a2, a3), copy-engine prefetcher with event-gated layer handoff (a4, a5) and
// the decode-step executor (a0, a6-a9). See include/mirage.h for the contract
// and DESIGN.md for the readings of the paper this follows.
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <numeric>
#include <cmath>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <tuple>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/mirage.h"
#include "kernels.cuh"

namespace mirage {
std::vector<int32_t> uniform_placement(int32_t n, int32_t m, int32_t anchor);
}

namespace {

using bf16 = __nv_bfloat16;
constexpr int kBlockTokens = MIRAGE_BLOCK_TOKENS;
constexpr int kMaxSplits = 128;        // split-K partitions per (sequence, kv head) (kernel agrees)
constexpr int kTargetCtas = 148 * 16;     // sizing bound for the attention work-item list
constexpr uint64_t kAlign = 256;
constexpr size_t kCublasWs = 32u << 20;

enum LayerState { RESIDENT = 0, SLOT = 1, RECLAIMED = 2 };

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Shape {
  int family, n, d, H, Hk, D, f, V, max_pos;
  float eps, theta;
};

struct Sizes {
  uint64_t S, G, BB;
};

uint64_t layer_params(const Shape& m) {
  const uint64_t d = m.d, f = m.f;
  if (m.family == MIRAGE_FAMILY_OPT) return 4 * d * d + 2 * d * f + 9 * d + f;
  const uint64_t qkv = (uint64_t)(m.H + 2 * m.Hk) * m.D;
  return qkv * d + d * (uint64_t)m.H * m.D + 3 * f * d + 2 * d;
}

uint64_t global_params(const Shape& m) {
  const uint64_t d = m.d, V = m.V;
  if (m.family == MIRAGE_FAMILY_OPT) return V * d + (uint64_t)(m.max_pos + 2) * d + 2 * d;
  return 2 * V * d + d;
}

Sizes sizes_of(const Shape& m) {
  Sizes z;
  z.S = 2 * layer_params(m);
  z.G = 2 * global_params(m);
  z.BB = (uint64_t)m.n * m.Hk * 2 * kBlockTokens * m.D * 2;
  return z;
}

// Per-layer tensor pointers (blob order documented in include/mirage.h).
struct LayerW {
  const bf16 *w_qkv, *w_o, *w_1, *w_2;  // w_1 = fc1 / gateup, w_2 = fc2 / down
  const bf16 *b_qkv, *b_o, *b_1, *b_2;  // OPT only
  const bf16 *n1_g, *n1_b, *n2_g, *n2_b;
};

LayerW layer_ptrs(const Shape& m, const char* base) {
  LayerW w{};
  const bf16* p = reinterpret_cast<const bf16*>(base);
  const size_t d = m.d, f = m.f;
  if (m.family == MIRAGE_FAMILY_OPT) {
    w.w_qkv = p; p += 3 * d * d;
    w.w_o = p; p += d * d;
    w.w_1 = p; p += f * d;
    w.w_2 = p; p += d * f;
    w.b_qkv = p; p += 3 * d;
    w.b_o = p; p += d;
    w.b_1 = p; p += f;
    w.b_2 = p; p += d;
    w.n1_g = p; p += d;
    w.n1_b = p; p += d;
    w.n2_g = p; p += d;
    w.n2_b = p; p += d;
  } else {
    const size_t qkv = (size_t)(m.H + 2 * m.Hk) * m.D;
    w.w_qkv = p; p += qkv * d;
    w.w_o = p; p += d * (size_t)m.H * m.D;
    w.w_1 = p; p += 2 * f * d;
    w.w_2 = p; p += d * f;
    w.n1_g = p; p += d;
    w.n2_g = p; p += d;
  }
  return w;
}

struct GlobalW {
  const bf16 *embed, *pos_embed, *nf_g, *nf_b, *lm_head;
};

GlobalW global_ptrs(const Shape& m, const char* base) {
  GlobalW g{};
  const bf16* p = reinterpret_cast<const bf16*>(base);
  const size_t d = m.d, V = m.V;
  g.embed = p; p += V * d;
  if (m.family == MIRAGE_FAMILY_OPT) {
    g.pos_embed = p; p += (size_t)(m.max_pos + 2) * d;
    g.nf_g = p; p += d;
    g.nf_b = p; p += d;
    g.lm_head = g.embed;  // tied
  } else {
    g.nf_g = p; p += d;
    g.lm_head = p; p += V * d;
  }
  return g;
}

// One reclaimed region: a maximal run of consecutive donor layers carved in one
// remap call into blocks [first_id, first_id + n_blocks) of the recipient.
struct Region {
  int32_t donor, first_layer, n_layers, first_id, n_blocks;
  bool cycle;    // part of a streaming self-remap (reverted only with the whole cycle)
  bool retired;  // reverted: ids retired, bytes back to parameters
};

struct CopyTiming {
  cudaEvent_t t0, t1;
  uint64_t bytes;
};

struct Model {
  Shape shp;
  Sizes sz;
  int id = 0;
  char* w_dev = nullptr;      // layer 0 of the device weights
  const char* host = nullptr; // pinned host blob
  char* pool = nullptr;       // native KV pool
  int64_t n_native = 0;
  bool active = true;
  // ---- allocator (a2, a3) ----
  int32_t next_id = 0;
  std::set<int32_t> free_ids;
  std::unordered_map<int64_t, std::vector<int32_t>> tables;
  std::unordered_map<int64_t, int32_t> lens;
  std::unordered_map<int64_t, int32_t> swapped;  // seq -> cached length while swapped out
  std::vector<int32_t> loc_donor;  // -1 native
  std::vector<uint64_t> loc_off;
  std::vector<uint64_t> bbase_host;
  uint64_t* bbase_dev = nullptr;
  int64_t bbase_cap = 0;
  uint64_t reclaimed_bytes = 0, donated_bytes = 0;
  std::vector<int> layer_state;
  std::vector<Region> regions;  // as recipient, in creation order
  // ---- prefetcher (a4, a5) ----
  std::vector<int32_t> cycle;
  int32_t beta = 0;
  std::vector<int> cyc_index;  // layer -> index in cycle or -1
  uint64_t uses = 0;           // cycled uses enqueued since install
  int64_t cyc_steps = 0;
  std::vector<int64_t> slot_log;  // rows of 5
  std::vector<cudaEvent_t> ready_ev, free_ev;
  // asynchronous reloads (mirage_unremap): layer l's weights land on the copy
  // stream; the first kernel that reads layer l waits for reload_ev[l]
  std::vector<cudaEvent_t> reload_ev;  // per layer, created on first use
  std::vector<char> reload_pending;
  // layers whose reload is requested but not yet enqueued: the copies are issued
  // by the model's next step right after its metadata upload (the host->device
  // copy engine is FIFO across streams, so copies queued earlier would hold the
  // step's own upload back until all of them finished)
  std::vector<int32_t> reload_queue;
  uint32_t* slot_tag = nullptr;   // device [MAX_CYCLE] tag of the layer each slot holds (SLOT_TAGS)
  uint32_t* tag_err = nullptr;    // device [2] mismatch count, last bad tag
  uint32_t* host_tags = nullptr;  // pinned [n_layers] tag values copied behind each layer DMA
  std::deque<CopyTiming> pending;
  uint64_t h2d_copies = 0, h2d_bytes = 0;
  double h2d_ms = 0;
  // ---- workspace (arena) ----
  float* h = nullptr;
  bf16* x = nullptr;
  float* y = nullptr;
  uint32_t* q = nullptr;  // [B][H][2][D/2] split-format q (AttnParams::q)
  bf16* f = nullptr;
  float* partial = nullptr;
  int32_t* tickets = nullptr;
  int32_t* argmax = nullptr;
  int y_ld_max = 0;
  // ---- attention kernel timing (MIRAGE_FLAG_TIME_ATTN) ----
  struct AttnTiming {
    cudaEvent_t t0, t1;
    uint64_t bytes;
    int reps = 1;  // launches between t0 and t1
  };
  std::deque<AttnTiming> attn_pending;
  std::deque<AttnTiming> stall_pending;  // (before, after) a slot ready-wait on the compute stream
  int64_t stall_waits = 0;
  double stall_ms = 0;
  std::vector<cudaEvent_t> ev_pool;
  int64_t attn_launches = 0;
  double attn_ms = 0;
  uint64_t attn_bytes = 0;
  uint64_t last_meta = 0;
  int32_t last_units = 0, last_split = 0;
  // ---- CUDA graphs of the decode step (MIRAGE_FLAG_CUDA_GRAPHS) ----
  // Key: batch size and, for a streaming cycle, the slot parity of the step's first
  // use (uses % lcm(m, beta)): the slots and copy sources of a step repeat with it.
  // A graph of a cycling model holds the copy stream's re-streaming DMAs as a
  // captured branch (fork on the free events, join before the graph ends).
  struct Graph {
    cudaGraphExec_t exec;
    int64_t kernels;
    // timed graphs (MIRAGE_FLAG_CUDA_GRAPHS + MIRAGE_FLAG_TIME_ATTN): event nodes before
    // and after each layer's attention launch, 2 per layer, read after the replay
    std::vector<cudaEvent_t> tev;
  };
  std::map<int64_t, Graph> graphs;
  std::set<int64_t> graph_seen;  // keys run once eagerly (plans/autotune done)
  const Graph* tpend = nullptr;  // the last timed replay whose attention times are not harvested
  uint64_t tpend_bytes = 0;      // algorithmic bytes of each of its attention launches
  cudaEvent_t join_ev = nullptr; // the copy branch rejoins the compute stream at the end of a capture
  // slot events used inside captures (an event recorded in a capture cannot be
  // waited on outside it, so the eager ready/free events stay separate)
  std::vector<cudaEvent_t> cap_ready_ev, cap_free_ev;
  uint64_t graph_copies = 0;     // re-streaming DMAs run inside graphs (not individually timed)
  // ---- tensor parallelism over peer memory (MIRAGE_FLAG_TP_IPC) ----
  // pull (TP_IPC): [flag u64 | pad][partial par 0][partial par 1];
  // push (TP_IPC + TC_GEMM): [flag | cnt[tp] u64 | pad][par 0: tp slots][par 1: tp slots]
  char* xfer = nullptr;
  size_t xfer_part = 0;               // bytes of one partial buffer (max_batch * d * 4)
  bool tp_push = false;               // fused GEMM + all-reduce (the GEMM pushes to every rank)
  float** push_dst_dev = nullptr;     // device [2][tp-1]: my slot in each OTHER rank's buffer
  float** local_slots_dev = nullptr;  // device [2][tp]: the tp slots of my own buffer
  unsigned long long** push_cnt_dev = nullptr;  // device [tp]: my arrival counter in every rank's header
  unsigned long long push_expect = 0; // tiles each counter has received once the last GEMM lands
  std::vector<char*> peer_base;       // rank -> base of its xfer (own or IPC-opened)
  float** parts_dev = nullptr;        // device [2][tp]
  unsigned long long** flags_dev = nullptr;  // device [tp]
  unsigned int* tp_err = nullptr;     // device counter of lost-peer timeouts
  unsigned long long tp_epoch = 0;
  bool tp_ready = false;
  // ---- step timing ----
  cudaEvent_t st0 = nullptr, st1 = nullptr;
  bool step_timed = false;
  double last_step_ms = 0;
  int64_t steps = 0;
};

}  // namespace

struct mirage_ctx {
  mirage_init_cfg cfg{};
  cudaStream_t cs = nullptr, xs = nullptr;
  bool own_xs = false;
  char* arena = nullptr;
  uint64_t arena_used = 0;
  std::vector<Model*> models;
  cublasHandle_t blas = nullptr;
  cublasLtHandle_t lt = nullptr;
  void* blas_ws = nullptr;

  struct LtPlan {
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
    cublasLtMatmulAlgo_t algo{};
    bool has_algo = false;
  };
  std::map<std::tuple<int, int, int, int, int>, LtPlan> lt_plans;  // (B, N, K, out_bf16, epi)
  // step metadata: pinned staging ring -> device
  size_t meta_bytes = 0;
  char* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  int stage_i = 0;
  char* meta_dev = nullptr;
  int max_units = 0;
  int sms = 148;  // multiprocessors of the device (split planning)
  static constexpr int kTraceCtas = 4096;
  uint64_t* attn_trace = nullptr;  // MIRAGE_ATTN_TRACE: [kTraceCtas][8] stamps of the last attn_only launch
  int32_t attn_trace_ctas = 0;
  int max_blk = 0;
  std::string err;
  int32_t sticky = MIRAGE_OK;
  int64_t launches = 0;
  bool host_only = false;  // MIRAGE_FLAG_HOST_ONLY: allocator/planner state only, no device
  ncclComm_t nccl = nullptr;  // tensor-parallel communicator (tp_size > 1)
  int tp = 1, tp_rank = 0;
};

namespace {

int32_t fail(mirage_ctx* c, int32_t code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (code == MIRAGE_ERR_CUDA || code == MIRAGE_ERR_NCCL) c->sticky = code;
  }
  return code;
}

#define CK(ctx, expr)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(ctx, MIRAGE_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define CKB(ctx, expr)                                                                        \
  do {                                                                                        \
    cublasStatus_t e_ = (expr);                                                               \
    if (e_ != CUBLAS_STATUS_SUCCESS)                                                          \
      return fail(ctx, MIRAGE_ERR_CUDA, "%s: cublas status %d (%s:%d)", #expr, (int)e_, __FILE__, \
                  __LINE__);                                                                  \
  } while (0)

#define KL(ctx, expr)      \
  do {                     \
    ++(ctx)->launches;     \
    CK(ctx, (expr));       \
  } while (0)

#define CKN(ctx, expr)                                                                             \
  do {                                                                                             \
    ncclResult_t e_ = (expr);                                                                      \
    if (e_ != ncclSuccess)                                                                         \
      return fail(ctx, MIRAGE_ERR_NCCL, "%s: %s (%s:%d)", #expr, ncclGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                       \
  } while (0)

// every call makes the ctx's device current on the calling thread (a process may
// drive several GPUs, e.g. a peer-HBM weight source on another device)
#define GUARD(ctx)                                                      \
  do {                                                                  \
    if (!(ctx)) return MIRAGE_ERR_CONFIG;                               \
    if ((ctx)->sticky) return (ctx)->sticky;                            \
    if (!(ctx)->host_only) cudaSetDevice((ctx)->cfg.device);            \
  } while (0)

Shape shape_of(const mirage_model_cfg* m) {
  Shape s;
  s.family = m->family;
  s.n = m->n_layers;
  s.d = m->d_model;
  s.H = m->n_heads;
  s.Hk = m->n_kv_heads;
  s.D = m->head_dim;
  s.f = m->ffn_dim;
  s.V = m->vocab;
  s.max_pos = m->max_pos;
  s.eps = m->norm_eps;
  s.theta = m->rope_theta;
  return s;
}

const char* check_shape(const Shape& s) {
  if (s.family != MIRAGE_FAMILY_OPT && s.family != MIRAGE_FAMILY_LLAMA) return "family";
  if (s.n <= 0 || s.n > MIRAGE_MAX_CYCLE) return "n_layers";
  if (s.d <= 0 || s.d % 128 || s.d > 8192) return "d_model (multiple of 128, <= 8192)";
  if (s.D != 64 && s.D != 128) return "head_dim (64 or 128)";
  if (s.H <= 0 || s.Hk <= 0 || s.H % s.Hk) return "n_heads % n_kv_heads";
  const int g = s.H / s.Hk;
  if (g != 1 && g != 2 && g != 4 && g != 8) return "group size (1,2,4,8)";
  if (s.family == MIRAGE_FAMILY_OPT && (s.H * s.D != s.d || s.Hk != s.H)) return "OPT: H*D == d, MHA";
  if (s.f <= 0 || s.f % 128) return "ffn_dim (multiple of 128)";
  if (s.V <= 0 || s.max_pos <= 0) return "vocab/max_pos";
  return nullptr;
}

// workspace element counts of a model under the ctx limits
struct WsPlan {
  uint64_t h, x, y, q, f, partial, tickets, argmax;
  int y_ld;
};

WsPlan ws_plan(const Shape& s, int Bm, int max_units) {
  WsPlan w;
  const int qkv = (s.H + 2 * s.Hk) * s.D;
  const int ffn_out = s.family == MIRAGE_FAMILY_LLAMA ? 2 * s.f : s.f;
  w.y_ld = std::max(std::max(qkv, ffn_out), std::max(s.V, s.d));
  w.h = (uint64_t)Bm * s.d * 4;
  w.x = (uint64_t)Bm * std::max(s.d, s.H * s.D) * 2;
  w.y = (uint64_t)Bm * w.y_ld * 4;
  w.q = (uint64_t)Bm * s.H * s.D * 4;
  w.f = (uint64_t)Bm * s.f * 2;
  w.partial = (uint64_t)max_units * s.H * (s.D + 4) * 4;
  w.tickets = (uint64_t)Bm * s.Hk * 4 + 8;  // split tickets + the attention work counter
  w.argmax = (uint64_t)Bm * 4;
  return w;
}

uint64_t model_arena(const Shape& s, int64_t n_native, int Bm, int max_units) {
  const Sizes z = sizes_of(s);
  const WsPlan w = ws_plan(s, Bm, max_units);
  uint64_t t = 0;
  t += align_up((uint64_t)s.n * z.S + z.G, kAlign);
  t += align_up((uint64_t)n_native * z.BB, kAlign);
  for (uint64_t b : {w.h, w.x, w.y, w.q, w.f, w.partial, w.tickets, w.argmax}) t += align_up(b, kAlign);
  return t;
}

int units_cap(int Bm) { return 2 * Bm + 2 * kTargetCtas; }

char* carve(mirage_ctx* c, uint64_t bytes) {
  const uint64_t off = align_up(c->arena_used, kAlign);
  if (off + bytes > c->cfg.dev_arena_bytes) return nullptr;
  c->arena_used = off + bytes;
  return c->arena + off;
}

Model* get_model(mirage_ctx* c, int32_t id) {
  if (id < 0 || id >= (int32_t)c->models.size()) return nullptr;
  return c->models[id];
}

// ---- step metadata packing ---------------------------------------------------
// One pinned staging buffer per step, uploaded with one H2D:
//   tokens | positions | lengths | seq_off | attention units | block addresses
// The block addresses are the step's table rows resolved through block_base on
// the host (addrs[seq_off[i] + j] = block_base[table[i][j]]), so the kernels
// need no dependent table lookups. The KV hooks reuse the address region for a
// plain int32 table row.
constexpr int kMaxRanges = 512;  // balanced-range mode: ranges (= grid / H_kv) per launch
struct MetaView {
  int32_t* hdr;  // [4]: n_units, attention mode (0 = LPT queue, 1 = balanced ranges), ...
  int32_t *tokens, *pos, *len, *seq_off;
  int32_t* rfirst;  // [kMaxRanges + 1]: first unit of each balanced range (mode 1)
  mirage::AttnUnit* units;
  uint64_t* addrs;
  int32_t* tables;  // aliases addrs (fill/write hooks only)
};

MetaView meta_view(mirage_ctx* c, char* base) {
  MetaView v;
  const int Bm = c->cfg.max_batch;
  char* p = base;
  v.hdr = reinterpret_cast<int32_t*>(p); p += 16;
  v.tokens = reinterpret_cast<int32_t*>(p); p += align_up((uint64_t)Bm * 4, 16);
  v.pos = reinterpret_cast<int32_t*>(p); p += align_up((uint64_t)Bm * 4, 16);
  v.len = reinterpret_cast<int32_t*>(p); p += align_up((uint64_t)Bm * 4, 16);
  v.seq_off = reinterpret_cast<int32_t*>(p); p += align_up((uint64_t)Bm * 4, 16);
  v.rfirst = reinterpret_cast<int32_t*>(p); p += align_up((uint64_t)(kMaxRanges + 1) * 4, 16);
  v.units = reinterpret_cast<mirage::AttnUnit*>(p); p += align_up((uint64_t)c->max_units * sizeof(mirage::AttnUnit), 16);
  v.addrs = reinterpret_cast<uint64_t*>(p);
  v.tables = reinterpret_cast<int32_t*>(p);
  return v;
}

size_t meta_size(mirage_ctx* c) {
  const int Bm = c->cfg.max_batch;
  return 16 + 4 * align_up((uint64_t)Bm * 4, 16) + align_up((uint64_t)(kMaxRanges + 1) * 4, 16) + align_up((uint64_t)c->max_units * sizeof(mirage::AttnUnit), 16) +
         (uint64_t)Bm * c->max_blk * 8;
}

// Upload a packed step (header and row arrays at capacity, n_addr addresses)
// from staging buffer `host` to the device copy, on the compute stream.
int32_t upload_meta(mirage_ctx* c, char* host, int n_addr, size_t* bytes_out = nullptr) {
  MetaView hv = meta_view(c, host);
  const size_t bytes = (size_t)(reinterpret_cast<char*>(hv.addrs) - host) + (size_t)n_addr * 8;
  CK(c, cudaMemcpyAsync(c->meta_dev, host, bytes, cudaMemcpyHostToDevice, c->cs));
  if (bytes_out) *bytes_out = bytes;
  return MIRAGE_OK;
}

int32_t acquire_stage(mirage_ctx* c, char** host) {
  c->stage_i ^= 1;
  CK(c, cudaEventSynchronize(c->stage_ev[c->stage_i]));
  *host = c->stage[c->stage_i];
  return MIRAGE_OK;
}

// Build attention units for lens[] (logical lengths only -> placement
// independent splits). Returns the unit count and split size in blocks.
// Split-K planning for the persistent attention kernel (a9). Work items are
// (sequence, split, kv head), claimed dynamically by `grid` resident CTAs in
// longest-first order (greedy LPT). Splitting adds per-item overhead and a
// combine, so the split size P (blocks) is the LARGEST one that still gives
// every resident CTA about one item to start with: items(P) >= f * grid, with
// f = 0.8 (f = 0.6 for G = 8); when even the unsplit batch has fewer items than
// the grid, the smallest P with items(P) <= grid (one item per CTA, equal SM
// loads). Equalised so the longest sequence has no runt last split, and at most
// kMaxSplits splits per sequence. Calibrated on B200 (tools/attn_bench.py
// --split sweeps). P depends on logical lengths only, never on
// block placement.
int choose_split(const int32_t* lens, int B, int Hk, int G, int grid, int warps) {
  (void)warps;
  int max_nb = 0;
  std::vector<int> nbs(B);
  for (int b = 0; b < B; ++b) {
    nbs[b] = (lens[b] + kBlockTokens - 1) / kBlockTokens;
    max_nb = std::max(max_nb, nbs[b]);
  }
  const int p_lo = std::max(1, (max_nb + kMaxSplits - 1) / kMaxSplits);
  const double need = (G >= 8 ? 0.6 : 0.8) * std::max(grid, 1);
  auto items = [&](int P) {
    int64_t n = 0;
    for (int b = 0; b < B; ++b) n += (nbs[b] + P - 1) / P;
    return (double)n * Hk;
  };
  int P = std::max(p_lo, max_nb);
  const bool lpt = items(P) >= grid;  // the unsplit batch already has an item for every CTA
  if (!lpt) {
    // Fewer items than resident CTAs: split until the items just fill the grid
    // (the smallest P with items(P) <= grid). Every CTA then holds one item, so
    // the SMs carry equal loads (ncu on 1 x 32k: SMs with 2 CTAs ran ~1.6x
    // longer than SMs with 1 under the "items >= f * grid" rule).
    int lo = p_lo, hi = P;  // items(P) is non-increasing in P
    while (lo < hi) {
      const int mid = (lo + hi) / 2;
      if (items(mid) <= grid) hi = mid;
      else lo = mid + 1;
    }
    P = lo;
  }
  while (P > p_lo && items(P) < need) {
    const int next = std::max(p_lo, std::min(P - 1, (int)(P * 0.97)));
    P = next;
  }
  // a skewed batch (ShareGPT lengths at small B): with enough items for the grid,
  // the longest item still bounds the LPT makespan, so no item may exceed 0.6 of
  // the average load per CTA (C2 P-paper B=29, OPT-13B: split 95 -> 33 blocks,
  // 41.9 -> ~37 us per launch in the tools/attn_bench.py --split sweep)
  if (lpt) {
    int64_t total = 0;
    for (int b = 0; b < B; ++b) total += nbs[b];
    const int cap = (int)std::ceil(0.6 * (double)total * Hk / std::max(grid, 1));
    P = std::max(p_lo, std::min(P, std::max(cap, 1)));
  }
  // equalise the longest sequence's splits (no runt last split)
  const int ns = (max_nb + P - 1) / P;
  return std::max(1, (max_nb + ns - 1) / ns);
}

bool ranges_enabled();

// Balanced ranges (stream-K over the batch): when the one-item-per-CTA split of
// choose_split leaves CTAs idle (e.g. 70B-TP8, 64 sequences x 1 kv head: 256
// equal items on 296 CTAs, so 40 SMs carry one CTA and 108 carry two), the
// concatenated block stream of the batch (sequence order) is cut into
// R = grid / Hk equal ranges instead; range r runs on the Hk CTAs r*Hk ..
// r*Hk + Hk - 1 (one per kv head) as the one or more pieces (units) of the
// sequences it overlaps. A sequence's pieces are its splits, in order, folded by
// the same split-K combine. Depends on logical lengths only (placement
// independent). Returns the unit count (units in range order, rfirst[r] = the
// first unit of range r, rfirst[R] = count) or -1.
int build_units_ranges(const int32_t* lens, const int32_t* seq_off, int B, int Hk, int grid,
                       mirage::AttnUnit* units, int max_units, int32_t* rfirst) {
  const int R = grid / Hk;
  if (R < 1 || R > kMaxRanges) return -1;
  std::vector<int> nbs(B), pieces(B, 0), pbase(B, 0);
  int64_t T = 0;
  for (int b = 0; b < B; ++b) {
    nbs[b] = (lens[b] + kBlockTokens - 1) / kBlockTokens;
    T += nbs[b];
  }
  int n = 0, b = 0;
  int64_t seq_start = 0;  // stream offset of sequence b's block 0
  for (int r = 0; r < R; ++r) {
    const int64_t lo = T * r / R, hi = T * (r + 1) / R;
    rfirst[r] = n;
    while (b < B && seq_start + nbs[b] <= lo) seq_start += nbs[b++];  // skip sequences that end before lo
    int64_t at = lo;
    int bb = b;
    int64_t st = seq_start;
    while (at < hi && bb < B) {
      const int64_t end = std::min(hi, st + nbs[bb]);
      if (end > at) {
        if (n >= max_units) return -1;
        units[n++] = mirage::AttnUnit{bb, (int16_t)pieces[bb], 0, 0, lens[bb], (int32_t)(at - st), (int32_t)(end - st),
                                      seq_off[bb], 1};
        ++pieces[bb];
        at = end;
      }
      if (at >= st + nbs[bb]) {
        st += nbs[bb];
        ++bb;
      }
    }
  }
  rfirst[R] = n;
  int pb = 0;
  for (int q = 0; q < B; ++q) {
    if (pieces[q] > kMaxSplits) return -1;
    pbase[q] = pb;
    if (pieces[q] > 1) pb += pieces[q];
  }
  for (int i = 0; i < n; ++i) {
    const int q = units[i].seq;
    units[i].nsplit = (int16_t)pieces[q];
    units[i].pbase = pieces[q] > 1 ? pbase[q] : 0;
  }
  return n;
}

// Use balanced ranges? Only when choose_split's one-item-per-CTA plan fills less
// than 0.97 of the grid (decode steps, grid a multiple of Hk) and every range is
// long (>= 256 blocks): a CTA's second piece costs a merge during which its TMA
// rings stall, which outweighs the balance gain on short ranges (70B-TP8 64 x 4k,
// 55 blocks per range: 32.9 -> 35.1 us; 32 x 32k, 1771 blocks: 601.8 -> 595.6 us,
// 16 x 16k: 159.0 -> 157.4 us; profiles/r02g_attn_ranges_b2b.jsonl).
bool want_ranges(const int32_t* lens, int B, int Hk, int grid, int P) {
  if (grid % Hk || grid / Hk > kMaxRanges || B < 1) return false;
  int64_t items = 0, T = 0;
  for (int b = 0; b < B; ++b) {
    const int nb = (lens[b] + kBlockTokens - 1) / kBlockTokens;
    items += (nb + P - 1) / P;
    T += nb;
  }
  items *= Hk;
  return items < grid && items < (int64_t)(0.97 * grid) && T >= 256ll * (grid / Hk);
}

int build_units(const int32_t* lens, const int32_t* seq_off, int B, int Hk, int G, int grid, int warps,
                int override_blocks, mirage::AttnUnit* units, int max_units, int* split_blocks,
                int32_t* mode = nullptr, int32_t* rfirst = nullptr) {
  int P = choose_split(lens, B, Hk, G, grid, warps);
  if (override_blocks > 0) P = override_blocks;
  if (mode) *mode = 0;
  // (override_blocks < 0: the test hook that forces the balanced-range schedule)
  if (mode && rfirst && (override_blocks < 0 || (override_blocks == 0 && ranges_enabled() &&
                                                  want_ranges(lens, B, Hk, grid, P)))) {
    const int n = build_units_ranges(lens, seq_off, B, Hk, grid, units, max_units, rfirst);
    if (n > 0) {
      *mode = 1;
      *split_blocks = 0;
      return n;
    }
  }
  int n = 0, pbase = 0;
  for (int b = 0; b < B; ++b) {
    const int nb = (lens[b] + kBlockTokens - 1) / kBlockTokens;
    const int ns = std::max(1, (nb + P - 1) / P);
    if (n + ns > max_units || ns > kMaxSplits) return -1;
    for (int i = 0; i < ns; ++i)
      units[n++] = mirage::AttnUnit{b, (int16_t)i, (int16_t)ns, ns > 1 ? pbase : 0, lens[b], i * P,
                                    std::min(nb, (i + 1) * P), seq_off[b], 1};
    if (ns > 1) pbase += ns;
  }
  // longest-first order for the persistent kernel's round-robin item assignment
  auto size_of = [&](const mirage::AttnUnit& u) { return u.b1 - u.b0; };
  std::stable_sort(units, units + n, [&](const mirage::AttnUnit& a, const mirage::AttnUnit& b) {
    return size_of(a) > size_of(b);
  });
  *split_blocks = P;
  return n;
}

// Units of a step that holds prefill rows: runs of up to qp consecutive rows of
// one sequence at consecutive positions become one unit (the kernel's QP
// variant serves them from one pass over the K|V tiles); never split.
int build_units_rows(const int32_t* lens, const int32_t* seq_off, const int64_t* seq_ids, int B, int qp,
                     mirage::AttnUnit* units, int max_units) {
  int n = 0;
  for (int i = 0; i < B;) {
    int j = i + 1;
    while (j < B && j - i < qp && seq_ids[j] == seq_ids[i] && lens[j] == lens[j - 1] + 1) ++j;
    if (n >= max_units) return -1;
    const int nb = (lens[j - 1] + kBlockTokens - 1) / kBlockTokens;
    units[n++] = mirage::AttnUnit{i, 0, 1, 0, lens[i], 0, nb, seq_off[i], j - i};
    i = j;
  }
  std::stable_sort(units, units + n, [](const mirage::AttnUnit& a, const mirage::AttnUnit& b) {
    return a.b1 - a.b0 > b.b1 - b.b0;
  });
  return n;
}

void harvest_copy_times(Model* M) {
  while (!M->pending.empty()) {
    CopyTiming& t = M->pending.front();
    if (cudaEventQuery(t.t1) != cudaSuccess) break;
    float ms = 0;
    cudaEventElapsedTime(&ms, t.t0, t.t1);
    M->h2d_ms += ms;
    M->h2d_bytes += t.bytes;
    M->h2d_copies += 1;
    M->ev_pool.push_back(t.t0);  // recycled (no event create/destroy on the step path)
    M->ev_pool.push_back(t.t1);
    M->pending.pop_front();
  }
  (void)cudaGetLastError();
}

void harvest_stall_times(Model* M) {
  while (!M->stall_pending.empty()) {
    auto& t = M->stall_pending.front();
    if (cudaEventQuery(t.t1) != cudaSuccess) break;
    float ms = 0;
    cudaEventElapsedTime(&ms, t.t0, t.t1);
    M->stall_ms += ms;
    M->stall_waits += 1;
    M->ev_pool.push_back(t.t0);
    M->ev_pool.push_back(t.t1);
    M->stall_pending.pop_front();
  }
  (void)cudaGetLastError();
}

// attention times of the last timed graph replay: its event pairs are re-recorded
// by the next replay of that graph, so a new timed replay harvests (blocking) first
void harvest_graph_attn(Model* M, bool block) {
  if (!M->tpend) return;
  const std::vector<cudaEvent_t>& ev = M->tpend->tev;
  if (!block && cudaEventQuery(ev.back()) != cudaSuccess) return;
  cudaEventSynchronize(ev.back());
  for (size_t i = 0; i + 1 < ev.size(); i += 2) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
    M->attn_ms += ms;
    M->attn_bytes += M->tpend_bytes;
    M->attn_launches += 1;
  }
  M->tpend = nullptr;
  (void)cudaGetLastError();
}

void harvest_attn_times(Model* M) {
  harvest_graph_attn(M, false);
  while (!M->attn_pending.empty()) {
    auto& t = M->attn_pending.front();
    if (cudaEventQuery(t.t1) != cudaSuccess) break;
    float ms = 0;
    cudaEventElapsedTime(&ms, t.t0, t.t1);
    M->attn_ms += ms;
    M->attn_bytes += t.bytes;
    M->attn_launches += t.reps;
    M->ev_pool.push_back(t.t0);
    M->ev_pool.push_back(t.t1);
    M->attn_pending.pop_front();
  }
  (void)cudaGetLastError();
}

// The captured graphs of M bake in its weight/slot pointers and copy sources:
// drop them whenever its cycle or weight source changes.
void drop_graphs(Model* M) {
  harvest_graph_attn(M, true);
  for (auto& g : M->graphs) {
    cudaGraphExecDestroy(g.second.exec);
    for (auto e : g.second.tev) cudaEventDestroy(e);
  }
  M->graphs.clear();
  M->graph_seen.clear();
  for (auto e : M->cap_ready_ev) cudaEventDestroy(e);
  for (auto e : M->cap_free_ev) cudaEventDestroy(e);
  M->cap_ready_ev.clear();
  M->cap_free_ev.clear();
}

// MIRAGE_ATTN_RANGES=0 disables the balanced-range attention schedule
bool ranges_enabled() {
  static const bool v = !(getenv("MIRAGE_ATTN_RANGES") && atoi(getenv("MIRAGE_ATTN_RANGES")) == 0);
  return v;
}

// One producer lane per consumer warp (AttnParams::prod_lanes; MIRAGE_ATTN_PRODUCER=0: lane 0
// issues every tile in order). Back to back: 1x32k 28.0 -> 27.4 us, 4x16k 46.1 -> 45.1,
// OPT-13B B=400 365.7 -> 362.5; B=64 64.9 -> 65.3, B=29 37.9 -> 38.2 (profiles/r02g/attn_producer_lanes.jsonl)
int attn_prod_lanes() {
  static const int v = !(getenv("MIRAGE_ATTN_PRODUCER") && atoi(getenv("MIRAGE_ATTN_PRODUCER")) == 0);
  return v;
}

// MIRAGE_KV_EVICT_FIRST=0 loads the attention's K|V tiles with the default L2 policy
int kv_evict_first() {
  static const int v = !(getenv("MIRAGE_KV_EVICT_FIRST") && atoi(getenv("MIRAGE_KV_EVICT_FIRST")) == 0);
  return v;
}

// MIRAGE_PDL=0 disables programmatic dependent launch of the attention kernel
int use_pdl() {
  static const int v = !(getenv("MIRAGE_PDL") && atoi(getenv("MIRAGE_PDL")) == 0);
  return v;
}

int prefetch_debug() {
  static const int v = getenv("MIRAGE_PREFETCH_DEBUG") ? atoi(getenv("MIRAGE_PREFETCH_DEBUG")) : 0;
  return v;
}

cudaEvent_t pool_event(Model* M) {
  if (!M->ev_pool.empty()) {
    cudaEvent_t e = M->ev_pool.back();
    M->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void harvest_step_time(Model* M) {
  if (M->step_timed && cudaEventQuery(M->st1) == cudaSuccess) {
    float ms = 0;
    cudaEventElapsedTime(&ms, M->st0, M->st1);
    M->last_step_ms = ms;
    M->step_timed = false;
  }
  (void)cudaGetLastError();
}

// The row-parallel projections (O-proj, FC2/down) of a decode step: with
// MIRAGE_FLAG_TC_GEMM the tcgen05 decode GEMM (decode_gemm.cu) writing split-K
// slices that the residual kernel sums (*nsplit of them); otherwise, or above 256
// rows, cuBLASLt (one fp32 output).

int32_t gemm_lt(mirage_ctx* c, int B, int N, int K, const bf16* W, const bf16* x, void* y, int out_bf16,
                const bf16* bias, int epi);

int32_t gemm_rowpar(mirage_ctx* c, int B, int N, int K, const bf16* W, const bf16* x, float* y, long long y_cap,
                    int* nsplit) {
  *nsplit = 1;
  if (!(c->cfg.flags & MIRAGE_FLAG_TC_GEMM) || B > 256 || K % 8) return gemm_lt(c, B, N, K, W, x, y, 0, nullptr, 0);
  int s = mirage::decode_gemm_splits(N, K, B, c->sms);
  s = (int)std::max<long long>(1, std::min<long long>(s, y_cap / ((long long)B * N)));
  // the slices are summed by the residual kernel (the in-kernel cluster reduction
  // measured slower: decode_gemm.cu)
  KL(c, mirage::launch_decode_gemm(W, N, K, K, x, B, K, y, N, (long long)B * N, s, nullptr, 0, 0, c->cs));
  *nsplit = s;
  return MIRAGE_OK;
}

// NEXT-4: the row-parallel GEMM of a tensor-parallel rank, fused with the one-shot
// all-reduce: one K split (so each rank sends B x N once), the epilogue stores the
// partial tile into this rank's own slot and into its slot of every other rank's
// exchange buffer (parity ep & 1), then bumps each rank's arrival counter for this
// rank; every counter therefore gains `tiles` per GEMM (push_expect).
int32_t tp_push_gemm(mirage_ctx* c, Model* M, int B, int N, int K, const bf16* W, const bf16* x, uint64_t ep) {
  const int par = (int)(ep & 1);
  float* mine = reinterpret_cast<float*>(M->xfer + kAlign + (par * c->tp + c->tp_rank) * M->xfer_part);
  // one K split, so every rank receives B x N exactly once (summing the splits in
  // the kernel through a cluster's distributed shared memory first measured slower:
  // 13.1 vs 12.4 ms per 70B-TP8 shard step, profiles/r02_tp_push_vs_pull_per_rank.jsonl)
  // column groups (batch cut into >= 32-row groups, one CTA each) spread the one
  // split over more SMs: each group re-reads its tile's weights, from L2
  static const int cg_env = getenv("MIRAGE_PUSH_CG") ? atoi(getenv("MIRAGE_PUSH_CG")) : 0;
  const int cg = std::max((B + 255) / 256,
                          cg_env > 0 ? std::min(cg_env, 8) : mirage::decode_gemm_cgroups(N, B, c->sms));
  KL(c, mirage::launch_decode_gemm(W, N, K, K, x, B, K, mine, N, 0, 1, M->push_dst_dev + par * (c->tp - 1),
                                   c->tp - 1, 0, c->cs, M->push_cnt_dev, c->tp, false, nullptr, cg));
  // every CTA signals once
  M->push_expect += (unsigned long long)mirage::decode_gemm_ctas_per_split(N, B, cg);
  return MIRAGE_OK;
}

// y[B][N] = epilogue(x[B][K] W[N][K]^T (+ bias[N])), fp32 accumulate, via cuBLASLt.
// epi: 0 none, 1 bias, 2 relu(+bias). out_bf16 selects the output type.
int32_t gemm_lt(mirage_ctx* c, int B, int N, int K, const bf16* W, const bf16* x, void* y, int out_bf16,
                const bf16* bias, int epi) {
  auto key = std::make_tuple(B, N, K, out_bf16, epi);
  auto it = c->lt_plans.find(key);
  if (it == c->lt_plans.end()) {
    mirage_ctx::LtPlan pl;
    CKB(c, cublasLtMatmulDescCreate(&pl.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    CKB(c, cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta));
    CKB(c, cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb));
    cublasLtEpilogue_t e = epi == 2 ? CUBLASLT_EPILOGUE_RELU_BIAS
                           : epi == 1 ? CUBLASLT_EPILOGUE_BIAS : CUBLASLT_EPILOGUE_DEFAULT;
    CKB(c, cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof e));
    if (epi) {
      const cudaDataType_t bt = CUDA_R_16BF;
      CKB(c, cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof bt));
    }
    CKB(c, cublasLtMatrixLayoutCreate(&pl.a, CUDA_R_16BF, K, N, K));
    CKB(c, cublasLtMatrixLayoutCreate(&pl.b, CUDA_R_16BF, K, B, K));
    CKB(c, cublasLtMatrixLayoutCreate(&pl.d, out_bf16 ? CUDA_R_16BF : CUDA_R_32F, N, B, N));
    cublasLtMatmulPreference_t pref;
    CKB(c, cublasLtMatmulPreferenceCreate(&pref));
    const uint64_t ws = kCublasWs;
    CKB(c, cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof ws));
    static const int kCand = getenv("MIRAGE_GEMM_CANDIDATES") ? std::max(1, std::min(64, atoi(getenv("MIRAGE_GEMM_CANDIDATES")))) : 12;
    cublasLtMatmulHeuristicResult_t res[64];
    int n = 0;
    cublasLtMatmulAlgoGetHeuristic(c->lt, pl.op, pl.a, pl.b, pl.d, pl.d, pref, kCand, res, &n);
    cublasLtMatmulPreferenceDestroy(pref);
    if (n > 0) {
      pl.algo = res[0].algo;
      pl.has_algo = true;
    }
    // Autotune once per shape on the real operands (first decode step = warm-up):
    // time every heuristic candidate on the compute stream, keep the fastest.
    static const bool tune = !getenv("MIRAGE_GEMM_AUTOTUNE") || atoi(getenv("MIRAGE_GEMM_AUTOTUNE")) != 0;
    if (tune && n > 1) {
      if (epi)
        CKB(c, cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof bias));
      cudaEvent_t e0, e1;
      CK(c, cudaEventCreate(&e0));
      CK(c, cudaEventCreate(&e1));
      const float one = 1.f, zero = 0.f;
      float best = 1e30f;
      for (int i = 0; i < n; ++i) {
        if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
        float tot = 0.f;
        bool ok = true;
        for (int r = 0; r < 4 && ok; ++r) {
          CK(c, cudaEventRecord(e0, c->cs));
          ok = cublasLtMatmul(c->lt, pl.op, &one, W, pl.a, x, pl.b, &zero, y, pl.d, y, pl.d, &res[i].algo,
                              c->blas_ws, kCublasWs, c->cs) == CUBLAS_STATUS_SUCCESS;
          CK(c, cudaEventRecord(e1, c->cs));
          CK(c, cudaEventSynchronize(e1));
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          if (r) tot += ms;  // first run is a warm-up
        }
        if (ok && tot < best) {
          best = tot;
          pl.algo = res[i].algo;
        }
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      (void)cudaGetLastError();
    }
    it = c->lt_plans.emplace(key, pl).first;
  }
  const mirage_ctx::LtPlan& pl = it->second;
  if (epi)
    CKB(c, cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof bias));
  const float one = 1.f, zero = 0.f;
  CKB(c, cublasLtMatmul(c->lt, pl.op, &one, W, pl.a, x, pl.b, &zero, y, pl.d, y, pl.d,
                        pl.has_algo ? &pl.algo : nullptr, c->blas_ws, kCublasWs, c->cs));
  return MIRAGE_OK;
}

}  // namespace

// ============================================================================
extern "C" {

int32_t mirage_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return MIRAGE_ERR_RANGE;
  return cudaHostRegister(ptr, bytes, cudaHostRegisterPortable) == cudaSuccess ? MIRAGE_OK : MIRAGE_ERR_CUDA;
}

int32_t mirage_host_unregister(void* ptr) {
  if (!ptr) return MIRAGE_ERR_RANGE;
  return cudaHostUnregister(ptr) == cudaSuccess ? MIRAGE_OK : MIRAGE_ERR_CUDA;
}

int32_t mirage_nccl_unique_id(void* out) {
  if (!out) return MIRAGE_ERR_RANGE;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return MIRAGE_ERR_NCCL;
  std::memcpy(out, &id, sizeof id);
  return MIRAGE_OK;
}

int32_t mirage_model_sizes(const mirage_model_cfg* m, uint64_t* layer_bytes, uint64_t* global_bytes,
                           uint64_t* block_bytes) {
  if (!m) return MIRAGE_ERR_CONFIG;
  const Shape s = shape_of(m);
  if (check_shape(s)) return MIRAGE_ERR_CONFIG;
  const Sizes z = sizes_of(s);
  if (layer_bytes) *layer_bytes = z.S;
  if (global_bytes) *global_bytes = z.G;
  if (block_bytes) *block_bytes = z.BB;
  return MIRAGE_OK;
}

int32_t mirage_model_arena_bytes(const mirage_model_cfg* m, int64_t native_kv_blocks,
                                 int32_t max_batch, int32_t max_ctx, uint64_t* bytes) {
  if (!m || !bytes || native_kv_blocks < 0 || max_batch <= 0 || max_ctx <= 0)
    return MIRAGE_ERR_CONFIG;
  const Shape s = shape_of(m);
  if (check_shape(s)) return MIRAGE_ERR_CONFIG;
  *bytes = model_arena(s, native_kv_blocks, max_batch, units_cap(max_batch)) + kAlign;
  return MIRAGE_OK;
}

int32_t mirage_init(const mirage_init_cfg* cfg, mirage_ctx** out) {
  if (!cfg || !out) return MIRAGE_ERR_CONFIG;
  *out = nullptr;
  if (cfg->block_tokens != kBlockTokens || cfg->tp_size < 1 || cfg->tp_rank < 0 ||
      cfg->tp_rank >= cfg->tp_size ||
      (cfg->tp_size > 1 && !cfg->nccl_id && !(cfg->flags & MIRAGE_FLAG_TP_IPC)) ||
      !cfg->dev_arena || (!cfg->compute_stream && !(cfg->flags & MIRAGE_FLAG_HOST_ONLY)) ||
      cfg->max_batch <= 0 || cfg->max_ctx <= 0 ||
      (reinterpret_cast<uintptr_t>(cfg->dev_arena) % kAlign))
    return MIRAGE_ERR_CONFIG;
  mirage_ctx* c = new mirage_ctx();
  c->cfg = *cfg;
  c->arena = reinterpret_cast<char*>(cfg->dev_arena);
  c->cs = reinterpret_cast<cudaStream_t>(cfg->compute_stream);
  c->max_units = units_cap(cfg->max_batch);
  c->max_blk = (cfg->max_ctx + kBlockTokens - 1) / kBlockTokens;
  auto bail = [&](int32_t code) {
    mirage_destroy(c);
    return code;
  };
  if (cfg->flags & MIRAGE_FLAG_HOST_ONLY) {  // no CUDA calls at all
    c->host_only = true;
    c->cs = nullptr;
    *out = c;
    return MIRAGE_OK;
  }
  if (cudaSetDevice(cfg->device) != cudaSuccess) return bail(MIRAGE_ERR_CUDA);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, cfg->device);
  if (cfg->copy_stream) {
    c->xs = reinterpret_cast<cudaStream_t>(cfg->copy_stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking) != cudaSuccess)
      return bail(MIRAGE_ERR_CUDA);
    c->own_xs = true;
  }
  if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) return bail(MIRAGE_ERR_CUDA);
  if (cublasLtCreate(&c->lt) != CUBLAS_STATUS_SUCCESS) return bail(MIRAGE_ERR_CUDA);
  if (cudaMalloc(&c->blas_ws, kCublasWs) != cudaSuccess) return bail(MIRAGE_ERR_CUDA);

  if (cublasSetWorkspace(c->blas, c->blas_ws, kCublasWs) != CUBLAS_STATUS_SUCCESS ||
      cublasSetStream(c->blas, c->cs) != CUBLAS_STATUS_SUCCESS)
    return bail(MIRAGE_ERR_CUDA);
  c->meta_bytes = meta_size(c);
  for (int i = 0; i < 2; ++i) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&c->stage[i]), c->meta_bytes, cudaHostAllocDefault) !=
            cudaSuccess ||
        cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(MIRAGE_ERR_CUDA);
  }
  if (getenv("MIRAGE_ATTN_TRACE") &&
      cudaMalloc(reinterpret_cast<void**>(&c->attn_trace), (size_t)mirage_ctx::kTraceCtas * 16 * 8) != cudaSuccess)
    c->attn_trace = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&c->meta_dev), c->meta_bytes) != cudaSuccess)
    return bail(MIRAGE_ERR_CUDA);
  c->tp = cfg->tp_size;
  c->tp_rank = cfg->tp_rank;
  if (cfg->nccl_id) {  // tp_size == 1 with an id runs the same all-reduce path on one rank
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof id);
    if (ncclCommInitRank(&c->nccl, c->tp, id, c->tp_rank) != ncclSuccess) return bail(MIRAGE_ERR_NCCL);
  }
  *out = c;
  return MIRAGE_OK;
}

void mirage_destroy(mirage_ctx* c) {
  if (!c) return;
  if (c->host_only) {
    for (Model* M : c->models) delete M;
    delete c;
    return;
  }
  if (c->cs) cudaStreamSynchronize(c->cs);
  if (c->xs) cudaStreamSynchronize(c->xs);
  for (Model* M : c->models) {
    for (auto e : M->ready_ev) cudaEventDestroy(e);
    for (auto e : M->free_ev) cudaEventDestroy(e);
    for (auto e : M->reload_ev)
      if (e) cudaEventDestroy(e);
    for (auto& t : M->pending) {
      cudaEventDestroy(t.t0);
      cudaEventDestroy(t.t1);
    }
    if (M->st0) cudaEventDestroy(M->st0);
    if (M->st1) cudaEventDestroy(M->st1);
    if (M->bbase_dev) cudaFree(M->bbase_dev);
    if (M->slot_tag) cudaFree(M->slot_tag);
    if (M->tag_err) cudaFree(M->tag_err);
    if (M->host_tags) cudaFreeHost(M->host_tags);
    for (auto& t : M->stall_pending) {
      cudaEventDestroy(t.t0);
      cudaEventDestroy(t.t1);
    }
    for (auto& t : M->attn_pending) {
      cudaEventDestroy(t.t0);
      cudaEventDestroy(t.t1);
    }
    for (auto e : M->ev_pool) cudaEventDestroy(e);
    drop_graphs(M);
    if (M->join_ev) cudaEventDestroy(M->join_ev);
    for (size_t r = 0; r < M->peer_base.size(); ++r)
      if (M->peer_base[r] && M->peer_base[r] != M->xfer) cudaIpcCloseMemHandle(M->peer_base[r]);
    if (M->xfer) cudaFree(M->xfer);
    if (M->push_dst_dev) cudaFree(M->push_dst_dev);
    if (M->local_slots_dev) cudaFree(M->local_slots_dev);
    if (M->push_cnt_dev) cudaFree(M->push_cnt_dev);
    if (M->parts_dev) cudaFree(M->parts_dev);
    if (M->flags_dev) cudaFree(M->flags_dev);
    if (M->tp_err) cudaFree(M->tp_err);
    delete M;
  }
  for (int i = 0; i < 2; ++i) {
    if (c->stage[i]) cudaFreeHost(c->stage[i]);
    if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
  }
  if (c->meta_dev) cudaFree(c->meta_dev);
  if (c->attn_trace) cudaFree(c->attn_trace);
  if (c->blas) cublasDestroy(c->blas);
  for (auto& kv : c->lt_plans) {
    cublasLtMatmulDescDestroy(kv.second.op);
    cublasLtMatrixLayoutDestroy(kv.second.a);
    cublasLtMatrixLayoutDestroy(kv.second.b);
    cublasLtMatrixLayoutDestroy(kv.second.d);
  }
  if (c->lt) cublasLtDestroy(c->lt);
  if (c->blas_ws) cudaFree(c->blas_ws);

  if (c->own_xs && c->xs) cudaStreamDestroy(c->xs);
  if (c->nccl) ncclCommDestroy(c->nccl);
  (void)cudaGetLastError();
  delete c;
}

const char* mirage_last_error(const mirage_ctx* c) { return c ? c->err.c_str() : "null ctx"; }

int64_t mirage_kernel_launches(const mirage_ctx* c) { return c ? c->launches : 0; }


int32_t mirage_decode_gemm(void* stream, const void* w_dev, int32_t N, int32_t K, const void* x_dev, int32_t B,
                           float* y_dev, int32_t splits, int32_t reduce, int32_t col_groups, int32_t* splits_out) {
  if (!w_dev || !x_dev || !y_dev || N <= 0 || K <= 0 || K % 8 || B <= 0 || col_groups < 0 || col_groups > 8 ||
      B > 256 * std::max(1, col_groups) || splits < 0 || splits > mirage::kMaxGemmSplits)
    return MIRAGE_ERR_RANGE;
  if (splits == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    splits = mirage::decode_gemm_splits(N, K, B, sms);
  }
  if (reduce) splits = std::min(splits, 8);
  int slices = splits;
  const cudaError_t e = mirage::launch_decode_gemm(
      reinterpret_cast<const bf16*>(w_dev), N, K, K, reinterpret_cast<const bf16*>(x_dev), B, K, y_dev, N,
      (long long)B * N, splits, nullptr, 0, 0, reinterpret_cast<cudaStream_t>(stream), nullptr, 0, reduce != 0,
      &slices, col_groups > 0 ? col_groups : 1);
  if (splits_out) *splits_out = slices;
  return e == cudaSuccess ? MIRAGE_OK : MIRAGE_ERR_CUDA;
}

int32_t mirage_set_flags(mirage_ctx* c, uint32_t flags, uint32_t mask) {
  GUARD(c);
  const uint32_t allowed = MIRAGE_FLAG_TIME_ATTN | MIRAGE_FLAG_CUDA_GRAPHS;
  if (mask & ~allowed) return fail(c, MIRAGE_ERR_CONFIG, "set_flags: only TIME_ATTN / CUDA_GRAPHS may change");
  c->cfg.flags = (c->cfg.flags & ~mask) | (flags & mask);
  return MIRAGE_OK;
}

int32_t mirage_sk_gemm(void* stream, const void* w_dev, int32_t N, int32_t K, const void* x_dev, int32_t B,
                       float* y_dev, void* y16_dev, const void* bias_dev, int32_t relu) {
  if (!w_dev || !x_dev || (!y_dev && !y16_dev) || N <= 0 || K <= 0 || K % 8 || B <= 0 || B > 256)
    return MIRAGE_ERR_RANGE;
  // process-wide workspace of the hook, one per device: partial slots and flags for
  // one wave (calls on one device must be stream-ordered: they share it)
  static std::mutex mu;
  static std::map<int, std::pair<float*, int*>> wsmap;
  float* ws = nullptr;
  int* flags = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return MIRAGE_ERR_CUDA;
    auto it = wsmap.find(dev);
    if (it == wsmap.end()) {
      const size_t n = (size_t)mirage::sk_gemm_max_ctas() * 256 * 128;
      if (cudaMalloc(&ws, n * 4) != cudaSuccess) return MIRAGE_ERR_CUDA;
      if (cudaMalloc(&flags, (size_t)mirage::sk_gemm_max_ctas() * 4) != cudaSuccess) return MIRAGE_ERR_CUDA;
      if (cudaMemset(flags, 0, (size_t)mirage::sk_gemm_max_ctas() * 4) != cudaSuccess) return MIRAGE_ERR_CUDA;
      it = wsmap.emplace(dev, std::make_pair(ws, flags)).first;
    }
    ws = it->second.first;
    flags = it->second.second;
  }
  const cudaError_t e = mirage::launch_sk_gemm(
      reinterpret_cast<const bf16*>(w_dev), N, K, K, reinterpret_cast<const bf16*>(x_dev), B, K, y_dev,
      y_dev ? nullptr : reinterpret_cast<bf16*>(y16_dev), N, reinterpret_cast<const bf16*>(bias_dev), relu, ws, flags,
      nullptr, 0, 0, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MIRAGE_OK : MIRAGE_ERR_CUDA;
}

int32_t mirage_attn_trace(mirage_ctx* c, uint64_t* host_out, int32_t cap_ctas, int32_t* n_ctas) {
  GUARD(c);
  if (!c->attn_trace) return fail(c, MIRAGE_ERR_STATE, "attn_trace: set MIRAGE_ATTN_TRACE before mirage_init");
  if (n_ctas) *n_ctas = c->attn_trace_ctas;
  if (!host_out || cap_ctas < c->attn_trace_ctas) return fail(c, MIRAGE_ERR_RANGE, "attn_trace: capacity");
  CK(c, cudaStreamSynchronize(c->cs));
  CK(c, cudaMemcpy(host_out, c->attn_trace, (size_t)c->attn_trace_ctas * 16 * 8, cudaMemcpyDeviceToHost));
  return MIRAGE_OK;
}

int32_t mirage_add_model(mirage_ctx* c, const mirage_model_cfg* mc, const void* host_blob,
                         uint64_t host_bytes, int64_t native_kv_blocks, int32_t* model_id) {
  GUARD(c);
  if (!mc || !host_blob || !model_id || native_kv_blocks < 0)
    return fail(c, MIRAGE_ERR_CONFIG, "add_model: null argument or negative pool");
  Shape s = shape_of(mc);
  if (const char* why = check_shape(s)) return fail(c, MIRAGE_ERR_CONFIG, "add_model: bad %s", why);
  if (c->tp > 1) {  // this rank's head shard (include/mirage.h)
    if (s.family != MIRAGE_FAMILY_LLAMA || s.H % c->tp || s.Hk % c->tp || s.f % (128 * c->tp))
      return fail(c, MIRAGE_ERR_CONFIG, "add_model: tensor parallelism needs a Llama shape divisible by tp");
    s.H /= c->tp;
    s.Hk /= c->tp;
    s.f /= c->tp;
  }
  const Sizes z = sizes_of(s);
  if (host_bytes != (uint64_t)s.n * z.S + z.G)
    return fail(c, MIRAGE_ERR_CONFIG, "add_model: host_bytes %llu != n*S+G %llu",
                (unsigned long long)host_bytes, (unsigned long long)((uint64_t)s.n * z.S + z.G));
  cudaPointerAttributes attr;
  if (!c->host_only &&
      (cudaPointerGetAttributes(&attr, host_blob) != cudaSuccess || attr.type != cudaMemoryTypeHost)) {
    (void)cudaGetLastError();
    return fail(c, MIRAGE_ERR_CONFIG, "add_model: host blob must be pinned host memory");
  }
  Model* M = new Model();
  M->shp = s;
  M->sz = z;
  M->host = reinterpret_cast<const char*>(host_blob);
  M->n_native = native_kv_blocks;
  const int Bm = c->cfg.max_batch;
  const WsPlan w = ws_plan(s, Bm, c->max_units);
  auto C = [&](uint64_t b) { return carve(c, b); };
  M->w_dev = C((uint64_t)s.n * z.S + z.G);
  M->pool = native_kv_blocks ? C((uint64_t)native_kv_blocks * z.BB) : c->arena;
  M->h = reinterpret_cast<float*>(C(w.h));
  M->x = reinterpret_cast<bf16*>(C(w.x));
  M->y = reinterpret_cast<float*>(C(w.y));
  M->q = reinterpret_cast<uint32_t*>(C(w.q));
  M->f = reinterpret_cast<bf16*>(C(w.f));
  M->partial = reinterpret_cast<float*>(C(w.partial));
  M->tickets = reinterpret_cast<int32_t*>(C(w.tickets));
  M->argmax = reinterpret_cast<int32_t*>(C(w.argmax));
  M->y_ld_max = w.y_ld;
  if (!M->w_dev || !M->pool || !M->h || !M->x || !M->y || !M->q || !M->f || !M->partial ||
      !M->tickets || !M->argmax) {
    delete M;
    return fail(c, MIRAGE_ERR_CAPACITY, "add_model: arena exhausted (%llu of %llu bytes used)",
                (unsigned long long)c->arena_used, (unsigned long long)c->cfg.dev_arena_bytes);
  }
  // block_base (library-owned): native ids + everything the arena could donate
  const uint64_t cap = (uint64_t)native_kv_blocks + c->cfg.dev_arena_bytes / z.BB + 16;
  if (!c->host_only && cudaMalloc(reinterpret_cast<void**>(&M->bbase_dev), cap * 8) != cudaSuccess) {
    delete M;
    return fail(c, MIRAGE_ERR_CUDA, "add_model: block_base allocation");
  }
  M->bbase_cap = (int64_t)cap;
  M->next_id = (int32_t)native_kv_blocks;
  for (int32_t i = 0; i < native_kv_blocks; ++i) {
    M->free_ids.insert(M->free_ids.end(), i);
    M->loc_donor.push_back(-1);
    M->loc_off.push_back((uint64_t)i * z.BB);
    M->bbase_host.push_back(reinterpret_cast<uint64_t>(M->pool) + (uint64_t)i * z.BB);
  }
  M->layer_state.assign(s.n, RESIDENT);
  M->cyc_index.assign(s.n, -1);
  if (c->host_only) {
    M->id = (int32_t)c->models.size();
    c->models.push_back(M);
    *model_id = M->id;
    return MIRAGE_OK;
  }
  if (c->cfg.flags & MIRAGE_FLAG_SLOT_TAGS) {
    CK(c, cudaMalloc(reinterpret_cast<void**>(&M->slot_tag), MIRAGE_MAX_CYCLE * 4));
    CK(c, cudaMalloc(reinterpret_cast<void**>(&M->tag_err), 8));
    CK(c, cudaMemsetAsync(M->tag_err, 0, 8, c->cs));
    CK(c, cudaHostAlloc(reinterpret_cast<void**>(&M->host_tags), (size_t)s.n * 4, cudaHostAllocDefault));
    for (int l = 0; l < s.n; ++l)
      M->host_tags[l] = 0xA5000000u | ((uint32_t)(c->models.size() & 0xff) << 16) | (uint32_t)l;
  }
  CK(c, cudaMemcpyAsync(M->w_dev, host_blob, host_bytes, cudaMemcpyHostToDevice, c->cs));
  if (native_kv_blocks)
    CK(c, cudaMemcpyAsync(M->bbase_dev, M->bbase_host.data(), native_kv_blocks * 8,
                          cudaMemcpyHostToDevice, c->cs));
  CK(c, cudaMemsetAsync(M->tickets, 0, w.tickets, c->cs));
  CK(c, cudaEventCreate(&M->st0));
  CK(c, cudaEventCreate(&M->st1));
  CK(c, cudaStreamSynchronize(c->cs));
  M->id = (int32_t)c->models.size();
  c->models.push_back(M);
  *model_id = M->id;
  return MIRAGE_OK;
}

int32_t mirage_tp_export(mirage_ctx* c, int32_t model, void* handle_out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !handle_out) return fail(c, MIRAGE_ERR_RANGE, "tp_export: arguments");
  if (!(c->cfg.flags & MIRAGE_FLAG_TP_IPC) || c->host_only)
    return fail(c, MIRAGE_ERR_CONFIG, "tp_export: needs MIRAGE_FLAG_TP_IPC");
  if (!M->xfer) {
    M->xfer_part = align_up((uint64_t)c->cfg.max_batch * M->shp.d * 4, kAlign);
    M->tp_push = (c->cfg.flags & MIRAGE_FLAG_TC_GEMM) && c->cfg.max_batch <= 256;
    const size_t bytes = kAlign + 2 * (M->tp_push ? (size_t)c->tp : 1) * M->xfer_part;
    CK(c, cudaMalloc(reinterpret_cast<void**>(&M->xfer), bytes));
    CK(c, cudaMemset(M->xfer, 0, bytes));
  }
  cudaIpcMemHandle_t h;
  CK(c, cudaIpcGetMemHandle(&h, M->xfer));
  std::memcpy(handle_out, &h, sizeof h);
  return MIRAGE_OK;
}

int32_t mirage_tp_import(mirage_ctx* c, int32_t model, const void* handles) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !handles || !M->xfer) return fail(c, MIRAGE_ERR_STATE, "tp_import: export first");
  const int tp = c->tp;
  M->peer_base.assign(tp, nullptr);
  for (int r = 0; r < tp; ++r) {
    if (r == c->tp_rank) {
      M->peer_base[r] = M->xfer;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, reinterpret_cast<const char*>(handles) + (size_t)r * sizeof h, sizeof h);
    void* p = nullptr;
    CK(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    M->peer_base[r] = reinterpret_cast<char*>(p);
  }
  std::vector<float*> parts(2 * tp);
  std::vector<unsigned long long*> flags(tp);
  for (int r = 0; r < tp; ++r) {
    flags[r] = reinterpret_cast<unsigned long long*>(M->peer_base[r]);
    for (int par = 0; par < 2; ++par)
      parts[par * tp + r] = reinterpret_cast<float*>(M->peer_base[r] + kAlign + par * M->xfer_part);
  }
  if (M->tp_push) {  // fused GEMM + all-reduce: where my GEMM pushes, where I read, whom I signal
    const int me = c->tp_rank;
    std::vector<float*> dst(2 * (tp - 1)), mine(2 * tp);
    std::vector<unsigned long long*> cnt(tp);
    for (int par = 0; par < 2; ++par) {
      int k = 0;
      for (int r = 0; r < tp; ++r) {
        mine[par * tp + r] = reinterpret_cast<float*>(M->xfer + kAlign + (par * tp + r) * M->xfer_part);
        if (r != me)
          dst[par * (tp - 1) + k++] =
              reinterpret_cast<float*>(M->peer_base[r] + kAlign + (par * tp + me) * M->xfer_part);
      }
    }
    for (int r = 0; r < tp; ++r) cnt[r] = reinterpret_cast<unsigned long long*>(M->peer_base[r] + 8 + 8 * me);
    CK(c, cudaMalloc(reinterpret_cast<void**>(&M->push_dst_dev), std::max<size_t>(1, dst.size()) * sizeof(float*)));
    CK(c, cudaMalloc(reinterpret_cast<void**>(&M->local_slots_dev), mine.size() * sizeof(float*)));
    CK(c, cudaMalloc(reinterpret_cast<void**>(&M->push_cnt_dev), cnt.size() * sizeof(void*)));
    if (!dst.empty())
      CK(c, cudaMemcpy(M->push_dst_dev, dst.data(), dst.size() * sizeof(float*), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(M->local_slots_dev, mine.data(), mine.size() * sizeof(float*), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(M->push_cnt_dev, cnt.data(), cnt.size() * sizeof(void*), cudaMemcpyHostToDevice));
  }
  CK(c, cudaMalloc(reinterpret_cast<void**>(&M->parts_dev), parts.size() * sizeof(float*)));
  CK(c, cudaMalloc(reinterpret_cast<void**>(&M->flags_dev), flags.size() * sizeof(void*)));
  CK(c, cudaMalloc(reinterpret_cast<void**>(&M->tp_err), 4));
  CK(c, cudaMemcpy(M->parts_dev, parts.data(), parts.size() * sizeof(float*), cudaMemcpyHostToDevice));
  CK(c, cudaMemcpy(M->flags_dev, flags.data(), flags.size() * sizeof(void*), cudaMemcpyHostToDevice));
  CK(c, cudaMemset(M->tp_err, 0, 4));
  M->tp_ready = true;
  return MIRAGE_OK;
}

int32_t mirage_set_weight_source(mirage_ctx* c, int32_t model, const void* src, uint64_t bytes) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !src) return fail(c, MIRAGE_ERR_RANGE, "weight_source: arguments");
  if (bytes != (uint64_t)M->shp.n * M->sz.S + M->sz.G)
    return fail(c, MIRAGE_ERR_CONFIG, "weight_source: %llu bytes, blob is %llu", (unsigned long long)bytes,
                (unsigned long long)((uint64_t)M->shp.n * M->sz.S + M->sz.G));
  if (!c->host_only) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, src) != cudaSuccess ||
        (a.type != cudaMemoryTypeHost && a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)) {
      (void)cudaGetLastError();
      return fail(c, MIRAGE_ERR_CONFIG, "weight_source: must be pinned host or device memory");
    }
    if (a.type == cudaMemoryTypeDevice && a.device != c->cfg.device) {  // a peer GPU's HBM over NVLink
      cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();
        return fail(c, MIRAGE_ERR_CONFIG, "weight_source: no peer access to device %d", a.device);
      }
      (void)cudaGetLastError();
    }
    CK(c, cudaStreamSynchronize(c->xs));  // no copy from the old source is in flight
  }
  M->host = reinterpret_cast<const char*>(src);
  drop_graphs(M);  // captured copies read the old source
  return MIRAGE_OK;
}

// Enqueue M's requested reloads on the copy stream, ordered after everything
// enqueued so far on the compute stream (the last readers of the bytes as KV,
// and the caller's metadata upload), one event per layer (reload_ev).
static int32_t flush_reloads(mirage_ctx* c, Model* D) {
  if (D->reload_queue.empty() || c->host_only) return MIRAGE_OK;
  std::vector<int32_t> layers;
  layers.swap(D->reload_queue);
  std::sort(layers.begin(), layers.end());
  layers.erase(std::unique(layers.begin(), layers.end()), layers.end());
  cudaEvent_t e;
  CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(c, cudaEventRecord(e, c->cs));
  CK(c, cudaStreamWaitEvent(c->xs, e, 0));
  cudaEventDestroy(e);
  if (D->reload_ev.empty()) {
    D->reload_ev.assign(D->shp.n, nullptr);
    D->reload_pending.assign(D->shp.n, 0);
  }
  for (int32_t l : layers) {
    if (!D->reload_ev[l]) CK(c, cudaEventCreateWithFlags(&D->reload_ev[l], cudaEventDisableTiming));
    CopyTiming t{pool_event(D), pool_event(D), D->sz.S};
    if (!t.t0 || !t.t1) return fail(c, MIRAGE_ERR_CUDA, "reload: event pool");
    CK(c, cudaEventRecord(t.t0, c->xs));
    if (prefetch_debug() == 3 || prefetch_debug() == 4)  // test hook: a slow link
      KL(c, mirage::launch_spin(20000000ull, c->xs));
    CK(c, cudaMemcpyAsync(D->w_dev + (uint64_t)l * D->sz.S, D->host + (uint64_t)l * D->sz.S, D->sz.S,
                          cudaMemcpyDefault, c->xs));
    CK(c, cudaEventRecord(t.t1, c->xs));
    CK(c, cudaEventRecord(D->reload_ev[l], c->xs));
    D->pending.push_back(t);
    D->reload_pending[l] = 1;
  }
  return MIRAGE_OK;
}

// Order the compute stream after every pending asynchronous reload of M (before
// M's weight bytes are handed out again, swapped or re-streamed).
static int32_t settle_reloads(mirage_ctx* c, Model* M) {
  if (int32_t e = flush_reloads(c, M)) return e;
  for (size_t l = 0; l < M->reload_pending.size(); ++l)
    if (M->reload_pending[l]) {
      CK(c, cudaStreamWaitEvent(c->cs, M->reload_ev[l], 0));
      M->reload_pending[l] = 0;
    }
  return MIRAGE_OK;
}

int32_t mirage_set_active(mirage_ctx* c, int32_t model, int32_t active) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M) return fail(c, MIRAGE_ERR_RANGE, "set_active: model %d", model);
  if (active && !M->active) {
    // a reclaimed layer runs only if it is streamed through this model's own cycle
    for (int32_t l = 0; l < M->shp.n; ++l)
      if (M->layer_state[l] == RECLAIMED && M->cyc_index[l] < 0)
        return fail(c, MIRAGE_ERR_STATE, "set_active: model %d layer %d is reclaimed outside its cycle", model, l);
  }
  M->active = active != 0;
  return MIRAGE_OK;
}

int32_t mirage_remap_layers(mirage_ctx* c, int32_t donor, int32_t recipient, const int32_t* cycle,
                            int32_t m, int32_t beta, int64_t* blocks_gained,
                            uint64_t* reclaimed_bytes) {
  GUARD(c);
  Model* D = get_model(c, donor);
  Model* R = get_model(c, recipient);
  if (!D || !R) return fail(c, MIRAGE_ERR_RANGE, "remap: model id");
  if (m <= 0 || m > D->shp.n || !cycle || beta < 0 || beta > m)
    return fail(c, MIRAGE_ERR_RANGE, "remap: m=%d beta=%d", m, beta);
  for (int i = 0; i < m; ++i) {
    if (cycle[i] < 0 || cycle[i] >= D->shp.n) return fail(c, MIRAGE_ERR_RANGE, "remap: layer %d", cycle[i]);
    if (i && cycle[i] <= cycle[i - 1])
      return fail(c, MIRAGE_ERR_RANGE, "remap: cycle must be strictly ascending");
  }
  for (int i = 0; i < m; ++i)
    if (D->layer_state[cycle[i]] != RESIDENT)
      return fail(c, MIRAGE_ERR_STATE, "remap: layer %d already cycled or reclaimed", cycle[i]);
  if (beta == 0 && D->active) return fail(c, MIRAGE_ERR_STATE, "remap: beta=0 needs an inactive donor");
  if (beta > 0 && donor != recipient)
    return fail(c, MIRAGE_ERR_STATE, "remap: streaming remap must be a self-remap");
  if (beta > 0 && !D->cycle.empty()) return fail(c, MIRAGE_ERR_STATE, "remap: donor already has a cycle");
  if (!c->host_only)  // bytes still being reloaded must land before they become KV or slots again
    if (int32_t e = settle_reloads(c, D)) return e;
  // carve R = cycle[beta:] into runs of consecutive layers
  std::vector<int32_t> Rl(cycle + beta, cycle + m);
  int64_t gained = 0;
  std::vector<std::pair<int32_t, int32_t>> runs;  // (first, count)
  for (int32_t l : Rl) {
    if (!runs.empty() && runs.back().first + runs.back().second == l) runs.back().second++;
    else runs.push_back({l, 1});
  }
  int64_t total_new = 0;
  for (auto& r : runs) total_new += (int64_t)((uint64_t)r.second * D->sz.S / R->sz.BB);
  if ((int64_t)R->next_id + total_new > R->bbase_cap) {  // grow the device block_base mirror
    if (c->host_only) {
      R->bbase_cap = std::max<int64_t>(2 * R->bbase_cap, R->next_id + total_new);
    } else {
      const int64_t cap = std::max<int64_t>(2 * R->bbase_cap, R->next_id + total_new + 16);
      uint64_t* nb = nullptr;
      CK(c, cudaStreamSynchronize(c->cs));
      CK(c, cudaMalloc(reinterpret_cast<void**>(&nb), cap * 8));
      if (R->next_id)
        CK(c, cudaMemcpy(nb, R->bbase_host.data(), (size_t)R->next_id * 8, cudaMemcpyHostToDevice));
      cudaFree(R->bbase_dev);
      R->bbase_dev = nb;
      R->bbase_cap = cap;
    }
  }
  const int32_t first_new = R->next_id;
  for (auto& r : runs) {
    const uint64_t off = (uint64_t)r.first * D->sz.S;
    const uint64_t len = (uint64_t)r.second * D->sz.S;
    const int64_t k = (int64_t)(len / R->sz.BB);
    R->regions.push_back(Region{donor, r.first, r.second, R->next_id, (int32_t)k, beta > 0, false});
    for (int64_t i = 0; i < k; ++i) {
      const int32_t id = R->next_id++;
      R->free_ids.insert(id);
      R->loc_donor.push_back(donor);
      R->loc_off.push_back(off + (uint64_t)i * R->sz.BB);
      R->bbase_host.push_back(reinterpret_cast<uint64_t>(D->w_dev) + off + (uint64_t)i * R->sz.BB);
    }
    gained += k;
  }
  R->reclaimed_bytes += (uint64_t)Rl.size() * D->sz.S;
  D->donated_bytes += (uint64_t)Rl.size() * D->sz.S;
  for (int i = 0; i < beta; ++i) D->layer_state[cycle[i]] = SLOT;
  for (int32_t l : Rl) D->layer_state[l] = RECLAIMED;
  if ((c->cfg.flags & MIRAGE_FLAG_POISON) && !c->host_only)  // debug: reclaimed bytes become NaN
    for (auto& r : runs)
      CK(c, cudaMemsetAsync(D->w_dev + (uint64_t)r.first * D->sz.S, 0xFF, (uint64_t)r.second * D->sz.S, c->cs));
  if (gained && !c->host_only)  // stream-ordered after every kernel that read these bytes as weights
    CK(c, cudaMemcpyAsync(R->bbase_dev + first_new, R->bbase_host.data() + first_new, gained * 8,
                          cudaMemcpyHostToDevice, c->cs));
  if (beta > 0) {
    D->cycle.assign(cycle, cycle + m);
    D->beta = beta;
    for (int i = 0; i < m; ++i) D->cyc_index[cycle[i]] = i;
    D->uses = 0;
    D->cyc_steps = 0;
    D->slot_log.clear();
    if (D->slot_tag && !c->host_only)
      for (int j = 0; j < beta; ++j)
        CK(c, cudaMemcpyAsync(D->slot_tag + j, D->host_tags + cycle[j], 4, cudaMemcpyHostToDevice, c->cs));
    for (int j = 0; j < beta && !c->host_only; ++j) {
      cudaEvent_t a, b;
      CK(c, cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      CK(c, cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      D->ready_ev.push_back(a);
      D->free_ev.push_back(b);
    }
    if (beta > 0) drop_graphs(D);
  }
  if (gained && !c->host_only) CK(c, cudaStreamSynchronize(c->cs));  // the host staging above is a pageable vector
  if (blocks_gained) *blocks_gained = gained;
  if (reclaimed_bytes) *reclaimed_bytes = (uint64_t)Rl.size() * D->sz.S;
  return MIRAGE_OK;
}

int32_t mirage_region_count(mirage_ctx* c, int32_t model, int32_t* n) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !n) return fail(c, MIRAGE_ERR_RANGE, "region_count: model %d", model);
  *n = (int32_t)M->regions.size();
  return MIRAGE_OK;
}

int32_t mirage_region_info(mirage_ctx* c, int32_t model, int32_t idx, mirage_region* out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !out || idx < 0 || idx >= (int32_t)M->regions.size())
    return fail(c, MIRAGE_ERR_RANGE, "region_info: model %d region %d", model, idx);
  const Region& r = M->regions[idx];
  out->donor = r.donor;
  out->first_layer = r.first_layer;
  out->n_layers = r.n_layers;
  out->first_id = r.first_id;
  out->n_blocks = r.n_blocks;
  out->n_free = 0;
  for (int32_t i = r.first_id; i < r.first_id + r.n_blocks; ++i) out->n_free += M->free_ids.count(i);
  out->cycle = r.cycle;
  out->retired = r.retired;
  return MIRAGE_OK;
}

// Dynamic Reversion.
int32_t mirage_unremap(mirage_ctx* c, int32_t recipient, int32_t region) {
  GUARD(c);
  Model* R = get_model(c, recipient);
  if (!R || region < 0 || region >= (int32_t)R->regions.size())
    return fail(c, MIRAGE_ERR_RANGE, "unremap: model %d region %d", recipient, region);
  if (R->regions[region].retired) return fail(c, MIRAGE_ERR_STATE, "unremap: region %d already reverted", region);
  const int32_t donor = R->regions[region].donor;
  Model* D = get_model(c, donor);
  // a streaming cycle is reverted as a whole (all of its regions); otherwise one region
  std::vector<int32_t> which;
  if (R->regions[region].cycle) {
    for (int32_t i = 0; i < (int32_t)R->regions.size(); ++i)
      if (R->regions[i].cycle && R->regions[i].donor == donor && !R->regions[i].retired) which.push_back(i);
  } else {
    which.push_back(region);
  }
  int64_t used = 0;
  for (int32_t i : which) {
    const Region& r = R->regions[i];
    for (int32_t b = r.first_id; b < r.first_id + r.n_blocks; ++b) used += !R->free_ids.count(b);
  }
  if (used) return fail(c, MIRAGE_ERR_PRESSURE, "unremap: %lld blocks of the region still hold KV", (long long)used);
  // retire the ids: never handed out again
  std::vector<int32_t> layers;
  for (int32_t i : which) {
    Region& r = R->regions[i];
    for (int32_t b = r.first_id; b < r.first_id + r.n_blocks; ++b) R->free_ids.erase(b);
    r.retired = true;
    for (int32_t l = r.first_layer; l < r.first_layer + r.n_layers; ++l) layers.push_back(l);
    R->reclaimed_bytes -= (uint64_t)r.n_layers * D->sz.S;
    D->donated_bytes -= (uint64_t)r.n_layers * D->sz.S;
  }
  const bool was_cycle = R->regions[region].cycle;
  if (was_cycle)  // the slot holders' storage may hold another cycled layer's weights
    for (int i = 0; i < D->beta; ++i) layers.push_back(D->cycle[i]);
  if (!c->host_only) {
    // The reload runs on the copy stream, ordered after every kernel enqueued so
    // far on the compute stream (the last readers of these bytes as KV, or of
    // the slots) and, by stream order, after in-flight prefetches. Layer l's
    // event gates the first kernel that reads it (mirage_decode_step /
    // mirage_prefill), so a cold start's prefill overlaps the reload layer by
    // layer (T_T * N <= T_Compute of the prefill).
    D->reload_queue.insert(D->reload_queue.end(), layers.begin(), layers.end());
    if (was_cycle)  // the slots are needed now: no deferral
      if (int32_t e = flush_reloads(c, D)) return e;
  }
  for (int32_t l : layers) D->layer_state[l] = RESIDENT;
  if (was_cycle) {
    for (int32_t l : D->cycle) D->cyc_index[l] = -1;
    D->cycle.clear();
    D->beta = 0;
    if (!c->host_only) {
      CK(c, cudaStreamSynchronize(c->xs));
      for (auto e : D->ready_ev) cudaEventDestroy(e);
      for (auto e : D->free_ev) cudaEventDestroy(e);
    }
    D->ready_ev.clear();
    D->free_ev.clear();
    drop_graphs(D);
  }
  return MIRAGE_OK;
}

// Block migration before reversion (reading #29).
int32_t mirage_migrate_region(mirage_ctx* c, int32_t model, int32_t region, int32_t* n_moved) {
  GUARD(c);
  Model* R = get_model(c, model);
  if (n_moved) *n_moved = 0;
  if (!R || region < 0 || region >= (int32_t)R->regions.size())
    return fail(c, MIRAGE_ERR_RANGE, "migrate: model %d region %d", model, region);
  const Region rg = R->regions[region];
  if (rg.retired) return fail(c, MIRAGE_ERR_STATE, "migrate: region %d already reverted", region);
  // the region's ids (a streaming cycle: all of its regions)
  std::vector<char> in_x(R->next_id, 0);
  for (int32_t i = 0; i < (int32_t)R->regions.size(); ++i) {
    const Region& g = R->regions[i];
    const bool take = rg.cycle ? (g.cycle && g.donor == rg.donor && !g.retired) : i == region;
    if (take)
      for (int32_t b = g.first_id; b < g.first_id + g.n_blocks; ++b) in_x[b] = 1;
  }
  std::vector<int32_t> live, outside;
  for (int32_t b = 0; b < R->next_id; ++b)
    if (in_x[b] && !R->free_ids.count(b)) live.push_back(b);
  for (int32_t b : R->free_ids)  // ascending
    if (!in_x[b] && outside.size() < live.size()) outside.push_back(b);
  if (outside.size() < live.size())
    return fail(c, MIRAGE_ERR_NO_BLOCKS, "migrate: %zu live blocks, %zu free outside", live.size(), outside.size());
  std::unordered_map<int32_t, int32_t> ren;
  for (size_t i = 0; i < live.size(); ++i) ren[live[i]] = outside[i];
  if (!c->host_only) {  // stream-ordered after every kernel that wrote the old blocks
    mirage::BlockMoves mv{};
    for (size_t i = 0; i < live.size(); ++i) {
      mv.src[mv.n] = R->bbase_host[live[i]];
      mv.dst[mv.n] = R->bbase_host[outside[i]];
      if (++mv.n == 16 || i + 1 == live.size()) {
        KL(c, mirage::launch_block_copy(mv, R->sz.BB, c->cs));
        mv.n = 0;
      }
    }
  }
  for (auto& kv : R->tables)
    for (int32_t& b : kv.second) {
      auto it = ren.find(b);
      if (it != ren.end()) b = it->second;
    }
  for (size_t i = 0; i < live.size(); ++i) {
    R->free_ids.erase(outside[i]);
    R->free_ids.insert(live[i]);
  }
  if (n_moved) *n_moved = (int32_t)live.size();
  return MIRAGE_OK;
}

int32_t mirage_alloc_blocks(mirage_ctx* c, int32_t model, int64_t seq_id, int32_t n, int32_t* ids_out,
                            int32_t* shortfall_out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || n < 0) return fail(c, MIRAGE_ERR_RANGE, "alloc: model %d n %d", model, n);
  if (shortfall_out) *shortfall_out = 0;
  if ((size_t)n > M->free_ids.size()) {
    if (shortfall_out) *shortfall_out = n - (int32_t)M->free_ids.size();
    return fail(c, MIRAGE_ERR_NO_BLOCKS, "alloc: shortfall %d", n - (int32_t)M->free_ids.size());
  }
  // every check before any state changes: a failed call leaves no table behind
  const auto found = M->tables.find(seq_id);
  const int64_t have = found == M->tables.end() ? 0 : (int64_t)found->second.size();
  if (have + n > c->max_blk)
    return fail(c, MIRAGE_ERR_RANGE, "alloc: table of seq %lld would exceed max_ctx", (long long)seq_id);
  auto& t = M->tables[seq_id];
  for (int i = 0; i < n; ++i) {
    const int32_t id = *M->free_ids.begin();
    M->free_ids.erase(M->free_ids.begin());
    t.push_back(id);
    if (ids_out) ids_out[i] = id;
  }
  M->lens.emplace(seq_id, 0);
  return MIRAGE_OK;
}

int32_t mirage_free_blocks(mirage_ctx* c, int32_t model, int64_t seq_id) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M) return fail(c, MIRAGE_ERR_RANGE, "free: model %d", model);
  auto it = M->tables.find(seq_id);
  if (it == M->tables.end()) return fail(c, MIRAGE_ERR_DOUBLE_FREE, "free: seq %lld", (long long)seq_id);
  for (int32_t id : it->second) M->free_ids.insert(id);
  M->tables.erase(it);
  M->lens.erase(seq_id);
  return MIRAGE_OK;
}

// KV swapping (the Pie-style baseline MIRAGE is compared against, PAPER.md:82-86,
// :212-221, :778-790): bidirectional KV movement over the host link.
int32_t mirage_swap_out(mirage_ctx* c, int32_t model, int64_t seq_id, void* host_dst, uint64_t bytes) {
  GUARD(c);
  if (c->host_only) return fail(c, MIRAGE_ERR_STATE, "host-only context has no device");
  Model* M = get_model(c, model);
  if (!M || !host_dst) return fail(c, MIRAGE_ERR_RANGE, "swap_out: arguments");
  auto it = M->tables.find(seq_id);
  if (it == M->tables.end()) return fail(c, MIRAGE_ERR_RANGE, "swap_out: unknown seq %lld", (long long)seq_id);
  const int32_t len = M->lens.count(seq_id) ? M->lens[seq_id] : 0;
  const int nb = (len + kBlockTokens - 1) / kBlockTokens;
  if ((uint64_t)nb * M->sz.BB > bytes) return fail(c, MIRAGE_ERR_RANGE, "swap_out: host buffer too small");
  char* dst = reinterpret_cast<char*>(host_dst);
  for (int j = 0; j < nb; ++j)  // ordered after every kernel that wrote the KV
    CK(c, cudaMemcpyAsync(dst + (uint64_t)j * M->sz.BB, reinterpret_cast<const void*>(M->bbase_host[it->second[j]]),
                          M->sz.BB, cudaMemcpyDeviceToHost, c->cs));
  // the blocks are free for later work on the same stream (ordered after the copies)
  for (int32_t id : it->second) M->free_ids.insert(id);
  M->tables.erase(it);
  M->lens.erase(seq_id);
  M->swapped[seq_id] = len;
  return MIRAGE_OK;
}

int32_t mirage_swap_in(mirage_ctx* c, int32_t model, int64_t seq_id, const void* host_src) {
  GUARD(c);
  if (c->host_only) return fail(c, MIRAGE_ERR_STATE, "host-only context has no device");
  Model* M = get_model(c, model);
  if (!M || !host_src) return fail(c, MIRAGE_ERR_RANGE, "swap_in: arguments");
  auto sw = M->swapped.find(seq_id);
  if (sw == M->swapped.end() || M->tables.count(seq_id))
    return fail(c, MIRAGE_ERR_STATE, "swap_in: seq %lld is not swapped out", (long long)seq_id);
  const int32_t len = sw->second;
  const int nb = (len + kBlockTokens - 1) / kBlockTokens;
  int32_t short_n = 0;
  if (int32_t e = mirage_alloc_blocks(c, model, seq_id, nb, nullptr, &short_n)) return e;
  const auto& t = M->tables[seq_id];
  const char* src = reinterpret_cast<const char*>(host_src);
  for (int j = 0; j < nb; ++j)
    CK(c, cudaMemcpyAsync(reinterpret_cast<void*>(M->bbase_host[t[j]]), src + (uint64_t)j * M->sz.BB, M->sz.BB,
                          cudaMemcpyHostToDevice, c->cs));
  M->lens[seq_id] = len;
  M->swapped.erase(sw);
  return MIRAGE_OK;
}

int32_t mirage_get_block_table(mirage_ctx* c, int32_t model, int64_t seq_id, int32_t* out, int32_t cap,
                               int32_t* n_out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M) return fail(c, MIRAGE_ERR_RANGE, "table: model %d", model);
  auto it = M->tables.find(seq_id);
  if (it == M->tables.end()) {
    if (n_out) *n_out = 0;
    return fail(c, MIRAGE_ERR_RANGE, "table: unknown seq %lld", (long long)seq_id);
  }
  if (n_out) *n_out = (int32_t)it->second.size();
  if ((int32_t)it->second.size() > cap || (!out && !it->second.empty()))
    return fail(c, MIRAGE_ERR_RANGE, "table: cap %d < %zu", cap, it->second.size());
  std::copy(it->second.begin(), it->second.end(), out);
  return MIRAGE_OK;
}

int32_t mirage_block_location(mirage_ctx* c, int32_t model, int32_t block_id, int32_t* donor,
                              uint64_t* offset) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || block_id < 0 || block_id >= M->next_id)
    return fail(c, MIRAGE_ERR_RANGE, "location: model %d block %d", model, block_id);
  if (donor) *donor = M->loc_donor[block_id];
  if (offset) *offset = M->loc_off[block_id];
  return MIRAGE_OK;
}

int32_t mirage_seq_len(mirage_ctx* c, int32_t model, int64_t seq_id, int32_t* len_out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !len_out) return fail(c, MIRAGE_ERR_RANGE, "seq_len: model %d", model);
  auto it = M->lens.find(seq_id);
  *len_out = it == M->lens.end() ? 0 : it->second;
  return MIRAGE_OK;
}

// ---- decode step -------------------------------------------------------------
int32_t mirage_decode_step(mirage_ctx* c, int32_t model, int32_t B, const int64_t* seq_ids,
                           const int32_t* tokens, const int32_t* positions, void* hidden_out,
                           int32_t* argmax_out) {
  GUARD(c);
  if (c->host_only) return fail(c, MIRAGE_ERR_STATE, "host-only context has no device");
  Model* M = get_model(c, model);
  if (!M) return fail(c, MIRAGE_ERR_RANGE, "step: model %d", model);
  if (B <= 0 || B > c->cfg.max_batch || !seq_ids || !tokens || !positions)
    return fail(c, MIRAGE_ERR_RANGE, "step: batch %d", B);
  const Shape& s = M->shp;
  if (!M->active) return fail(c, MIRAGE_ERR_STATE, "step: model %d inactive", model);
  for (int32_t l = 0; l < s.n; ++l)
    if (M->layer_state[l] == RECLAIMED && M->cyc_index[l] < 0)
      return fail(c, MIRAGE_ERR_STATE, "step: model %d layer %d is reclaimed outside its cycle", model, l);
  // ---- validate (before any enqueue) ----
  // A row is one token. Several rows may belong to one sequence (a prefill or
  // extend chunk): in row order they must take consecutive positions starting at
  // the sequence's cached length. Each row attends causally over positions
  // 0..positions[i] (prefill = the prompt's tokens in parallel).
  std::vector<const std::vector<int32_t>*> rows(B);
  std::unordered_map<int64_t, int32_t> next_pos;  // seq -> expected position of its next row
  std::vector<int32_t> first_row(B);               // row whose address list this row shares
  std::unordered_map<int64_t, int32_t> first_of;
  for (int i = 0; i < B; ++i) {
    auto it = M->tables.find(seq_ids[i]);
    auto np = next_pos.find(seq_ids[i]);
    const int32_t len = np != next_pos.end() ? np->second
                                             : (M->lens.count(seq_ids[i]) ? M->lens[seq_ids[i]] : 0);
    if (positions[i] != len)
      return fail(c, MIRAGE_ERR_STATE, "step: seq %lld position %d != expected %d",
                  (long long)seq_ids[i], positions[i], len);
    next_pos[seq_ids[i]] = len + 1;
    first_row[i] = first_of.emplace(seq_ids[i], i).first->second;
    if (positions[i] + 1 > c->cfg.max_ctx || positions[i] + 1 > s.max_pos)
      return fail(c, MIRAGE_ERR_RANGE, "step: seq %lld exceeds max_ctx", (long long)seq_ids[i]);
    if (tokens[i] < 0 || tokens[i] >= s.V) return fail(c, MIRAGE_ERR_RANGE, "step: token %d", tokens[i]);
    const int need = (positions[i] + 1 + kBlockTokens - 1) / kBlockTokens;
    if (it == M->tables.end() || (int)it->second.size() < need)
      return fail(c, MIRAGE_ERR_NO_BLOCKS, "step: seq %lld needs %d blocks", (long long)seq_ids[i], need);
    rows[i] = &it->second;
  }
  harvest_copy_times(M);
  harvest_step_time(M);
  // ---- pack metadata ----
  char* host;
  if (int32_t e = acquire_stage(c, &host)) return e;
  MetaView hv = meta_view(c, host), dv = meta_view(c, c->meta_dev);
  // one resolved address list per sequence, long enough for its last row
  int n_addr = 0;
  for (int i = 0; i < B; ++i) {
    hv.tokens[i] = tokens[i];
    hv.pos[i] = positions[i];
    hv.len[i] = positions[i] + 1;
    if (first_row[i] != i) {
      hv.seq_off[i] = hv.seq_off[first_row[i]];
      continue;
    }
    hv.seq_off[i] = n_addr;
    const int need = (next_pos[seq_ids[i]] + kBlockTokens - 1) / kBlockTokens;
    for (int j = 0; j < need; ++j) hv.addrs[n_addr + j] = M->bbase_host[(*rows[i])[j]];
    n_addr += need;
  }
  int split_blocks = 1;
  bool multi_row = false;  // a prefill / extend step: some sequence has several rows
  for (int i = 0; i < B && !multi_row; ++i) multi_row = first_row[i] != i;
  const int qp = multi_row ? mirage::attention_prefill_rows(s.H, s.Hk) : 1;
  int32_t attn_mode = 0;
  const int n_units =
      qp > 1 ? build_units_rows(hv.len, hv.seq_off, seq_ids, B, qp, hv.units, c->max_units)
             : build_units(hv.len, hv.seq_off, B, s.Hk, s.H / s.Hk, mirage::attention_grid_ctas(s.H, s.Hk, s.D),
                           mirage::attention_cta_warps(s.Hk), 0, hv.units, c->max_units, &split_blocks, &attn_mode,
                           hv.rfirst);
  if (n_units < 0) return fail(c, MIRAGE_ERR_RANGE, "step: too many attention units");
  hv.hdr[0] = n_units;
  hv.hdr[1] = attn_mode;
  cudaStream_t cs = c->cs;
  const bool timed = !M->step_timed && !multi_row;  // T_Compute = a decode step, not a prefill
  if (timed) CK(c, cudaEventRecord(M->st0, cs));
  size_t meta_bytes = 0;
  if (int32_t e = upload_meta(c, host, n_addr, &meta_bytes)) return e;
  CK(c, cudaEventRecord(c->stage_ev[c->stage_i], cs));
  M->last_meta = meta_bytes;
  if (int32_t e = flush_reloads(c, M)) return e;  // requested reloads start behind this step's upload
  M->last_units = n_units;
  M->last_split = split_blocks;

  const GlobalW gw = global_ptrs(s, M->w_dev + (uint64_t)s.n * M->sz.S);
  const int d = s.d, H = s.H, Hk = s.Hk, D = s.D, qkvN = (H + 2 * Hk) * D;
  const bool opt = s.family == MIRAGE_FAMILY_OPT;
  const long long y_cap = (long long)c->cfg.max_batch * M->y_ld_max;  // floats of the y workspace
  const int m = (int)M->cycle.size();
  const int beta = M->beta;
  // weights of layer l for this step (slot if cycled) and its use index
  std::vector<const char*> wptr(s.n);
  std::vector<int64_t> use_of(s.n, -1);
  uint64_t k = M->uses;
  for (int l = 0; l < s.n; ++l) {
    if (M->cyc_index[l] >= 0) {
      use_of[l] = (int64_t)k;
      const int slot = (int)(k % beta);
      wptr[l] = M->w_dev + (uint64_t)M->cycle[slot] * M->sz.S;
      ++k;
    } else {
      wptr[l] = M->w_dev + (uint64_t)l * M->sz.S;
    }
  }
  // test/experiment hooks (MIRAGE_PREFETCH_DEBUG): 1 = events only, no DMA; 2 = no waits;
  // 3 = no waits + a 20 ms stall before each copy (slow link); 4 = slow link, waits kept
  static const int dbg_nowait = prefetch_debug() == 2 || prefetch_debug() == 3;
  bool reloading = false;
  for (char r : M->reload_pending) reloading |= r != 0;
  bool capturing = false;  // this step's body is being captured into a CUDA graph
  auto gate = [&](int l) -> int32_t {  // wait until layer l's weights are in its slot
    if (reloading && l < s.n && M->reload_pending[l]) {  // an asynchronous reload (mirage_unremap)
      if (!dbg_nowait) CK(c, cudaStreamWaitEvent(cs, M->reload_ev[l], 0));
      M->reload_pending[l] = 0;
    }
    // (inside a graph capture, a copy issued by an earlier step is covered by the
    // pre-capture waits and, on replays, by the previous graph's joined copy branch)
    const bool prior_copy = use_of[l] - beta < (int64_t)M->uses;
    if (!dbg_nowait && l < s.n && use_of[l] >= beta && use_of[l] >= 0 && !(capturing && prior_copy)) {
      if ((c->cfg.flags & MIRAGE_FLAG_TIME_ATTN) && !capturing) {  // measured stall of this handoff
        Model::AttnTiming t{pool_event(M), pool_event(M), 0};
        CK(c, cudaEventRecord(t.t0, cs));
        CK(c, cudaStreamWaitEvent(cs, M->ready_ev[use_of[l] % beta], 0));
        CK(c, cudaEventRecord(t.t1, cs));
        M->stall_pending.push_back(t);
      } else {
        CK(c, cudaStreamWaitEvent(cs, (capturing ? M->cap_ready_ev : M->ready_ev)[use_of[l] % beta], 0));
      }
    }
    if (M->slot_tag && l < s.n && use_of[l] >= 0)  // SLOT_TAGS: the slot must hold layer l now
      KL(c, mirage::launch_tag_check(M->slot_tag + use_of[l] % beta, M->host_tags[l], M->tag_err, cs));
    return MIRAGE_OK;
  };
  auto release = [&](int l) -> int32_t {  // layer l done reading its slot; prefetch use+beta
    if (use_of[l] < 0) return MIRAGE_OK;
    const uint64_t u = (uint64_t)use_of[l];
    const int slot = (int)(u % beta);
    M->slot_log.insert(M->slot_log.end(),
                       {(int64_t)u, M->cyc_steps, l, slot, (int64_t)(u >= (uint64_t)beta)});
    cudaEvent_t fev = (capturing ? M->cap_free_ev : M->free_ev)[slot];
    CK(c, cudaEventRecord(fev, cs));
    const uint64_t nu = u + beta;
    const int nl = M->cycle[nu % m];
    CK(c, cudaStreamWaitEvent(c->xs, fev, 0));  // (in a capture: forks the copy branch)
    CopyTiming t{nullptr, nullptr, M->sz.S};
    if (!capturing) {  // copy timing events are per step: eager steps only
      t = CopyTiming{pool_event(M), pool_event(M), M->sz.S};
      if (!t.t0 || !t.t1) return fail(c, MIRAGE_ERR_CUDA, "release: event pool");
      CK(c, cudaEventRecord(t.t0, c->xs));
    }
    const int dbg_mode = prefetch_debug();
    if (dbg_mode == 3 || dbg_mode == 4) KL(c, mirage::launch_spin(20000000ull, c->xs));  // a slow link
    if (dbg_mode != 1) {  // experiment hook: 1 = events only, no DMA
      void* dst = M->w_dev + (uint64_t)M->cycle[slot] * M->sz.S;
      const void* src = M->host + (uint64_t)nl * M->sz.S;
      CK(c, cudaMemcpyAsync(dst, src, M->sz.S, cudaMemcpyDefault, c->xs));
    }
    if (M->slot_tag)  // same stream, after the weights: a correct tag proves they landed
      CK(c, cudaMemcpyAsync(M->slot_tag + slot, M->host_tags + nl, 4, cudaMemcpyHostToDevice, c->xs));
    if (!capturing) {
      CK(c, cudaEventRecord(t.t1, c->xs));
      M->pending.push_back(t);
    } else {
      M->graph_copies += 1;
    }
    CK(c, cudaEventRecord((capturing ? M->cap_ready_ev : M->ready_ev)[slot], c->xs));
    return MIRAGE_OK;
  };

  // CUDA graph of the step body (embed ... argmax): models without a streaming
  // cycle, one graph per batch size, captured on the second step of that size
  // (the first runs eagerly so cuBLASLt plans/autotuning happen outside capture)
  // With MIRAGE_FLAG_TIME_ATTN too, the graphs are separate timed variants: an event
  // node before and after each attention launch (the measurement pass of bench.py)
  const bool time_attn = c->cfg.flags & MIRAGE_FLAG_TIME_ATTN;
  uint64_t attn_bytes = 0;
  for (int i = 0; i < B; ++i) attn_bytes += (uint64_t)hv.len[i] * 2 * Hk * D * 2;
  const bool graphable = (c->cfg.flags & MIRAGE_FLAG_CUDA_GRAPHS) && !reloading && qp == 1 &&
                         !M->tp_ready && !dbg_nowait && prefetch_debug() == 0 && !M->slot_tag;
  if (c->tp > 1 && !c->nccl && !M->tp_ready)
    return fail(c, MIRAGE_ERR_STATE, "step: tensor parallel model without a collective (tp_import first)");
  bool body_done = false;
  int64_t l0 = 0;
  const int64_t par_period = m ? (int64_t)std::lcm(m, beta) : 1;
  const int64_t gkey = ((int64_t)B * 64 + (m ? (int64_t)(M->uses % par_period) : 0)) * 2 + (time_attn ? 1 : 0);
  std::vector<cudaEvent_t> cap_tev;  // a timed capture's attention event pairs
  if (graphable) {
    auto g = M->graphs.find(gkey);
    if (g != M->graphs.end() || M->graph_seen.count(gkey)) {
      // a cycling model: copies issued by earlier (eager) steps must land before the graph
      for (int sl = 0; sl < beta; ++sl) CK(c, cudaStreamWaitEvent(cs, M->ready_ev[sl], 0));
    }
    if (g != M->graphs.end()) {
      if (time_attn) harvest_graph_attn(M, true);  // its events are about to be re-recorded
      CK(c, cudaGraphLaunch(g->second.exec, cs));
      if (time_attn) {
        M->tpend = &g->second;
        M->tpend_bytes = attn_bytes;
      }
      c->launches += g->second.kernels;
      body_done = true;
      // host bookkeeping of the replayed step: the slot log and the copy count
      for (int l = 0; l < s.n; ++l)
        if (use_of[l] >= 0) {
          const uint64_t u = (uint64_t)use_of[l];
          M->slot_log.insert(M->slot_log.end(),
                             {(int64_t)u, M->cyc_steps, l, (int64_t)(u % beta), (int64_t)(u >= (uint64_t)beta)});
          M->graph_copies += 1;
        }
    } else if (M->graph_seen.count(gkey)) {
      while ((int)M->cap_ready_ev.size() < beta) {
        cudaEvent_t a, b;
        CK(c, cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CK(c, cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        M->cap_ready_ev.push_back(a);
        M->cap_free_ev.push_back(b);
      }
      if (time_attn) {
        harvest_graph_attn(M, true);
        cap_tev.resize(2 * (size_t)s.n, nullptr);
        for (auto& e : cap_tev) CK(c, cudaEventCreate(&e));
      }
      CK(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      capturing = true;
      l0 = c->launches;
    } else {
      M->graph_seen.insert(gkey);
    }
  }
  if (!body_done) {
  // embedding + layer 0's first norm
  if (int32_t e = gate(0)) return e;
  {
    const LayerW w0 = layer_ptrs(s, wptr[0]);
    KL(c, mirage::launch_embed_norm(s.family, B, d, dv.tokens, dv.pos, gw.embed, gw.pos_embed, w0.n1_g,
                                   w0.n1_b, s.eps, M->h, M->x, cs));
  }
  mirage::AttnParams ap{};
  ap.q = M->q;
  ap.addrs = dv.addrs;
  ap.units = dv.units;
  ap.hdr = dv.hdr;
  ap.rfirst = dv.rfirst;
  ap.full_grid = attn_mode == 1;
  ap.n_units = n_units;
  ap.n_units_dev = nullptr;
  if (capturing) {  // replays keep the full persistent grid; the unit count comes from the metadata
    ap.n_units = c->max_units;
    ap.n_units_dev = dv.hdr;
  }
  ap.H = H;
  ap.H_kv = Hk;
  ap.D = D;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
  ap.partial = M->partial;
  ap.tickets = M->tickets;
  ap.sched = M->tickets + (size_t)c->cfg.max_batch * Hk;
  ap.out = M->x;  // bf16 [B][H*D]: the O-projection input
  ap.out_fp32 = 0;
  ap.qp = qp;
  ap.pdl = use_pdl();  // programmatic dependency on qkv_post (which precedes it in the stream)
  ap.kv_evict_first = kv_evict_first();
  ap.prod_lanes = attn_prod_lanes();
  if (time_attn && !capturing) {  // (no event queries inside a stream capture)
    harvest_attn_times(M);
    harvest_stall_times(M);
  }
  for (int l = 0; l < s.n; ++l) {
    const LayerW w = layer_ptrs(s, wptr[l]);
    const uint64_t layer_off = (uint64_t)l * Hk * 2 * kBlockTokens * D * 2;
    if (int32_t e = gemm_lt(c, B, qkvN, d, w.w_qkv, M->x, M->y, 0, nullptr, 0)) return e;
    KL(c, mirage::launch_qkv_post(s.family, B, H, Hk, D, M->y, opt ? w.b_qkv : nullptr, dv.pos,
                                 dv.seq_off, dv.addrs, layer_off, s.theta, ap.scale_log2, M->q, cs, use_pdl()));
    ap.layer_off = layer_off;
    if (time_attn && capturing) {  // event record nodes of the timed graph (external: they
      // record at replay time; a plain record inside a capture is only a dependency marker)
      CK(c, cudaEventRecordWithFlags(cap_tev[2 * l], cs, cudaEventRecordExternal));
      KL(c, mirage::launch_paged_attention(ap, cs));
      CK(c, cudaEventRecordWithFlags(cap_tev[2 * l + 1], cs, cudaEventRecordExternal));
    } else if (time_attn) {
      Model::AttnTiming at{pool_event(M), pool_event(M), attn_bytes};
      CK(c, cudaEventRecord(at.t0, cs));
      KL(c, mirage::launch_paged_attention(ap, cs));
      CK(c, cudaEventRecord(at.t1, cs));
      M->attn_pending.push_back(at);
    } else {
      KL(c, mirage::launch_paged_attention(ap, cs));
    }
    if (M->tp_ready && M->tp_push) {  // NEXT-4: the O-proj GEMM pushes its partial to every rank
      const uint64_t ep = ++M->tp_epoch;
      if (int32_t e = tp_push_gemm(c, M, B, d, H * D, w.w_o, M->x, ep)) return e;
      KL(c, mirage::launch_tp_push_residual_norm(s.family, B, d, M->local_slots_dev + (ep & 1) * c->tp, c->tp,
                                                reinterpret_cast<unsigned long long*>(M->xfer + 8), M->push_expect,
                                                M->tp_err, opt ? w.b_o : nullptr, w.n2_g, opt ? w.n2_b : nullptr,
                                                s.eps, M->h, M->x, cs));
    } else if (M->tp_ready) {  // a10 over peer memory: partial O-proj -> fused all-reduce + residual + norm
      const uint64_t ep = ++M->tp_epoch;
      float* part = reinterpret_cast<float*>(M->xfer + kAlign + (ep & 1) * M->xfer_part);
      if (int32_t e = gemm_lt(c, B, d, H * D, w.w_o, M->x, part, 0, nullptr, 0)) return e;
      KL(c, mirage::launch_tp_residual_norm(s.family, B, d, M->parts_dev + (ep & 1) * c->tp, c->tp, c->tp_rank,
                                           M->flags_dev, ep, M->tp_err, opt ? w.b_o : nullptr, w.n2_g,
                                           opt ? w.n2_b : nullptr, s.eps, M->h, M->x, cs));
    } else {
      int ns_o = 1;
      if (c->nccl) {
        if (int32_t e = gemm_lt(c, B, d, H * D, w.w_o, M->x, M->y, 0, nullptr, 0)) return e;
        // a10: sum the heads' partial O-projections over the TP ranks
        CKN(c, ncclAllReduce(M->y, M->y, (size_t)B * d, ncclFloat32, ncclSum, c->nccl, cs));
      } else if (int32_t e = gemm_rowpar(c, B, d, H * D, w.w_o, M->x, M->y, y_cap, &ns_o)) {
        return e;
      }
      KL(c, mirage::launch_residual_norm(s.family, B, d, M->y, d, opt ? w.b_o : nullptr, w.n2_g,
                                        opt ? w.n2_b : nullptr, s.eps, M->h, M->x, cs, ns_o, (long long)B * d,
                                        use_pdl()));
    }
    if (opt) {
      // FC1 + bias + ReLU fused in the GEMM epilogue, bf16 out (one rounding, as before)
      if (int32_t e = gemm_lt(c, B, s.f, d, w.w_1, M->x, M->f, 1, w.b_1, 2)) return e;
    } else {
      if (int32_t e = gemm_lt(c, B, 2 * s.f, d, w.w_1, M->x, M->y, 0, nullptr, 0)) return e;
      KL(c, mirage::launch_act(s.family, B, s.f, M->y, nullptr, M->f, cs));
    }
    uint64_t ep2 = 0;
    int ns_2 = 1;
    if (M->tp_ready && M->tp_push) {
      ep2 = ++M->tp_epoch;
      if (int32_t e = tp_push_gemm(c, M, B, d, s.f, w.w_2, M->f, ep2)) return e;
    } else if (M->tp_ready) {
      ep2 = ++M->tp_epoch;
      float* part = reinterpret_cast<float*>(M->xfer + kAlign + (ep2 & 1) * M->xfer_part);
      if (int32_t e = gemm_lt(c, B, d, s.f, w.w_2, M->f, part, 0, nullptr, 0)) return e;
    } else if (c->nccl) {
      if (int32_t e = gemm_lt(c, B, d, s.f, w.w_2, M->f, M->y, 0, nullptr, 0)) return e;
    } else if (int32_t e = gemm_rowpar(c, B, d, s.f, w.w_2, M->f, M->y, y_cap, &ns_2)) {
      return e;
    }
    if (c->nccl)  // a10: sum the FFN shards' partial down-projections
      CKN(c, ncclAllReduce(M->y, M->y, (size_t)B * d, ncclFloat32, ncclSum, c->nccl, cs));
    // residual of layer l (+ the next norm): plain, or fused with the peer all-reduce
    auto residual = [&](const bf16* bias2, const bf16* g2, const bf16* b2) -> int32_t {
      if (M->tp_ready && M->tp_push) {
        KL(c, mirage::launch_tp_push_residual_norm(s.family, B, d, M->local_slots_dev + (ep2 & 1) * c->tp, c->tp,
                                                  reinterpret_cast<unsigned long long*>(M->xfer + 8),
                                                  M->push_expect, M->tp_err, bias2, g2, b2, s.eps, M->h, M->x, cs));
      } else if (M->tp_ready) {
        KL(c, mirage::launch_tp_residual_norm(s.family, B, d, M->parts_dev + (ep2 & 1) * c->tp, c->tp, c->tp_rank,
                                             M->flags_dev, ep2, M->tp_err, bias2, g2, b2, s.eps, M->h, M->x, cs));
      } else {
        KL(c, mirage::launch_residual_norm(s.family, B, d, M->y, d, bias2, g2, b2, s.eps, M->h, M->x, cs, ns_2,
                                          (long long)B * d, use_pdl()));
      }
      return MIRAGE_OK;
    };
    // residual, then the next layer's first norm (or the final norm)
    const bool last = l + 1 == s.n;
    const bf16* ng = last ? gw.nf_g : nullptr;
    const bf16* nb = last ? gw.nf_b : nullptr;
    const bool split_gate = !last && use_of[l] >= 0 && use_of[l + 1] >= 0 && beta == 1;
    if (split_gate) {
      // l and l+1 share the single slot: finish l, hand the slot over, then norm
      if (int32_t e = residual(opt ? w.b_2 : nullptr, nullptr, nullptr)) return e;
      if (int32_t e = release(l)) return e;
      if (int32_t e = gate(l + 1)) return e;
      const LayerW wn = layer_ptrs(s, wptr[l + 1]);
      KL(c, mirage::launch_residual_norm(s.family, B, d, nullptr, d, nullptr, wn.n1_g,
                                        opt ? wn.n1_b : nullptr, s.eps, M->h, M->x, cs));
    } else {
      if (!last) {
        if (int32_t e = gate(l + 1)) return e;
        const LayerW wn = layer_ptrs(s, wptr[l + 1]);
        ng = wn.n1_g;
        nb = opt ? wn.n1_b : nullptr;
      }
      if (int32_t e = residual(opt ? w.b_2 : nullptr, ng, opt ? nb : nullptr)) return e;
      if (int32_t e = release(l)) return e;
    }
  }
  // LM head + argmax
  if (int32_t e = gemm_lt(c, B, s.V, d, gw.lm_head, M->x, M->y, 0, nullptr, 0)) return e;
  KL(c, mirage::launch_argmax(B, s.V, M->y, M->argmax, cs));
  if (capturing) {
    if (m) {  // rejoin the copy branch: the graph ends when its DMAs have landed
      if (!M->join_ev) CK(c, cudaEventCreateWithFlags(&M->join_ev, cudaEventDisableTiming));
      CK(c, cudaEventRecord(M->join_ev, c->xs));
      CK(c, cudaStreamWaitEvent(cs, M->join_ev, 0));
    }
    cudaGraph_t graph;
    CK(c, cudaStreamEndCapture(cs, &graph));
    cudaGraphExec_t exec;
    CK(c, cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    M->graphs[gkey] = Model::Graph{exec, c->launches - l0, cap_tev};
    CK(c, cudaGraphLaunch(exec, cs));
    if (time_attn) {
      M->tpend = &M->graphs[gkey];
      M->tpend_bytes = attn_bytes;
    }
  }
  }  // !body_done
  if (hidden_out)
    CK(c, cudaMemcpyAsync(hidden_out, M->x, (size_t)B * d * 2, cudaMemcpyDeviceToDevice, cs));
  if (argmax_out) CK(c, cudaMemcpyAsync(argmax_out, M->argmax, (size_t)B * 4, cudaMemcpyDeviceToHost, cs));
  if (timed) {
    CK(c, cudaEventRecord(M->st1, cs));
    M->step_timed = true;
  }
  // commit host state
  M->uses = k;
  if (m) M->cyc_steps++;
  M->steps++;
  for (int i = 0; i < B; ++i) M->lens[seq_ids[i]] = positions[i] + 1;
  return MIRAGE_OK;
}

// Prefill / extend (§2.1; the cold-start prefill of P:395-397).
// The prompts' tokens are laid out as rows of decode steps (one row per token,
// rows of one sequence at consecutive positions) and run in chunks of at most
// max_batch rows. Each chunk is one layer-major pass, so a chunk's layer l waits
// only for layer l's weights (an asynchronous reload, mirage_unremap, overlaps
// with the chunk's earlier layers).
int32_t mirage_prefill(mirage_ctx* c, int32_t model, int32_t n_seqs, const int64_t* seq_ids,
                       const int32_t* prompt_lens, const int32_t* tokens, int32_t* last_argmax_out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || n_seqs <= 0 || !seq_ids || !prompt_lens || !tokens)
    return fail(c, MIRAGE_ERR_RANGE, "prefill: arguments");
  std::vector<int64_t> rs;
  std::vector<int32_t> rt, rp, last_row(n_seqs);
  int64_t tok = 0;
  for (int i = 0; i < n_seqs; ++i) {
    if (prompt_lens[i] <= 0) return fail(c, MIRAGE_ERR_RANGE, "prefill: prompt %d has length %d", i, prompt_lens[i]);
    for (int j = 0; j < i; ++j)
      if (seq_ids[j] == seq_ids[i]) return fail(c, MIRAGE_ERR_RANGE, "prefill: duplicate seq");
    const int32_t p0 = M->lens.count(seq_ids[i]) ? M->lens[seq_ids[i]] : 0;
    auto it = M->tables.find(seq_ids[i]);  // all blocks checked before the first chunk runs
    const int need = (p0 + prompt_lens[i] + kBlockTokens - 1) / kBlockTokens;
    if (it == M->tables.end() || (int)it->second.size() < need)
      return fail(c, MIRAGE_ERR_NO_BLOCKS, "prefill: seq %lld needs %d blocks", (long long)seq_ids[i], need);
    if (p0 + prompt_lens[i] > c->cfg.max_ctx || p0 + prompt_lens[i] > M->shp.max_pos)
      return fail(c, MIRAGE_ERR_RANGE, "prefill: seq %lld exceeds max_ctx", (long long)seq_ids[i]);
    for (int32_t t = 0; t < prompt_lens[i]; ++t) {
      rs.push_back(seq_ids[i]);
      rt.push_back(tokens[tok++]);
      rp.push_back(p0 + t);
    }
    last_row[i] = (int32_t)rs.size() - 1;
  }
  const int64_t R = (int64_t)rs.size();
  std::vector<int32_t> am(last_argmax_out ? R : 0);
  for (int64_t r0 = 0; r0 < R; r0 += c->cfg.max_batch) {
    const int32_t n = (int32_t)std::min<int64_t>(c->cfg.max_batch, R - r0);
    if (int32_t e = mirage_decode_step(c, model, n, rs.data() + r0, rt.data() + r0, rp.data() + r0, nullptr,
                                       last_argmax_out ? am.data() + r0 : nullptr))
      return e;
  }
  if (last_argmax_out) {
    CK(c, cudaStreamSynchronize(c->cs));
    for (int i = 0; i < n_seqs; ++i) last_argmax_out[i] = am[last_row[i]];
  }
  return MIRAGE_OK;
}

int32_t mirage_attn_only(mirage_ctx* c, int32_t model, int32_t layer, int32_t B, const int64_t* seq_ids,
                         const float* q_dev, void* out_dev, int32_t out_fp32,
                         int32_t split_tokens_override) {
  GUARD(c);
  if (c->host_only) return fail(c, MIRAGE_ERR_STATE, "host-only context has no device");
  Model* M = get_model(c, model);
  if (!M || layer < 0 || layer >= M->shp.n || B <= 0 || B > c->cfg.max_batch || !seq_ids || !q_dev ||
      !out_dev || split_tokens_override < -1 || (split_tokens_override > 0 && split_tokens_override % kBlockTokens))
    return fail(c, MIRAGE_ERR_RANGE, "attn_only: arguments");
  char* host;
  if (int32_t e = acquire_stage(c, &host)) return e;
  MetaView hv = meta_view(c, host), dv = meta_view(c, c->meta_dev);
  int n_addr = 0;
  for (int i = 0; i < B; ++i) {
    auto it = M->tables.find(seq_ids[i]);
    const int32_t len = M->lens.count(seq_ids[i]) ? M->lens[seq_ids[i]] : 0;
    if (it == M->tables.end() || len <= 0)
      return fail(c, MIRAGE_ERR_STATE, "attn_only: seq %lld has no tokens", (long long)seq_ids[i]);
    hv.len[i] = len;
    hv.seq_off[i] = n_addr;
    const int nb = (len + kBlockTokens - 1) / kBlockTokens;
    for (int j = 0; j < nb; ++j) hv.addrs[n_addr + j] = M->bbase_host[it->second[j]];
    n_addr += nb;
  }
  int split_blocks = 1;
  const int n_units = build_units(hv.len, hv.seq_off, B, M->shp.Hk, M->shp.H / M->shp.Hk,
                                  mirage::attention_grid_ctas(M->shp.H, M->shp.Hk, M->shp.D),
                                  mirage::attention_cta_warps(M->shp.Hk),
                                  split_tokens_override < 0 ? -1 : split_tokens_override / kBlockTokens,
                                  hv.units, c->max_units, &split_blocks, &hv.hdr[1], hv.rfirst);
  if (n_units < 0) return fail(c, MIRAGE_ERR_RANGE, "attn_only: too many units for the split override");
  hv.hdr[0] = n_units;
    if (int32_t e = upload_meta(c, host, n_addr)) return e;
  CK(c, cudaEventRecord(c->stage_ev[c->stage_i], c->cs));
  M->last_units = n_units;
  M->last_split = split_blocks;
  const Shape& s = M->shp;
  mirage::AttnParams ap{};
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)M->shp.D));
  KL(c, mirage::launch_q_split((int64_t)B * M->shp.H * M->shp.D, M->shp.D, q_dev, ap.scale_log2, M->q, c->cs));
  ap.q = M->q;
  ap.addrs = dv.addrs;
  ap.layer_off = (uint64_t)layer * s.Hk * 2 * kBlockTokens * s.D * 2;
  ap.units = dv.units;
  ap.hdr = dv.hdr;
  ap.rfirst = dv.rfirst;
  ap.full_grid = hv.hdr[1] == 1;
  ap.n_units = n_units;
  ap.H = s.H;
  ap.H_kv = s.Hk;
  ap.D = s.D;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)s.D));
  ap.partial = M->partial;
  ap.tickets = M->tickets;
  ap.sched = M->tickets + (size_t)c->cfg.max_batch * s.Hk;
  ap.out = out_dev;
  ap.out_fp32 = out_fp32;
  ap.pdl = use_pdl();  // programmatic dependency on q_split (or the previous repeat)
  ap.kv_evict_first = kv_evict_first();
  ap.prod_lanes = attn_prod_lanes();
  if (c->attn_trace) {
    const int ctas = mirage::attention_grid_ctas(s.H, s.Hk, s.D);
    c->attn_trace_ctas = std::min(mirage_ctx::kTraceCtas, std::min(ctas, n_units * s.Hk));
    CK(c, cudaMemsetAsync(c->attn_trace, 0, (size_t)mirage_ctx::kTraceCtas * 16 * 8, c->cs));
    ap.trace = c->attn_trace;
  }
  if (c->cfg.flags & MIRAGE_FLAG_TIME_ATTN) {  // kernel-only time, excluding the metadata upload
    harvest_attn_times(M);
    uint64_t nbytes = 0;
    for (int i = 0; i < B; ++i) nbytes += (uint64_t)hv.len[i] * 2 * s.Hk * s.D * 2;
    // MIRAGE_ATTN_REPEAT=R (bench hook): R back-to-back launches over layers
    // layer, layer+1, ... (mod n: every launch reads other HBM) inside one timed
    // pair of events, reported as R launches (per-launch time = total / R)
    static const int reps = getenv("MIRAGE_ATTN_REPEAT") ? std::max(1, atoi(getenv("MIRAGE_ATTN_REPEAT"))) : 1;
    Model::AttnTiming at{pool_event(M), pool_event(M), nbytes * reps, reps};
    CK(c, cudaEventRecord(at.t0, c->cs));
    for (int r = 0; r < reps; ++r) {
      ap.layer_off = (uint64_t)((layer + r) % s.n) * s.Hk * 2 * kBlockTokens * s.D * 2;
      KL(c, mirage::launch_paged_attention(ap, c->cs));
    }
    CK(c, cudaEventRecord(at.t1, c->cs));
    M->attn_pending.push_back(at);
    return MIRAGE_OK;
  }
  KL(c, mirage::launch_paged_attention(ap, c->cs));
  return MIRAGE_OK;
}

static int32_t kv_hook_prepare(mirage_ctx* c, Model* M, int64_t seq_id, int32_t n, int32_t* p0) {
  auto it = M->tables.find(seq_id);
  const int32_t len = M->lens.count(seq_id) ? M->lens[seq_id] : 0;
  const int need = (len + n + kBlockTokens - 1) / kBlockTokens;
  if (it == M->tables.end() || (int)it->second.size() < need)
    return fail(c, MIRAGE_ERR_NO_BLOCKS, "kv: seq %lld needs %d blocks", (long long)seq_id, need);
  if (len + n > c->cfg.max_ctx) return fail(c, MIRAGE_ERR_RANGE, "kv: exceeds max_ctx");
  char* host;
  if (int32_t e = acquire_stage(c, &host)) return e;
  MetaView hv = meta_view(c, host);
  std::copy(it->second.begin(), it->second.begin() + need, hv.tables);
  const size_t head = reinterpret_cast<char*>(hv.tables) - host;
  CK(c, cudaMemcpyAsync(c->meta_dev + head, host + head, (size_t)need * 4, cudaMemcpyHostToDevice, c->cs));
  CK(c, cudaEventRecord(c->stage_ev[c->stage_i], c->cs));
  *p0 = len;
  return MIRAGE_OK;
}

int32_t mirage_fill_kv(mirage_ctx* c, int32_t model, int64_t seq_id, int32_t n, uint64_t seed) {
  GUARD(c);
  if (c->host_only) return fail(c, MIRAGE_ERR_STATE, "host-only context has no device");
  Model* M = get_model(c, model);
  if (!M || n < 0) return fail(c, MIRAGE_ERR_RANGE, "fill_kv: arguments");
  int32_t p0 = 0;
  if (int32_t e = kv_hook_prepare(c, M, seq_id, n, &p0)) return e;
  MetaView dv = meta_view(c, c->meta_dev);
  const Shape& s = M->shp;
  KL(c, mirage::launch_fill_kv(seed, seq_id, s.n, s.Hk, s.D, p0, n, dv.tables, M->bbase_dev, c->cs));
  M->lens[seq_id] = p0 + n;
  return MIRAGE_OK;
}

int32_t mirage_write_kv(mirage_ctx* c, int32_t model, int64_t seq_id, int32_t n, const void* host_kv) {
  GUARD(c);
  if (c->host_only) return fail(c, MIRAGE_ERR_STATE, "host-only context has no device");
  Model* M = get_model(c, model);
  if (!M || n < 0 || (!host_kv && n)) return fail(c, MIRAGE_ERR_RANGE, "write_kv: arguments");
  int32_t p0 = 0;
  if (int32_t e = kv_hook_prepare(c, M, seq_id, n, &p0)) return e;
  const Shape& s = M->shp;
  const size_t bytes = (size_t)s.n * s.Hk * 2 * n * s.D * 2;
  void* tmp = nullptr;
  if (bytes) {
    CK(c, cudaMalloc(&tmp, bytes));
    CK(c, cudaMemcpyAsync(tmp, host_kv, bytes, cudaMemcpyHostToDevice, c->cs));
    MetaView dv = meta_view(c, c->meta_dev);
    ++c->launches;
    cudaError_t e = mirage::launch_write_kv(s.n, s.Hk, s.D, p0, n, reinterpret_cast<const bf16*>(tmp),
                                            dv.tables, M->bbase_dev, c->cs);
    cudaError_t e2 = cudaStreamSynchronize(c->cs);
    cudaFree(tmp);
    CK(c, e);
    CK(c, e2);
  }
  M->lens[seq_id] = p0 + n;
  return MIRAGE_OK;
}

int32_t mirage_query(mirage_ctx* c, int32_t model, mirage_stats* o) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M || !o) return fail(c, MIRAGE_ERR_RANGE, "query: model %d", model);
  if (!c->host_only) {
    harvest_copy_times(M);
    harvest_step_time(M);
    harvest_attn_times(M);
    harvest_stall_times(M);
  }
  std::memset(o, 0, sizeof *o);
  o->native_blocks = M->n_native;
  o->total_blocks = M->next_id;
  o->free_blocks = (int64_t)M->free_ids.size();
  o->layer_bytes = M->sz.S;
  o->block_bytes = M->sz.BB;
  o->reclaimed_bytes = M->reclaimed_bytes;
  o->donated_bytes = M->donated_bytes;
  o->m = (int32_t)M->cycle.size();
  o->beta = M->beta;
  o->active = M->active;
  o->n_seqs = (int32_t)M->tables.size();
  for (size_t i = 0; i < M->cycle.size() && i < MIRAGE_MAX_CYCLE; ++i) o->cycle[i] = M->cycle[i];
  o->uses = M->uses;
  o->h2d_copies = M->h2d_copies;
  o->h2d_bytes = M->h2d_bytes;
  o->h2d_ms = M->h2d_ms;
  o->last_step_ms = M->last_step_ms;
  o->steps = M->steps;
  o->attn_launches = M->attn_launches;
  o->stall_waits = M->stall_waits;
  o->stall_ms = M->stall_ms;
  o->attn_ms = M->attn_ms;
  o->attn_bytes = M->attn_bytes;
  o->last_meta_h2d_bytes = M->last_meta;
  if (M->tp_err) {
    uint32_t e = 0;
    CK(c, cudaMemcpy(&e, M->tp_err, 4, cudaMemcpyDeviceToHost));
    o->tp_peer_timeouts = e;
  }
  if (M->tag_err) {
    uint32_t e[2] = {0, 0};
    CK(c, cudaMemcpy(e, M->tag_err, 8, cudaMemcpyDeviceToHost));
    o->slot_tag_errors = e[0];
  }
  o->last_attn_units = M->last_units;
  o->last_split_blocks = M->last_split;
  return MIRAGE_OK;
}

int32_t mirage_slot_log(mirage_ctx* c, int32_t model, int64_t* out, int32_t cap, int32_t* n_out) {
  GUARD(c);
  Model* M = get_model(c, model);
  if (!M) return fail(c, MIRAGE_ERR_RANGE, "slot_log: model %d", model);
  const int32_t n = (int32_t)(M->slot_log.size() / 5);
  if (n_out) *n_out = n;
  if (n > cap || (!out && n)) return fail(c, MIRAGE_ERR_RANGE, "slot_log: cap %d < %d", cap, n);
  std::copy(M->slot_log.begin(), M->slot_log.end(), out);
  return MIRAGE_OK;
}

int32_t mirage_sync(mirage_ctx* c) {
  GUARD(c);
  if (c->host_only) return MIRAGE_OK;
  for (Model* M : c->models)
    if (M)
      if (int32_t e = flush_reloads(c, M)) return e;
  CK(c, cudaStreamSynchronize(c->cs));
  CK(c, cudaStreamSynchronize(c->xs));
  CK(c, cudaGetLastError());
  return MIRAGE_OK;
}

}  // extern "C"
