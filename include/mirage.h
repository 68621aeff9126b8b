/*
 * mirage.h — C-ABI of the B200-native MIRAGE decode-step hot path
 * (arXiv 2507.11507, "MIRAGE: ... Dynamic Remapping Engine", PAPER.md in the
 * reference tree; SURVEY.md §8(b) is the interface contract).
 *
 * What the library does (PAPER.md:297-329 §4, :552-564 §6):
 *   - parameter bytes of chosen layers (or of an inactive tenant's whole model)
 *     are reclaimed as paged KV-cache blocks       (mirage_remap_layers)
 *   - per-sequence block tables over one id space that spans the native pool
 *     and the reclaimed regions                     (mirage_alloc/free_blocks)
 *   - a decode step whose paged-attention kernel reads through that table and
 *     whose cycled layers' weights are re-streamed one-way from pinned host
 *     memory, one layer ahead of use, gated by events (mirage_decode_step)
 *
 * Conventions (all functions):
 *   - extern "C", fixed-width types, no C++ or torch types.
 *   - Every call returns int32_t status: MIRAGE_OK (0) or a negative code.
 *     Nothing throws across the ABI. mirage_last_error() gives the message.
 *   - One mirage_ctx per GPU per process; a ctx is NOT thread-safe.
 *   - Device work is enqueued on the caller's compute stream and the call
 *     returns before it finishes. Host metadata (allocator, tables, remap sets,
 *     slot log) is updated synchronously and deterministically at call time.
 *   - Ownership: the caller owns and must keep alive, for the ctx's lifetime,
 *     the device arena, every host weight blob and the compute stream. The
 *     library owns its metadata, events, the copy stream (unless supplied), the
 *     cuBLAS handle, pinned staging buffers and everything it carves from the
 *     arena.
 *   - Sticky failure: a CUDA error puts the ctx in a failed state; every later
 *     call returns MIRAGE_ERR_CUDA until mirage_destroy.
 *   - There is no CPU fallback: every step of the decode path runs in this
 *     library's sm_100a kernels (GEMMs via cuBLAS).
 */
#ifndef MIRAGE_H_
#define MIRAGE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (SPEC.md error vocabulary) ------------ */
#define MIRAGE_OK 0
#define MIRAGE_ERR_CONFIG -1      /* bad configuration (SPEC ConfigError)              */
#define MIRAGE_ERR_CAPACITY -2    /* arena too small (SPEC CapacityError)              */
#define MIRAGE_ERR_RANGE -3       /* argument out of range (SPEC RangeError)           */
#define MIRAGE_ERR_STATE -4       /* illegal in current state (SPEC StateError)        */
#define MIRAGE_ERR_NO_BLOCKS -5   /* not enough free blocks; shortfall is data         */
#define MIRAGE_ERR_DOUBLE_FREE -6 /* free of an unknown / already freed sequence       */
#define MIRAGE_ERR_INFEASIBLE -7  /* no zero-stall plan (SPEC InfeasibleAlpha)         */
#define MIRAGE_ERR_PRESSURE -8    /* reserved: unremap with live blocks (NEXT-1)       */
#define MIRAGE_ERR_CUDA -9        /* CUDA / cuBLAS failure (sticky)                     */
#define MIRAGE_ERR_NCCL -10       /* reserved: NCCL failure (sticky)                    */

/* ---- families and flags -------------------------------------------------- */
#define MIRAGE_FAMILY_OPT 0   /* pre-LN, ReLU MLP, learned positions (+2), tied head */
#define MIRAGE_FAMILY_LLAMA 1 /* RMSNorm, rotate-half RoPE, SiLU-gated MLP, GQA      */

#define MIRAGE_BETA_1 1       /* one staging slot          (Eq. 4, :472)  */
#define MIRAGE_BETA_2 2       /* double buffering          (Eq. 5, :478)  */
#define MIRAGE_BETA_DYNAMIC 3 /* smallest m with zero predicted stall (reading #6) */

#define MIRAGE_FLAG_TIME_ATTN 1u /* init flag: time every attention launch and every
                                  * slot ready-wait (mirage_stats.stall_ms) with events */
#define MIRAGE_FLAG_SLOT_TAGS 4u /* init flag: race detector for re-streaming. Behind every
                                  * layer DMA the copy stream writes a 4-byte tag
                                  * {0xA5, model, layer} into the slot's tag word; before
                                  * the first kernel of a cycled layer a check kernel
                                  * compares it (mirage_stats.slot_tag_errors).      */
#define MIRAGE_FLAG_CUDA_GRAPHS 8u /* init flag: capture the decode-step body (embed .. argmax)
                                    * into CUDA graphs, one per batch size and, for a
                                    * streaming cycle, per slot parity (uses mod
                                    * lcm(m, beta)); the re-streaming DMAs are a captured
                                    * branch forked from the slot-free events and joined
                                    * before the graph ends (captured on the second step
                                    * of a key; ignored with MIRAGE_FLAG_SLOT_TAGS, during
                                    * reloads and for prefill steps). Together with
                                    * MIRAGE_FLAG_TIME_ATTN the graphs are separate timed
                                    * variants with an event node before and after each
                                    * attention launch (read after each replay; handoff
                                    * stalls and copies are timed in eager steps only) */
#define MIRAGE_FLAG_TP_IPC 16u /* init flag: tensor parallelism without NCCL: after
                                * mirage_tp_export/import, each partial O-/down-projection
                                * is summed by one kernel that reads the peers' partials
                                * over peer memory (NVLink) and applies the residual and
                                * next norm (a one-shot all-reduce fused into its
                                * consumer; fixed rank order, bit-identical on all ranks) */
#define MIRAGE_FLAG_POISON 32u /* init flag (debug): when layers are reclaimed,
                                * their bytes are filled with 0xFF (bf16 NaN) on the compute
                                * stream before any block is handed out, so a kernel that
                                * still read a reclaimed layer as weights would produce NaN.
                                * Blocks carry KV before they are read, so outputs are
                                * unchanged.                                               */
#define MIRAGE_FLAG_TC_GEMM 64u /* init flag: the row-parallel projections (O-proj and
                                 * FC2/down, batch <= 256) run on the library's tcgen05
                                 * decode GEMM (see mirage_decode_gemm) instead of
                                 * cuBLASLt; its split-K slices are summed in fixed order
                                 * by the residual kernel. With MIRAGE_FLAG_TP_IPC the
                                 * GEMM's epilogue stores each partial tile straight into
                                 * every rank's exchange buffer and bumps that rank's
                                 * arrival counter (GEMM fused with a one-shot all-reduce,
                                 * SURVEY NEXT-4); the consumer then reads only local
                                 * memory, in fixed rank order.                        */
#define MIRAGE_FLAG_HOST_ONLY 2u /* init flag: no device; allocator/remap/table/query
                                  * calls only (the arena pointer is used for address
                                  * arithmetic, never dereferenced); device calls
                                  * return MIRAGE_ERR_STATE. For CPU-only replay,
                                  * fuzzing and multi-rank allocator checks.       */

#define MIRAGE_BLOCK_TOKENS 16
#define MIRAGE_MAX_CYCLE 256

typedef struct mirage_ctx mirage_ctx;

typedef struct mirage_init_cfg {
  int32_t device;           /* CUDA device ordinal                                  */
  void* dev_arena;          /* caller-owned device allocation (borrowed)            */
  uint64_t dev_arena_bytes; /* its size; everything the library needs is carved here */
  int32_t block_tokens;     /* tokens per KV block; must be 16                      */
  void* compute_stream;     /* cudaStream_t on which all compute is enqueued        */
  void* copy_stream;        /* cudaStream_t for H2D re-streaming, NULL -> library's */
  int32_t max_batch;        /* max sequences per decode step                        */
  int32_t max_ctx;          /* max tokens per sequence                              */
  uint32_t flags;           /* MIRAGE_FLAG_* bits                                   */
  int32_t tp_rank, tp_size; /* head-sharded tensor parallelism (a10): rank / size     */
  const void* nccl_id;      /* tp_size > 1: 128-byte ncclUniqueId from
                             * mirage_nccl_unique_id() on rank 0, broadcast by the
                             * caller; the library creates and owns the communicator.
                             * NULL: no communicator (tp_size must be 1). With
                             * tp_size == 1 and an id, the all-reduce path runs on
                             * a one-rank communicator (identity; for testing).   */
} mirage_init_cfg;

typedef struct mirage_model_cfg {
  int32_t family;     /* MIRAGE_FAMILY_*                                           */
  int32_t n_layers;   /* hidden layers n                                           */
  int32_t d_model;    /* d; multiple of 128                                        */
  int32_t n_heads;    /* H                                                         */
  int32_t n_kv_heads; /* H_kv; H % H_kv == 0, H/H_kv in {1,2,4,8}                  */
  int32_t head_dim;   /* D in {64, 128}                                            */
  int32_t ffn_dim;    /* multiple of 128                                           */
  int32_t vocab;
  int32_t max_pos;    /* OPT: learned position table has max_pos + 2 rows          */
  float norm_eps;
  float rope_theta;   /* Llama only                                                */
} mirage_model_cfg;

/*
 * Weight blob layout (host, bf16, little-endian; the device copy is identical):
 *   [layer 0][layer 1] ... [layer n-1][globals]
 * Each layer occupies exactly S = mirage_layer_bytes bytes (a multiple of 256),
 * tensors back to back in this order (row-major, PyTorch Linear [out, in]):
 *   OPT  : w_qkv[3d,d] w_o[d,d] w_fc1[f,d] w_fc2[d,f] b_qkv[3d] b_o[d] b_fc1[f]
 *          b_fc2[d] ln1_g[d] ln1_b[d] ln2_g[d] ln2_b[d]
 *   Llama: w_qkv[(H+2H_kv)D,d] w_o[d,HD] w_gateup[2f,d] (gate rows, then up rows)
 *          w_down[d,f] rms1_g[d] rms2_g[d]
 *   w_qkv rows are [q heads | k heads | v heads], head h at rows h*D..h*D+D-1.
 * Globals: OPT: embed[V,d] pos_embed[max_pos+2,d] lnf_g[d] lnf_b[d]
 *          Llama: embed[V,d] normf_g[d] lm_head[V,d]
 *
 * KV block layout (device): one physical block holds 16 tokens of ALL layers:
 *   [L][H_kv][2 (K,V)][16 rows][D] bf16, BB = L*H_kv*2*16*D*2 bytes. Within a
 *   row r (token pos % 16), element c is stored at position
 *   ((c / 8) ^ (r % 8)) * 8 + c % 8 (16-byte chunks XOR-swizzled by row) so the
 *   attention kernel's tensor-core fragment loads are bank-conflict free.
 * Block ids [0, N0) are the native pool; reclaimed ids are appended after.
 */

/* Sizes of one model: S (one hidden layer), globals, and BB (one KV block). */
int32_t mirage_model_sizes(const mirage_model_cfg* m, uint64_t* layer_bytes,
                           uint64_t* global_bytes, uint64_t* block_bytes);

/* Arena bytes mirage_add_model will carve for a model with n_native blocks
 * under the given init limits (weights + native pool + workspace). */
int32_t mirage_model_arena_bytes(const mirage_model_cfg* m, int64_t native_kv_blocks,
                                 int32_t max_batch, int32_t max_ctx, uint64_t* bytes);

/* Bind device and streams; create events, the cuBLAS handle, staging and, for
 * tp_size > 1, the NCCL communicator (collective over the tp_size ranks).
 * Errors: CONFIG (block_tokens != 16, bad tp rank/size, null arena/stream),
 * CUDA, NCCL. */
int32_t mirage_init(const mirage_init_cfg* cfg, mirage_ctx** out);

/* Fill out[128] with a fresh ncclUniqueId (call on TP rank 0 only). */
int32_t mirage_nccl_unique_id(void* out);

/* Synchronise the compute and copy streams, release everything the library
 * owns. Borrowed pointers are not freed. Safe on NULL. */
void mirage_destroy(mirage_ctx* ctx);

/* Message of the last failing call on this ctx ("" if none). Never NULL. */
const char* mirage_last_error(const mirage_ctx* ctx);

/* Add a tenant model. host_blob (pinned, caller-owned, must outlive ctx) holds
 * the layout above and is copied once H2D into the arena. Under tensor
 * parallelism (tp_size > 1, Llama family only; SURVEY.md §8(e) head sharding)
 * m describes the FULL model and the blob holds this rank's shard in the same
 * layout with H/tp q heads, H_kv/tp kv heads and ffn/tp: w_qkv = [the rank's q
 * heads | its k heads | its v heads] rows, w_o = columns of the rank's heads,
 * w_gateup = [the rank's gate rows | its up rows], w_down = the rank's columns;
 * norms, embeddings and the LM head are replicated. The decode step then sums
 * the O-projection and down-projection partials with ncclAllReduce (a10); it stays the
 * authoritative copy re-streamed for cycled layers (PAPER.md:555 footnote: the
 * serving framework keeps a complete host copy of the parameters). The native
 * KV pool gets ids [0, native_kv_blocks). Model ids are 0,1,2,... in call order.
 * Errors: CONFIG (shape constraints, host_bytes mismatch, blob not pinned),
 * CAPACITY (arena exhausted), CUDA. */
int32_t mirage_add_model(mirage_ctx* ctx, const mirage_model_cfg* m, const void* host_blob,
                         uint64_t host_bytes, int64_t native_kv_blocks, int32_t* model_id);

/* MIRAGE_FLAG_TP_IPC setup: tp_export writes this rank's 64-byte CUDA IPC handle
 * of its partial-sum exchange buffer ([flag][2 x max_batch x d fp32]); the caller
 * all-gathers the tp handles (rank order) and passes them to tp_import, which
 * maps the peers' buffers. Errors: CONFIG, STATE, RANGE, CUDA. */
int32_t mirage_tp_export(mirage_ctx* ctx, int32_t model, void* handle_out);
int32_t mirage_tp_import(mirage_ctx* ctx, int32_t model, const void* handles);

/* Re-streaming source tier: point the model's authoritative
 * weight copy -- used for cycled-layer re-streaming and reversion reloads -- at
 * `src` (same layout as the blob): pinned host memory (the default
 * fn.), or device memory, e.g. a peer B200's HBM reached over NVLink 5 (peer
 * access is enabled here), which restores the GH200-like T_T/T_c regime
 * (P:60, :883-890). Caller-owned, must outlive the ctx. Errors: RANGE, CONFIG
 * (size mismatch, pageable memory, no peer access), CUDA. */
int32_t mirage_set_weight_source(mirage_ctx* ctx, int32_t model, const void* src, uint64_t bytes);

/* Pure planner (§5.3-5.4, Eqs. 1-5). Writes the
 * cycle C (ascending, m entries; cycle_out capacity >= n_layers), m and beta.
 * Slot holders are C[0..beta), reclaimed layers R = C[beta..m).
 * Errors: RANGE (bad arguments, alpha + beta > n), INFEASIBLE (dynamic policy
 * found no zero-stall plan). */
int32_t mirage_plan(int32_t n_layers, int32_t alpha, int32_t beta_policy,
                    uint64_t t_transfer_ns, uint64_t t_compute_layer_ns, int32_t anchor,
                    int32_t* cycle_out, int32_t* m_out, int32_t* beta_out);

/* Predicted steady-state stall per decode step (ns) of an explicit cycle: the
 * planner's event simulation of the copy-engine / compute timeline (PAPER.md
 * :310-314, :463-482; the 8th simulated step minus n * t_compute). cycle:
 * ascending layer ids, m entries, beta slots (0 = nothing streamed). Pure, no
 * context. Errors: RANGE. */
int32_t mirage_predict_stall(int32_t n_layers, const int32_t* cycle, int32_t m, int32_t beta,
                             uint64_t t_transfer_ns, uint64_t t_compute_layer_ns, int64_t* stall_ns_out);

/* Reclaim the parameter memory of R = cycle[beta..m) of `donor` as KV blocks of
 * `recipient`. R is split into maximal runs
 * of consecutive layers; each run yields floor(run_bytes / BB_recipient) blocks
 * at byte offsets first*S + i*BB of the donor's weights, appended to the
 * recipient's id space and usable at once. beta > 0 (self-remap of an active
 * model) also installs the cycle: the beta slot holders' storage becomes the
 * staging slots through which all m cycled layers rotate (PAPER.md:411-413,
 * :463-482); the change takes effect at the next decode step. beta == 0
 * requires an inactive donor (its layers are never executed). Eqs. 4/5 are not
 * enforced here (speed, not correctness). KV writes into reclaimed bytes are
 * stream-ordered after every previously enqueued kernel that read them.
 * Errors: RANGE (ids, cycle not strictly ascending, beta > m), STATE (layer
 * already cycled/reclaimed, active donor with beta 0, beta > 0 with donor !=
 * recipient or a cycle already installed), CUDA. */
int32_t mirage_remap_layers(mirage_ctx* ctx, int32_t donor, int32_t recipient,
                            const int32_t* cycle, int32_t m, int32_t beta,
                            int64_t* blocks_gained, uint64_t* reclaimed_bytes);

/* One reclaimed region of a recipient: a maximal run of consecutive donor
 * layers carved by one mirage_remap_layers call. */
typedef struct mirage_region {
  int32_t donor, first_layer, n_layers; /* donor model and its layers [first, first+n)     */
  int32_t first_id, n_blocks;           /* recipient block ids [first_id, first_id+n)      */
  int32_t n_free;                       /* of those, currently free                        */
  int32_t cycle;                        /* 1: part of a streaming self-remap (beta > 0)    */
  int32_t retired;                      /* 1: reverted by mirage_unremap                   */
} mirage_region;

int32_t mirage_region_count(mirage_ctx* ctx, int32_t model, int32_t* n);
int32_t mirage_region_info(mirage_ctx* ctx, int32_t model, int32_t idx, mirage_region* out);

/* Dynamic Reversion (§5.1 "the reclaimed memory is then
 * restored for parameter usage", :830-839 §7.6.1): give region `region` of
 * `recipient` back to its donor's parameters. Every block of the region must be
 * free; the ids are retired (never handed out again, reading #13); the layers'
 * weights are reloaded from the host copy on the COPY stream, one event per
 * layer. The call returns without waiting and enqueues nothing: the donor's next
 * decode step / prefill issues the copies right after its own metadata upload
 * (the host-to-device copy engine is FIFO across streams, so copies queued
 * earlier would hold that upload back), ordered after every kernel enqueued
 * before it on the compute stream (the last readers of the bytes as KV); its
 * first kernel that reads layer l waits for layer l's event only, so a cold
 * start's prefill overlaps the reload layer by layer (PAPER.md:387, :395-397
 * "T_T * N <= T_Compute" with T_Compute = prefill). mirage_sync also issues
 * requested reloads. A
 * region of a streaming self-remap reverts the donor's whole cycle (all its
 * regions, slot holders reloaded, streaming stops at the next step).
 * Errors: RANGE; STATE (already reverted); PRESSURE (blocks still hold KV);
 * CUDA. */
int32_t mirage_unremap(mirage_ctx* ctx, int32_t recipient, int32_t region);

/* Block migration before Dynamic Reversion (reading #29: the paper restores
 * reclaimed memory "when KV cache space is sufficient", PAPER.md:352-354,
 * :830-834, and is silent on blocks still live in it). The region's live block
 * ids (a streaming cycle: all of its regions'), ascending, take the lowest free
 * ids outside it, ascending, one for one; every block-table entry is renamed in
 * place, the old ids become free, and each moved block's bytes (block_bytes, all
 * layers) are copied on the compute stream after every kernel enqueued before.
 * The region can then be reverted with mirage_unremap. *n_moved (may be NULL)
 * receives the number of blocks moved. Errors: RANGE; STATE (already reverted);
 * NO_BLOCKS (fewer free ids outside the region than live blocks; nothing changed). */
int32_t mirage_migrate_region(mirage_ctx* ctx, int32_t model, int32_t region, int32_t* n_moved);

/* Mark a tenant active (1) or inactive (0) (temporal sharing).
 * Errors: RANGE; STATE (activating a model with reclaimed layers: unremap its
 * regions first; the reload then overlaps the next prefill). */
int32_t mirage_set_active(mirage_ctx* ctx, int32_t model, int32_t active);

/* Allocate n blocks for seq_id: the n lowest free ids, ascending, appended to
 * its table; all-or-nothing (reading #14). ids_out (capacity n, may be NULL).
 * Errors: RANGE; NO_BLOCKS with *shortfall_out = n - free (state unchanged). */
int32_t mirage_alloc_blocks(mirage_ctx* ctx, int32_t model, int64_t seq_id, int32_t n,
                            int32_t* ids_out, int32_t* shortfall_out);

/* Return all blocks of seq_id and forget the sequence (reading #15).
 * Errors: RANGE; DOUBLE_FREE for an unknown or already freed sequence. */
int32_t mirage_free_blocks(mirage_ctx* ctx, int32_t model, int64_t seq_id);

/* KV swapping baseline (Pie-style):
 * swap_out copies seq_id's KV blocks (all layers, ceil(len/16) * BB bytes, in
 * table order) to host_dst (pinned, >= that size) on the compute stream and
 * frees the blocks; swap_in allocates blocks again and copies them back. The
 * cached length is kept while swapped out. Errors: RANGE, STATE, NO_BLOCKS, CUDA. */
int32_t mirage_swap_out(mirage_ctx* ctx, int32_t model, int64_t seq_id, void* host_dst, uint64_t bytes);
int32_t mirage_swap_in(mirage_ctx* ctx, int32_t model, int64_t seq_id, const void* host_src);

/* Copy of the host block table of seq_id. Errors: RANGE (unknown seq, cap too
 * small; *n_out still receives the length). */
int32_t mirage_get_block_table(mirage_ctx* ctx, int32_t model, int64_t seq_id, int32_t* out,
                               int32_t cap, int32_t* n_out);

/* Where block `block_id` of `model` lives: donor = -1 for the native pool
 * (offset from the pool start), else the donor model id and the byte offset
 * from the start of the donor's layer-0 weights. Errors: RANGE. */
int32_t mirage_block_location(mirage_ctx* ctx, int32_t model, int32_t block_id, int32_t* donor,
                              uint64_t* offset);

/* Tokens cached for seq_id (0 if unknown). */
int32_t mirage_seq_len(mirage_ctx* ctx, int32_t model, int64_t seq_id, int32_t* len_out);

/* One decode step for `batch` rows (Alg. 1 line 13
 * "GPU LLM Kernel(enable_remap, remapped_layer_list)"). A row is one token of
 * seq_ids[i] at positions[i]; the step appends the row's K/V at that position
 * and attends over positions[i]+1 tokens (causal), so the sequence needs
 * >= ceil((positions[i]+1)/16) blocks. Normally every row is a different
 * sequence and positions[i] equals its cached length. Several rows may name one
 * sequence (a prefill / extend chunk): in row order they must take consecutive
 * positions starting at its cached length; all rows' K/V are appended before any
 * row attends. tokens are teacher-forced by the caller.
 * hidden_out: device bf16 [batch, d] (final normalised hidden) or NULL.
 * argmax_out: host int32 [batch] (greedy token, lowest index on ties) or NULL;
 * valid after the compute stream is synchronised.
 * Errors: RANGE (batch, ids), NO_BLOCKS (a missing block, checked before any
 * enqueue), STATE (position != cached length, model inactive or fully
 * reclaimed), CUDA. */
int32_t mirage_decode_step(mirage_ctx* ctx, int32_t model, int32_t batch, const int64_t* seq_ids,
                           const int32_t* tokens, const int32_t* positions, void* hidden_out,
                           int32_t* argmax_out);

/* Prefill (§2.1: the prompt is processed in parallel and its
 * KV cached; the cold-start phase of :395-397). n_seqs prompts; prompt i has
 * prompt_lens[i] > 0 tokens, concatenated in `tokens` (host int32, sum of
 * lengths). Each prompt is appended at its sequence's cached length (0 for a
 * new sequence: prefill; > 0: extend). The rows run as mirage_decode_step
 * chunks of at most max_batch rows, each one layer-major pass, so a pending
 * asynchronous reload gates each layer separately. last_argmax_out: host int32
 * [n_seqs], the greedy next token after each prompt (the call then synchronises
 * the compute stream), or NULL (asynchronous). Blocks must be allocated.
 * Errors: RANGE (lengths, duplicate seq), NO_BLOCKS, STATE, CUDA. */
int32_t mirage_prefill(mirage_ctx* ctx, int32_t model, int32_t n_seqs, const int64_t* seq_ids,
                       const int32_t* prompt_lens, const int32_t* tokens, int32_t* last_argmax_out);

typedef struct mirage_stats {
  int64_t native_blocks, total_blocks, free_blocks;
  uint64_t layer_bytes, block_bytes;
  uint64_t reclaimed_bytes; /* bytes of R carved into this model's pool           */
  uint64_t donated_bytes;   /* bytes of this model's layers reclaimed            */
  int32_t m, beta, active, n_seqs;
  int32_t cycle[MIRAGE_MAX_CYCLE];
  uint64_t uses;            /* cycled-layer uses enqueued so far                 */
  uint64_t h2d_copies, h2d_bytes;
  double h2d_ms;            /* summed event time of completed H2D copies         */
  double last_step_ms;      /* event time of the last completed decode step (steps with prefill rows excluded: T_Compute) */
  int64_t steps;
  /* with MIRAGE_FLAG_TIME_ATTN: completed attention launches, their summed event
   * time and algorithmic KV bytes (sum over sequences of ctx_len * 2 * H_kv * D * 2) */
  int64_t attn_launches;
  double attn_ms;
  uint64_t attn_bytes;
  uint64_t last_meta_h2d_bytes; /* step metadata uploaded by the last decode step    */
  int32_t last_attn_units;      /* attention work units of the last decode step      */
  int32_t last_split_blocks;    /* blocks per split-K partition of the last step     */
  int64_t slot_tag_errors;      /* MIRAGE_FLAG_SLOT_TAGS: cycled layers that started
                                 * before their weights had landed (must stay 0)     */
  int64_t tp_peer_timeouts;     /* MIRAGE_FLAG_TP_IPC: all-reduce waits that gave up
                                 * on a peer (must stay 0)                            */
  /* with MIRAGE_FLAG_TIME_ATTN: the compute stream's measured stall on the slot
   * handoff (a5): event time from reaching a cycled layer's ready-wait to passing
   * it, summed over completed waits (0 when re-streaming is hidden)  */
  int64_t stall_waits;
  double stall_ms;
} mirage_stats;

int32_t mirage_query(mirage_ctx* ctx, int32_t model, mirage_stats* out);

/* Slot-assignment log of `model` since its cycle was installed: rows of
 * (k, step, layer, slot, copied) as int64, row-major [n][5]; equals the
 * oracle's c5 log. Errors: RANGE (cap too small; *n_out gets the length). */
int32_t mirage_slot_log(mirage_ctx* ctx, int32_t model, int64_t* out, int32_t cap, int32_t* n_out);

/* Change the measurement-mode init flags of a live ctx: the bits of `mask`
 * among MIRAGE_FLAG_TIME_ATTN and MIRAGE_FLAG_CUDA_GRAPHS are set to their
 * values in `flags` (other bits of mask: CONFIG). Takes effect at the next step;
 * captured graphs are kept (they are replayed again once MIRAGE_FLAG_CUDA_GRAPHS
 * is set and MIRAGE_FLAG_TIME_ATTN clear). Errors: CONFIG. */
int32_t mirage_set_flags(mirage_ctx* ctx, uint32_t flags, uint32_t mask);

/* Block until all work enqueued by this ctx has finished; reports sticky errors. */
int32_t mirage_sync(mirage_ctx* ctx);

/* ---- test / bench hooks --------------------------------------------------- */

/* Paged attention of one layer only (a8+a9), over the sequences' current
 * cached lengths. q_dev: device fp32 [batch, H, D]; out_dev: device [batch, H,
 * D] fp32 (out_fp32 = 1) or bf16. split_tokens_override > 0 forces the split
 * size (multiple of 16); -1 forces the balanced-range schedule.
 * Errors: RANGE, STATE (a sequence with 0 tokens). */
int32_t mirage_attn_only(mirage_ctx* ctx, int32_t model, int32_t layer, int32_t batch,
                         const int64_t* seq_ids, const float* q_dev, void* out_dev,
                         int32_t out_fp32, int32_t split_tokens_override);

/* Append n_tokens synthetic tokens of KV to seq_id (all layers), values from
 * the counter-based generator documented in oracle/kvgen.py's header (the
 * kernel implements it independently). Needs the blocks. Errors: RANGE,
 * NO_BLOCKS. */
int32_t mirage_fill_kv(mirage_ctx* ctx, int32_t model, int64_t seq_id, int32_t n_tokens,
                       uint64_t seed);

/* Append n_tokens of caller KV to seq_id: host_kv bf16 [L][H_kv][2][n][D]
 * (any host memory; copied synchronously). Errors: RANGE, NO_BLOCKS. */
int32_t mirage_write_kv(mirage_ctx* ctx, int32_t model, int64_t seq_id, int32_t n_tokens,
                        const void* host_kv);

/* Page-lock (cudaHostRegister, portable) / release caller host memory, e.g. a
 * weight blob in a file mapping shared by the replicas on one node, so it can
 * serve as a pinned host blob. Errors: RANGE (null/zero), CUDA. */
int32_t mirage_host_register(void* ptr, uint64_t bytes);
int32_t mirage_host_unregister(void* ptr);

/* Number of kernels this ctx has launched (its own kernels, not cuBLAS). */
int64_t mirage_kernel_launches(const mirage_ctx* ctx);

/* Test/bench hook: the decode GEMM of the step on the 5th-generation tensor
 * cores (tcgen05 + TMEM, TMA-fed; SURVEY §8(a) a6 supporting row, NEXT-4):
 * Y_s[b][n] = sum over split s's share of K of X[b][k] * W[n][k], for
 * W = w_dev bf16 [N][K] and X = x_dev bf16 [B][K] (row-major, device memory,
 * K % 8 == 0, 1 <= B <= 256, or <= 256 * col_groups), written to y_dev fp32 [splits][B][N]; the splits
 * partition K in order and sum to Y. splits = 0 picks the library's choice
 * (a per-SM load model) and reports it in *splits_out. reduce != 0: splits
 * of a tile run as one thread-block cluster and are summed in split order
 * through distributed shared memory inside the kernel (at most 8 splits,
 * B <= 128), so y_dev receives ONE slice [B][N] and *splits_out is set to 1.
 * col_groups (0 or 1 = none, at most 8): the batch rows are cut into that many
 * groups (each rounded up to 32/64/128/256 rows; empty groups dropped), one CTA
 * per (128-row tile, split, group), each re-reading its tile's weights (the
 * fused tensor-parallel push GEMM runs one split this way; not with reduce);
 * B may then reach 256 * col_groups.
 * Enqueued on `stream` (a cudaStream_t; NULL = legacy default stream).
 * Errors: RANGE, CUDA. */
int32_t mirage_decode_gemm(void* stream, const void* w_dev, int32_t N, int32_t K, const void* x_dev, int32_t B,
                           float* y_dev, int32_t splits, int32_t reduce, int32_t col_groups, int32_t* splits_out);

/* Test/bench hook: the persistent stream-K form of the tcgen05 decode GEMM
 * (SURVEY §8(a) a6 supporting row, NEXT-4): one wave of CTAs
 * walks the tiles x 64-wide K blocks in order, and a tile cut between CTAs is
 * finished inside the GEMM by the CTA holding its first K block, which adds the
 * others' parked fp32 partials in K order (deterministic). Computes
 * y = epilogue(X W^T) for W = w_dev bf16 [N][K], X = x_dev bf16 [B][K]
 * (row-major, device memory, K % 8 == 0, 1 <= B <= 256): + bias_dev[N] (bf16,
 * or NULL), then max(., 0) if relu, stored to y_dev fp32 [B][N] or, if y_dev is
 * NULL, to y16_dev bf16 [B][N]. Uses a library-owned workspace per device
 * (allocated on first use, kept for the process), so calls on one device must
 * be ordered on one stream. Enqueued on `stream` (a cudaStream_t; NULL = legacy
 * default stream) on the current device. Errors: RANGE, CUDA. */
int32_t mirage_sk_gemm(void* stream, const void* w_dev, int32_t N, int32_t K, const void* x_dev, int32_t B,
                       float* y_dev, void* y16_dev, const void* bias_dev, int32_t relu);

/* Profiling hook. With the environment variable MIRAGE_ATTN_TRACE set when the
 * ctx is created, every attention launch of mirage_attn_only records 16
 * %globaltimer slots per CTA (ns: entry, first tiles issued, first tile
 * landed, last tile consumed, last output written, last split combine, exit;
 * slot 7 = items processed; 9 = every consumer warp done with the last item;
 * 8, 10 = phases of the last combine: ticket taken, weights computed; 12-15 =
 * SM cycles from the merge start to the ticket, the first head's max, the
 * weights barrier and the end of the fold). This call synchronizes the compute stream and
 * copies the last launch's [n_ctas][16] uint64 slots to host_out (capacity
 * cap_ctas CTAs). Errors: STATE (tracing off), RANGE (cap too small; *n_ctas
 * still receives the count), CUDA. */
int32_t mirage_attn_trace(mirage_ctx* ctx, uint64_t* host_out, int32_t cap_ctas, int32_t* n_ctas);

#ifdef __cplusplus
}
#endif
#endif /* MIRAGE_H_ */
