/*
 * hgnn.h — C-ABI of the B200-native HydraGNN (PNA-GCNN) data-parallel training step.
 *
 * The calls follow the paper's problem statement — pack a batch of graphs,
 * forward, backward, allreduce gradients, step (BASELINE.json north_star;
 * PAPER.md:160-164 §3.2 "each iteration consists of a forward, backward, and
 * optimization step"; §4 gradient aggregation with NCCL) —
 * and mirror the SPEC.md interfaces for this path (SPEC.md:266-283 dataload,
 * 337-384 gcnn, 435-455 ddp). Everything below is plain C: host or device
 * pointers, sizes and status codes; no PyTorch types.
 *
 * Conventions
 *  - Every call returns hg_status; HG_OK == 0. On failure hg_last_error()
 *    returns a thread-local message describing the most recent failure.
 *  - Argument / shape validation is synchronous. Device work is enqueued
 *    asynchronously on the ctx's compute stream (the caller's stream handed to
 *    hg_ctx_create). CUDA / NCCL failures are sticky: once one is seen the ctx
 *    returns HG_E_STATE from every later device call; hg_sync() reports it.
 *  - Floating point: fp32 storage and fp32 arithmetic on the device (GEMMs in
 *    fp32-accurate form); the CPU oracle (tests only) is float64.
 *  - Ownership: the caller owns every pointer it passes. hg_store_create
 *    copies (or, with copy == 0, borrows) the arrays; the device workspace is
 *    caller-owned and must outlive the ctx.
 */
#ifndef HGNN_H
#define HGNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_ABI_VERSION 2

typedef enum {
  HG_OK = 0,
  HG_E_INVALID = 1,    /* bad argument (null pointer, negative size, ...) */
  HG_E_SHAPE = 2,      /* InconsistentFeatureWidth / ShapeMismatch */
  HG_E_RANGE = 3,      /* IndexOutOfRange: graph id or node id out of range */
  HG_E_EMPTY = 4,      /* EmptyBatch / EmptyGraphSlot */
  HG_E_ASYMMETRIC = 5, /* edge list not symmetric with identical attributes */
  HG_E_DEGREE = 6,     /* a node degree exceeds HG_MAX_DEGREE / max_degree, or a batch holds more
                          distinct node degrees than the ctx's degree-class slots */
  HG_E_CAPACITY = 7,   /* batch exceeds the ctx capacities (max_graphs / max_nodes / max_edges) */
  HG_E_CUDA = 8,       /* CUDA runtime failure */
  HG_E_NCCL = 9,       /* NCCL failure (TransportFailure) */
  HG_E_STATE = 10,     /* ctx unusable after a sticky failure, or call out of order */
  HG_E_UNSORTED = 11,  /* per-graph edges not sorted by (src, dst) */
  HG_E_IO = 12         /* container / object file missing, truncated, bad magic or checksum */
} hg_status;

/* Largest supported node degree: argmin/argmax positions are stored as u8
 * with bit 7 reserved for the std variance-floor flag. */
#define HG_MAX_DEGREE 127

const char *hg_last_error(void);
int32_t hg_abi_version(void);

/* ======================================================================
 * Graph store — the Table-1 global arrays (§3.3)
 * ====================================================================== */
typedef struct hg_store hg_store;

typedef struct {
  int64_t num_graphs, num_nodes, num_edges;
  int32_t f_node, f_edge;            /* F0 = |vocab| + 3, Fe = 4 */
  const int64_t *node_offset;        /* [num_graphs + 1], starts at 0, non-decreasing */
  const int64_t *edge_offset;        /* [num_graphs + 1], starts at 0, non-decreasing */
  const float *x;                    /* [num_nodes][f_node] row-major */
  const int32_t *edge_index;         /* [2][num_edges]: row 0 = src, row 1 = dst, graph-local ids,
                                        per graph sorted by (src, dst), each bond in both directions */
  const float *edge_attr;            /* [num_edges][f_edge] */
  const float *y;                    /* [num_graphs] target (eV) */
  const float *y_node;               /* [num_nodes] node-level targets (node-level head), nullable = 0 */
} hg_store_desc;

/* Validate and adopt a store. copy != 0: arrays are copied (caller may free on
 * return); copy == 0: arrays are borrowed and must outlive the store.
 * Validation (multi-threaded over graphs, `threads` <= 0 = all cores):
 * ids in range (HG_E_RANGE), per-graph (src, dst) order strictly increasing
 * (HG_E_UNSORTED), symmetry with identical attributes (HG_E_ASYMMETRIC),
 * degree <= HG_MAX_DEGREE (HG_E_DEGREE), every graph non-empty (HG_E_EMPTY).
 * Also derives, per directed edge, slot = position of src inside dst's
 * neighbour row. */
hg_status hg_store_create(const hg_store_desc *d, int32_t copy, int32_t threads, hg_store **out);
hg_status hg_store_destroy(hg_store *s);
/* One copy of the store shared by every rank of the node: hg_store_create_shared
 * validates `d` like hg_store_create, derives the slots and writes everything into the new POSIX
 * shared-memory object `name` ("/..."; HG_E_IO if it exists); hg_store_open_shared maps an
 * existing one read-only in another process (HG_E_IO: missing, or not a store). pin_memory != 0
 * page-locks the mapping (cudaHostRegister; HG_E_CUDA if that fails, e.g. without a GPU).
 * hg_store_destroy unmaps; hg_store_unlink_shared removes the name (once every rank opened it). */
hg_status hg_store_create_shared(const hg_store_desc *d, const char *name, int32_t pin_memory, int32_t threads,
                                 hg_store **out);
hg_status hg_store_open_shared(const char *name, int32_t pin_memory, hg_store **out);
hg_status hg_store_unlink_shared(const char *name);
/* Totals and maxima over the store (Table 2 style summary). */
hg_status hg_store_stats(const hg_store *s, int64_t *graphs, int64_t *nodes, int64_t *edges,
                         int32_t *max_nodes_per_graph, int32_t *max_degree);
/* PNA degree statistic delta = mean over the nodes of graphs `ids` of ln(d+1),
 * float64. ids == NULL: all graphs. */
hg_status hg_degree_stat(const hg_store *s, const int64_t *ids, int64_t n, double *delta);
/* delta_lin = mean in-degree over the nodes of graphs `ids` (NULL: all), float64: the
 * normaliser of the linear scalers (hg_config.delta_lin). */
hg_status hg_degree_stat_linear(const hg_store *s, const int64_t *ids, int64_t n, double *delta_lin);

/* ======================================================================
 * Sharding ("shuffled and disjointed subsets")
 * Global per-epoch permutation of [0, n) ascending by (splitmix64(seed ^
 * epoch*0x9E3779B97F4A7C15 ^ i*0xD1B54A32D192ED03), i); rank takes positions
 * p == rank (mod world), drop-last to floor(n/world).
 * ids_out capacity >= n / world. Host-only, deterministic.
 * ====================================================================== */
hg_status hg_shard(uint64_t seed, int64_t epoch, int32_t rank, int32_t world, int64_t n,
                   int64_t *ids_out, int64_t *n_out);

/* ======================================================================
 * Model configuration
 * ====================================================================== */
typedef struct {
  int32_t f_node, f_edge;            /* input widths F0, Fe */
  int32_t hidden;                    /* H in [1, 1024]; not a multiple of 32 => channel-padded
                                        internally (hg_config_internal) */
  int32_t layers;                    /* L >= 1 conv layers */
  int32_t fc_hidden;                 /* Hf: head hidden width (= H) */
  int32_t max_graphs;                /* capacity: graphs per batch */
  int32_t max_nodes;                 /* capacity: nodes per batch */
  int32_t max_edges;                 /* capacity: directed edges per batch */
  int32_t n_slots;                   /* device batch slots (>= 1; 2+ to overlap H2D with compute) */
  int32_t flags;                     /* HG_FLAG_*; 0 = defaults */
  double delta;                      /* PNA degree statistic (hg_degree_stat) */
  float var_floor;                   /* epsilon_v for the std aggregator, 1e-10 */
  int32_t max_degree;                /* capacity: largest node degree in a batch (0 = HG_MAX_DEGREE).
                                        Degree-class slots = min(max_degree + 1, 32): a batch may hold
                                        at most that many DISTINCT node degrees (HG_E_DEGREE at pack
                                        time otherwise; molecules: <= 6). DESIGN.md §6. */
  int32_t scalers;                   /* PNA degree scalers, HG_SCALER_* bit set (0 = the default
                                        IDENTITY | AMPLIFICATION | ATTENUATION); identity
                                        required. U holds 4 * popcount(scalers) blocks of H columns,
                                        scaler-major in bit order, aggregator-minor. */
  double delta_lin;                  /* mean in-degree over the training set (hg_degree_stat_linear):
                                        normaliser of the LINEAR / INVERSE_LINEAR scalers (> 0 if used) */
  float node_weight;                 /* HG_FLAG_NODE_HEAD: weight of the node-level MSE in the loss (>= 0) */
} hg_config;

/* Degree scalers (SURVEY §8(f) row 3 adds PNA's linear pair, DESIGN.md
 * reading R-scalers): identity 1, amplification ln(d+1)/delta, attenuation delta/ln(d+1),
 * linear d/delta_lin, inverse_linear delta_lin/d; every scaler is 1 at d = 0. */
#define HG_SCALER_IDENTITY 1
#define HG_SCALER_AMPLIFICATION 2
#define HG_SCALER_ATTENUATION 4
#define HG_SCALER_LINEAR 8
#define HG_SCALER_INVERSE_LINEAR 16

/* hg_config.flags: HG_FLAG_TF32 selects the reduced-precision GEMM mode (
 * PAPER.md:212): every tensor-core contraction runs ONE tf32 pass (operands truncated to
 * tf32, fp32 accumulate) instead of the fp32-accurate 3xTF32 default. Everything else
 * (aggregation, head, loss, AdamW, the exchange) stays fp32. Its parity bars are looser
 * (DESIGN.md §3 "TF32 mode": forward 2e-2 max-scaled, gradients / moments / parameters 5e-2). */
#define HG_FLAG_TF32 1
/* hg_config.flags: HG_FLAG_SELF_TERM selects the PNA self-term variant (SURVEY C1 / §8(f)
 * row 3, reading R-self): the message is M [x_j || x_i || e_ij] + b_M and the update
 * [scaled aggregates || x_i] [U | U_x]^T + b_U, with the extra parameters conv<l>.M_s [H, F_l]
 * (after M_x) and conv<l>.U_x [H, F_l] (after U). Requires f_node <= hidden. */
#define HG_FLAG_SELF_TERM 2
/* hg_config.flags: HG_FLAG_NODE_HEAD adds a node-level head beside the graph head (PAPER.md:77
 * "multitask prediction of hybrid node-level and graph-level properties", PAPER.md:144 atom-level
 * properties; reading R-node-head): per node yhat_i = W2n ReLU(W1n x_L,i + b1n) + b2n
 * (parameters head_n.W1 [fc_hidden, H], head_n.b1, head_n.W2 [1, fc_hidden], head_n.b2 after the
 * graph head's), and loss = graph MSE + node_weight * mean over the batch's nodes of
 * (yhat_i - y_node,i)^2 with the store's y_node targets. */
#define HG_FLAG_NODE_HEAD 4

/* Channel padding for widths that are not a multiple of the tensor-core tile (128),
 * e.g. the paper's H = 55 and H = 200 (SURVEY §8(d) "Padding
 * hazard"), or config A's H = 32. Writes to *out the configuration the kernels
 * actually run: hidden rounded up to a multiple of 128 and fc_hidden padded alike
 * when it equals hidden; *out = *c when hidden % 128 == 0.
 * The padded channels compute exact zeros: padded parameter entries start at
 * zero, the std aggregator of a padded channel is forced to 0 (not
 * sqrt(var_floor)), so every padded gradient is exactly zero and AdamW keeps
 * the padding at zero. Everything public stays logical: hg_param_info, the
 * params / grads / optimizer-state arenas of get/set are in the layout of *c
 * (hg_param_layout(c)); only hg_workspace_view buffers are internal-width.
 * Host-only. Errors: HG_E_INVALID as hg_workspace_bytes. */
hg_status hg_config_internal(const hg_config *c, hg_config *out);

typedef struct {
  float lr, beta1, beta2, eps, weight_decay;  /* 1e-3, 0.9, 0.999, 1e-8, 0.01 */
} hg_adamw;

/* ---- packed batch layout -----------------------------------
 * One contiguous blob per batch (host staging and device slot alike):
 *   header   int32[16]: B, N, E, F0, Fe, then zeros
 *   graph_ptr int32[B+1]   cumulative node counts
 *   y         float[B]
 *   y_node    float[N]     node-level targets (zeros when the store has none)
 *   rowptr    int32[N+1]   CSR over destination nodes
 *   col       int32[E]     in-neighbour ids, ascending within a row
 *   x         float[N*F0]
 *   eattr     float[E*Fe]  attribute of edge col -> row
 *   slot      uint8[E]     position of row inside col's row
 * each array starting at a 16-byte aligned offset given by hg_batch_offsets. */
typedef struct {
  int64_t graph_ptr, y, y_node, rowptr, col, x, eattr, slot, total;  /* byte offsets; total = blob size */
} hg_batch_offsets;
hg_status hg_batch_offsets_get(int32_t B, int32_t N, int32_t E, int32_t f_node, int32_t f_edge,
                               hg_batch_offsets *off);

/* Host-only collate: gather graphs `ids` (B of them, in
 * order) from the store into `dst` (capacity `cap` bytes) in the layout above.
 * Fails with HG_E_EMPTY (B == 0), HG_E_RANGE, HG_E_SHAPE (widths differ from
 * cfg), HG_E_CAPACITY (exceeds cfg capacities or cap). *used = blob bytes. */
hg_status hg_pack_host(const hg_store *s, const int64_t *ids, int32_t B, const hg_config *cfg,
                       void *dst, size_t cap, size_t *used);
/* Host threads one collation (hg_pack / hg_pack_host) uses, process-wide (default 4; the
 * packed bytes do not depend on it). HG_E_INVALID outside [1, 1024]. */
hg_status hg_pack_threads_set(int32_t threads);

/* Host-side parameter initialisation into a flat fp32 array laid out like the
 * device arena (hg_param_info offsets; padding zero). SPEC.md:339, 401 with the
 * counter-based rule of SURVEY C12. n_elems = hg_param_layout total. */
hg_status hg_param_layout(const hg_config *c, int32_t *n_tensors, int64_t *n_elems);
hg_status hg_param_layout_info(const hg_config *c, int32_t i, const char **name, int64_t *offset,
                               int32_t *rows, int32_t *cols);
hg_status hg_params_init_host(const hg_config *c, uint64_t seed, float *dst);

/* ======================================================================
 * Device context (one per rank / GPU)
 * ====================================================================== */
typedef struct hg_ctx hg_ctx;

/* Bytes of device workspace the ctx needs (params, grads, Adam moments,
 * batch slots, per-layer activations, backward scratch), 256-byte aligned. */
hg_status hg_workspace_bytes(const hg_config *c, size_t *bytes);
/* workspace: caller-owned device memory of >= hg_workspace_bytes bytes on
 * `device`; stream: the caller's cudaStream_t (NULL = legacy default stream).
 * Parameters start zeroed; call hg_params_init or hg_params_set. */
hg_status hg_ctx_create(const hg_config *c, int32_t device, void *workspace, size_t bytes,
                        void *stream, hg_ctx **out);
hg_status hg_ctx_destroy(hg_ctx *x);

hg_status hg_param_count(const hg_ctx *x, int32_t *n_tensors, int64_t *n_elems);
hg_status hg_param_info(const hg_ctx *x, int32_t i, const char **name, int64_t *offset,
                        int32_t *rows, int32_t *cols);
hg_status hg_params_init(hg_ctx *x, uint64_t seed);
/* on_device != 0: src/dst are device pointers; else host pointers. Arrays are
 * the flat arena (n_elems floats). Synchronous w.r.t. the compute stream. */
hg_status hg_params_set(hg_ctx *x, const float *src, int32_t on_device);
hg_status hg_params_get(hg_ctx *x, float *dst, int32_t on_device);
hg_status hg_grads_get(hg_ctx *x, float *dst, int32_t on_device);
hg_status hg_opt_state_get(hg_ctx *x, float *m, float *v, int64_t *step, int32_t on_device);
hg_status hg_opt_state_set(hg_ctx *x, const float *m, const float *v, int64_t step, int32_t on_device);

/* Checkpoint / resume ("versioned binary dump of config + named parameter tensors +
 * optimizer state, little-endian, with CRC"). File: "HGNNCKPT", u32 version 1, the
 * model part of hg_config (f_node, f_edge, hidden, layers, fc_hidden, flags, scalers, delta,
 * delta_lin, var_floor, node_weight), the named tensor table (name, offset, rows, cols), the
 * parameter arena, the Adam step, m and v (logical widths, hg_param_layout), then a CRC-32C of
 * everything before it. Save gathers sharded moments first (peer-memory exchange) and writes
 * path atomically (path.tmp, then rename). Load requires the same model configuration (the
 * TF32 flag may differ) and tensor table: HG_E_SHAPE otherwise; HG_E_IO for a missing,
 * truncated or corrupt file (nothing is changed then). Synchronous. */
hg_status hg_checkpoint_save(hg_ctx *x, const char *path);
hg_status hg_checkpoint_load(hg_ctx *x, const char *path);

/* Debug / parity views into the workspace: byte offset and size of a named
 * buffer. what: 0 = P_l [N,H] ([N,2H] = [P | Q] with the self-term), 1 = A_l [N,4H]
 * (mean|min|max|std, degree-sorted rows; [N,5H] with the self-term's x_i block), 2 = arg_l
 * [N,2H] u8 (argmin | argmax with bit7 = var>floor), 3 = X_{l+1} [N,H],
 * 4 = batch slot `layer` blob, 5 = yhat [B], 6 = loss [1], 7 = head hidden
 * pre-activation [B,Hf], 8 = params, 9 = grads, 10 = amp [N] and 11 = att [N] of batch slot
 * `layer` (the node scalers, computed with the slot's degree classes when its batch is
 * uploaded), 12 = node-level head yhat [N], 13 = its hidden pre-activation [N,Hf]
 * (HG_FLAG_NODE_HEAD). */
hg_status hg_workspace_view(const hg_ctx *x, int32_t what, int32_t layer, int64_t *offset, int64_t *bytes);

/* Debug: copy batch slot `slot`'s packed blob (layout above; its header gives B, N, E) to
 * host memory dst (capacity cap bytes), after the slot's pending H2D copy and the compute
 * stream's work. *used = blob bytes. HG_E_RANGE bad slot, HG_E_CAPACITY cap too small. */
hg_status hg_batch_get(hg_ctx *x, int32_t slot, void *dst, size_t cap, size_t *used);

/* Collate `ids` from the store on the host (pinned staging buffer of `slot`)
 * and enqueue the H2D copy on the ctx's copy stream, followed there by the batch's degree
 * classes (stable sort by in-degree, class table, GEMM tiles, per-graph ranges: DESIGN.md §5,
 * one CTA beside any running step); later device work on that slot waits for both. The
 * staging buffer is reused only after its previous copy completed. Errors as hg_pack_host. */
hg_status hg_pack(hg_ctx *x, const hg_store *s, const int64_t *ids, int32_t B, int32_t slot);
/* Copy an already packed blob (host pointer, e.g. from hg_pack_host) into `slot`. The blob is
 * validated first (header, capacities, offsets, degrees, distinct-degree count); the degree
 * classes follow on the copy stream as in hg_pack. */
hg_status hg_upload_packed(hg_ctx *x, const void *blob, size_t bytes, int32_t slot);

/* Forward pass on the batch in `slot`: L GC layers, global
 * mean pool, FC head, MSE
 * loss written to the device loss cell. */
hg_status hg_forward(hg_ctx *x, int32_t slot);
/* Backward pass of the last forward on `slot`: writes every
 * parameter gradient (overwrites, no accumulation). */
hg_status hg_backward(hg_ctx *x, int32_t slot);

/* NCCL data-parallel plumbing. The 128-byte unique id is
 * produced on rank 0 and distributed by the caller (e.g. torch.distributed).
 * hg_comm_init: world == 1 with id128 == NULL sets rank/world only (no communicator:
 * the exchange is a no-op); with an id (world >= 1) it creates the NCCL communicator, so
 * a one-rank communicator runs the bucketed average path too. HG_E_STATE if called twice. */
hg_status hg_nccl_unique_id(void *out128);
hg_status hg_comm_init(hg_ctx *x, const void *id128, int32_t rank, int32_t world);
/* Mean over ranks of the gradient arena; no-op without a communicator. */
hg_status hg_allreduce_grads(hg_ctx *x);
/* The gradient buckets of a configuration (host-only): *n = bucket count; ranges (capacity
 * `cap` buckets, nullable) receives [begin, end) float offsets into the flat parameter arena
 * of the INTERNAL layout (hg_config_internal), in backward (launch) order: bucket 0 = head +
 * the last layers ... last bucket = conv0. Together they cover the arena exactly once. */
hg_status hg_bucket_layout(const hg_config *c, int64_t *ranges, int32_t cap, int32_t *n);

/* Gradient exchange over NVLink peer memory (reduce-scatter ->
 * sharded fused AdamW -> all-gather, as ONE kernel; PAPER.md:206-212 DDP averaging).
 * hg_p2p_handle writes this rank's HG_P2P_HANDLE_BYTES record (CUDA IPC handle of the
 * workspace allocation + the workspace's byte offset in it; the workspace must be a
 * cudaMalloc-backed allocation, e.g. torch's default caching allocator, not
 * expandable segments -> HG_E_CUDA). After every rank's records are gathered (rank
 * order, world x HG_P2P_HANDLE_BYTES bytes) hg_p2p_open maps the peers' workspaces
 * (requires hg_comm_init with 2 <= world <= 8; all ranks use the same config).
 * From then on hg_train_step / hg_capture_step end every step with: this rank's
 * gradients ready -> flag in every rank; each rank sums the W gradient copies of its
 * 1/W shard of the flat arena in rank order over peer loads, divides by W, applies
 * AdamW and stores the new parameters into every rank's arena; a done flag per rank
 * closes the step. Deterministic; parameters stay bitwise identical across ranks.
 * The Adam moments become sharded (rank r updates m, v of its shard only); every call that
 * needs whole moments first gathers the peers' shards over peer memory, stream-ordered:
 * hg_opt_state_get, hg_step, hg_profile_step and hg_p2p_open(x, NULL) (which returns this
 * ctx to the NCCL exchange; captured graphs are rebuilt on their next use). Such calls are
 * collective: every rank makes them at the same point of its step sequence. The eager
 * hg_train_step(graph = 0) returns HG_E_STATE while the peer-memory exchange is on.
 * Every flag wait is bounded by hg_set_timeout (a dead peer traps the step: HG_E_CUDA). */
#define HG_P2P_HANDLE_BYTES 72
hg_status hg_p2p_handle(hg_ctx *x, void *out);
hg_status hg_p2p_open(hg_ctx *x, const void *all);

/* Validation entry for the peer-memory exchange on ONE device: world (2..8) contexts of one
 * process and one configuration act as the ranks. After every context ran its backward,
 * the exchange kernels of every rank (the same k_p2p_signal / k_p2p_adamw as
 * hg_p2p_open's captured step) run back to back on ctxs[0]'s stream with the flag waits
 * elided (ranks that spin on one another must not share a GPU, B200_PROFILING.md), then
 * synchronise. Afterwards the contexts are ranks 0..world-1 with sharded moments (see above).
 * HG_E_STATE if a context holds a communicator. */
hg_status hg_p2p_emulate(hg_ctx *const *ctxs, int32_t world, const hg_adamw *h);

/* Measurement: run this ctx's gradient exchange alone `iters` times back to back on the
 * compute stream (peer-memory reduce + AdamW + all-gather when hg_p2p_open is on, else the
 * NCCL average of the whole arena) and return the mean device milliseconds per exchange.
 * Collective (every rank calls it); the peer-memory variant applies AdamW to the current
 * gradients, so it advances the optimizer state. HG_E_STATE without an exchange. */
hg_status hg_exchange_time(hg_ctx *x, const hg_adamw *h, int32_t iters, float *ms);

/* Fail-stop bound, seconds (0 = none, the default): every device
 * flag wait of the peer-memory exchange traps past it (the step then fails with HG_E_CUDA),
 * and hg_sync returns HG_E_NCCL after aborting the NCCL communicator when its streams have
 * not drained within it. Captured graphs are rebuilt on their next use. */
hg_status hg_set_timeout(hg_ctx *x, double seconds);

/* Fused AdamW over the whole parameter arena. */
hg_status hg_step(hg_ctx *x, const hg_adamw *h);

/* forward + backward + allreduce + AdamW in one call; the device work is
 * captured once per slot into a CUDA graph and replayed (graph == 0 disables). */
hg_status hg_train_step(hg_ctx *x, int32_t slot, const hg_adamw *h, int32_t graph);

/* Capture (without running) the CUDA graph hg_train_step replays for `slot`. */
hg_status hg_capture_step(hg_ctx *x, int32_t slot, const hg_adamw *h);

/* Instrumented step: forward + backward + allreduce + AdamW captured on ONE
 * stream (no side-stream overlap) with CUDA timing events around every kernel
 * class, replayed once as a graph; returns, per phase, the summed device
 * milliseconds (ms[HG_PHASE_COUNT]) and kernel launches (launches[HG_PHASE_COUNT],
 * nullable). Advances the training state like hg_train_step. Synchronises.
 * HG_PHASE_SCALERS covers the degree sort, scalers and the degree-class weight
 * preparation; HG_PHASE_DMX also covers the dM_e reduction.
 * (SPEC.md:429-432 PhaseTimings) */
enum {
  HG_PHASE_SCALERS = 0, HG_PHASE_PROJ = 1, HG_PHASE_AGG_FWD = 2, HG_PHASE_UPDATE = 3, HG_PHASE_HEAD_FWD = 4,
  HG_PHASE_HEAD_BWD = 5, HG_PHASE_DA = 6, HG_PHASE_DU = 7, HG_PHASE_AGG_BWD = 8, HG_PHASE_DMX = 9,
  HG_PHASE_DX = 10, HG_PHASE_ALLREDUCE = 11, HG_PHASE_ADAMW = 12, HG_PHASE_COUNT = 13
};
hg_status hg_profile_step(hg_ctx *x, int32_t slot, const hg_adamw *h, float *ms, int64_t *launches);

/* ---- On-disk packed container with subfiles: the ADIOS
 * stand-in of PAPER.md:183-192 — the Table-1 variables as
 * global arrays with per-graph offsets, split over `n_subfiles` files that hold
 * contiguous graph ranges ("control the number of subfiles").
 * Format (little-endian, version 1): `dir`/meta.idx = header {"HGPK", version,
 * G, N, E, F0, Fe, n_sub}, node_offset[G+1], edge_offset[G+1] (int64),
 * sub_graph[n_sub+1], CRC-32C; `dir`/data.<k> = header {"HGPD", version, global
 * graph/node/edge ranges} then x, src, dst, edge_attr, y blocks each followed by
 * its CRC-32C. The index is written last.
 * hg_container_write: writes the store (threads: one per subfile). Creates `dir`
 *   if needed and overwrites its files. HG_E_IO on any write failure.
 * hg_container_open: reads every subfile straight into owned global arrays
 *   (parallel), validates CRCs and index consistency (HG_E_IO: missing subfile,
 *   bad magic/version, truncation, checksum), then validates the graphs exactly
 *   like hg_store_create; the returned store owns its memory (hg_store_destroy).
 * hg_container_info: header counts only (no data read).
 * hg_objfiles_write / hg_objfiles_open: the comparison backend of PAPER.md:341-347
 *   (one object file per graph, `dir`/g<id>.obj), same store result. */
hg_status hg_container_write(const hg_store *s, const char *dir, int32_t n_subfiles, int32_t threads);
hg_status hg_container_open(const char *dir, int32_t threads, hg_store **out);
hg_status hg_container_info(const char *dir, int64_t *graphs, int64_t *nodes, int64_t *edges, int32_t *subfiles);
hg_status hg_objfiles_write(const hg_store *s, const char *dir, int32_t threads);
hg_status hg_objfiles_open(const char *dir, int64_t num_graphs, int32_t threads, hg_store **out);

/* ---- Forward-only evaluation (SPEC.md:385-389 `evaluate`;
 * PAPER.md:377-381 reports MAE). hg_eval_reset zeroes the device accumulators;
 * hg_eval_batch runs the forward of the batch in `slot` (graph != 0: captured
 * once per slot and replayed) and adds sum (yhat-y)^2, sum |yhat-y| and the
 * graph count to fp64 device accumulators in a fixed order (deterministic);
 * hg_eval_result synchronises and returns MSE = sum sq / n, MAE = sum abs / n
 * over every graph since the reset (HG_E_EMPTY if none). hg_eval_pairs copies
 * the (y, yhat) parity pairs of the last forward of `slot` to caller host
 * buffers of capacity `cap` (HG_E_CAPACITY if the batch is larger), *n = B.
 * Parameters are not modified. */
hg_status hg_eval_reset(hg_ctx *x);
hg_status hg_eval_batch(hg_ctx *x, int32_t slot, int32_t graph);
hg_status hg_eval_result(hg_ctx *x, double *mse, double *mae, int64_t *count);
hg_status hg_eval_pairs(hg_ctx *x, int32_t slot, float *y, float *yhat, int32_t cap, int32_t *n);

/* Read the loss of the last forward (synchronises the compute stream). */
hg_status hg_loss_get(hg_ctx *x, float *loss);
/* Pipelined loss read-back: hg_loss_enqueue copies the loss of the last enqueued
 * forward into entry `i` (0 <= i < HG_LOSS_RING) of a pinned host ring owned by
 * the ctx, on the compute stream, without synchronising; hg_loss_fetch waits for
 * that copy only and returns the value. Lets a training loop read step k's loss
 * after step k+1 has been launched. HG_E_RANGE for a bad index. */
#define HG_LOSS_RING 4
hg_status hg_loss_enqueue(hg_ctx *x, int32_t i);
hg_status hg_loss_fetch(hg_ctx *x, int32_t i, float *loss);
/* Synchronise the ctx's streams; surfaces sticky CUDA/NCCL errors. Polls NCCL's async error
 * while waiting: an NCCL failure, a CUDA fault or the hg_set_timeout bound aborts the
 * communicator and makes the ctx unusable (fail-stop). */
hg_status hg_sync(hg_ctx *x);
/* Number of kernels this ctx has launched (graph replays count their kernel nodes). */
hg_status hg_launch_count(const hg_ctx *x, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* HGNN_H */
