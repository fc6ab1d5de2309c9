/* sidp.h — C ABI of the B200-native SiDP decode hot path (libsidp.so).
 *
 * SiDP ("Memory-Efficient Data Parallelism for Offline LLM Inference", PAPER.md): inside a
 * data-parallel group of d GPUs every transformer layer's pooled weights are owned by exactly
 * one rank (§4.2); other ranks either stream the layer over NVLink into a small
 * HBM cache ring (Weight-as-a-Service, WaS) or ship activations to the owner
 * (Compute-as-a-Service, CaS).  Both modes compute exactly what replicated
 * DP computes.
 *
 * Conventions (all functions):
 *  - Every pointer argument is a plain host or device pointer as documented per argument;
 *    no framework types cross this boundary.  Streams are cudaStream_t passed as void*.
 *  - All device work is enqueued asynchronously on the caller's stream (plus the library's
 *    internal fetch stream for WaS).  Nothing blocks the host except sidp_alloc, the
 *    synthetic init helpers' error checks, sidp_import_handles and sidp_destroy.
 *  - Return value: SIDP_OK or a negative sidp_status; nothing throws across the ABI.
 *    SIDP_EINVAL means no work was enqueued.  CUDA failures are sticky (SIDP_ECUDA for the
 *    rest of the context's life).  sidp_last_error() gives a thread-local message.
 *  - Ownership: the library owns what it allocates (owned-weight arena, cache slots, CaS
 *    staging/flags, workspaces, peer mappings, schedule tables) and frees it in
 *    sidp_destroy.  The caller owns activations, KV caches, token/position buffers.
 *  - One host thread per context; a context is not thread-safe.
 */
#ifndef SIDP_H_
#define SIDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sidp_ctx sidp_ctx; /* opaque, owned by the library */

typedef enum {
  SIDP_OK = 0,
  SIDP_EINVAL = -1,   /* bad argument; nothing enqueued */
  SIDP_ECUDA = -2,    /* CUDA runtime/driver error (sticky) */
  SIDP_ENOMEM = -3,   /* device allocation failed */
  SIDP_ESTATE = -4,   /* call out of protocol order (e.g. layer order, not allocated) */
  SIDP_EPEER = -5,    /* peer handle import failed */
  SIDP_ETIMEOUT = -6  /* a device-side flag wait timed out (CaS peer did not arrive) */
} sidp_status;

typedef enum {
  SIDP_WAS = 0,        /* Weight-as-a-Service: stream remote layers into the cache ring */
  SIDP_CAS = 1,        /* Compute-as-a-Service: ship activations to the owner */
  SIDP_REPLICATED = 2  /* baseline: every layer local (requires world == 1) */
} sidp_mode;

typedef enum {
  SIDP_ORDER_EXEC = 0,  /* remote layers in execution order (+ C-S7 stagger); any S >= 1 */
  SIDP_ORDER_PAPER = 1  /* peak-shifting cycles of PAPER.md:200; requires S >= d-1 */
} sidp_order;

typedef enum {
  SIDP_POOL_LAYER = 0,  /* pool QKV, O, gate/up, down (north_star; per-GPU ~W/d) */
  SIDP_POOL_FFN = 1     /* pool gate/up/down only, attention replicated */
} sidp_pool;

typedef enum {
  SIDP_FETCH_SM = 0,    /* hand-written K1 (TMA bulk copies through shared memory, CTA pairs) over
                           peer memory; device epoch flags per slot; the compute kernels size
                           their grids for the SMs the fetch does not hold */
  SIDP_FETCH_CE = 1     /* copy-engine cudaMemcpyAsync + CUDA events (the paper's mechanism,
                           PAPER.md:236-237; baseline) */
} sidp_fetch_engine;

/* Decoder model dimensions (HF-Llama block; Qwen3 qk_norm and Qwen2.5 QKV-bias variants).
 * Constraints: hidden, intermediate, n_q_heads*head_dim multiples of 64; head_dim 64 or 128;
 * n_q_heads % n_kv_heads == 0 and n_q_heads/n_kv_heads <= 16. */
typedef struct {
  int32_t num_layers, hidden, n_q_heads, n_kv_heads, head_dim, intermediate, vocab;
  int32_t qkv_bias; /* 0/1 */
  int32_t qk_norm;  /* 0/1 */
  float rms_eps, rope_theta;
} sidp_model_desc;

/* Group / runtime configuration.  PAPER.md:164 (init: assign owners, load only owned
 * weights, register buffers and export handles), PAPER.md:238 (slot budgets). */
typedef struct {
  int32_t rank, world;          /* this rank r in [0, d), d = DP group size */
  const int32_t* layer_owner;   /* host int32[num_layers], each in [0, world); NULL => l % world
                                   (exactly one owner per layer) */
  int32_t was_slots;            /* S >= 1 cache slots (north_star default 2; paper d-1) */
  int32_t cas_slots;            /* CaS staging buffers >= 1 (2) */
  int32_t order;                /* sidp_order */
  int32_t pool_scope;           /* sidp_pool */
  int32_t max_batch;            /* max rows per rank per step */
  int32_t max_ctx;              /* KV positions per sequence; a step needs pos + 1 <= max_ctx */
  int32_t fetch_sms;            /* SMs (CTAs, rounded to CTA pairs) the SM fetch kernel holds
                                   (0 => 24: one bulk-copy CTA moves ~50 GB/s (its SM's TMA unit
                                   carries both the load and the store of every chunk), so 24 keep
                                   NVLink 5's ~770 GB/s reader rate with headroom under a loaded
                                   HBM); the WaS compute kernels then use the remaining SMs.  Ignored by SIDP_FETCH_CE and when d == 1 */
  int32_t fetch_engine;         /* sidp_fetch_engine */
  int32_t stagger;              /* 1 => C-S7 start offsets t_r = (-r) mod (d-1) fetch ticks */
  int32_t device;               /* CUDA device ordinal the context lives on */
  uint64_t seed;                /* seed of the synthetic (counter-hash) weights, K12 */
  float fetch_pace_gbps;        /* > 0: the SM fetch kernel paces itself to at most this rate
                                   (GB/s).  Only for emulating NVLink with local-HBM owners on
                                   one GPU (bench.py --emulate-world); 0 on real NVLink, which
                                   caps the rate by itself. */
  int32_t compute_sms;          /* SMs the compute grids are sized for: 0 = automatic (all SMs,
                                   minus fetch_sms while an SM-fetch WaS ring is active); > 0 =
                                   explicit (e.g. a replicated baseline sized like a WaS rank,
                                   so both run bitwise-identical kernels) */
  int32_t slot_parts;           /* WaS cache granularity ("tensor
                                   tiles"): 1 = whole layers (a slot is filled, made ready and
                                   released as one unit); 2 = tiles: each pooled component (W_qkv,
                                   W_o, W_gate/up, W_down; FFN scope W_gate/up, W_down) of a slot has
                                   its own fill / ready / release flags, so a GEMM starts once its
                                   own weights have landed and the next layer's component refills
                                   as soon as this layer's GEMM released it — which makes a single
                                   slot (was_slots = 1, about one layer of memory) pipeline;
                                   0 = 1.  Tiles need the SM fetch (SIDP_FETCH_SM) and
                                   was_slots x parts <= 16 (else SIDP_EINVAL at sidp_alloc), and one
                                   computing context per GPU (its fetch is one windowed launch
                                   whose CTAs gate each part in-kernel; else SIDP_ESTATE at the
                                   step). */
  float fetch_ce_share;         /* hybrid WaS fetch (SIDP_FETCH_SM, whole-layer slots): this share of
                                   each layer (a prefix, in 32 KB chunks) is copied by the copy
                                   engine on its own stream, the rest by the SM fetch kernel; both
                                   count into the same fill epoch and whichever completes it
                                   publishes.  An SM reads ~50 GB/s, so moving part of
                                   the layer to the copy engine lets fewer fetch SMs hold the link
                                   rate at compute-bound batches.  [0, 1); 0 = SM fetch only. */
} sidp_config;

/* Caller-owned KV cache of this rank (never pooled).
 * Contiguous (block_table == NULL): k_cache / v_cache device bf16
 *   [num_layers][max_batch][n_kv_heads][max_ctx][head_dim].
 * Paged (block_table != NULL; the serving engines' block layout): k_cache /
 *   v_cache are block pools, device bf16 [num_layers][num_blocks][n_kv_heads][16][head_dim], and
 *   block_table is device int32 [max_batch][max_blocks]: token t of row b lives in pool block
 *   block_table[b][t / 16] at slot t % 16.  block_tokens must be 16 (the attention chunk);
 *   max_blocks * 16 >= max_ctx; every entry the step reads (t <= pos[b]) must be a valid block
 *   < num_blocks, owned by that row alone.  The table may change between steps (graph replays
 *   read it on the device); SIDP_EINVAL on bad sizes.
 * pos: device int32[batch], tokens already cached per row; the step writes the new k/v at
 * position pos[b] and attends over [0, pos[b]].  max_pos: host hint >= max_b pos[b]. */
typedef struct {
  void* k_cache;
  void* v_cache;
  const int32_t* pos;
  int32_t max_pos;
  const int32_t* block_table;   /* NULL: contiguous layout */
  int32_t block_tokens;         /* 16 when paged */
  int32_t max_blocks;           /* block_table row stride */
  int32_t num_blocks;           /* pool blocks per layer */
} sidp_kv;

/* One decode step of this rank. tokens/next: device int32[batch].  batch == 0 marks a
 * dummy step: no data movement and no compute in CaS; the owner still
 * serves peers.  logits (optional): device fp32 [batch][vocab].  layer_inputs (optional):
 * device bf16 [num_layers][batch][hidden], receives each layer's input x (teacher-forcing
 * parity dumps). */
typedef struct {
  const int32_t* tokens;
  int32_t* next;        /* may alias tokens (written after the last read of tokens) */
  int32_t batch;
  sidp_kv kv;
  float* logits;
  void* layer_inputs;
  int32_t* pos_out;     /* optional device int32[batch]: receives pos[b] + 1 at the end of
                           the step (may alias kv.pos) — a decode loop needs no other kernel */
} sidp_batch;

typedef struct {
  uint64_t steps;           /* completed sidp_step calls */
  uint64_t fetches;         /* remote-layer fetches enqueued */
  uint64_t bytes_fetched;   /* verbatim bytes copied into slots */
  uint64_t launches;        /* device kernels (and copy-engine copies) enqueued */
  uint64_t cas_round_trips; /* CaS round trips this rank took part in */
  int32_t mode;             /* current sidp_mode */
  int32_t timeouts;         /* device flag-wait timeouts observed */
  uint64_t layer_bytes;     /* pooled bytes of one layer (what one fetch moves) */
  uint64_t local_layer_bytes;  /* un-pooled per-layer bytes every rank keeps */
  uint64_t owned_bytes;     /* owned-weight arena */
  uint64_t slot_bytes;      /* S x layer_bytes */
  uint64_t replicated_bytes;   /* embedding + final norm + LM head + local layer parts */
  uint64_t workspace_bytes; /* activations, split-K / split-KV workspaces, staging */
  double timed_ms[8];       /* per kernel class: summed CUDA-event durations (sidp_set_timing) */
  uint64_t timed_launches[8];  /* per kernel class: timed launches */
  int32_t fetch_sms_held;   /* SMs the SM fetch kernel holds (0: copy engine, or no remote layer) */
  int32_t compute_sms;      /* SMs the WaS compute grids are sized for (0 = all) */
  double stagger_tick_ns;   /* measured single-reader layer fetch (C-S7 tick; 0 = not measured) */
  uint64_t graph_replays;   /* sidp_step calls that replayed a captured CUDA graph */
  uint64_t slot_checks;     /* debug SIDP_SLOT_VERIFY=1 (read at sidp_init): landed slots (or slot
                               parts) compared word for word with the owner's blob before the
                               layer's first reader */
  uint64_t slot_mismatches; /* differing 16-byte words found by those checks (0 = verbatim) */
} sidp_stats_t;

/* ---- lifecycle --------------------------------------------------------------------- */

/* Validate model + config, build the owner map, prefetch plan and FIFO slot recurrence
 * (host only; no device work, callable without a GPU).  SIDP_EINVAL on: bad dims, rank not
 * in [0, world), owner not in [0, world), was_slots < 1, SIDP_ORDER_PAPER with
 * was_slots < world-1 (deadlock), max_batch/max_ctx < 1.
 * *out receives a context owned by the library (free with sidp_destroy). */
sidp_status sidp_init(const sidp_model_desc* model, const sidp_config* cfg, sidp_ctx** out);

/* Allocate device state on cfg->device: owned-weight arena (owned layers only; non-owned
 * layers get no memory — the paper's "placeholders"), S cache slots,
 * replicated tensors, CaS staging + flags, workspaces, the fetch stream and events. */
sidp_status sidp_alloc(sidp_ctx* ctx);

/* Bytes of the owned-weight arena this context lays out (its owned layers' pooled blobs,
 * contiguous; "each GPU holds only its own layers"): what sidp_alloc_owned needs.
 * Host-only; valid after sidp_init. */
sidp_status sidp_owned_bytes(const sidp_ctx* ctx, uint64_t* bytes);

/* sidp_alloc with a CALLER-OWNED owned-weight arena (SURVEY.md §8(b) sidp_alloc_owned; e.g. a
 * torch allocation): arena is device memory on the context's device, >= sidp_owned_bytes bytes,
 * 256-byte aligned.  The library lays the owned layers out in it (sidp_init_weights_synthetic
 * fills them), never frees it, and exports it to peers as its allocation's IPC handle plus the
 * arena's offset inside that allocation, so an arena carved from a larger (caching-allocator)
 * segment works — so it must be cudaMalloc-backed (torch's default caching allocator; not a
 * cuMemCreate / expandable-segments allocation, which has no legacy IPC handle: peers then fail
 * sidp_import_handles with SIDP_EPEER).  The caller keeps it alive and unmodified until
 * sidp_destroy.  Everything else
 * (local layers, slots, workspaces, CaS staging) is allocated as by sidp_alloc.  SIDP_EINVAL
 * (nothing allocated) if the arena is too small, misaligned or not device memory of the
 * context's device; otherwise as sidp_alloc. */
sidp_status sidp_alloc_owned(sidp_ctx* ctx, void* arena, uint64_t bytes);

/* Alternative to sidp_alloc for a serve-only rank: allocate only the owned-weight arena (and a
 * CaS flag block so the exported blob is well formed; no local per-layer parts).
 * The rank owns, initialises (sidp_init_weights_synthetic fills only its owned and local
 * parts) and exports its layers for WaS peers to fetch ("each GPU ... serves its
 * layers to peers"), but never computes: sidp_step / sidp_decode_layer return SIDP_ESTATE and
 * it cannot serve CaS.  Used to emulate the d-1 owners of a DP group beside one computing rank
 * on a single GPU (bench.py --emulate-world).  SIDP_ESTATE if already allocated, SIDP_ENOMEM
 * on allocation failure (nothing left allocated is leaked: sidp_destroy frees it). */
sidp_status sidp_alloc_serve_only(sidp_ctx* ctx);

/* TIMING EMULATION ONLY.  A serve-only context whose owned arena IS `donor`'s (same device, same
 * pooled layout, donor owns at least as many layers): d-1 emulated owners of a big model then
 * cost one arena of HBM, which frees the memory for the KV cache of the configured point (M3:
 * Llama-3.1-70B at B_e ~ 1536 with max KV).  The fetched bytes, their sizes and the schedule are
 * a real rank's, but a slot then holds the donor's layer values, so the results are NOT the
 * model's: never used by a parity test.  sidp_init_weights_synthetic is a no-op on it; destroy
 * leaves the donor's arena alone (destroy the donor last).  SIDP_EINVAL: null donor or a
 * mismatching layout. */
sidp_status sidp_alloc_serve_only_alias(sidp_ctx* ctx, const sidp_ctx* donor);

/* K12: fill owned layers, local layer parts and replicated tensors with the counter-hash
 * synthetic values (same function as sidp_inputs/gen.py), on `stream`. */
sidp_status sidp_init_weights_synthetic(sidp_ctx* ctx, void* stream);

/* Export this rank's owned arena / staging / flag handles into blob (host buffer of
 * *len bytes; on return *len = bytes written; pass blob = NULL to query the size). */
sidp_status sidp_export_handles(sidp_ctx* ctx, void* blob, size_t* len);

/* Import all ranks' blobs (host pointers, rank order, world entries; this rank's own entry
 * is ignored).  Same-process blobs map directly; others via CUDA IPC (peer access enabled).
 * SIDP_EPEER if a handle cannot be opened. */
sidp_status sidp_import_handles(sidp_ctx* ctx, const void* const* blobs, const size_t* lens);

void sidp_destroy(sidp_ctx* ctx);

/* ---- the hot path ------------------------------------------------------------------- */

/* One decoder layer on x (device bf16 [batch][hidden], in/out), §4.2 / §4.3:
 * RMSNorm -> QKV (+bias) -> (qk-norm) RoPE, KV append -> GQA attention -> O + residual ->
 * RMSNorm -> gate/up + SiLU*mul -> down + residual.
 *  mode SIDP_WAS: an owned layer runs from the arena; a remote layer waits for its slot
 *    (filled by the fetch stream in plan order) and frees it after the down GEMM.  Layers
 *    must be called in execution order (0..L-1, step after step): else SIDP_ESTATE.
 *  mode SIDP_CAS: collective per layer — every rank of the group calls it for every layer
 *    in order; batch == 0 (dummy) returns after serving peers if this rank owns the layer.
 *  mode SIDP_REPLICATED: world == 1 only.
 * batch > max_batch, layer out of range, or pos out of range => SIDP_EINVAL.
 * A CaS flag wait that exceeds the timeout (20 s; SIDP_CAS_TIMEOUT_MS read at sidp_init) writes
 * a mapped host word: every later call on this context returns SIDP_ETIMEOUT (sticky) and
 * sidp_stats reports it in `timeouts`. */
sidp_status sidp_decode_layer(sidp_ctx* ctx, void* x, int32_t batch, int32_t layer,
                              int32_t mode, const sidp_kv* kv, void* stream);

/* One full decode step: embedding gather -> L layers in the current
 * mode -> final RMSNorm -> LM head GEMM with fused argmax (ties -> lowest index). */
sidp_status sidp_step(sidp_ctx* ctx, const sidp_batch* batch, void* stream);

/* Globally consistent mode directive: must be called with identical
 * arguments on every rank.  Takes effect at the start of step `effective_step`
 * (0-based count of sidp_step calls).  Switching drains the WaS ring and resets the plan. */
sidp_status sidp_set_mode(sidp_ctx* ctx, int32_t mode, int64_t effective_step);

/* Control plane for CaS: per-rank rows of the coming step (host int32[world], identical on
 * all ranks; 0 = dummy).  Sets the fused-GEMM offsets (exclusive prefix sums). */
sidp_status sidp_set_batches(sidp_ctx* ctx, const int32_t* batches);

/* ---- introspection (host only; no GPU needed) ------------------------------------------ */

sidp_status sidp_owner_of(const sidp_ctx* ctx, int32_t layer, int32_t* owner);

/* This rank's per-pass prefetch plan (layers in fetch order). */
sidp_status sidp_get_plan(const sidp_ctx* ctx, int32_t* layers, int32_t capacity, int32_t* n);

/* The (step, layer, slot) fetch schedule of the first `steps` passes from the FIFO
 * free-list recurrence — compared bit-exactly with the oracle. */
sidp_status sidp_get_schedule(const sidp_ctx* ctx, int32_t steps, int32_t* fetch_step,
                              int32_t* fetch_layer, int32_t* fetch_slot, int32_t capacity,
                              int32_t* n);

/* Fetch-tick offset of this rank's fetch stream (C-S7 stagger). */
sidp_status sidp_stagger_ticks(const sidp_ctx* ctx, int32_t* ticks);

/* The fetches performed since the last reset of the plan, as (step, layer, slot).
 * SIDP_FETCH_SM: read back from the device log that the fetch kernel's publishing CTA appends
 * to (the layer id and slot it actually copied; the last 4096 entries); synchronises the fetch
 * stream.  SIDP_FETCH_CE: the host's enqueue log (the copy engine writes no log).
 * fetch_step == NULL: *n = count only; else capacity must be >= the count (SIDP_EINVAL). */
sidp_status sidp_get_fetch_log(const sidp_ctx* ctx, int32_t* fetch_step, int32_t* fetch_layer,
                               int32_t* fetch_slot, int32_t capacity, int32_t* n);

/* SIDP_FETCH_SM only (else *n = 0): the device fetch log with timing — int64 [n][7] =
 * {fetch index j, layer, slot, owner rank, fill epoch of the slot, %globaltimer ns of the first
 * fetch CTA's start, %globaltimer ns of the publish}.  Per-owner reader traces (C-S7) and the
 * achieved per-fetch GB/s come from it.  Synchronises the fetch stream. */
sidp_status sidp_get_fetch_trace(const sidp_ctx* ctx, int64_t* out, int32_t capacity, int32_t* n);

/* SIDP_FETCH_SM only (else *n = 0): the compute side's device log of slot consumptions —
 * int64 [n][5] = {layer expected, slot, layer tag found in the slot, consumption epoch,
 * %globaltimer ns when the weights were ready}.  A tag != layer also raises the sticky error
 * word (protocol violation).  Synchronises the device. */
sidp_status sidp_get_consume_log(const sidp_ctx* ctx, int64_t* out, int32_t capacity, int32_t* n);

sidp_status sidp_stats(const sidp_ctx* ctx, sidp_stats_t* out);

/* Time every launch of the kernel classes in `class_mask` (bit c = class c) with CUDA events
 * on the stream each launch goes to: 1 gate/up GEMM, 2 attention, 3 fetch, 4 down GEMM,
 * 5 QKV GEMM, 6 O GEMM, 7 LM head (0 = off).  Resets the accumulators;
 * sidp_stats().timed_ms[c] sums them (that read synchronises on the recorded events). */
sidp_status sidp_set_timing(sidp_ctx* ctx, int32_t class_mask);

const char* sidp_last_error(void);

/* ---- test hooks (parity tests of single kernels; same kernels as the hot path) ---------- */

/* tcgen05 GEMM: out = epilogue(x[M,K] . w[N,K]^T).  epi: 0 fp32, 1 bf16, 2 bf16 + resid,
 * 3 SiLU(gate)*up over 16-row [gate 8 | up 8] groups, 4 fused argmax (u64 packed; call
 * with out zeroed).  k_splits 0 = auto, 1 = whole tiles, >1 = forced stream-K, -1 = token-major
 * orientation (X as the UMMA A operand; not for epilogue 5).  Device pointers; enqueued on stream. */
sidp_status sidp_test_gemm(const void* x, int32_t ldx, const void* w, int32_t ldw, int32_t M,
                           int32_t N, int32_t K, int32_t epi, void* out, int32_t ldo,
                           const void* resid, int32_t ldr, const void* bias, int32_t k_splits,
                           void* stream);

/* Test hook for the fused QKV GEMM (PAPER.md:163 — the KV cache is local):
 * Y = X W^T (+ bias) with X [M,K] (row stride ldx) and W [N = (nq + 2 nkv) hd, K] bf16
 * row-major; per token m and head: q/k heads get the per-head RMSNorm (gains gq / gk, null =
 * off; Qwen3 qk_norm) and rotate-half RoPE with rope[pos[m]] ((cos, sin) fp32 pairs [.][hd/2]),
 * then q -> q[m][head][hd] bf16, k / v -> kc / vc[(m nkv + g) smax + pos[m]][hd] bf16.
 * k_splits 0 = the runtime's choice (token-major head tiles with an in-kernel stream-K fix-up
 * from M >= 128, else W-major whole tiles), 1 = W-major whole tiles.  hd 64 or 128.  SIDP_EINVAL
 * on bad shapes.  Device pointers; enqueued on stream. */
sidp_status sidp_test_gemm_qkv(const void* x, int32_t ldx, const void* w, int32_t M, int32_t K,
                               const void* bias, int32_t nq, int32_t nkv, int32_t hd,
                               const void* gq, const void* gk, float eps, const void* rope,
                               const int32_t* pos, void* q, void* kc, void* vc, int32_t smax,
                               int32_t k_splits, void* stream);

/* Test hook for the deferred stream-K fix-up (SURVEY.md a8+a9, a11+a5): the EPI_PARTIAL GEMM
 * Y = X W^T (X [M,K] row stride ldx, W [N,K] contiguous, bf16) leaves fp32 k-range partials
 * that resid_norm sums in slice order: xout = bf16(Y + resid) ([M,N], resid row stride ldr,
 * may alias xout) and u = bf16(xout * rsqrt(mean(xout^2) + eps) * g) ([M,N]).  SIDP_EINVAL
 * (nothing enqueued) if the shape fills the machine with whole tiles or its slices exceed the
 * hook's 256 MB workspace.  Device pointers; enqueued on stream. */
sidp_status sidp_test_gemm_resid_norm(const void* x, int32_t ldx, const void* w, int32_t M,
                                      int32_t N, int32_t K, const void* resid, int32_t ldr,
                                      const void* g, float eps, void* xout, void* u, void* stream);

/* Test hook for the fused gate/up -> down launch (SURVEY.md a10 + a11 + next a5): act =
 * SiLU(u Wg^T) * (u Wu^T) (wgu [2I][h], gate/up rows interleaved in 16-row groups), then the down
 * projection's partial slices summed by resid_norm: xout = bf16(resid + act Wd^T) (wd [h][I]) and
 * unorm = RMSNorm(xout) * g.  u, resid, xout, unorm [M][h], act [M][I], all contiguous bf16.
 * SIDP_EINVAL (nothing enqueued) if M > 256, h % 256 or I % 128.  Device pointers. */
sidp_status sidp_test_mlp_fused(const void* u, const void* wgu, const void* wd, const void* resid,
                                int32_t M, int32_t h, int32_t I, const void* g, float eps,
                                void* act, void* xout, void* unorm, void* stream);

/* Host-only (no GPU): the fused MLP's list schedule for G gate/up tiles of nks1 k-steps and D
 * down tiles of nks2 k-steps, MT token tiles of 256 rows, over C CTA pairs, down split into
 * <= max_seg chunks per (tile, token tile).  units: int32 [cap][4] = {phase | seg << 8 |
 * mt << 16, tile, kb0, kb1}; off [C + 1] (pair c owns units [off[c], off[c+1])); nseg [D * MT]
 * (index tile * MT + mt); *n_units = count.  SIDP_EINVAL on bad arguments or cap too small. */
sidp_status sidp_test_mlp_schedule(int32_t G, int32_t nks1, int32_t D, int32_t nks2, int32_t C,
                                   int32_t max_seg, int32_t MT, int32_t* units, int32_t cap,
                                   int32_t* off, int32_t* nseg, int32_t* n_units);

/* K12 on an arbitrary buffer: dst[r*ld + c] = value(seed, tensor, layer, (row0+r)*lcols + c)
 * with kind 0 weight (scale from scale_k), 1 gain, 2 bias, 3 unit; row_map 1 = packed
 * gate/up interleave. */
sidp_status sidp_test_gen(void* dst, int64_t ld, int64_t rows, int64_t cols, uint64_t seed,
                          int32_t tensor, int32_t layer, int32_t kind, int32_t scale_k,
                          int64_t row0, int64_t lcols, int32_t row_map, void* stream);

/* K1 fetch of `bytes` (multiple of 16, 16-byte aligned pointers) from src (local or peer VA) to
 * dst: engine 0 = the TMA bulk-copy kernel on `ctas` CTAs (rounded to CTA pairs) with a static
 * chunk split, 1 = the copy engine (cudaMemcpyAsync), 2 = the vectorised LDG/STG copy kernel
 * (round-1 design, kept for A/B), 3 = the same kernel exactly as the WaS ring runs it (chunks
 * claimed in groups, completion published to a scratch ring; no gates) — for ncu.  Device
 * pointers; enqueued on stream; no flag of any context is posted. */
sidp_status sidp_test_fetch(void* dst, const void* src, size_t bytes, int32_t ctas, int32_t engine,
                            void* stream);

/* Synthetic KV cache fill: cache[b][g][t][d] (b < B, t < T) from logical b_global = b0 + b. */
sidp_status sidp_test_gen_kv(void* cache, int32_t B, int32_t nkv, int32_t smax, int32_t hd,
                             int32_t T, int64_t b0, uint64_t seed, int32_t tensor, int32_t layer,
                             void* stream);

/* Copy this rank's CaS flag words (arrive[world], done, served) to host out[n] (debugging). */
sidp_status sidp_debug_flags(const sidp_ctx* ctx, uint64_t* out, int32_t n);

/* Pointer to layer `layer`'s pooled blob as resident on this rank (owned arena, else NULL)
 * and the byte offsets of its components. */
sidp_status sidp_layer_ptr(const sidp_ctx* ctx, int32_t layer, void** pooled, void** local);

#ifdef __cplusplus
}
#endif

#endif /* SIDP_H_ */
