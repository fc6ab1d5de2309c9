// kernels.h — internal launchers of the SiDP device kernels (below the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace sidp {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------- tcgen05 decode GEMM
// Y[m, n] = sum_k X[m, k] * W[n, k]  (X [M,K] bf16 row-major, W [N,K] bf16 row-major)
// computed swap-AB: W tiles are the UMMA "A" operand (128 features per tile), the
// tokens are the UMMA "N" dimension, accumulators live in TMEM.
enum GemmEpilogue : int {
  EPI_F32 = 0,        // out fp32 = acc (+ bias)
  EPI_BF16 = 1,       // out bf16 = acc (+ bias)
  EPI_RESID = 2,      // out bf16 = acc + resid (bf16); out may alias resid
  EPI_SILU_MUL = 3,   // W rows interleaved in 16-row groups g: [gate 8g..8g+7 | up 8g..8g+7];
                      // out[m, f] bf16 = silu(gate f) * up f, f = 8g + i
  EPI_ARGMAX = 4,     // fused argmax over n: packed (value, lowest index) into out u64[M]
  EPI_QKV = 5,        // fused QKV post-processing: (+bias) (qk-norm) RoPE -> q bf16, k/v -> KV cache
  EPI_PARTIAL = 6,    // deferred reduction: stream-K over all CTA pairs, EVERY unit writes its fp32
                      // k-range partial to the workspace slice of its segment; no fix-up kernel —
                      // the consumer (resid_norm, qkv_post) sums the slices (see PartialSrc)
};

// Where an EPI_PARTIAL GEMM left Y: Y[m, n] = sum_{s < nseg(tile(m, n))} ws[s][m][n] in slice
// order (deterministic: depends only on the shapes and the launch's cluster count).  Tiles
// are (tile_m tokens x tile_f features); tile index t = sw ? (m / tile_m) * f_tiles + n / tile_f
// : (n / tile_f) * m_tiles + m / tile_m; the t-th tile covers k-steps [t nks, (t+1) nks) of
// the stream-K range split evenly over `clusters` CTA pairs.
constexpr int kPartialMaxTiles = 128;
struct PartialSrc {
  const float* ws;
  int M, N;
  int sw, tile_m, tile_f, m_tiles, f_tiles;
  int nks, clusters;
  long long total_kb;
  unsigned char nseg[kPartialMaxTiles];   // partial_nseg of every tile (tiles <= 128), host-built
};
__host__ __device__ inline int partial_cluster_of(long long g, long long total, int C) {
  return (int)(((g + 1) * (long long)C + total - 1) / total) - 1;
}
__host__ __device__ inline int partial_tile(const PartialSrc& p, int m, int n) {
  return p.sw ? (m / p.tile_m) * p.f_tiles + n / p.tile_f : (n / p.tile_f) * p.m_tiles + m / p.tile_m;
}
__host__ __device__ inline int partial_nseg(const PartialSrc& p, int m, int n) {
  const long long t = p.sw ? (long long)(m / p.tile_m) * p.f_tiles + n / p.tile_f
                           : (long long)(n / p.tile_f) * p.m_tiles + m / p.tile_m;
  return partial_cluster_of((t + 1) * p.nks - 1, p.total_kb, p.clusters) -
         partial_cluster_of(t * p.nks, p.total_kb, p.clusters) + 1;
}

// Paged KV (16-token blocks, sidp_kv.block_table): element offset of (row b, kv head g, token t)
// in a layer's cache — contiguous [B][nkv][smax][hd], or the block pool [nblk][nkv][16][hd].
constexpr int kKvBlock = 16;
__host__ __device__ inline size_t kv_off(const int32_t* bt, int bt_stride, int nkv, int smax,
                                         int hd, int b, int g, int t) {
  if (!bt) return (((size_t)b * nkv + g) * smax + t) * hd;
  const size_t blk = (size_t)bt[(size_t)b * bt_stride + t / kKvBlock];
  return ((blk * nkv + g) * kKvBlock + (t % kKvBlock)) * hd;
}

// Destination of the fused QKV epilogue (rows of W_qkv = [q heads | k heads | v heads]).
struct QkvEpi {
  bf16* q;                       // [M, nq, hd]
  bf16* kc; bf16* vc;            // this layer's caches [Bmax, nkv, smax, hd]
  const int32_t* pos;            // [M] position of the new token
  const float2* rope;            // [max_pos, hd/2] (cos, sin)
  const bf16* gq; const bf16* gk;   // qk-norm gains (null = off)
  float eps;
  int nq, nkv, hd, smax;
  const int32_t* bt; int bt_stride;   // paged KV (null: contiguous)
};

// A CaS flag wait folded into a consumer kernel's prologue (no standalone wait launch): the
// kernel's loads of the guarded data start once every *p[i] >= value (system-scope acquire);
// n == 0: no wait.  Timeout -> *err (mapped host word), surfaced as SIDP_ETIMEOUT.
struct FlagWait {
  const uint64_t* p[16];
  int n;
  uint64_t value;
  uint64_t timeout_ns;
  int* err;
  const uint64_t* base;        // optional: value is relative to *base (CaS graph replay)
};

// CaS owner: the GEMM's output rows scattered straight into the requesters'
// receive buffers — rows [row0[q], row0[q+1]) of the fused staging batch go to base[q] (a peer
// VA; row stride = the GEMM's ldo).  n == 0: plain output.
struct RowScatter {
  int n;
  int row0[17];
  void* base[16];
};

// Flags a grid posts once ALL its CTAs' stores are done (the last CTA to finish releases them at
// system scope): the CaS owner's done + served flags ride on its last GEMM instead of a launch.
struct PostFlags {
  uint64_t* flag[17];
  int n;
  uint64_t value;
  unsigned int* counter;       // last-CTA election (0 between launches)
  const uint64_t* base;        // optional: value is relative to *base
};

struct GemmArgs {
  const bf16* x; int ldx;      // [M, K]
  const bf16* w; int ldw;      // [N, K]
  int M, N, K;
  int epi;
  void* out; int ldo;
  const bf16* resid; int ldr;
  const bf16* bias;            // [N] or null
  int k_splits;                // 0 = auto, 1 = whole tiles, >1 stream-K, -1 = token-major (SW)
  int max_ctas;                // 0 = all SMs
  const QkvEpi* qkv;           // EPI_QKV only
  int w_kbmajor;               // 1: W is k-block-major [K/64][N][64] (one 3-D TMA box per stage)
  int x_kbmajor;               // 1: X is k-block-major [K/64][M][64] (layout experiment)
  PartialSrc* partial_out;     // EPI_PARTIAL: receives the slice geometry for the consumer
  const FlagWait* wait;        // optional: the activation loads wait for these flags (CaS owner)
  const RowScatter* scatter;   // optional (EPI_F32 / EPI_BF16 / EPI_RESID): output rows -> peers
  const PostFlags* post;       // optional: posted by the last CTA of the GEMM's last launch
};

struct GemmWorkspace {
  float* ws; size_t ws_bytes;  // split-K partials
  int* counters; int n_counters;
};

cudaError_t gemm_launch(const GemmArgs& a, const GemmWorkspace& w, cudaStream_t s);
// Grid-sizing SM budget of the persistent / one-wave compute kernels (GEMMs, fused MLP,
// attention) on this host thread: 0 = every SM of the device; n > 0 = the first n (even) — set
// by the runtime while a WaS fetch kernel holds dedicated SMs, so no compute CTA (pair) ever
// waits for an SM the fetch occupies.  SIDP_SM_BUDGET overrides the default 0.
void set_compute_sms(int n);
int get_compute_sms_budget();
int compute_sms();
int gemm_pick_splits(int tiles, int nkb, int sms);
// true when an EPI_PARTIAL launch of this shape is both possible (slices fit the workspace)
// and worthwhile (whole 256x256 tiles would leave CTA pairs idle, so the GEMM is stream-K
// anyway and the fix-up can move into the consumer)
bool gemm_partial_ok(int M, int N, int K, size_t ws_bytes);
int gemm_last_launch_count();   // kernels enqueued by the last gemm_launch on this thread

// Fused gate/up -> down (SURVEY.md a10 + a11) in one persistent tcgen05 launch: gate/up tiles
// (SiLU*mul -> act) and down k-range units (fp32 partial slices, summed by resid_norm in slice
// order) in host-scheduled per-pair lists; a down unit's act k-block is loaded once the gate/up
// tile producing it is stored (device tile counters in GemmWorkspace.counters).
struct MlpArgs {
  const bf16* u; int ldu;        // [M][h] gate/up input
  const bf16* wgu;               // [2I][h], gate/up rows interleaved in 16-row groups
  const bf16* wd;                // [h][I]
  bf16* act; int ldact;          // [M][I] SiLU(gate) * up
  int M, h, I;
  PartialSrc* partial_out;       // down partial slices for resid_norm
};
// max_tt: most 256-row token tiles allowed (0 = the runtime policy, SIDP_MLP_MAX_TT, default 1;
// the kernel supports 2).
bool mlp_fused_ok(int M, int h, int I, size_t ws_bytes, int n_counters, int max_tt = 0);
// true when an EPI_QKV launch of this shape takes the token-major head-tile path (qk-norm, RoPE
// and the KV append in the GEMM epilogue; stream-K with an in-kernel fix-up of split tiles)
bool gemm_qkv_sw_ok(int M, int N, int K, int hd, size_t ws_bytes, int n_counters);
void mlp_prepare(int h, int I, size_t ws_bytes);   // builds the schedule (call before capture)
// The host list schedule (no CUDA calls): per-pair unit lists {phase | seg << 8, tile, kb0, kb1}
// (flat, cluster c at [off[c], off[c+1])) and the down segments per tile.
void plan_mlp_units(int G, int nks1, int D, int nks2, int C, int max_seg, int MT,
                    std::vector<int4>& flat, std::vector<int>& off, std::vector<int>& nseg);
cudaError_t mlp_launch(const MlpArgs& a, const GemmWorkspace& w, cudaStream_t s);

// ---------------------------------------------------------------- element-wise / small kernels
cudaError_t rmsnorm_launch(const bf16* x, int ldx, const bf16* g, float eps, bf16* y, int ldy,
                           int rows, int h, cudaStream_t s);
// Deferred stream-K fix-up fused with the residual add and the next RMSNorm (SURVEY.md a8 + a9,
// a11 + next layer's a5): per row m, x_out = bf16(sum of the partial slices + resid) and
// u = bf16(x_out * rsqrt(mean(x_out^2) + eps) * g).  resid may alias x_out.  post (optional):
// a WaS slot's release counter, incremented (release) once the predecessor kernel completed.
cudaError_t resid_norm_launch(const PartialSrc& ps, const bf16* resid, int ldr, bf16* xout, int ldx,
                              const bf16* g, float eps, bf16* u, int ldu, int rows, int h,
                              cudaStream_t s, unsigned long long* post = nullptr);
cudaError_t embed_launch(const bf16* E, int h, const int32_t* tokens, bf16* x, int rows,
                         cudaStream_t s);
// CaS requester, round trip 1 (the send fused into the producing kernel):
// waits for the owner's previous round trip to be served (its staging slot is free), computes
// u = RMSNorm(x) g and stores [u | x] straight into the owner's staging rows (peer VA), then the
// last CTA posts the arrival flag (release, system scope).  One launch replaces rmsnorm + wait +
// transfer.
struct CasSendArgs {
  const bf16* x; int ldx;
  const bf16* g; float eps;
  int rows, h;
  bf16* dst; int ldd;          // owner staging rows, u -> cols [0, h), x -> cols [h, 2h)
  FlagWait wait;               // owner's previous round trip served
  uint64_t* arrive; uint64_t value;
  unsigned int* counter;       // last-CTA election (0 between launches)
  const uint64_t* base;        // optional: value (and wait.value via wait.base) relative to *base
};
cudaError_t cas_send_norm_launch(const CasSendArgs& a, cudaStream_t s);
// qkv fp32 [B, (nq+2nkv)*hd] -> q bf16 [B, nq, hd]; k, v appended to caches at pos[b]
struct QkvPostArgs {
  const float* qkv; int B, nq, nkv, hd;
  const bf16* gq; const bf16* gk; float eps;    // qk_norm gains (null = off)
  const float2* rope;                           // [max_pos, hd/2] (cos, sin)
  const int32_t* pos;
  bf16* q;
  bf16* kc; bf16* vc;                           // [Bmax, nkv, Smax, hd] (or block pools)
  int smax;
  const int32_t* bt; int bt_stride;             // paged KV: block table [B][bt_stride] (null: contiguous)
  PartialSrc part;                              // part.ws != null: qkv is the sum of these slices
  const bf16* bias;                             // added in the partial form only (else by the GEMM)
  int ldqkv;                                    // qkv row stride in floats (0 = (nq + 2 nkv) hd)
  FlagWait wait;                                // optional: qkv is read once these flags are set
};
cudaError_t qkv_post_launch(const QkvPostArgs& a, cudaStream_t s);

struct AttnArgs {
  const bf16* q;              // [B, nq, hd]
  const bf16* kc; const bf16* vc;   // [Bmax, nkv, Smax, hd]
  const int32_t* pos;         // attend over [0, pos_b]
  bf16* o;                    // [B, nq*hd], row stride ldo (0 = nq*hd; may be a peer VA)
  int ldo;
  int B, nq, nkv, hd, smax;
  const int32_t* bt; int bt_stride;   // paged KV: block table [B][bt_stride], 16-token blocks
  int max_tokens;             // host hint: max_b (pos_b + 1) <= smax (sizes the grid)
  float* ws; size_t ws_bytes; // partials of (b, g) pairs split across CTAs
  int* cnt; int n_cnt;        // [B * nkv] arrival counters, zero between launches
};
cudaError_t attention_launch(const AttnArgs& a, cudaStream_t s);
int attention_last_launch_count();

// next[b] = decoded argmax; if pos_out: pos_out[b] = pos[b] + 1 (may alias pos)
cudaError_t argmax_finalize_launch(const unsigned long long* packed, int32_t* next,
                                   int32_t* pos_out, const int32_t* pos, int rows, cudaStream_t s);
cudaError_t argmax_reset_launch(unsigned long long* packed, int rows, cudaStream_t s);

// ---------------------------------------------------------------- K12 synthetic init
// dst[i] = value(seed, tensor, layer, logical(i)) for a strided 2-D block of a logical
// [rows, cols] tensor: logical index = (row0 + r) * lcols + c; dst = base + r*ld + c.
enum GenKind : int { GEN_WEIGHT = 0, GEN_GAIN = 1, GEN_BIAS = 2, GEN_UNIT = 3 };
struct GenArgs {
  bf16* dst; int64_t ld;
  int64_t rows, cols;
  uint64_t seed; int tensor; int layer;
  int kind; int scale_k;          // GEN_WEIGHT scale from K = scale_k
  int64_t row0, lcols;            // logical row offset and logical row length
  int row_map;                    // 0: identity; 1: gate/up interleave (see init.cu)
  int inter;                      // intermediate size for row_map 1
};
cudaError_t gen_launch(const GenArgs& a, cudaStream_t s);
// KV cache: cache[b, g, t, d] for b < B, t < T (logical b_global = b0 + b)
cudaError_t gen_kv_launch(bf16* cache, int B, int nkv, int smax, int hd, int T, int64_t b0,
                          uint64_t seed, int tensor, int layer, cudaStream_t s);

// ---------------------------------------------------------------- WaS fetch
// Verbatim copy of one pooled layer, owner HBM (possibly a peer VA) -> local slot.
cudaError_t fetch_launch(void* dst, const void* src, size_t bytes, int ctas, cudaStream_t s,
                         float pace_gbps = 0.0f);
cudaError_t delay_launch(uint64_t ns, cudaStream_t s);
// copy-engine fetch pacing: first != 0 stamps *t0; else waits until *t0 + offset_ns
cudaError_t pace_launch(unsigned long long* t0, int first, uint64_t offset_ns, cudaStream_t s);

// ---------------------------------------------------------------- WaS ring on the device
// (kernels/ring.cu): epoch flags per slot + device-side logs of what was actually fetched and
// consumed.  One FetchRing per context, library-owned, zeroed (t_first = ~0) at alloc and at
// every plan reset.
constexpr int kRingMaxSlots = 16;
constexpr int kFetchLogCap = 4096;
constexpr int kFetchStages = 6;                 // shared-memory ring of the bulk fetch
constexpr int kFetchChunk = 32 * 1024;          // bytes per bulk copy
constexpr int kFetchClaim = 8;                  // chunks per atomic claim (SIDP_FETCH_CLAIM)
struct FetchLogEnt {
  unsigned long long j;        // fetch index since the last reset
  int layer, slot, owner, pad;
  unsigned long long epoch;    // fill number of the slot (1-based)
  unsigned long long t_start, t_end;   // %globaltimer ns: first CTA start, publish
};
struct ConsLogEnt {
  int layer, slot, tag, pad;
  unsigned long long epoch;    // consumption number of the slot (1-based)
  unsigned long long t;        // %globaltimer ns when the layer's weights were ready
};
struct FetchRing {
  unsigned long long fill[kRingMaxSlots];   // completed fills per slot (fetch side)
  unsigned long long rel[kRingMaxSlots];    // releases per slot (compute side)
  unsigned long long cons[kRingMaxSlots];   // consumptions started (compute side)
  unsigned long long t_first[kRingMaxSlots];   // earliest CTA start of the slot's current fill
  unsigned int arrive[kRingMaxSlots];       // CTAs done with the slot's current fill (static split)
  int tag[kRingMaxSlots];                   // layer held by the slot (last fill)
  // dynamic chunk claiming (fetch_bulk_kernel): fill n of slot s owns claim indices
  // [n (nch + F), (n + 1)(nch + F)) — each CTA over-claims at most once per fill — and is complete
  // when done[s] reaches (n + 1) nch; t0[s] = paced start of fill t0_fill[s] - 1
  unsigned long long claim[kRingMaxSlots];
  unsigned long long done[kRingMaxSlots];
  unsigned long long t0[kRingMaxSlots];
  unsigned long long t0_fill[kRingMaxSlots];
  unsigned long long link_t;                // emulated link: due end of the last started fill
  unsigned long long nfetch, ncons;
  FetchLogEnt log[kFetchLogCap];
  ConsLogEnt clog[kFetchLogCap];
};
// One fetch of a window: layer `layer` of owner `owner` from src into slot `slot`, fill number
// `fill` of that slot (0-based; host-counted, so the gate needs no device read of fill[slot]).
struct FetchEnt {
  const uint8_t* src;
  int layer, slot, owner;
  unsigned int fill;
};
constexpr int kFetchWindow = 96;   // fetches one launch can carry (>= remote layers per pass)
struct FetchArgs {
  uint8_t* slots; size_t slot_stride; size_t bytes;   // destination slot s = slots + s * stride
  FetchRing* ring;             // null: plain copy (test hook: src -> slots), no gate / publish
  int n;                       // entries in this launch
  int gate;                    // 1: each CTA waits for rel[slot] >= fill in-kernel (windowed)
  uint64_t ns_per_chunk;       // > 0: emulated link rate (chunk c starts >= c x ns after start)
  uint64_t delay_ns;           // start offset (C-S7 stagger) before the first entry
  uint64_t timeout_ns; int* err;   // gate timeout -> *err (mapped host word)
  int chunk, stages;           // set by fetch_bulk_launch (shared-memory ring geometry)
  int claim_group;             // set by fetch_bulk_launch: chunks per atomic claim
  int nparts;                  // tile-granular slots: parts per blob (0/1 = whole layers)
  int ce_chunks;               // hybrid fetch (whole layers): chunks [0, ce_chunks) of every fill
                               // come from the copy engine (ring_ce_done adds them to `done`)
  size_t part_off[4], part_bytes[4];   // byte range of each part within the blob
  FetchEnt ent[kFetchWindow];
};
size_t fetch_bulk_smem();
cudaError_t fetch_bulk_launch(const FetchArgs& a, int ctas, cudaStream_t s);
cudaError_t ring_free_wait_launch(FetchRing* r, int slot, unsigned long long fill,
                                  uint64_t timeout_ns, int* err, cudaStream_t s);
cudaError_t ring_ready_wait_launch(FetchRing* r, int slot, int layer, uint64_t timeout_ns, int* err,
                                   cudaStream_t s);
// Debug: compare `bytes` of a landed slot with its owner's source; cnt[0] += 1, cnt[1] +=
// differing 16-byte words (SIDP_SLOT_VERIFY=1, sidp_stats slot_checks / slot_mismatches).
cudaError_t slot_verify_launch(const void* slot, const void* src, size_t bytes,
                               unsigned long long* cnt, cudaStream_t s);
cudaError_t ring_release_launch(unsigned long long* rel, cudaStream_t s,
                                unsigned long long* b = nullptr);
cudaError_t ring_delay_launch(uint64_t ns, cudaStream_t s);
// Hybrid fetch: after the copy engine wrote chunks [0, ce_chunks) of fill e.fill of e.slot, count
// them into the fill (the SM kernel counts the rest); whichever side completes it publishes.
cudaError_t ring_ce_done_launch(FetchRing* r, const FetchEnt& e, unsigned long long nchunks,
                                unsigned ce_chunks, cudaStream_t s);
cudaError_t ring_preload();

// ---------------------------------------------------------------- CaS signalling
struct FlagSet {
  uint64_t* p[16];
  int n;
};
cudaError_t signal_launch(uint64_t* flag, uint64_t value, cudaStream_t s,
                          const uint64_t* base = nullptr);
cudaError_t wait_launch(const FlagSet& flags, uint64_t value, uint64_t timeout_ns, int* err,
                        cudaStream_t s, const uint64_t* base = nullptr);
// *base += delta (the CaS round-trip counter of a step; first kernel of a CaS step)
cudaError_t base_add_launch(uint64_t* base, uint64_t delta, cudaStream_t s);
cudaError_t copy_rows_launch(void* dst, int ldd, const void* src, int lds, int rows, int row_bytes,
                             cudaStream_t s);
// Fused CaS transfer ("V2": fewer, fused transfer launches): copy every job's
// rows (row_bytes % 16 == 0; destinations may be peer VAs) and, once ALL of them are globally
// visible, release-store `value` into every flag.  One launch replaces njobs copy kernels plus
// nflags signal kernels.  `counter` (device int, 0 between launches) elects the last CTA.
struct XferJob { void* dst; const void* src; int ldd, lds, rows, row_bytes; };
struct XferSet {
  XferJob job[16]; int njobs;
  uint64_t* flag[18]; int nflags;
  uint64_t value;
  unsigned int* counter;
};
cudaError_t xfer_launch(const XferSet& x, cudaStream_t s);

// Wait for the flags, then copy rows (CaS requester: the owner's returned slice -> x).
cudaError_t wait_copy_launch(const FlagWait& w, void* dst, int ldd, const void* src, int lds,
                             int rows, int row_bytes, cudaStream_t s);

// Eager module loading of every kernel (called once by sidp_alloc).
cudaError_t gemm_preload();
cudaError_t attention_preload();
cudaError_t norm_preload();
cudaError_t fetch_preload();

}  // namespace sidp
