/*
 * odmoe.h — C ABI of the B200-native OD-MoE decode hot path (arXiv 2512.03927).
 *
 * "P:L" cites /root/reference/PAPER.md line L; "S:L" cites SPEC.md line L; "Qn" is a
 * reading of the paper listed in DESIGN.md §4.
 *
 * The library (paper_2512_03927_b200/libodmoe.so) is CUDA sm_100a code plus a C++
 * runtime. Every entry point returns an odmoe_status; nothing aborts and no C++
 * exception crosses this boundary. Two families of calls:
 *
 *  1. Stateless kernels (odmoe_route_topk, odmoe_expert_ffn, odmoe_shadow_expert_ffn,
 *     odmoe_lm_head_argmax, odmoe_quantize_int8_rows, odmoe_gen_weights):
 *     every pointer is CALLER-OWNED DEVICE memory on the current CUDA device, row-major,
 *     16-byte aligned; `stream` is a cudaStream_t (NULL = legacy default stream).
 *     They only enqueue work and return; results are valid when the stream reaches them.
 *     Shape errors return ODMOE_E_CONFIG before anything is enqueued; a launch error
 *     returns ODMOE_E_CUDA.
 *
 *  2. The stateful decode engine (odmoe_create ... odmoe_destroy): one odmoe_ctx per
 *     process, bound to one GPU (one process per GPU; ranks talk over NCCL). The ctx
 *     owns the pinned host expert pool, the device expert slots, the resident
 *     non-expert weights, the INT8 shadow model (rank 0), the copy-stream loader thread,
 *     the NCCL communicators, streams and events. Host output buffers of these calls are
 *     caller-owned and valid when the call returns. A ctx is used by one host thread.
 *
 * Data layout of one expert blob (host pool and device slot, dtype T = bf16 | fp32):
 *   W13 [F][2][d]  row 2f = W1 row f ("gate"), row 2f+1 = W3 row f ("up")   (interleaved)
 *   W2  [d][F]                                                               (row-major)
 *   blob = W13 followed immediately by W2; 3*d*F*sizeof(T) bytes.
 */
#ifndef ODMOE_H_
#define ODMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ODMOE_ABI_VERSION 2

typedef enum {
  ODMOE_OK = 0,
  ODMOE_E_CONFIG = 1,    /* bad shape/config: k>E, zero dims, d%8, world % G, ... */
  ODMOE_E_RANGE = 2,     /* layer / expert / token out of range                      */
  ODMOE_E_NONFINITE = 3, /* NaN/Inf in a hidden state or logits                             */
  ODMOE_E_BUDGET = 4,    /* a load would exceed the per-GPU slot budget                    */
  ODMOE_E_STATE = 5,     /* evict of a non-resident expert, call on a destroyed/poisoned ctx, ...  */
  ODMOE_E_PLAN = 6,      /* cardinality mismatch in placement                              */
  ODMOE_E_NOMEM = 7,     /* host pin or device allocation failed                                   */
  ODMOE_E_CUDA = 8,      /* CUDA error; the ctx is poisoned (every later call returns E_STATE)     */
  ODMOE_E_NCCL = 9       /* NCCL error; the ctx is poisoned                                         */
} odmoe_status;

typedef enum { ODMOE_BF16 = 0, ODMOE_FP32 = 1 } odmoe_dtype;

/* Where the loader's expert IDs come from (P:250-258 ablation cases in B200 form). */
typedef enum {
  ODMOE_PRED_SHADOW_INT8 = 0, /* SEP with an INT8-row quantised shadow (Q9, Q10)    */
  ODMOE_PRED_NONE = 1,        /* load only after the main router (P:257 case 6)                         */
  ODMOE_PRED_RANDOM = 2,      /* uniformly random k experts per layer (P:256 case 5; E[recall] = k/E)    */
  ODMOE_PRED_PERFECT = 3,     /* replay of the true routing recorded by an earlier run of the same ctx   */
  ODMOE_PRED_SHADOW_SAME = 4, /* shadow with the main model's own weights (recall must be exactly 1.0)   */
  ODMOE_PRED_GATE_REUSE = 5,  /* prior work: after the main router of layer l,
                                 apply the gates of layers l+1..l+D to layer l's normalised input   */
  ODMOE_PRED_SHADOW_BF16 = 6, /* SEP with a BF16 shadow of an FP32 main model: the B200 analogue of the
                                 paper's FP16 shadow (99.94 % recall); needs dtype FP32 */
  ODMOE_PRED_SHADOW_NF4 = 7,  /* SEP with an NF4 shadow (95.67 % recall; reading Q27):
                                 expert matrices NF4 in 64-weight blocks, embedding/routers int8-row;
                                 needs d, F multiples of 64 */
  ODMOE_PRED_SHADOW_FP8 = 8   /* SEP with an FP8 (E4M3, row-scaled) shadow: the precision axis between
                                 INT8 and BF16 (reading Q28); embedding/routers int8 */
} odmoe_predictor;

/* Where expert work goes at N > 1 GPUs. */
typedef enum {
  ODMOE_PLACE_GROUPS = 0,  /* the paper's placement: G = min(k, N) GPUs per group, layer l on
                              group l mod N_G, sorted experts <-> sorted GPUs; one whole expert per GPU   */
  ODMOE_PLACE_SLICED = 1   /* SURVEY §8(f)3 "sliced loading": every GPU holds, loads and computes 1/N of
                              every expert (W13 rows of its F/N gate/up pairs, the matching W2 columns),
                              sums its k gated partials and the N partials are reduced on GPU 0. All N host
                              links serve every layer, so lookahead 1 suffices. Needs F % (16 N) == 0; not
                              with SHADOW_SAME; slots_per_gpu counts slice slots                        */
} odmoe_placement;

typedef struct {
  int32_t L, E, k, d, F, V;  /* Mixtral 32,8,2,4096,14336,32000; tiny 4,8,2,256,512,1024           */
  int32_t dtype;             /* odmoe_dtype of the main model's weights and of the normalised input u */
  int32_t predictor;         /* odmoe_predictor                                                       */
  int32_t lookahead;         /* D >= 1: loads may be issued for layers <= current + D (Q11)           */
  int32_t slots_per_gpu;     /* device expert slots per GPU (>= 1); -1 = fully resident baseline. With
                                fewer slots than this GPU's experts of a layer (FP32 Mixtral: 1 slot
                                under the 1 GB budget) the experts that found no slot
                                before the router are loaded after the previous expert's compute frees
                                one; like misprediction reloads they count as post-router loads
                                (reloads, reload_ids)                                                  */
  float rms_eps;             /* RMSNorm epsilon (1e-5, Q7)                                             */
  uint64_t weight_seed;      /* synthetic weights: counter-based generator               */
  uint64_t aux_seed;         /* RANDOM predictor stream                                                */
  int32_t rank, world_size;  /* this process's rank; number of GPUs (1, 2, 4, 8)                       */
  int32_t group_size;        /* G; 0 => min(k, world_size) (Q14)                                */
  int32_t device;            /* CUDA device ordinal of this rank                                       */
  int64_t chunk_bytes;       /* H2D copy chunk (0 => 32 MiB)                                            */
  int32_t debug_capture;     /* 1 => keep every per-layer intermediate on the host (parity tests)      */
  int32_t time_kernels;      /* CUDA events around kernels: 1 => expert FFN launches only (the roofline
                                kernel; keeps the PDL chains of the other kernels intact), 2 => every
                                kernel family (per-family stats)                                        */
  int32_t pool_threads;      /* host threads used to build the pool (0 => all)                         */
  int32_t refine_depth;      /* R >= 0: SEP refinement ("Mode B"): after the main router of
                                layer l the shadow re-runs layers l..l+R-1 from the main model's exact
                                state and corrects the loads of layers l+1..l+R; 0 = off (paper's Mode A) */
  int32_t placement;         /* odmoe_placement: 0 = the paper's worker groups, 1 = sliced      */
  int32_t n_heads;           /* attention block (reading Q29): query heads H, 0 = no
                                attention (the MoE-only hot path); head_dim = d / H in {32, 64, 128}     */
  int32_t n_kv_heads;        /* key/value heads (GQA), H % Hkv == 0, H / Hkv <= 8                       */
  int32_t max_seq;           /* KV-cache capacity in tokens (0 => 4096 when n_heads > 0)                */
  int32_t emulate_world;     /* 0/1 = off; N in {2, 4, 8} with world_size == 1: run the expert arithmetic
                                of an N-GPU run of `placement` on this one GPU -- SLICED: each routed
                                expert as N F/N slices computed with the kernels and grid a real rank
                                uses, each emulated rank's k gated partials summed in router rank order,
                                the N partials summed in rank order (the P2P combine's order); GROUPS:
                                the experts summed per emulated rank of layer l's group (sorted pairing)
                                then over the group's ranks in rank order. Values are bitwise those of
                                the real N-GPU run (parity of the multi-GPU arithmetic on one GPU; time
                                is NOT emulated). On-demand decode only (no prefill)                   */
  int32_t expert_layer_period; /* 0 => off; P in 1..L: the expert weights of layer l are generated as
                                those of layer l mod P (a synthetic model whose expert tensors repeat
                                with period P; routers, embedding, LM head stay per layer). The host pool
                                holds P layers' blobs, every load still moves one full blob, so loads and
                                bytes per token are the full model's: used for the FP32 leg whose
                                L-layer pool (180 GB) exceeds the GPU box's host RAM. Not with groups
                                placement at N > 1                                                      */
  const void* nccl_id;       /* 128-byte ncclUniqueId from rank 0 (NULL when world_size == 1)          */
} odmoe_config;

/* One per layer per decode step (S:154-157 RoutingRecord). k <= 8. Filled on every rank that passes
 * a non-NULL rec; true_ids / pred_ids / weights / correct are the same on every rank, the load fields
 * (issued_ids, reload_ids, n_reloads, load_wait_us) describe THIS rank's loads. */
typedef struct {
  int32_t true_ids[8];       /* main-router top-k, rank order                                          */
  int32_t pred_ids[8];       /* the predictor's ids for this layer (Mode A for the shadows; -1 = none) */
  float weights[8];          /* mixture weights, aligned with true_ids                                 */
  int32_t pred_available;    /* 1 => the predictor produced ids for this layer in this step (Eq. 3
                                counts them: prediction accuracy); 0 => none (c = 0)     */
  int32_t correct;           /* c(n, l) = |true ∩ pred| (Eq. 2 numerator term)                   */
  int32_t n_reloads;         /* experts loaded after the router because the prediction missed  */
  float load_wait_us;        /* host-observed wait for this layer's router ids                         */
  int32_t pred_in_time;      /* 1 => pred_ids had reached the host BEFORE this layer's router ids did
                                (the prediction could drive the loads: "prediction
                                available at decision time")                                          */
  int32_t correct_in_time;   /* correct if pred_in_time else 0 (the conservative c of S:197)           */
  int32_t issued_ids[8];     /* experts of this layer whose loads THIS rank issued before the router ids
                                reached the host (predicted loads, incl. ones later stopped), ascending,
                                -1 padded                                                             */
  int32_t reload_ids[8];     /* experts of this layer THIS rank loaded after the router (misprediction
                                fallback), ascending, -1 padded                    */
} odmoe_layer_record;

typedef struct {
  int64_t tokens;            /* decode steps since reset                                              */
  int64_t loads_issued;      /* expert loads started (incl. reloads and wasted loads)                 */
  int64_t loads_completed;
  int64_t loads_cancelled;   /* mispredicted loads stopped before their last chunk                    */
  int64_t reloads;           /* loads issued after the router (misprediction fallback)         */
  int64_t bytes_h2d;         /* bytes copied host->device by the loader                              */
  int64_t kernel_launches;   /* kernels this library launched                                        */
  int64_t max_resident;      /* peak number of occupied expert slots on this GPU (S:326 audit)       */
  int64_t resident_bytes;    /* device bytes of expert slots (slots_per_gpu * blob)                   */
  int64_t shadow_bytes;      /* device bytes of the shadow model on this GPU                          */
  int64_t pool_bytes;        /* pinned host pool bytes on this rank                                   */
  double pool_build_s;       /* seconds spent pinning + generating the pool                           */
  /* time_kernels: summed device time (ms) and launch count per kernel family */
  double ms_router, ms_w13, ms_w2, ms_shadow, ms_lm_head, ms_embed;
  int64_t n_router, n_w13, n_w2, n_shadow, n_lm_head, n_embed;
  double wait_us;            /* host time blocked on loads                                            */
  int64_t correct, predicted_total; /* Σc and Σ k over layers with a prediction (rank 0)              */
  int64_t refine_corrections;        /* layer predictions changed by the SEP refinement                */
  int64_t refine_correct, refine_total; /* Σc, Σk of the refined predictions (rank 0)                  */
  double ms_attn;                    /* attention block kernels (QKV, RoPE, attention, W_o), rank 0     */
  int64_t n_attn;
  int64_t correct_in_time;           /* Σc over layers whose prediction arrived before the router */
  int64_t spec_steps;                /* decode steps whose predictions came from a speculative shadow pass
                                        (token alignment period > 1, the shadow's own token)            */
  int64_t early_loads;               /* loads issued for the NEXT token while this one was decoding     */
  /* time_kernels = 2: the shadow's expert phases (one launch per phase for its k experts; also in
     ms_shadow): W13 + SwiGLU, W2 + gate; n_* count experts */
  double ms_sh_w13, ms_sh_w2;
  int64_t n_sh_w13, n_sh_w2;
  /* option 9: device time of whole shadow passes (embed .. last expert; one event pair per pass, so
     the kernels inside keep their PDL chains) and their count */
  double ms_sh_pass;
  int64_t n_sh_pass;
} odmoe_stats;

/* ------------------------------------------------------------------ lifecycle */
int32_t odmoe_abi_version(void);
odmoe_status odmoe_create(const odmoe_config* cfg, void** ctx_out);
/* Generates the synthetic model from cfg->weight_seed, pins + fills this rank's host pool,
 * quantises the shadow (rank 0), allocates slots, joins the NCCL communicator.
 * Errors: E_CONFIG (validation), E_NOMEM, E_CUDA, E_NCCL. *ctx_out is NULL on error. */
void odmoe_destroy(void* ctx);
const char* odmoe_last_error(const void* ctx); /* ctx==NULL => last create error of this thread */
odmoe_status odmoe_get_stats(const void* ctx, odmoe_stats* out);
odmoe_status odmoe_reset_stats(void* ctx);
int odmoe_nccl_unique_id(void* out128); /* fills a 128-byte ncclUniqueId; returns 0 on success */

/* ------------------------------------------------------------------ placement plan (host only) */

/* Experts of `layer` that `rank` computes for router output ids[k] (P:104 groups of G workers,
 * one-to-one assignment; P:113-120 layer -> group l mod N_G round robin
 * sorted pairing; Q14 G = min(k, N) when group_size == 0, a GPU takes k/G experts when G < k).
 * Writes *n_out (0..k) ascending expert ids to out[k] (host). Pure function; no GPU needed.
 * E_CONFIG on invalid sizes (world % G, k % G, rank range). */
odmoe_status odmoe_plan_layer(int k, int world_size, int group_size, int layer, const int32_t* ids,
                              int rank, int32_t* out, int32_t* n_out);
/* 1 if `rank`'s host pool must hold expert (layer, expert) (some routing can send it there under
 * the sorted pairing), 0 if not, -1 on invalid sizes. Pure function. */
int32_t odmoe_plan_pool_holds(int E, int k, int world_size, int group_size, int layer, int expert,
                              int rank);

/* ------------------------------------------------------------------ stateless kernels */

/* Fused residual-combine + RMSNorm + router GEMV + softmax/top-k + renormalise
 * (a2+a3 of SURVEY §8(a); Q2, Q3, Q7).
 *   h      [m,d] fp32 residual stream (in/out): h += y_add[0] + ... + y_add[n_add-1]
 *          (added in the order given), written back to h.
 *   y_add  device array of n_add device pointers to fp32 [m,d] partial outputs (may be NULL)
 *   gamma  [d] of dtype dt, or NULL (=1)
 *   w_gate [E,d] of dtype dt
 *   u_out  [m,d] dtype dt: RMSNorm(h) rounded to dt (RNE)
 *   ids    [m,k] int32, rank order (logit desc, lower index on ties)
 *   w      [m,k] fp32 softmax over the selected logits
 *   logits [m,E] fp32 or NULL
 *   flag   int32 device scalar or NULL: set to 1 if any logit is non-finite
 * Limits: 1 <= k <= E <= 64, k <= 8, d % 8 == 0. */
odmoe_status odmoe_route_topk(float* h, const float* const* y_add, int n_add, const void* gamma,
                              const void* w_gate, int m, int E, int d, int k, int dt, float eps,
                              void* u_out, int32_t* ids, float* w, float* logits, int32_t* flag,
                              void* stream);

/* Expert SwiGLU FFN at batch 1 (a8; Q1, Q8):
 *   a = silu(W1 u) * (W3 u)  (fp32, scratch [F]),  y = gate_w[gate_idx] * (W2 a)  (fp32 [d]).
 *   w13 [F][2][d] dt, w2 [d][F] dt, u [d] dt, gate_w device fp32 array (NULL => 1.0),
 *   a_scratch fp32 [F] device, y fp32 [d] (overwritten).
 * Limits: d % 8 == 0, F % 8 == 0. */
odmoe_status odmoe_expert_ffn(const void* w13, const void* w2, const void* u, const float* gate_w,
                              int gate_idx, int d, int F, int dt, float* a_scratch, float* y,
                              void* stream);

/* Shadow expert FFN with INT8-row weights (a4; Q9):
 *   q13 [F][2][d] int8 with s13 [2F] fp32 row scales; q2 [d][F] int8 with s2 [d] fp32;
 *   u [d] bf16. Same math as odmoe_expert_ffn with W = s_r * q_r. */
odmoe_status odmoe_shadow_expert_ffn(const int8_t* q13, const float* s13, const int8_t* q2,
                                     const float* s2, const void* u, const float* gate_w,
                                     int gate_idx, int d, int F, float* a_scratch, float* y,
                                     void* stream);

/* The same INT8 shadow expert on the tensor cores (reading Q32; the engine's default shadow path):
 * q13p / q2p are the codes in the fragment-packed layout written by odmoe_pack_int8_frag (W13 with
 * pair_rows = 1, W2 with pair_rows = 0), s13 / s2 natural-order row scales as above. d, F multiples
 * of 32. Same math as odmoe_shadow_expert_ffn (fp32 accumulation in the tensor cores' order);
 * a_scratch (4F bytes) receives the SwiGLU activation in the tensor cores' B-fragment form (f16 hi +
 * lo per element), not as fp32. */
odmoe_status odmoe_shadow_expert_ffn_packed(const uint8_t* q13p, const float* s13, const uint8_t* q2p,
                                            const float* s2, const void* u, const float* gate_w, int gate_idx,
                                            int d, int F, float* a_scratch, float* y, void* stream);
/* int8 codes q [R][C] (row-major, signed) -> the fragment-packed layout of mma.sync m16n8k16
 * (16-row tiles x 32-column blocks of 512 B; each lane's 16 B = its A fragments of two k-blocks, the
 * codes stored biased q + 128). pair_rows = 1: tile row g / g+8 = rows 2(8t+g) / 2(8t+g)+1 (W13's
 * gate/up pairs). R % 16 == 0, C % 32 == 0 else E_CONFIG. out: R*C bytes (device). */
odmoe_status odmoe_pack_int8_frag(const int8_t* q, int64_t R, int64_t C, int pair_rows, uint8_t* out, void* stream);

/* NF4 shadow expert FFN (reading Q27): like odmoe_shadow_expert_ffn with W = c[code] * absmax.
 * q13: codes of W13 [2F][d/2] bytes (two codes per byte, low nibble = even column), a13: fp32
 * absmax [2F][d/64]; q2 [d][F/2], a2 [d][F/64]; u bf16 [d]. d, F multiples of 64 (the flat
 * kernel needs multiples of 1024; other shapes take a warp-per-row kernel). */
odmoe_status odmoe_shadow_expert_ffn_nf4(const uint8_t* q13, const float* a13, const uint8_t* q2,
                                         const float* a2, const void* u, const float* gate_w, int gate_idx,
                                         int d, int F, float* a_scratch, float* y, void* stream);

/* FP8 shadow expert FFN (reading Q28): like odmoe_shadow_expert_ffn with W = s_r * e4m3(q_rj):
 * q13 E4M3 codes [2F][d], s13 [2F]; q2 [d][F], s2 [d]; u bf16 [d]. */
odmoe_status odmoe_shadow_expert_ffn_fp8(const uint8_t* q13, const float* s13, const uint8_t* q2,
                                         const float* s2, const void* u, const float* gate_w, int gate_idx,
                                         int d, int F, float* a_scratch, float* y, void* stream);

/* Router over INT8-row weights (shadow gating): like odmoe_route_topk with w_gate = s_e*q_e,
 * gamma = 1, u_out bf16. */
odmoe_status odmoe_shadow_route_topk(float* h, const float* const* y_add, int n_add,
                                     const int8_t* q_gate, const float* s_gate, int m, int E, int d,
                                     int k, float eps, void* u_out, int32_t* ids, float* w,
                                     float* logits, int32_t* flag, void* stream);

/* Prefill grouping ("embeddings are grouped by their desired experts"): stable
 * counting sort of the T*k (token, slot) pairs of ids [T,k] by expert. Outputs (device):
 * offsets [E+1] (rows of expert e are [offsets[e], offsets[e+1])), src_pair [T*k] (pair index
 * t*k+j of each grouped row), inv [T*k] (grouped row of each pair), gate_perm [T*k] (w of that
 * pair). Stable: within an expert, pairs keep ascending (t, j) order. */
odmoe_status odmoe_prefill_group(const int32_t* ids, const float* w, int T, int k, int E,
                                 int32_t* offsets, int32_t* src_pair, int32_t* inv,
                                 float* gate_perm, void* stream);

/* Grouped expert SwiGLU FFN for prefill on the tcgen05 tensor cores (a11; Q8):
 * for every expert e and grouped row r in [offsets[e], offsets[e+1]):
 *   a2[r] = bf16(silu(W1_e x[r]) * (W3_e x[r]))   and   y[r] = gate_perm[r] * (W2_e a2[r]).
 * w13[e], w2[e]: HOST arrays of DEVICE pointers (bf16 [F][2][d] and [d][F]); x_perm [M,d] bf16,
 * gate_perm [M] fp32, a2_scratch [M,F] bf16, y_perm [M,d] fp32 (device); offsets [n_experts+1]
 * HOST int32, M = offsets[n_experts]; tiles_scratch device >= 16*(M/128 + n_experts)*(2F/224 +
 * d/128) bytes. Limits: n_experts <= 8, d % 256 == 0, F % 128 == 0, bf16 only. Synchronous on
 * `stream` (returns after the GEMMs complete). */
odmoe_status odmoe_expert_ffn_grouped(const void* const* w13, const void* const* w2, int n_experts,
                                      const void* x_perm, const int32_t* offsets,
                                      const float* gate_perm, int d, int F, void* a2_scratch,
                                      float* y_perm, void* tiles_scratch,
                                      int64_t tiles_scratch_bytes, void* stream);

/* Final RMSNorm + LM head GEMV + greedy argmax (a10; S:95 lowest id on ties).
 *   h [d] fp32 (h_L), lm_head [V,d] dt; token_out int32 device scalar;
 *   logits [V] fp32 or NULL; scratch: device buffer of >= 16*4096 bytes. */
odmoe_status odmoe_lm_head_argmax(const float* h, const void* lm_head, int V, int d, int dt,
                                  float eps, int32_t* token_out, float* logits, void* scratch,
                                  void* stream);

/* INT8 per-row quantiser (Q9): q = clamp(RNE((W*127)/m_r), -127, 127) in fp64,
 * s = fl32(m_r/127); zero rows -> q = 0, s = 1.  w [R,C] dt -> q [R,C] int8, s [R] fp32. */
odmoe_status odmoe_quantize_int8_rows(const void* w, int64_t R, int64_t C, int dt, int8_t* q,
                                      float* s, void* stream);

/* NF4 blockwise quantiser (reading Q27; QLoRA's codebook): per block of 64 consecutive weights
 * of a row, absmax[r][b] = max|w| (fp32), code = nearest codebook entry to w/absmax compared in
 * fp64 (lower index on a tie; zero block -> code 7). w [R][C] of dtype dt (device), q [R][C/2]
 * bytes (low nibble = even column), absmax [R][C/64]. C % 64 == 0 else E_CONFIG. */
odmoe_status odmoe_quantize_nf4(const void* w, int64_t R, int64_t C, int dt, uint8_t* q, float* absmax,
                                void* stream);

/* FP8 row quantiser (reading Q28): s_r = fl32(max|w_r|/448), code = E4M3(RNE, satfinite) of
 * fl32(w/s_r) (fp64 quotient); zero row -> codes 0, s = 1. q [R][C] bytes, s [R] (device). */
odmoe_status odmoe_quantize_fp8_rows(const void* w, int64_t R, int64_t C, int dt, uint8_t* q, float* s,
                                     void* stream);

/* Synthetic weight generator: out[i] = dt(fl32(v_i * fl32(1/sqrt(fan_in)))),
 * v_i from splitmix64(seed, tensor_id, i). kind: 1 emb, 2 router, 3 W1, 4 W3, 5 W2, 6 LM head;
 * kind 0 = the interleaved expert blob of (layer, expert) (W13 then W2; rows/cols ignored). */
odmoe_status odmoe_gen_weights(void* out, int kind, int layer, int expert, int64_t rows,
                               int64_t cols, int64_t fan_in, int d, int F, uint64_t seed, int dt,
                               void* stream);

/* ------------------------------------------------------------------ stateful engine */

/* Async H2D load of expert (layer, expert) into a free slot of this rank's GPU,
 * through the same copy-stream loader the decode step uses (most urgent first). OK no-op if
 * already resident or loading; E_BUDGET if every slot is occupied; E_RANGE if this rank's pool
 * does not hold that expert; E_STATE on a fully-resident ctx. A slot filled this way stays
 * occupied (and unavailable to odmoe_decode_step) until odmoe_evict. */
odmoe_status odmoe_load(void* ctx, int layer, int expert);
/* Block until (layer, expert) is resident; *w13 / *w2 receive its device pointers. */
odmoe_status odmoe_load_wait(void* ctx, int layer, int expert, void** w13, void** w2);
/* Free the slot once work already enqueued on the compute stream is done ("promptly evicts
 * it afterward"; Q16). Only the engine's compute stream is ordered before the slot's reuse:
 * a caller that read the weights from kernels on its own streams must synchronise those streams
 * first. E_STATE if the expert is not resident/loading. */
odmoe_status odmoe_evict(void* ctx, int layer, int expert);

/* Event trace of the decode engine (S:350-358 event schema; Eq. 1 analysis). Enabled with
 * odmoe_set_option(ctx, 7, 1); every decode step then appends events on this rank. Times are device
 * times in microseconds since the trace was enabled (CUDA events on the compute and copy streams of
 * this GPU); host-only events carry t_us = NaN. */
typedef enum {
  ODMOE_EV_STEP_START = 0,    /* compute stream reached the start of decode step `step`            */
  ODMOE_EV_LOAD_ISSUE = 1,    /* host: load of (layer, expert) submitted to the loader; l_cur = the
                                 main layer the host was at (the lookahead window, Q11: layer (counted
                                 from this step's layer 0; L + m for layer m of the next token) must
                                 be <= l_cur + D); aux = 0 predicted, 1 reload after the router,
                                 2 refined prediction, 3 next-token (cross-token speculation)       */
  ODMOE_EV_LOAD_START = 2,    /* copy engine began the first chunk (after the slot's free event)   */
  ODMOE_EV_LOAD_END = 3,      /* copy engine finished the last chunk it issued; bytes = bytes copied */
  ODMOE_EV_LOAD_CANCEL = 4,   /* host: a mispredicted load was stopped                      */
  ODMOE_EV_ROUTER_DONE = 5,   /* layer's routing known on this GPU (router kernel, or the packet
                                 broadcast at N > 1)                                                  */
  ODMOE_EV_COMPUTE_START = 6, /* expert kernel of (layer, expert) may start: its load has landed and
                                 the compute stream reached it                                        */
  ODMOE_EV_COMPUTE_END = 7,   /* expert kernel of (layer, expert) finished                          */
  ODMOE_EV_MISPREDICT = 8,    /* host: (layer, expert) was routed but not loaded -> reload   */
  ODMOE_EV_STEP_END = 9       /* compute stream finished the step (token on the host next)          */
} odmoe_event_type;

typedef struct {
  int32_t type;              /* odmoe_event_type                                                      */
  int32_t step;              /* decode step (ctx-local counter) the event belongs to                  */
  int32_t layer, expert;     /* -1 when not applicable                                                */
  int32_t slot;              /* device expert slot, -1 when not applicable                            */
  int32_t l_cur;             /* LOAD_ISSUE: main layer at issue time (-1 = before layer 0's router)    */
  int32_t aux;               /* LOAD_ISSUE kind (see above)                                           */
  int32_t rank;              /* this rank                                                              */
  int64_t bytes;             /* LOAD_END / LOAD_CANCEL: bytes copied for this load                    */
  double t_us;               /* device time (µs since the trace was enabled), NaN for host-only events */
} odmoe_trace_event;

/* Move up to `cap` resolved trace events (in emission order) into `out` (host, caller-owned) and
 * set *n_out; events whose device times are not final yet (loads still in flight) stay queued.
 * E_STATE if tracing was never enabled. */
odmoe_status odmoe_trace_read(void* ctx, odmoe_trace_event* out, int32_t cap, int32_t* n_out);

/* Runtime options (take effect at the next decode step; every rank must set the same value):
 *   key 1 = lookahead D (>= 1, Q11); key 2 = predictor (odmoe_predictor; the shadow predictors
 *   need a ctx created with a shadow predictor: E_STATE otherwise); key 3 = refine_depth R (0..4;
 *   only with a shadow predictor); key 4 = KV-cache position of the next decode step (attention
 *   ctx only; 0 starts a new sequence; E_RANGE outside [0, max_seq)); key 5 = KV alignment of the
 *   shadow (Fig. 3: 1 = attend over the main model's cache (default), 0 = the shadow keeps
 *   its own cache from its own passes; attention ctx with a shadow); key 6 = time_kernels level (0..2,
 *   see odmoe_config); key 7 = event trace (0 off, 1 on; odmoe_trace_read); key 8 = token alignment
 *   period T_p of the shadow (Fig. 6 "T_i": 1 = the main model's token every iteration
 *   (Mode A, default); T_p > 1 = at iterations n with n mod T_p != 0 (n counted from the first step
 *   or the last key-8 / key-4 call) the shadow decodes with its OWN greedy token from its INT8 LM
 *   head, so its pass for token n+1 starts right after its pass for n, before the main model has
 *   finished n, and loads for layers 0.. of n+1 may be issued inside the lookahead window (cross-
 *   token speculation); shadow predictors only, T_p in 1..64); key 9 = shadow-pass
 *   timing (0/1: odmoe_stats.ms_sh_pass / n_sh_pass). E_CONFIG on a bad key/value. */
odmoe_status odmoe_set_option(void* ctx, int key, int64_t value);

/* SEP Mode A (Q10): run the shadow from the main model's token `token`
 * through all L layers (token alignment, T1), cache the predictions for that token and
 * copy P[from_layer .. from_layer+depth) x k (rank order) into pred_ids (host, int32).
 * Rank 0 only (E_STATE elsewhere). */
odmoe_status odmoe_predict_ahead(void* ctx, int32_t token, int from_layer, int depth,
                                 int32_t* pred_ids);

/* One decode iteration: embed token_in, L x [router -> (prediction check,
 * reload) -> expert FFNs on their GPUs -> combine], LM head, argmax. Collective: every rank
 * calls it with the same token_in. token_out (host) is valid on every rank. rec [L] host or
 * NULL (filled on rank 0). Synchronous. */
odmoe_status odmoe_decode_step(void* ctx, int32_t token_in, int32_t* token_out,
                               odmoe_layer_record* rec);

/* Batched prefill of T tokens: no prediction; layer by layer: batched router (T rows),
 * grouping by expert, tcgen05 grouped expert GEMMs, deterministic scatter-combine. Layer l's E
 * experts are loaded onto the G GPUs of group l mod N_G (expert e -> position e*G/E), so loads
 * round-robin over the groups. token_out = greedy token after the last prompt token;
 * expert_counts [L,E] host or NULL (tokens routed per expert, P:214 footnote). Needs the bf16
 * model and 2*E/G extra device expert slots. Collective, synchronous. */
odmoe_status odmoe_prefill(void* ctx, const int32_t* tokens, int T, int32_t* token_out,
                           int32_t* expert_counts);

/* Prefill capture (cfg.debug_capture == 1), rank 0, last prefill: what 0 = residual h entering
 * layer `layer` ([T][d] fp32; layer == L gives the final h), what 1 = router ids of `layer`
 * ([T][k] int32). */
odmoe_status odmoe_prefill_debug_read(const void* ctx, int what, int layer, void* dst, int64_t bytes);

/* Parity capture (cfg.debug_capture == 1), rank 0, last decode step. Copies `bytes` bytes of
 * field `what` for `layer` into host `dst`. Fields and sizes:
 *   0 H_IN fp32[d] (the MoE input: after the attention block when n_heads > 0)  1 U dt[d]
 *   2 LOGITS fp32[E]  3 IDS int32[k]  4 W fp32[k]
 *   5 Y fp32[d] (combined)  6 Y_PART fp32[k][d] (N=1: per selected expert, rank order)
 *   7 SH_H_IN fp32[d]  8 SH_U bf16[d]  9 SH_LOGITS fp32[E]  10 SH_IDS int32[k]
 *   11 H_FINAL fp32[d] (layer ignored)  12 LM_LOGITS fp32[V] (layer ignored)
 *   13 H_PRE fp32[d] (n_heads > 0: h before the attention block of the layer)
 *   with a token alignment period > 1, the shadow pass that produced this step's predictions:
 *   14 SH_H_FINAL fp32[d] (its h_L)  15 SH_TOK int32[1] (its own greedy token)
 *   16 SH_LM_LOGITS fp32[V] (its INT8-row LM head logits)   (layer ignored for 11, 12, 14-16)
 *   with emulate_world = N: 5 Y fp32[d] = the combined output of the N emulated ranks;
 *   17 Y_RANK fp32[N][d] = each emulated rank's partial (sliced: its F/N slices of the k experts,
 *   summed in router rank order; groups: its experts) */
odmoe_status odmoe_debug_read(const void* ctx, int what, int layer, void* dst, int64_t bytes);

/* Device pointers of ctx-owned tensors (tests): 0 emb, 1 lm_head, 2 router[layer],
 * 3 shadow q_gate[layer], 4 shadow s_gate[layer], 5 shadow q13[layer*E+e] (layer, expert via
 * `index` = layer*E+expert), 6 s13, 7 q2, 8 s2, 9 shadow q_emb, 10 shadow s_emb. */
odmoe_status odmoe_tensor_ptr(const void* ctx, int what, int index, void** ptr);

#ifdef __cplusplus
}
#endif
#endif /* ODMOE_H_ */
