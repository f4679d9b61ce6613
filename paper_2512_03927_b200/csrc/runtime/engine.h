// Decode engine state (internal to libodmoe.so). See odmoe.h for the contract and DESIGN.md §5
// for the HBM layout.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../../include/odmoe.h"
#include "../kernels/kernels.h"
#include "loader.h"

namespace odmoe {

enum Family { K_ROUTER = 0, K_W13, K_W2, K_SHADOW, K_LM, K_EMBED, K_ATTN, K_SH_W13, K_SH_W2, K_SH_PASS, K_NFAM };

struct Slot {
  char* dev = nullptr;
  int layer = -1, expert = -1;
  bool occupied = false;
  int64_t token = -1;              // decode step the occupant belongs to
  cudaEvent_t ev_w13 = nullptr, ev_done = nullptr, ev_free = nullptr;
  bool free_recorded = false;
  uint32_t* flag = nullptr;         // device [2]: epoch of the last load whose W13 / whole blob landed
  uint32_t epoch = 0;               // epoch of the current occupant's load
  std::shared_ptr<LoadReq> req;
};

struct Ctx {
  odmoe_config cfg{};
  std::string err;
  bool poisoned = false;
  int L = 0, E = 0, k = 0, d = 0, F = 0, V = 0;
  WType wt = W_BF16;
  size_t esz = 2;
  int64_t blob_elems = 0, blob_bytes = 0, w13_bytes = 0;
  int world = 1, rank = 0, G = 1, NG = 1, my_group = 0, my_pos = 0;
  bool sliced = false;    // ODMOE_PLACE_SLICED: this rank's experts are F/N-wide slices
  int Fs = 0;             // F of the blobs this rank holds (F, or F / world when sliced)
  int64_t full_bytes = 0; // one whole expert blob (generator output)
  // emulate_world (world 1): the expert arithmetic of an N-GPU run on this GPU (odmoe.h)
  int elp = 0;                   // expert_layer_period (0 = off)
  int emu = 0;                   // emulated ranks (0 = off)
  bool emu_sliced = false;       // SLICED: blob = N slice blobs (slice r laid out as rank r's pool blob)
  int emu_G = 1, emu_NG = 1;     // GROUPS: group size and number of groups of the emulated run
  int64_t emu_slice_bytes = 0, emu_w13s = 0;
  float* d_yemu = nullptr;       // [N][k][d] sliced: expert j's partial of slice r
  float* d_prank = nullptr;      // [N][d] each emulated rank's partial
  const float** d_emu_ptr = nullptr;   // device pointer arrays [L][N + N*k]
  const float** h_emu_ptr = nullptr;   // pinned staging of the same
  float* dbg_yrank = nullptr;    // [L][N][d] (debug capture)
  bool resident = false;
  int built_pred = -1;           // predictor the ctx was created with (decides whether a shadow exists)
  int dev = 0;
  cudaStream_t s_main = nullptr, s_shadow = nullptr, s_copy = nullptr;

  // non-expert weights (rank 0): embedding [V,d], LM head [V,d], routers [L][E][d]
  void* d_emb = nullptr;
  void* d_lm = nullptr;
  void* d_router = nullptr;

  // attention block (rank 0; reading Q29): fused QKV [L][(H+2Hkv)*hd][d], W_o [L][d][H*hd] in the
  // main dtype; KV cache [L][max_seq][Hkv*hd] bf16; pos = tokens already in the cache
  int H = 0, Hkv = 0, hd = 0, qkv_rows = 0, kvd = 0, max_seq = 0;
  int kv_esz = 2;               // KV-cache element: bf16 (bf16 model) or fp32 (fp32 model)
  int64_t pos = 0;
  void* d_wqkv = nullptr;
  void* d_wo = nullptr;
  void* d_kc = nullptr;
  void* d_vc = nullptr;
  float* d_qkv = nullptr;       // [qkv_rows]
  float* d_attn_o = nullptr;    // [H*hd]
  float* d_attn_part = nullptr; // split partials
  float* dbg_hpre = nullptr;    // [L][d] h before the attention block (debug capture)
  // prefill attention buffers (T_cap rows)
  void* pa_x = nullptr;         // bf16 [T][d] RMSNorm(h) / attention output o
  float* pa_qkv = nullptr;      // fp32 [T][qkv_rows]
  float* pa_part = nullptr;     // split partials
  float* pa_out = nullptr;      // fp32 [T][d] W_o o
  int4* pa_tiles = nullptr;
  // shadow attention: int8-row copies, its own current-position k/v (past from the main cache)
  void* sh_wqkv = nullptr;
  float* sh_sqkv = nullptr;
  void* sh_wo = nullptr;
  float* sh_so = nullptr;
  float* sh_qkv = nullptr;
  float* sh_attn_o = nullptr;
  float* sh_attn_part = nullptr;
  void* sh_kcur = nullptr;
  void* sh_vcur = nullptr;
  // KV alignment (Fig. 3 "KV1"): 1 = the shadow attends over the MAIN model's cache;
  // 0 ("KV0") = the shadow keeps its own cache, filled by its own token-aligned passes
  int kv_align = 1;
  void* sh_kc = nullptr;
  void* sh_vc = nullptr;

  // shadow model (rank 0)
  bool has_shadow = false;
  WType sh_wt = W_I8;    // shadow embedding / router weights
  WType sh_ewt = W_I8;   // shadow expert weights (W_NF4 for the NF4 shadow)
  void* sh_emb = nullptr;      // int8 [V,d] (or main dtype for SHADOW_SAME)
  float* sh_semb = nullptr;    // [V]
  void* sh_router = nullptr;   // [L][E][d]
  float* sh_srouter = nullptr; // [L][E]
  std::vector<void*> sh_blob;  // [L*E] int8 blobs (q13 then q2)
  std::vector<float*> sh_sc;   // [L*E] scales (s13 [2F] then s2 [d])
  void** d_sh_tbl = nullptr;
  float** d_sh_stbl = nullptr;

  // host pool (pinned): blob of (l, e) at pool + pool_off[l*E+e] (-1 if not on this rank)
  char* pool = nullptr;
  int64_t pool_bytes = 0;
  std::vector<int64_t> pool_off;

  // resident experts (slots_per_gpu == -1, or SHADOW_SAME)
  std::vector<char*> res_blob;
  void** d_res_tbl = nullptr;

  std::vector<Slot> slots;
  Loader loader;

  // device work buffers
  float* d_h = nullptr;          // residual [d]
  char* d_pkt = nullptr;         // [L] packets: u [d] dt | ids [k] int32 | w [k] fp32
  int64_t pkt_bytes = 0, pkt_ids_off = 0, pkt_w_off = 0;
  float* d_logits = nullptr;     // [L][E]
  float* d_a = nullptr;          // [k][F]
  float* d_y = nullptr;          // [k][d] per-expert outputs (this GPU)
  float* d_yred = nullptr;       // [d] reduced output (rank 0, N > 1)
  float* d_zero = nullptr;       // [d] zeros (idle ranks' reduce contribution)
  float* d_ysum = nullptr;       // [d] sliced placement: sum of this rank's k gated partials
  // P2P combine (N > 1): GPU 0 owns part [world][d] + flags [world]; every rank maps them (CUDA IPC)
  bool p2p = false;
  float* p2p_part = nullptr;     // GPU 0's receive rows (local on rank 0, IPC-mapped elsewhere)
  float* p2p_own_part = nullptr; // rank 0: the allocation (freed at destroy)
  uint32_t p2p_seq = 0;          // epoch of the next layer combine (same sequence on every rank)
  bool p2p_fused_sent = false;   // this layer's partials already went out from the W2 epilogue
  const float** d_y1ptr = nullptr;  // device array {d_y} (one partial)
  const float** d_yptr = nullptr;    // [k] -> d_y parts (N = 1)
  const float** d_yredptr = nullptr; // [1] -> d_yred
  int32_t* d_tok_in = nullptr;
  int32_t* d_tok_out = nullptr;
  int32_t* d_flag = nullptr;
  void* d_lmscratch = nullptr;
  float* d_lmlogits = nullptr;   // [V] (debug)

  // shadow work buffers (rank 0)
  float* sh_h = nullptr;
  void* sh_u = nullptr;
  int32_t* sh_ids = nullptr;     // [L][k]
  float* sh_w = nullptr;         // [L][k]
  float* sh_logits = nullptr;    // [L][E]
  float* sh_a = nullptr;         // [k][F]
  float* sh_y = nullptr;         // [k][d]
  const float** sh_yptr = nullptr;

  // pinned host mirrors
  int32_t* h_ids = nullptr;      // [L][k]
  float* h_w = nullptr;          // [L][k]
  int32_t* h_pred = nullptr;     // [L][k]
  int32_t* h_tok = nullptr;      // [2]: in, out
  int32_t* h_flag = nullptr;
  cudaEvent_t ev_ids = nullptr, ev_tok = nullptr, ev_shadow_done = nullptr, ev_step = nullptr;
  cudaEvent_t* ev_pred = nullptr;    // [L] view of ev_pred_all for this step's buffer (per layer at N = 1;
                                     // per chunk at N > 1)
  int pred_chunk = 4;

  // Prediction buffers: the shadow pass of step n writes buffer n & 1 (so a speculative pass for
  // n + 1 can run while step n still reads its own); buffer 2 belongs to odmoe_predict_ahead.
  // sh_ids / h_pred / sh_logits / dbg_sh_h / dbg_sh_u / ev_pred are views of this step's buffer.
  static constexpr int kPredBufs = 3;
  int32_t* sh_ids_all = nullptr;        // device [3][L][k]
  int32_t* h_pred_all = nullptr;        // pinned [3][L][k]
  float* sh_logits_all = nullptr;       // device [3][L][E]
  float* dbg_sh_h_all = nullptr;        // device [3][L][d] (debug capture)
  char* dbg_sh_u_all = nullptr;         // device [3][L][d*4] (debug capture)
  float* dbg_sh_hf_all = nullptr;       // device [3][d]: the shadow's final hidden state (debug capture)
  std::vector<cudaEvent_t> ev_pred_all; // [3][L]
  int cur_buf = 0;

  // Cross-token speculation (token alignment period T_p > 1): at iterations
  // n with n mod T_p != 0 the shadow decodes with its own greedy token (INT8-row LM head), so its pass
  // for n + 1 is enqueued right after the pass for n and loads of the next token's first layers may
  // be issued inside the lookahead window while the main model still decodes n.
  void* sh_lm = nullptr;                // shadow LM head [V][d] (int8-row; main / bf16 weights for SAME / BF16)
  float* sh_slm = nullptr;              // its row scales [V] (int8)
  int32_t* sh_tok = nullptr;            // device [3]: the shadow's own greedy token of each buffer's pass
  void* sh_lmscratch = nullptr;         // argmax scratch of the shadow LM head (own ticket)
  float* sh_lmlogits = nullptr;         // device [V] (debug capture)
  int align_period = 1;                 // T_p
  int64_t align_n = 0;                  // iteration index since the last alignment reset
  int64_t spec_step = -1;               // the step whose shadow pass is already enqueued (speculative)
  int next_plan_nx = 0;                 // next layer of the NEXT token whose predicted loads are unplanned
  std::vector<char> nx_ready;           // [L] next token's prediction of layer m on the host
  std::vector<int32_t> nx_tbl;          // [L][k]

  ncclComm_t comm = nullptr, comm_pred = nullptr;

  // per-step scheduler state
  int64_t step = 0;
  std::vector<char> pred_ready;  // [L]
  bool pred_valid = false;       // a prediction source exists this step
  int next_plan = 0;             // next layer whose predicted loads are not yet planned
  int l_cur = 0;
  std::vector<int32_t> pred_tbl; // [L][k] predictions this step (host)

  // SEP refinement ("Mode B"; refine_depth R > 0): after the main router of layer l the shadow
  // re-runs from the main's exact state (h_l, u_l, true ids of layer l) and predicts l+1..l+R.
  int R = 0;
  std::vector<cudaEvent_t> ev_router;   // [L] main router of layer l done (h_hist[l], pkt[l] valid)
  std::vector<cudaEvent_t> ev_ref;      // [L] refined predictions of refinement l on the host
  std::vector<char> ref_enq;            // [L] refinement l enqueued this step (its event is current)
  float* h_hist = nullptr;              // device [L][d] residual entering layer l (rank 0)
  float* rf_h = nullptr;
  void* rf_u = nullptr;
  int32_t* rf_ids = nullptr;            // device [L][4][k] refined ids (received at N > 1)
  float* rf_w = nullptr;                // device [4][k]
  float* rf_y = nullptr;                // device [k][d]
  float* rf_a = nullptr;                // device [k][F]
  const float** rf_yptr = nullptr;
  int32_t* h_ref = nullptr;             // pinned [L][4][k]
  int ref_next = 0;                     // next refinement to apply (host, this step)
  std::vector<int32_t> predA_tbl;       // [L][k] Mode A predictions (the paper's SEP: recall Eq. 3)
  std::vector<char> predA_ready;        // [L] Mode A prediction of layer l copied to predA_tbl
  std::vector<int32_t> predB_tbl;       // [L][k] refined predictions (-1 = none)

  // PERFECT predictor: routing recorded per input token (Mode A: routing is a function of the
  // token only, there is no KV state on the hot path)
  // PERFECT predictor: routing recorded per input token (and position, with attention)
  std::map<int64_t, std::vector<int32_t>> route_cache;
  int32_t predict_cache_token = -1;

  // kernel timing (time_kernels)
  struct Timed { int fam; cudaEvent_t a, b; int units; bool graph = false; };  // units: experts per launch
  cudaGraphExec_t graph_exec = nullptr;  // fully-resident 1-GPU step (captured once, replayed)
  int64_t graph_launches = 0;
  std::vector<Timed> graph_timers;
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> tev_pool;

  odmoe_stats stats{};

  // event trace (option key 7; odmoe_trace_read). Entries are kept in emission order; an entry is
  // resolved when its device event (if any) has completed and, for load entries, its request settled.
  struct TraceRec {
    odmoe_trace_event ev;
    cudaEvent_t e = nullptr;               // timing event (nullptr: host-only entry)
    std::shared_ptr<LoadReq> req;          // load entries: bytes + settled state
    bool own_event = true;                 // return `e` to the pool on resolution
  };
  int trace = 0;
  int pass_timing = 0;           // option 9: CUDA events around every whole shadow pass (stats.ms_sh_pass)
  cudaEvent_t tr_origin = nullptr;
  std::vector<TraceRec> tr_pending;
  std::vector<odmoe_trace_event> tr_done;
  std::vector<cudaEvent_t> tr_pool;

  // per-step load bookkeeping for the layer records (this rank): experts whose loads were issued
  // before the router ids reached the host / loaded after them (misprediction fallback)
  std::vector<std::vector<int>> issued_pre, reloaded;   // [L]
  std::vector<std::vector<int>> issued_nx;              // [L] the next token's early loads
  std::vector<char> in_time;                            // [L] prediction on the host before the router ids

  // prefill: batch buffers sized for T_cap tokens, E/G expert slots x 2 (double buffer)
  int T_cap = 0;
  float* p_h = nullptr;          // [T, d] residual
  char* p_pkt = nullptr;         // [T] u (bf16 [T,d]) | ids [T,k] | w [T,k]  (broadcast at N > 1)
  int64_t p_pkt_bytes = 0, p_ids_off = 0, p_w_off = 0;
  int32_t* p_tok = nullptr;      // [T]
  int32_t* p_off = nullptr;      // [E+1]
  int32_t* p_src = nullptr;      // [T*k]
  int32_t* p_inv = nullptr;      // [T*k]
  float* p_gate = nullptr;       // [T*k]
  void* p_x = nullptr;           // [T*k, d] bf16 grouped rows
  void* p_a2 = nullptr;          // [T*k, F] bf16
  float* p_y = nullptr;          // [T*k, d] fp32
  float* p_part = nullptr;       // [T, d] fp32 (N > 1 partial combine)
  int4* p_tiles = nullptr;       // [tiles_cap]
  int tiles_cap = 0;
  int32_t* h_off = nullptr;      // pinned [E+1]
  std::vector<Slot> pslots;
  std::vector<float> p_dbg;      // debug: [L+1][T][d] h per layer (rank 0)
  std::vector<int32_t> p_dbg_ids;  // [L][T][k]

  // debug capture (rank 0)
  float* dbg_h = nullptr;        // device [L][d]
  float* dbg_ypart = nullptr;    // device [L][k][d]
  float* dbg_yred = nullptr;     // device [L][d]
  float* dbg_sh_h = nullptr;     // device [L][d]
  void* dbg_sh_u = nullptr;      // device [L][d] bf16/dt
  float* dbg_hfinal = nullptr;   // device [d]
  std::vector<char> hdbg;        // host copy of everything after the step
  std::map<int, std::pair<int64_t, int64_t>> hdbg_index;  // what -> (offset, per-layer bytes)
};

}  // namespace odmoe
