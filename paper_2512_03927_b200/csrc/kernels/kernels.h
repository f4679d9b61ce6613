// Host-side launchers of the OD-MoE sm_100a kernels (internal to libodmoe.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace odmoe {

enum WType { W_BF16 = 0, W_F32 = 1, W_I8 = 2, W_NF4 = 3, W_F8 = 4, W_U8 = 5, W_I8P = 6 };
// W_I8P (INT8 shadow experts, mma_gemv.cu): the biased codes q + 128 in the fragment-packed layout of
// mma.sync m16n8k16 (16-row tiles x 32-column blocks of 512 B; W13 tiles pair gate/up rows), same
// natural-order row scales; expert blob = packed W13 (2Fd bytes) then packed W2 (dF bytes).
// W_U8 (shadow experts on the flat engine only): the INT8-row codes q stored as the byte q + 128,
// same row scales; the dot product then widens a byte without flipping its sign bit first.
// W_F8 (shadow experts only, reading Q28): E4M3 codes, one fp32 scale per row (int8's layout).
// W_NF4 (shadow experts only, reading Q27): two 4-bit codes per byte (low nibble = even column),
// "scales" = fp32 absmax per 64-weight block of a row, [R][C/64]; expert blob = codes of W13 then
// W2 (3dF/2 bytes), scale array = W13 blocks then W2 blocks.

int num_sms();  // cached SM count of the current device
int stream_grid_sms();            // num_sms() minus the reserve below (grid of the flat engine)
void set_stream_sm_reserve(int n);  // SMs the flat engine leaves free on the current device

// a2+a3: h += sum(y_add); u = RMSNorm(h) (rounded to u's dtype); logits = W_g u; top-k; softmax.
// wt: weight type of w_gate (W_I8 uses wg_scale[E]); u dtype = fp32 iff wt == W_F32, else bf16.
cudaError_t launch_router(float* h, const float* const* y_add, int n_add, const void* gamma,
                          const void* w_gate, const float* wg_scale, WType wt, int m, int E, int d,
                          int k, float eps, void* u_out, int32_t* ids, float* w, float* logits,
                          int32_t* flag, cudaStream_t s, bool pdl = false);

// h += (y_0 + ... + y_{n-1}) (final residual combine before the LM head).
cudaError_t launch_combine(float* h, const float* const* y_add, int n_add, int d, cudaStream_t s);

// Which expert a GEMV reads. Direct: blob/scales given. Indirect (tbl != NULL): the expert id is
// read on the device, so routing never round-trips through the host:
//   pick = sorted ? (index of the `sel`-th smallest id among ids[0..k)) : sel
//   blob = tbl[base + ids[pick]], scales = stbl ? stbl[base + ids[pick]] : NULL, gate = gate_w[pick]
// Blob layout: W13 [F][2][d] then W2 [d][F]; int8 scales: s13 [2F] then s2 [d].
struct ExpertRef {
  const void* blob;
  const float* scales;
  const void* const* tbl;
  const float* const* stbl;
  const int32_t* ids;
  int sel, base, k, sorted;
};
inline ExpertRef direct_ref(const void* blob, const float* scales, int gate_idx) {
  return ExpertRef{blob, scales, nullptr, nullptr, nullptr, gate_idx, 0, 0, 0};
}

// a8 phase 1: a[f] = silu(g_f) * v_f with [g_f; v_f] = W13[2f:2f+2] u (int8: row scales).
// pdl: launch with programmatic stream serialization (only when the previous operation on the
// stream is a kernel of this library; the weights are prefetched before the dependency wait).
cudaError_t launch_w13(ExpertRef ex, WType wt, const void* u, int u_f32, float* a, int d, int F,
                       cudaStream_t s, bool pdl = false);
// a8 phase 2: y = gate_w[pick] * (W2 a) (int8: row scales); gate_w may be NULL (=1).
cudaError_t launch_w2(ExpertRef ex, WType wt, const float* a, const float* gate_w, float* y, int d,
                      int F, cudaStream_t s, bool pdl = false);

// GEMV engines: 2 = flat per-warp streams (flat_gemv.cu, default), 0 = per-row register streaming
// (gemv.cu); env ODMOE_GEMV=flat|ldg. (The measured TMA bulk-ring engine of round 1 lives in
// tools/ab/stream_gemv.cu, outside the library.)
int gemv_engine();
cudaError_t launch_w13_flat(ExpertRef ex, WType wt, const void* u, int u_f32, float* a, int d, int F,
                            cudaStream_t s, bool pdl);
struct P2PSend;
cudaError_t launch_w2_flat(ExpertRef ex, WType wt, const float* act, const float* gate_w, float* y, int d,
                           int F, cudaStream_t s, bool pdl, const P2PSend* send = nullptr);
cudaError_t launch_lm_head_flat(const float* h, const void* W, WType wt, int V, int d, float eps,
                                int32_t* token_out, float* logits, void* scratch, cudaStream_t s, bool pdl,
                                const float* scales = nullptr);
bool use_fused_expert();  // env ODMOE_FUSED=0 disables (A/B)
// Graph capture of cooperative kernels: restart the grid-barrier targets of stream s at 0 and return
// its arrival counter (the captured step memsets it to 0 first, so every replay sees the same targets).
unsigned int* barrier_capture_reset(cudaStream_t s);
// NF4 / FP8 rows shorter than one flat group: warp-per-row kernel (x: bf16 unless x_f32; W2 x = fp32)
cudaError_t launch_lowbit_small(ExpertRef ex, WType wt, int second, const void* x, int x_f32, int d, int F,
                                const float* gate_w, float* out, cudaStream_t s);
// FP8 row quantiser (reading Q28): codes [R][C] E4M3, s [R]
cudaError_t launch_quantize_fp8(const void* w, int64_t R, int64_t C, WType wt, uint8_t* q, float* s, cudaStream_t st);
// NF4 blockwise quantiser (reading Q27): codes [R][C/2] bytes, absmax [R][C/64]; C % 64 == 0
cudaError_t launch_quantize_nf4(const void* w, int64_t R, int64_t C, WType wt, uint8_t* q, float* absmax,
                                cudaStream_t s);
// The P2P combine fused into the W2 epilogue of a GPU's LAST expert of a layer:
// every thread stores, for its rows, prev[0] + ... + prev[nprev-1] + (this expert's gated output) --
// the order of launch_p2p_send -- straight into GPU 0's receive row over NVLink as one 8-byte
// {value, epoch} pair (the format launch_p2p_gather polls; no fence, no flag, no counter).
struct P2PSend {
  float* dst;                 // this rank's row of GPU 0's buffer (peer memory), 2 words per element
  uint32_t epoch;
  const float* const* prev;   // device array: this GPU's earlier gated partials of the layer
  int nprev;
};

// Fused expert FFN (flat engine): W13+SwiGLU -> grid barrier -> W2+gate in ONE cooperative
// launch. Direct mode: ex.blob/ex.scales = W13 (+ scales), w2_direct/s2_direct = W2 (+ scales);
// indirect mode: the expert table entries (whole blobs). a_buf: fp32 [F] scratch.
// The n (<= 4) experts one GPU computes for a layer in ONE cooperative launch (W13 of all, one grid
// barrier, W2 of all); a_buf: fp32 [n][F]; y[i]: output of expert i (gate-weighted). bf16 / fp32.
cudaError_t launch_experts_fused(int n, const ExpertRef* ex, const void* const* w2_direct, const float* const* s2_direct,
                                 WType wt, const void* u, int u_f32, float* a_buf, const float* gate_w,
                                 float* const* y, int d, int F, cudaStream_t s, bool pdl,
                                 const P2PSend* send = nullptr);  // send: fused into the last expert
// The n (<= 4) experts of one layer, one phase per launch, not cooperative (the shadow's k experts):
// W13+SwiGLU of all -> a_buf [n][F]; W2+gate of all -> y_buf [n][d]. Each expert's result is bitwise
// that of launch_w13 / launch_w2; shapes the flat engine does not take fall back to those launches.
bool multi_flat_ok(int n, WType wt, int d, int F);  // one launch per phase for these shapes
cudaError_t launch_w13_multi(int n, const ExpertRef* ex, WType wt, const void* u, int u_f32, float* a_buf, int d,
                             int F, cudaStream_t s, bool pdl);
cudaError_t launch_w2_multi(int n, const ExpertRef* ex, WType wt, const float* a_buf, const float* gate_w, float* y_buf,
                            int d, int F, cudaStream_t s, bool pdl);
cudaError_t launch_expert_fused(ExpertRef ex, const void* w2_direct, const float* s2_direct, WType wt,
                                const void* u, int u_f32, float* a_buf, const float* gate_w, float* y, int d,
                                int F, cudaStream_t s, bool pdl, const P2PSend* send = nullptr);
// Rows the flat engine takes for a [R, C] matrix of type wt (whole 512-byte groups).
bool stream_ok(WType wt, int C);

// a10: token = argmax_v (W_o RMSNorm(h))_v, lowest id on ties. scratch >= 8*(grid+2) bytes.
// W_I8 (the shadow's LM head, cross-token speculation): logit_v = scales[v] * (q_v . bf16(RMSNorm(h))).
cudaError_t launch_lm_head(const float* h, const void* W, WType wt, int V, int d, float eps,
                           int32_t* token_out, float* logits, void* scratch, cudaStream_t s,
                           bool pdl = false, const float* scales = nullptr);

// a1: h = Emb[token] (fp32); int8 rows use emb_scale.
cudaError_t launch_embed(const void* emb, const float* emb_scale, WType wt, const int32_t* token,
                         int d, float* h, cudaStream_t s);

// Prefill grouped expert GEMM on tcgen05. Tiles are {expert, row0, rows, n0} (device
// int4 array): rows [row0, row0+rows) of A belong to `expert`; A is [M, K] bf16 (rows of all
// experts, grouped), b[e] is expert e's [N, K] bf16 matrix (K-major), out is
// mode 0: SwiGLU of interleaved column pairs -> bf16 [M, N/2]; mode 1: gate[row] * C -> fp32 [M, N].
constexpr int kMaxGGExperts = 8;
struct GroupedGemmArgs {
  const void* a;
  const void* b[kMaxGGExperts];
  int n_experts;
  const int4* tiles;
  int n_tiles;
  int M, N, K;
  int mode;
  void* out;
  const float* gate;
};
cudaError_t launch_grouped_gemm(const GroupedGemmArgs& g, cudaStream_t s);
int grouped_gemm_bn(int mode, int N);  // output-tile width for the mode and N (tile n0 step)
int grouped_gemm_bm();          // rows per tile (tile row0 step, <= 256)

// Prefill permutation: stable counting sort of the T*k pairs by expert.
cudaError_t launch_route_group(const int32_t* ids, const float* w, int n_pairs, int E, int32_t* offsets,
                               int32_t* src_pair, int32_t* inv, float* gate_perm, cudaStream_t s);
cudaError_t launch_gather_rows(const void* u, const int32_t* src_pair, int k, int M, int d, void* out,
                               cudaStream_t s);
// h[t] += sum_j y[inv[t*k+j]] (partial == 0), or h[t] = that sum (partial == 1, N > 1 share).
cudaError_t launch_scatter_combine(float* h, const float* y, const int32_t* inv, int T, int k, int d,
                                   int partial, cudaStream_t s);
cudaError_t launch_add_rows(float* h, const float* y, long long n, cudaStream_t s);
cudaError_t launch_embed_rows(const void* emb, WType wt, const int32_t* tokens, int T, int d, float* h,
                              cudaStream_t s);

// Synthetic weights. kind 1..6 plain tensor rows x cols; kind 0 = expert blob.
cudaError_t launch_gen(void* out, int kind, int layer, int expert, int64_t rows, int64_t cols,
                       int64_t fan_in, int d, int F, uint64_t seed, WType wt, cudaStream_t s);

// ---- attention block (reading Q29; attention.cu + flat_gemv.cu)
// out[R] = W RMSNorm(h) (flat GEMV, RMSNorm fused in the prologue); needs (C * elem) % 512 == 0
cudaError_t launch_gemv_rmsnorm(const float* h, const void* W, const float* scales, WType wt, int R, int C, float eps,
                                float* out, cudaStream_t s, bool pdl);
// out[R] += W x (x fp32 [C])
cudaError_t launch_gemv_acc(const void* W, const float* scales, WType wt, int R, int C, const float* x, float* out,
                            cudaStream_t s, bool pdl);
// rotate q, k of T positions pos0.. in qkv rows ([q H*hd | k Hkv*hd | v Hkv*hd], fp32, stride
// qkv_stride); k (rotated) and v stored as rows of kv_stride elements at kc / vc (row t), bf16 or
// (kv_f32) fp32
cudaError_t launch_rope_kv(float* qkv, int qkv_stride, int T, int H, int Hkv, int hd, int pos0, void* kc, void* vc,
                           int kv_stride, int kv_f32, cudaStream_t s);
// causal GQA attention of T queries at positions pos0..: keys/values < pos0 from *_past (rows by
// position), >= pos0 from *_cur (row t = position pos0 + t); part: attn_part_floats(...) fp32;
// o [T][H*hd] as fp32 and/or bf16 (either may be NULL)
int attn_splits(int max_pos);
cudaError_t launch_rmsnorm_rows(const float* h, int T, int d, float eps, void* x_bf16, cudaStream_t s);
cudaError_t launch_attention(const float* q, int q_stride, int T, int H, int Hkv, int hd, int pos0, const void* kc_past,
                             const void* vc_past, const void* kc_cur, const void* vc_cur, int kv_stride, int kv_f32,
                             float* part, float* o_f32, void* o_bf16, int o_stride, cudaStream_t s);

// P2P combine over NVLink (p2p.cu): sender sums its n partials into its row of GPU 0's buffer as
// {value, epoch} pairs (2 words per element; no fence, no flag); GPU 0 polls the rows in `mask` until
// every pair carries `epoch` and sums them in rank order.
cudaError_t launch_p2p_send(const float* const* y, int n, int d, float* dst, uint32_t epoch, cudaStream_t s);
cudaError_t launch_p2p_gather(const float* part, uint32_t mask, int d, uint32_t epoch, float* out, int32_t* err_flag,
                              cudaStream_t s);

// INT8 shadow experts on the tensor cores (mma_gemv.cu): one phase (mode 0 = W13 + SwiGLU -> out
// [n][F], x = bf16 u; mode 1 = W2 + gate -> out [n][d], x = fp32 a [n][F]) of n <= 4 W_I8P experts.
bool mma_shadow_ok(int d, int F);
cudaError_t launch_mma_shadow(int n, const ExpertRef* ex, int mode, const void* x, const float* gate_w,
                              float* out, int d, int F, cudaStream_t s, bool pdl);
// Both phases of the n W_I8P experts (indirect refs) in ONE cooperative launch with a grid barrier.
cudaError_t launch_mma_shadow_layer(int n, const ExpertRef* ex, const void* u, float* a_buf, const float* gate_w,
                                    float* y_buf, int d, int F, cudaStream_t s, bool pdl);
// Next grid-barrier target of stream s for a cooperative grid of `grid` CTAs (flat engine's counter).
cudaError_t coop_barrier_next(cudaStream_t s, int grid, unsigned int** counter, unsigned int* target);
// biased codes [R][C] (row-major) -> W_I8P layout; pair_rows: W13's gate/up pairing
cudaError_t launch_pack_i8_frag(const uint8_t* q_biased, uint8_t* out, int R, int C, int pair_rows, cudaStream_t s,
                                bool signed_codes = false);  // signed_codes: input q (not q + 128)

// One warp spins until *flag reaches epoch (the copy stream writes it after a load): keeps the GPU out of
// its idle state while the compute stream waits for an expert (p2p.cu). Timeout ~30 s -> *err_flag = 3.
cudaError_t launch_wait_flag(const uint32_t* flag, uint32_t epoch, int32_t* err_flag, cudaStream_t s);

// BF16 (round to nearest even) copy of an fp32 tensor: the BF16 shadow of an FP32 main model.
cudaError_t launch_f32_to_bf16(const float* in, void* out, int64_t n, cudaStream_t s);

// Q9 int8-row quantiser of a [R, C] matrix of type wt (bf16 / fp32).
cudaError_t launch_quantize(const void* w, int64_t R, int64_t C, WType wt, int8_t* q, float* sc,
                            cudaStream_t s,
                            bool biased = false);  // biased: store q + 128 (W_U8)

}  // namespace odmoe
