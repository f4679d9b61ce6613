// C ABI of libodmoe.so: stateless kernel entry points and the stateful OD-MoE decode engine.
// Contract: include/odmoe.h. Design: DESIGN.md §5-§7.
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"

using namespace odmoe;

namespace {

thread_local std::string t_create_err;

struct Fail {
  odmoe_status st;
};

// Every internal error path throws Fail (caught at the ABI boundary).
[[noreturn]] void fail(Ctx* c, odmoe_status st, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (st == ODMOE_E_CUDA || st == ODMOE_E_NCCL) c->poisoned = true;
  } else {
    t_create_err = msg;
  }
  throw Fail{st};
}

#define CUDA_OK(c, x)                                                                          \
  do {                                                                                         \
    cudaError_t _e = (x);                                                                      \
    if (_e != cudaSuccess)                                                                     \
      fail((c), ODMOE_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e) + " @" +         \
                                  std::to_string(__LINE__));                                   \
  } while (0)

#define NCCL_OK(c, x)                                                                          \
  do {                                                                                         \
    ncclResult_t _r = (x);                                                                     \
    if (_r != ncclSuccess)                                                                     \
      fail((c), ODMOE_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(_r));                \
  } while (0)

template <typename F>
odmoe_status guard(Ctx* c, F&& f) {
  try {
    f();
    return ODMOE_OK;
  } catch (const Fail& e) {
    return e.st;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return ODMOE_E_NOMEM;
  } catch (...) {
    if (c) c->err = "unexpected exception";
    return ODMOE_E_STATE;
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool is_shadow(int p) {
  return p == ODMOE_PRED_SHADOW_INT8 || p == ODMOE_PRED_SHADOW_SAME || p == ODMOE_PRED_SHADOW_BF16 ||
         p == ODMOE_PRED_SHADOW_NF4 || p == ODMOE_PRED_SHADOW_FP8;
}
inline WType wtype(int dt) { return dt == ODMOE_FP32 ? W_F32 : W_BF16; }
inline size_t dsize(int dt) { return dt == ODMOE_FP32 ? 4 : 2; }
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename T>
T* dmalloc(Ctx* c, size_t n, const char* what) {
  void* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) fail(c, ODMOE_E_NOMEM, std::string("cudaMalloc ") + what + " (" + std::to_string(n * sizeof(T)) + " B): " + cudaGetErrorString(e));
  return reinterpret_cast<T*>(p);
}

template <typename T>
T* hmalloc(Ctx* c, size_t n, const char* what) {
  void* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable);
  if (e != cudaSuccess) fail(c, ODMOE_E_NOMEM, std::string("cudaHostAlloc ") + what + " (" + std::to_string(n * sizeof(T)) + " B): " + cudaGetErrorString(e));
  return reinterpret_cast<T*>(p);
}

// ------------------------------------------------------------------ kernel timing + counting
struct KTimer {
  Ctx* c;
  int fam;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  int units;
  KTimer(Ctx* c_, int fam_, cudaStream_t s_, int units_ = 1) : c(c_), fam(fam_), s(s_), units(units_) {
    c->stats.kernel_launches++;
    // level 1: only the expert FFN launches (the roofline kernel) -- events between kernels cut the
    // programmatic-dependent-launch overlap, so the other families are timed only at level 2
    if (!c->cfg.time_kernels || (c->cfg.time_kernels == 1 && fam != K_W13 && fam != K_W2)) return;
    a = get();
    b = get();
    record(a);
  }
  ~KTimer() {
    if (!a) return;
    record(b);
    c->timed.push_back(Ctx::Timed{fam, a, b, units, false});
  }
  // inside a stream capture a plain record is only a dependency marker; External makes it a
  // timestamp node of the graph
  void record(cudaEvent_t e) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  }
  cudaEvent_t get() {
    if (!c->tev_pool.empty()) {
      cudaEvent_t e = c->tev_pool.back();
      c->tev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

void harvest_timers(Ctx* c) {
  for (auto& t : c->timed) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
      switch (t.fam) {
        case K_ROUTER: c->stats.ms_router += ms; c->stats.n_router++; break;
        case K_W13: c->stats.ms_w13 += ms; c->stats.n_w13 += t.units; break;
        case K_W2: c->stats.ms_w2 += ms; c->stats.n_w2++; break;
        case K_SHADOW: c->stats.ms_shadow += ms; c->stats.n_shadow++; break;
        case K_LM: c->stats.ms_lm_head += ms; c->stats.n_lm_head++; break;
        case K_EMBED: c->stats.ms_embed += ms; c->stats.n_embed++; break;
        case K_ATTN: c->stats.ms_attn += ms; c->stats.n_attn++; break;
        case K_SH_W13:  // the shadow's expert phases also count in ms_shadow
          c->stats.ms_shadow += ms; c->stats.n_shadow++; c->stats.ms_sh_w13 += ms; c->stats.n_sh_w13 += t.units; break;
        case K_SH_W2:
          c->stats.ms_shadow += ms; c->stats.n_shadow++; c->stats.ms_sh_w2 += ms; c->stats.n_sh_w2 += t.units; break;
        case K_SH_PASS: c->stats.ms_sh_pass += ms; c->stats.n_sh_pass++; break;
      }
    }
    if (!t.graph) {  // graph-owned events stay with the graph
      c->tev_pool.push_back(t.a);
      c->tev_pool.push_back(t.b);
    }
  }
  c->timed.clear();
}

// ------------------------------------------------------------------ event trace
cudaEvent_t tr_event(Ctx* c) {
  if (!c->tr_pool.empty()) {
    cudaEvent_t e = c->tr_pool.back();
    c->tr_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  CUDA_OK(c, cudaEventCreate(&e));
  return e;
}

odmoe_trace_event tr_make(const Ctx* c, int type, int layer, int expert, int slot, int l_cur, int aux, int64_t step) {
  odmoe_trace_event ev{};
  ev.type = type;
  ev.step = (int32_t)step;
  ev.layer = layer;
  ev.expert = expert;
  ev.slot = slot;
  ev.l_cur = l_cur;
  ev.aux = aux;
  ev.rank = c->rank;
  ev.bytes = 0;
  ev.t_us = std::nan("");
  return ev;
}

// host-only entry (t_us = NaN); `req` makes it wait for that load to settle (bytes copied)
void tr_host(Ctx* c, int type, int layer, int expert, int slot, int aux, std::shared_ptr<LoadReq> req = nullptr) {
  if (!c->trace) return;
  Ctx::TraceRec r;
  r.ev = tr_make(c, type, layer, expert, slot, c->l_cur, aux, c->step);
  r.req = std::move(req);
  c->tr_pending.push_back(std::move(r));
}

// device-timed entry: an event recorded on `s` now
void tr_dev(Ctx* c, int type, cudaStream_t s, int layer, int expert = -1, int slot = -1) {
  if (!c->trace) return;
  Ctx::TraceRec r;
  r.ev = tr_make(c, type, layer, expert, slot, c->l_cur, 0, c->step);
  r.e = tr_event(c);
  CUDA_OK(c, cudaEventRecord(r.e, s));
  c->tr_pending.push_back(std::move(r));
}

// Move every resolvable entry (in order) to tr_done.
void tr_resolve(Ctx* c) {
  std::vector<Ctx::TraceRec> keep;
  for (auto& r : c->tr_pending) {
    int64_t bytes = 0;
    if (r.req && !c->loader.settled(r.req, &bytes)) { keep.push_back(std::move(r)); continue; }
    if (r.e) {
      const cudaError_t q = cudaEventQuery(r.e);
      if (q == cudaErrorNotReady) { keep.push_back(std::move(r)); continue; }
      float ms = 0.f;
      if (q == cudaSuccess && cudaEventElapsedTime(&ms, c->tr_origin, r.e) == cudaSuccess) r.ev.t_us = 1e3 * (double)ms;
      cudaGetLastError();  // never-recorded events (a load stopped before its first chunk) leave NaN
      if (r.own_event) c->tr_pool.push_back(r.e);
    }
    if (r.req) r.ev.bytes = bytes;
    c->tr_done.push_back(r.ev);
  }
  c->tr_pending.swap(keep);
}

// ------------------------------------------------------------------ placement
// Pure placement functions (also exported as odmoe_plan_* for host-side tests).
// Experts of layer l that `rank` computes for routing S (k ids): none unless the rank is in group
// l mod N_G; sorted experts paired with sorted group GPUs; with G < k a GPU takes k/G
// consecutive sorted experts (reading Q14).
int plan_layer(int k, int world, int G, int l, const int32_t* S, int rank, int32_t* out) {
  const int NG = world / G;
  if ((l % NG) != rank / G) return 0;
  const int pos = rank % G;
  int32_t s[8];
  if (k < 1 || k > 8) return 0;
  for (int i = 0; i < k; ++i) s[i] = S[i];
  // insertion sort (k <= 8)
  for (int i = 1; i < k; ++i)
    for (int j = i; j > 0 && s[j - 1] > s[j]; --j) std::swap(s[j - 1], s[j]);
  int n = 0;
  for (int i = 0; i < k; ++i)
    if (i * G / k == pos) out[n++] = s[i];
  return n;
}

// Can the sorted pairing ever send (l, e) to `rank`? Position p receives the i-th smallest of k
// distinct ids for i in [p*k/G, (p+1)*k/G), so it needs >= p*k/G smaller and >= (G-1-p)*k/G larger
// ids among E experts.
bool plan_pool_holds(int E, int k, int world, int G, int l, int e, int rank) {
  if (G == 0) return true;  // sliced placement: every rank holds a slice of every expert
  const int NG = world / G;
  if ((l % NG) != rank / G) return false;
  const int pos = rank % G;
  const int lo = pos * (k / G);
  const int hi = (G - 1 - pos) * (k / G);
  return e >= lo && e <= E - 1 - hi;
}

std::vector<int> my_experts(const Ctx* c, int l, const int32_t* S) {
  if (c->sliced) return std::vector<int>(S, S + c->k);  // every rank: its slice of all k experts
  int32_t buf[8];
  const int n = plan_layer(c->k, c->world, c->G, l, S, c->rank, buf);
  return std::vector<int>(buf, buf + n);
}

bool holds_expert(const Ctx* c, int l, int e) { return c->pool_off[(size_t)l * c->E + e] >= 0; }

// Expert weights of layer l are generated as those of layer l mod P (config expert_layer_period P;
// 0 => every layer its own). The host pool then holds P layers' blobs and layer l's loads read layer
// (l mod P)'s: the bytes per load and the loads per token are those of the full model.
int wl(const Ctx* c, int l) { return c->elp > 0 ? l % c->elp : l; }

// ------------------------------------------------------------------ validation
void validate(const odmoe_config* g) {
  auto bad = [](const std::string& m) { fail(nullptr, ODMOE_E_CONFIG, m); };
  if (!g) bad("null config");
  if (g->L < 1 || g->E < 1 || g->k < 1 || g->d < 8 || g->F < 8 || g->V < 2) bad("non-positive dimension");
  if (g->k > g->E || g->k > 8 || g->E > 64) bad("need 1 <= k <= E <= 64 and k <= 8");
  if (g->d % 8 || g->F % 8) bad("d and F must be multiples of 8");
  if (g->dtype != ODMOE_BF16 && g->dtype != ODMOE_FP32) bad("dtype");
  if (g->predictor < 0 || g->predictor > 8) bad("predictor");
  if (g->placement != ODMOE_PLACE_GROUPS && g->placement != ODMOE_PLACE_SLICED) bad("placement");
  if (g->placement == ODMOE_PLACE_SLICED && g->world_size > 1) {
    if (g->F % (16 * g->world_size)) bad("sliced placement needs F % (16 N) == 0");
    if (g->predictor == ODMOE_PRED_SHADOW_SAME) bad("sliced placement: SHADOW_SAME keeps whole experts");
    if (g->group_size != 0) bad("sliced placement: group_size must be 0");
    if (g->slots_per_gpu != -1 && g->slots_per_gpu < 1) bad("slots_per_gpu must be >= 1 or -1");
  }
  if (g->predictor == ODMOE_PRED_SHADOW_NF4 && (g->d % 64 || g->F % 64)) bad("the NF4 shadow needs d, F multiples of 64");
  if (g->emulate_world > 1) {
    const int N = g->emulate_world;
    if (N != 2 && N != 4 && N != 8) bad("emulate_world must be 0, 1, 2, 4 or 8");
    if (g->world_size != 1) bad("emulate_world runs on one GPU (world_size 1)");
    if (g->slots_per_gpu == -1) bad("emulate_world: on-demand decode only");
    if (g->placement == ODMOE_PLACE_SLICED && g->F % (16 * N)) bad("emulated sliced placement needs F % (16 N) == 0");
    if (g->placement == ODMOE_PLACE_GROUPS) {
      const int Ge = g->group_size > 0 ? g->group_size : std::min(g->k, N);
      if (N % Ge || g->k % Ge) bad("emulate_world: N and k must be divisible by the group size");
    }
  } else if (g->emulate_world < 0) {
    bad("emulate_world must be 0, 1, 2, 4 or 8");
  }
  if (g->expert_layer_period < 0 || g->expert_layer_period > g->L) bad("expert_layer_period must be in 0..L");
  if (g->expert_layer_period > 0 && g->world_size > 1 && g->placement == ODMOE_PLACE_GROUPS)
    bad("expert_layer_period: groups placement at N > 1 keeps per-layer pools (use sliced)");
  if (g->lookahead < 1) bad("lookahead must be >= 1");
  if (g->world_size < 1 || g->rank < 0 || g->rank >= g->world_size) bad("rank/world_size");
  const int G = g->group_size > 0 ? g->group_size : std::min(g->k, g->world_size);
  if (g->world_size % G && g->emulate_world <= 1) bad("world_size must be divisible by the group size (S:251, S:269)");
  if (g->k % G) bad("k must be divisible by the group size");
  if (g->slots_per_gpu != -1 && g->slots_per_gpu < 1) bad("slots_per_gpu must be >= 1 or -1");
  if (g->world_size > 1 && g->nccl_id == nullptr) bad("nccl_id required when world_size > 1");
  if (g->refine_depth < 0 || g->refine_depth > 4) bad("refine_depth must be in 0..4");
  if (g->refine_depth > 0 && !is_shadow(g->predictor)) bad("refine_depth needs a shadow predictor");
  if (g->predictor == ODMOE_PRED_SHADOW_BF16 && g->dtype != ODMOE_FP32)
    bad("the BF16 shadow is for an FP32 main model");
  if (g->refine_depth > 0 && g->dtype != ODMOE_BF16) bad("refine_depth needs the bf16 model");
  if (g->n_heads < 0 || g->n_kv_heads < 0 || g->max_seq < 0) bad("attention sizes");
  if (g->n_heads > 0) {
    const int hd = g->d / g->n_heads;
    if (g->d % g->n_heads || (hd != 32 && hd != 64 && hd != 128)) bad("attention: head_dim = d / n_heads must be 32, 64 or 128");
    if (g->n_kv_heads < 1 || g->n_heads % g->n_kv_heads || g->n_heads / g->n_kv_heads > 8)
      bad("attention: n_heads % n_kv_heads == 0 and n_heads / n_kv_heads <= 8");
    if (g->predictor == ODMOE_PRED_SHADOW_BF16) bad("attention: the BF16 shadow has no attention weights yet");
    if (((int64_t)g->d * (g->dtype == ODMOE_FP32 ? 4 : 2)) % 512) bad("attention: d * sizeof(dtype) % 512 == 0");
  }
}

// ------------------------------------------------------------------ setup
void build_nonexpert(Ctx* c) {
  const int L = c->L, E = c->E, d = c->d, V = c->V;
  const uint64_t seed = c->cfg.weight_seed;
  c->d_emb = dmalloc<char>(c, (size_t)V * d * c->esz, "emb");
  c->d_lm = dmalloc<char>(c, (size_t)V * d * c->esz, "lm_head");
  c->d_router = dmalloc<char>(c, (size_t)L * E * d * c->esz, "router");
  CUDA_OK(c, launch_gen(c->d_emb, 1, 0, 0, V, d, d, d, c->F, seed, c->wt, c->s_main));
  CUDA_OK(c, launch_gen(c->d_lm, 6, 0, 0, V, d, d, d, c->F, seed, c->wt, c->s_main));
  for (int l = 0; l < L; ++l)
    CUDA_OK(c, launch_gen((char*)c->d_router + (size_t)l * E * d * c->esz, 2, l, 0, E, d, d, d, c->F, seed, c->wt, c->s_main));
  if (c->H > 0) {
    // fused QKV rows [q H*hd | k Hkv*hd | v Hkv*hd] x d and W_o [d][H*hd] per layer; KV cache
    const size_t qkv = (size_t)c->qkv_rows * d * c->esz, wo = (size_t)d * c->H * c->hd * c->esz;
    c->d_wqkv = dmalloc<char>(c, qkv * L, "wqkv");
    c->d_wo = dmalloc<char>(c, wo * L, "wo");
    for (int l = 0; l < L; ++l) {
      char* b = (char*)c->d_wqkv + qkv * l;
      const int64_t qr = (int64_t)c->H * c->hd, kr = (int64_t)c->kvd;
      CUDA_OK(c, launch_gen(b, 9, l, 0, qr, d, d, d, c->F, seed, c->wt, c->s_main));
      CUDA_OK(c, launch_gen(b + qr * d * c->esz, 10, l, 0, kr, d, d, d, c->F, seed, c->wt, c->s_main));
      CUDA_OK(c, launch_gen(b + (qr + kr) * d * c->esz, 11, l, 0, kr, d, d, d, c->F, seed, c->wt, c->s_main));
      CUDA_OK(c, launch_gen((char*)c->d_wo + wo * l, 12, l, 0, d, qr, d, d, c->F, seed, c->wt, c->s_main));
    }
    const size_t kv = (size_t)L * c->max_seq * c->kvd * c->kv_esz;
    c->d_kc = dmalloc<char>(c, kv, "k cache");
    c->d_vc = dmalloc<char>(c, kv, "v cache");
    CUDA_OK(c, cudaMemsetAsync(c->d_kc, 0, kv, c->s_main));
    CUDA_OK(c, cudaMemsetAsync(c->d_vc, 0, kv, c->s_main));
  }
}

// Attention block of layer l at position c->pos on stream s: h += W_o attn(RMSNorm(h)) (Q29).
// Main model: its weights, k/v of this position written into the cache. Shadow: int8-row weights,
// this position's k/v in a private buffer, earlier positions from the MAIN model's cache (KV
// alignment).
void enqueue_attention(Ctx* c, int l, cudaStream_t s, float* h, bool shadow, bool mode_a = false) {
  const int d = c->d, hq = c->H * c->hd;
  const size_t kv_l = (size_t)l * c->max_seq * c->kvd * c->kv_esz;
  char* kc = (char*)c->d_kc + kv_l;
  char* vc = (char*)c->d_vc + kv_l;
  const size_t cur = (size_t)c->pos * c->kvd * c->kv_esz;
  const int kvf = c->kv_esz == 4;
  if (!shadow) {
    const size_t qkv = (size_t)c->qkv_rows * d * c->esz, wo = (size_t)d * hq * c->esz;
    { KTimer t(c, K_ATTN, s);
      CUDA_OK(c, launch_gemv_rmsnorm(h, (const char*)c->d_wqkv + qkv * l, nullptr, c->wt, c->qkv_rows, d,
                                     c->cfg.rms_eps, c->d_qkv, s, true)); }
    { KTimer t(c, K_ATTN, s);
      CUDA_OK(c, launch_rope_kv(c->d_qkv, c->qkv_rows, 1, c->H, c->Hkv, c->hd, (int)c->pos, kc + cur, vc + cur,
                                c->kvd, kvf, s)); }
    { KTimer t(c, K_ATTN, s);
      CUDA_OK(c, launch_attention(c->d_qkv, c->qkv_rows, 1, c->H, c->Hkv, c->hd, (int)c->pos, kc, vc, kc + cur,
                                  vc + cur, c->kvd, kvf, c->d_attn_part, c->d_attn_o, nullptr, hq, s)); }
    { KTimer t(c, K_ATTN, s);
      CUDA_OK(c, launch_gemv_acc((const char*)c->d_wo + wo * l, nullptr, c->wt, d, hq, c->d_attn_o, h, s, true)); }
    return;
  }
  const bool same = c->sh_wt != W_I8;  // SHADOW_SAME: the main weights
  const size_t qkv = (size_t)c->qkv_rows * d * (same ? c->esz : 1), wo = (size_t)d * hq * (same ? c->esz : 1);
  // KV0: past positions from the shadow's own cache; its token-aligned pass (Mode A) appends this
  // position there, the refinement passes use the private buffer
  void* kcur = c->sh_kcur;
  void* vcur = c->sh_vcur;
  if (!c->kv_align) {
    kc = (char*)c->sh_kc + kv_l;
    vc = (char*)c->sh_vc + kv_l;
    if (mode_a) {
      kcur = kc + cur;
      vcur = vc + cur;
    }
  }
  { KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_gemv_rmsnorm(h, (const char*)c->sh_wqkv + qkv * l,
                                   same ? nullptr : c->sh_sqkv + (size_t)l * c->qkv_rows, c->sh_wt, c->qkv_rows, d,
                                   c->cfg.rms_eps, c->sh_qkv, s, true)); }
  { KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_rope_kv(c->sh_qkv, c->qkv_rows, 1, c->H, c->Hkv, c->hd, (int)c->pos, kcur, vcur,
                              c->kvd, kvf, s)); }
  { KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_attention(c->sh_qkv, c->qkv_rows, 1, c->H, c->Hkv, c->hd, (int)c->pos, kc, vc, kcur,
                                vcur, c->kvd, kvf, c->sh_attn_part, c->sh_attn_o, nullptr, hq, s)); }
  { KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_gemv_acc((const char*)c->sh_wo + wo * l, same ? nullptr : c->sh_so + (size_t)l * d, c->sh_wt,
                               d, hq, c->sh_attn_o, h, s, true)); }
}

void build_shadow(Ctx* c, char* staging) {
  const int L = c->L, E = c->E, d = c->d, V = c->V, F = c->F;
  if (c->cfg.predictor == ODMOE_PRED_SHADOW_SAME) {
    // The shadow runs the main model's own weights (recall must be exactly 1.0).
    c->sh_wt = c->sh_ewt = c->wt;
    c->sh_emb = c->d_emb;
    c->sh_lm = c->d_lm;
    c->sh_router = c->d_router;
    c->sh_wqkv = c->d_wqkv;
    c->sh_wo = c->d_wo;
    c->d_sh_tbl = c->d_res_tbl;
    c->d_sh_stbl = nullptr;
    return;
  }
  if (c->cfg.predictor == ODMOE_PRED_SHADOW_BF16) {
    // BF16 copy of the FP32 main model (round to nearest even), no scales
    c->sh_wt = c->sh_ewt = W_BF16;
    c->sh_emb = dmalloc<char>(c, (size_t)V * d * 2, "shadow emb bf16");
    c->sh_router = dmalloc<char>(c, (size_t)L * E * d * 2, "shadow router bf16");
    c->sh_lm = dmalloc<char>(c, (size_t)V * d * 2, "shadow lm head bf16");
    CUDA_OK(c, launch_f32_to_bf16((const float*)c->d_emb, c->sh_emb, (int64_t)V * d, c->s_main));
    CUDA_OK(c, launch_f32_to_bf16((const float*)c->d_lm, c->sh_lm, (int64_t)V * d, c->s_main));
    CUDA_OK(c, launch_f32_to_bf16((const float*)c->d_router, c->sh_router, (int64_t)L * E * d, c->s_main));
    c->sh_blob.assign((size_t)L * E, nullptr);
    c->sh_sc.assign((size_t)L * E, nullptr);
    for (int l = 0; l < L; ++l)
      for (int e = 0; e < E; ++e) {
        const size_t i = (size_t)l * E + e;
        char* q = dmalloc<char>(c, (size_t)3 * F * d * 2, "shadow expert bf16");
        CUDA_OK(c, launch_gen(staging, 0, wl(c, l), e, 0, 0, 0, d, F, c->cfg.weight_seed, c->wt, c->s_main));
        CUDA_OK(c, launch_f32_to_bf16((const float*)staging, q, 3LL * F * d, c->s_main));
        c->sh_blob[i] = q;
        c->stats.shadow_bytes += (int64_t)3 * F * d * 2;
      }
    c->stats.shadow_bytes += (int64_t)2 * V * d * 2 + (int64_t)L * E * d * 2;
    c->d_sh_tbl = dmalloc<void*>(c, (size_t)L * E, "shadow tbl");
    c->d_sh_stbl = nullptr;
    CUDA_OK(c, cudaMemcpyAsync(c->d_sh_tbl, c->sh_blob.data(), sizeof(void*) * L * E, cudaMemcpyHostToDevice, c->s_main));
    CUDA_OK(c, cudaStreamSynchronize(c->s_main));
    return;
  }
  const bool nf4 = c->cfg.predictor == ODMOE_PRED_SHADOW_NF4;
  const bool fp8 = c->cfg.predictor == ODMOE_PRED_SHADOW_FP8;
  c->sh_wt = W_I8;
  // INT8 experts on the flat engine are stored biased (W_U8: q + 128), which saves the sign flip of
  // every weight word in the dot product; other shapes keep signed codes (ODMOE_SHADOW_U8=0: A/B)
  const char* u8e = getenv("ODMOE_SHADOW_U8");
  const bool u8 = !nf4 && !fp8 && !(u8e && u8e[0] == '0') && gemv_engine() == 2 && stream_ok(W_U8, d) &&
                  stream_ok(W_U8, F);
  // INT8 experts on the tensor cores (mma_gemv.cu): biased codes in the fragment-packed layout;
  // ODMOE_SHADOW_MMA=0 keeps the CUDA-core flat engine (A/B)
  const char* mme = getenv("ODMOE_SHADOW_MMA");
  const bool mma = !nf4 && !fp8 && !(mme && mme[0] == '0') && mma_shadow_ok(d, F);
  c->sh_ewt = nf4 ? W_NF4 : (fp8 ? W_F8 : (mma ? W_I8P : (u8 ? W_U8 : W_I8)));
  c->sh_emb = dmalloc<int8_t>(c, (size_t)V * d, "shadow emb");
  c->sh_semb = dmalloc<float>(c, V, "shadow emb scales");
  c->sh_router = dmalloc<int8_t>(c, (size_t)L * E * d, "shadow router");
  c->sh_srouter = dmalloc<float>(c, (size_t)L * E, "shadow router scales");
  CUDA_OK(c, launch_quantize(c->d_emb, V, d, c->wt, (int8_t*)c->sh_emb, c->sh_semb, c->s_main));
  // int8-row LM head: the shadow's own greedy token (cross-token speculation)
  c->sh_lm = dmalloc<int8_t>(c, (size_t)V * d, "shadow lm head");
  c->sh_slm = dmalloc<float>(c, V, "shadow lm head scales");
  CUDA_OK(c, launch_quantize(c->d_lm, V, d, c->wt, (int8_t*)c->sh_lm, c->sh_slm, c->s_main));
  CUDA_OK(c, launch_quantize(c->d_router, (int64_t)L * E, d, c->wt, (int8_t*)c->sh_router, c->sh_srouter, c->s_main));
  if (c->H > 0) {  // attention projections: int8-row like the routers (reading Q29)
    const int64_t hq = (int64_t)c->H * c->hd;
    c->sh_wqkv = dmalloc<int8_t>(c, (size_t)L * c->qkv_rows * d, "shadow wqkv");
    c->sh_sqkv = dmalloc<float>(c, (size_t)L * c->qkv_rows, "shadow sqkv");
    c->sh_wo = dmalloc<int8_t>(c, (size_t)L * d * hq, "shadow wo");
    c->sh_so = dmalloc<float>(c, (size_t)L * d, "shadow so");
    CUDA_OK(c, launch_quantize(c->d_wqkv, (int64_t)L * c->qkv_rows, d, c->wt, (int8_t*)c->sh_wqkv, c->sh_sqkv, c->s_main));
    CUDA_OK(c, launch_quantize(c->d_wo, (int64_t)L * d, hq, c->wt, (int8_t*)c->sh_wo, c->sh_so, c->s_main));
    c->stats.shadow_bytes += (int64_t)L * (c->qkv_rows * d + d * hq) + (int64_t)L * (c->qkv_rows + d) * 4;
  }
  c->sh_blob.assign((size_t)L * E, nullptr);
  c->sh_sc.assign((size_t)L * E, nullptr);
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e) {
      const size_t i = (size_t)l * E + e;
      const char* src = staging;
      if (!c->res_blob.empty() && c->res_blob[i]) {
        src = c->res_blob[i];
      } else {
        CUDA_OK(c, launch_gen(staging, 0, wl(c, l), e, 0, 0, 0, d, F, c->cfg.weight_seed, c->wt, c->s_main));
      }
      if (nf4) {  // codes W13 [2F][d/2] then W2 [d][F/2]; absmax W13 [2F][d/64] then W2 [d][F/64]
        uint8_t* q = dmalloc<uint8_t>(c, (size_t)3 * F * d / 2, "shadow expert nf4");
        float* s = dmalloc<float>(c, (size_t)3 * F * d / 64, "shadow nf4 absmax");
        CUDA_OK(c, launch_quantize_nf4(src, 2LL * F, d, c->wt, q, s, c->s_main));
        CUDA_OK(c, launch_quantize_nf4(src + (size_t)2 * F * d * c->esz, d, F, c->wt, q + (size_t)F * d,
                                       s + (size_t)2 * F * d / 64, c->s_main));
        c->sh_blob[i] = q;
        c->sh_sc[i] = s;
        c->stats.shadow_bytes += (int64_t)3 * F * d / 2 + (int64_t)3 * F * d / 64 * 4;
        continue;
      }
      int8_t* q = dmalloc<int8_t>(c, (size_t)3 * F * d, "shadow expert");
      float* s = dmalloc<float>(c, (size_t)2 * F + d, "shadow scales");
      if (fp8) {  // E4M3 codes, int8's layout (rows of W13 then W2; row scales s13 then s2)
        CUDA_OK(c, launch_quantize_fp8(src, 2LL * F, d, c->wt, (uint8_t*)q, s, c->s_main));
        CUDA_OK(c, launch_quantize_fp8(src + (size_t)2 * F * d * c->esz, d, F, c->wt, (uint8_t*)q + (size_t)2 * F * d,
                                       s + 2 * F, c->s_main));
      } else if (mma) {  // biased codes row-major into scratch, then the fragment-packed layout
        int8_t* qs = reinterpret_cast<int8_t*>(staging + c->full_bytes);
        CUDA_OK(c, launch_quantize(src, 2LL * F, d, c->wt, qs, s, c->s_main, true));
        CUDA_OK(c, launch_quantize(src + (size_t)2 * F * d * c->esz, d, F, c->wt, qs + (size_t)2 * F * d, s + 2 * F,
                                   c->s_main, true));
        CUDA_OK(c, launch_pack_i8_frag((const uint8_t*)qs, (uint8_t*)q, 2 * F, d, 1, c->s_main));
        CUDA_OK(c, launch_pack_i8_frag((const uint8_t*)qs + (size_t)2 * F * d, (uint8_t*)q + (size_t)2 * F * d, d, F, 0,
                                       c->s_main));
      } else {
        CUDA_OK(c, launch_quantize(src, 2LL * F, d, c->wt, q, s, c->s_main, u8));
        CUDA_OK(c, launch_quantize(src + (size_t)2 * F * d * c->esz, d, F, c->wt, q + (size_t)2 * F * d, s + 2 * F,
                                   c->s_main, u8));
      }
      c->sh_blob[i] = q;
      c->sh_sc[i] = s;
      c->stats.shadow_bytes += (int64_t)3 * F * d + (int64_t)(2 * F + d) * 4;
    }
  c->stats.shadow_bytes += 2 * ((int64_t)V * d + V * 4) + (int64_t)L * E * d + L * E * 4;
  c->d_sh_tbl = dmalloc<void*>(c, (size_t)L * E, "shadow tbl");
  c->d_sh_stbl = dmalloc<float*>(c, (size_t)L * E, "shadow stbl");
  CUDA_OK(c, cudaMemcpyAsync(c->d_sh_tbl, c->sh_blob.data(), sizeof(void*) * L * E, cudaMemcpyHostToDevice, c->s_main));
  CUDA_OK(c, cudaMemcpyAsync(c->d_sh_stbl, c->sh_sc.data(), sizeof(float*) * L * E, cudaMemcpyHostToDevice, c->s_main));
  CUDA_OK(c, cudaStreamSynchronize(c->s_main));
}

// Which (layer, expert) blobs this rank may ever need.
bool rank_may_need(const Ctx* c, int l, int e) {
  return plan_pool_holds(c->E, c->k, c->world, c->sliced ? 0 : c->G, l, e, c->rank);
}

// Generate expert (l, e) into dst: the whole blob, or (sliced placement) this rank's slice: W13
// gate/up pairs [f0, f0 + Fs) (contiguous rows of the interleaved W13) and W2 columns [f0, f0 + Fs)
// (a pitched copy), laid out as a blob of an expert with F = Fs. `full` is whole-blob scratch.
void gen_blob(Ctx* c, int l, int e, char* dst, char* full) {
  const int d = c->d, F = c->F;
  if (c->emu > 1 && c->emu_sliced) {  // N slice blobs back to back, slice r as rank r would hold it
    CUDA_OK(c, launch_gen(full, 0, wl(c, l), e, 0, 0, 0, d, F, c->cfg.weight_seed, c->wt, c->s_main));
    const size_t es = c->esz;
    for (int r = 0; r < c->emu; ++r) {
      char* o = dst + (size_t)r * c->emu_slice_bytes;
      const size_t f0 = (size_t)r * c->Fs;
      CUDA_OK(c, cudaMemcpyAsync(o, full + 2 * f0 * d * es, (size_t)c->emu_w13s, cudaMemcpyDeviceToDevice, c->s_main));
      CUDA_OK(c, cudaMemcpy2DAsync(o + c->emu_w13s, (size_t)c->Fs * es, full + (size_t)2 * F * d * es + f0 * es,
                                   (size_t)F * es, (size_t)c->Fs * es, (size_t)d, cudaMemcpyDeviceToDevice, c->s_main));
    }
    return;
  }
  if (!c->sliced) {
    CUDA_OK(c, launch_gen(dst, 0, wl(c, l), e, 0, 0, 0, d, F, c->cfg.weight_seed, c->wt, c->s_main));
    return;
  }
  CUDA_OK(c, launch_gen(full, 0, wl(c, l), e, 0, 0, 0, d, F, c->cfg.weight_seed, c->wt, c->s_main));
  const size_t es = c->esz, f0 = (size_t)c->rank * c->Fs;
  CUDA_OK(c, cudaMemcpyAsync(dst, full + 2 * f0 * d * es, (size_t)c->w13_bytes, cudaMemcpyDeviceToDevice, c->s_main));
  CUDA_OK(c, cudaMemcpy2DAsync(dst + c->w13_bytes, (size_t)c->Fs * es, full + (size_t)2 * F * d * es + f0 * es,
                               (size_t)F * es, (size_t)c->Fs * es, (size_t)d, cudaMemcpyDeviceToDevice, c->s_main));
}

// NUMA node of this rank's GPU from sysfs (-1 when unknown / single node)
int gpu_numa_node(int dev) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, (int)sizeof(bus), dev) != cudaSuccess) return -1;
  for (char* p = bus; *p; ++p) *p = (char)std::tolower((unsigned char)*p);
  const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) return -1;
  int n = -1;
  if (std::fscanf(f, "%d", &n) != 1) n = -1;
  std::fclose(f);
  return n;
}

// While alive, this thread's page allocations prefer `node` (MPOL_PREFERRED), so the pinned expert
// pool lands next to its GPU's PCIe root on multi-socket hosts. Best effort: any error
// leaves the default policy; a no-op on single-node hosts.
struct NumaPreferred {
  bool set = false;
  explicit NumaPreferred(int node) {
    const char* e = getenv("ODMOE_NUMA");  // ODMOE_NUMA=0: leave page placement to the kernel
    if (node < 0 || node >= 64 || (e && e[0] == '0')) return;
    unsigned long mask = 1ul << node;
    set = syscall(SYS_set_mempolicy, 1 /* MPOL_PREFERRED */, &mask, 64ul) == 0;
  }
  ~NumaPreferred() {
    if (set) syscall(SYS_set_mempolicy, 0 /* MPOL_DEFAULT */, nullptr, 0ul);
  }
};

void build_pool(Ctx* c, char* staging) {
  const int L = c->L, E = c->E, d = c->d, F = c->F;
  const double t0 = now_s();
  c->pool_off.assign((size_t)L * E, -1);
  int64_t n = 0;
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e)
      if (l != wl(c, l)) c->pool_off[(size_t)l * E + e] = c->pool_off[(size_t)wl(c, l) * E + e];
      else if (rank_may_need(c, l, e)) c->pool_off[(size_t)l * E + e] = (n++) * c->blob_bytes;
  c->pool_bytes = n * c->blob_bytes;
  if (c->resident) {
    // fully-resident baseline: every blob this rank may need lives in HBM (same placement)
    c->res_blob.assign((size_t)L * E, nullptr);
    for (int l = 0; l < L; ++l)
      for (int e = 0; e < E; ++e)
        if (l != wl(c, l)) {
          c->res_blob[(size_t)l * E + e] = c->res_blob[(size_t)wl(c, l) * E + e];
        } else if (c->pool_off[(size_t)l * E + e] >= 0 || (c->rank == 0 && c->cfg.predictor == ODMOE_PRED_SHADOW_SAME)) {
          char* p = dmalloc<char>(c, c->blob_bytes, "resident expert");
          gen_blob(c, l, e, p, staging);
          c->res_blob[(size_t)l * E + e] = p;
          c->stats.resident_bytes += c->blob_bytes;
        }
    c->pool_bytes = 0;
  } else {
    if (c->rank == 0 && c->cfg.predictor == ODMOE_PRED_SHADOW_SAME) {
      // SHADOW_SAME keeps a device copy of every expert for the shadow (tiny configs)
      c->res_blob.assign((size_t)L * E, nullptr);
      for (int l = 0; l < L; ++l)
        for (int e = 0; e < E; ++e) {
          char* p = dmalloc<char>(c, c->blob_bytes, "shadow-same expert");
          CUDA_OK(c, launch_gen(p, 0, wl(c, l), e, 0, 0, 0, d, F, c->cfg.weight_seed, c->wt, c->s_main));
          c->res_blob[(size_t)l * E + e] = p;
        }
    }
    {
      NumaPreferred np(gpu_numa_node(c->cfg.device));  // pages are placed when cudaHostAlloc pins them
      c->pool = hmalloc<char>(c, (size_t)c->pool_bytes, "expert pool");
    }
    // Fill the pool: generate each blob on the GPU, copy D2H into its pinned slot.
    char* stg[2] = {staging + c->full_bytes, staging + c->full_bytes + c->blob_bytes};
    cudaEvent_t done[2];
    CUDA_OK(c, cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    CUDA_OK(c, cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    bool used[2] = {false, false};
    int i = 0;
    for (int l = 0; l < L; ++l)
      for (int e = 0; e < E; ++e) {
        const int64_t off = c->pool_off[(size_t)l * E + e];
        if (off < 0 || l != wl(c, l)) continue;
        const int b = i++ & 1;
        if (used[b]) CUDA_OK(c, cudaEventSynchronize(done[b]));
        gen_blob(c, l, e, stg[b], staging);
        CUDA_OK(c, cudaMemcpyAsync(c->pool + off, stg[b], c->blob_bytes, cudaMemcpyDeviceToHost, c->s_main));
        CUDA_OK(c, cudaEventRecord(done[b], c->s_main));
        used[b] = true;
      }
    CUDA_OK(c, cudaStreamSynchronize(c->s_main));
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
  }
  if (!c->res_blob.empty()) {
    c->d_res_tbl = dmalloc<void*>(c, (size_t)L * E, "resident tbl");
    CUDA_OK(c, cudaMemcpy(c->d_res_tbl, c->res_blob.data(), sizeof(void*) * L * E, cudaMemcpyHostToDevice));
  }
  c->stats.pool_bytes = c->pool_bytes;
  c->stats.pool_build_s = now_s() - t0;
}

// ODMOE_WARM_WAIT=0: the compute stream waits on the copy events and idles (A/B of the ramp)
bool warm_wait_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_WARM_WAIT");
    v = (e && e[0] == '0') ? 0 : (stream_write_available() ? 1 : 0);
  }
  return v == 1;
}

// The compute stream waits for part (0 = W13, 1 = whole blob) of the slot's current load: a spinning
// warp (warm wait) when the slot has flags, else the copy event.
void wait_load(Ctx* c, Slot& sl, int part, cudaStream_t s) {
  if (sl.flag) {
    CUDA_OK(c, launch_wait_flag(sl.flag + part, sl.epoch, c->d_flag, s));
    c->stats.kernel_launches++;
  } else {
    CUDA_OK(c, cudaStreamWaitEvent(s, part == 0 ? sl.ev_w13 : sl.ev_done, 0));
  }
}

void build_slots(Ctx* c) {
  if (c->resident) return;
  const int n = c->cfg.slots_per_gpu;
  c->slots.resize(n);
  for (auto& s : c->slots) {
    s.dev = dmalloc<char>(c, c->blob_bytes, "expert slot");
    CUDA_OK(c, cudaEventCreateWithFlags(&s.ev_w13, cudaEventDisableTiming));
    CUDA_OK(c, cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
    CUDA_OK(c, cudaEventCreateWithFlags(&s.ev_free, cudaEventDisableTiming));
    if (warm_wait_enabled()) {
      s.flag = dmalloc<uint32_t>(c, 2, "slot flag");
      CUDA_OK(c, cudaMemset(s.flag, 0, 2 * sizeof(uint32_t)));
    }
    s.req = std::make_shared<LoadReq>();
  }
  c->stats.resident_bytes = (int64_t)n * c->blob_bytes;
}

// Point the per-step prediction views (sh_ids, h_pred, sh_logits, dbg_sh_*, ev_pred) at buffer b.
void select_buf(Ctx* c, int b) {
  const size_t L = c->L, k = c->k, E = c->E, d = c->d;
  c->cur_buf = b;
  c->sh_ids = c->sh_ids_all ? c->sh_ids_all + b * L * k : nullptr;
  c->h_pred = c->h_pred_all + b * L * k;
  c->sh_logits = c->sh_logits_all ? c->sh_logits_all + b * L * E : nullptr;
  c->dbg_sh_h = c->dbg_sh_h_all ? c->dbg_sh_h_all + b * L * d : nullptr;
  c->dbg_sh_u = c->dbg_sh_u_all ? c->dbg_sh_u_all + b * L * d * 4 : nullptr;
  c->ev_pred = c->ev_pred_all.data() + b * L;
}

void build_buffers(Ctx* c) {
  const int L = c->L, E = c->E, k = c->k, d = c->d, F = c->F, V = c->V;
  c->pkt_ids_off = (int64_t)d * c->esz;
  c->pkt_w_off = c->pkt_ids_off + 4 * k;
  c->pkt_bytes = (c->pkt_w_off + 4 * k + 15) / 16 * 16;
  c->d_h = dmalloc<float>(c, d, "h");
  c->d_pkt = dmalloc<char>(c, (size_t)L * c->pkt_bytes, "packets");
  c->d_logits = dmalloc<float>(c, (size_t)L * E, "logits");
  c->d_a = dmalloc<float>(c, (size_t)k * F, "a");
  c->d_y = dmalloc<float>(c, (size_t)k * d, "y");
  c->d_yred = dmalloc<float>(c, d, "yred");
  c->d_zero = dmalloc<float>(c, d, "zero");
  c->d_ysum = dmalloc<float>(c, d, "ysum");
  CUDA_OK(c, cudaMemset(c->d_zero, 0, sizeof(float) * d));
  CUDA_OK(c, cudaMemset(c->d_y, 0, sizeof(float) * k * d));
  c->d_yptr = dmalloc<const float*>(c, k, "yptr");
  c->d_yredptr = dmalloc<const float*>(c, 1, "yredptr");
  std::vector<const float*> yp(k);
  for (int j = 0; j < k; ++j) yp[j] = c->d_y + (size_t)j * d;
  CUDA_OK(c, cudaMemcpy(c->d_yptr, yp.data(), sizeof(float*) * k, cudaMemcpyHostToDevice));
  const float* yr = c->d_yred;
  CUDA_OK(c, cudaMemcpy(c->d_yredptr, &yr, sizeof(float*), cudaMemcpyHostToDevice));
  c->d_tok_in = dmalloc<int32_t>(c, 1, "tok_in");
  c->d_tok_out = dmalloc<int32_t>(c, 1, "tok_out");
  c->d_flag = dmalloc<int32_t>(c, 1, "flag");
  CUDA_OK(c, cudaMemset(c->d_flag, 0, 4));
  c->d_lmscratch = dmalloc<char>(c, 16 * 4096, "lm scratch");
  CUDA_OK(c, cudaMemset(c->d_lmscratch, 0, 16 * 4096));
  c->d_lmlogits = dmalloc<float>(c, V, "lm logits");
  c->h_ids = hmalloc<int32_t>(c, (size_t)L * k, "h_ids");
  c->h_w = hmalloc<float>(c, (size_t)L * k, "h_w");
  c->h_pred_all = hmalloc<int32_t>(c, (size_t)Ctx::kPredBufs * L * k, "h_pred");
  c->h_tok = hmalloc<int32_t>(c, 2, "h_tok");
  c->h_flag = hmalloc<int32_t>(c, 1, "h_flag");
  CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_ids, cudaEventDisableTiming));
  CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_tok, cudaEventDisableTiming));
  CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_shadow_done, cudaEventDisableTiming));
  CUDA_OK(c, cudaEventCreateWithFlags(&c->ev_step, cudaEventDisableTiming));
  c->ev_pred_all.assign((size_t)Ctx::kPredBufs * L, nullptr);
  for (auto& e : c->ev_pred_all) CUDA_OK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c->nx_ready.assign(L, 0);
  c->nx_tbl.assign((size_t)L * k, -1);
  c->issued_nx.assign(L, {});
  c->pred_ready.assign(L, 0);
  c->pred_tbl.assign((size_t)L * k, -1);
  if (c->has_shadow) {
    c->sh_h = dmalloc<float>(c, d, "sh_h");
    c->sh_u = dmalloc<char>(c, (size_t)d * 4, "sh_u");
    c->sh_ids_all = dmalloc<int32_t>(c, (size_t)Ctx::kPredBufs * L * k, "sh_ids");
    c->sh_w = dmalloc<float>(c, (size_t)L * k, "sh_w");
    c->sh_logits_all = dmalloc<float>(c, (size_t)Ctx::kPredBufs * L * E, "sh_logits");
    c->sh_tok = dmalloc<int32_t>(c, Ctx::kPredBufs, "sh_tok");
    c->sh_lmscratch = dmalloc<char>(c, 16 * 4096, "shadow lm scratch");
    CUDA_OK(c, cudaMemset(c->sh_lmscratch, 0, 16 * 4096));
    CUDA_OK(c, cudaMemset(c->sh_tok, 0, sizeof(int32_t) * Ctx::kPredBufs));
    c->sh_a = dmalloc<float>(c, (size_t)k * F, "sh_a");
    c->sh_y = dmalloc<float>(c, (size_t)k * d, "sh_y");
    c->sh_yptr = dmalloc<const float*>(c, k, "sh_yptr");
    for (int j = 0; j < k; ++j) yp[j] = c->sh_y + (size_t)j * d;
    CUDA_OK(c, cudaMemcpy(c->sh_yptr, yp.data(), sizeof(float*) * k, cudaMemcpyHostToDevice));
  } else if (c->world > 1) {
    c->sh_ids_all = dmalloc<int32_t>(c, (size_t)Ctx::kPredBufs * L * k, "sh_ids");  // receive buffers for P
  }
  // SEP refinement buffers (allocated for any shadow ctx so the depth can be switched at run time)
  if (is_shadow(c->built_pred) || c->built_pred == ODMOE_PRED_GATE_REUSE) {
    c->ev_router.resize(L);
    c->ev_ref.resize(L);
    for (auto& e : c->ev_router) CUDA_OK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->ev_ref) CUDA_OK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ref_enq.assign(L, 0);
    c->rf_ids = dmalloc<int32_t>(c, (size_t)L * 4 * k, "rf_ids");
    c->h_ref = hmalloc<int32_t>(c, (size_t)L * 4 * k, "h_ref");
    if (c->rank == 0) {
      c->h_hist = dmalloc<float>(c, (size_t)L * d, "h_hist");
      c->rf_h = dmalloc<float>(c, d, "rf_h");
      c->rf_u = dmalloc<char>(c, (size_t)d * 4, "rf_u");
      c->rf_w = dmalloc<float>(c, (size_t)4 * k, "rf_w");
      c->rf_y = dmalloc<float>(c, (size_t)k * d, "rf_y");
      c->rf_a = dmalloc<float>(c, (size_t)k * F, "rf_a");
      c->rf_yptr = dmalloc<const float*>(c, k, "rf_yptr");
      for (int j = 0; j < k; ++j) yp[j] = c->rf_y + (size_t)j * d;
      CUDA_OK(c, cudaMemcpy(c->rf_yptr, yp.data(), sizeof(float*) * k, cudaMemcpyHostToDevice));
    }
  }
  if (c->H > 0 && c->rank == 0) {
    const size_t part = (size_t)c->H * attn_splits(c->max_seq - 1) * (c->hd + 2);
    c->d_qkv = dmalloc<float>(c, c->qkv_rows, "qkv");
    c->d_attn_o = dmalloc<float>(c, (size_t)c->H * c->hd, "attn o");
    c->d_attn_part = dmalloc<float>(c, part, "attn part");
    if (c->has_shadow) {
      c->sh_qkv = dmalloc<float>(c, c->qkv_rows, "sh qkv");
      c->sh_attn_o = dmalloc<float>(c, (size_t)c->H * c->hd, "sh attn o");
      c->sh_attn_part = dmalloc<float>(c, part, "sh attn part");
      c->sh_kcur = dmalloc<char>(c, (size_t)c->kvd * c->kv_esz, "sh kcur");
      c->sh_vcur = dmalloc<char>(c, (size_t)c->kvd * c->kv_esz, "sh vcur");
    }
    if (c->cfg.debug_capture) c->dbg_hpre = dmalloc<float>(c, (size_t)L * d, "dbg_hpre");
  }
  c->predA_tbl.assign((size_t)L * k, -1);
  c->predA_ready.assign(L, 0);
  c->issued_pre.assign(L, {});
  c->reloaded.assign(L, {});
  c->in_time.assign(L, 0);
  select_buf(c, 0);
  if (c->emu > 1) {
    const int N = c->emu;
    c->d_yemu = dmalloc<float>(c, (size_t)N * k * d, "emulated slice outputs");
    c->d_prank = dmalloc<float>(c, (size_t)N * d, "emulated rank partials");
    c->d_emu_ptr = dmalloc<const float*>(c, (size_t)L * (N + N * k), "emulation pointer arrays");
    c->h_emu_ptr = hmalloc<const float*>(c, (size_t)L * (N + N * k), "emulation pointer arrays (host)");
    if (c->cfg.debug_capture) c->dbg_yrank = dmalloc<float>(c, (size_t)L * N * d, "dbg_yrank");
  }
  c->predB_tbl.assign((size_t)L * k, -1);
  if (c->cfg.debug_capture && c->rank == 0) {
    c->dbg_h = dmalloc<float>(c, (size_t)L * d, "dbg_h");
    c->dbg_ypart = dmalloc<float>(c, (size_t)L * k * d, "dbg_ypart");
    c->dbg_yred = dmalloc<float>(c, (size_t)L * d, "dbg_yred");
    c->dbg_sh_h_all = dmalloc<float>(c, (size_t)Ctx::kPredBufs * L * d, "dbg_sh_h");
    c->dbg_sh_u_all = dmalloc<char>(c, (size_t)Ctx::kPredBufs * L * d * 4, "dbg_sh_u");
    c->dbg_sh_hf_all = dmalloc<float>(c, (size_t)Ctx::kPredBufs * d, "dbg_sh_hf");
    if (c->has_shadow) c->sh_lmlogits = dmalloc<float>(c, (size_t)Ctx::kPredBufs * V, "shadow lm logits");
    c->dbg_hfinal = dmalloc<float>(c, d, "dbg_hfinal");
    CUDA_OK(c, cudaMemset(c->dbg_ypart, 0, sizeof(float) * L * k * d));
    CUDA_OK(c, cudaMemset(c->dbg_yred, 0, sizeof(float) * L * d));
  }
}

// ODMOE_SHADOW_FUSED=1: both tensor-core shadow phases in one cooperative launch per layer. Off by
// default: measured 83.4 us per layer vs 49.0 + 31.5 us for the two launches (ncu, profiles/
// launches_r02_shadow_layer_fused.csv) -- the grid barrier costs more than the launch it saves.
bool shadow_fused_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_SHADOW_FUSED");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// The shadow's k experts of one layer (a8 on the quantised weights): W13+SwiGLU of all k in one
// launch, W2+gate of all k in a second one (launch_w13_multi / launch_w2_multi; bitwise the
// per-expert launches). a: [k][F] scratch, y: [k][d] gate-weighted outputs.
void shadow_experts(Ctx* c, const ExpertRef* ex, const void* u, int u_f32, float* a, const float* gate_w, float* y,
                    bool pdl_first, cudaStream_t s) {
  const int k = c->k, d = c->d, F = c->F;
  // the tensor-core INT8 shadow: both phases in one cooperative launch (ODMOE_SHADOW_FUSED=0: two)
  if (c->sh_ewt == W_I8P && ex[0].tbl != nullptr && shadow_fused_enabled() && multi_flat_ok(k, c->sh_ewt, d, F)) {
    KTimer t(c, K_SH_W13, s, k);
    CUDA_OK(c, launch_mma_shadow_layer(k, ex, u, a, gate_w, y, d, F, s, pdl_first));
    return;
  }
  // shapes the flat engine does not take run one launch per expert (count them all)
  if (!multi_flat_ok(k, c->sh_ewt, d, F)) c->stats.kernel_launches += 2 * (k - 1);
  { KTimer t(c, K_SH_W13, s, k); CUDA_OK(c, launch_w13_multi(k, ex, c->sh_ewt, u, u_f32, a, d, F, s, pdl_first)); }
  { KTimer t(c, K_SH_W2, s, k); CUDA_OK(c, launch_w2_multi(k, ex, c->sh_ewt, a, gate_w, y, d, F, s, true)); }
}

// ------------------------------------------------------------------ shadow forward (SEP, Mode A)
// Enqueue one shadow pass on s_shadow into prediction buffer b: embed the token at token_dev (the
// main model's token, Mode A / token alignment, or the shadow's own previous token at an unaligned
// iteration), then L x [router, k expert FFNs] with the shadow's own routing chosen on the device
// (Q10). Predictions land in sh_ids_all[b] [L][k]; at N = 1 each layer's ids are
// copied to h_pred_all[b] with event ev_pred_all[b][l]; at N > 1 rank 0 broadcasts them in chunks of
// pred_chunk layers as soon as each chunk's last router has run. want_token: also run the shadow's
// final norm + INT8-row LM head + argmax into sh_tok[b] (its own next token).
void enqueue_shadow(Ctx* c, const int32_t* token_dev, int b, bool want_token) {
  const int L = c->L, E = c->E, k = c->k, d = c->d;
  cudaStream_t s = c->s_shadow;
  const WType swt = c->sh_wt;
  const bool same = swt != W_I8;  // no row scales (main-dtype or BF16 shadow)
  const size_t sesz = swt == W_I8 ? 1 : (swt == W_BF16 ? 2 : 4);
  int32_t* ids = c->sh_ids_all + (size_t)b * L * k;
  float* logits = c->sh_logits_all + (size_t)b * L * E;
  int32_t* hp = c->h_pred_all + (size_t)b * L * k;
  cudaEvent_t* evp = c->ev_pred_all.data() + (size_t)b * L;
  float* dh = c->dbg_sh_h_all ? c->dbg_sh_h_all + (size_t)b * L * d : nullptr;
  char* du = c->dbg_sh_u_all ? c->dbg_sh_u_all + (size_t)b * L * d * 4 : nullptr;
  cudaEvent_t pa = nullptr, pz = nullptr;
  if (c->pass_timing) {
    for (cudaEvent_t* ev : {&pa, &pz}) {
      if (!c->tev_pool.empty()) { *ev = c->tev_pool.back(); c->tev_pool.pop_back(); }
      else CUDA_OK(c, cudaEventCreate(ev));
    }
    CUDA_OK(c, cudaEventRecord(pa, s));
  }
  {
    KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_embed(c->sh_emb, c->sh_semb, swt, token_dev, d, c->sh_h, s));
  }
  if (token_dev == c->d_tok_in) CUDA_OK(c, cudaEventRecord(c->ev_shadow_done, s));  // d_tok_in consumed
  for (int l = 0; l < L; ++l) {
    int n_add = l > 0 ? k : 0;
    if (c->H > 0) {  // the shadow's own attention block (past keys/values from the main cache)
      if (n_add > 0) CUDA_OK(c, launch_combine(c->sh_h, c->sh_yptr, n_add, d, s));
      n_add = 0;
      enqueue_attention(c, l, s, c->sh_h, true, true);
    }
    {
      KTimer t(c, K_SHADOW, s);
      CUDA_OK(c, launch_router(c->sh_h, c->sh_yptr, n_add, nullptr,
                               (const char*)c->sh_router + (size_t)l * E * d * sesz,
                               same ? nullptr : c->sh_srouter + (size_t)l * E, swt, 1, E, d, k,
                               c->cfg.rms_eps, c->sh_u, ids + (size_t)l * k,
                               c->sh_w + (size_t)l * k, logits + (size_t)l * E, nullptr, s, true));
    }
    if (dh) {
      CUDA_OK(c, cudaMemcpyAsync(dh + (size_t)l * d, c->sh_h, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
      CUDA_OK(c, cudaMemcpyAsync(du + (size_t)l * d * 4, c->sh_u, (size_t)d * (swt == W_F32 ? 4 : 2), cudaMemcpyDeviceToDevice, s));
    }
    if (c->world == 1) {
      CUDA_OK(c, cudaMemcpyAsync(hp + (size_t)l * k, ids + (size_t)l * k, 4 * k, cudaMemcpyDeviceToHost, s));
      CUDA_OK(c, cudaEventRecord(evp[l], s));
    } else if ((l + 1) % c->pred_chunk == 0 || l == L - 1) {
      // this chunk's predictions go out now, not after the whole pass (receivers post the same
      // broadcasts in the same comm_pred order: enqueue_pred_broadcast)
      const int l0 = l / c->pred_chunk * c->pred_chunk, n = l + 1 - l0;
      NCCL_OK(c, ncclBroadcast(ids + (size_t)l0 * k, ids + (size_t)l0 * k, (size_t)n * k, ncclInt32, 0, c->comm_pred, s));
      CUDA_OK(c, cudaMemcpyAsync(hp + (size_t)l0 * k, ids + (size_t)l0 * k, 4 * n * k, cudaMemcpyDeviceToHost, s));
      CUDA_OK(c, cudaEventRecord(evp[l0], s));
    }
    const int u_f32 = swt == W_F32;
    std::vector<ExpertRef> ex(k);
    for (int j = 0; j < k; ++j)
      ex[j] = ExpertRef{nullptr, nullptr, (const void* const*)c->d_sh_tbl, (const float* const*)c->d_sh_stbl,
                        ids + (size_t)l * k, j, l * E, k, 0};
    shadow_experts(c, ex.data(), c->sh_u, u_f32, c->sh_a, c->sh_w + (size_t)l * k, c->sh_y, true, s);
  }
  if (want_token) {  // h_L = h_{L-1} + y_{L-1}; own greedy token (lowest id on ties)
    CUDA_OK(c, launch_combine(c->sh_h, c->sh_yptr, k, d, s));
    if (c->dbg_sh_hf_all)
      CUDA_OK(c, cudaMemcpyAsync(c->dbg_sh_hf_all + (size_t)b * d, c->sh_h, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_lm_head(c->sh_h, c->sh_lm, swt, c->V, d, c->cfg.rms_eps, c->sh_tok + b,
                              c->sh_lmlogits ? c->sh_lmlogits + (size_t)b * c->V : nullptr, c->sh_lmscratch, s,
                              false, same ? nullptr : c->sh_slm));
  }
  if (pa) {
    CUDA_OK(c, cudaEventRecord(pz, s));
    c->timed.push_back(Ctx::Timed{K_SH_PASS, pa, pz, 1, false});
  }
}

// At N > 1 the non-zero ranks receive rank 0's prediction table of buffer b in chunks of pred_chunk
// layers over comm_pred on s_shadow, copy each chunk to h_pred_all[b] and record its event.
void enqueue_pred_broadcast(Ctx* c, int b) {
  const int L = c->L, k = c->k;
  cudaStream_t s = c->s_shadow;
  int32_t* ids = c->sh_ids_all + (size_t)b * L * k;
  int32_t* hp = c->h_pred_all + (size_t)b * L * k;
  cudaEvent_t* evp = c->ev_pred_all.data() + (size_t)b * L;
  for (int l0 = 0; l0 < L; l0 += c->pred_chunk) {
    const int n = std::min(c->pred_chunk, L - l0);
    NCCL_OK(c, ncclBroadcast(ids + (size_t)l0 * k, ids + (size_t)l0 * k, (size_t)n * k, ncclInt32, 0, c->comm_pred, s));
    CUDA_OK(c, cudaMemcpyAsync(hp + (size_t)l0 * k, ids + (size_t)l0 * k, 4 * n * k, cudaMemcpyDeviceToHost, s));
    CUDA_OK(c, cudaEventRecord(evp[l0], s));
  }
}

// The NEXT token's prediction for layer m (speculative pass, buffer (step + 1) & 1) on the host?
bool next_pred_available(Ctx* c, int m) {
  if (c->spec_step != c->step + 1) return false;
  if (c->nx_ready[m]) return true;
  const int b = (int)((c->step + 1) & 1), L = c->L, k = c->k;
  const int evl = c->world == 1 ? m : (m / c->pred_chunk) * c->pred_chunk;
  const cudaError_t q = cudaEventQuery(c->ev_pred_all[(size_t)b * L + evl]);
  if (q == cudaErrorNotReady) return false;
  CUDA_OK(c, q);
  const int hi = c->world == 1 ? m + 1 : std::min(L, evl + c->pred_chunk);
  const int32_t* hp = c->h_pred_all + (size_t)b * L * k;
  for (int l = evl; l < hi; ++l) {
    c->nx_ready[l] = 1;
    std::copy(hp + (size_t)l * k, hp + (size_t)(l + 1) * k, c->nx_tbl.begin() + (size_t)l * k);
  }
  return true;
}

// Prediction for layer m available on the host? (non-blocking). Mode A (token-start shadow)
// results are copied to predA_tbl as their events complete; the plan (pred_tbl) takes Mode A
// unless a refined prediction for that layer already arrived.
bool pred_available(Ctx* c, int m) {
  if (!c->pred_valid) return false;
  const int p = c->cfg.predictor;
  if (is_shadow(p) && !c->predA_ready[m]) {
    const int evl = c->world == 1 ? m : (m / c->pred_chunk) * c->pred_chunk;
    const cudaError_t q = cudaEventQuery(c->ev_pred[evl]);
    if (q == cudaErrorNotReady) return c->pred_ready[m] != 0;
    CUDA_OK(c, q);
    const int hi = c->world == 1 ? m + 1 : std::min(c->L, evl + c->pred_chunk);
    for (int l = evl; l < hi; ++l) {
      c->predA_ready[l] = 1;
      std::copy(c->h_pred + (size_t)l * c->k, c->h_pred + (size_t)(l + 1) * c->k, c->predA_tbl.begin() + (size_t)l * c->k);
      if (c->predB_tbl[(size_t)l * c->k] < 0) {  // a refined prediction, if any, supersedes Mode A
        std::copy(c->h_pred + (size_t)l * c->k, c->h_pred + (size_t)(l + 1) * c->k, c->pred_tbl.begin() + (size_t)l * c->k);
        c->pred_ready[l] = 1;
      }
    }
  }
  return c->pred_ready[m] != 0;
}

// RANDOM predictor (P:256 case 5): k distinct uniform experts from splitmix64(aux_seed, step, l).
uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void random_prediction(Ctx* c, int64_t step, int l, int32_t* out) {
  uint64_t x = sm64(sm64(c->cfg.aux_seed) ^ ((uint64_t)step << 20) ^ (uint64_t)l);
  int n = 0;
  while (n < c->k) {
    x = sm64(x);
    const int e = (int)(x % (uint64_t)c->E);
    bool dup = false;
    for (int i = 0; i < n; ++i) dup |= out[i] == e;
    if (!dup) out[n++] = e;
  }
}

// ------------------------------------------------------------------ SEP refinement ("Mode B")
// Rank 0, shadow stream, after the main router of layer j: re-anchor the INT8 shadow at the main
// model's exact state -- h_j, u_j and the TRUE experts of layer j -- and run it R layers ahead:
// y'_j = sum_i w_i Q-FFN_i(u_j); h' = h_j + y'_j; router_{j+1}(h') -> P_B[j+1]; (experts, router)...
// Its error covers at most R quantised layers instead of the whole token (Mode A), so it corrects
// most mispredictions one or two layers before the main router would discover them.
// Gate reuse (prior work): the MAIN model's gates of layers j+1..j+R applied to layer j's
// state h_j (no expert outputs, no shadow): HOBBIT-style multi-layer look-ahead.
void enqueue_gate_reuse(Ctx* c, int j) {
  const int L = c->L, E = c->E, k = c->k, d = c->d, R = c->R;
  cudaStream_t s = c->s_shadow;
  int32_t* out = c->rf_ids + (size_t)j * 4 * k;
  CUDA_OK(c, cudaStreamWaitEvent(s, c->ev_router[j], 0));
  CUDA_OK(c, cudaMemsetAsync(out, 0xff, sizeof(int32_t) * 4 * k, s));
  for (int r = 1; r <= R && j + r < L; ++r) {
    const int m = j + r;
    CUDA_OK(c, cudaMemcpyAsync(c->rf_h, c->h_hist + (size_t)j * d, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    KTimer t(c, K_SHADOW, s);
    CUDA_OK(c, launch_router(c->rf_h, nullptr, 0, nullptr, (const char*)c->d_router + (size_t)m * E * d * c->esz,
                             nullptr, c->wt, 1, E, d, k, c->cfg.rms_eps, c->rf_u, out + (size_t)(r - 1) * k,
                             c->rf_w + (size_t)(r - 1) * k, nullptr, nullptr, s, false));
  }
}

void enqueue_refine(Ctx* c, int j) {
  if (c->cfg.predictor == ODMOE_PRED_GATE_REUSE) return enqueue_gate_reuse(c, j);
  const int L = c->L, E = c->E, k = c->k, d = c->d, R = c->R;
  cudaStream_t s = c->s_shadow;
  const WType swt = c->sh_wt;
  const size_t sesz = swt == W_I8 ? 1 : (swt == W_BF16 ? 2 : 4);
  const bool same = swt != W_I8;
  char* pkt = c->d_pkt + (size_t)j * c->pkt_bytes;
  int32_t* out = c->rf_ids + (size_t)j * 4 * k;
  CUDA_OK(c, cudaStreamWaitEvent(s, c->ev_router[j], 0));
  CUDA_OK(c, cudaMemcpyAsync(c->rf_h, c->h_hist + (size_t)j * d, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
  CUDA_OK(c, cudaMemsetAsync(out, 0xff, sizeof(int32_t) * 4 * k, s));
  // layer j with the main's u_j and true ids
  std::vector<ExpertRef> ex(k);
  for (int i = 0; i < k; ++i)
    ex[i] = ExpertRef{nullptr, nullptr, (const void* const*)c->d_sh_tbl, (const float* const*)c->d_sh_stbl,
                      (const int32_t*)(pkt + c->pkt_ids_off), i, j * E, k, 0};
  shadow_experts(c, ex.data(), pkt, 0, c->rf_a, (const float*)(pkt + c->pkt_w_off), c->rf_y, false, s);
  for (int r = 1; r <= R && j + r < L; ++r) {
    const int m = j + r;
    int n_add = k;
    if (c->H > 0) {
      CUDA_OK(c, launch_combine(c->rf_h, c->rf_yptr, k, d, s));
      n_add = 0;
      enqueue_attention(c, m, s, c->rf_h, true);
    }
    {
      KTimer t(c, K_SHADOW, s);
      CUDA_OK(c, launch_router(c->rf_h, c->rf_yptr, n_add, nullptr, (const char*)c->sh_router + (size_t)m * E * d * sesz,
                               same ? nullptr : c->sh_srouter + (size_t)m * E, swt, 1, E, d, k, c->cfg.rms_eps,
                               c->rf_u, out + (size_t)(r - 1) * k, c->rf_w + (size_t)(r - 1) * k, nullptr, nullptr, s, true));
    }
    if (r < R && m + 1 < L) {
      for (int i = 0; i < k; ++i)
        ex[i] = ExpertRef{nullptr, nullptr, (const void* const*)c->d_sh_tbl, (const float* const*)c->d_sh_stbl,
                          out + (size_t)(r - 1) * k, i, m * E, k, 0};
      shadow_experts(c, ex.data(), c->rf_u, 0, c->rf_a, c->rf_w + (size_t)(r - 1) * k, c->rf_y, true, s);
    }
  }
}

// Broadcast (N > 1) and copy to the host the refined ids of refinement j; record ev_ref[j].
void enqueue_refine_delivery(Ctx* c, int j) {
  const int k = c->k;
  cudaStream_t s = c->s_shadow;
  int32_t* buf = c->rf_ids + (size_t)j * 4 * k;
  if (c->world > 1) NCCL_OK(c, ncclBroadcast(buf, buf, (size_t)4 * k, ncclInt32, 0, c->comm_pred, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_ref + (size_t)j * 4 * k, buf, sizeof(int32_t) * 4 * k, cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaEventRecord(c->ev_ref[j], s));
  c->ref_enq[j] = 1;
}

// ------------------------------------------------------------------ slots + loads
int find_slot(Ctx* c, int64_t tok, int l, int e) {
  for (int i = 0; i < (int)c->slots.size(); ++i) {
    const Slot& s = c->slots[i];
    if (s.occupied && s.token == tok && s.layer == l && s.expert == e) return i;
  }
  return -1;
}
int free_slot(Ctx* c) {
  for (int i = 0; i < (int)c->slots.size(); ++i)
    if (!c->slots[i].occupied) return i;
  return -1;
}
int occupied_count(const Ctx* c) {
  int n = 0;
  for (auto& s : c->slots) n += s.occupied;
  return n;
}

// kind: 0 predicted, 1 reload after the router, 2 refined prediction, 3 next-token
// (cross-token speculation), 4 user load (odmoe_load), 5 prefill
enum LoadKind { LK_PRED = 0, LK_RELOAD = 1, LK_REFINE = 2, LK_NEXT = 3, LK_USER = 4, LK_PREFILL = 5 };

void submit_into(Ctx* c, Slot& s, int slot, int64_t tok, int l, int e, int64_t key, int kind) {
  if (!holds_expert(c, l, e)) fail(c, ODMOE_E_RANGE, "expert not in this rank's pool");
  s.occupied = true;
  s.token = tok;
  s.layer = l;
  s.expert = e;
  auto r = std::make_shared<LoadReq>();
  r->layer = l;
  r->expert = e;
  r->slot = slot;
  r->key = key;
  r->src = c->pool + c->pool_off[(size_t)l * c->E + e];
  r->dst = s.dev;
  r->bytes = c->blob_bytes;
  r->w13_bytes = c->w13_bytes;
  r->ev_w13 = s.ev_w13;
  r->ev_done = s.ev_done;
  r->wait_ev = s.free_recorded ? s.ev_free : nullptr;
  if (s.flag) {
    r->flag = s.flag;
    r->epoch = ++s.epoch;
  }
  if (c->trace) {
    r->tr_start = tr_event(c);
    r->tr_end = tr_event(c);
    // the window position of the load: layer m of the next token is L + m (Q11)
    const int pos = (int)((tok > c->step ? (tok - c->step) * c->L : 0) + l);
    Ctx::TraceRec a, b, i;
    i.ev = tr_make(c, ODMOE_EV_LOAD_ISSUE, pos, e, slot, c->l_cur, kind, tok < 0 ? c->step : tok);
    a.ev = tr_make(c, ODMOE_EV_LOAD_START, l, e, slot, c->l_cur, kind, tok < 0 ? c->step : tok);
    a.e = r->tr_start;
    a.req = r;
    b.ev = tr_make(c, ODMOE_EV_LOAD_END, l, e, slot, c->l_cur, kind, tok < 0 ? c->step : tok);
    b.e = r->tr_end;
    b.req = r;
    c->tr_pending.push_back(std::move(i));
    c->tr_pending.push_back(std::move(a));
    c->tr_pending.push_back(std::move(b));
  }
  if (tok == c->step && l >= 0 && l < c->L && !c->issued_pre.empty()) {
    if (kind == LK_RELOAD) c->reloaded[l].push_back(e);
    else if (kind != LK_USER && kind != LK_PREFILL) c->issued_pre[l].push_back(e);
  } else if (tok == c->step + 1 && kind == LK_NEXT && l >= 0 && l < c->L) {
    c->issued_nx[l].push_back(e);
  }
  s.req = r;
  c->loader.submit(r);
}

void submit_load(Ctx* c, int slot, int64_t tok, int l, int e, int64_t key, int kind) {
  submit_into(c, c->slots[slot], slot, tok, l, e, key, kind);
  c->stats.max_resident = std::max<int64_t>(c->stats.max_resident, occupied_count(c));
}

void release_slot(Ctx* c, int slot) {
  Slot& s = c->slots[slot];
  if (s.req && c->loader.cancel(s.req)) tr_host(c, ODMOE_EV_LOAD_CANCEL, s.layer, s.expert, slot, 0, s.req);
  s.occupied = false;
  s.layer = s.expert = -1;
  s.token = -1;
}

int64_t load_key(const Ctx* c, int64_t tok, int l, int j) { return (tok * c->L + l) * 16 + j; }

// Consume finished refinements in order; for every layer whose refined prediction differs from the
// plan: take it as the plan and, if that layer's loads were already issued, stop the wrong ones and
// load the right experts now (before the main router of that layer runs).
void apply_refinements(Ctx* c) {
  const int k = c->k;
  while (c->ref_next < c->L - 1 && c->ref_enq[c->ref_next]) {
    const int j = c->ref_next;
    const cudaError_t q = cudaEventQuery(c->ev_ref[j]);
    if (q == cudaErrorNotReady) return;
    CUDA_OK(c, q);
    c->ref_next++;
    for (int r = 1; r <= c->R && j + r < c->L; ++r) {
      const int m = j + r;
      const int32_t* P = c->h_ref + ((size_t)j * 4 + (r - 1)) * k;
      if (P[0] < 0) continue;
      int32_t* B = c->predB_tbl.data() + (size_t)m * k;
      std::copy(P, P + k, B);
      if (m <= c->l_cur) continue;  // that layer's router already decided
      pred_available(c, m);          // compare against Mode A's prediction if it has arrived
      int32_t* plan = c->pred_tbl.data() + (size_t)m * k;
      bool same = c->pred_ready[m] != 0;
      for (int a = 0; a < k && same; ++a) {
        bool found = false;
        for (int b = 0; b < k; ++b) found |= P[a] == plan[b];
        same &= found;
      }
      if (same) continue;
      c->stats.refine_corrections++;
      std::copy(P, P + k, plan);
      c->pred_ready[m] = 1;
      if (m >= c->next_plan) continue;  // not planned yet: pump() will use the refined plan
      const std::vector<int> mine = my_experts(c, m, P);
      for (int i = 0; i < (int)c->slots.size(); ++i) {
        Slot& sl = c->slots[i];
        if (sl.occupied && sl.token == c->step && sl.layer == m &&
            std::find(mine.begin(), mine.end(), sl.expert) == mine.end())
          release_slot(c, i);
      }
      for (size_t jj = 0; jj < mine.size(); ++jj) {
        if (find_slot(c, c->step, m, mine[jj]) >= 0) continue;
        const int fs = free_slot(c);
        if (fs < 0) {  // no room now: re-plan this layer when a slot frees
          c->next_plan = std::min(c->next_plan, m);
          break;
        }
        submit_load(c, fs, c->step, m, mine[jj], load_key(c, c->step, m, 1 + (int)jj), LK_REFINE);
      }
    }
  }
}

// Issue predicted loads for layers next_plan .. l_cur + D while slots are free (Q11).
void pump(Ctx* c) {
  if (c->resident) return;
  if (c->R > 0) apply_refinements(c);
  while (c->next_plan < c->L) {
    const int m = c->next_plan;
    if (m > c->l_cur + c->cfg.lookahead) break;
    if (!pred_available(c, m)) break;
    std::vector<int> mine = my_experts(c, m, c->pred_tbl.data() + (size_t)m * c->k);
    std::vector<int> todo;
    for (int e : mine)
      if (find_slot(c, c->step, m, e) < 0) todo.push_back(e);
    int nfree = 0;
    for (auto& s : c->slots) nfree += !s.occupied;
    if (nfree < (int)todo.size()) break;
    for (size_t j = 0; j < todo.size(); ++j)
      submit_load(c, free_slot(c), c->step, m, todo[j], load_key(c, c->step, m, 1 + (int)j), LK_PRED);
    c->next_plan++;
  }
  // Cross-token speculation: once every layer of this token is planned, the next
  // token's layers m whose window position L + m <= l_cur + D are loaded from the speculative
  // shadow pass's predictions while the main model is still finishing this token.
  if (c->next_plan < c->L || c->spec_step != c->step + 1) return;
  const int64_t tn = c->step + 1;
  while (c->next_plan_nx < c->L) {
    const int m = c->next_plan_nx;
    if (c->L + m > c->l_cur + c->cfg.lookahead) break;
    if (!next_pred_available(c, m)) break;
    std::vector<int> mine = my_experts(c, m, c->nx_tbl.data() + (size_t)m * c->k);
    std::vector<int> todo;
    for (int e : mine)
      if (find_slot(c, tn, m, e) < 0) todo.push_back(e);
    int nfree = 0;
    for (auto& s : c->slots) nfree += !s.occupied;
    if (nfree < (int)todo.size()) break;
    for (size_t j = 0; j < todo.size(); ++j) {
      submit_load(c, free_slot(c), tn, m, todo[j], load_key(c, tn, m, 1 + (int)j), LK_NEXT);
      c->stats.early_loads++;
    }
    c->next_plan_nx++;
  }
}

// ------------------------------------------------------------------ P2P combine setup
// GPU 0 allocates the receive rows and flags, exports them with CUDA IPC and broadcasts the handles
// over NCCL; the other ranks map them (NVLink peer access). ODMOE_P2P=0 keeps the NCCL reduce.
void setup_p2p(Ctx* c) {
  const char* e = getenv("ODMOE_P2P");
  if ((e && e[0] == '0') || c->world > 32) return;
  struct Handles { cudaIpcMemHandle_t part; int ok; };
  Handles h{};
  if (c->rank == 0) {
    // receive rows: {value, epoch} pairs, 2 words per element (the LL format of p2p.cu)
    c->p2p_own_part = dmalloc<float>(c, (size_t)2 * c->world * c->d, "p2p part");
    CUDA_OK(c, cudaMemset(c->p2p_own_part, 0, sizeof(float) * 2 * c->world * c->d));
    h.ok = cudaIpcGetMemHandle(&h.part, c->p2p_own_part) == cudaSuccess;
  }
  char* dbuf = dmalloc<char>(c, sizeof(Handles), "p2p handles");
  CUDA_OK(c, cudaMemcpy(dbuf, &h, sizeof(h), cudaMemcpyHostToDevice));
  NCCL_OK(c, ncclBroadcast(dbuf, dbuf, sizeof(Handles), ncclChar, 0, c->comm, c->s_main));
  CUDA_OK(c, cudaStreamSynchronize(c->s_main));
  CUDA_OK(c, cudaMemcpy(&h, dbuf, sizeof(h), cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  int ok = h.ok;
  if (c->rank == 0) {
    c->p2p_part = c->p2p_own_part;
  } else if (ok) {
    void* pp = nullptr;
    ok = cudaIpcOpenMemHandle(&pp, h.part, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (!ok) cudaGetLastError();
    c->p2p_part = (float*)pp;
  }
  // every rank must agree (a rank that could not map falls back with everyone else)
  int32_t* dok = dmalloc<int32_t>(c, 1, "p2p ok");
  CUDA_OK(c, cudaMemcpy(dok, &ok, 4, cudaMemcpyHostToDevice));
  NCCL_OK(c, ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->comm, c->s_main));
  CUDA_OK(c, cudaStreamSynchronize(c->s_main));
  CUDA_OK(c, cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost));
  cudaFree(dok);
  c->p2p = ok != 0;
  c->p2p_seq = 1;
}

// Ranks whose expert work feeds layer l's combine (bit r = rank r).
uint32_t p2p_mask(const Ctx* c, int l) {
  if (c->sliced) return c->world >= 32 ? 0xffffffffu : ((1u << c->world) - 1u);
  const int g = l % c->NG;
  uint32_t m = 0;
  for (int p = 0; p < c->G; ++p) m |= 1u << (g * c->G + p);
  return m;
}

// ------------------------------------------------------------------ one decode step
// emulate_world: layer l's combine as an N-GPU run performs it (odmoe.h): each emulated rank sums its
// gated partials in router rank order (p2p_send's order), then the ranks' partials are summed in rank
// order into d_yred (p2p_gather's order); the next router adds d_yred (n_add = 1).
void emu_combine(Ctx* c, int l, const int32_t* S, cudaStream_t s) {
  const int N = c->emu, k = c->k, d = c->d;
  const float** hp = c->h_emu_ptr + (size_t)l * (N + N * k);
  const float** dp = c->d_emu_ptr + (size_t)l * (N + N * k);
  std::vector<int> nrank(N, 0);
  int r0 = 0, nr = N;
  if (c->emu_sliced) {
    for (int r = 0; r < N; ++r) {
      for (int j = 0; j < k; ++j) hp[N + r * k + j] = c->d_yemu + ((size_t)r * k + j) * d;
      nrank[r] = k;
    }
  } else {  // layer l's group; each rank's experts by the sorted pairing
    r0 = (l % c->emu_NG) * c->emu_G;
    nr = c->emu_G;
    for (int r = r0; r < r0 + nr; ++r) {
      int32_t mine[8];
      const int n = plan_layer(k, N, c->emu_G, l, S, r, mine);
      for (int j = 0; j < k; ++j)
        for (int i = 0; i < n; ++i)
          if (S[j] == mine[i]) hp[N + r * k + nrank[r]++] = c->d_y + (size_t)j * d;
    }
  }
  int np = 0;
  for (int r = r0; r < r0 + nr; ++r)
    if (nrank[r] > 0) hp[np++] = c->d_prank + (size_t)r * d;
  CUDA_OK(c, cudaMemcpyAsync(dp, hp, sizeof(float*) * (N + N * k), cudaMemcpyHostToDevice, s));
  for (int r = r0; r < r0 + nr; ++r) {
    if (nrank[r] == 0) continue;
    float* pr = c->d_prank + (size_t)r * d;
    CUDA_OK(c, cudaMemsetAsync(pr, 0, sizeof(float) * d, s));
    CUDA_OK(c, launch_combine(pr, dp + N + r * k, nrank[r], d, s));
    c->stats.kernel_launches++;
  }
  CUDA_OK(c, cudaMemsetAsync(c->d_yred, 0, sizeof(float) * d, s));
  CUDA_OK(c, launch_combine(c->d_yred, dp, np, d, s));
  c->stats.kernel_launches++;
  if (c->dbg_yrank) {
    CUDA_OK(c, cudaMemsetAsync(c->dbg_yrank + (size_t)l * N * d, 0, sizeof(float) * N * d, s));
    for (int r = r0; r < r0 + nr; ++r)
      if (nrank[r] > 0)
        CUDA_OK(c, cudaMemcpyAsync(c->dbg_yrank + ((size_t)l * N + r) * d, c->d_prank + (size_t)r * d, sizeof(float) * d,
                                   cudaMemcpyDeviceToDevice, s));
  }
  if (c->dbg_yred) CUDA_OK(c, cudaMemcpyAsync(c->dbg_yred + (size_t)l * d, c->d_yred, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
}

// The cooperative fused expert kernel at N > 1 (default since round 2; ODMOE_FUSED_NGPU=0 restores the
// split W13 / W2 launches). Safe because every kernel that can spin beside it is either stream-ordered
// with it (layer NCCL, P2P gather, warm wait) or the one-CTA prediction communicator, and the flat
// engine's grid leaves one SM free at N > 1.
bool fused_ngpu_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_FUSED_NGPU");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// The P2P send in the last expert's W2 epilogue instead of the one-CTA send kernel (ODMOE_P2P_FUSED=0:
// the send kernel). With a flag release it needed a system-scope fence per CTA (~30 us per launch,
// profiles/r02_m2c_*.json); since every value travels with its epoch in one 8-byte store (p2p.cu) no
// fence is needed, and the fused send is the default: resident N = 2 295.7 vs 280.4 tok/s,
// on-demand tok/s unchanged (profiles/r02_n2_p2p_ll_{fused_send,send_kernel}.json).
bool p2p_fused_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_P2P_FUSED");  // default on since the {value, epoch} format (no fences)
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// The P2P combine of this rank's layer partials, fused into its last expert's W2 (odmoe.h, kernels.h)
P2PSend p2p_send_args(Ctx* c, int nprev) {
  P2PSend ps{};
  ps.dst = c->p2p_part + (size_t)2 * c->rank * c->d;
  ps.epoch = c->p2p_seq;  // the epoch the layer-end send would use
  ps.prev = c->d_yptr;
  ps.nprev = nprev;
  return ps;
}

bool graph_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ODMOE_GRAPH");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

void decode_step_impl(Ctx* c, int32_t token_in, int32_t* token_out, odmoe_layer_record* rec) {
  const int L = c->L, E = c->E, k = c->k, d = c->d, F = c->F;
  if (token_in < 0 || token_in >= c->V) fail(c, ODMOE_E_RANGE, "token out of range");
  if (c->H > 0 && c->pos >= c->max_seq) fail(c, ODMOE_E_RANGE, "KV cache full (max_seq)");
  // a step is a function of its token (no attention) or of (token, position) over a replayed context
  const int64_t route_key = c->H > 0 ? ((int64_t)c->pos << 32) | (uint32_t)token_in : (int64_t)token_in;
  cudaStream_t s = c->s_main;
  const int p = c->cfg.predictor;
  const bool r0 = c->rank == 0;
  const int u_f32 = c->wt == W_F32;
  // Fused W13->W2 cooperative kernel: only on the compute stream and only where no kernel that
  // spins on ANOTHER GPU can occupy SMs concurrently (N = 1, or fully resident where the
  // prediction communicator is idle). At N > 1 the prediction broadcasts spin on the shadow
  // stream; a cooperative grid that cannot become fully resident would wait at its barrier for
  // SMs held by a kernel that waits for a peer that waits for us.
  // ODMOE_FUSED_NGPU=1 also allows it at N > 1: the prediction communicator is limited to one CTA
  // and the grid leaves one SM free, so the grid can always become resident beside it.
  const bool fused = use_fused_expert() && stream_ok(c->wt, d) && stream_ok(c->wt, c->Fs) && c->emu <= 1 &&
                     (c->world == 1 || c->resident || fused_ngpu_enabled());

  // Fully-resident 1-GPU steps (no attention, no debug capture) are the same sequence of launches
  // every token: the second step is captured into a CUDA graph (token H2D ... token D2H) and later
  // steps replay it -- one launch per token instead of ~200 (ODMOE_GRAPH=0 disables).
  const bool graphable = c->resident && c->world == 1 && c->H == 0 && !c->cfg.debug_capture && !c->trace && graph_enabled();
  c->predict_cache_token = -1;  // this step's shadow pass overwrites sh_ids (odmoe_predict_ahead's cache)
  for (int l = 0; l < L; ++l) {
    c->issued_pre[l].clear();
    c->reloaded[l].clear();
    c->in_time[l] = 0;
  }
  const bool replay = graphable && c->graph_exec != nullptr;
  const bool capture = graphable && !replay && c->step >= 1;
  const int64_t launches0 = c->stats.kernel_launches;
  const size_t timers0 = c->timed.size();
  if (capture) {
    unsigned int* counter = barrier_capture_reset(s);  // grid-barrier targets restart at 0 in every replay
    if (!counter) fail(c, ODMOE_E_CUDA, "barrier counter");
    CUDA_OK(c, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    CUDA_OK(c, cudaMemsetAsync(counter, 0, sizeof(unsigned int), s));
  }

  // token in (pinned -> device); the previous step's shadow must be done with d_tok_in
  c->h_tok[0] = token_in;
  if (!replay) {
    if (!c->resident) CUDA_OK(c, cudaStreamWaitEvent(s, c->ev_shadow_done, 0));
    CUDA_OK(c, cudaMemcpyAsync(c->d_tok_in, c->h_tok, 4, cudaMemcpyHostToDevice, s));
    if (!c->resident) CUDA_OK(c, cudaEventRecord(c->ev_tok, s));
  }
  c->l_cur = -1;
  tr_dev(c, ODMOE_EV_STEP_START, s, -1);

  // predictions for this step
  std::fill(c->pred_ready.begin(), c->pred_ready.end(), 0);
  std::fill(c->pred_tbl.begin(), c->pred_tbl.end(), -1);
  std::fill(c->predA_tbl.begin(), c->predA_tbl.end(), -1);
  std::fill(c->predA_ready.begin(), c->predA_ready.end(), 0);
  std::fill(c->predB_tbl.begin(), c->predB_tbl.end(), -1);
  const bool shadow_pred = is_shadow(p);
  const bool gate_reuse = p == ODMOE_PRED_GATE_REUSE;
  c->R = c->resident ? 0 : (shadow_pred ? c->cfg.refine_depth : (gate_reuse ? std::min(4, c->cfg.lookahead) : 0));
  c->ref_next = 0;
  std::fill(c->ref_enq.begin(), c->ref_enq.end(), 0);
  c->pred_valid = false;
  // Prediction buffer of this step; cross-token speculation state (token alignment period T_p):
  // this step's shadow pass may already have run during the previous step from the shadow's own
  // token (have_spec); the next step's pass is speculative iff iteration align_n + 1 is unaligned.
  const int pb = (int)(c->step & 1);
  select_buf(c, pb);
  const bool have_spec = shadow_pred && !c->resident && c->spec_step == c->step;
  const bool next_spec = shadow_pred && !c->resident && c->align_period > 1 &&
                         ((c->align_n + 1) % c->align_period) != 0;
  if (!have_spec) {  // early loads of an abandoned speculation (options changed in between) are dropped
    for (int i = 0; i < (int)c->slots.size(); ++i)
      if (c->slots[i].occupied && c->slots[i].token == c->step) release_slot(c, i);
  } else {
    for (int l = 0; l < L; ++l) c->issued_pre[l] = c->issued_nx[l];
  }
  for (int l = 0; l < L; ++l) c->issued_nx[l].clear();
  if (!c->resident) {
    if (shadow_pred) {
      if (r0) {
        if (!have_spec) {
          CUDA_OK(c, cudaStreamWaitEvent(c->s_shadow, c->ev_tok, 0));
          enqueue_shadow(c, c->d_tok_in, pb, c->align_period > 1);
        }
        if (next_spec) enqueue_shadow(c, c->sh_tok + pb, pb ^ 1, true);  // the shadow's own token
      } else if (c->world > 1) {
        if (!have_spec) enqueue_pred_broadcast(c, pb);
        if (next_spec) enqueue_pred_broadcast(c, pb ^ 1);
      }
      c->pred_valid = true;
      if (have_spec) c->stats.spec_steps++;
    } else if (gate_reuse) {
      c->pred_valid = true;  // predictions arrive per layer through the refinement path
    } else if (p == ODMOE_PRED_RANDOM) {
      for (int l = 0; l < L; ++l) random_prediction(c, c->step, l, c->pred_tbl.data() + (size_t)l * k);
      c->predA_tbl = c->pred_tbl;
      std::fill(c->pred_ready.begin(), c->pred_ready.end(), 1);
      c->pred_valid = true;
    } else if (p == ODMOE_PRED_PERFECT) {
      auto it = c->route_cache.find(route_key);
      if (it != c->route_cache.end()) {
        std::copy(it->second.begin(), it->second.end(), c->pred_tbl.begin());
        c->predA_tbl = c->pred_tbl;
        std::fill(c->pred_ready.begin(), c->pred_ready.end(), 1);
        c->pred_valid = true;
      }
    }
  }
  c->next_plan = have_spec ? c->next_plan_nx : 0;
  c->spec_step = next_spec ? c->step + 1 : -1;
  c->next_plan_nx = 0;
  std::fill(c->nx_ready.begin(), c->nx_ready.end(), 0);
  c->l_cur = 0;
  for (int m = 0; m < c->next_plan; ++m) pred_available(c, m);  // early-loaded layers: predictions on the host
  pump(c);

  std::vector<int32_t> true_ids((size_t)L * k);
  if (!replay) {
  // embedding (rank 0)
  if (r0) {
    KTimer t(c, K_EMBED, s);
    CUDA_OK(c, launch_embed(c->d_emb, nullptr, c->wt, c->d_tok_in, d, c->d_h, s));
  }

  const bool multi = c->world > 1 || c->emu > 1;  // the next router adds one reduced partial
  const float* const* yadd = multi ? c->d_yredptr : c->d_yptr;
  int n_add = 0;
  for (int l = 0; l < L; ++l) {
    c->l_cur = l;
    // Receivers enqueue refinement l's broadcast only now, after their layer l-1 reduce: a receive
    // that spins on the shadow stream must never sit (in a shared hardware queue) in front of the
    // layer traffic rank 0 needs before it can send it. Same comm_pred order as rank 0.
    if (c->world > 1 && !r0 && c->R > 0 && l < L - 1) enqueue_refine_delivery(c, l);
    char* pkt = c->d_pkt + (size_t)l * c->pkt_bytes;
    int32_t* ids_dev = (int32_t*)(pkt + c->pkt_ids_off);
    float* w_dev = (float*)(pkt + c->pkt_w_off);
    if (r0 && c->p2p && l > 0) {  // layer l-1's partials from the peers (NVLink) -> d_yred
      CUDA_OK(c, launch_p2p_gather(c->p2p_part, p2p_mask(c, l - 1), d, c->p2p_seq - 1, c->d_yred, c->d_flag, s));
      c->stats.kernel_launches++;
      if (c->dbg_yred) CUDA_OK(c, cudaMemcpyAsync(c->dbg_yred + (size_t)(l - 1) * d, c->d_yred, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    }
    if (r0 && c->H > 0) {
      // attention block of layer l (Q29): h += y_{l-1}; h += W_o attn(RMSNorm(h)); router sees that h
      if (n_add > 0) {
        CUDA_OK(c, launch_combine(c->d_h, yadd, n_add, d, s));
        c->stats.kernel_launches++;
        n_add = 0;
      }
      if (c->dbg_hpre) CUDA_OK(c, cudaMemcpyAsync(c->dbg_hpre + (size_t)l * d, c->d_h, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
      enqueue_attention(c, l, s, c->d_h, false);
    }
    if (r0) {
      KTimer t(c, K_ROUTER, s);
      CUDA_OK(c, launch_router(c->d_h, yadd, n_add, nullptr, (const char*)c->d_router + (size_t)l * E * d * c->esz,
                               nullptr, c->wt, 1, E, d, k, c->cfg.rms_eps, pkt, ids_dev, w_dev,
                               c->d_logits + (size_t)l * E, c->d_flag, s, true));
      if (c->dbg_h) CUDA_OK(c, cudaMemcpyAsync(c->dbg_h + (size_t)l * d, c->d_h, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
      if (c->R > 0 && l < L - 1) {
        CUDA_OK(c, cudaMemcpyAsync(c->h_hist + (size_t)l * d, c->d_h, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
        CUDA_OK(c, cudaEventRecord(c->ev_router[l], s));
        enqueue_refine(c, l);
        enqueue_refine_delivery(c, l);
      }
    }
    if (c->world > 1) NCCL_OK(c, ncclBroadcast(pkt, pkt, c->pkt_bytes, ncclChar, 0, c->comm, s));
    tr_dev(c, ODMOE_EV_ROUTER_DONE, s, l);
    n_add = multi ? 1 : k;

    const bool in_group = (l % c->NG) == c->my_group;
    // the P2P combine rides in the last expert's W2 epilogue (fused kernel, or a flat W2 launch)
    const bool flat_w2 = gemv_engine() == 2 && stream_ok(c->wt, c->Fs);
    const bool fuse_send = c->world > 1 && c->p2p && (fused || flat_w2) && p2p_fused_enabled();
    c->p2p_fused_sent = false;
    if (c->resident) {
      // routing consumed on the device: no host round trip per layer
      if (in_group) {
        const int mine = c->sliced ? k : k / c->G;
        const bool own = c->world == 1 || c->sliced;  // this rank computes (a slice of) every expert
        if (fused && mine <= 4) {
          // all of this GPU's experts of the layer in one cooperative launch
          ExpertRef exs[4];
          float* ys[4];
          for (int j = 0; j < mine; ++j) {
            exs[j] = ExpertRef{nullptr, nullptr, (const void* const*)c->d_res_tbl, nullptr, ids_dev,
                               own ? j : c->my_pos * mine + j, l * E, k, own ? 0 : 1};
            ys[j] = c->d_y + (size_t)j * d;
          }
          KTimer t(c, K_W13, s, mine);
          const P2PSend ps = fuse_send ? p2p_send_args(c, mine - 1) : P2PSend{};
          CUDA_OK(c, launch_experts_fused(mine, exs, nullptr, nullptr, c->wt, pkt, u_f32, c->d_a, w_dev, ys, d,
                                          c->Fs, s, true, fuse_send ? &ps : nullptr));
          c->p2p_fused_sent = fuse_send;
        }
        for (int j = 0; j < mine; ++j) {
          ExpertRef ex{nullptr, nullptr, (const void* const*)c->d_res_tbl, nullptr, ids_dev,
                       own ? j : c->my_pos * mine + j, l * E, k, own ? 0 : 1};
          float* y = c->d_y + (size_t)j * d;
          if (fused && mine <= 4) {
            // launched above
          } else if (fused) {
            KTimer t(c, K_W13, s);
            CUDA_OK(c, launch_expert_fused(ex, nullptr, nullptr, c->wt, pkt, u_f32, c->d_a + (size_t)j * F, w_dev, y, d, c->Fs, s, true));
          } else {
            { KTimer t(c, K_W13, s); CUDA_OK(c, launch_w13(ex, c->wt, pkt, u_f32, c->d_a + (size_t)j * F, d, c->Fs, s, true)); }
            { KTimer t(c, K_W2, s); CUDA_OK(c, launch_w2(ex, c->wt, c->d_a + (size_t)j * F, w_dev, y, d, c->Fs, s, true)); }
          }
          if (c->dbg_ypart) CUDA_OK(c, cudaMemcpyAsync(c->dbg_ypart + ((size_t)l * k + j) * d, y, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
        }
      }
    } else {
      // the host learns the router's ids (every rank: they arrive with the broadcast packet)
      CUDA_OK(c, cudaMemcpyAsync(c->h_ids + (size_t)l * k, ids_dev, 4 * k, cudaMemcpyDeviceToHost, s));
      CUDA_OK(c, cudaEventRecord(c->ev_ids, s));
      const double tw = now_s();
      for (;;) {
        const cudaError_t q = cudaEventQuery(c->ev_ids);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) CUDA_OK(c, q);
        pump(c);
        if (c->loader.error() != cudaSuccess) CUDA_OK(c, c->loader.error());
        std::this_thread::sleep_for(std::chrono::microseconds(5));
      }
      const double wait_us = (now_s() - tw) * 1e6;
      const int32_t* S = c->h_ids + (size_t)l * k;
      std::copy(S, S + k, true_ids.begin() + (size_t)l * k);
      // the prediction that could drive this layer's loads had reached the host before the ids did
      c->in_time[l] = c->pred_valid && (shadow_pred ? c->predA_ready[l] : c->pred_ready[l]);
      pred_available(c, l);  // refresh (shadow may have finished meanwhile)
      int reloads = 0;
      if (in_group) {
        std::vector<int> mine = my_experts(c, l, S);
        // Misprediction fallback: experts of this layer loaded for a wrong prediction
        // are stopped and their slots reused for the true experts (Q15).
        for (int i = 0; i < (int)c->slots.size(); ++i) {
          Slot& sl = c->slots[i];
          if (sl.occupied && sl.token == c->step && sl.layer == l &&
              std::find(mine.begin(), mine.end(), sl.expert) == mine.end())
            release_slot(c, i);
        }
        // a slot for a post-router load of layer l: a free one, else the furthest future prefetch
        // is dropped and re-planned later (never a slot held by odmoe_load, token -2; the next
        // token's early loads are furthest); -1 if every slot holds layer l's own experts
        auto take_slot = [&]() {
          int fs = free_slot(c);
          if (fs >= 0) return fs;
          int far = -1;
          auto wpos = [&](const Slot& q) { return (q.token - c->step) * (int64_t)L + q.layer; };
          for (int i = 0; i < (int)c->slots.size(); ++i)
            if (c->slots[i].occupied && c->slots[i].token >= c->step && (far < 0 || wpos(c->slots[i]) > wpos(c->slots[far]))) far = i;
          if (far < 0 || wpos(c->slots[far]) <= l) return -1;
          if (c->slots[far].token == c->step) c->next_plan = std::min(c->next_plan, c->slots[far].layer);
          else c->next_plan_nx = std::min(c->next_plan_nx, c->slots[far].layer);
          release_slot(c, far);
          return far;
        };
        for (int e : mine) {
          if (find_slot(c, c->step, l, e) >= 0) continue;
          const int fs = take_slot();
          if (fs < 0) {
            // fewer slots than experts of the layer (e.g. FP32 Mixtral, 1 slot under the 1 GB
            // budget): loaded in the compute loop below once an expert's slot frees
            if ((int)c->slots.size() >= (int)mine.size()) fail(c, ODMOE_E_BUDGET, "no slot for a reload");
            continue;
          }
          tr_host(c, ODMOE_EV_MISPREDICT, l, e, fs, 0);
          submit_load(c, fs, c->step, l, e, load_key(c, c->step, l, 0), LK_RELOAD);
          reloads++;
          c->stats.reloads++;
        }
        // compute, in rank order of the router's output; with a slot shortage the experts
        // already in slots go first and the deferred ones follow as slots free (each expert writes
        // its own output row ypos, so the combine order is unchanged)
        int ord[8], rpos[8], nord = 0;
        bool deferred = false;
        for (int pass = 0; pass < 2; ++pass)
          for (int j = 0, p = 0; j < k; ++j) {
            if (std::find(mine.begin(), mine.end(), S[j]) == mine.end()) continue;
            const bool has = find_slot(c, c->step, l, S[j]) >= 0;
            if (pass == 0) { rpos[j] = p; deferred |= !has; }
            if (has == (pass == 0)) ord[nord++] = j;
            p++;
          }
        const bool fuse_send_l = fuse_send && !deferred;
        int jj = 0;
        for (int oi = 0; oi < nord; ++oi) {
          const int j = ord[oi];
          int si = find_slot(c, c->step, l, S[j]);
          if (si < 0) {  // deferred (slot shortage): the slot the previous expert just freed; the copy
                         // waits for that expert's compute (the slot's free event)
            si = take_slot();
            if (si < 0) fail(c, ODMOE_E_BUDGET, "no slot for a deferred load");
            submit_load(c, si, c->step, l, S[j], load_key(c, c->step, l, 0), LK_RELOAD);
            reloads++;
            c->stats.reloads++;
          }
          Slot& sl = c->slots[si];
          if (!c->loader.wait_issued(sl.req)) {
            if (c->loader.error() != cudaSuccess) CUDA_OK(c, c->loader.error());
            fail(c, ODMOE_E_STATE, "load was cancelled before compute");
          }
          const int ypos = (c->world == 1 || c->sliced) ? j : rpos[j];
          float* y = c->d_y + (size_t)ypos * d;
          ExpertRef e13 = direct_ref(sl.dev, nullptr, j);
          ExpertRef e2 = direct_ref(sl.dev + c->w13_bytes, nullptr, j);
          if (c->emu > 1) {  // the N-GPU run's launches on this GPU (split W13 / W2, reserve-1 grid)
            wait_load(c, sl, 1, s);
            tr_dev(c, ODMOE_EV_COMPUTE_START, s, l, S[j], si);
            const int nsl = c->emu_sliced ? c->emu : 1;
            for (int r = 0; r < nsl; ++r) {
              const char* base = sl.dev + (size_t)r * c->emu_slice_bytes;
              const char* b2 = c->emu_sliced ? base + c->emu_w13s : sl.dev + c->w13_bytes;
              float* yo = c->emu_sliced ? c->d_yemu + ((size_t)r * k + j) * d : y;
              { KTimer t(c, K_W13, s); CUDA_OK(c, launch_w13(direct_ref(base, nullptr, j), c->wt, pkt, u_f32, c->d_a + (size_t)ypos * F, d, c->Fs, s)); }
              { KTimer t(c, K_W2, s); CUDA_OK(c, launch_w2(direct_ref(b2, nullptr, j), c->wt, c->d_a + (size_t)ypos * F, w_dev, yo, d, c->Fs, s)); }
            }
          } else if (fused) {  // one launch once the whole blob has landed
            wait_load(c, sl, 1, s);
            tr_dev(c, ODMOE_EV_COMPUTE_START, s, l, S[j], si);
            KTimer t(c, K_W13, s);
            const int nmine = (int)mine.size();
            const bool last = jj == nmine - 1;
            const P2PSend ps = (fuse_send_l && last) ? p2p_send_args(c, nmine - 1) : P2PSend{};
            CUDA_OK(c, launch_expert_fused(e13, sl.dev + c->w13_bytes, nullptr, c->wt, pkt, u_f32, c->d_a + (size_t)ypos * F,
                                           w_dev, y, d, c->Fs, s, false, (fuse_send_l && last) ? &ps : nullptr));
            if (fuse_send_l && last) c->p2p_fused_sent = true;
          } else {  // W13 starts as soon as its part has landed, W2 after the rest
            wait_load(c, sl, 0, s);
            tr_dev(c, ODMOE_EV_COMPUTE_START, s, l, S[j], si);
            { KTimer t(c, K_W13, s); CUDA_OK(c, launch_w13(e13, c->wt, pkt, u_f32, c->d_a + (size_t)ypos * F, d, c->Fs, s)); }
            wait_load(c, sl, 1, s);
            const int nmine = (int)mine.size();
            const bool last = jj == nmine - 1;
            if (fuse_send_l && last) {  // flat W2 launch with the layer's P2P send in its epilogue
              const P2PSend ps = p2p_send_args(c, nmine - 1);
              KTimer t(c, K_W2, s);
              CUDA_OK(c, launch_w2_flat(e2, c->wt, c->d_a + (size_t)ypos * F, w_dev, y, d, c->Fs, s, false, &ps));
              c->p2p_fused_sent = true;
            } else {
              KTimer t(c, K_W2, s);
              CUDA_OK(c, launch_w2(e2, c->wt, c->d_a + (size_t)ypos * F, w_dev, y, d, c->Fs, s));
            }
          }
          tr_dev(c, ODMOE_EV_COMPUTE_END, s, l, S[j], si);
          // evict right after use: the slot is reusable once this event fires (Q16)
          CUDA_OK(c, cudaEventRecord(sl.ev_free, s));
          sl.free_recorded = true;
          sl.req.reset();
          sl.occupied = false;
          sl.layer = sl.expert = -1;
          sl.token = -1;
          if (c->dbg_ypart) CUDA_OK(c, cudaMemcpyAsync(c->dbg_ypart + ((size_t)l * k + j) * d, y, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
          jj++;
        }
      }
      if (c->emu > 1) emu_combine(c, l, S, s);
      if (c->next_plan <= l) c->next_plan = l + 1;
      pump(c);
      if (rec) {
        odmoe_layer_record& R = rec[l];
        std::memset(&R, 0, sizeof(R));
        for (int j = 0; j < 8; ++j) { R.true_ids[j] = -1; R.pred_ids[j] = -1; R.issued_ids[j] = -1; R.reload_ids[j] = -1; }
        for (int j = 0; j < k; ++j) R.true_ids[j] = S[j];
        R.n_reloads = reloads;
        R.load_wait_us = (float)wait_us;
      }
      c->stats.wait_us += wait_us;
    }
    if (c->world > 1 && c->p2p) {
      // this rank's gated partials, summed in router rank order, stored into its row of GPU 0's
      // buffer over NVLink and published with a release flag (one kernel; no NCCL reduce)
      const uint32_t ep = c->p2p_seq++;
      if (in_group && !c->p2p_fused_sent) {
        CUDA_OK(c, launch_p2p_send(c->d_yptr, c->sliced ? k : k / c->G, d, c->p2p_part + (size_t)2 * c->rank * d,
                                   ep, s));
        c->stats.kernel_launches++;
      }
    } else if (c->world > 1) {
      const float* send = (in_group ? c->d_y : c->d_zero);
      const int nmine = c->sliced ? k : k / c->G;
      if (in_group && nmine > 1) {  // this rank's gated partials, summed in router rank order
        CUDA_OK(c, cudaMemsetAsync(c->d_ysum, 0, sizeof(float) * d, s));
        CUDA_OK(c, launch_combine(c->d_ysum, c->d_yptr, nmine, d, s));
        c->stats.kernel_launches++;
        send = c->d_ysum;
      }
      NCCL_OK(c, ncclReduce(send, c->d_yred, d, ncclFloat32, ncclSum, 0, c->comm, s));
      if (c->dbg_yred && r0) CUDA_OK(c, cudaMemcpyAsync(c->dbg_yred + (size_t)l * d, c->d_yred, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    }
  }

  // final combine + LM head + argmax (rank 0)
  if (r0) {
    if (c->p2p) {
      CUDA_OK(c, launch_p2p_gather(c->p2p_part, p2p_mask(c, L - 1), d, c->p2p_seq - 1, c->d_yred, c->d_flag, s));
      c->stats.kernel_launches++;
      if (c->dbg_yred) CUDA_OK(c, cudaMemcpyAsync(c->dbg_yred + (size_t)(L - 1) * d, c->d_yred, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    }
    CUDA_OK(c, launch_combine(c->d_h, yadd, n_add, d, s));
    c->stats.kernel_launches++;
    if (c->dbg_hfinal) CUDA_OK(c, cudaMemcpyAsync(c->dbg_hfinal, c->d_h, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    KTimer t(c, K_LM, s);
    CUDA_OK(c, launch_lm_head(c->d_h, c->d_lm, c->wt, c->V, d, c->cfg.rms_eps, c->d_tok_out,
                              c->cfg.debug_capture ? c->d_lmlogits : nullptr, c->d_lmscratch, s));
  }
  if (c->world > 1) NCCL_OK(c, ncclBroadcast(c->d_tok_out, c->d_tok_out, 1, ncclInt32, 0, c->comm, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_tok + 1, c->d_tok_out, 4, cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_flag, c->d_flag, 4, cudaMemcpyDeviceToHost, s));
  c->l_cur = L;  // the window now reaches into the next token (positions <= L + D)
  tr_dev(c, ODMOE_EV_STEP_END, s, -1);
  if (c->resident) CUDA_OK(c, cudaMemcpyAsync(c->h_ids, c->d_pkt + c->pkt_ids_off, 4 * k, cudaMemcpyDeviceToHost, s));
  if (c->resident && r0) {
    for (int l = 0; l < L; ++l)
      CUDA_OK(c, cudaMemcpyAsync(c->h_ids + (size_t)l * k, c->d_pkt + (size_t)l * c->pkt_bytes + c->pkt_ids_off, 4 * k, cudaMemcpyDeviceToHost, s));
  }
  }  // !replay
  if (capture) {
    cudaGraph_t graph = nullptr;
    CUDA_OK(c, cudaStreamEndCapture(s, &graph));
    const cudaError_t ie = cudaGraphInstantiate(&c->graph_exec, graph, 0);
    cudaGraphDestroy(graph);
    CUDA_OK(c, ie);
    c->graph_launches = c->stats.kernel_launches - launches0;
    c->graph_timers.assign(c->timed.begin() + timers0, c->timed.end());  // events owned by the graph
    for (auto& t : c->graph_timers) t.graph = true;
    c->timed.resize(timers0);
  }
  if (capture || replay) {
    CUDA_OK(c, cudaGraphLaunch(c->graph_exec, s));
    if (replay) c->stats.kernel_launches += c->graph_launches;
    c->timed.insert(c->timed.end(), c->graph_timers.begin(), c->graph_timers.end());
  }
  if (c->spec_step == c->step + 1 && !replay) {
    // keep issuing the next token's early loads while the LM head and the token copy finish
    for (;;) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) CUDA_OK(c, q);
      pump(c);
      if (c->loader.error() != cudaSuccess) CUDA_OK(c, c->loader.error());
      std::this_thread::sleep_for(std::chrono::microseconds(5));
    }
  }
  CUDA_OK(c, cudaStreamSynchronize(s));
  if (!c->resident && (shadow_pred || gate_reuse) && (r0 || c->world > 1)) CUDA_OK(c, cudaStreamSynchronize(c->s_shadow));
  if (c->spec_step == c->step + 1) pump(c);  // the speculative pass has finished: plan what fits now
  if (c->h_flag[0] == 2) fail(c, ODMOE_E_STATE, "peer partials did not arrive (P2P combine timeout)");
  if (c->h_flag[0] == 3) fail(c, ODMOE_E_STATE, "an expert load did not land (warm-wait timeout)");
  if (c->h_flag[0]) fail(c, ODMOE_E_NONFINITE, "non-finite router logits");
  if (c->resident) std::copy(c->h_ids, c->h_ids + (size_t)L * k, true_ids.begin());

  // predictions as they stood (recall accounting, Eqs. 2-3): the paper's SEP (Mode A) predictions
  // drive recall_eq3; the refined ones are counted separately
  for (int l = 0; l < L; ++l) pred_available(c, l);
  if (c->R > 0) apply_refinements(c);
  if (gate_reuse) c->predA_tbl = c->predB_tbl;  // the gate-reuse predictions are this predictor's output
  {
    for (int l = 0; l < L; ++l) {
      const int32_t* S = true_ids.data() + (size_t)l * k;
      const int32_t* P = c->predA_tbl.data() + (size_t)l * k;
      const bool have = c->pred_valid && P[0] >= 0;
      int corr = 0;
      if (have)
        for (int a = 0; a < k; ++a)
          for (int b = 0; b < k; ++b) corr += S[a] == P[b];
      const int corr_t = c->in_time[l] ? corr : 0;
      if (have && r0) { c->stats.correct += corr; c->stats.predicted_total += k; c->stats.correct_in_time += corr_t; }
      const int32_t* PB = c->predB_tbl.data() + (size_t)l * k;
      if (PB[0] >= 0 && r0) {
        int cb = 0;
        for (int a = 0; a < k; ++a)
          for (int b = 0; b < k; ++b) cb += S[a] == PB[b];
        c->stats.refine_correct += cb;
        c->stats.refine_total += k;
      }
      if (rec) {
        odmoe_layer_record& R = rec[l];
        if (c->resident) {
          std::memset(&R, 0, sizeof(R));
          for (int j = 0; j < 8; ++j) { R.true_ids[j] = -1; R.pred_ids[j] = -1; R.issued_ids[j] = -1; R.reload_ids[j] = -1; }
          for (int j = 0; j < k; ++j) R.true_ids[j] = S[j];
        }
        for (int j = 0; j < k; ++j) R.pred_ids[j] = have ? P[j] : -1;
        R.pred_available = have;
        R.correct = corr;
        R.pred_in_time = c->in_time[l];
        R.correct_in_time = corr_t;
        std::vector<int> a = c->issued_pre[l], b = c->reloaded[l];
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        for (int j = 0; j < (int)a.size() && j < 8; ++j) R.issued_ids[j] = a[j];
        for (int j = 0; j < (int)b.size() && j < 8; ++j) R.reload_ids[j] = b[j];
      }
    }
    if (rec) {
      std::vector<float> wv((size_t)L * k);
      for (int l = 0; l < L; ++l)
        CUDA_OK(c, cudaMemcpy(wv.data() + (size_t)l * k, c->d_pkt + (size_t)l * c->pkt_bytes + c->pkt_w_off, 4 * k, cudaMemcpyDeviceToHost));
      for (int l = 0; l < L; ++l)
        for (int j = 0; j < k; ++j) rec[l].weights[j] = wv[(size_t)l * k + j];
    }
  }
  c->route_cache[route_key] = true_ids;
  *token_out = c->h_tok[1];
  c->stats.tokens++;
  c->step++;
  c->align_n++;
  if (c->H > 0) c->pos++;
  if (c->cfg.time_kernels || c->pass_timing) harvest_timers(c);
  if (c->trace) tr_resolve(c);
  // loader statistics
  c->stats.loads_issued = c->loader.loads_issued.load();
  c->stats.loads_completed = c->loader.loads_completed.load();
  c->stats.loads_cancelled = c->loader.loads_cancelled.load();
  c->stats.bytes_h2d = c->loader.bytes_h2d.load();

  if (c->cfg.debug_capture && r0) {
    // host copy of the capture
    auto& H = c->hdbg;
    auto& I = c->hdbg_index;
    H.clear();
    I.clear();
    auto add = [&](int what, const void* dev, int64_t per_layer, int layers) {
      const int64_t off = (int64_t)H.size();
      H.resize(H.size() + (size_t)per_layer * layers);
      if (dev) CUDA_OK(c, cudaMemcpy(H.data() + off, dev, (size_t)per_layer * layers, cudaMemcpyDeviceToHost));
      I[what] = {off, per_layer};
    };
    std::vector<char> ubuf((size_t)L * d * c->esz), idb((size_t)L * k * 4), wb((size_t)L * k * 4);
    for (int l = 0; l < L; ++l) {
      const char* pk = c->d_pkt + (size_t)l * c->pkt_bytes;
      CUDA_OK(c, cudaMemcpy(ubuf.data() + (size_t)l * d * c->esz, pk, (size_t)d * c->esz, cudaMemcpyDeviceToHost));
      CUDA_OK(c, cudaMemcpy(idb.data() + (size_t)l * k * 4, pk + c->pkt_ids_off, 4 * k, cudaMemcpyDeviceToHost));
      CUDA_OK(c, cudaMemcpy(wb.data() + (size_t)l * k * 4, pk + c->pkt_w_off, 4 * k, cudaMemcpyDeviceToHost));
    }
    add(0, c->dbg_h, (int64_t)d * 4, L);
    {
      const int64_t off = (int64_t)H.size();
      H.insert(H.end(), ubuf.begin(), ubuf.end());
      I[1] = {off, (int64_t)d * (int64_t)c->esz};
    }
    add(2, c->d_logits, (int64_t)E * 4, L);
    {
      int64_t off = (int64_t)H.size();
      H.insert(H.end(), idb.begin(), idb.end());
      I[3] = {off, (int64_t)k * 4};
      off = (int64_t)H.size();
      H.insert(H.end(), wb.begin(), wb.end());
      I[4] = {off, (int64_t)k * 4};
    }
    add(5, c->dbg_yred, (int64_t)d * 4, L);
    add(6, c->dbg_ypart, (int64_t)k * d * 4, L);
    if (c->has_shadow && c->dbg_sh_h) {
      add(7, c->dbg_sh_h, (int64_t)d * 4, L);
      add(8, c->dbg_sh_u, (int64_t)d * 4, L);
      add(9, c->sh_logits, (int64_t)E * 4, L);
      add(10, c->sh_ids, (int64_t)k * 4, L);
      if (c->align_period > 1) {  // the pass that produced this step's predictions: its final state + own token
        add(14, c->dbg_sh_hf_all + (size_t)pb * d, (int64_t)d * 4, 1);
        add(15, c->sh_tok + pb, 4, 1);
        add(16, c->sh_lmlogits + (size_t)pb * c->V, (int64_t)c->V * 4, 1);
      }
    }
    add(11, c->dbg_hfinal, (int64_t)d * 4, 1);
    if (c->dbg_yrank) add(17, c->dbg_yrank, (int64_t)c->emu * d * 4, L);
    add(12, c->d_lmlogits, (int64_t)c->V * 4, 1);
    if (c->dbg_hpre) add(13, c->dbg_hpre, (int64_t)d * 4, L);
  }
}

// ------------------------------------------------------------------ prefill
// Layer l's E experts are split over the G GPUs of group l mod N_G in sorted order (expert e ->
// position e*G/E): with N = E = G this is the paper's "each worker handles one expert of every
// layer"; with fewer GPUs it keeps the decode pool placement and round-robins the loads over the
// groups, so group g loads layer l + 1 while another group computes layer l.
bool prefill_mine(const Ctx* c, int l, int e) {
  if (c->sliced) return true;  // every rank: its slice of every expert
  return (l % c->NG) == c->my_group && e * c->G / c->E == c->my_pos;
}

constexpr int kPrefillQChunk = 256;  // prefill attention queries per launch

void ensure_prefill(Ctx* c, int T) {
  const int E = c->E, k = c->k, d = c->d, F = c->F;
  if (c->pslots.empty() && !c->resident) {
    c->pslots.resize((size_t)2 * (c->sliced ? E : std::max(1, E / c->G)));
    for (auto& s : c->pslots) {
      s.dev = dmalloc<char>(c, c->blob_bytes, "prefill slot");
      CUDA_OK(c, cudaEventCreateWithFlags(&s.ev_w13, cudaEventDisableTiming));
      CUDA_OK(c, cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
      CUDA_OK(c, cudaEventCreateWithFlags(&s.ev_free, cudaEventDisableTiming));
    }
  }
  if (!c->h_off) c->h_off = hmalloc<int32_t>(c, (size_t)E + 1, "h_off");
  if (T <= c->T_cap) return;
  auto F_ = [](void* p) { if (p) cudaFree(p); };
  F_(c->p_h); F_(c->p_pkt); F_(c->p_tok); F_(c->p_off); F_(c->p_src); F_(c->p_inv); F_(c->p_gate);
  F_(c->p_x); F_(c->p_a2); F_(c->p_y); F_(c->p_part); F_(c->p_tiles);
  const int64_t M = (int64_t)T * k;
  c->p_ids_off = (int64_t)T * d * 2;
  c->p_w_off = c->p_ids_off + 4 * M;
  c->p_pkt_bytes = c->p_w_off + 4 * M;
  c->p_h = dmalloc<float>(c, (size_t)T * d, "p_h");
  c->p_pkt = dmalloc<char>(c, (size_t)c->p_pkt_bytes, "p_pkt");
  c->p_tok = dmalloc<int32_t>(c, T, "p_tok");
  c->p_off = dmalloc<int32_t>(c, (size_t)E + 1, "p_off");
  c->p_src = dmalloc<int32_t>(c, M, "p_src");
  c->p_inv = dmalloc<int32_t>(c, M, "p_inv");
  c->p_gate = dmalloc<float>(c, M, "p_gate");
  c->p_x = dmalloc<char>(c, (size_t)M * d * 2, "p_x");
  c->p_a2 = dmalloc<char>(c, (size_t)M * F * 2, "p_a2");
  c->p_y = dmalloc<float>(c, (size_t)M * d, "p_y");
  c->p_part = dmalloc<float>(c, (size_t)T * d, "p_part");
  c->tiles_cap = (int)(((M + 127) / 128 + E) * (2 * c->Fs / grouped_gemm_bn(0, 2 * c->Fs) + d / grouped_gemm_bn(1, d)));
  c->p_tiles = dmalloc<int4>(c, (size_t)c->tiles_cap, "p_tiles");
  if (c->H > 0 && c->rank == 0) {
    F_(c->pa_x); F_(c->pa_qkv); F_(c->pa_part); F_(c->pa_out); F_(c->pa_tiles);
    c->pa_x = dmalloc<char>(c, (size_t)T * d * 2, "pa_x");
    c->pa_qkv = dmalloc<float>(c, (size_t)T * c->qkv_rows, "pa_qkv");
    c->pa_part = dmalloc<float>(c, (size_t)std::min(T, kPrefillQChunk) * c->H * attn_splits(T - 1) * (c->hd + 2),
                                "pa_part");
    c->pa_out = dmalloc<float>(c, (size_t)T * d, "pa_out");
    c->pa_tiles = dmalloc<int4>(c, (size_t)((T + 255) / 256 + 1) * (c->qkv_rows / 128 + d / 128 + 2), "pa_tiles");
  }
  c->T_cap = T;
}

// Tile list {expert, row0, rows, n0} for the experts in `mine` (host offsets).
void build_tiles(const std::vector<int32_t>& off, const std::vector<int>& mine, int N, int BN,
                 std::vector<int4>& out) {
  for (int e : mine) {
    const int m = off[e + 1] - off[e];
    const int BM = grouped_gemm_bm();
    for (int m0 = 0; m0 < m; m0 += BM)
      for (int n0 = 0; n0 < N; n0 += BN) out.push_back(make_int4(e, off[e] + m0, std::min(BM, m - m0), n0));
  }
}

// Prefill attention of layer l for positions 0..T-1 (rank 0): x = RMSNorm(h) (bf16), QKV = x W^T on
// the tcgen05 GEMM, RoPE + KV cache rows, causal GQA attention, h += o W_o^T (GEMM + row add).
void prefill_attention(Ctx* c, int l, int T, cudaStream_t s) {
  const int d = c->d, hq = c->H * c->hd;
  const size_t qkv_b = (size_t)c->qkv_rows * d * c->esz, wo_b = (size_t)d * hq * c->esz;
  const size_t kv_l = (size_t)l * c->max_seq * c->kvd * c->kv_esz;
  char* kc = (char*)c->d_kc + kv_l;
  char* vc = (char*)c->d_vc + kv_l;
  const int kvf = c->kv_esz == 4;
  auto gemm = [&](const void* a, const void* w, int N, int K, float* out) {
    std::vector<int4> tiles;
    const int BM = grouped_gemm_bm(), BN = grouped_gemm_bn(1, N);
    for (int m0 = 0; m0 < T; m0 += BM)
      for (int n0 = 0; n0 < N; n0 += BN) tiles.push_back(make_int4(0, m0, std::min(BM, T - m0), n0));
    CUDA_OK(c, cudaMemcpyAsync(c->pa_tiles, tiles.data(), sizeof(int4) * tiles.size(), cudaMemcpyHostToDevice, s));
    GroupedGemmArgs g{};
    g.a = a; g.b[0] = w; g.n_experts = 1; g.tiles = c->pa_tiles; g.n_tiles = (int)tiles.size();
    g.M = T; g.N = N; g.K = K; g.mode = 1; g.out = out; g.gate = nullptr;
    CUDA_OK(c, launch_grouped_gemm(g, s));
    CUDA_OK(c, cudaStreamSynchronize(s));  // the host tile list is reused by the next GEMM
  };
  KTimer t(c, K_ATTN, s);
  CUDA_OK(c, launch_rmsnorm_rows(c->p_h, T, d, c->cfg.rms_eps, c->pa_x, s));
  gemm(c->pa_x, (const char*)c->d_wqkv + qkv_b * l, c->qkv_rows, d, c->pa_qkv);
  CUDA_OK(c, launch_rope_kv(c->pa_qkv, c->qkv_rows, T, c->H, c->Hkv, c->hd, 0, kc, vc, c->kvd, kvf, s));
  for (int t0 = 0; t0 < T; t0 += kPrefillQChunk) {  // query chunks bound the split-partial buffer
    const int tc = std::min(kPrefillQChunk, T - t0);
    const size_t cur = (size_t)t0 * c->kvd * c->kv_esz;
    CUDA_OK(c, launch_attention(c->pa_qkv + (size_t)t0 * c->qkv_rows, c->qkv_rows, tc, c->H, c->Hkv, c->hd, t0, kc, vc,
                                kc + cur, vc + cur, c->kvd, kvf, c->pa_part, nullptr,
                                (char*)c->pa_x + (size_t)t0 * hq * 2, hq, s));
  }
  gemm(c->pa_x, (const char*)c->d_wo + wo_b * l, d, hq, c->pa_out);
  CUDA_OK(c, launch_add_rows(c->p_h, c->pa_out, (long long)T * d, s));
  c->stats.kernel_launches += 6;
}

void prefill_impl(Ctx* c, const int32_t* tokens, int T, int32_t* token_out, int32_t* counts_out) {
  const int L = c->L, E = c->E, k = c->k, d = c->d;
  if (c->wt != W_BF16) fail(c, ODMOE_E_CONFIG, "prefill runs the bf16 tensor-core GEMM: needs dtype BF16");
  if (c->H > 0 && T > c->max_seq) fail(c, ODMOE_E_RANGE, "prompt longer than the KV cache (max_seq)");
  if (E > kMaxGGExperts) fail(c, ODMOE_E_CONFIG, "prefill supports E <= 8");
  if (d % 256 || c->Fs % 128) fail(c, ODMOE_E_CONFIG, "prefill needs d % 256 == 0 and F (per rank) % 128 == 0");
  if (T < 1 || !tokens) fail(c, ODMOE_E_CONFIG, "empty prompt (S:108)");
  if (c->emu > 1) fail(c, ODMOE_E_CONFIG, "emulate_world emulates the decode step only");
  c->predict_cache_token = -1;  // the KV position changes (odmoe_predict_ahead's cache)
  c->align_n = 0;                // a new sequence starts aligned
  c->spec_step = -1;
  for (int t = 0; t < T; ++t)
    if (tokens[t] < 0 || tokens[t] >= c->V) fail(c, ODMOE_E_RANGE, "token out of range");
  ensure_prefill(c, T);
  cudaStream_t s = c->s_main;
  const bool r0 = c->rank == 0;
  const int64_t M = (int64_t)T * k;
  if (r0) {
    CUDA_OK(c, cudaMemcpy(c->p_tok, tokens, 4 * (size_t)T, cudaMemcpyHostToDevice));
    CUDA_OK(c, launch_embed_rows(c->d_emb, c->wt, c->p_tok, T, d, c->p_h, s));
    c->stats.kernel_launches++;
  }
  // this rank's expert loads, in layer order (no prediction in prefill)
  std::vector<std::pair<int, int>> need;
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e)
      if (prefill_mine(c, l, e)) need.push_back({l, e});
  size_t next = 0;
  auto find_p = [&](int l, int e) {
    for (int i = 0; i < (int)c->pslots.size(); ++i)
      if (c->pslots[i].occupied && c->pslots[i].layer == l && c->pslots[i].expert == e) return i;
    return -1;
  };
  auto ppump = [&]() {
    if (c->resident) return;
    while (next < need.size()) {
      int fs = -1;
      for (int i = 0; i < (int)c->pslots.size(); ++i)
        if (!c->pslots[i].occupied) { fs = i; break; }
      if (fs < 0) break;
      submit_into(c, c->pslots[fs], fs, -3, need[next].first, need[next].second, (int64_t)need[next].first * 16, LK_PREFILL);
      next++;
    }
  };
  ppump();
  if (c->cfg.debug_capture && r0) {
    c->p_dbg.assign((size_t)(L + 1) * T * d, 0.f);
    c->p_dbg_ids.assign((size_t)L * T * k, -1);
    CUDA_OK(c, cudaMemcpyAsync(c->p_dbg.data(), c->p_h, sizeof(float) * T * d, cudaMemcpyDeviceToHost, s));
  }
  std::vector<int32_t> counts((size_t)L * E, 0), off(E + 1);
  std::vector<int4> tiles;
  char* u = c->p_pkt;
  int32_t* ids = (int32_t*)(c->p_pkt + c->p_ids_off);
  float* w = (float*)(c->p_pkt + c->p_w_off);
  if (c->H > 0) c->pos = 0;  // a prompt starts a new sequence
  for (int l = 0; l < L; ++l) {
    if (r0 && c->H > 0) prefill_attention(c, l, T, s);
    if (r0) {
      KTimer t(c, K_ROUTER, s);
      CUDA_OK(c, launch_router(c->p_h, nullptr, 0, nullptr, (const char*)c->d_router + (size_t)l * E * d * c->esz,
                               nullptr, c->wt, T, E, d, k, c->cfg.rms_eps, u, ids, w, nullptr, c->d_flag, s));
    }
    if (c->world > 1) NCCL_OK(c, ncclBroadcast(c->p_pkt, c->p_pkt, (size_t)c->p_pkt_bytes, ncclChar, 0, c->comm, s));
    CUDA_OK(c, launch_route_group(ids, w, (int)M, E, c->p_off, c->p_src, c->p_inv, c->p_gate, s));
    CUDA_OK(c, cudaMemcpyAsync(c->h_off, c->p_off, 4 * (size_t)(E + 1), cudaMemcpyDeviceToHost, s));
    CUDA_OK(c, cudaEventRecord(c->ev_ids, s));
    for (;;) {
      const cudaError_t q = cudaEventQuery(c->ev_ids);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) CUDA_OK(c, q);
      ppump();
      if (c->loader.error() != cudaSuccess) CUDA_OK(c, c->loader.error());
      std::this_thread::sleep_for(std::chrono::microseconds(5));
    }
    std::copy(c->h_off, c->h_off + E + 1, off.begin());
    for (int e = 0; e < E; ++e) counts[(size_t)l * E + e] = off[e + 1] - off[e];
    if (c->cfg.debug_capture && r0)
      CUDA_OK(c, cudaMemcpy(c->p_dbg_ids.data() + (size_t)l * T * k, ids, 4 * (size_t)M, cudaMemcpyDeviceToHost));
    const bool in_group = (l % c->NG) == c->my_group;
    if (in_group) {
      std::vector<int> mine;
      for (int e = 0; e < E; ++e)
        if (prefill_mine(c, l, e)) mine.push_back(e);
      CUDA_OK(c, launch_gather_rows(u, c->p_src, k, (int)M, d, c->p_x, s));
      tiles.clear();
      build_tiles(off, mine, 2 * c->Fs, grouped_gemm_bn(0, 2 * c->Fs), tiles);
      const int n1 = (int)tiles.size();
      build_tiles(off, mine, d, grouped_gemm_bn(1, d), tiles);
      const int n2 = (int)tiles.size() - n1;
      if ((int)tiles.size() > c->tiles_cap) fail(c, ODMOE_E_STATE, "tile list overflow");
      if (!tiles.empty())
        CUDA_OK(c, cudaMemcpyAsync(c->p_tiles, tiles.data(), sizeof(int4) * tiles.size(), cudaMemcpyHostToDevice, s));
      GroupedGemmArgs g1{}, g2{};
      g1.n_experts = g2.n_experts = E;
      std::vector<int> used;
      for (int e : mine) {
        const char* blob = nullptr;
        if (c->resident) {
          blob = c->res_blob[(size_t)l * E + e];
        } else {
          const int si = find_p(l, e);
          if (si < 0) fail(c, ODMOE_E_STATE, "prefill expert not loading");
          Slot& sl = c->pslots[si];
          if (!c->loader.wait_issued(sl.req)) {
            if (c->loader.error() != cudaSuccess) CUDA_OK(c, c->loader.error());
            fail(c, ODMOE_E_STATE, "prefill load cancelled");
          }
          CUDA_OK(c, cudaStreamWaitEvent(s, sl.ev_done, 0));
          blob = sl.dev;
          used.push_back(si);
        }
        g1.b[e] = blob;
        g2.b[e] = blob + c->w13_bytes;
      }
      g1.a = c->p_x; g1.tiles = c->p_tiles; g1.n_tiles = n1; g1.M = (int)M; g1.N = 2 * c->Fs; g1.K = d;
      g1.mode = 0; g1.out = c->p_a2; g1.gate = nullptr;
      g2.a = c->p_a2; g2.tiles = c->p_tiles + n1; g2.n_tiles = n2; g2.M = (int)M; g2.N = d; g2.K = c->Fs;
      g2.mode = 1; g2.out = c->p_y; g2.gate = c->p_gate;
      if (c->world > 1) CUDA_OK(c, cudaMemsetAsync(c->p_y, 0, sizeof(float) * M * d, s));
      { KTimer t(c, K_W13, s); CUDA_OK(c, launch_grouped_gemm(g1, s)); }
      { KTimer t(c, K_W2, s); CUDA_OK(c, launch_grouped_gemm(g2, s)); }
      for (int si : used) {
        Slot& sl = c->pslots[si];
        CUDA_OK(c, cudaEventRecord(sl.ev_free, s));
        sl.free_recorded = true;
        sl.req.reset();
        sl.occupied = false;
        sl.layer = sl.expert = -1;
      }
    }
    if (c->world == 1) {
      CUDA_OK(c, launch_scatter_combine(c->p_h, c->p_y, c->p_inv, T, k, d, 0, s));
    } else {
      if (in_group) CUDA_OK(c, launch_scatter_combine(c->p_part, c->p_y, c->p_inv, T, k, d, 1, s));
      else CUDA_OK(c, cudaMemsetAsync(c->p_part, 0, sizeof(float) * T * d, s));
      NCCL_OK(c, ncclReduce(c->p_part, c->p_y, (size_t)T * d, ncclFloat32, ncclSum, 0, c->comm, s));
      if (r0) CUDA_OK(c, launch_add_rows(c->p_h, c->p_y, (long long)T * d, s));
    }
    c->stats.kernel_launches += 4;
    ppump();
    if (c->cfg.debug_capture && r0)
      CUDA_OK(c, cudaMemcpyAsync(c->p_dbg.data() + (size_t)(l + 1) * T * d, c->p_h, sizeof(float) * T * d,
                                 cudaMemcpyDeviceToHost, s));
  }
  if (r0) {
    KTimer t(c, K_LM, s);
    CUDA_OK(c, launch_lm_head(c->p_h + (size_t)(T - 1) * d, c->d_lm, c->wt, c->V, d, c->cfg.rms_eps,
                              c->d_tok_out, c->cfg.debug_capture ? c->d_lmlogits : nullptr, c->d_lmscratch, s));
  }
  if (c->world > 1) NCCL_OK(c, ncclBroadcast(c->d_tok_out, c->d_tok_out, 1, ncclInt32, 0, c->comm, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_tok + 1, c->d_tok_out, 4, cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaMemcpyAsync(c->h_flag, c->d_flag, 4, cudaMemcpyDeviceToHost, s));
  CUDA_OK(c, cudaStreamSynchronize(s));
  if (c->h_flag[0]) fail(c, ODMOE_E_NONFINITE, "non-finite router logits");
  if (c->H > 0) c->pos = T;
  if (c->H > 0 && c->sh_kc) {  // KV0 shadow: it shares the prompt's keys/values once, then keeps its own
    const size_t row = (size_t)c->kvd * c->kv_esz, layer = (size_t)c->max_seq * row;
    for (int l = 0; l < L; ++l) {
      CUDA_OK(c, cudaMemcpyAsync((char*)c->sh_kc + l * layer, (char*)c->d_kc + l * layer, row * T, cudaMemcpyDeviceToDevice, s));
      CUDA_OK(c, cudaMemcpyAsync((char*)c->sh_vc + l * layer, (char*)c->d_vc + l * layer, row * T, cudaMemcpyDeviceToDevice, s));
    }
    CUDA_OK(c, cudaStreamSynchronize(s));
  }
  if (c->cfg.time_kernels) harvest_timers(c);
  c->stats.bytes_h2d = c->loader.bytes_h2d.load();
  c->stats.loads_issued = c->loader.loads_issued.load();
  c->stats.loads_completed = c->loader.loads_completed.load();
  *token_out = c->h_tok[1];
  if (counts_out) std::copy(counts.begin(), counts.end(), counts_out);
  if (c->cfg.debug_capture && r0) {
    // last-token LM logits for the argmax check
    c->hdbg_index.erase(12);
    const int64_t off12 = (int64_t)c->hdbg.size();
    c->hdbg.resize(c->hdbg.size() + (size_t)c->V * 4);
    CUDA_OK(c, cudaMemcpy(c->hdbg.data() + off12, c->d_lmlogits, (size_t)c->V * 4, cudaMemcpyDeviceToHost));
    c->hdbg_index[12] = {off12, (int64_t)c->V * 4};
  }
}

void destroy_ctx(Ctx* c) {
  if (!c) return;
  cudaSetDevice(c->dev);
  c->loader.stop();
  if (c->s_main) cudaStreamSynchronize(c->s_main);
  if (c->s_shadow) cudaStreamSynchronize(c->s_shadow);
  if (c->s_copy) cudaStreamSynchronize(c->s_copy);
  auto F = [](void* p) { if (p) cudaFree(p); };
  for (auto& r : c->tr_pending)
    if (r.e) cudaEventDestroy(r.e);
  for (auto e : c->tr_pool) cudaEventDestroy(e);
  if (c->tr_origin) cudaEventDestroy(c->tr_origin);
  F(c->d_emb); F(c->d_lm); F(c->d_router);
  F(c->d_wqkv); F(c->d_wo); F(c->d_kc); F(c->d_vc); F(c->d_qkv); F(c->d_attn_o); F(c->d_attn_part); F(c->dbg_hpre);
  F(c->sh_qkv); F(c->sh_attn_o); F(c->sh_attn_part); F(c->sh_kcur); F(c->sh_vcur);
  F(c->pa_x); F(c->pa_qkv); F(c->pa_part); F(c->pa_out); F(c->pa_tiles); F(c->sh_kc); F(c->sh_vc);
  if (c->built_pred != ODMOE_PRED_SHADOW_SAME) {
    F(c->sh_wqkv); F(c->sh_sqkv); F(c->sh_wo); F(c->sh_so);
    F(c->sh_emb); F(c->sh_semb); F(c->sh_router); F(c->sh_srouter); F(c->sh_lm); F(c->sh_slm);
    for (auto p : c->sh_blob) F(p);
    for (auto p : c->sh_sc) F(p);
    F(c->d_sh_tbl); F(c->d_sh_stbl);
  }
  for (auto p : c->res_blob) F(p);
  F(c->d_res_tbl);
  for (auto& s : c->slots) {
    F(s.dev);
    if (s.ev_w13) cudaEventDestroy(s.ev_w13);
    if (s.ev_done) cudaEventDestroy(s.ev_done);
    if (s.flag) cudaFree(s.flag);
    if (s.ev_free) cudaEventDestroy(s.ev_free);
  }
  F(c->d_h); F(c->d_pkt); F(c->d_logits); F(c->d_a); F(c->d_y); F(c->d_yred); F(c->d_zero);
  F((void*)c->d_yptr); F((void*)c->d_yredptr); F(c->d_tok_in); F(c->d_tok_out); F(c->d_flag);
  F(c->d_lmscratch); F(c->d_lmlogits);
  F(c->sh_h); F(c->sh_u); F(c->sh_ids_all); F(c->sh_w); F(c->sh_logits_all); F(c->sh_a); F(c->sh_y); F((void*)c->sh_yptr);
  F(c->sh_tok); F(c->sh_lmscratch); F(c->sh_lmlogits);
  F(c->d_yemu); F(c->d_prank); F((void*)c->d_emu_ptr); F(c->dbg_yrank);
  if (c->h_emu_ptr) cudaFreeHost((void*)c->h_emu_ptr);
  F(c->dbg_h); F(c->dbg_ypart); F(c->dbg_yred); F(c->dbg_sh_h_all); F(c->dbg_sh_u_all); F(c->dbg_sh_hf_all); F(c->dbg_hfinal);
  F(c->p_h); F(c->p_pkt); F(c->p_tok); F(c->p_off); F(c->p_src); F(c->p_inv); F(c->p_gate);
  F(c->p_x); F(c->p_a2); F(c->p_y); F(c->p_part); F(c->p_tiles);
  for (auto& s : c->pslots) {
    F(s.dev);
    if (s.ev_w13) cudaEventDestroy(s.ev_w13);
    if (s.ev_done) cudaEventDestroy(s.ev_done);
    if (s.flag) cudaFree(s.flag);
    if (s.ev_free) cudaEventDestroy(s.ev_free);
  }
  if (c->h_off) cudaFreeHost(c->h_off);
  F(c->h_hist); F(c->rf_h); F(c->rf_u); F(c->rf_ids); F(c->rf_w); F(c->rf_y); F(c->rf_a); F((void*)c->rf_yptr);
  if (c->h_ref) cudaFreeHost(c->h_ref);
  for (auto e : c->ev_router) cudaEventDestroy(e);
  for (auto e : c->ev_ref) cudaEventDestroy(e);
  auto FH = [](void* p) { if (p) cudaFreeHost(p); };
  FH(c->pool); FH(c->h_ids); FH(c->h_w); FH(c->h_pred_all); FH(c->h_tok); FH(c->h_flag);
  for (auto e : c->ev_pred_all) cudaEventDestroy(e);
  for (auto e : {c->ev_ids, c->ev_tok, c->ev_shadow_done, c->ev_step}) if (e) cudaEventDestroy(e);
  for (auto& t : c->timed) { c->tev_pool.push_back(t.a); c->tev_pool.push_back(t.b); }
  for (auto e : c->tev_pool) cudaEventDestroy(e);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  for (auto& t : c->graph_timers) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (c->rank != 0) {
    if (c->p2p_part) cudaIpcCloseMemHandle(c->p2p_part);
  } else {
    if (c->p2p_own_part) cudaFree(c->p2p_own_part);
  }
  if (c->comm_pred) ncclCommDestroy(c->comm_pred);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->s_main) cudaStreamDestroy(c->s_main);
  if (c->s_shadow) cudaStreamDestroy(c->s_shadow);
  if (c->s_copy) cudaStreamDestroy(c->s_copy);
  delete c;
}

}  // namespace

// ==================================================================== C ABI
extern "C" {

int32_t odmoe_abi_version(void) { return ODMOE_ABI_VERSION; }

odmoe_status odmoe_plan_layer(int k, int world_size, int group_size, int layer, const int32_t* ids,
                              int rank, int32_t* out, int32_t* n_out) {
  const int G = group_size > 0 ? group_size : std::min(k, world_size);
  if (k < 1 || k > 8 || world_size < 1 || G < 1 || world_size % G || k % G || rank < 0 ||
      rank >= world_size || layer < 0 || !ids || !out || !n_out)
    return ODMOE_E_CONFIG;
  *n_out = plan_layer(k, world_size, G, layer, ids, rank, out);
  return ODMOE_OK;
}

int32_t odmoe_plan_pool_holds(int E, int k, int world_size, int group_size, int layer, int expert, int rank) {
  const int G = group_size > 0 ? group_size : std::min(k, world_size);
  if (k < 1 || E < k || world_size < 1 || G < 1 || world_size % G || k % G || rank < 0 || rank >= world_size)
    return -1;
  return plan_pool_holds(E, k, world_size, G, layer, expert, rank) ? 1 : 0;
}

int odmoe_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return 1;
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

odmoe_status odmoe_create(const odmoe_config* cfg, void** ctx_out) {
  if (ctx_out) *ctx_out = nullptr;
  Ctx* c = nullptr;
  t_create_err.clear();
  odmoe_status st = guard(nullptr, [&] {
    validate(cfg);
    if (!ctx_out) fail(nullptr, ODMOE_E_CONFIG, "null ctx_out");
    c = new Ctx();
    c->cfg = *cfg;
    if (c->cfg.rms_eps <= 0.f) c->cfg.rms_eps = 1e-5f;
    c->L = cfg->L; c->E = cfg->E; c->k = cfg->k; c->d = cfg->d; c->F = cfg->F; c->V = cfg->V;
    c->wt = wtype(cfg->dtype);
    c->esz = dsize(cfg->dtype);
    c->world = cfg->world_size;
    c->rank = cfg->rank;
    c->sliced = cfg->placement == ODMOE_PLACE_SLICED && c->world > 1;
    c->elp = cfg->expert_layer_period;
    c->Fs = c->sliced ? c->F / c->world : c->F;
    c->full_bytes = 3LL * c->F * c->d * (int64_t)c->esz;
    c->blob_elems = 3LL * c->Fs * c->d;
    c->blob_bytes = c->blob_elems * (int64_t)c->esz;
    c->w13_bytes = 2LL * c->Fs * c->d * (int64_t)c->esz;
    if (cfg->emulate_world > 1) {
      c->emu = cfg->emulate_world;
      c->emu_sliced = cfg->placement == ODMOE_PLACE_SLICED;
      if (c->emu_sliced) {
        c->Fs = c->F / c->emu;  // every kernel launch runs one F/N slice, as on a real rank
        c->emu_slice_bytes = 3LL * c->Fs * c->d * (int64_t)c->esz;
        c->emu_w13s = 2LL * c->Fs * c->d * (int64_t)c->esz;
        c->w13_bytes = c->blob_bytes;  // no W13 prefix in a blob of N slices: compute waits for all of it
      } else {
        c->emu_G = cfg->group_size > 0 ? cfg->group_size : std::min(c->k, c->emu);
        c->emu_NG = c->emu / c->emu_G;
      }
    }
    // (an emulated multi-GPU run keeps this process's own placement: one GPU holds everything)
    c->G = c->sliced ? c->world
                     : (cfg->emulate_world > 1 ? 1 : (cfg->group_size > 0 ? cfg->group_size : std::min(c->k, c->world)));
    c->NG = c->world / c->G;
    c->my_group = c->rank / c->G;
    c->my_pos = c->rank % c->G;
    c->resident = cfg->slots_per_gpu == -1;
    if (cfg->n_heads > 0) {
      c->H = cfg->n_heads;
      c->Hkv = cfg->n_kv_heads;
      c->hd = c->d / c->H;
      c->kvd = c->Hkv * c->hd;
      c->qkv_rows = (c->H + 2 * c->Hkv) * c->hd;
      c->max_seq = cfg->max_seq > 0 ? cfg->max_seq : 4096;
      c->kv_esz = cfg->dtype == ODMOE_FP32 ? 4 : 2;
    }
    c->built_pred = cfg->predictor;
    c->dev = cfg->device;
    c->has_shadow = c->rank == 0 && !c->resident &&
                    is_shadow(cfg->predictor);
    try {
      CUDA_OK(c, cudaSetDevice(c->dev));
      // The main model's stream gets the highest priority: when a shadow kernel (SEP, refinement)
      // and a main-model kernel are both pending, the block scheduler hands freed SMs to the main one.
      int prio_lo = 0, prio_hi = 0;
      CUDA_OK(c, cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
      CUDA_OK(c, cudaStreamCreateWithPriority(&c->s_main, cudaStreamNonBlocking, prio_hi));
      CUDA_OK(c, cudaStreamCreateWithPriority(&c->s_shadow, cudaStreamNonBlocking, prio_lo));
      CUDA_OK(c, cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
      if (c->emu > 1) set_stream_sm_reserve(1);  // the flat engine's grid of a rank of a multi-GPU run
      if (c->world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_id, sizeof(id));
        NCCL_OK(c, ncclCommInitRank(&c->comm, c->world, id, c->rank));
        // the prediction communicator moves a few hundred bytes at a time and its receives spin on
        // the shadow stream beside the expert kernels: one CTA, and the flat engine leaves one SM
        ncclConfig_t pcfg = NCCL_CONFIG_INITIALIZER;
        pcfg.minCTAs = 1;
        pcfg.maxCTAs = 1;
        NCCL_OK(c, ncclCommSplit(c->comm, 0, c->rank, &c->comm_pred, &pcfg));
        set_stream_sm_reserve(1);
        setup_p2p(c);
      }
      char* staging = dmalloc<char>(c, (size_t)(c->full_bytes + 2 * c->blob_bytes), "staging");
      if (c->rank == 0) build_nonexpert(c);
      build_pool(c, staging);
      if (c->has_shadow) build_shadow(c, staging);
      CUDA_OK(c, cudaStreamSynchronize(c->s_main));
      cudaFree(staging);
      build_slots(c);
      build_buffers(c);
      if (!c->resident) c->loader.start(c->dev, c->s_copy, cfg->chunk_bytes > 0 ? cfg->chunk_bytes : (32LL << 20), 2);
      CUDA_OK(c, cudaDeviceSynchronize());
    } catch (const Fail& f) {
      t_create_err = c->err;
      destroy_ctx(c);
      c = nullptr;
      throw;
    }
  });
  if (st == ODMOE_OK) *ctx_out = c;
  return st;
}

void odmoe_destroy(void* ctx) { destroy_ctx(reinterpret_cast<Ctx*>(ctx)); }

const char* odmoe_last_error(const void* ctx) {
  if (!ctx) return t_create_err.c_str();
  return reinterpret_cast<const Ctx*>(ctx)->err.c_str();
}

odmoe_status odmoe_get_stats(const void* ctx, odmoe_stats* out) {
  if (!ctx || !out) return ODMOE_E_STATE;
  *out = reinterpret_cast<const Ctx*>(ctx)->stats;
  return ODMOE_OK;
}

odmoe_status odmoe_reset_stats(void* ctx) {
  if (!ctx) return ODMOE_E_STATE;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  odmoe_stats keep = c->stats;
  c->stats = odmoe_stats{};
  c->stats.resident_bytes = keep.resident_bytes;
  c->stats.shadow_bytes = keep.shadow_bytes;
  c->stats.pool_bytes = keep.pool_bytes;
  c->stats.pool_build_s = keep.pool_build_s;
  c->loader.bytes_h2d = 0;
  c->loader.loads_issued = 0;
  c->loader.loads_completed = 0;
  c->loader.loads_cancelled = 0;
  return ODMOE_OK;
}

// Every ctx entry re-applies its flat-engine grid (a multi-GPU rank, real or emulated, leaves one SM
// free); several ctxs may share a device within one process.
#define CTX_GUARD(ctxp)                                                   \
  Ctx* c = reinterpret_cast<Ctx*>(ctxp);                                  \
  if (!c || c->poisoned) return ODMOE_E_STATE;                            \
  cudaSetDevice(c->dev);                                                  \
  set_stream_sm_reserve((c->world > 1 || c->emu > 1) ? 1 : 0);

odmoe_status odmoe_decode_step(void* ctx, int32_t token_in, int32_t* token_out, odmoe_layer_record* rec) {
  CTX_GUARD(ctx);
  if (!token_out) return ODMOE_E_CONFIG;
  return guard(c, [&] { decode_step_impl(c, token_in, token_out, rec); });
}

odmoe_status odmoe_predict_ahead(void* ctx, int32_t token, int from_layer, int depth, int32_t* pred_ids) {
  CTX_GUARD(ctx);
  return guard(c, [&] {
    if (!c->has_shadow) fail(c, ODMOE_E_STATE, "no shadow on this rank");
    CUDA_OK(c, cudaStreamSynchronize(c->s_shadow));  // a previous step's shadow work is done with sh_ids
    if (token < 0 || token >= c->V || from_layer < 0 || depth < 0 || from_layer + depth > c->L)
      fail(c, ODMOE_E_RANGE, "range");
    const int pbuf = Ctx::kPredBufs - 1;  // its own prediction buffer: a speculative pass may hold the others
    if (c->predict_cache_token != token) {
      c->h_tok[0] = token;
      CUDA_OK(c, cudaMemcpyAsync(c->d_tok_in, c->h_tok, 4, cudaMemcpyHostToDevice, c->s_shadow));
      enqueue_shadow(c, c->d_tok_in, pbuf, false);
      CUDA_OK(c, cudaStreamSynchronize(c->s_shadow));
      if (c->cfg.time_kernels || c->pass_timing) harvest_timers(c);
      c->predict_cache_token = token;
    }
    std::vector<int32_t> P((size_t)c->L * c->k);
    CUDA_OK(c, cudaMemcpy(P.data(), c->sh_ids_all + (size_t)pbuf * c->L * c->k, 4 * P.size(), cudaMemcpyDeviceToHost));
    std::copy(P.begin() + (size_t)from_layer * c->k, P.begin() + (size_t)(from_layer + depth) * c->k, pred_ids);
  });
}

odmoe_status odmoe_set_option(void* ctx, int key, int64_t value) {
  CTX_GUARD(ctx);
  return guard(c, [&] {
    if (key == 1) {
      if (value < 1) fail(c, ODMOE_E_CONFIG, "lookahead must be >= 1");
      c->cfg.lookahead = (int32_t)value;
    } else if (key == 2) {
      if (value < 0 || value > 8) fail(c, ODMOE_E_CONFIG, "predictor");
      const bool wants_shadow = is_shadow((int)value);
      if (wants_shadow && value != c->built_pred)
        fail(c, ODMOE_E_STATE, "this ctx was not created with that shadow predictor");
      if (c->resident && value != ODMOE_PRED_NONE) fail(c, ODMOE_E_STATE, "fully-resident ctx loads nothing");
      if (value == ODMOE_PRED_GATE_REUSE && (c->ev_ref.empty() || c->wt != W_BF16))
        fail(c, ODMOE_E_STATE, "gate reuse needs a bf16 ctx created with a shadow or gate-reuse predictor");
      c->cfg.predictor = (int32_t)value;
    } else if (key == 3) {
      if (value < 0 || value > 4) fail(c, ODMOE_E_CONFIG, "refine_depth must be in 0..4");
      if (value > 0 && (c->ev_ref.empty() || c->wt != W_BF16))
        fail(c, ODMOE_E_STATE, "refinement needs a bf16 ctx created with a shadow predictor");
      c->cfg.refine_depth = (int32_t)value;
    } else if (key == 5) {
      if (value != 0 && value != 1) fail(c, ODMOE_E_CONFIG, "kv_align is 0 or 1");
      if (c->H == 0 || !c->has_shadow) fail(c, ODMOE_E_STATE, "kv_align needs an attention ctx with a shadow");
      if (value == 0 && !c->sh_kc) {  // the shadow's own cache (zero: nothing seen yet)
        const size_t kv = (size_t)c->L * c->max_seq * c->kvd * c->kv_esz;
        c->sh_kc = dmalloc<char>(c, kv, "shadow k cache");
        c->sh_vc = dmalloc<char>(c, kv, "shadow v cache");
        CUDA_OK(c, cudaMemset(c->sh_kc, 0, kv));
        CUDA_OK(c, cudaMemset(c->sh_vc, 0, kv));
      }
      c->kv_align = (int)value;
    } else if (key == 6) {
      if (value < 0 || value > 2) fail(c, ODMOE_E_CONFIG, "time_kernels is 0, 1 or 2");
      CUDA_OK(c, cudaStreamSynchronize(c->s_main));
      if (c->cfg.time_kernels) harvest_timers(c);
      c->cfg.time_kernels = (int32_t)value;
      if (c->graph_exec) {  // its timestamp nodes follow the old level: capture again
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
        for (auto& t : c->graph_timers) {
          cudaEventDestroy(t.a);
          cudaEventDestroy(t.b);
        }
        c->graph_timers.clear();
      }
    } else if (key == 4) {
      if (value < 0 || value >= c->max_seq || c->H == 0) fail(c, ODMOE_E_RANGE, "position outside the KV cache");
      c->pos = value;
      c->predict_cache_token = -1;
    } else if (key == 7) {
      if (value != 0 && value != 1) fail(c, ODMOE_E_CONFIG, "trace is 0 or 1");
      if (value && !c->tr_origin) {
        CUDA_OK(c, cudaEventCreate(&c->tr_origin));
        CUDA_OK(c, cudaEventRecord(c->tr_origin, c->s_main));
        CUDA_OK(c, cudaStreamSynchronize(c->s_main));
      }
      c->trace = (int)value;
    } else if (key == 9) {
      if (value != 0 && value != 1) fail(c, ODMOE_E_CONFIG, "pass timing is 0 or 1");
      c->pass_timing = (int)value;
    } else if (key == 8) {
      if (value < 1 || value > 64) fail(c, ODMOE_E_CONFIG, "token alignment period must be in 1..64");
      if (value > 1 && (!is_shadow(c->built_pred) || c->resident || c->H > 0))
        fail(c, ODMOE_E_STATE, "cross-token speculation needs an on-demand shadow ctx without attention");
      c->align_period = (int)value;
      c->align_n = 0;
      c->spec_step = -1;
    } else {
      fail(c, ODMOE_E_CONFIG, "unknown option key");
    }
  });
}

odmoe_status odmoe_trace_read(void* ctx, odmoe_trace_event* out, int32_t cap, int32_t* n_out) {
  CTX_GUARD(ctx);
  return guard(c, [&] {
    if (!c->tr_origin) fail(c, ODMOE_E_STATE, "trace was never enabled");
    if (!n_out || cap < 0 || (cap > 0 && !out)) fail(c, ODMOE_E_CONFIG, "bad output buffer");
    tr_resolve(c);
    const int n = std::min<int>(cap, (int)c->tr_done.size());
    std::copy(c->tr_done.begin(), c->tr_done.begin() + n, out);
    c->tr_done.erase(c->tr_done.begin(), c->tr_done.begin() + n);
    *n_out = n;
  });
}

odmoe_status odmoe_load(void* ctx, int layer, int expert) {
  CTX_GUARD(ctx);
  return guard(c, [&] {
    if (c->resident) fail(c, ODMOE_E_STATE, "fully-resident ctx has no loader");
    if (layer < 0 || layer >= c->L || expert < 0 || expert >= c->E) fail(c, ODMOE_E_RANGE, "range");
    if (!holds_expert(c, layer, expert)) fail(c, ODMOE_E_RANGE, "expert not in this rank's pool");
    if (find_slot(c, -2, layer, expert) >= 0) return;
    const int fs = free_slot(c);
    if (fs < 0) fail(c, ODMOE_E_BUDGET, "all slots occupied");
    submit_load(c, fs, -2, layer, expert, -1, LK_USER);
  });
}

odmoe_status odmoe_load_wait(void* ctx, int layer, int expert, void** w13, void** w2) {
  CTX_GUARD(ctx);
  return guard(c, [&] {
    const int si = find_slot(c, -2, layer, expert);
    if (si < 0) fail(c, ODMOE_E_STATE, "not loading");
    Slot& s = c->slots[si];
    if (!c->loader.wait_issued(s.req)) fail(c, ODMOE_E_STATE, "load cancelled");
    CUDA_OK(c, cudaEventSynchronize(s.ev_done));
    if (w13) *w13 = s.dev;
    if (w2) *w2 = s.dev + c->w13_bytes;
  });
}

odmoe_status odmoe_evict(void* ctx, int layer, int expert) {
  CTX_GUARD(ctx);
  return guard(c, [&] {
    const int si = find_slot(c, -2, layer, expert);
    if (si < 0) fail(c, ODMOE_E_STATE, "expert not resident");
    Slot& s = c->slots[si];
    // after work already on the compute stream: kernels a caller ran on its own streams on the
    // slot's pointers must be ordered before this call by the caller (header contract)
    CUDA_OK(c, cudaEventRecord(s.ev_free, c->s_main));
    s.free_recorded = true;
    release_slot(c, si);
  });
}

odmoe_status odmoe_prefill(void* ctx, const int32_t* tokens, int T, int32_t* token_out, int32_t* expert_counts) {
  CTX_GUARD(ctx);
  if (!token_out) return ODMOE_E_CONFIG;
  return guard(c, [&] { prefill_impl(c, tokens, T, token_out, expert_counts); });
}

odmoe_status odmoe_prefill_debug_read(const void* ctx, int what, int layer, void* dst, int64_t bytes) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !dst) return ODMOE_E_STATE;
  if (what == 0) {  // h entering layer `layer` (layer == L: final), [T][d] fp32
    const int64_t per = (int64_t)c->T_cap * c->d * 4;
    if (c->p_dbg.empty() || layer < 0 || layer > c->L) return ODMOE_E_RANGE;
    const int64_t T = (int64_t)c->p_dbg.size() / ((int64_t)(c->L + 1) * c->d);
    const int64_t per_l = T * c->d * 4;
    (void)per;
    if (bytes > per_l) return ODMOE_E_RANGE;
    std::memcpy(dst, reinterpret_cast<const char*>(c->p_dbg.data()) + layer * per_l, (size_t)bytes);
    return ODMOE_OK;
  }
  if (what == 1) {  // router ids of layer `layer`, [T][k] int32
    if (c->p_dbg_ids.empty() || layer < 0 || layer >= c->L) return ODMOE_E_RANGE;
    const int64_t per_l = (int64_t)c->p_dbg_ids.size() / c->L * 4;
    if (bytes > per_l) return ODMOE_E_RANGE;
    std::memcpy(dst, reinterpret_cast<const char*>(c->p_dbg_ids.data()) + layer * per_l, (size_t)bytes);
    return ODMOE_OK;
  }
  return ODMOE_E_RANGE;
}

odmoe_status odmoe_debug_read(const void* ctx, int what, int layer, void* dst, int64_t bytes) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !dst) return ODMOE_E_STATE;
  auto it = c->hdbg_index.find(what);
  if (it == c->hdbg_index.end()) return ODMOE_E_STATE;
  const bool single = what == 11 || what == 12 || what == 14 || what == 15 || what == 16;
  const int64_t off = it->second.first + (int64_t)(single ? 0 : layer) * it->second.second;
  if (layer < 0 || layer >= c->L || bytes > it->second.second || off + bytes > (int64_t)c->hdbg.size()) return ODMOE_E_RANGE;
  std::memcpy(dst, c->hdbg.data() + off, (size_t)bytes);
  return ODMOE_OK;
}

odmoe_status odmoe_tensor_ptr(const void* ctx, int what, int index, void** ptr) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !ptr) return ODMOE_E_STATE;
  const int LE = c->L * c->E;
  switch (what) {
    case 0: *ptr = c->d_emb; break;
    case 1: *ptr = c->d_lm; break;
    case 2: if (index < 0 || index >= c->L) return ODMOE_E_RANGE; *ptr = (char*)c->d_router + (size_t)index * c->E * c->d * c->esz; break;
    case 3: if (!c->sh_srouter || index < 0 || index >= c->L) return ODMOE_E_RANGE; *ptr = (char*)c->sh_router + (size_t)index * c->E * c->d; break;
    case 4: if (!c->sh_srouter || index < 0 || index >= c->L) return ODMOE_E_RANGE; *ptr = c->sh_srouter + (size_t)index * c->E; break;
    case 5: if (c->sh_blob.empty() || index < 0 || index >= LE) return ODMOE_E_RANGE; *ptr = c->sh_blob[index]; break;
    case 6: if (c->sh_sc.empty() || index < 0 || index >= LE) return ODMOE_E_RANGE; *ptr = c->sh_sc[index]; break;
    case 7: if (c->sh_blob.empty() || index < 0 || index >= LE) return ODMOE_E_RANGE; *ptr = (int8_t*)c->sh_blob[index] + 2LL * c->F * c->d; break;
    case 8: if (c->sh_sc.empty() || index < 0 || index >= LE) return ODMOE_E_RANGE; *ptr = c->sh_sc[index] + 2 * c->F; break;
    case 9: if (!c->sh_semb) return ODMOE_E_RANGE; *ptr = c->sh_emb; break;
    case 10: if (!c->sh_semb) return ODMOE_E_RANGE; *ptr = c->sh_semb; break;
    default: return ODMOE_E_RANGE;
  }
  return ODMOE_OK;
}

// ------------------------------------------------------------------ stateless kernels
static bool router_shape_ok(int m, int E, int d, int k) {
  return m >= 1 && E >= 1 && E <= 64 && k >= 1 && k <= 8 && k <= E && d >= 8 && d % 8 == 0;
}

odmoe_status odmoe_route_topk(float* h, const float* const* y_add, int n_add, const void* gamma,
                              const void* w_gate, int m, int E, int d, int k, int dt, float eps,
                              void* u_out, int32_t* ids, float* w, float* logits, int32_t* flag,
                              void* stream) {
  if (!router_shape_ok(m, E, d, k) || (dt != ODMOE_BF16 && dt != ODMOE_FP32) || n_add < 0 ||
      (n_add > 0 && !y_add) || !h || !w_gate || !u_out || !ids || !w)
    return ODMOE_E_CONFIG;
  return launch_router(h, y_add, n_add, gamma, w_gate, nullptr, wtype(dt), m, E, d, k, eps, u_out,
                       ids, w, logits, flag, S(stream)) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_shadow_route_topk(float* h, const float* const* y_add, int n_add,
                                     const int8_t* q_gate, const float* s_gate, int m, int E, int d,
                                     int k, float eps, void* u_out, int32_t* ids, float* w,
                                     float* logits, int32_t* flag, void* stream) {
  if (!router_shape_ok(m, E, d, k) || d % 16 || n_add < 0 || (n_add > 0 && !y_add) || !h || !q_gate ||
      !s_gate || !u_out || !ids || !w)
    return ODMOE_E_CONFIG;
  return launch_router(h, y_add, n_add, nullptr, q_gate, s_gate, W_I8, m, E, d, k, eps, u_out, ids, w,
                       logits, flag, S(stream)) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_expert_ffn(const void* w13, const void* w2, const void* u, const float* gate_w,
                              int gate_idx, int d, int F, int dt, float* a_scratch, float* y,
                              void* stream) {
  if (!w13 || !w2 || !u || !a_scratch || !y || d < 8 || F < 8 || d % 8 || F % 8 || gate_idx < 0 ||
      (dt != ODMOE_BF16 && dt != ODMOE_FP32))
    return ODMOE_E_CONFIG;
  const WType wt = wtype(dt);
  if (use_fused_expert() && stream_ok(wt, d) && stream_ok(wt, F))
    return launch_expert_fused(direct_ref(w13, nullptr, gate_idx), w2, nullptr, wt, u, dt == ODMOE_FP32, a_scratch,
                               gate_w, y, d, F, S(stream), false) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
  if (launch_w13(direct_ref(w13, nullptr, gate_idx), wt, u, dt == ODMOE_FP32, a_scratch, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  if (launch_w2(direct_ref(w2, nullptr, gate_idx), wt, a_scratch, gate_w, y, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  return ODMOE_OK;
}

odmoe_status odmoe_expert_ffn_grouped(const void* const* w13, const void* const* w2, int n_experts,
                                      const void* x_perm, const int32_t* offsets, const float* gate_perm,
                                      int d, int F, void* a2_scratch, float* y_perm, void* tiles_scratch,
                                      int64_t tiles_scratch_bytes, void* stream) {
  if (!w13 || !w2 || !x_perm || !offsets || !gate_perm || !a2_scratch || !y_perm || !tiles_scratch ||
      n_experts < 1 || n_experts > kMaxGGExperts || d % 256 || F % 128 || d < 256 || F < 128)
    return ODMOE_E_CONFIG;
  std::vector<int32_t> off(offsets, offsets + n_experts + 1);
  for (int e = 0; e < n_experts; ++e)
    if (off[e + 1] < off[e]) return ODMOE_E_CONFIG;
  std::vector<int> all(n_experts);
  for (int e = 0; e < n_experts; ++e) all[e] = e;
  std::vector<int4> tiles;
  build_tiles(off, all, 2 * F, grouped_gemm_bn(0, 2 * F), tiles);
  const int n1 = (int)tiles.size();
  build_tiles(off, all, d, grouped_gemm_bn(1, d), tiles);
  if ((int64_t)(tiles.size() * sizeof(int4)) > tiles_scratch_bytes) return ODMOE_E_CONFIG;
  const int M = off[n_experts];
  if (M == 0) return ODMOE_OK;
  if (cudaMemcpyAsync(tiles_scratch, tiles.data(), sizeof(int4) * tiles.size(), cudaMemcpyHostToDevice, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  GroupedGemmArgs g1{}, g2{};
  g1.n_experts = g2.n_experts = n_experts;
  for (int e = 0; e < n_experts; ++e) { g1.b[e] = w13[e]; g2.b[e] = w2[e]; }
  g1.a = x_perm; g1.tiles = (const int4*)tiles_scratch; g1.n_tiles = n1; g1.M = M; g1.N = 2 * F; g1.K = d;
  g1.mode = 0; g1.out = a2_scratch;
  g2.a = a2_scratch; g2.tiles = (const int4*)tiles_scratch + n1; g2.n_tiles = (int)tiles.size() - n1;
  g2.M = M; g2.N = d; g2.K = F; g2.mode = 1; g2.out = y_perm; g2.gate = gate_perm;
  if (launch_grouped_gemm(g1, S(stream)) != cudaSuccess) return ODMOE_E_CUDA;
  if (launch_grouped_gemm(g2, S(stream)) != cudaSuccess) return ODMOE_E_CUDA;
  // the host tile list must outlive the async copy from pageable memory
  if (cudaStreamSynchronize(S(stream)) != cudaSuccess) return ODMOE_E_CUDA;
  return ODMOE_OK;
}

odmoe_status odmoe_prefill_group(const int32_t* ids, const float* w, int T, int k, int E, int32_t* offsets,
                                 int32_t* src_pair, int32_t* inv, float* gate_perm, void* stream) {
  if (!ids || !w || !offsets || !src_pair || !inv || !gate_perm || T < 0 || k < 1 || E < 1 || E > 64)
    return ODMOE_E_CONFIG;
  return launch_route_group(ids, w, T * k, E, offsets, src_pair, inv, gate_perm, S(stream)) == cudaSuccess
             ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_shadow_expert_ffn(const int8_t* q13, const float* s13, const int8_t* q2,
                                     const float* s2, const void* u, const float* gate_w,
                                     int gate_idx, int d, int F, float* a_scratch, float* y,
                                     void* stream) {
  if (!q13 || !s13 || !q2 || !s2 || !u || !a_scratch || !y || d < 16 || F < 16 || d % 16 || F % 16 || gate_idx < 0)
    return ODMOE_E_CONFIG;
  if (use_fused_expert() && stream_ok(W_I8, d) && stream_ok(W_I8, F))
    return launch_expert_fused(direct_ref(q13, s13, gate_idx), q2, s2, W_I8, u, 0, a_scratch, gate_w, y, d, F,
                               S(stream), false) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
  if (launch_w13(direct_ref(q13, s13, gate_idx), W_I8, u, 0, a_scratch, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  if (launch_w2(direct_ref(q2, s2, gate_idx), W_I8, a_scratch, gate_w, y, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  return ODMOE_OK;
}

odmoe_status odmoe_shadow_expert_ffn_packed(const uint8_t* q13p, const float* s13, const uint8_t* q2p,
                                            const float* s2, const void* u, const float* gate_w, int gate_idx,
                                            int d, int F, float* a_scratch, float* y, void* stream) {
  if (!q13p || !s13 || !q2p || !s2 || !u || !a_scratch || !y || !mma_shadow_ok(d, F) || gate_idx < 0)
    return ODMOE_E_CONFIG;
  if (launch_w13(direct_ref(q13p, s13, gate_idx), W_I8P, u, 0, a_scratch, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  if (launch_w2(direct_ref(q2p, s2, gate_idx), W_I8P, a_scratch, gate_w, y, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  return ODMOE_OK;
}

odmoe_status odmoe_pack_int8_frag(const int8_t* q, int64_t R, int64_t C, int pair_rows, uint8_t* out, void* stream) {
  if (!q || !out || R < 16 || C < 32 || R % 16 || C % 32 || R > INT32_MAX || C > INT32_MAX) return ODMOE_E_CONFIG;
  return launch_pack_i8_frag((const uint8_t*)q, out, (int)R, (int)C, pair_rows, S(stream), true) == cudaSuccess
             ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_shadow_expert_ffn_nf4(const uint8_t* q13, const float* a13, const uint8_t* q2,
                                         const float* a2, const void* u, const float* gate_w, int gate_idx,
                                         int d, int F, float* a_scratch, float* y, void* stream) {
  if (!q13 || !a13 || !q2 || !a2 || !u || !a_scratch || !y || d < 64 || F < 64 || d % 64 || F % 64 || gate_idx < 0)
    return ODMOE_E_CONFIG;
  if (use_fused_expert() && stream_ok(W_NF4, d) && stream_ok(W_NF4, F))
    return launch_expert_fused(direct_ref(q13, a13, gate_idx), q2, a2, W_NF4, u, 0, a_scratch, gate_w, y, d, F,
                               S(stream), false) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
  if (launch_w13(direct_ref(q13, a13, gate_idx), W_NF4, u, 0, a_scratch, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  if (launch_w2(direct_ref(q2, a2, gate_idx), W_NF4, a_scratch, gate_w, y, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  return ODMOE_OK;
}

odmoe_status odmoe_shadow_expert_ffn_fp8(const uint8_t* q13, const float* s13, const uint8_t* q2,
                                         const float* s2, const void* u, const float* gate_w, int gate_idx,
                                         int d, int F, float* a_scratch, float* y, void* stream) {
  if (!q13 || !s13 || !q2 || !s2 || !u || !a_scratch || !y || d < 16 || F < 16 || d % 16 || F % 16 || gate_idx < 0)
    return ODMOE_E_CONFIG;
  if (use_fused_expert() && stream_ok(W_F8, d) && stream_ok(W_F8, F))
    return launch_expert_fused(direct_ref(q13, s13, gate_idx), q2, s2, W_F8, u, 0, a_scratch, gate_w, y, d, F,
                               S(stream), false) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
  if (launch_w13(direct_ref(q13, s13, gate_idx), W_F8, u, 0, a_scratch, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  if (launch_w2(direct_ref(q2, s2, gate_idx), W_F8, a_scratch, gate_w, y, d, F, S(stream)) != cudaSuccess)
    return ODMOE_E_CUDA;
  return ODMOE_OK;
}

odmoe_status odmoe_lm_head_argmax(const float* h, const void* lm_head, int V, int d, int dt, float eps,
                                  int32_t* token_out, float* logits, void* scratch, void* stream) {
  if (!h || !lm_head || !token_out || !scratch || V < 1 || d < 8 || d % 8 || (dt != ODMOE_BF16 && dt != ODMOE_FP32))
    return ODMOE_E_CONFIG;
  // zero the ticket word (the kernel re-zeroes it after use)
  if (cudaMemsetAsync((char*)scratch + 1024 * 8, 0, 8, S(stream)) != cudaSuccess) return ODMOE_E_CUDA;
  return launch_lm_head(h, lm_head, wtype(dt), V, d, eps, token_out, logits, scratch, S(stream)) == cudaSuccess
             ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_quantize_int8_rows(const void* w, int64_t R, int64_t C, int dt, int8_t* q, float* s,
                                      void* stream) {
  if (!w || !q || !s || R < 0 || C < 1 || (dt != ODMOE_BF16 && dt != ODMOE_FP32)) return ODMOE_E_CONFIG;
  return launch_quantize(w, R, C, wtype(dt), q, s, S(stream)) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_quantize_nf4(const void* w, int64_t R, int64_t C, int dt, uint8_t* q, float* absmax,
                                void* stream) {
  if (!w || !q || !absmax || R < 0 || C < 64 || C % 64 || (dt != ODMOE_BF16 && dt != ODMOE_FP32))
    return ODMOE_E_CONFIG;
  return launch_quantize_nf4(w, R, C, wtype(dt), q, absmax, S(stream)) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_quantize_fp8_rows(const void* w, int64_t R, int64_t C, int dt, uint8_t* q, float* s,
                                     void* stream) {
  if (!w || !q || !s || R < 0 || C < 1 || (dt != ODMOE_BF16 && dt != ODMOE_FP32)) return ODMOE_E_CONFIG;
  return launch_quantize_fp8(w, R, C, wtype(dt), q, s, S(stream)) == cudaSuccess ? ODMOE_OK : ODMOE_E_CUDA;
}

odmoe_status odmoe_gen_weights(void* out, int kind, int layer, int expert, int64_t rows, int64_t cols,
                               int64_t fan_in, int d, int F, uint64_t seed, int dt, void* stream) {
  if (!out || kind < 0 || kind > 6 || (dt != ODMOE_BF16 && dt != ODMOE_FP32)) return ODMOE_E_CONFIG;
  if (kind == 0 && (d < 1 || F < 1)) return ODMOE_E_CONFIG;
  if (kind != 0 && (rows < 0 || cols < 0 || fan_in < 1)) return ODMOE_E_CONFIG;
  return launch_gen(out, kind, layer, expert, rows, cols, fan_in, d, F, seed, wtype(dt), S(stream)) == cudaSuccess
             ? ODMOE_OK : ODMOE_E_CUDA;
}

}  // extern "C"
