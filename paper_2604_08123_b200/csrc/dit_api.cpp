// dit_api.cpp -- host side of libdit: context, borrowed weights, adapter pool,
// ControlNet slots, batch plan and the dit_step launch sequence (include/dit.h).
//
// dit_step = one LegoDiffusion model-execution node of the shared base model
// over a cross-workflow batch plus
// denoise().  Launch sequence per step:
//   conditioning MLPs (skinny) -> ALL adaLN modulations (one skinny launch)
//   -> img_in/txt_in (one grouped GEMM, EPI_STORE_H)
//   -> 19 x double block: LN-mod(2 streams) -> [LoRA shrink] -> QKV GEMM
//      (EPI_QKV) -> attention -> [shrink] proj (EPI_RESID) -> LN-mod ->
//      [shrink] fc1 (EPI_GELU) -> [ControlNet wait] [shrink] fc2 (EPI_RESID+CN)
//   -> 38 x single block: LN-mod -> [shrink] linear1 (EPI_QKV split GELU) ->
//      attention -> [shrink] linear2 (EPI_RESID)
//   -> final LN-mod -> final GEMM with the Euler update fused (EPI_FINAL).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <ctime>
#include <vector>

#include "../../include/dit.h"
#include "kernels.h"

using namespace dit;
typedef uint16_t bf16_t;

namespace {

thread_local std::string g_create_error;

struct Lin {
  const void* w = nullptr;
  const void* b = nullptr;
  int out = 0, in = 0;
  CUtensorMap tm;    // weight [out][in], box {64, 128}
  CUtensorMap tm_m;  // merged (patched) copy W' = W + s B A while a lora_merge is active
  bool has_m = false;
};

struct LoraPool {     // one adapted module
  int in = 0, out = 0;
  void* A = nullptr;  // bf16 [slots][r_alloc][in]
  void* B = nullptr;  // bf16 [slots][out][r_alloc]
  CUtensorMap tmA, tmB;
};

struct DoubleStream {
  Lin mod, qkv, proj, fc1, fc2;
  const void* qn = nullptr;
  const void* kn = nullptr;
  int lora[4];  // module index of qkv, proj, fc1, fc2
};
struct SingleBlk {
  Lin mod, l1, l2;
  const void* qn = nullptr;
  const void* kn = nullptr;
  int lora[2];
};

struct RowSpace {     // LoRA bookkeeping for one GEMM row space (txt, img or joint)
  int M = 0, rows_per_req = 0, tiles_m = 0;
  int* row_slot = nullptr;        // device [M]
  int* tile_slots = nullptr;      // device [tiles_m][slot_cap]
  int* tile_cnt = nullptr;        // device [tiles_m]
  int2* shrink_list = nullptr;    // device [n_shrink]
  int n_shrink = 0;
  double rank_rows = 0;           // sum over rows of the adapter rank
  std::vector<int> h_row_slot;    // host copy (debug export)
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

// In-process communicator for tests: one host thread per rank, all ranks'
// contexts in one process (same or peer-accessible devices).  The all-to-all
// is event-ordered device-to-device copies; host barriers make every rank see
// the others' send buffers and events.  Test-only (dit_local_group_create).
struct LocalGroup {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int count = 0;
  long gen = 0;
  std::vector<const void*> send;
  std::vector<cudaEvent_t> ready, done;
  // fused exchange: every rank's peer-visible buffers (same process: plain device pointers)
  std::vector<void*> qkv, o, cat, vcfg;
  std::vector<uint32_t*> flags;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long g = gen;
    if (++count == world) {
      count = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  void a2a(int rank, const void* sendbuf, void* recvbuf, size_t bytes, cudaStream_t s) {
    cudaEventRecord(ready[rank], s);
    send[rank] = sendbuf;
    barrier();
    for (int r = 0; r < world; ++r) {
      cudaStreamWaitEvent(s, ready[r], 0);
      cudaMemcpyAsync(static_cast<uint8_t*>(recvbuf) + (size_t)r * bytes,
                      static_cast<const uint8_t*>(send[r]) + (size_t)rank * bytes, bytes, cudaMemcpyDeviceToDevice, s);
    }
    cudaEventRecord(done[rank], s);
    barrier();
    for (int r = 0; r < world; ++r) cudaStreamWaitEvent(s, done[r], 0);
    barrier();
  }
  // in-place all-gather: rank r's chunk lives at buf + r * bytes in every rank's buf
  void allgather(int rank, void* buf, size_t bytes, cudaStream_t s) {
    cudaEventRecord(ready[rank], s);
    send[rank] = buf;
    barrier();
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      cudaStreamWaitEvent(s, ready[r], 0);
      cudaMemcpyAsync(static_cast<uint8_t*>(buf) + (size_t)r * bytes,
                      static_cast<const uint8_t*>(send[r]) + (size_t)r * bytes, bytes, cudaMemcpyDeviceToDevice, s);
    }
    cudaEventRecord(done[rank], s);
    barrier();
    for (int r = 0; r < world; ++r) cudaStreamWaitEvent(s, done[r], 0);
    barrier();
  }
};

struct dit_ctx {
  dit_config cfg;
  int device = 0;
  int num_sms = 148;
  std::string err;
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
  int D, H, d, F, C, Ct, Cp, Ld, Ls;
  int Nmax, Rmax;
  int r_alloc;
  int mod_total;
  // weights
  std::map<std::string, dit_tensor> tensors;
  bool weights_ready = false;
  Lin img_in, txt_in, t_in, t_out, g_in, g_out, y_in, y_out, fin_mod, fin_lin;
  std::vector<DoubleStream> dbl[2];  // [stream][block], stream 0 = img, 1 = txt
  std::vector<SingleBlk> sgl;
  // adapter pool
  std::vector<LoraPool> pools;
  std::map<int, int> adapter_slot;      // adapter id -> pool slot
  std::vector<float> slot_scale_h;
  std::vector<cudaEvent_t> slot_last_use;
  // asynchronous adapter loading: lora_register / lora_merge run on the caller's
  // side stream; the step waits on these events on ITS stream (no host stall)
  std::vector<cudaEvent_t> slot_ready;   // recorded after lora_register's copies
  cudaEvent_t merge_ready = nullptr;     // recorded after lora_merge's kernel
  cudaEvent_t merged_last_use = nullptr; // recorded by every dit_step that reads the merged copy
  cudaEvent_t step_done = nullptr;       // recorded at the end of every dit_step (in-place merge waits)
  // pinned staging of every per-step host->device upload (plan tables, parameters, ControlNet
  // tables, segment table): a ring of PIN_RING blocks, block i reused only after its copies ran
  static constexpr int PIN_RING = 4;
  uint8_t* pin = nullptr;                // PIN_RING x stage_bytes, cudaHostAlloc
  size_t stage_bytes = 0;
  cudaEvent_t pin_ev[PIN_RING] = {};
  int pin_next = 0;
  // the block the current dit_step stages into (a ring block, or a graph's own block)
  uint8_t* st_base = nullptr;
  size_t st_off = 0;
  cudaEvent_t st_event = nullptr;        // capture: recorded once the graph's staging copies are done
  // in-place merge (lora_merge_inplace): W' written over the base weights, undo log of the elements
  // the inverse cannot recover
  bool merged_inplace = false;
  unsigned long long* inplace_log = nullptr;
  unsigned long long inplace_entries = 0;
  int inplace_tiles = 0, inplace_njobs = 0;
  unsigned long long* mcount = nullptr;  // device counter (workspace)
  int merged_adapter = -1;           // lora_merge: adapter patched into tm_m copies (-1: none)
  // ControlNet registrations for the next step
  struct CnReg { const void* ptr; float scale; cudaEvent_t ready; const uint32_t* flag; uint32_t expect; };
  std::map<std::pair<int, int>, std::vector<CnReg>> cn;   // (slot, block) -> up to CN_FANIN residuals
  // SP
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  LocalGroup* local_group = nullptr;
  bool force_sp = false;             // test-only: SP data path at world == 1 (DIT_FORCE_SP)
  // fused Ulysses exchange (default at P > 1; DIT_SP_NCCL=1 selects the NCCL all-to-all path):
  // the QKV epilogue and the attention epilogue store straight into the owning rank's buffers
  // (peer-mapped through CUDA IPC), with device flag barriers instead of all-to-alls
  bool sp_fused = false;
  bool peers_ready = false;
  void* peer_qkv[8] = {};
  void* peer_o[8] = {};
  void* peer_cat[8] = {};
  PeerFlags peer_flags = {};
  uint32_t* flags = nullptr;         // [8] arrival epochs, written by the peers
  // attention split tail (opt-in, DIT_ATTN_SPLIT_TAIL=1 at dit_create): partials + merge counters
  bool attn_split_tail = false;
  float* attn_tail_ws = nullptr;
  uint32_t* attn_tail_cnt = nullptr;
  uint32_t sp_epoch = 0;
  std::vector<void*> ipc_opened;
  // latent (CFG) parallelism: rank 0 conditional, rank 1 unconditional branch
  int lp_world = 1, lp_rank = 0;
  bool lp_fused = false;             // the final GEMM epilogue stores v into the peer's vcfg too
  float* peer_vcfg[2] = {};
  uint32_t lp_steps = 0;             // step parity selects the vcfg buffer (peer-store WAR safety)
  ncclComm_t lp_comm = nullptr;
  LocalGroup* lp_group = nullptr;
  bf16_t* sp = nullptr;              // [send1 | recv1 | send2 | recv2] at P > 1
  bf16_t* qkv = nullptr;             // attention layout [3][B][H/P][N][d]
  // workspace carve-outs
  float* h = nullptr;
  bf16_t* u = nullptr;
  bf16_t* o = nullptr;
  bf16_t* cat = nullptr;
  bf16_t* sext = nullptr;
  bf16_t* xb = nullptr;
  float* vcfg = nullptr;             // CFG: v of every sequence [2][B][ni][C] (cond block, uncond block)
  uint8_t* mjobs = nullptr;          // lora_merge: device job table (one per adapted linear)
  float2* rope = nullptr;
  float* mod = nullptr;
  float* vec = nullptr;
  float* h1 = nullptr;
  bf16_t* xprep = nullptr;
  bf16_t* temb = nullptr;
  SkinnySeg* segs = nullptr;
  int nsegs = 0, seg_rows = 0;
  bool segs_dirty = true;
  // per-step device params
  float* p_dsig = nullptr;
  float* p_cn_scale = nullptr;
  float* p_sigma = nullptr;
  float* p_guid = nullptr;
  float* p_cfg = nullptr;            // [MAX_SEQ] CFG scale per request
  const void** p_cn_ptr = nullptr;   // [Ld + Ls][CN_FANIN][MAX_SEQ]
  float* p_slot_scale = nullptr;     // [max_adapters]
  float* p_cn_kappa = nullptr;       // [Ld + Ls][CN_FANIN][MAX_SEQ] cn_scale_b * inject scale
  const uint32_t** p_cn_flag = nullptr;   // [Ld + Ls][CN_FANIN][8] device ready flags (controlnet_inject_flag)
  uint32_t* p_cn_expect = nullptr;        // [Ld + Ls][CN_FANIN][MAX_SEQ]
  int* p_img_valid = nullptr;             // [MAX_SEQ] ragged batch: image rows of each sequence
  int* p_seq_valid = nullptr;             // [MAX_SEQ] ragged batch: joint rows of each sequence
  std::vector<int> plan_hw;               // ragged grids the rope tables were built for
  bool cn_flags = false;                  // any flag registration in the current step
  RowSpace rs[3];                    // 0 txt stream, 1 img stream, 2 joint
  int slot_cap = 1;
  // plan cache key
  int plan_B = -1, plan_h = -1, plan_w = -1, plan_nt = -1;
  std::vector<int> plan_slots;
  int rope_key[3] = {-1, -1, -1};
  int last_launches = 0;
  int launches = 0;
  // per-launch profiling (bench.py roofline): events on the launch stream
  struct ProfRec { int kind; double flops; cudaEvent_t a, b; };
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  cudaEvent_t prof_a = nullptr;
  std::vector<int> slot_rank_h;
  int gemm_label = 0;   // profiling sub-kind of the next GEMM launch (10..18)

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
};

// ------------------------------------------------------------------ sizes
namespace {

struct Carve {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  }
};

int n_lora_modules(const dit_config& c) { return c.depth_double * 2 * 4 + c.depth_single * 2; }

// SD3: the last joint block's text stream is context_pre_only (no proj / fc1 / fc2; reading C21).
bool pre_only(const dit_config& c, int block, int stream) {
  return c.arch == DIT_ARCH_SD3 && stream == 1 && block == c.depth_double - 1;
}

bool cfg_valid(const dit_config* c, std::string* why) {
  auto bad = [&](const char* s) { if (why) *why = s; return false; };
  if (!c) return bad("cfg is NULL");
  if (c->hidden <= 0 || c->heads <= 0 || c->hidden % c->heads) return bad("hidden must be a positive multiple of heads");
  int d = c->hidden / c->heads;
  if (d != 32 && d != 64 && d != 128) return bad("head dim must be 32, 64 or 128");
  if (c->hidden % 64) return bad("hidden must be a multiple of 64");
  if (c->hidden > 3072 * 1) { if (c->hidden / 4 > 24 * 32) return bad("hidden > 3072 unsupported"); }
  if (c->arch != DIT_ARCH_FLUX && c->arch != DIT_ARCH_SD3) return bad("arch must be DIT_ARCH_FLUX or DIT_ARCH_SD3");
  if (c->arch == DIT_ARCH_FLUX) {
    if (c->rope_axes[0] + c->rope_axes[1] + c->rope_axes[2] != d) return bad("rope axes must sum to head dim");
    if (c->rope_axes[0] % 2 || c->rope_axes[1] % 2 || c->rope_axes[2] % 2) return bad("rope axes must be even");
  } else {
    if (c->depth_single != 0) return bad("SD3 has no single-stream blocks (depth_single must be 0)");
    if (c->depth_double < 1) return bad("SD3 needs at least one joint block");
    if (c->guidance_embed) return bad("SD3 has no guidance embedding");
    if (c->hidden % 4) return bad("SD3 position table needs hidden % 4 == 0");
    if (c->pos_embed_max < 1 || c->pos_embed_base < 1) return bad("pos_embed_max / pos_embed_base must be positive");
    if (c->qk_norm != 0 && c->qk_norm != 1) return bad("qk_norm must be 0 or 1");
  }
  if (c->depth_double < 0 || c->depth_single < 0) return bad("negative depth");
  if (c->in_channels <= 0 || c->in_channels % 8) return bad("in_channels must be a positive multiple of 8");
  if (c->txt_dim <= 0 || c->txt_dim % 8) return bad("txt_dim must be a positive multiple of 8");
  if (c->pooled_dim <= 0 || c->pooled_dim % 8) return bad("pooled_dim must be a positive multiple of 8");
  if (c->mlp_ratio <= 0) return bad("mlp_ratio must be positive");
  if (c->max_batch < 1 || c->max_batch > MAX_SEQ) return bad("max_batch must be in [1, 16]");
  if (c->max_img_tokens < 1 || c->max_txt_tokens < 1) return bad("token maxima must be positive");
  if (c->max_rank < 0 || c->max_rank > 128) return bad("max_rank must be in [0, 128]");
  if (c->max_adapters < 0 || c->max_adapters > 64) return bad("max_adapters must be in [0, 64]");
  if (c->max_sp_world < 0 || c->max_sp_world > 64) return bad("max_sp_world must be in [0, 64]");
  return true;
}

struct Layout {
  size_t h, u, qkv, sp, o, cat, sext, xb, rope, mod, vec, h1, xprep, temb, segs, params, rowspace, pools, vcfg, mjobs,
      total;
  size_t pool_bytes_per_slot;
};

Layout layout_of(const dit_config& c) {
  Layout L{};
  const size_t D = c.hidden, F = (size_t)c.mlp_ratio * c.hidden, d = D / c.heads;
  const size_t N = (size_t)c.max_img_tokens + c.max_txt_tokens;
  const size_t R = (size_t)c.max_batch * N;
  const size_t r_alloc = c.max_rank > 0 ? align_up(c.max_rank, 64) : 0;
  const size_t mod_total = 12 * D * c.depth_double + 3 * D * c.depth_single + 2 * D;
  const size_t nseg = 2 * c.depth_double + c.depth_single + 1;
  const size_t tiles = (R + GEMM_BM - 1) / GEMM_BM + 4;
  Carve cv;
  L.h = cv.take(R * D * 4);
  L.u = cv.take(R * D * 2);
  L.qkv = cv.take(3 * R * D * 2);
  // SP all-to-all send / recv buffers (8 B*N_loc*D*P elements at any P, incl. the forced P = 1
  // test path); a single-GPU workspace (max_sp_world = 1) keeps only a 64 KB scratch
  L.sp = cv.take(c.max_sp_world == 1 ? (size_t)65536 : 8 * R * D * 2);
  L.o = cv.take(R * D * 2);
  L.cat = cv.take(R * (D + F) * 2);
  L.sext = cv.take(R * (size_t)std::max(c.max_adapters, 1) * std::max<size_t>(r_alloc, 64) * 2);
  L.xb = cv.take((size_t)c.max_batch * c.max_img_tokens * c.in_channels * 2);
  // CFG: v of both branches, twice (latent parallelism over peer stores alternates buffers by step parity)
  L.vcfg = cv.take(4 * (size_t)c.max_batch * c.max_img_tokens * c.in_channels * 4);
  L.mjobs = cv.take((size_t)n_lora_modules(c) * merge_job_bytes() + 256);   // lora_merge job table + counter
  L.rope = cv.take((size_t)c.max_batch * N * (d / 2) * 8);   // one table per sequence for ragged batches
  L.mod = cv.take(MAX_SEQ * mod_total * 4);
  L.vec = cv.take(MAX_SEQ * D * 4);
  L.h1 = cv.take(MAX_SEQ * D * 4);
  L.xprep = cv.take(MAX_SEQ * std::max<size_t>({D, 256, (size_t)c.pooled_dim}) * 2);
  L.temb = cv.take(MAX_SEQ * 256 * 2);
  L.segs = cv.take((nseg + 6) * sizeof(SkinnySeg));
  L.params = cv.take(4096 + (size_t)std::max(c.depth_double + c.depth_single, 1) * CN_FANIN * MAX_SEQ * 2 * (sizeof(void*) + 4) + 2048);
  L.rowspace = cv.take(3 * (R * 4 + tiles * MAX_SEQ * 4 + tiles * 4 + tiles * MAX_SEQ * 8) + 3 * 1024);
  size_t per_slot = 0;
  if (c.max_adapters > 0 && r_alloc > 0) {
    auto add = [&](size_t in, size_t out) { per_slot += r_alloc * in * 2 + out * r_alloc * 2; };
    for (int i = 0; i < c.depth_double * 2; ++i) { add(D, 3 * D); add(D, D); add(D, F); add(F, D); }
    for (int j = 0; j < c.depth_single; ++j) { add(D, 3 * D + F); add(D + F, D); }
  }
  L.pool_bytes_per_slot = per_slot;
  L.pools = cv.take(per_slot * c.max_adapters + n_lora_modules(c) * 2 * 256);
  L.total = cv.off;
  return L;
}

}  // namespace

namespace {
// upper bound of one dit_step's staged host->device bytes (16-byte aligned pieces)
size_t stage_bytes_of(const dit_config& c) {
  const size_t N = (size_t)c.max_img_tokens + c.max_txt_tokens;
  const size_t R = (size_t)c.max_batch * N;
  const size_t tiles = (R + GEMM_TM - 1) / GEMM_TM + 4;
  const size_t ncn = (size_t)std::max(c.depth_double + c.depth_single, 1) * CN_FANIN * MAX_SEQ;
  const size_t nseg = 2 * c.depth_double + c.depth_single + 1 + 6;
  return 3 * (R * 4 + tiles * c.max_batch * 4 + tiles * 4 + tiles * MAX_SEQ * 8 + 64) + MAX_SEQ * 64 + 64 * 4 + 16 * 4 +
         ncn * (2 * sizeof(void*) + 8) + 64 + nseg * sizeof(SkinnySeg) + 4096;
}
}  // namespace

extern "C" size_t dit_workspace_bytes(const dit_config* cfg) {
  if (!cfg_valid(cfg, nullptr)) return 0;
  return layout_of(*cfg).total;
}

// ------------------------------------------------------------------ create / destroy
extern "C" int dit_create(const dit_config* cfg, int device, void* workspace, size_t ws_bytes, dit_ctx** out) {
  std::string why;
  if (!out) { g_create_error = "out is NULL"; return DIT_EINVAL; }
  *out = nullptr;
  if (!cfg_valid(cfg, &why)) { g_create_error = why; return DIT_EINVAL; }
  Layout L = layout_of(*cfg);
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255)) {
    g_create_error = "workspace must be a non-NULL 256-byte aligned device pointer";
    return DIT_EINVAL;
  }
  if (ws_bytes < L.total) {
    g_create_error = "workspace too small: need " + std::to_string(L.total) + " bytes";
    return DIT_ENOMEM;
  }
  if (cudaSetDevice(device) != cudaSuccess) { g_create_error = "cudaSetDevice failed"; return DIT_ECUDA; }
  {
    // every libdit kernel loaded now, not at its first launch (common.cuh preload_module_of): a
    // lazy load while a spinning kernel of this process waits on it (exchange barriers, ControlNet
    // flags, in-process ranks) can stall until the spin gives up
    static std::once_flag once;
    std::call_once(once, [] {
      const cudaError_t e[5] = {gemm_preload(), attention_tc_preload(), attention_mma_preload(), elementwise_preload(),
                                merge_preload()};
      for (cudaError_t x : e)
        if (x != cudaSuccess) fprintf(stderr, "[libdit] eager kernel loading unavailable (%s)\n", cudaGetErrorString(x));
    });
  }
  dit_ctx* c = new dit_ctx();
  c->cfg = *cfg;
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  c->ws = static_cast<uint8_t*>(workspace);
  c->ws_bytes = ws_bytes;
  c->D = cfg->hidden;
  c->H = cfg->heads;
  c->d = c->D / c->H;
  c->F = cfg->mlp_ratio * c->D;
  c->C = cfg->in_channels;
  c->Ct = cfg->txt_dim;
  c->Cp = cfg->pooled_dim;
  c->Ld = cfg->depth_double;
  c->Ls = cfg->depth_single;
  c->Nmax = cfg->max_img_tokens + cfg->max_txt_tokens;
  c->Rmax = cfg->max_batch * c->Nmax;
  c->r_alloc = cfg->max_rank > 0 ? (int)align_up(cfg->max_rank, 64) : 64;
  {
    const char* st = getenv("DIT_ATTN_SPLIT_TAIL");
    if (st && st[0] == '1') {
      const size_t wsb = attn_tail_ws_bytes(std::max(cfg->hidden / std::max(cfg->heads, 1), 64));
      if (cudaMalloc(&c->attn_tail_ws, wsb) == cudaSuccess &&
          cudaMalloc(&c->attn_tail_cnt, ATTN_TAIL_UNITS * 2 * 4) == cudaSuccess &&
          cudaMemset(c->attn_tail_cnt, 0, ATTN_TAIL_UNITS * 2 * 4) == cudaSuccess)
        c->attn_split_tail = true;
    }
  }
  c->mod_total = 12 * c->D * c->Ld + 3 * c->D * c->Ls + 2 * c->D;
  uint8_t* w = c->ws;
  c->h = reinterpret_cast<float*>(w + L.h);
  c->u = reinterpret_cast<bf16_t*>(w + L.u);
  c->qkv = reinterpret_cast<bf16_t*>(w + L.qkv);
  c->sp = reinterpret_cast<bf16_t*>(w + L.sp);
  c->o = reinterpret_cast<bf16_t*>(w + L.o);
  c->cat = reinterpret_cast<bf16_t*>(w + L.cat);
  c->sext = reinterpret_cast<bf16_t*>(w + L.sext);
  c->xb = reinterpret_cast<bf16_t*>(w + L.xb);
  c->vcfg = reinterpret_cast<float*>(w + L.vcfg);
  c->mjobs = w + L.mjobs;
  c->mcount = reinterpret_cast<unsigned long long*>(w + L.mjobs + align_up((size_t)n_lora_modules(*cfg) * merge_job_bytes(), 256));
  c->rope = reinterpret_cast<float2*>(w + L.rope);
  c->mod = reinterpret_cast<float*>(w + L.mod);
  c->vec = reinterpret_cast<float*>(w + L.vec);
  c->h1 = reinterpret_cast<float*>(w + L.h1);
  c->xprep = reinterpret_cast<bf16_t*>(w + L.xprep);
  c->temb = reinterpret_cast<bf16_t*>(w + L.temb);
  c->segs = reinterpret_cast<SkinnySeg*>(w + L.segs);
  {
    Carve cv;
    uint8_t* p = w + L.params;
    c->p_dsig = reinterpret_cast<float*>(p + cv.take(MAX_SEQ * 4));
    c->p_cn_scale = reinterpret_cast<float*>(p + cv.take(MAX_SEQ * 4));
    c->p_sigma = reinterpret_cast<float*>(p + cv.take(MAX_SEQ * 4));
    c->p_guid = reinterpret_cast<float*>(p + cv.take(MAX_SEQ * 4));
    c->p_cfg = reinterpret_cast<float*>(p + cv.take(MAX_SEQ * 4));
    c->p_slot_scale = reinterpret_cast<float*>(p + cv.take(64 * 4));
    const size_t ncn = (size_t)std::max(c->Ld + c->Ls, 1) * CN_FANIN * MAX_SEQ;
    c->p_cn_ptr = reinterpret_cast<const void**>(p + cv.take(ncn * sizeof(void*)));
    c->p_cn_kappa = reinterpret_cast<float*>(p + cv.take(ncn * 4));
    c->p_cn_flag = reinterpret_cast<const uint32_t**>(p + cv.take(ncn * sizeof(void*)));
    c->p_cn_expect = reinterpret_cast<uint32_t*>(p + cv.take(ncn * 4));
    c->p_img_valid = reinterpret_cast<int*>(p + cv.take(MAX_SEQ * 4));
    c->p_seq_valid = reinterpret_cast<int*>(p + cv.take(MAX_SEQ * 4));
    c->flags = reinterpret_cast<uint32_t*>(p + cv.take(8 * 4));
  }
  {
    const size_t tiles = (c->Rmax + GEMM_BM - 1) / GEMM_BM + 4;
    Carve cv;
    uint8_t* p = w + L.rowspace;
    for (int s = 0; s < 3; ++s) {
      c->rs[s].row_slot = reinterpret_cast<int*>(p + cv.take(c->Rmax * 4));
      c->rs[s].tile_slots = reinterpret_cast<int*>(p + cv.take(tiles * MAX_SEQ * 4));
      c->rs[s].tile_cnt = reinterpret_cast<int*>(p + cv.take(tiles * 4));
      c->rs[s].shrink_list = reinterpret_cast<int2*>(p + cv.take(tiles * MAX_SEQ * 8));
    }
  }
  c->slot_cap = cfg->max_batch;
  // adapter pools
  const int nmod = n_lora_modules(*cfg);
  c->pools.resize(nmod);
  {
    size_t off = L.pools;
    int mi = 0;
    const int D = c->D, F = c->F;
    auto add = [&](int in, int out) {
      LoraPool& P = c->pools[mi++];
      P.in = in;
      P.out = out;
      if (cfg->max_adapters > 0 && cfg->max_rank > 0) {
        P.A = w + off;
        off = align_up(off + (size_t)cfg->max_adapters * c->r_alloc * in * 2, 256);
        P.B = w + off;
        off = align_up(off + (size_t)cfg->max_adapters * out * c->r_alloc * 2, 256);
        // A pool viewed [slots*r_alloc][in]; B pool viewed [slots*out][r_alloc]
        make_tmap_2d(&P.tmA, P.A, in, (uint64_t)cfg->max_adapters * c->r_alloc, (uint64_t)in * 2, 64, 128);
        make_tmap_2d(&P.tmB, P.B, c->r_alloc, (uint64_t)cfg->max_adapters * out, (uint64_t)c->r_alloc * 2, 64, 128);
      }
    };
    for (int i = 0; i < c->Ld; ++i)
      for (int s = 0; s < 2; ++s) { add(D, 3 * D); add(D, D); add(D, F); add(F, D); }
    for (int j = 0; j < c->Ls; ++j) { add(D, 3 * D + F); add(D + F, D); }
  }
  c->slot_scale_h.assign(std::max(cfg->max_adapters, 1), 0.f);
  c->slot_rank_h.assign(std::max(cfg->max_adapters, 1), 0);
  c->slot_last_use.assign(std::max(cfg->max_adapters, 1), nullptr);
  for (auto& e : c->slot_last_use) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  c->slot_ready.assign(std::max(cfg->max_adapters, 1), nullptr);
  for (auto& e : c->slot_ready) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->merge_ready, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->merged_last_use, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->step_done, cudaEventDisableTiming);
  c->stage_bytes = align_up(stage_bytes_of(*cfg), 256);
  if (cudaHostAlloc(reinterpret_cast<void**>(&c->pin), c->stage_bytes * dit_ctx::PIN_RING, cudaHostAllocDefault) !=
      cudaSuccess) {
    g_create_error = "cudaHostAlloc of the pinned staging ring failed";
    delete c;
    return DIT_ECUDA;
  }
  for (auto& e : c->pin_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  c->dbl[0].resize(c->Ld);
  c->dbl[1].resize(c->Ld);
  c->sgl.resize(c->Ls);
  {
    int mi = 0;
    for (int i = 0; i < c->Ld; ++i)
      for (int s = 0; s < 2; ++s)
        for (int t = 0; t < 4; ++t) c->dbl[s][i].lora[t] = mi++;
    for (int j = 0; j < c->Ls; ++j)
      for (int t = 0; t < 2; ++t) c->sgl[j].lora[t] = mi++;
  }
  if (cudaGetLastError() != cudaSuccess) {
    g_create_error = "CUDA error during context creation";
    delete c;
    return DIT_ECUDA;
  }
  *out = c;
  return DIT_OK;
}

extern "C" void dit_destroy(dit_ctx* c) {
  if (!c) return;
  for (auto& e : c->ev_pool) cudaEventDestroy(e);
  for (auto& e : c->slot_last_use)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->slot_ready)
    if (e) cudaEventDestroy(e);
  if (c->merge_ready) cudaEventDestroy(c->merge_ready);
  if (c->merged_last_use) cudaEventDestroy(c->merged_last_use);
  if (c->step_done) cudaEventDestroy(c->step_done);
  for (auto& e : c->pin_ev)
    if (e) cudaEventDestroy(e);
  if (c->pin) cudaFreeHost(c->pin);
  if (c->attn_tail_ws) cudaFree(c->attn_tail_ws);
  if (c->attn_tail_cnt) cudaFree(c->attn_tail_cnt);
  for (void* ptr : c->ipc_opened) dit_ipc_close(ptr);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->lp_comm) ncclCommDestroy(c->lp_comm);
  delete c;
}

extern "C" const char* dit_last_error(const dit_ctx* c) {
  if (!c) return g_create_error.c_str();
  return c->err.c_str();
}

// ------------------------------------------------------------------ weights
namespace {

struct Expect {
  std::string name;
  int64_t s0, s1;   // s1 = -1 for rank-1
};

void expected_tensors(const dit_ctx* c, std::vector<Expect>& e) {
  const int D = c->D, C = c->C, Ct = c->Ct, Cp = c->Cp, F = c->F, d = c->d;
  auto lin = [&](const std::string& n, int out, int in) {
    e.push_back({n + ".w", out, in});
    e.push_back({n + ".b", out, -1});
  };
  lin("img_in", D, C);
  lin("txt_in", D, Ct);
  lin("time_in.in", D, 256);
  lin("time_in.out", D, D);
  if (c->cfg.guidance_embed) { lin("guidance_in.in", D, 256); lin("guidance_in.out", D, D); }
  lin("vector_in.in", D, Cp);
  lin("vector_in.out", D, D);
  const bool norms = c->cfg.arch == DIT_ARCH_FLUX || c->cfg.qk_norm;
  for (int i = 0; i < c->Ld; ++i)
    for (int st = 0; st < 2; ++st) {
      std::string p = "double." + std::to_string(i) + (st == 0 ? ".img." : ".txt.");
      const bool po = pre_only(c->cfg, i, st);
      lin(p + "mod", (po ? 2 : 6) * D, D);
      lin(p + "qkv", 3 * D, D);
      if (norms) {
        e.push_back({p + "q_norm", d, -1});
        e.push_back({p + "k_norm", d, -1});
      }
      if (po) continue;
      lin(p + "proj", D, D);
      lin(p + "fc1", F, D);
      lin(p + "fc2", D, F);
    }
  for (int j = 0; j < c->Ls; ++j) {
    std::string p = "single." + std::to_string(j) + ".";
    lin(p + "mod", 3 * D, D);
    lin(p + "linear1", 3 * D + F, D);
    e.push_back({p + "q_norm", d, -1});
    e.push_back({p + "k_norm", d, -1});
    lin(p + "linear2", D, D + F);
  }
  lin("final.mod", 2 * D, D);
  lin("final.linear", C, D);
}

bool bind_lin(dit_ctx* c, Lin& L, const std::string& name) {
  auto w = c->tensors.find(name + ".w");
  auto b = c->tensors.find(name + ".b");
  if (w == c->tensors.end() || b == c->tensors.end()) return false;
  L.w = w->second.ptr;
  L.b = b->second.ptr;
  L.out = (int)w->second.shape[0];
  L.in = (int)w->second.shape[1];
  return make_tmap_2d(&L.tm, L.w, L.in, L.out, (uint64_t)L.in * 2, 64, 128);
}

int bind_all(dit_ctx* c) {
  std::vector<Expect> ex;
  expected_tensors(c, ex);
  for (auto& e : ex)
    if (!c->tensors.count(e.name)) return 0;
  bool ok = true;
  ok &= bind_lin(c, c->img_in, "img_in");
  ok &= bind_lin(c, c->txt_in, "txt_in");
  ok &= bind_lin(c, c->t_in, "time_in.in");
  ok &= bind_lin(c, c->t_out, "time_in.out");
  if (c->cfg.guidance_embed) {
    ok &= bind_lin(c, c->g_in, "guidance_in.in");
    ok &= bind_lin(c, c->g_out, "guidance_in.out");
  }
  ok &= bind_lin(c, c->y_in, "vector_in.in");
  ok &= bind_lin(c, c->y_out, "vector_in.out");
  for (int i = 0; i < c->Ld; ++i)
    for (int s = 0; s < 2; ++s) {
      std::string p = "double." + std::to_string(i) + (s == 0 ? ".img." : ".txt.");
      DoubleStream& B = c->dbl[s][i];
      ok &= bind_lin(c, B.mod, p + "mod");
      ok &= bind_lin(c, B.qkv, p + "qkv");
      if (!pre_only(c->cfg, i, s)) {
        ok &= bind_lin(c, B.proj, p + "proj");
        ok &= bind_lin(c, B.fc1, p + "fc1");
        ok &= bind_lin(c, B.fc2, p + "fc2");
      }
      B.qn = B.kn = nullptr;   // SD3-medium: no QK-norm (the epilogue skips it)
      if (c->cfg.arch == DIT_ARCH_FLUX || c->cfg.qk_norm) {
        B.qn = c->tensors[p + "q_norm"].ptr;
        B.kn = c->tensors[p + "k_norm"].ptr;
      }
    }
  for (int j = 0; j < c->Ls; ++j) {
    std::string p = "single." + std::to_string(j) + ".";
    SingleBlk& S = c->sgl[j];
    ok &= bind_lin(c, S.mod, p + "mod");
    ok &= bind_lin(c, S.l1, p + "linear1");
    ok &= bind_lin(c, S.l2, p + "linear2");
    S.qn = c->tensors[p + "q_norm"].ptr;
    S.kn = c->tensors[p + "k_norm"].ptr;
  }
  ok &= bind_lin(c, c->fin_mod, "final.mod");
  ok &= bind_lin(c, c->fin_lin, "final.linear");
  return ok ? 1 : -1;
}

}  // namespace

extern "C" int dit_load_weights(dit_ctx* c, const dit_tensor* t, int n) {
  if (!c) return DIT_EINVAL;
  // the merged copies W' were computed from the current base weights: replacing a base tensor
  // under them would leave the step running a stale patch
  if (c->merged_adapter >= 0)
    return c->fail(DIT_EINVAL, "adapter %d is merged; lora_unmerge before replacing base weights", c->merged_adapter);
  if (n < 0 || (n > 0 && !t)) return c->fail(DIT_EINVAL, "bad tensor list");
  std::vector<Expect> ex;
  expected_tensors(c, ex);
  std::map<std::string, Expect> want;
  for (auto& e : ex) want[e.name] = e;
  std::map<std::string, int> seen;
  for (int i = 0; i < n; ++i) {
    if (!t[i].name) return c->fail(DIT_EINVAL, "tensor %d has no name", i);
    auto it = want.find(t[i].name);
    if (it == want.end()) return c->fail(DIT_EINVAL, "unknown tensor '%s'", t[i].name);
    if (seen.count(t[i].name)) return c->fail(DIT_EINVAL, "duplicate tensor '%s'", t[i].name);
    seen[t[i].name] = 1;
    if (t[i].dtype != 0) return c->fail(DIT_EINVAL, "tensor '%s': dtype must be bf16 (0)", t[i].name);
    if (!t[i].ptr || (reinterpret_cast<uintptr_t>(t[i].ptr) & 15))
      return c->fail(DIT_EINVAL, "tensor '%s': NULL or not 16-byte aligned", t[i].name);
    const Expect& e = it->second;
    const bool r1 = e.s1 < 0;
    if ((r1 && (t[i].rank != 1 || t[i].shape[0] != e.s0)) ||
        (!r1 && (t[i].rank != 2 || t[i].shape[0] != e.s0 || t[i].shape[1] != e.s1)))
      return c->fail(DIT_EINVAL, "tensor '%s': wrong shape", t[i].name);
  }
  for (int i = 0; i < n; ++i) {
    dit_tensor copy = t[i];
    c->tensors[t[i].name] = copy;
    c->tensors[t[i].name].name = nullptr;
  }
  int r = bind_all(c);
  if (r < 0) return c->fail(DIT_ECUDA, "tensor map encoding failed");
  c->weights_ready = (r == 1);
  c->segs_dirty = true;
  return DIT_OK;
}

// ------------------------------------------------------------------ LoRA registry
extern "C" int lora_register(dit_ctx* c, int32_t adapter_id, int32_t rank, float scale, const dit_tensor* t, int n,
                             void* stream) {
  if (!c) return DIT_EINVAL;
  if (adapter_id < 0) return c->fail(DIT_EINVAL, "adapter id must be >= 0");
  if (c->adapter_slot.count(adapter_id)) return c->fail(DIT_EEXIST, "adapter %d already registered", adapter_id);
  if (rank <= 0 || rank > c->cfg.max_rank) return c->fail(DIT_ERANK, "rank %d not in [1, %d]", rank, c->cfg.max_rank);
  if (!std::isfinite(scale)) return c->fail(DIT_EINVAL, "scale must be finite");
  if (n < 0 || (n > 0 && !t)) return c->fail(DIT_EINVAL, "bad tensor list");
  int slot = -1;
  for (int s = 0; s < c->cfg.max_adapters; ++s) {
    bool used = false;
    for (auto& kv : c->adapter_slot)
      if (kv.second == s) used = true;
    if (!used) { slot = s; break; }
  }
  if (slot < 0) return c->fail(DIT_ENOSPC, "adapter pool full (%d slots)", c->cfg.max_adapters);
  // module name -> index
  std::map<std::string, int> modidx;
  for (int i = 0; i < c->Ld; ++i)
    for (int s = 0; s < 2; ++s) {
      const char* names[4] = {"qkv", "proj", "fc1", "fc2"};
      for (int q = 0; q < (pre_only(c->cfg, i, s) ? 1 : 4); ++q)
        modidx["double." + std::to_string(i) + (s == 0 ? ".img." : ".txt.") + names[q]] = c->dbl[s][i].lora[q];
    }
  for (int j = 0; j < c->Ls; ++j) {
    modidx["single." + std::to_string(j) + ".linear1"] = c->sgl[j].lora[0];
    modidx["single." + std::to_string(j) + ".linear2"] = c->sgl[j].lora[1];
  }
  struct Job { int mod; bool isA; const dit_tensor* t; };
  std::vector<Job> jobs;
  std::map<std::string, int> seen;
  for (int i = 0; i < n; ++i) {
    if (!t[i].name || !t[i].ptr) return c->fail(DIT_EINVAL, "tensor %d: NULL name or pointer", i);
    std::string nm = t[i].name;
    bool isA;
    std::string mod;
    if (nm.size() > 7 && nm.compare(nm.size() - 7, 7, ".lora_A") == 0) { isA = true; mod = nm.substr(0, nm.size() - 7); }
    else if (nm.size() > 7 && nm.compare(nm.size() - 7, 7, ".lora_B") == 0) { isA = false; mod = nm.substr(0, nm.size() - 7); }
    else return c->fail(DIT_EINVAL, "tensor '%s' is not <module>.lora_A/B", t[i].name);
    auto it = modidx.find(mod);
    if (it == modidx.end()) return c->fail(DIT_EINVAL, "'%s' is not an adapted module", mod.c_str());
    if (seen.count(nm)) return c->fail(DIT_EINVAL, "duplicate tensor '%s'", t[i].name);
    seen[nm] = 1;
    const LoraPool& P = c->pools[it->second];
    if (t[i].dtype != 0 || t[i].rank != 2) return c->fail(DIT_EINVAL, "'%s': must be a rank-2 bf16 tensor", t[i].name);
    if (isA && (t[i].shape[0] != rank || t[i].shape[1] != P.in))
      return c->fail(DIT_EINVAL, "'%s': expected [%d][%d]", t[i].name, rank, P.in);
    if (!isA && (t[i].shape[0] != P.out || t[i].shape[1] != rank))
      return c->fail(DIT_EINVAL, "'%s': expected [%d][%d]", t[i].name, P.out, rank);
    jobs.push_back({it->second, isA, &t[i]});
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int ra = c->r_alloc;
  // zero the whole slot of every module, then copy the given matrices
  for (auto& P : c->pools) {
    cudaMemsetAsync(static_cast<uint8_t*>(P.A) + (size_t)slot * ra * P.in * 2, 0, (size_t)ra * P.in * 2, s);
    cudaMemsetAsync(static_cast<uint8_t*>(P.B) + (size_t)slot * P.out * ra * 2, 0, (size_t)P.out * ra * 2, s);
  }
  // sources may be device memory or pinned host memory (cudaMemcpyDefault, UVA): an adapter can be
  // loaded straight from host RAM over PCIe on a side stream while steps run
  for (auto& j : jobs) {
    LoraPool& P = c->pools[j.mod];
    if (j.isA) {
      cudaMemcpyAsync(static_cast<uint8_t*>(P.A) + (size_t)slot * ra * P.in * 2, j.t->ptr, (size_t)rank * P.in * 2,
                      cudaMemcpyDefault, s);
    } else {
      cudaMemcpy2DAsync(static_cast<uint8_t*>(P.B) + (size_t)slot * P.out * ra * 2, (size_t)ra * 2, j.t->ptr,
                        (size_t)rank * 2, (size_t)rank * 2, P.out, cudaMemcpyDefault, s);
    }
  }
  cudaEventRecord(c->slot_ready[slot], s);   // every dit_step using the slot waits on this, on its stream
  if (cudaGetLastError() != cudaSuccess) return c->fail(DIT_ECUDA, "adapter copy failed");
  c->adapter_slot[adapter_id] = slot;
  c->slot_scale_h[slot] = scale;
  c->slot_rank_h[slot] = rank;
  c->plan_B = -1;  // slot tables may change
  return DIT_OK;
}

extern "C" int lora_unregister(dit_ctx* c, int32_t adapter_id) {
  if (!c) return DIT_EINVAL;
  auto it = c->adapter_slot.find(adapter_id);
  if (it == c->adapter_slot.end()) return c->fail(DIT_ENOENT, "adapter %d not registered", adapter_id);
  if (adapter_id == c->merged_adapter) return c->fail(DIT_EINVAL, "adapter %d is merged; lora_unmerge first", adapter_id);
  cudaEventSynchronize(c->slot_last_use[it->second]);
  c->adapter_slot.erase(it);
  c->plan_B = -1;
  return DIT_OK;
}

// ------------------------------------------------------------------ merged LoRA (hot patch)
namespace {
// Adapted linears in LoRA-pool module order: double blocks (img then txt stream; qkv, proj,
// fc1, fc2), then single blocks (linear1, linear2).  (out, in) from the config alone.
void adapted_shapes(const dit_config& cfg, std::vector<std::pair<int, int>>& v) {
  const int D = cfg.hidden, F = cfg.mlp_ratio * cfg.hidden;
  v.clear();
  for (int i = 0; i < cfg.depth_double; ++i)
    for (int s = 0; s < 2; ++s) {
      v.push_back({3 * D, D});
      if (pre_only(cfg, i, s)) continue;
      v.push_back({D, D});
      v.push_back({F, D});
      v.push_back({D, F});
    }
  for (int j = 0; j < cfg.depth_single; ++j) {
    v.push_back({3 * D + F, D});
    v.push_back({D, D + F});
  }
}
std::vector<std::pair<Lin*, int>> adapted_lins(dit_ctx* c) {
  std::vector<std::pair<Lin*, int>> v;
  for (int i = 0; i < c->Ld; ++i)
    for (int s = 0; s < 2; ++s) {
      DoubleStream& X = c->dbl[s][i];
      Lin* L[4] = {&X.qkv, &X.proj, &X.fc1, &X.fc2};
      for (int q = 0; q < (pre_only(c->cfg, i, s) ? 1 : 4); ++q) v.push_back({L[q], X.lora[q]});
    }
  for (int j = 0; j < c->Ls; ++j) {
    v.push_back({&c->sgl[j].l1, c->sgl[j].lora[0]});
    v.push_back({&c->sgl[j].l2, c->sgl[j].lora[1]});
  }
  return v;
}
}  // namespace

extern "C" size_t dit_merge_bytes(const dit_config* cfg) {
  if (!cfg_valid(cfg, nullptr)) return 0;
  std::vector<std::pair<int, int>> v;
  adapted_shapes(*cfg, v);
  size_t off = 0;
  for (auto& oi : v) off = align_up(off + (size_t)oi.first * oi.second * 2, 256);
  return off;
}

namespace {
// Job table of every adapted linear for the tensor-core merge kernel (merge_tc.cu), copied to the
// workspace on `s` (staged: the host buffer is reusable at once).  out_maps == nullptr: in place
// (the output map is the weight map itself).
bool upload_merge_jobs(dit_ctx* c, int slot, const std::vector<CUtensorMap>* out_maps, cudaStream_t s, int* tiles) {
  auto lins = adapted_lins(c);
  const int ra = c->r_alloc;
  const float scale = c->slot_scale_h[slot];
  const size_t jb = merge_job_bytes();
  std::vector<uint8_t> store(align_up(lins.size() * jb, 64) + 64);
  uint8_t* host = reinterpret_cast<uint8_t*>(align_up(reinterpret_cast<uintptr_t>(store.data()), 64));
  int t = 0;
  long long elem = 0;
  for (size_t k = 0; k < lins.size(); ++k) {
    Lin& L = *lins[k].first;
    const LoraPool& P = c->pools[lins[k].second];
    if (!merge_job_fill(host + k * jb, L.tm, out_maps ? (*out_maps)[k] : L.tm,
                        static_cast<const uint8_t*>(P.A) + (size_t)slot * ra * P.in * 2,
                        static_cast<const uint8_t*>(P.B) + (size_t)slot * P.out * ra * 2, L.out, L.in, ra, scale, t,
                        L.w, elem))
      return false;
    t += merge_job_tiles(host + k * jb);
    elem += (long long)L.out * L.in;
  }
  // pageable source: the runtime stages it before returning, so `store` may die right after
  cudaMemcpyAsync(c->mjobs, host, lins.size() * jb, cudaMemcpyHostToDevice, s);
  *tiles = t;
  return true;
}
}  // namespace

extern "C" int lora_merge(dit_ctx* c, int32_t adapter_id, void* merged, size_t bytes, void* stream) {
  if (!c) return DIT_EINVAL;
  auto it = c->adapter_slot.find(adapter_id);
  if (it == c->adapter_slot.end()) return c->fail(DIT_ENOENT, "adapter %d not registered", adapter_id);
  if (c->merged_adapter >= 0) return c->fail(DIT_EEXIST, "adapter %d is already merged", c->merged_adapter);
  if (!c->weights_ready) return c->fail(DIT_ENOWEIGHTS, "base weights not (fully) loaded");
  if (!merged || (reinterpret_cast<uintptr_t>(merged) & 255)) return c->fail(DIT_EINVAL, "merged buffer must be 256-byte aligned");
  const size_t need = dit_merge_bytes(&c->cfg);
  if (bytes < need) return c->fail(DIT_ENOMEM, "merged buffer %zu bytes < %zu", bytes, need);
  const int slot = it->second;
  const float scale = c->slot_scale_h[slot];
  const int ra = c->r_alloc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto lins = adapted_lins(c);
  // a previous merged copy in `merged` may still be read by an in-flight step; the adapter's pool
  // copy may still be in flight on its registration stream
  cudaStreamWaitEvent(s, c->merged_last_use, 0);
  cudaStreamWaitEvent(s, c->slot_ready[slot], 0);
  // validate everything before enqueuing anything
  std::vector<CUtensorMap> maps(lins.size());
  size_t off = 0;
  std::vector<size_t> offs(lins.size());
  for (size_t k = 0; k < lins.size(); ++k) {
    const Lin& L = *lins[k].first;
    offs[k] = off;
    if (!make_tmap_2d(&maps[k], static_cast<uint8_t*>(merged) + off, L.in, L.out, (uint64_t)L.in * 2, 64, 128))
      return c->fail(DIT_EINVAL, "tensor map for the merged copy failed");
    off = align_up(off + (size_t)L.out * L.in * 2, 256);
  }
  // tensor-core merge (merge_tc.cu); DIT_MERGE_MMA_SYNC=1 selects the mma.sync kernel (comparison)
  const char* legacy = getenv("DIT_MERGE_MMA_SYNC");
  const bool use_tc = !(legacy && legacy[0] == '1') && (ra == 64 || ra == 128);
  if (use_tc) {   // one job per adapted linear, one persistent launch
    int tiles = 0;
    if (!upload_merge_jobs(c, slot, &maps, s, &tiles)) return c->fail(DIT_EINVAL, "tensor map for the merge operands failed");
    cudaError_t e = lora_merge_tc_launch(c->mjobs, (int)lins.size(), tiles, ra, c->num_sms, s);
    if (e != cudaSuccess) return c->fail(DIT_ECUDA, "lora_merge kernel: %s", cudaGetErrorString(e));
  } else {
    for (size_t k = 0; k < lins.size(); ++k) {
      Lin& L = *lins[k].first;
      const LoraPool& P = c->pools[lins[k].second];
      cudaError_t e = lora_merge_launch(L.w, static_cast<const uint8_t*>(P.A) + (size_t)slot * ra * P.in * 2,
                                        static_cast<const uint8_t*>(P.B) + (size_t)slot * P.out * ra * 2,
                                        static_cast<uint8_t*>(merged) + offs[k], L.out, L.in, ra, scale, s);
      if (e != cudaSuccess) return c->fail(DIT_ECUDA, "lora_merge kernel: %s", cudaGetErrorString(e));
    }
  }
  for (size_t k = 0; k < lins.size(); ++k) {
    lins[k].first->tm_m = maps[k];
    lins[k].first->has_m = true;
  }
  cudaStreamWaitEvent(s, c->slot_last_use[slot], 0);   // keep slot_last_use covering earlier steps too
  cudaEventRecord(c->slot_last_use[slot], s);
  cudaEventRecord(c->merge_ready, s);                    // the next dit_step waits on this (its stream)
  c->merged_adapter = adapter_id;
  c->plan_B = -1;
  return DIT_OK;
}

extern "C" int lora_merge_inplace(dit_ctx* c, int32_t adapter_id, void* undo, size_t undo_bytes,
                                  uint64_t* undo_entries, void* stream) {
  if (!c) return DIT_EINVAL;
  auto it = c->adapter_slot.find(adapter_id);
  if (it == c->adapter_slot.end()) return c->fail(DIT_ENOENT, "adapter %d not registered", adapter_id);
  if (c->merged_adapter >= 0) return c->fail(DIT_EEXIST, "adapter %d is already merged", c->merged_adapter);
  if (!c->weights_ready) return c->fail(DIT_ENOWEIGHTS, "base weights not (fully) loaded");
  if ((undo_bytes > 0 && !undo) || (reinterpret_cast<uintptr_t>(undo) & 7))
    return c->fail(DIT_EINVAL, "undo log must be an 8-byte aligned device buffer");
  const int ra = c->r_alloc;
  if (ra != 64 && ra != 128) return c->fail(DIT_EINVAL, "in-place merge needs r_alloc 64 or 128");
  const int slot = it->second;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // every step enqueued so far reads the base weights; the adapter's copies may still be in flight
  cudaStreamWaitEvent(s, c->step_done, 0);
  cudaStreamWaitEvent(s, c->slot_ready[slot], 0);
  int tiles = 0;
  if (!upload_merge_jobs(c, slot, nullptr, s, &tiles)) return c->fail(DIT_EINVAL, "tensor map for the merge operands failed");
  const int nj = (int)adapted_lins(c).size();
  // pass 1: count the elements the inverse cannot recover (nothing is written)
  cudaMemsetAsync(c->mcount, 0, 8, s);
  cudaError_t e = lora_merge_tc_launch(c->mjobs, nj, tiles, ra, c->num_sms, s, 1, nullptr, c->mcount);
  if (e != cudaSuccess) return c->fail(DIT_ECUDA, "merge count kernel: %s", cudaGetErrorString(e));
  unsigned long long need = 0;
  if (cudaMemcpyAsync(&need, c->mcount, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return c->fail(DIT_ECUDA, "merge count readback failed");
  if (undo_entries) *undo_entries = need;
  if (need * 8 > undo_bytes)
    return c->fail(DIT_ENOMEM, "undo log needs %llu entries (%llu bytes), got %zu bytes; weights untouched", need,
                   need * 8, undo_bytes);
  // pass 2: W' over W, the unrecoverable elements logged
  cudaMemsetAsync(c->mcount, 0, 8, s);
  e = lora_merge_tc_launch(c->mjobs, nj, tiles, ra, c->num_sms, s, 2, static_cast<unsigned long long*>(undo), c->mcount);
  if (e != cudaSuccess) return c->fail(DIT_ECUDA, "in-place merge kernel: %s", cudaGetErrorString(e));
  cudaStreamWaitEvent(s, c->slot_last_use[slot], 0);
  cudaEventRecord(c->slot_last_use[slot], s);
  cudaEventRecord(c->merge_ready, s);
  c->merged_adapter = adapter_id;
  c->merged_inplace = true;
  c->inplace_log = static_cast<unsigned long long*>(undo);
  c->inplace_entries = need;
  c->inplace_tiles = tiles;
  c->inplace_njobs = nj;
  c->plan_B = -1;
  return DIT_OK;
}

extern "C" int lora_unmerge(dit_ctx* c) {
  if (!c) return DIT_EINVAL;
  if (c->merged_adapter < 0) return c->fail(DIT_ENOENT, "no adapter is merged");
  // the caller may free / reuse the merged buffer after this returns: wait for its last reader
  if (cudaEventSynchronize(c->merged_last_use) != cudaSuccess) return c->fail(DIT_ECUDA, "merged copy still in use");
  if (c->merged_inplace) {   // W = bf16(W' - s B A) everywhere, then the logged elements exactly
    cudaStream_t s = nullptr;   // (legacy default stream; synchronised below)
    cudaError_t e = lora_merge_tc_launch(c->mjobs, c->inplace_njobs, c->inplace_tiles, c->r_alloc, c->num_sms, s, 3,
                                         nullptr, nullptr);
    if (e == cudaSuccess) e = restore_log_launch(c->mjobs, c->inplace_njobs, c->inplace_log, c->inplace_entries, c->num_sms, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return c->fail(DIT_ECUDA, "restore: %s", cudaGetErrorString(e));
    c->merged_inplace = false;
    c->inplace_log = nullptr;
    c->inplace_entries = 0;
  }
  for (auto& lm : adapted_lins(c)) lm.first->has_m = false;   // copy mode: base weights never written
  c->merged_adapter = -1;
  c->plan_B = -1;
  return DIT_OK;
}

// ------------------------------------------------------------------ ControlNet
extern "C" int controlnet_inject(dit_ctx* c, int32_t slot, int32_t block, const void* residual, float scale,
                                 void* ready) {
  if (!c) return DIT_EINVAL;
  if (slot < 0 || slot >= c->cfg.max_batch) return c->fail(DIT_EINVAL, "slot %d not in [0, %d)", slot, c->cfg.max_batch);
  if (block < 0 || block >= c->Ld + c->Ls)
    return c->fail(DIT_EINVAL, "block %d not in [0, %d) (double blocks, then single blocks)", block, c->Ld + c->Ls);
  if (!residual || (reinterpret_cast<uintptr_t>(residual) & 15))
    return c->fail(DIT_EINVAL, "residual must be a non-NULL 16-byte aligned device pointer");
  if (!std::isfinite(scale)) return c->fail(DIT_EINVAL, "scale must be finite");
  auto& lst = c->cn[{slot, block}];
  if ((int)lst.size() >= CN_FANIN)
    return c->fail(DIT_ENOSPC, "request %d block %d already has %d ControlNet residuals (fan-in limit)", slot, block, CN_FANIN);
  lst.push_back({residual, scale, reinterpret_cast<cudaEvent_t>(ready), nullptr, 0});
  return DIT_OK;
}

extern "C" int controlnet_inject_flag(dit_ctx* c, int32_t slot, int32_t block, const void* residual, float scale,
                                      const uint32_t* flag, uint32_t expect) {
  if (!c) return DIT_EINVAL;
  if (!flag || (reinterpret_cast<uintptr_t>(flag) & 3)) return c->fail(DIT_EINVAL, "flag must be a 4-byte aligned device pointer");
  const int r = controlnet_inject(c, slot, block, residual, scale, nullptr);
  if (r != DIT_OK) return r;
  auto& e = c->cn[{slot, block}].back();
  e.flag = flag;
  e.expect = expect;
  return DIT_OK;
}

extern "C" int controlnet_clear(dit_ctx* c) {
  if (!c) return DIT_EINVAL;
  c->cn.clear();
  return DIT_OK;
}

namespace {
void CUDART_CB host_delay_cb(void* arg) {
  const uint64_t ns = reinterpret_cast<uint64_t>(arg);
  struct timespec ts;
  ts.tv_sec = (time_t)(ns / 1000000000ull);
  ts.tv_nsec = (long)(ns % 1000000000ull);
  nanosleep(&ts, nullptr);
}
}  // namespace

extern "C" int dit_debug_host_delay(void* stream, uint64_t delay_ns) {
  return cudaLaunchHostFunc(reinterpret_cast<cudaStream_t>(stream), host_delay_cb,
                            reinterpret_cast<void*>(delay_ns)) == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

extern "C" int dit_debug_delayed_publish(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                                         uint64_t delay_ns, void* stream) {
  return delayed_publish_launch(dst, src, bytes, flag, value, delay_ns, reinterpret_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? DIT_OK : DIT_ECUDA;
}

// ------------------------------------------------------------------ SP
// the workspace's SP capacity (dit_config.max_sp_world): 1 = no exchange buffers, n > 1 = at most n ranks
static int sp_world_ok(dit_ctx* c, int world) {
  const int cap = c->cfg.max_sp_world;
  if (cap == 1 && world > 1)
    return c->fail(DIT_EPARALLEL, "workspace sized for one GPU (max_sp_world = 1): no sequence parallelism");
  if (cap > 1 && world > cap) return c->fail(DIT_EPARALLEL, "world %d > max_sp_world %d", world, cap);
  return DIT_OK;
}

extern "C" void* dit_local_group_create(int32_t world) {
  if (world < 1 || world > 64) return nullptr;
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->send.assign(world, nullptr);
  g->qkv.assign(world, nullptr);
  g->o.assign(world, nullptr);
  g->cat.assign(world, nullptr);
  g->vcfg.assign(world, nullptr);
  g->flags.assign(world, nullptr);
  g->ready.assign(world, nullptr);
  g->done.assign(world, nullptr);
  for (int r = 0; r < world; ++r) {
    cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming);
  }
  return g;
}

extern "C" void dit_local_group_destroy(void* grp) {
  LocalGroup* g = static_cast<LocalGroup*>(grp);
  if (!g) return;
  for (auto e : g->ready) cudaEventDestroy(e);
  for (auto e : g->done) cudaEventDestroy(e);
  delete g;
}

extern "C" int sp_init_local(dit_ctx* c, void* grp, int32_t rank) {
  if (!c) return DIT_EINVAL;
  LocalGroup* g = static_cast<LocalGroup*>(grp);
  if (!g || rank < 0 || rank >= g->world) return c->fail(DIT_EINVAL, "bad local group / rank");
  if (int e = sp_world_ok(c, g->world)) return e;
  if (c->H % g->world) return c->fail(DIT_EPARALLEL, "world %d does not divide heads %d", g->world, c->H);
  if (c->lp_world > 1) return c->fail(DIT_EPARALLEL, "latent parallelism is active (lp_init)");
  const char* nccl_path = getenv("DIT_SP_NCCL");
  // the fused exchange's peer tables and flag words are sized for 8 ranks (PeerFlags, qkv_peer,
  // out_peer); larger in-process groups use the all-to-all path
  c->sp_fused = g->world > 1 && g->world <= 8 && !(nccl_path && nccl_path[0] == '1');
  if (c->sp_fused) {   // peers resolve at the first dit_step, once every rank has registered
    cudaMemset(c->flags, 0, 8 * 4);
    cudaDeviceSynchronize();
    g->qkv[rank] = c->qkv;
    g->o[rank] = c->o;
    g->cat[rank] = c->cat;
    g->flags[rank] = c->flags;
    c->peers_ready = false;
    c->sp_epoch = 0;
  }
  c->local_group = g;
  c->world = g->world;
  c->rank = rank;
  c->plan_B = -1;
  c->rope_key[0] = -1;
  return DIT_OK;
}

// Peer handle of a context: the CUDA IPC handle of its workspace + the workspace size.  One
// handle per rank suffices: the carve-out layout is identical on every rank (same dit_config),
// so a peer's qkv / o / cat / vcfg / flags sit at my offsets from its base.
constexpr int PEER_HANDLE = DIT_IPC_HANDLE_BYTES + 8;
static_assert(PEER_HANDLE == DIT_PEER_HANDLE_BYTES, "peer handle layout");

extern "C" int dit_peer_handle(dit_ctx* c, void* out) {
  if (!c || !out) return DIT_EINVAL;
  if (cudaSetDevice(c->device) != cudaSuccess) return c->fail(DIT_ECUDA, "cudaSetDevice");
  // zero my arrival flags BEFORE the handle leaves this process: no peer can signal before it has
  // every handle, and it has mine only after this call returned
  if (cudaMemset(c->flags, 0, 8 * 4) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return c->fail(DIT_ECUDA, "flag reset failed");
  uint8_t* o = static_cast<uint8_t*>(out);
  if (dit_ipc_export(c->ws, o) != DIT_OK) return c->fail(DIT_ECUDA, "cudaIpcGetMemHandle of the workspace failed");
  const uint64_t wsb = c->ws_bytes;
  memcpy(o + DIT_IPC_HANDLE_BYTES, &wsb, 8);
  return DIT_OK;
}

namespace {
// Map every peer's workspace from the all-gathered handles (P x PEER_HANDLE bytes, rank order).
// base[me] = my own workspace.  Returns false (nothing left open) if any handle is unusable.
bool open_peer_bases(dit_ctx* c, int P, int me, const uint8_t* all, uint8_t** base, std::vector<void*>& opened) {
  opened.clear();
  for (int r = 0; r < P; ++r) {
    uint64_t b = 0;
    memcpy(&b, all + (size_t)r * PEER_HANDLE + DIT_IPC_HANDLE_BYTES, 8);
    if (b != c->ws_bytes) return false;   // an export failed (zeroed) or layouts differ
  }
  for (int r = 0; r < P; ++r) {
    if (r == me) { base[r] = c->ws; continue; }
    void* ptr = nullptr;
    if (dit_ipc_open(all + (size_t)r * PEER_HANDLE, &ptr) != DIT_OK) {
      for (void* x : opened) dit_ipc_close(x);
      opened.clear();
      cudaGetLastError();
      return false;
    }
    opened.push_back(ptr);
    base[r] = static_cast<uint8_t*>(ptr);
  }
  return true;
}

void* at_peer(const dit_ctx* c, uint8_t* const* base, int r, const void* mine_ptr) {
  return static_cast<void*>(base[r] + (static_cast<const uint8_t*>(mine_ptr) - c->ws));
}

void bind_sp_peers(dit_ctx* c, uint8_t* const* base, int P) {
  for (int r = 0; r < P; ++r) {
    c->peer_qkv[r] = at_peer(c, base, r, c->qkv);
    c->peer_o[r] = at_peer(c, base, r, c->o);
    c->peer_cat[r] = at_peer(c, base, r, c->cat);
    c->peer_flags.f[r] = static_cast<uint32_t*>(at_peer(c, base, r, c->flags));
  }
  c->sp_fused = true;
  c->peers_ready = true;
  c->sp_epoch = 0;
}

void bind_lp_peers(dit_ctx* c, uint8_t* const* base) {
  for (int r = 0; r < 2; ++r) {
    c->peer_vcfg[r] = static_cast<float*>(at_peer(c, base, r, c->vcfg));
    c->peer_flags.f[r] = static_cast<uint32_t*>(at_peer(c, base, r, c->flags));
  }
  c->lp_fused = true;
  c->peers_ready = true;
  c->sp_epoch = 0;
  c->lp_steps = 0;
}

void close_opened(dit_ctx* c) {
  for (void* x : c->ipc_opened) dit_ipc_close(x);
  c->ipc_opened.clear();
}

// All-gather every rank's peer handle over an NCCL communicator and map the peers, with a
// consensus all-reduce: every rank mapped every peer, or all ranks report false together.
bool nccl_gather_and_open(dit_ctx* c, ncclComm_t comm, int P, int me, uint8_t** base, std::vector<void*>& opened) {
  std::vector<uint8_t> mine(PEER_HANDLE, 0), all((size_t)P * PEER_HANDLE);
  // the exchange runs even when the export failed (a zeroed handle marks it), so no rank hangs
  if (dit_peer_handle(c, mine.data()) != DIT_OK) std::fill(mine.begin(), mine.end(), 0);
  uint8_t* dev = reinterpret_cast<uint8_t*>(c->sp);
  cudaMemcpy(dev, mine.data(), mine.size(), cudaMemcpyHostToDevice);
  if (ncclAllGather(dev, dev + 4096, PEER_HANDLE, ncclUint8, comm, 0) != ncclSuccess) return false;
  if (cudaStreamSynchronize(0) != cudaSuccess) return false;
  cudaMemcpy(all.data(), dev + 4096, all.size(), cudaMemcpyDeviceToHost);
  int ok_open = open_peer_bases(c, P, me, all.data(), base, opened) ? 1 : 0;
  int* dflag = reinterpret_cast<int*>(dev + 8192);
  cudaMemcpy(dflag, &ok_open, 4, cudaMemcpyHostToDevice);
  if (ncclAllReduce(dflag, dflag, 1, ncclInt32, ncclMin, comm, 0) != ncclSuccess) ok_open = 0;
  cudaStreamSynchronize(0);
  int all_ok = 0;
  cudaMemcpy(&all_ok, dflag, 4, cudaMemcpyDeviceToHost);
  if (!ok_open || !all_ok) {
    for (void* x : opened) dit_ipc_close(x);
    opened.clear();
    cudaGetLastError();
    return false;
  }
  return true;
}
}  // namespace

// Fused exchange setup over NCCL: map the peers' workspaces through the new communicator.  Any
// failure leaves sp_fused off (the NCCL all-to-all path then runs) -- a capability check.
static void setup_fused_peers(dit_ctx* c) {
  uint8_t* base[8] = {};
  std::vector<void*> opened;
  if (!nccl_gather_and_open(c, c->comm, c->world, c->rank, base, opened)) return;
  close_opened(c);
  c->ipc_opened = opened;
  bind_sp_peers(c, base, c->world);
}

extern "C" int sp_init(dit_ctx* c, int32_t world, int32_t rank, const void* uid) {
  if (!c) return DIT_EINVAL;
  if (world < 1 || rank < 0 || rank >= world) return c->fail(DIT_EINVAL, "bad world/rank %d/%d", world, rank);
  if (int e = sp_world_ok(c, world)) return e;
  if (world == 1 && c->cfg.max_sp_world == 1 && getenv("DIT_FORCE_SP") && uid != nullptr)
    return c->fail(DIT_EPARALLEL, "DIT_FORCE_SP needs the SP buffers (max_sp_world != 1)");
  if (c->H % world) return c->fail(DIT_EPARALLEL, "world %d does not divide heads %d", world, c->H);
  if (c->lp_world > 1 && world > 1) return c->fail(DIT_EPARALLEL, "latent parallelism is active (lp_init)");
  // DIT_FORCE_SP=1 (test-only): a 1-rank NCCL communicator drives the full
  // sequence-parallel data path (all-to-alls + gather/scatter) at world == 1.
  const char* force = getenv("DIT_FORCE_SP");
  c->force_sp = force && force[0] == '1' && uid != nullptr;
  if (world == 1 && !c->force_sp) {
    c->world = 1;
    c->rank = 0;
    c->local_group = nullptr;
    c->rope_key[0] = -1;
    return DIT_OK;
  }
  if (!uid) return c->fail(DIT_EINVAL, "nccl unique id is NULL");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  cudaSetDevice(c->device);
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return c->fail(DIT_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  if (c->comm) ncclCommDestroy(c->comm);
  c->comm = comm;
  c->local_group = nullptr;
  c->world = world;
  c->rank = rank;
  c->plan_B = -1;
  c->rope_key[0] = -1;
  c->sp_fused = false;
  const char* nccl_path = getenv("DIT_SP_NCCL");
  if (world > 1 && world <= 8 && !(nccl_path && nccl_path[0] == '1')) setup_fused_peers(c);
  return DIT_OK;
}

extern "C" int sp_init_peers(dit_ctx* c, int32_t world, int32_t rank, const void* handles) {
  if (!c) return DIT_EINVAL;
  if (world < 2 || world > 8 || rank < 0 || rank >= world)
    return c->fail(DIT_EINVAL, "sp_init_peers: world must be in [2, 8] and rank in [0, world), got %d/%d", world, rank);
  if (!handles) return c->fail(DIT_EINVAL, "handles is NULL");
  if (int e = sp_world_ok(c, world)) return e;
  if (c->H % world) return c->fail(DIT_EPARALLEL, "world %d does not divide heads %d", world, c->H);
  if (c->lp_world > 1) return c->fail(DIT_EPARALLEL, "latent parallelism is active (lp_init)");
  if (cudaSetDevice(c->device) != cudaSuccess) return c->fail(DIT_ECUDA, "cudaSetDevice");
  uint8_t* base[8] = {};
  std::vector<void*> opened;
  if (!open_peer_bases(c, world, rank, static_cast<const uint8_t*>(handles), base, opened))
    return c->fail(DIT_ECUDA, "a peer workspace could not be mapped (cudaIpcOpenMemHandle / size mismatch)");
  close_opened(c);
  c->ipc_opened = opened;
  if (c->comm) ncclCommDestroy(c->comm);
  c->comm = nullptr;
  c->local_group = nullptr;
  c->force_sp = false;
  c->world = world;
  c->rank = rank;
  c->plan_B = -1;
  c->rope_key[0] = -1;
  bind_sp_peers(c, base, world);
  return DIT_OK;
}

// ------------------------------------------------------------------ ControlNet producer side (f2)
extern "C" int controlnet_push(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                               void* stream) {
  if (!dst || !src || !flag || bytes % 16 || (reinterpret_cast<uintptr_t>(dst) & 15) ||
      (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(flag) & 3))
    return DIT_EINVAL;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return controlnet_push_launch(dst, src, bytes, flag, value, sms, reinterpret_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? DIT_OK
             : DIT_ECUDA;
}

namespace {
struct IpcHandle {
  cudaIpcMemHandle_t h;   // 64 bytes
  uint64_t offset;        // dev_ptr - allocation base
};
static_assert(sizeof(IpcHandle) == DIT_IPC_HANDLE_BYTES, "ipc handle layout");
// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda link)
CUresult mem_range(CUdeviceptr* base, size_t* size, CUdeviceptr p) {
  typedef CUresult (*Fn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return CUDA_ERROR_NOT_FOUND;
    fn = reinterpret_cast<Fn>(f);
  }
  return fn(base, size, p);
}
}  // namespace

extern "C" int dit_ipc_export(const void* dev_ptr, void* out) {
  if (!dev_ptr || !out) return DIT_EINVAL;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (mem_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return DIT_EINVAL;
  IpcHandle ih;
  memset(&ih, 0, sizeof(ih));
  if (cudaIpcGetMemHandle(&ih.h, reinterpret_cast<void*>(base)) != cudaSuccess) return DIT_ECUDA;
  ih.offset = reinterpret_cast<CUdeviceptr>(dev_ptr) - base;
  memcpy(out, &ih, sizeof(ih));
  return DIT_OK;
}

extern "C" int dit_ipc_open(const void* handle, void** out) {
  if (!handle || !out) return DIT_EINVAL;
  IpcHandle ih;
  memcpy(&ih, handle, sizeof(ih));
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, ih.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return DIT_ECUDA;
  *out = static_cast<uint8_t*>(base) + ih.offset;
  return DIT_OK;
}

extern "C" int dit_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return DIT_EINVAL;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (mem_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) return DIT_EINVAL;
  return cudaIpcCloseMemHandle(reinterpret_cast<void*>(base)) == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

// ------------------------------------------------------------------ latent parallelism
extern "C" int lp_init(dit_ctx* c, int32_t world, int32_t rank, const void* uid) {
  if (!c) return DIT_EINVAL;
  if (world != 2) return c->fail(DIT_EPARALLEL, "latent parallelism splits the 2 CFG branches: world must be 2, got %d", world);
  if (rank < 0 || rank >= world) return c->fail(DIT_EINVAL, "bad rank %d", rank);
  if (c->world > 1 || c->force_sp) return c->fail(DIT_EPARALLEL, "sequence parallelism is active (sp_init)");
  if (!uid) return c->fail(DIT_EINVAL, "nccl unique id is NULL");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  cudaSetDevice(c->device);
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return c->fail(DIT_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  if (c->lp_comm) ncclCommDestroy(c->lp_comm);
  c->lp_comm = comm;
  c->lp_group = nullptr;
  c->lp_world = world;
  c->lp_rank = rank;
  c->lp_fused = false;
  c->plan_B = -1;
  // fused v exchange: the final GEMM epilogue stores this branch's v into the peer's buffer as
  // well (peer-mapped through CUDA IPC); else ncclAllGather (DIT_SP_NCCL=1 forces it)
  const char* nccl_path = getenv("DIT_SP_NCCL");
  if (!(nccl_path && nccl_path[0] == '1')) {
    uint8_t* base[8] = {};
    std::vector<void*> opened;
    if (nccl_gather_and_open(c, comm, 2, rank, base, opened)) {
      close_opened(c);
      c->ipc_opened = opened;
      bind_lp_peers(c, base);
    }
  }
  return DIT_OK;
}

extern "C" int lp_init_peers(dit_ctx* c, int32_t world, int32_t rank, const void* handles) {
  if (!c) return DIT_EINVAL;
  if (world != 2) return c->fail(DIT_EPARALLEL, "latent parallelism splits the 2 CFG branches: world must be 2, got %d", world);
  if (rank < 0 || rank >= world) return c->fail(DIT_EINVAL, "bad rank %d", rank);
  if (!handles) return c->fail(DIT_EINVAL, "handles is NULL");
  if (c->world > 1 || c->force_sp) return c->fail(DIT_EPARALLEL, "sequence parallelism is active (sp_init)");
  if (cudaSetDevice(c->device) != cudaSuccess) return c->fail(DIT_ECUDA, "cudaSetDevice");
  uint8_t* base[8] = {};
  std::vector<void*> opened;
  if (!open_peer_bases(c, 2, rank, static_cast<const uint8_t*>(handles), base, opened))
    return c->fail(DIT_ECUDA, "the peer workspace could not be mapped (cudaIpcOpenMemHandle / size mismatch)");
  close_opened(c);
  c->ipc_opened = opened;
  if (c->lp_comm) ncclCommDestroy(c->lp_comm);
  c->lp_comm = nullptr;
  c->lp_group = nullptr;
  c->lp_world = 2;
  c->lp_rank = rank;
  c->plan_B = -1;
  bind_lp_peers(c, base);
  return DIT_OK;
}

extern "C" int lp_init_local(dit_ctx* c, void* grp, int32_t rank) {
  if (!c) return DIT_EINVAL;
  LocalGroup* g = static_cast<LocalGroup*>(grp);
  if (!g || g->world != 2 || rank < 0 || rank >= 2) return c->fail(DIT_EPARALLEL, "latent parallelism needs a 2-rank group");
  if (c->world > 1 || c->force_sp) return c->fail(DIT_EPARALLEL, "sequence parallelism is active (sp_init)");
  c->lp_group = g;
  c->lp_world = 2;
  c->lp_rank = rank;
  // fused v exchange over the group's (same-process) pointers unless DIT_SP_NCCL=1; the peer
  // resolves at the first dit_step, once both ranks have registered
  const char* nccl_path = getenv("DIT_SP_NCCL");
  c->lp_fused = !(nccl_path && nccl_path[0] == '1');
  c->peers_ready = false;
  if (c->lp_fused) {
    cudaMemset(c->flags, 0, 8 * 4);
    cudaDeviceSynchronize();
    g->vcfg[rank] = c->vcfg;
    g->flags[rank] = c->flags;
    c->sp_epoch = 0;
    c->lp_steps = 0;
  }
  c->plan_B = -1;
  return DIT_OK;
}

// ------------------------------------------------------------------ plan
namespace {

int build_rowspace(dit_ctx* c, RowSpace& R, int M, int rows_per_req, const std::vector<int>& req_slot,
                   std::vector<int>& h_tiles, std::vector<int>& h_cnt, std::vector<int2>& h_shrink) {
  R.M = M;
  R.rows_per_req = rows_per_req;
  R.tiles_m = (M + GEMM_TM - 1) / GEMM_TM;
  R.h_row_slot.assign(M, -1);
  for (int r = 0; r < M; ++r) R.h_row_slot[r] = req_slot[r / rows_per_req];
  h_tiles.assign((size_t)R.tiles_m * c->slot_cap, 0);
  h_cnt.assign(R.tiles_m, 0);
  h_shrink.clear();
  for (int m = 0; m < R.tiles_m; ++m) {
    std::vector<int> sl;
    for (int r = m * GEMM_TM; r < std::min(M, (m + 1) * GEMM_TM); ++r) {
      int s = R.h_row_slot[r];
      if (s >= 0 && std::find(sl.begin(), sl.end(), s) == sl.end()) sl.push_back(s);
    }
    std::sort(sl.begin(), sl.end());
    if ((int)sl.size() > c->slot_cap) return -1;
    h_cnt[m] = (int)sl.size();
    for (size_t i = 0; i < sl.size(); ++i) {
      h_tiles[(size_t)m * c->slot_cap + i] = sl[i];
      h_shrink.push_back(make_int2(m, sl[i]));
    }
  }
  R.n_shrink = (int)h_shrink.size();
  R.rank_rows = 0;
  for (int r = 0; r < M; ++r)
    if (R.h_row_slot[r] >= 0) R.rank_rows += c->slot_rank_h[R.h_row_slot[r]];
  return 0;
}

}  // namespace

// ------------------------------------------------------------------ GEMM helpers
namespace {

cudaEvent_t prof_event(dit_ctx* c) {
  if (c->ev_next == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_next++];
}
// NVTX ranges (nsys timelines): one per dit_step, per block and per launch, named
// by the profiling kind.  Header-only NVTX v3: without an attached tool a push / pop is a few ns.
// DIT_NVTX=0 turns them off.
bool nvtx_on() {
  static const bool on = [] {
    const char* e = getenv("DIT_NVTX");
    return !(e && e[0] == '0');
  }();
  return on;
}
const char* kind_name(int kind) {
  static const char* const names[19] = {"gemm",        "attention",   "lnmod",       "modulation", "other",
                                        "sp_exchange", "sp_layout",   "",            "",           "",
                                        "gemm:embed",  "gemm:dbl_qkv", "gemm:dbl_proj", "gemm:dbl_fc1", "gemm:dbl_fc2",
                                        "gemm:sgl_linear1", "gemm:sgl_linear2", "gemm:final", "gemm:lora_shrink"};
  return kind >= 0 && kind < 19 ? names[kind] : "launch";
}
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(nvtx_on()) {
    if (on) nvtxRangePushA(name);
  }
  NvtxRange(const char* fmt, int i) : on(nvtx_on()) {
    if (on) {
      char buf[64];
      snprintf(buf, sizeof(buf), fmt, i);
      nvtxRangePushA(buf);
    }
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

void prof_begin(dit_ctx* c, cudaStream_t s, int kind) {
  if (nvtx_on()) nvtxRangePushA(kind_name(kind));
  if (!c->prof_on) return;
  c->prof_a = prof_event(c);
  cudaEventRecord(c->prof_a, s);
}
void prof_end(dit_ctx* c, cudaStream_t s, int kind, double flops) {
  if (nvtx_on()) nvtxRangePop();
  if (!c->prof_on) return;
  cudaEvent_t b = prof_event(c);
  cudaEventRecord(b, s);
  c->prof.push_back({kind, flops, c->prof_a, b});
}

// Algorithmic FLOPs: 2MNK for the base product; LoRA counts
// 2 r in (shrink) + 2 r out (expand) per adapted row -- padding excluded.
double problem_flops(const dit_ctx* c, const GemmProblem& P) {
  (void)c;
  if (P.shrink) return 2.0 * P.K * P.rank_rows;
  double f = 2.0 * P.M * P.N * (double)P.K;
  if (P.ext_kblocks > 0) f += 2.0 * P.N * P.rank_rows;
  return f;
}

GemmProblem base_problem(dit_ctx* c, const void* A, int M, int K, int lda, const Lin& W, const EpiParams& epi) {
  GemmProblem P;
  memset(&P, 0, sizeof(P));
  make_tmap_2d(&P.tmA, A, K, M, (uint64_t)lda * 2, 64, GEMM_BM);
  P.tmB = (c->merged_adapter >= 0 && W.has_m) ? W.tm_m : W.tm;
  P.M = M;
  P.N = W.out;
  P.K = K;
  P.tiles_m = (M + GEMM_TM - 1) / GEMM_TM;
  P.tiles_n = (P.N + GEMM_BN - 1) / GEMM_BN;
  P.num_tiles = P.tiles_m * P.tiles_n;
  P.epi = epi;
  P.slot_cap = c->slot_cap;
  if (epi.kind == EPI_RESID)   // h [R_max][D] fp32 for the epilogue's TMA reduce-add
    P.tmH_ok = make_tmap_2d_f32(&P.tmH, epi.h, (uint64_t)epi.D, (uint64_t)c->Rmax, (uint64_t)epi.D * 4, 32, 32) ? 1 : 0;
  return P;
}

void add_lora_ext(dit_ctx* c, GemmProblem& P, const RowSpace& R, int module, const void* sext) {
  if (R.n_shrink == 0 || c->pools.empty() || !c->pools[module].A) return;
  const int nslots = std::max(c->cfg.max_adapters, 1);
  make_tmap_2d(&P.tmAx, sext, (uint64_t)nslots * c->r_alloc, P.M, (uint64_t)nslots * c->r_alloc * 2, 64, GEMM_BM);
  P.tmBx = c->pools[module].tmB;
  P.tile_slots = R.tile_slots;
  P.tile_slot_cnt = R.tile_cnt;
  P.ext_kblocks = c->r_alloc / 64;
  P.epi.r_alloc = c->r_alloc;
  P.rank_rows = R.rank_rows;
}

GemmProblem shrink_problem(dit_ctx* c, const void* A, int M, int K, int lda, const RowSpace& R, int module,
                           void* sext) {
  GemmProblem P;
  memset(&P, 0, sizeof(P));
  const LoraPool& L = c->pools[module];
  const int nslots = std::max(c->cfg.max_adapters, 1);
  make_tmap_2d(&P.tmA, A, K, M, (uint64_t)lda * 2, 64, GEMM_BM);
  P.tmB = L.tmA;
  P.M = M;
  P.N = c->r_alloc;
  P.K = K;
  P.tiles_m = (M + GEMM_TM - 1) / GEMM_TM;
  P.tiles_n = 1;
  P.num_tiles = R.n_shrink;
  P.shrink = 1;
  P.shrink_list = R.shrink_list;
  P.rank_rows = R.rank_rows;
  P.epi.kind = EPI_SHRINK;
  P.epi.out = sext;
  P.epi.ld_out = nslots * c->r_alloc;
  P.epi.row_slot = R.row_slot;
  P.epi.slot_scale = c->p_slot_scale;
  P.epi.r_alloc = c->r_alloc;
  P.epi.rows_per_req = R.rows_per_req;
  P.epi.joint_n = 1;
  return P;
}

int run_gemm(dit_ctx* c, GemmProblem* probs, int np, cudaStream_t s, double flops = -1.0) {
  if (flops < 0) {
    flops = 0;
    for (int i = 0; i < np; ++i) flops += problem_flops(c, probs[i]);
  }
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  int t = 0;
  int k = 0;
  for (int i = 0; i < np; ++i) {
    if (probs[i].num_tiles <= 0 || probs[i].M <= 0) continue;
    a.p[k] = probs[i];
    a.p[k].tile_begin = t;
    t += probs[i].num_tiles;
    ++k;
  }
  a.num_problems = k;
  a.total_tiles = t;
  if (t == 0) return DIT_OK;
  prof_begin(c, s, c->gemm_label);
  cudaError_t e = gemm_launch(a, c->num_sms, s);
  prof_end(c, s, c->gemm_label, flops);
  c->launches++;
  if (e != cudaSuccess) return c->fail(DIT_ECUDA, "gemm launch: %s", cudaGetErrorString(e));
  return DIT_OK;
}

// LoRA shrink for up to two (A, rowspace, module) triples, as one launch.
// S_ext of stream problem i lives at sext_of(c, i): the txt stream's rows first,
// then the img stream's (a single-block problem uses the start).
void* sext_of(dit_ctx* c, int stream_rows_before) {
  const int nslots = std::max(c->cfg.max_adapters, 1);
  return c->sext + (size_t)stream_rows_before * nslots * c->r_alloc;
}

int run_shrink(dit_ctx* c, int np, const void* const* A, const int* M, const int* K, const int* lda,
               const RowSpace* const* R, const int* module, const int* row_base, cudaStream_t s) {
  GemmProblem p[2];
  int k = 0;
  for (int i = 0; i < np; ++i)
    if (R[i]->n_shrink > 0 && c->pools[module[i]].A)
      p[k++] = shrink_problem(c, A[i], M[i], K[i], lda[i], *R[i], module[i], sext_of(c, row_base[i]));
  if (k == 0) return DIT_OK;
  c->gemm_label = 18;
  return run_gemm(c, p, k, s);
}

}  // namespace

// ------------------------------------------------------------------ step
extern "C" double dit_step_flops(const dit_ctx* c, const dit_batch* b) {
  if (!c || !b || b->batch < 1) return 0.0;
  // sequences computed on this GPU: CFG doubles the batch unless latent parallelism splits it;
  // a ragged batch counts each request at its own grid (padding is not algorithmic work)
  const int seq = (b->cfg_scale && c->lp_world == 1) ? 2 * b->batch : b->batch;
  const double Nt = b->txt_tokens, D = c->D, F = c->F, C = c->C, Ct = c->Ct;
  const bool sd3 = c->cfg.arch == DIT_ARCH_SD3;
  double f = 0;
  for (int q = 0; q < seq; ++q) {
    const int r = q % b->batch;
    const double Ni = b->img_hw ? (double)b->img_hw[2 * r] * b->img_hw[2 * r + 1] : (double)b->img_h * b->img_w;
    const double N = Ni + Nt;
    // embedders, final
    f += 2 * Ni * D * C + 2 * Nt * D * Ct + 2 * Ni * D * C;
    // double blocks: qkv, proj, fc1, fc2 per stream + attention; SD3's context_pre_only last
    // block has no text proj / MLP
    f += c->Ld * (2 * N * D * (3 * D) + 2 * N * D * D + 2 * 2 * N * D * F + 4 * N * N * D);
    if (sd3) f -= 2 * Nt * D * D + 2 * 2 * Nt * D * F;
    // single blocks
    f += c->Ls * (2 * N * D * (3 * D + F) + 2 * N * (D + F) * D + 4 * N * N * D);
    // LoRA: 2 r (in + out) per row per adapted linear
    const int aid = b->adapter_id ? b->adapter_id[r] : -1;
    if (aid < 0 || c->merged_adapter >= 0) continue;   // merged: the delta is inside the base GEMMs
    auto slot = c->adapter_slot.find(aid);
    if (slot == c->adapter_slot.end()) continue;       // unregistered: dit_step would reject it
    const double rk = c->slot_rank_h[slot->second];    // the adapter's registered rank (padding excluded)
    f += c->Ld * 2 * rk * N * ((D + 3 * D) + (D + D) + (D + F) + (F + D));
    if (sd3) f -= 2 * rk * Nt * ((D + D) + (D + F) + (F + D));
    f += c->Ls * 2 * rk * N * ((D + 3 * D + F) + (D + F + D));
  }
  return f;
}

extern "C" int dit_last_launch_count(const dit_ctx* c) { return c ? c->last_launches : 0; }

extern "C" int dit_sp_exchange(const dit_ctx* c) {
  if (c && c->lp_world > 1) return c->lp_fused ? 2 : 1;
  if (!c || (c->world == 1 && !c->force_sp)) return 0;
  return c->sp_fused ? 2 : 1;
}

#define CK(x)                                                                        \
  do {                                                                               \
    int _r = (x);                                                                    \
    if (_r != DIT_OK) return _r;                                                     \
  } while (0)
#define CKC(x) CKK(x, 4, 0.0)
#define CKK(x, kind, flops)                                                          \
  do {                                                                               \
    prof_begin(c, s, kind);                                                          \
    cudaError_t _e = (x);                                                            \
    prof_end(c, s, kind, flops);                                                     \
    c->launches++;                                                                   \
    if (_e != cudaSuccess) return c->fail(DIT_ECUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
  } while (0)

// mode: STEP_RUN a normal step; STEP_CAPTURE the same enqueue sequence under stream capture (every
// upload forced, staged in the graph's own pinned block; waits on outside events as external
// nodes); STEP_STAGE validation + host tables staged into the graph's block, nothing enqueued
// (dit_graph_launch refreshes the block its graph's copy nodes read, then replays the graph).
enum { STEP_RUN = 0, STEP_CAPTURE = 1, STEP_STAGE = 2 };
static int step_impl(dit_ctx* c, const dit_batch* b, cudaStream_t s, int mode);

extern "C" int dit_step(dit_ctx* c, const dit_batch* b, void* stream) {
  if (!c) return DIT_EINVAL;
  return step_impl(c, b, reinterpret_cast<cudaStream_t>(stream), STEP_RUN);
}

static int step_impl(dit_ctx* c, const dit_batch* b, cudaStream_t s, int mode) {
  NvtxRange nv_step(mode == STEP_CAPTURE ? "dit_step (capture)" : mode == STEP_STAGE ? "dit_step (stage)" : "dit_step");
  // ControlNet registrations apply to exactly one dit_step call: cleared on EVERY exit (a
  // validation error or a failed launch included), so no stale borrowed pointer outlives it
  struct CnClear {
    dit_ctx* c;
    ~CnClear() { c->cn.clear(); }
  } cn_guard{c};
  if (!b) return c->fail(DIT_EINVAL, "batch is NULL");
  if (!c->weights_ready) return c->fail(DIT_ENOWEIGHTS, "base weights not (fully) loaded");
  const int B = b->batch;   // requests
  if (B < 1 || B > c->cfg.max_batch) return c->fail(DIT_EBATCH, "batch %d not in [1, %d]", B, c->cfg.max_batch);
  // classifier-free guidance (reading C22): S sequences run here -- 2B (cond, then uncond)
  // on one GPU, B (this rank's branch) under latent parallelism
  const bool cfgon = b->cfg_scale != nullptr;
  const bool lpar = c->lp_world > 1;   // latent parallelism
  if (lpar && !cfgon) return c->fail(DIT_EINVAL, "latent parallelism (lp_init) needs cfg_scale");
  const int S = (cfgon && !lpar) ? 2 * B : B;
  if (S > c->cfg.max_batch)
    return c->fail(DIT_EBATCH, "CFG doubles the batch: %d sequences > B_max %d", S, c->cfg.max_batch);
  if (cfgon)
    for (int i = 0; i < B; ++i)
      if (!std::isfinite(b->cfg_scale[i])) return c->fail(DIT_EINVAL, "cfg_scale[%d] is not finite", i);
  if (b->img_h < 1 || b->img_w < 1 || b->txt_tokens < 1) return c->fail(DIT_ESHAPE, "empty token grid");
  const int Ni = b->img_h * b->img_w, Nt = b->txt_tokens;
  if (Ni > c->cfg.max_img_tokens || Nt > c->cfg.max_txt_tokens)
    return c->fail(DIT_ESHAPE, "tokens (%d img, %d txt) exceed the configured maxima", Ni, Nt);
  // ragged batch (reading C24): per-request grids inside the padded img_h x img_w slot
  const bool ragged = b->img_hw != nullptr;
  std::vector<int> seq_hw(2 * S), img_valid(S), seq_valid(S);
  for (int q = 0; q < S; ++q) {
    const int r = q % B;
    seq_hw[2 * q] = ragged ? b->img_hw[2 * r] : b->img_h;
    seq_hw[2 * q + 1] = ragged ? b->img_hw[2 * r + 1] : b->img_w;
    const int hq = seq_hw[2 * q], wq = seq_hw[2 * q + 1];
    if (hq < 1 || wq < 1 || (long long)hq * wq > (long long)b->img_h * b->img_w)
      return c->fail(DIT_ESHAPE, "request %d grid %dx%d does not fit the %dx%d slot", r, hq, wq, b->img_h, b->img_w);
    if (c->cfg.arch == DIT_ARCH_SD3 && (hq > c->cfg.pos_embed_max || wq > c->cfg.pos_embed_max))
      return c->fail(DIT_ESHAPE, "request %d grid %dx%d exceeds the %d^2 position table", r, hq, wq,
                     c->cfg.pos_embed_max);
    img_valid[q] = hq * wq;
    seq_valid[q] = b->txt_tokens + hq * wq;
  }
  if (ragged && (c->world > 1 || c->force_sp))
    return c->fail(DIT_EPARALLEL, "ragged batches (img_hw) run without sequence parallelism");
  if (c->cfg.arch == DIT_ARCH_SD3 && (b->img_h > c->cfg.pos_embed_max || b->img_w > c->cfg.pos_embed_max) && !ragged)
    return c->fail(DIT_ESHAPE, "token grid %dx%d exceeds the %d^2 position table", b->img_h, b->img_w,
                   c->cfg.pos_embed_max);
  const int P = c->world;
  if (Ni % P || Nt % P) return c->fail(DIT_EPARALLEL, "world %d does not divide Ni=%d / Nt=%d", P, Ni, Nt);
  if (P > 1 && !c->comm && !c->local_group && !c->peers_ready) return c->fail(DIT_EPARALLEL, "sp_init not called");
  if (!b->adapter_id || !b->sigma || !b->sigma_next || !b->guidance)
    return c->fail(DIT_EINVAL, "host arrays adapter_id/sigma/sigma_next/guidance required");
  if (!b->latents_in || !b->latents_out || !b->txt || !b->pooled) return c->fail(DIT_EINVAL, "NULL device pointer");
  const size_t lat_bytes = (size_t)B * (Ni / P) * c->C * 4;
  {
    const uint8_t* a0 = static_cast<const uint8_t*>((const void*)b->latents_in);
    const uint8_t* b0 = reinterpret_cast<const uint8_t*>(b->latents_out);
    if (a0 < b0 + lat_bytes && b0 < a0 + lat_bytes) return c->fail(DIT_EALIAS, "latents_out aliases latents_in");
  }
  if ((reinterpret_cast<uintptr_t>(b->txt) & 15)) return c->fail(DIT_EINVAL, "txt must be 16-byte aligned");
  if (b->cfg_scale) {   // cfg_euler_kernel moves latents / v as float4
    auto mis16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; };
    if (mis16(b->latents_in) || mis16(b->latents_out) || (b->v_out && mis16(b->v_out)))
      return c->fail(DIT_EINVAL, "with cfg_scale, latents_in / latents_out / v_out must be 16-byte aligned");
  }
  std::vector<int> req_slot(S, -1);   // pool slot of every sequence
  for (int i = 0; i < S; ++i) {
    const int aid = b->adapter_id[i % B];
    if (c->merged_adapter >= 0) {   // patched replica: specialised to its adapter
      if (aid != c->merged_adapter)
        return c->fail(DIT_EADAPTER, "adapter %d is merged; request %d uses %d", c->merged_adapter, i, aid);
      continue;                     // its LoRA is in the weights: no per-step LoRA work
    }
    if (aid < 0) continue;
    auto it = c->adapter_slot.find(aid);
    if (it == c->adapter_slot.end()) return c->fail(DIT_EADAPTER, "request %d uses unregistered adapter %d", i, aid);
    req_slot[i] = it->second;
  }
  for (auto& kv : c->cn)
    if (kv.first.first >= S) return c->fail(DIT_EINVAL, "ControlNet registered for slot %d >= sequences %d", kv.first.first, S);

  if (cudaSetDevice(c->device) != cudaSuccess) return c->fail(DIT_ECUDA, "cudaSetDevice");
  const bool capture = mode == STEP_CAPTURE, stage_only = mode == STEP_STAGE;
  // events recorded outside a capture are waited on as external nodes; ours recorded inside it
  // must stay usable outside the graph (lora_unregister / lora_unmerge wait on them)
  const unsigned wait_fl = capture ? cudaEventWaitExternal : 0;
  auto record = [&](cudaEvent_t e) {
    if (capture) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  };
  if (mode == STEP_RUN) {   // pinned ring block for this step's uploads
    const int i = c->pin_next++ % dit_ctx::PIN_RING;
    cudaEventSynchronize(c->pin_ev[i]);   // its copies of PIN_RING steps ago have run
    c->st_base = c->pin + (size_t)i * c->stage_bytes;
  }
  c->st_off = 0;
  // stage `bytes` from host `src` into the pinned block and (unless staging only) enqueue its copy
  auto UP = [&](void* dst, const void* src, size_t bytes) -> bool {
    if (c->st_off + bytes > c->stage_bytes) return false;
    uint8_t* p = c->st_base + c->st_off;
    memcpy(p, src, bytes);
    c->st_off = align_up(c->st_off + bytes, 16);
    if (!stage_only) cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s);
    return true;
  };
  struct ProfOff {   // no per-launch profiling events inside a graph
    dit_ctx* c;
    bool saved;
    ~ProfOff() { c->prof_on = saved; }
  } prof_guard{c, c->prof_on};
  if (capture) c->prof_on = false;
  if (capture || stage_only) {   // a graph carries every upload (its replays must not rely on caches)
    c->plan_B = -1;
    c->rope_key[0] = -1;
    c->segs_dirty = true;
  }
  {
    cudaError_t pe = cudaGetLastError();
    if (pe != cudaSuccess) return c->fail(DIT_ECUDA, "pending CUDA error: %s", cudaGetErrorString(pe));
  }
  c->launches = 0;
  // asynchronously loaded / patched adapters: order this step after their copies on THIS stream
  {
    std::vector<int> waited;
    for (int i = 0; i < S && !stage_only; ++i)
      if (req_slot[i] >= 0 && std::find(waited.begin(), waited.end(), req_slot[i]) == waited.end()) {
        cudaStreamWaitEvent(s, c->slot_ready[req_slot[i]], wait_fl);
        waited.push_back(req_slot[i]);
      }
    if (c->merged_adapter >= 0 && !stage_only) cudaStreamWaitEvent(s, c->merge_ready, wait_fl);
  }
  const int D = c->D, H = c->H, d = c->d, F = c->F, C = c->C, Ct = c->Ct;
  const int nt = Nt / P, ni = Ni / P, N = nt + ni;
  const int Mt = S * nt, Mi = S * ni, Mj = S * N;

  // ---- plan (cached by shape + adapter slots)
  bool any_lora = false;
  for (int i = 0; i < S; ++i) any_lora |= req_slot[i] >= 0;
  if (c->plan_B != S || c->plan_h != b->img_h || c->plan_w != b->img_w || c->plan_nt != Nt || c->plan_slots != req_slot) {
    std::vector<int> ht, hc;
    std::vector<int2> hs;
    const int Ms[3] = {Mt, Mi, Mj}, rpr[3] = {nt, ni, N};
    for (int r = 0; r < 3; ++r) {
      if (build_rowspace(c, c->rs[r], Ms[r], rpr[r], req_slot, ht, hc, hs) < 0)
        return c->fail(DIT_ESHAPE, "too many distinct adapters in one 128-row tile");
      bool ok = UP(c->rs[r].row_slot, c->rs[r].h_row_slot.data(), Ms[r] * 4);
      ok &= UP(c->rs[r].tile_slots, ht.data(), ht.size() * 4);
      ok &= UP(c->rs[r].tile_cnt, hc.data(), hc.size() * 4);
      if (!hs.empty()) ok &= UP(c->rs[r].shrink_list, hs.data(), hs.size() * 8);
      if (!ok) return c->fail(DIT_ENOMEM, "staging block overflow (plan tables)");
    }
    if (!any_lora)
      for (int r = 0; r < 3; ++r) c->rs[r].n_shrink = 0;
    c->plan_B = S;
    c->plan_h = b->img_h;
    c->plan_w = b->img_w;
    c->plan_nt = Nt;
    c->plan_slots = req_slot;
  }
  // RoPE tables: one shared by every sequence, or one per sequence of a ragged Flux batch
  const bool rope_per_seq = ragged && c->cfg.arch == DIT_ARCH_FLUX;
  const int rope_stride = rope_per_seq ? N * (d / 2) : 0;
  const std::vector<int> hw_key = rope_per_seq ? seq_hw : std::vector<int>();
  if (!stage_only && (c->rope_key[0] != nt || c->rope_key[1] != ni || c->rope_key[2] != b->img_w || c->plan_hw != hw_key)) {
    if (c->cfg.arch == DIT_ARCH_SD3)   // no RoPE: the QKV epilogue rotates by angle 0 (exact identity)
      CKC(rope_table_launch(c->rope, nt, ni, 0, 0, 1, 0, 0, d, 1.f, s));   // theta 1, width 1: angle 0
    else if (rope_per_seq)
      for (int q = 0; q < S; ++q)   // (P = 1) positions from request q's own grid width
        CKC(rope_table_launch(c->rope + (size_t)q * rope_stride, nt, ni, 0, 0, seq_hw[2 * q + 1],
                              c->cfg.rope_axes[0], c->cfg.rope_axes[1], c->cfg.rope_axes[2], c->cfg.rope_theta, s));
    else
      CKC(rope_table_launch(c->rope, nt, ni, c->rank * nt, c->rank * ni, b->img_w, c->cfg.rope_axes[0],
                            c->cfg.rope_axes[1], c->cfg.rope_axes[2], c->cfg.rope_theta, s));
    c->rope_key[0] = nt;
    c->rope_key[1] = ni;
    c->rope_key[2] = b->img_w;
    c->plan_hw = hw_key;
  }
  if (ragged) {
    std::vector<int> iv(2 * MAX_SEQ, 0);
    for (int q = 0; q < S; ++q) {
      iv[q] = img_valid[q];
      iv[MAX_SEQ + q] = seq_valid[q];
    }
    UP(c->p_img_valid, iv.data(), MAX_SEQ * 4);
    UP(c->p_seq_valid, iv.data() + MAX_SEQ, MAX_SEQ * 4);
  }
  // ---- per-step parameter block (staged in pinned memory: the host copies may be reused at once)
  {
    // per SEQUENCE (CFG: sequence q belongs to request q % B), CFG scale per request
    constexpr int M = MAX_SEQ;
    std::vector<float> pf(M * 5 + 64, 0.f);
    for (int q = 0; q < S; ++q) {
      const int i = q % B;
      pf[q] = b->sigma_next[i] - b->sigma[i];
      pf[M + q] = b->cn_scale ? b->cn_scale[i] : 1.f;
      pf[2 * M + q] = b->sigma[i];
      pf[3 * M + q] = b->guidance[i];
    }
    for (int i = 0; i < B && cfgon; ++i) pf[4 * M + i] = b->cfg_scale[i];
    UP(c->p_cfg, pf.data() + 4 * M, M * 4);
    UP(c->p_dsig, pf.data(), M * 4);
    UP(c->p_cn_scale, pf.data() + M, M * 4);
    UP(c->p_sigma, pf.data() + 2 * M, M * 4);
    UP(c->p_guid, pf.data() + 3 * M, M * 4);
    std::vector<float> ss(64, 0.f);
    for (size_t i = 0; i < c->slot_scale_h.size() && i < 64; ++i) ss[i] = c->slot_scale_h[i];
    UP(c->p_slot_scale, ss.data(), 64 * 4);
    c->cn_flags = false;
    if (!c->cn.empty()) {
      // [block][fan-in k][request] tables of the residuals registered for this step
      const size_t ncn = (size_t)(c->Ld + c->Ls) * CN_FANIN * MAX_SEQ;
      std::vector<const void*> cp(ncn, nullptr);
      std::vector<float> kap(ncn, 0.f);
      std::vector<const uint32_t*> fl(ncn, nullptr);
      std::vector<uint32_t> ex(ncn, 0);
      c->cn_flags = false;
      for (auto& kv : c->cn)
        for (size_t k = 0; k < kv.second.size(); ++k) {
          const size_t at = ((size_t)kv.first.second * CN_FANIN + k) * MAX_SEQ + kv.first.first;
          cp[at] = kv.second[k].ptr;
          kap[at] = kv.second[k].scale * (b->cn_scale ? b->cn_scale[kv.first.first % B] : 1.f);
          fl[at] = kv.second[k].flag;
          ex[at] = kv.second[k].expect;
          c->cn_flags |= kv.second[k].flag != nullptr;
        }
      UP(c->p_cn_ptr, cp.data(), cp.size() * sizeof(void*));
      UP(c->p_cn_kappa, kap.data(), kap.size() * 4);
      if (c->cn_flags) {
        UP(c->p_cn_flag, fl.data(), fl.size() * sizeof(void*));
        UP(c->p_cn_expect, ex.data(), ex.size() * 4);
      }
    }
  }
  if (c->segs_dirty) {
    std::vector<SkinnySeg> sg;
    for (int i = 0; i < c->Ld; ++i)
      for (int st = 0; st < 2; ++st) {
        const Lin& L = c->dbl[st][i].mod;
        sg.push_back({L.w, L.b, L.out, (i * 2 + st) * 6 * D});
      }
    for (int j = 0; j < c->Ls; ++j) sg.push_back({c->sgl[j].mod.w, c->sgl[j].mod.b, c->sgl[j].mod.out, 12 * D * c->Ld + j * 3 * D});
    sg.push_back({c->fin_mod.w, c->fin_mod.b, c->fin_mod.out, 12 * D * c->Ld + 3 * D * c->Ls});
    c->nsegs = (int)sg.size();
    c->seg_rows = 0;
    for (auto& x : sg) c->seg_rows += x.rows;
    // tail: conditioning MLPs (time in/out, guidance in/out, vector in/out)
    sg.push_back({c->t_in.w, c->t_in.b, D, 0});
    sg.push_back({c->t_out.w, c->t_out.b, D, 0});
    sg.push_back({c->g_in.w, c->g_in.b, D, 0});
    sg.push_back({c->g_out.w, c->g_out.b, D, 0});
    sg.push_back({c->y_in.w, c->y_in.b, D, 0});
    sg.push_back({c->y_out.w, c->y_out.b, D, 0});
    if (!UP(c->segs, sg.data(), sg.size() * sizeof(SkinnySeg))) return c->fail(DIT_ENOMEM, "staging block overflow");
    c->segs_dirty = false;
  }
  if (mode == STEP_RUN) cudaEventRecord(c->pin_ev[(c->pin_next - 1) % dit_ctx::PIN_RING], s);
  if (capture && c->st_event) record(c->st_event);   // the graph's block may be restaged after this
  if (stage_only) return DIT_OK;   // dit_graph_launch: the block its graph reads is refreshed
  const int mod_off_single = 12 * D * c->Ld;
  const int mod_off_final = mod_off_single + 3 * D * c->Ls;

  // ---- conditioning vec (tail segments nsegs+0..5) and all modulations (one launch)
  SkinnySeg* cs = c->segs + c->nsegs;
  CKC(temb_launch(c->p_sigma, S, c->temb, s));
  CKC(skinny_launch(c->temb, 256, cs + 0, 1, D, c->h1, D, S, 0, s));
  CKC(prep_x_launch(c->h1, S, D, 1, c->xprep, s));
  CKC(skinny_launch(c->xprep, D, cs + 1, 1, D, c->vec, D, S, 0, s));
  if (c->cfg.guidance_embed) {
    CKC(temb_launch(c->p_guid, S, c->temb, s));
    CKC(skinny_launch(c->temb, 256, cs + 2, 1, D, c->h1, D, S, 0, s));
    CKC(prep_x_launch(c->h1, S, D, 1, c->xprep, s));
    CKC(skinny_launch(c->xprep, D, cs + 3, 1, D, c->vec, D, S, 1, s));
  }
  cudaMemsetAsync(c->xprep, 0, (size_t)MAX_SEQ * c->Cp * 2, s);
  cudaMemcpyAsync(c->xprep, b->pooled, (size_t)S * c->Cp * 2, cudaMemcpyDeviceToDevice, s);
  CKC(skinny_launch(c->xprep, c->Cp, cs + 4, 1, D, c->h1, D, S, 0, s));
  CKC(prep_x_launch(c->h1, S, D, 1, c->xprep, s));
  CKC(skinny_launch(c->xprep, D, cs + 5, 1, D, c->vec, D, S, 1, s));
  CKC(prep_x_launch(c->vec, S, D, 1, c->xprep, s));
  CKK(skinny_launch(c->xprep, D, c->segs, c->nsegs, c->seg_rows, c->mod, c->mod_total, S, 0, s), 3,
      2.0 * S * (double)c->seg_rows * D);

  // ---- embeddings into the fp32 residual stream h [S][N][D] (txt rows first)
  if (ragged)   // padding rows of the latents become exact zeros (every padded row stays finite)
    CKC(cast_latents_ragged_launch(b->latents_in, c->xb, B, ni, C, c->p_img_valid, s));
  else
    CKC(cast_bf16_launch(b->latents_in, c->xb, (int64_t)B * ni * C, s));
  if (S > B)   // CFG on one GPU: both branches denoise the same latents
    cudaMemcpyAsync(c->xb + (size_t)B * ni * C, c->xb, (size_t)B * ni * C * 2, cudaMemcpyDeviceToDevice, s);
  {
    EpiParams ei;
    memset(&ei, 0, sizeof(ei));
    ei.kind = EPI_STORE_H;
    ei.h = c->h;
    ei.D = D;
    ei.joint_n = N;
    EpiParams et = ei;
    ei.bias = c->img_in.b;
    ei.rows_per_req = ni;
    ei.joint_off = nt;
    et.bias = c->txt_in.b;
    et.rows_per_req = nt;
    et.joint_off = 0;
    GemmProblem p[2] = {base_problem(c, c->xb, Mi, C, C, c->img_in, ei),
                        base_problem(c, b->txt, Mt, Ct, Ct, c->txt_in, et)};
    c->gemm_label = 10;
    CK(run_gemm(c, p, 2, s));
  }
  if (c->cfg.arch == DIT_ARCH_SD3) {   // SD3 position table on the image rows (reading C21)
    if (ragged)
      for (int q = 0; q < S; ++q)
        CKC(pos_embed_add_launch(c->h + (size_t)q * N * D, 1, N, nt, img_valid[q], 0, seq_hw[2 * q],
                                 seq_hw[2 * q + 1], D, c->cfg.pos_embed_max, c->cfg.pos_embed_base, s));
    else
      CKC(pos_embed_add_launch(c->h, S, N, nt, ni, c->rank * ni, b->img_h, b->img_w, D, c->cfg.pos_embed_max,
                               c->cfg.pos_embed_base, s));
  }

  const float scale_log2 = 1.4426950408889634f / std::sqrt((float)d);
  // ---- attention with the Ulysses exchange around it (P > 1): QKV epilogue wrote
  // [P][3][S][H/P][N_loc][d] -> a2a -> global order -> attention on H/P heads over the
  // full sequence -> O in [P][S][N_loc][H/P*d] -> a2a -> scatter into the local rows.
  const int Hl = H / P, Nglob = P * N;
  const bool sp = P > 1 || c->force_sp;   // Ulysses exchange active
  const bool fused = P > 1 && c->sp_fused;  // ... done by the epilogues over peer memory
  if (fused && !c->peers_ready) {          // in-process group: every rank has registered by now
    LocalGroup* g = c->local_group;
    for (int r = 0; r < P; ++r) {
      if (!g || !g->qkv[r]) return c->fail(DIT_EPARALLEL, "rank %d of the local group has not called sp_init_local", r);
      c->peer_qkv[r] = g->qkv[r];
      c->peer_o[r] = g->o[r];
      c->peer_cat[r] = g->cat[r];
      c->peer_flags.f[r] = g->flags[r];
    }
    c->peers_ready = true;
  }
  if (lpar && c->lp_fused && !c->peers_ready) {   // in-process latent-parallel group
    LocalGroup* g = c->lp_group;
    for (int r = 0; r < 2; ++r) {
      if (!g || !g->vcfg[r]) return c->fail(DIT_EPARALLEL, "rank %d of the local group has not called lp_init_local", r);
      c->peer_vcfg[r] = static_cast<float*>(g->vcfg[r]);
      c->peer_flags.f[r] = g->flags[r];
    }
    c->peers_ready = true;
  }
  // fused exchange barrier: my stores into the peers are done -> tell them; wait for theirs
  auto exchange_barrier = [&]() -> int {
    ++c->sp_epoch;
    prof_begin(c, s, 5);
    cudaError_t e1 = sp_signal_launch(c->peer_flags, c->rank, P, c->sp_epoch, s);
    cudaError_t e2 = sp_wait_launch(c->flags, c->rank, P, c->sp_epoch, s);
    prof_end(c, s, 5, 0.0);
    c->launches += 2;
    if (e1 != cudaSuccess || e2 != cudaSuccess) return c->fail(DIT_ECUDA, "sp barrier launch failed");
    return DIT_OK;
  };
  auto a2a = [&](const void* snd, void* rcv, size_t count) -> int {
    prof_begin(c, s, 5);
    if (c->comm) {
      ncclResult_t r = ncclAlltoAll(snd, rcv, count, ncclBfloat16, c->comm, s);
      if (r != ncclSuccess) return c->fail(DIT_ENCCL, "ncclAlltoAll: %s", ncclGetErrorString(r));
    } else {
      c->local_group->a2a(c->rank, snd, rcv, count * 2, s);
    }
    prof_end(c, s, 5, 0.0);
    c->launches++;
    return DIT_OK;
  };
  auto attention_stage = [&](void* out, int ld_out, int split) -> int {
    const size_t pp1 = (size_t)3 * S * Hl * N * d, pp2 = (size_t)S * N * Hl * d;
    bf16_t* send1 = c->sp;
    bf16_t* recv1 = send1 + (size_t)P * pp1;
    bf16_t* send2 = recv1 + (size_t)P * pp1;
    bf16_t* recv2 = send2 + (size_t)P * pp2;
    if (fused) {
      CK(exchange_barrier());   // every rank's q/k/v rows are in my attention buffer
    } else if (sp) {
      CK(a2a(send1, recv1, pp1));
      CKK(sp_gather_qkv_launch(recv1, c->qkv, P, S, Hl, nt, ni, d, s), 6, 0.0);
    }
    AttnParams ap;
    memset(&ap, 0, sizeof(ap));
    const size_t sec = (size_t)S * Hl * Nglob * d;
    ap.q = c->qkv;
    ap.k = c->qkv + sec;
    ap.v = c->qkv + 2 * sec;
    ap.B = S;
    ap.H = Hl;
    ap.N = Nglob;
    ap.d = d;
    ap.scale_log2 = scale_log2;
    ap.nt = nt;
    ap.ni = ni;
    ap.Nt = Nt;
    ap.seq_valid = ragged ? c->p_seq_valid : nullptr;
    ap.split_tail = c->attn_split_tail ? 1 : 0;
    ap.tail_ws = c->attn_tail_ws;
    ap.tail_cnt = c->attn_tail_cnt;
    if (fused) {   // O rows straight to their owners' buffers
      ap.split = 3;
      ap.out_split = split;
      ap.ld_out = ld_out;
      ap.head_off = c->rank * Hl;
      for (int r = 0; r < P; ++r) ap.out_peer[r] = (out == (void*)c->o) ? c->peer_o[r] : c->peer_cat[r];
    } else if (!sp) {
      ap.out = out;
      ap.ld_out = ld_out;
      ap.split = split;
    } else {
      ap.out = send2;
      ap.ld_out = Hl * d;
      ap.split = 2;
    }
    CKK(attention_launch(ap, s), 1, 4.0 * S * (double)Nglob * Nglob * Hl * d);
    if (fused) {
      CK(exchange_barrier());   // every rank's O rows of my tokens are in my buffer
    } else if (sp) {
      CK(a2a(send2, recv2, pp2));
      CKK(sp_scatter_o_launch(recv2, out, ld_out, split, P, S, Hl, nt, ni, d, s), 6, 0.0);
    }
    return DIT_OK;
  };
  // LN-modulate of the txt and/or img stream; shift / scale given as absolute mod columns
  // (txt_on = false: image stream only -- after SD3's context_pre_only attention)
  auto lnmod_st = [&](bool txt_on, int shT, int scT, int shI, int scI) -> int {
    LnModParams lp;
    memset(&lp, 0, sizeof(lp));
    lp.h = c->h;
    lp.D = D;
    lp.joint_n = N;
    lp.u = c->u;
    lp.mod_stride = c->mod_total;
    lp.nseg = 2;
    lp.seg_rows[0] = Mt;
    lp.seg_rows[1] = Mi;
    lp.seg_rows_per_req[0] = nt;
    lp.seg_rows_per_req[1] = ni;
    lp.seg_joint_off[0] = 0;
    lp.seg_joint_off[1] = nt;
    lp.seg_shift_off[0] = shT;
    lp.seg_scale_off[0] = scT;
    lp.seg_shift_off[1] = shI;
    lp.seg_scale_off[1] = scI;
    lp.seg_mod[0] = lp.seg_mod[1] = c->mod;
    if (!txt_on) {   // the image segment alone, written at its usual place (after the txt rows)
      lp.u = c->u + (size_t)Mt * D;
      lp.nseg = 1;
      lp.seg_rows[0] = Mi;
      lp.seg_rows_per_req[0] = ni;
      lp.seg_joint_off[0] = nt;
      lp.seg_shift_off[0] = shI;
      lp.seg_scale_off[0] = scI;
    }
    prof_begin(c, s, 2);
    cudaError_t e = lnmod_launch(lp, s);
    prof_end(c, s, 2, 0.0);
    c->launches++;
    return e == cudaSuccess ? DIT_OK : c->fail(DIT_ECUDA, "lnmod: %s", cudaGetErrorString(e));
  };
  auto lnmod2 = [&](int modT, int modI, int sh, int sc) -> int {
    return lnmod_st(true, modT + sh, modT + sc, modI + sh, modI + sc);
  };
  auto shrink2 = [&](const void* At, const void* Ai, int K, int lda, int modT, int modI, bool txt_on = true) -> int {
    if (!any_lora) return DIT_OK;
    const void* A[2] = {At, Ai};
    const int M[2] = {Mt, Mi}, Ks[2] = {K, K}, ld[2] = {lda, lda};
    const RowSpace* R[2] = {&c->rs[0], &c->rs[1]};
    const int mods[2] = {modT, modI};
    const int base[2] = {0, Mt};
    if (!txt_on) return run_shrink(c, 1, A + 1, M + 1, Ks + 1, ld + 1, R + 1, mods + 1, base + 1, s);
    return run_shrink(c, 2, A, M, Ks, ld, R, mods, base, s);
  };

  // deferred ControlNet inputs of block `blk` (double blocks 0..Ld-1, then single blocks):
  // wait on their producers' ready events right before the consuming GEMM
  auto cn_wait = [&](int blk) -> bool {
    bool any = false;
    for (auto& kv : c->cn)
      if (kv.first.second == blk)
        for (auto& r : kv.second) {
          any = true;
          if (r.ready) cudaStreamWaitEvent(s, r.ready, wait_fl);
        }
    return any;
  };

  // ---- double-stream blocks
  for (int i = 0; i < c->Ld; ++i) {
    NvtxRange nv_blk("double block %d", i);
    const DoubleStream& I = c->dbl[0][i];
    const DoubleStream& T = c->dbl[1][i];
    const int mI = (i * 2 + 0) * 6 * D, mT = (i * 2 + 1) * 6 * D;
    bf16_t* uT = c->u;
    bf16_t* uI = c->u + (size_t)Mt * D;
    // SD3 last block: the text stream is context_pre_only -- (scale, shift) modulation, then it
    // only feeds attention (reading C21)
    const bool po = pre_only(c->cfg, i, 1);
    if (po) CK(lnmod_st(true, mT + D, mT, mI, mI + D));
    else CK(lnmod2(mT, mI, 0, D));
    CK(shrink2(uT, uI, D, D, T.lora[0], I.lora[0]));
    {
      EpiParams e;
      memset(&e, 0, sizeof(e));
      e.kind = EPI_QKV;
      e.joint_n = N;
      e.D = D;
      e.qkv = (P == 1 && !c->force_sp) ? c->qkv : c->sp;
      if (fused) {
        for (int r = 0; r < P; ++r) e.qkv_peer[r] = c->peer_qkv[r];
        e.sp_rank = c->rank;
        e.sp_nt = nt;
        e.sp_ni = ni;
      }
      e.batch = S;
      e.sp_world = P;
      e.rope = c->rope;
      e.rope_stride = rope_stride;
      e.qkv_cols = 3 * D;
      e.heads = H;
      e.head_dim = d;
      e.seq_len = N;
      EpiParams eT = e, eI = e;
      eT.bias = T.qkv.b;
      eT.rows_per_req = nt;
      eT.joint_off = 0;
      eT.q_gamma = T.qn;
      eT.k_gamma = T.kn;
      eI.bias = I.qkv.b;
      eI.rows_per_req = ni;
      eI.joint_off = nt;
      eI.q_gamma = I.qn;
      eI.k_gamma = I.kn;
      GemmProblem p[2] = {base_problem(c, uT, Mt, D, D, T.qkv, eT), base_problem(c, uI, Mi, D, D, I.qkv, eI)};
      if (any_lora) {
        add_lora_ext(c, p[0], c->rs[0], T.lora[0], sext_of(c, 0));
        add_lora_ext(c, p[1], c->rs[1], I.lora[0], sext_of(c, Mt));
      }
      c->gemm_label = 11;
      CK(run_gemm(c, p, 2, s));
    }
    CK(attention_stage(c->o, D, 1));
    bf16_t* oT = c->o;
    bf16_t* oI = c->o + (size_t)Mt * D;
    auto resid_pair = [&](const Lin& LT, const Lin& LI, const void* AT, const void* AI, int K, int lda, int goff,
                          int modT_l, int modI_l, const void* const* cn_ptr) -> int {
      EpiParams e;
      memset(&e, 0, sizeof(e));
      e.kind = EPI_RESID;
      e.h = c->h;
      e.D = D;
      e.joint_n = N;
      e.mod = c->mod;
      e.mod_stride = c->mod_total;
      EpiParams eT = e, eI = e;
      eT.bias = LT.b;
      eT.rows_per_req = nt;
      eT.joint_off = 0;
      eT.gate_off = mT + goff;
      eI.bias = LI.b;
      eI.rows_per_req = ni;
      eI.joint_off = nt;
      eI.gate_off = mI + goff;
      if (cn_ptr) {
        eI.cn_ptr = cn_ptr;
        eI.cn_scale = c->p_cn_kappa + (size_t)i * CN_FANIN * MAX_SEQ;
        eI.cn_row0 = 0;   // the img-stream problem's rows are exactly the residual's rows
        eI.img_valid = ragged ? c->p_img_valid : nullptr;
        if (c->cn_flags) {
          eI.cn_flag = c->p_cn_flag + (size_t)i * CN_FANIN * MAX_SEQ;
          eI.cn_expect = c->p_cn_expect + (size_t)i * CN_FANIN * MAX_SEQ;
        }
      }
      GemmProblem p[2] = {base_problem(c, AT, Mt, K, lda, LT, eT), base_problem(c, AI, Mi, K, lda, LI, eI)};
      if (any_lora) {
        add_lora_ext(c, p[0], c->rs[0], modT_l, sext_of(c, 0));
        add_lora_ext(c, p[1], c->rs[1], modI_l, sext_of(c, Mt));
      }
      c->gemm_label = goff == 2 * D ? 12 : 14;
      if (po) return run_gemm(c, p + 1, 1, s);   // context_pre_only: image stream only
      return run_gemm(c, p, 2, s);
    };
    CK(shrink2(oT, oI, D, D, T.lora[1], I.lora[1], !po));
    CK(resid_pair(T.proj, I.proj, oT, oI, D, D, 2 * D, T.lora[1], I.lora[1], nullptr));
    CK(lnmod_st(!po, mT + 3 * D, mT + 4 * D, mI + 3 * D, mI + 4 * D));
    CK(shrink2(uT, uI, D, D, T.lora[2], I.lora[2], !po));
    bf16_t* aT = c->cat;
    bf16_t* aI = c->cat + (size_t)Mt * F;
    {
      EpiParams e;
      memset(&e, 0, sizeof(e));
      e.kind = EPI_GELU;
      e.ld_out = F;
      e.joint_n = N;
      EpiParams eT = e, eI = e;
      eT.bias = T.fc1.b;
      eT.rows_per_req = nt;
      eT.out = aT;
      eI.bias = I.fc1.b;
      eI.rows_per_req = ni;
      eI.joint_off = nt;
      eI.out = aI;
      GemmProblem p[2] = {base_problem(c, uT, Mt, D, D, T.fc1, eT), base_problem(c, uI, Mi, D, D, I.fc1, eI)};
      if (any_lora) {
        add_lora_ext(c, p[0], c->rs[0], T.lora[2], sext_of(c, 0));
        add_lora_ext(c, p[1], c->rs[1], I.lora[2], sext_of(c, Mt));
      }
      c->gemm_label = 13;
      if (po) CK(run_gemm(c, p + 1, 1, s));
      else CK(run_gemm(c, p, 2, s));
    }
    // deferred ControlNet input of block i: wait right before its consumer
    const bool has_cn = cn_wait(i);
    CK(shrink2(aT, aI, F, F, T.lora[3], I.lora[3], !po));
    CK(resid_pair(T.fc2, I.fc2, aT, aI, F, F, 5 * D, T.lora[3], I.lora[3],
                  has_cn ? (const void* const*)(c->p_cn_ptr + (size_t)i * CN_FANIN * MAX_SEQ) : nullptr));
  }

  // ---- single-stream blocks on the joint sequence
  for (int j = 0; j < c->Ls; ++j) {
    NvtxRange nv_blk("single block %d", j);
    const SingleBlk& SB = c->sgl[j];
    const int mj = mod_off_single + j * 3 * D;
    {
      LnModParams lp;
      memset(&lp, 0, sizeof(lp));
      lp.h = c->h;
      lp.D = D;
      lp.joint_n = N;
      lp.u = c->u;
      lp.mod_stride = c->mod_total;
      lp.nseg = 1;
      lp.seg_rows[0] = Mj;
      lp.seg_rows_per_req[0] = N;
      lp.seg_joint_off[0] = 0;
      lp.seg_shift_off[0] = mj;
      lp.seg_scale_off[0] = mj + D;
      lp.seg_mod[0] = c->mod;
      CKK(lnmod_launch(lp, s), 2, 0.0);
    }
    if (any_lora) {
      const void* A[1] = {c->u};
      const int M[1] = {Mj}, K[1] = {D}, ld[1] = {D};
      const RowSpace* R[1] = {&c->rs[2]};
      const int mods[1] = {SB.lora[0]};
      const int base[1] = {0};
      CK(run_shrink(c, 1, A, M, K, ld, R, mods, base, s));
    }
    {
      EpiParams e;
      memset(&e, 0, sizeof(e));
      e.kind = EPI_QKV;
      e.bias = SB.l1.b;
      e.rows_per_req = N;
      e.joint_off = 0;
      e.joint_n = N;
      e.D = D;
      e.qkv = (P == 1 && !c->force_sp) ? c->qkv : c->sp;
      if (fused) {
        for (int r = 0; r < P; ++r) e.qkv_peer[r] = c->peer_qkv[r];
        e.sp_rank = c->rank;
        e.sp_nt = nt;
        e.sp_ni = ni;
      }
      e.batch = S;
      e.sp_world = P;
      e.q_gamma = SB.qn;
      e.k_gamma = SB.kn;
      e.rope = c->rope;
      e.rope_stride = rope_stride;
      e.qkv_cols = 3 * D;
      e.heads = H;
      e.head_dim = d;
      e.seq_len = N;
      e.out = c->cat;
      e.ld_out = D + F;
      e.out_col0 = D;
      GemmProblem p = base_problem(c, c->u, Mj, D, D, SB.l1, e);
      if (any_lora) add_lora_ext(c, p, c->rs[2], SB.lora[0], sext_of(c, 0));
      c->gemm_label = 15;
      CK(run_gemm(c, &p, 1, s));
    }
    CK(attention_stage(c->cat, D + F, 0));
    if (any_lora) {
      const void* A[1] = {c->cat};
      const int M[1] = {Mj}, K[1] = {D + F}, ld[1] = {D + F};
      const RowSpace* R[1] = {&c->rs[2]};
      const int mods[1] = {SB.lora[1]};
      const int base[1] = {0};
      CK(run_shrink(c, 1, A, M, K, ld, R, mods, base, s));
    }
    {
      EpiParams e;
      memset(&e, 0, sizeof(e));
      e.kind = EPI_RESID;
      e.bias = SB.l2.b;
      e.rows_per_req = N;
      e.joint_off = 0;
      e.joint_n = N;
      e.h = c->h;
      e.D = D;
      e.mod = c->mod;
      e.mod_stride = c->mod_total;
      e.gate_off = mj + 2 * D;
      if (cn_wait(c->Ld + j)) {   // single-block ControlNet residual on the image rows (reading C20)
        e.cn_ptr = (const void* const*)(c->p_cn_ptr + (size_t)(c->Ld + j) * CN_FANIN * MAX_SEQ);
        e.cn_scale = c->p_cn_kappa + (size_t)(c->Ld + j) * CN_FANIN * MAX_SEQ;
        e.cn_row0 = nt;           // joint rows are [txt; img] per request
        e.img_valid = ragged ? c->p_img_valid : nullptr;
        if (c->cn_flags) {
          e.cn_flag = c->p_cn_flag + (size_t)(c->Ld + j) * CN_FANIN * MAX_SEQ;
          e.cn_expect = c->p_cn_expect + (size_t)(c->Ld + j) * CN_FANIN * MAX_SEQ;
        }
      }
      GemmProblem p = base_problem(c, c->cat, Mj, D + F, D + F, SB.l2, e);
      if (any_lora) add_lora_ext(c, p, c->rs[2], SB.lora[1], sext_of(c, 0));
      c->gemm_label = 16;
      CK(run_gemm(c, &p, 1, s));
    }
  }

  // ---- final layer + Euler update (fused epilogue)
  {
    LnModParams lp;
    memset(&lp, 0, sizeof(lp));
    lp.h = c->h;
    lp.D = D;
    lp.joint_n = N;
    lp.u = c->u;
    lp.mod_stride = c->mod_total;
    lp.nseg = 1;
    lp.seg_rows[0] = Mi;
    lp.seg_rows_per_req[0] = ni;
    lp.seg_joint_off[0] = nt;
    // Flux LastLayer (shift, scale); SD3 AdaLayerNormContinuous (scale, shift) [ext]
    const bool sd3 = c->cfg.arch == DIT_ARCH_SD3;
    lp.seg_shift_off[0] = mod_off_final + (sd3 ? D : 0);
    lp.seg_scale_off[0] = mod_off_final + (sd3 ? 0 : D);
    lp.seg_mod[0] = c->mod;
    CKK(lnmod_launch(lp, s), 2, 0.0);
    EpiParams e;
    memset(&e, 0, sizeof(e));
    e.kind = EPI_FINAL;
    e.bias = c->fin_lin.b;
    e.rows_per_req = ni;
    e.joint_n = N;
    e.lat_in = b->latents_in;
    e.lat_out = b->latents_out;
    e.v_out = b->v_out;
    e.dsig = c->p_dsig;
    const size_t vcount = (size_t)B * ni * C;   // one branch's v
    // latent parallelism over peer stores: the two halves of vcfg alternate by step parity, so a
    // peer one step ahead never overwrites the buffer this rank's combine is still reading
    const size_t vpar = (lpar && c->lp_fused && (c->lp_steps & 1))
                            ? 2 * (size_t)c->cfg.max_batch * c->cfg.max_img_tokens * C : 0;
    float* vbuf = c->vcfg + vpar;
    if (cfgon) {   // v of every sequence into vcfg [cond B | uncond B]; Euler after the combine
      e.lat_in = nullptr;
      e.lat_out = nullptr;
      e.v_out = vbuf + (lpar ? (size_t)c->lp_rank * vcount : 0);
      if (lpar && c->lp_fused)   // ... and into the peer's buffer at the same place: the all-gather, fused
        e.v_peer = c->peer_vcfg[1 - c->lp_rank] + vpar + (size_t)c->lp_rank * vcount;
    }
    GemmProblem p = base_problem(c, c->u, Mi, D, D, c->fin_lin, e);
    c->gemm_label = 17;
    CK(run_gemm(c, &p, 1, s));
    if (lpar) {   // latent parallelism: per-step gather of the two branches' v
      prof_begin(c, s, 5);
      if (c->lp_fused) {   // both halves are in place once the peer's epilogue has released its flag
        ++c->sp_epoch;
        ++c->lp_steps;
        cudaError_t e1 = sp_signal_launch(c->peer_flags, c->lp_rank, 2, c->sp_epoch, s);
        cudaError_t e2 = sp_wait_launch(c->flags, c->lp_rank, 2, c->sp_epoch, s);
        c->launches += 1;
        if (e1 != cudaSuccess || e2 != cudaSuccess) return c->fail(DIT_ECUDA, "lp barrier launch failed");
      } else if (c->lp_comm) {
        ncclResult_t r = ncclAllGather(vbuf + (size_t)c->lp_rank * vcount, vbuf, vcount, ncclFloat32,
                                       c->lp_comm, s);
        if (r != ncclSuccess) return c->fail(DIT_ENCCL, "ncclAllGather: %s", ncclGetErrorString(r));
      } else {
        c->lp_group->allgather(c->lp_rank, vbuf, vcount * 4, s);
      }
      prof_end(c, s, 5, 0.0);
      c->launches++;
    }
    if (cfgon)   // v = v_u + g (v_c - v_u); latents_out = latents_in + dsig v (reading C22)
      CKC(cfg_euler_launch(vbuf, vbuf + vcount, c->p_cfg, c->p_dsig, b->latents_in, b->latents_out, b->v_out,
                           B, ni * C, s));
  }

  for (int i = 0; i < S; ++i)
    if (req_slot[i] >= 0) record(c->slot_last_use[req_slot[i]]);
  if (c->merged_adapter >= 0) record(c->merged_last_use);
  record(c->step_done);
  c->last_launches = c->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return c->fail(DIT_ECUDA, "step: %s", cudaGetErrorString(e));
  return DIT_OK;
}

// ------------------------------------------------------------------ CUDA graphs
// One captured dit_step replayed with fresh per-step scalars (sigma, guidance, CFG / ControlNet
// scales, ControlNet residual pointers): dit_graph_launch re-runs the step's host logic in staging
// mode into the graph's own pinned block (which the graph's copy nodes read), then launches the
// graph -- no per-kernel launch cost.
struct dit_graph {
  dit_ctx* c = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint8_t* block = nullptr;     // pinned, stage_bytes
  cudaEvent_t staged = nullptr; // recorded by each replay once its copy nodes have read `block`
  dit_batch key{};              // captured shape and device pointers
  std::vector<int> ids, hw;
  std::vector<std::pair<std::pair<int, int>, std::vector<cudaEvent_t>>> cn_key;   // (slot, block) -> events
};

namespace {
std::vector<std::pair<std::pair<int, int>, std::vector<cudaEvent_t>>> cn_signature(const dit_ctx* c, bool* flags) {
  std::vector<std::pair<std::pair<int, int>, std::vector<cudaEvent_t>>> v;
  *flags = false;
  for (auto& kv : c->cn) {
    std::vector<cudaEvent_t> ev;
    for (auto& r : kv.second) {
      ev.push_back(r.ready);
      *flags |= r.flag != nullptr;
    }
    v.push_back({kv.first, ev});
  }
  return v;
}
bool same_shape(const dit_graph* g, const dit_batch* b) {
  const dit_batch& k = g->key;
  if (b->batch != k.batch || b->img_h != k.img_h || b->img_w != k.img_w || b->txt_tokens != k.txt_tokens) return false;
  if (b->latents_in != k.latents_in || b->latents_out != k.latents_out || b->txt != k.txt || b->pooled != k.pooled ||
      b->v_out != k.v_out)
    return false;
  if ((b->cfg_scale == nullptr) != (k.cfg_scale == nullptr) || (b->img_hw == nullptr) != (k.img_hw == nullptr))
    return false;
  for (int i = 0; i < b->batch; ++i)
    if (!b->adapter_id || b->adapter_id[i] != g->ids[i]) return false;
  for (size_t i = 0; i < g->hw.size(); ++i)
    if (b->img_hw[i] != g->hw[i]) return false;
  return true;
}
}  // namespace

extern "C" int dit_graph_create(dit_ctx* c, const dit_batch* b, void* stream, dit_graph** out) {
  if (!c) return DIT_EINVAL;
  if (!out || !b) return c->fail(DIT_EINVAL, "NULL argument");
  *out = nullptr;
  if (c->local_group || c->lp_group) return c->fail(DIT_EPARALLEL, "in-process groups are not capturable");
  if ((c->world > 1 && c->sp_fused) || (c->lp_world > 1 && c->lp_fused))
    return c->fail(DIT_EPARALLEL, "the fused peer exchange's epochs are per launch: not capturable");
  bool flags = false;
  auto sig = cn_signature(c, &flags);
  if (flags) return c->fail(DIT_EINVAL, "device-flag ControlNet inputs are single-use: not capturable");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (s == nullptr) return c->fail(DIT_EINVAL, "capture needs a non-default stream");
  dit_graph* g = new dit_graph();
  g->c = c;
  if (cudaHostAlloc(reinterpret_cast<void**>(&g->block), c->stage_bytes, cudaHostAllocDefault) != cudaSuccess) {
    delete g;
    return c->fail(DIT_ECUDA, "cudaHostAlloc of the graph's staging block failed");
  }
  g->key = *b;
  g->ids.assign(b->adapter_id ? b->adapter_id : nullptr, b->adapter_id ? b->adapter_id + b->batch : nullptr);
  if (b->img_hw) g->hw.assign(b->img_hw, b->img_hw + 2 * b->batch);
  g->cn_key = sig;
  cudaEventCreateWithFlags(&g->staged, cudaEventDisableTiming);
  c->st_base = g->block;
  c->st_event = g->staged;
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaFreeHost(g->block);
    delete g;
    return c->fail(DIT_ECUDA, "cudaStreamBeginCapture failed");
  }
  int r = step_impl(c, b, s, STEP_CAPTURE);
  c->st_event = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &graph);
  c->plan_B = -1;                        // the device tables now hold the graph's plan
  c->rope_key[0] = -1;
  if (r != DIT_OK || e != cudaSuccess ||
      cudaGraphInstantiate(&g->exec, graph, cudaGraphInstantiateFlagAutoFreeOnLaunch) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaFreeHost(g->block);
    cudaEventDestroy(g->staged);
    delete g;
    cudaGetLastError();
    return r != DIT_OK ? r : c->fail(DIT_ECUDA, "graph capture / instantiation failed: %s", cudaGetErrorString(e));
  }
  cudaGraphDestroy(graph);
  *out = g;
  return DIT_OK;
}

extern "C" int dit_graph_launch(dit_graph* g, const dit_batch* b, void* stream) {
  if (!g || !g->c) return DIT_EINVAL;
  dit_ctx* c = g->c;
  if (!b) return c->fail(DIT_EINVAL, "batch is NULL");
  if (!same_shape(g, b)) return c->fail(DIT_EINVAL, "batch shape / pointers / adapters differ from the captured step");
  bool flags = false;
  if (cn_signature(c, &flags) != g->cn_key || flags)
    return c->fail(DIT_EINVAL, "ControlNet registrations differ from the captured step (slots, blocks, events)");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // the previous replay's copy nodes may still have to read the block (the host runs <= 1 replay ahead)
  if (cudaEventSynchronize(g->staged) != cudaSuccess) return c->fail(DIT_ECUDA, "previous replay failed");
  c->st_base = g->block;
  const int r = step_impl(c, b, s, STEP_STAGE);
  if (r != DIT_OK) return r;
  const cudaError_t e = cudaGraphLaunch(g->exec, s);
  c->plan_B = -1;                        // device plan tables / rope now the graph's
  c->rope_key[0] = -1;
  c->launches = 1;
  return e == cudaSuccess ? DIT_OK : c->fail(DIT_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(e));
}

extern "C" void dit_graph_destroy(dit_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->block) cudaFreeHost(g->block);
  if (g->staged) cudaEventDestroy(g->staged);
  delete g;
}

// ------------------------------------------------------------------ profiling exports
extern "C" int dit_profile(dit_ctx* c, int enable) {
  if (!c) return DIT_EINVAL;
  c->prof_on = enable != 0;
  return DIT_OK;
}

extern "C" int dit_profile_read(dit_ctx* c, int kind, double* total_ms, double* flops, int* launches) {
  if (!c || kind < 0 || kind > 18) return DIT_EINVAL;
  double ms = 0, fl = 0;
  int n = 0;
  for (auto& r : c->prof) {
    const bool match = (r.kind == kind) || (kind == 0 && r.kind >= 10);
    if (!match) continue;
    cudaEventSynchronize(r.b);
    float e = 0.f;
    cudaEventElapsedTime(&e, r.a, r.b);
    ms += e;
    fl += r.flops;
    ++n;
  }
  if (total_ms) *total_ms = ms;
  if (flops) *flops = fl;
  if (launches) *launches = n;
  return DIT_OK;
}

extern "C" int dit_profile_reset(dit_ctx* c) {
  if (!c) return DIT_EINVAL;
  c->prof.clear();
  c->ev_next = 0;
  return DIT_OK;
}

// ------------------------------------------------------------------ test-only exports
extern "C" int dit_fill_synthetic(void* dst, int64_t n, uint64_t seed, uint64_t tid, float scale, float offset,
                                  void* stream) {
  if (!dst || n < 0) return DIT_EINVAL;
  cudaError_t e = fill_synthetic_launch(dst, n, seed, tid, scale, offset, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

namespace {
// req_slot per SEQUENCE (CFG without latent parallelism: 2B sequences, sequence q = request q % B)
int debug_prepare(dit_ctx* c, const dit_batch* b, std::vector<int>& req_slot, int& nt, int& ni) {
  if (!b || b->batch < 1 || b->batch > c->cfg.max_batch) return -DIT_EBATCH;
  const int P = c->world;
  const int Ni = b->img_h * b->img_w, Nt = b->txt_tokens;
  if (Ni <= 0 || Nt <= 0 || Ni % P || Nt % P) return -DIT_EPARALLEL;
  nt = Nt / P;
  ni = Ni / P;
  const int S = (b->cfg_scale && c->lp_world == 1) ? 2 * b->batch : b->batch;
  if (S > c->cfg.max_batch) return -DIT_EBATCH;
  req_slot.assign(S, -1);
  for (int i = 0; i < S; ++i) {
    const int aid = b->adapter_id ? b->adapter_id[i % b->batch] : -1;
    if (aid < 0 || c->merged_adapter >= 0) continue;
    auto it = c->adapter_slot.find(aid);
    if (it == c->adapter_slot.end()) return -DIT_EADAPTER;
    req_slot[i] = it->second;
  }
  return 0;
}
}  // namespace

extern "C" int dit_debug_row_adapter(dit_ctx* c, const dit_batch* b, int32_t* out, int cap) {
  if (!c || !out) return -DIT_EINVAL;
  std::vector<int> rs;
  int nt, ni;
  int r = debug_prepare(c, b, rs, nt, ni);
  if (r < 0) return r;
  const int S = (int)rs.size();
  const int rows = S * nt + S * ni;
  if (cap < rows) return -DIT_EINVAL;
  // the planner dit_step uses (build_rowspace), on scratch row spaces (the step's cache is untouched)
  int k = 0;
  const int Ms[2] = {S * nt, S * ni}, rpr[2] = {nt, ni};
  for (int q = 0; q < 2; ++q) {
    RowSpace R;
    std::vector<int> ht, hc;
    std::vector<int2> hs;
    if (build_rowspace(c, R, Ms[q], rpr[q], rs, ht, hc, hs) < 0) return -DIT_ESHAPE;
    for (int x = 0; x < Ms[q]; ++x) out[k++] = R.h_row_slot[x];
  }
  return rows;
}

// The integer tables the LAST dit_step uploaded for row space `which` (0 txt stream, 1 img stream,
// 2 joint sequence), read back from the device: kind 0 row -> pool slot [M], 1 tile -> sorted
// distinct slots [tiles_m][slot_cap] (unused entries 0), 2 distinct slots per tile [tiles_m],
// 3 shrink work list (tile, slot) pairs [n_shrink][2].  Test-only (synchronous).
extern "C" int dit_debug_plan(dit_ctx* c, int32_t which, int32_t kind, int32_t* out, int cap) {
  if (!c || !out || which < 0 || which > 2 || kind < 0 || kind > 3) return -DIT_EINVAL;
  if (c->plan_B < 0) return -DIT_ENOENT;
  const RowSpace& R = c->rs[which];
  const void* src = nullptr;
  int n = 0;
  switch (kind) {
    case 0: src = R.row_slot; n = R.M; break;
    case 1: src = R.tile_slots; n = R.tiles_m * c->slot_cap; break;
    case 2: src = R.tile_cnt; n = R.tiles_m; break;
    default: src = R.shrink_list; n = 2 * R.n_shrink; break;
  }
  if (n > cap) return -DIT_EINVAL;
  if (n > 0 && cudaMemcpy(out, src, (size_t)n * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return -DIT_ECUDA;
  return n;
}

// Bench-only: one plain projection out = bf16(A W^T + bias) through the tcgen05 GEMM (the same
// kernel and tile schedule as the step, EPI_BIAS epilogue) for the library bars.
extern "C" int dit_debug_gemm(const void* A, const void* W, const void* bias, void* out, int32_t M, int32_t N,
                              int32_t K, void* stream) {
  if (!A || !W || !bias || !out || M < 1 || N < 1 || K < 64 || K % 64) return DIT_EINVAL;
  GemmProblem P;
  memset(&P, 0, sizeof(P));
  if (!make_tmap_2d(&P.tmA, A, K, M, (uint64_t)K * 2, 64, GEMM_BM) ||
      !make_tmap_2d(&P.tmB, W, K, N, (uint64_t)K * 2, 64, 128))
    return DIT_EINVAL;
  P.M = M;
  P.N = N;
  P.K = K;
  P.tiles_m = (M + GEMM_TM - 1) / GEMM_TM;
  P.tiles_n = (N + GEMM_BN - 1) / GEMM_BN;
  P.num_tiles = P.tiles_m * P.tiles_n;
  P.epi.kind = EPI_BIAS;
  P.epi.bias = bias;
  P.epi.out = out;
  P.epi.ld_out = N;
  P.epi.rows_per_req = M;
  P.epi.joint_n = M;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.p[0] = P;
  a.num_problems = 1;
  a.total_tiles = P.num_tiles;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return gemm_launch(a, sms, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

// Bench-only: the gated-residual projection of the step alone: h[M][N] (fp32) += gate[N] * (A W^T +
// bias) through the same GEMM + EPI_RESID epilogue (profiling the epilogue's cost).
extern "C" int dit_debug_gemm_resid(const void* A, const void* W, const void* bias, float* h, const float* gate,
                                    int32_t M, int32_t N, int32_t K, void* stream) {
  if (!A || !W || !bias || !h || !gate || M < 1 || N < 1 || K < 64 || K % 64 || N % 32) return DIT_EINVAL;
  GemmProblem P;
  memset(&P, 0, sizeof(P));
  if (!make_tmap_2d(&P.tmA, A, K, M, (uint64_t)K * 2, 64, GEMM_BM) ||
      !make_tmap_2d(&P.tmB, W, K, N, (uint64_t)K * 2, 64, 128))
    return DIT_EINVAL;
  P.M = M;
  P.N = N;
  P.K = K;
  P.tiles_m = (M + GEMM_TM - 1) / GEMM_TM;
  P.tiles_n = (N + GEMM_BN - 1) / GEMM_BN;
  P.num_tiles = P.tiles_m * P.tiles_n;
  P.epi.kind = EPI_RESID;
  P.epi.bias = bias;
  P.epi.h = h;
  P.epi.D = N;
  P.epi.rows_per_req = M;
  P.epi.joint_n = M;
  P.epi.mod = gate;
  P.epi.mod_stride = 0;
  P.epi.gate_off = 0;
  P.tmH_ok = make_tmap_2d_f32(&P.tmH, h, (uint64_t)N, (uint64_t)M, (uint64_t)N * 4, 32, 32) ? 1 : 0;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.p[0] = P;
  a.num_problems = 1;
  a.total_tiles = P.num_tiles;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return gemm_launch(a, sms, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

// Test/bench-only: one attention launch on head-major q/k/v [B][H][N][d] (bf16),
// O written joint-row-major [B*N][H*d] (d = 128 -> tcgen05 kernel).
extern "C" int dit_debug_attention_ex(const void* q, const void* k, const void* v, int32_t B, int32_t H, int32_t N,
                                      int32_t d, void* out, int32_t split_tail, void* stream) {
  if (!q || !k || !v || !out || B < 1 || H < 1 || N < 1) return DIT_EINVAL;
  AttnParams ap;
  memset(&ap, 0, sizeof(ap));
  ap.q = q;
  ap.k = k;
  ap.v = v;
  ap.B = B;
  ap.H = H;
  ap.N = N;
  ap.d = d;
  ap.scale_log2 = 1.4426950408889634f / std::sqrt((float)d);
  ap.out = out;
  ap.ld_out = H * d;
  ap.split = 0;
  static float* tail_ws = nullptr;        // one process-wide tail workspace (debug / bench launches)
  static uint32_t* tail_cnt = nullptr;
  if (split_tail && d >= 64) {
    if (!tail_ws && (cudaMalloc(&tail_ws, attn_tail_ws_bytes(128)) != cudaSuccess ||
                     cudaMalloc(&tail_cnt, ATTN_TAIL_UNITS * 2 * 4) != cudaSuccess ||
                     cudaMemset(tail_cnt, 0, ATTN_TAIL_UNITS * 2 * 4) != cudaSuccess))
      return DIT_ENOMEM;
    ap.split_tail = 1;
    ap.tail_ws = tail_ws;
    ap.tail_cnt = tail_cnt;
  }
  return attention_launch(ap, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

extern "C" int dit_debug_attention(const void* q, const void* k, const void* v, int32_t B, int32_t H, int32_t N,
                                   int32_t d, void* out, void* stream) {
  static const bool split_tail = [] {   // DIT_ATTN_SPLIT_TAIL=1: the split tail for bench runs
    const char* e = getenv("DIT_ATTN_SPLIT_TAIL");
    return e && e[0] == '1';
  }();
  return dit_debug_attention_ex(q, k, v, B, H, N, d, out, split_tail ? 1 : 0, stream);
}

namespace dit { cudaError_t attention_set_trace(long long* buf); }
// Debug: record a clock64 timeline of CTA (0,0,0) of the tcgen05 attention kernel
// into buf (device, 10 events x 64 iterations of int64); NULL disables.
extern "C" int dit_debug_attention_trace(void* buf) {
  return dit::attention_set_trace(static_cast<long long*>(buf)) == cudaSuccess ? DIT_OK : DIT_ECUDA;
}

extern "C" int dit_nccl_unique_id(void* out128) {
  if (!out128) return DIT_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DIT_ENCCL;
  memcpy(out128, &id, sizeof(id));
  return DIT_OK;
}

// Host export of the SP index maps the kernels use (kernels.h), for CPU tests.
//  which 0: shard map, out[b*nloc + i] = global joint row b*N + n of local row i
//  which 1: QKV send: out[sp_attn-style (sec,b,head,i) index over [3][B][H][nloc]] = send d-vector index
//  which 2: gather: out[recv d-vector index] = attention-layout d-vector index
//  which 3: O send: out[(b, n, hl) over [B][N][Hl]] = send2 row index (attn_out_row, SP mode)
//  which 4: scatter (split = 1): out[recv2 row (rs, b, i)] = local output row
extern "C" int64_t dit_sp_layout(int32_t which, int32_t world, int32_t rank, int32_t B, int32_t H, int32_t Nt,
                                 int32_t Ni, int64_t* out, int64_t cap) {
  const int P = world;
  if (P < 1 || rank < 0 || rank >= P || B < 1 || H % P || Nt % P || Ni % P || !out) return -DIT_EINVAL;
  const int nt = Nt / P, ni = Ni / P, nloc = nt + ni, N = Nt + Ni, Hl = H / P;
  int64_t k = 0;
  auto put = [&](int64_t v) { if (k < cap) out[k] = v; ++k; };
  if (which == 0) {
    for (int b = 0; b < B; ++b)
      for (int i = 0; i < nloc; ++i) put((int64_t)b * N + sp_global_row(P, nt, ni, rank, i));
  } else if (which == 1) {
    for (int sec = 0; sec < 3; ++sec)
      for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h)
          for (int i = 0; i < nloc; ++i) put(sp_qkv_send_vec(B, Hl, nloc, h / Hl, sec, b, h % Hl, i));
  } else if (which == 2) {
    for (int rs = 0; rs < P; ++rs)
      for (int sec = 0; sec < 3; ++sec)
        for (int b = 0; b < B; ++b)
          for (int hl = 0; hl < Hl; ++hl)
            for (int i = 0; i < nloc; ++i) put(sp_attn_vec(B, Hl, N, sec, b, hl, sp_global_row(P, nt, ni, rs, i)));
  } else if (which == 3) {
    AttnParams p;
    memset(&p, 0, sizeof(p));
    p.B = B; p.H = Hl; p.N = N; p.split = 2; p.nt = nt; p.ni = ni; p.Nt = Nt;
    for (int b = 0; b < B; ++b)
      for (int n = 0; n < N; ++n)
        for (int hl = 0; hl < Hl; ++hl) put(attn_out_row(p, b, n));
  } else if (which == 4) {
    for (int rs = 0; rs < P; ++rs)
      for (int b = 0; b < B; ++b)
        for (int i = 0; i < nloc; ++i) put(sp_local_row(1, B, nt, ni, b, i));
  } else if (which == 5) {
    // fused exchange, QKV epilogue: (sec, b, head, local row i) -> dest * 3*B*Hl*N + index in
    // dest's attention buffer (the expression of the EPI_QKV peer store)
    const int64_t span = (int64_t)3 * B * Hl * N;
    for (int sec = 0; sec < 3; ++sec)
      for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h)
          for (int i = 0; i < nloc; ++i)
            put((h / Hl) * span + sp_attn_vec(B, Hl, N, sec, b, h % Hl, sp_global_row(P, nt, ni, rank, i)));
  } else if (which == 6) {
    // fused exchange, attention epilogue: (b, global query n, local head hl) -> dest * 2^40 +
    // element index (row * H + global head) in dest's stream-split O buffer (attn_out_addr itself)
    AttnParams p;
    memset(&p, 0, sizeof(p));
    p.B = B; p.H = Hl; p.N = N; p.split = 3; p.out_split = 1; p.nt = nt; p.ni = ni; p.Nt = Nt;
    p.ld_out = H; p.head_off = rank * Hl;
    for (int r = 0; r < P; ++r) p.out_peer[r] = reinterpret_cast<void*>((uintptr_t)r << 41);
    for (int b = 0; b < B; ++b)
      for (int n = 0; n < N; ++n)
        for (int hl = 0; hl < Hl; ++hl) {
          const uintptr_t a = reinterpret_cast<uintptr_t>(attn_out_addr(p, b, n, hl, 1));
          put((int64_t)(a >> 41) * ((int64_t)1 << 40) + (int64_t)((a & (((uintptr_t)1 << 41) - 1)) >> 1));
        }
  } else {
    return -DIT_EINVAL;
  }
  return k;
}

extern "C" int dit_debug_shard_map(dit_ctx* c, const dit_batch* b, int32_t* out, int cap) {
  if (!c || !out) return -DIT_EINVAL;
  std::vector<int> rs;
  int nt, ni;
  int r = debug_prepare(c, b, rs, nt, ni);
  if (r < 0) return r;
  const int B = b->batch, Nt = b->txt_tokens, N = b->txt_tokens + b->img_h * b->img_w;
  const int rows = B * (nt + ni);
  if (cap < rows) return -DIT_EINVAL;
  int k = 0;
  for (int bb = 0; bb < B; ++bb) {
    for (int x = 0; x < nt; ++x) out[k++] = bb * N + c->rank * nt + x;
    for (int x = 0; x < ni; ++x) out[k++] = bb * N + Nt + c->rank * ni + x;
  }
  return rows;
}
