// kernels.h -- internal launch interfaces of libdit (host side; no torch types).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dit {

// ------------------------------------------------------------------ GEMM (tcgen05)
// Tile 128 x 256 x 64, bf16 in, fp32 accumulate in TMEM, fused epilogues.
constexpr int GEMM_BM = 128;      // accumulator rows per CTA (= TMEM lanes)
constexpr int GEMM_TM = 256;      // rows per 2-SM (CTA pair) tile
constexpr int GEMM_BN = 256;
constexpr int GEMM_BK = 64;
constexpr int GEMM_MAX_PROBLEMS = 2;
constexpr int CN_FANIN = 2;   // ControlNet residuals summed per (request, block) (multi-ControlNet fan-in)
constexpr int MAX_SEQ = 16;   // B_max: sequences per dit_step (per-sequence parameter tables are sized by it)
#ifndef GEMM_GROUP_M_DEF
#define GEMM_GROUP_M_DEF 16
#endif
constexpr int GEMM_GROUP_M = GEMM_GROUP_M_DEF;   // rasterisation: tiles sweep all N within a group of M-tiles

enum EpiKind : int {
  EPI_STORE_H = 0,  // h[jrow][c] = acc + bias                (fp32, embeddings)
  EPI_QKV = 1,      // bias, QK-RMSNorm, RoPE, head-major scatter; cols >= qkv_cols -> GELU to out
  EPI_GELU = 2,     // out[r][out_col0 + c] = bf16(gelu_tanh(acc + bias))
  EPI_RESID = 3,    // h[jrow][c] += gate_b[c] * (acc + bias) (+ cn_scale_b * R_b[n][c])
  EPI_FINAL = 4,    // v = acc + bias; lat_out = lat_in + dsig_b * v
  EPI_SHRINK = 5,   // S[r][slot*r_alloc + c] = row_slot(r)==slot ? bf16(scale_slot*acc) : 0
  EPI_BIAS = 6,     // out[r][out_col0 + c] = bf16(acc + bias)  (plain projection; library-bar runs)
};

struct EpiParams {
  int kind;
  const void* bias;          // bf16 [N]
  // row map: local GEMM row r -> request b = r / rows_per_req, n = r % rows_per_req
  int rows_per_req;
  int joint_off;             // stream offset inside the joint (local) sequence
  int joint_n;               // local joint rows per request
  // fp32 residual stream h [B][joint_n][D]
  float* h;
  int D;
  const float* mod;          // modulation base [B][mod_stride]
  int mod_stride;
  int gate_off;              // column offset of the gate vector inside mod rows
  // ControlNet residual (EPI_RESID img stream)
  const void* const* cn_ptr; // device [CN_FANIN][MAX_SEQ] residual pointers (nullptr = none), bf16 [rows][D]
  const float* cn_scale;     // device [CN_FANIN][MAX_SEQ] kappa_b * inject scale
  int cn_row0;               // request-local row of residual row 0 (0: img-stream GEMM; Nt_loc: joint rows)
  const uint32_t* const* cn_flag;  // device [CN_FANIN][MAX_SEQ] ready flags (nullptr = resident / event-ordered)
  const uint32_t* cn_expect;       // device [CN_FANIN][MAX_SEQ] value the flag must reach
  const int* img_valid;            // device [MAX_SEQ] valid image rows per sequence (ragged batch; nullptr = all)
  // bf16 outputs
  void* out;
  int ld_out;
  int out_col0;
  // QKV scatter into the (SP send) layout [P][3][B][H/P][seq_len][d]; P = 1 is the
  // attention layout [3][B][H][N][d] itself.
  void* qkv;
  int batch;                 // B
  int sp_world;              // P
  const void* q_gamma;       // bf16 [d]
  const void* k_gamma;
  const float2* rope;        // [joint_n][d/2] (cos, sin) (+ b * rope_stride for a ragged batch)
  int rope_stride;           // float2 entries per sequence (0: one table shared by all sequences)
  int qkv_cols;              // 3D (columns beyond go to the GELU branch)
  int heads, head_dim;
  int seq_len;               // rows per (b, h) of q/k/v (= joint_n)
  // fused Ulysses exchange (qkv_peer[0] != nullptr): every q/k/v row is stored straight into
  // the attention buffer [3][B][H/P][P*seq_len][d] of the rank that owns its head
  // (qkv_peer[dest], peer-mapped), at its global joint position; no send buffer, no all-to-all
  void* qkv_peer[8];
  int sp_rank, sp_nt, sp_ni;  // this rank, local txt / img rows per request
  // final layer
  const float* lat_in;
  float* lat_out;
  float* v_out;
  float* v_peer;             // latent parallelism over peer memory: v also stored here (the peer's vcfg)
  const float* dsig;         // device [B] sigma_next - sigma
  // LoRA shrink
  const int* row_slot;       // device [M] pool slot of each row (-1 none)
  const float* slot_scale;   // device [max_adapters]
  int r_alloc;
};

struct GemmProblem {
  CUtensorMap tmA;       // A [M][K] bf16, box {64, 128}
  CUtensorMap tmB;       // B [N][K] bf16, box {64, 128} (each CTA of the pair loads half of N)
  CUtensorMap tmAx;      // LoRA K-extension A: S [M][slots*r_alloc], box {64, 128}
  CUtensorMap tmBx;      // LoRA K-extension B: pool viewed [slot*N][r_alloc], box {64, 128}
  CUtensorMap tmH;       // EPI_RESID: fp32 residual stream h [rows][D], box {32, 32} (TMA reduce-add)
  int tmH_ok;
  int M, N, K;
  int tiles_m, tiles_n;  // tiles_m: 256-row pair tiles
  int tile_begin;        // first global tile index of this problem
  int group_m;           // rasterisation group (M-tiles per N sweep; gemm_launch fills it)
  int num_tiles;
  // LoRA: per m-tile list of pool slots (device [tiles_m][slot_cap]) + counts
  const int* tile_slots;
  const int* tile_slot_cnt;
  int slot_cap;
  int ext_kblocks;       // k-blocks per slot (r_alloc / 64); 0 = no extension
  int shrink;            // 1: tiles enumerate (m_tile, slot) pairs from shrink_list
  const int2* shrink_list;  // device [num_tiles] (m_tile, slot)
  EpiParams epi;
  double rank_rows;      // host bookkeeping: sum over LoRA rows of the adapter rank (FLOP count)
};

struct GemmArgs {
  GemmProblem p[GEMM_MAX_PROBLEMS];
  int num_problems;
  int total_tiles;
};

// Encode a 2D/3D bf16 tensor map with SWIZZLE_128B (box inner = 64 elements).
bool make_tmap_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                  uint32_t box_inner, uint32_t box_outer);
// fp32 2D map, SWIZZLE_128B (box inner = 32 elements = 128 B)
bool make_tmap_2d_f32(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_outer);
bool make_tmap_3d(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1_bytes,
                  uint64_t stride2_bytes, uint32_t box0, uint32_t box1);

cudaError_t gemm_launch(const GemmArgs& args, int num_sms, cudaStream_t s);
// eager loading of each translation unit's kernels (common.cuh preload_module_of)
cudaError_t gemm_preload();
cudaError_t attention_tc_preload();
cudaError_t attention_mma_preload();
cudaError_t elementwise_preload();
cudaError_t merge_preload();
size_t gemm_smem_bytes();

// ------------------------------------------------------------------ attention
// q/k/v bf16 [B][H][N][d]; O rows written to out with the stream-split or joint map.
struct AttnParams {
  const void* q;
  const void* k;
  const void* v;
  int B, H, N, d;      // H = heads on this rank, N = full (global) joint sequence
  float scale_log2;    // log2(e) / sqrt(d)
  void* out;           // bf16
  int ld_out;          // elements per output row
  int split;           // 0 joint rows b*N+n; 1 stream-split (txt rows then img rows); 2 SP send layout
  int nt;              // txt rows per request (split: global Nt; SP: local nt)
  int ni;              // img rows per request (split: global Ni; SP: local ni)
  int Nt;              // global txt rows (SP mode)
  const int* seq_valid;  // device [B] valid joint rows per sequence (ragged batch; nullptr = N):
                         // keys beyond are masked, query rows beyond are written as zeros
  // split 3 = fused Ulysses exchange: O rows go straight to the owner rank's buffer
  // out_peer[dest] (peer-mapped) at its local row (out_split: 1 stream-split, 0 joint) and
  // columns (head_off + h) * d
  void* out_peer[8];
  int out_split;
  int head_off;
  // split tail (opt-in, attention_tc.cu TailSched): the last partial round's items split along the
  // keys; tail_ws = device fp32 [ATTN_TAIL_UNITS][2][128][d + 4] partials, tail_cnt = device u32
  // [ATTN_TAIL_UNITS * 2] merge counters (zero; the merging part resets them)
  int split_tail;
  float* tail_ws;
  uint32_t* tail_cnt;
};
constexpr int ATTN_TAIL_UNITS = 160;   // >= SMs: tail units never exceed the grid
inline size_t attn_tail_ws_bytes(int d) { return (size_t)ATTN_TAIL_UNITS * 2 * 128 * (d + 4) * 4; }
// Output row of query token n (global joint order) of request b; SP mode also
// returns the destination rank in *dest (rows are then [dest][B][N_loc]).
__host__ __device__ inline long long attn_out_row(const AttnParams& p, int b, int n) {
  if (p.split == 1)
    return (n < p.nt) ? (long long)b * p.nt + n : (long long)p.B * p.nt + (long long)b * p.ni + (n - p.nt);
  if (p.split == 2) {
    const int nloc = p.nt + p.ni;
    int dest, i;
    if (n < p.Nt) { dest = n / p.nt; i = n - dest * p.nt; }
    else { dest = (n - p.Nt) / p.ni; i = p.nt + (n - p.Nt) - dest * p.ni; }
    return ((long long)dest * p.B + b) * nloc + i;
  }
  return (long long)b * p.N + n;
}
cudaError_t attention_launch(const AttnParams& p, cudaStream_t s);

// ------------------------------------------------------------------ Ulysses SP index maps
// (host + device: the kernels use these, and dit_sp_layout exports them for tests)
// Global joint row (within one request) of rank rs's local row i (local rows: nt txt then ni img).
__host__ __device__ inline int sp_global_row(int P, int nt, int ni, int rs, int i) {
  return i < nt ? rs * nt + i : P * nt + rs * ni + (i - nt);
}
// d-vector index of (dest, sec, b, hl, i) in the QKV send layout [P][3][B][Hl][nloc].
__host__ __device__ inline long long sp_qkv_send_vec(int B, int Hl, int nloc, int dest, int sec, int b, int hl,
                                                     int i) {
  return (((long long)(dest * 3 + sec) * B + b) * Hl + hl) * nloc + i;
}
// d-vector index of (sec, b, hl, n) in the attention layout [3][B][Hl][N].
__host__ __device__ inline long long sp_attn_vec(int B, int Hl, int N, int sec, int b, int hl, int n) {
  return (((long long)sec * B + b) * Hl + hl) * N + n;
}
// Local output row of (b, i): split = 1 stream-split (txt rows of all requests first), 0 joint.
__host__ __device__ inline long long sp_local_row(int split, int B, int nt, int ni, int b, int i) {
  if (split) return (i < nt) ? (long long)b * nt + i : (long long)B * nt + (long long)b * ni + (i - nt);
  return (long long)b * (nt + ni) + i;
}

// Output address of (request b, global query n, local head h) for every split mode.
__host__ __device__ inline uint16_t* attn_out_addr(const AttnParams& p, int b, int n, int h, int hd) {
  if (p.split == 3) {
    int dest, i;
    if (n < p.Nt) { dest = n / p.nt; i = n - dest * p.nt; }
    else { dest = (n - p.Nt) / p.ni; i = p.nt + (n - p.Nt) - dest * p.ni; }
    const long long row = sp_local_row(p.out_split, p.B, p.nt, p.ni, b, i);
    return static_cast<uint16_t*>(p.out_peer[dest]) + row * p.ld_out + (long long)(p.head_off + h) * hd;
  }
  return static_cast<uint16_t*>(p.out) + attn_out_row(p, b, n) * p.ld_out + (long long)h * hd;
}

// Fused Ulysses exchange barrier over peer-mapped flags: signal stores epoch into every peer's
// flags[me] (fence.sys + st.release.sys, after the producing kernel on the same stream); wait
// spins (ld.acquire.sys, bounded -> trap) until flags[src] >= epoch for every peer src.
struct PeerFlags { uint32_t* f[8]; };
cudaError_t sp_signal_launch(const PeerFlags& peers, int me, int P, uint32_t epoch, cudaStream_t s);
cudaError_t sp_wait_launch(const uint32_t* flags, int me, int P, uint32_t epoch, cudaStream_t s);

// ------------------------------------------------------------------ Ulysses SP layout kernels
// recv [P][3][B][Hl][nloc][d] (chunk r_s = rank r_s's tokens, my heads) ->
// attention layout [3][B][Hl][N][d], global joint order (txt of all ranks, then img).
cudaError_t sp_gather_qkv_launch(const void* recv, void* out, int P, int B, int Hl, int nt_loc, int ni_loc, int d,
                                 cudaStream_t s);
// recv [P][B][nloc][Hl*d] (chunk r_s = heads of rank r_s for my tokens) -> rows of
// `out` (split = 1 stream-split rows, 0 joint rows b*nloc+i) at columns r_s*Hl*d.
cudaError_t sp_scatter_o_launch(const void* recv, void* out, int ld_out, int split, int P, int B, int Hl, int nt_loc,
                                int ni_loc, int d, cudaStream_t s);

// ------------------------------------------------------------------ elementwise / skinny
// u[r] = (1 + scale_b) * LN(h[jrow(r)]) + shift_b  (bf16 out), rows of up to 2 streams.
struct LnModParams {
  const float* h;
  int D;
  int joint_n;
  void* u;                 // bf16 [rows][D]
  const float* mod;
  int mod_stride;
  int nseg;
  int seg_rows[2];         // rows of each segment (stream)
  int seg_rows_per_req[2];
  int seg_joint_off[2];
  int seg_shift_off[2];    // column offsets of shift / scale inside mod rows
  int seg_scale_off[2];
  const float* seg_mod[2]; // per-segment modulation base (may differ per stream)
};
cudaError_t lnmod_launch(const LnModParams& p, cudaStream_t s);

// Merged LoRA (weight patching): out[o][i] = bf16(W[o][i] + scale * sum_k Bm[o][k] A[k][i]),
// W / out bf16 [rows][cols], Bm bf16 [rows][ra], A bf16 [ra][cols], ra a multiple of 16 (<= 128).
// Test/bench helper standing in for a remote ControlNet producer: after spinning `delay_ns`,
// copy `bytes` (multiple of 16) from src to dst and publish *flag = value with a system-scope
// release (so a consumer that acquires the flag sees the data).  One CTA.
cudaError_t delayed_publish_launch(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                                   uint64_t delay_ns, cudaStream_t s);
// ControlNet push (producer side, §8(f) f2): grid copy dst <- src (16-byte granules), then a
// one-thread kernel: fence.sys + st.release.sys *flag = value.
cudaError_t controlnet_push_launch(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                                   int num_sms, cudaStream_t s);
// Merged LoRA on the tensor cores (merge_tc.cu), one persistent launch over every adapted
// linear: the host fills one job per linear (merge_job_fill: w_map / out_map = the [rows][cols]
// box {64, 128} maps of W and of the output, tile_begin = running tile count) into device memory
// (merge_job_bytes each, 64-byte aligned); ra in {64, 128}.  Same result as lora_merge_launch.
// w / elem_base: the linear's weights and the index of its [0][0] in the concatenation of all
// adapted linears (undo-log addresses of the in-place merge).  mode: 0 merge into out, 1 count the
// elements the inverse cannot recover (*log_count +=), 2 merge in place (out = w) logging those
// elements (value << 48 | index) at log[atomicAdd(log_count)], 3 restore W = bf16(W' - s BA) in place.
size_t merge_job_bytes();
bool merge_job_fill(void* job, const CUtensorMap& w_map, const CUtensorMap& out_map, const void* A, const void* Bm,
                    int rows, int cols, int ra, float scale, int tile_begin, const void* w, long long elem_base);
int merge_job_tiles(const void* job);
cudaError_t lora_merge_tc_launch(const void* jobs_dev, int njobs, int total_tiles, int ra, int num_sms,
                                 cudaStream_t s, int mode = 0, unsigned long long* log = nullptr,
                                 unsigned long long* log_count = nullptr);
// after mode 3: rewrite the n logged elements exactly
cudaError_t restore_log_launch(const void* jobs_dev, int njobs, const unsigned long long* log, unsigned long long n,
                               int num_sms, cudaStream_t s);
cudaError_t lora_merge_launch(const void* W, const void* A, const void* Bm, void* out, int rows, int cols, int ra,
                              float scale, cudaStream_t s);

// out[b][n] (+)= sum_k x[b][k] * W[n][k] + bias[n] for b < B <= MAX_SEQ, with x bf16 [MAX_SEQ][K]
// (zero rows beyond B).  Segment table lets one launch cover many weights.
struct SkinnySeg {
  const void* w;       // bf16 [rows][K]
  const void* bias;    // bf16 [rows]
  int rows;
  int out_off;         // column offset into out rows
};
cudaError_t skinny_launch(const void* x, int K, const SkinnySeg* segs_dev, int nseg, int total_rows,
                          float* out, int out_stride, int B, int accumulate, cudaStream_t s);

// x_bf16[b][k] = bf16(act(x[b][k])) (act: 0 none, 1 SiLU), rows >= B zeroed (8 rows).
cudaError_t prep_x_launch(const float* x, int B, int K, int silu, void* out, cudaStream_t s);
// sinusoid embedding rows: out[b] = bf16([cos(1000 t w_k), sin(...)]), t = vals[b]; zero rows >= B.
cudaError_t temb_launch(const float* vals, int B, void* out, cudaStream_t s);
// rope table [n_rows][d/2] float2 from (Nt, img_w, first global joint row ...).
cudaError_t rope_table_launch(float2* tab, int nt_loc, int ni_loc, int nt_off, int ni_off, int img_w,
                              int a0, int a1, int a2, float theta, cudaStream_t s);
// SD3 2-D sincos position table added to the image rows of h [S][N][D] (reading C21).
cudaError_t pos_embed_add_launch(float* h, int S, int N, int nt, int ni, int ni_off, int img_h, int img_w, int D,
                                 int pe_max, int base, cudaStream_t s);
// CFG combine + Euler: v = vu + g_b (vc - vu), lat_out = lat_in + dsig_b v, v_out = v (nullable);
// per request b < B, count = Ni_loc * C fp32 (multiple of 4).
cudaError_t cfg_euler_launch(const float* vc, const float* vu, const float* g, const float* dsig, const float* lat_in,
                             float* lat_out, float* v_out, int B, int count, cudaStream_t s);
// x fp32 [n] -> bf16
cudaError_t cast_bf16_launch(const float* x, void* out, int64_t n, cudaStream_t s);
// ragged batch: latents [B][ni_pad][C] fp32 -> bf16, rows >= valid[b] (device) set to zero
cudaError_t cast_latents_ragged_launch(const float* x, void* out, int B, int ni_pad, int C, const int* valid,
                                       cudaStream_t s);
cudaError_t fill_synthetic_launch(void* dst, int64_t n, uint64_t seed, uint64_t tid, float scale, float offset,
                                  cudaStream_t s);

}  // namespace dit
