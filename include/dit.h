/*
 * dit.h -- C ABI of the B200-native denoise-step library (libdit.so).
 *
 * One call of dit_step() is one LegoDiffusion "model-execution node" of the
 * shared base diffusion model: execute(model_components, **kwargs) ->
 * {"noise_pred"} (Fig. flux_model_integration) over a
 * cross-workflow batch of up to B_max same-model nodes (PAPER.md:1152-1154,
 * :1178-1187), followed by denoise(noise_pred, latents).
 * The base model is a Flux-Dev-shaped MMDiT (the paper names Flux-Dev,
 * PAPER.md:154, :1306, but never defines it: DESIGN.md reading C1).
 *
 * Conventions
 *  - Every call returns an int status (DIT_OK = 0).  Every call validates ALL
 *    arguments before it enqueues any device work, so a failed call has no
 *    side effects.  dit_last_error() returns a human-readable reason.
 *  - Asynchronous device faults surface as DIT_ECUDA on the next call.
 *  - The CALLER owns all device memory (weights, workspace, inputs, outputs);
 *    the library never allocates device memory itself (NCCL internals aside).
 *  - A context is bound to one GPU and is not thread-safe: serialise calls.
 *  - Pointers documented "device" must be device-accessible; "host" pointers
 *    are read synchronously during the call and may be reused afterwards.
 *  - bf16 = IEEE bfloat16 stored as uint16; all matrices are row-major.
 *  - No C++ exceptions cross this boundary.
 */
#ifndef DIT_H_
#define DIT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum {
  DIT_OK = 0,
  DIT_EINVAL = 1,     /* bad argument / malformed tensor                        */
  DIT_ENOMEM = 2,     /* workspace too small                                   */
  DIT_ECUDA = 3,      /* CUDA runtime error (sticky for async faults)          */
  DIT_EEXIST = 4,     /* adapter id already registered (~DuplicateModelId)     */
  DIT_ERANK = 5,      /* LoRA rank > cfg.max_rank                              */
  DIT_ENOSPC = 6,     /* adapter pool full                                     */
  DIT_ENOENT = 7,     /* unknown adapter id                                    */
  DIT_EBATCH = 8,     /* B > B_max (~BatchExceedsMax)                          */
  DIT_ESHAPE = 9,     /* tokens exceed the configured maxima / not shardable   */
  DIT_EADAPTER = 10,  /* batch references an unregistered adapter              */
  DIT_EALIAS = 11,    /* latents_out aliases latents_in (immutability) */
  DIT_EPARALLEL = 12, /* world does not divide H, Nt, Ni (~ParallelismExceedsMax) */
  DIT_ENCCL = 13,     /* NCCL error                                            */
  DIT_ENOWEIGHTS = 14 /* dit_step before every base tensor was loaded          */
};

/* ------------------------------------------------------------------ config */
/* Model + capacity description (Model.__init__ / load). */
typedef struct dit_config {
  int32_t hidden;          /* D (3072)                                            */
  int32_t heads;           /* H (24); head dim d = D / H in {32, 64, 128}         */
  int32_t depth_double;    /* L_d double-stream blocks (19)                        */
  int32_t depth_single;    /* L_s single-stream blocks (38)                        */
  int32_t in_channels;     /* C packed latent channels (64)                        */
  int32_t txt_dim;         /* Ct text-embedding width (4096)                       */
  int32_t pooled_dim;      /* Cp pooled width (768)                                */
  int32_t mlp_ratio;       /* F = mlp_ratio * D (4)                                */
  int32_t rope_axes[3];    /* RoPE dims per position axis, sum = d (16, 56, 56)    */
  float rope_theta;        /* 10000                                                */
  int32_t guidance_embed;  /* 1 = guidance MLP present (Flux-Dev)                  */
  int32_t max_batch;       /* B_max sequences per dit_step, <= 16 */
  int32_t max_img_tokens;  /* largest Ni (global, before sharding)                */
  int32_t max_txt_tokens;  /* largest Nt (global, before sharding)                */
  int32_t max_rank;        /* largest LoRA rank (<= 128)                          */
  int32_t max_adapters;    /* adapter-pool slots (registered adapters)            */
  /* Model family (readings C1 / C21; the paper serves Flux-Dev, SD3 and
   * SD3.5-Large workflows, and loads
   * SD3Transformer2DModel at PAPER.md:841):
   *   DIT_ARCH_FLUX: depth_double double + depth_single single blocks, 3-axis RoPE.
   *   DIT_ARCH_SD3:  depth_double joint blocks (depth_single must be 0, no guidance
   *   embedding, rope_axes ignored); a 2-D sincos position table over a
   *   pos_embed_max^2 grid (positions * pos_embed_base / pos_embed_max, centre-
   *   cropped) is added to the embedded image tokens; the last block's text stream
   *   is context_pre_only (2-chunk (scale, shift) modulation, feeds attention only);
   *   final modulation (scale, shift).  qk_norm: 1 = per-head QK-RMSNorm with
   *   learned gamma (SD3.5), 0 = none (SD3-medium).  Ignored for Flux (always on). */
  int32_t arch;
  int32_t qk_norm;
  int32_t pos_embed_max;   /* 192 for SD3 / SD3.5                                 */
  int32_t pos_embed_base;  /* 64 for SD3 / SD3.5                                  */
  /* Sequence-parallel capacity of the workspace: 0 = default (the all-to-all send / recv
   * buffers, 16 B_max N D bytes, are carved; no cap on the world size), 1 = single GPU (no
   * exchange buffers: 1.8 GB less at Flux 1024^2 with B_max 8; sp_init with world > 1,
   * sp_init_local and sp_init_peers then fail with DIT_EPARALLEL), 2..64 = buffers carved,
   * worlds above the value refused with DIT_EPARALLEL. */
  int32_t max_sp_world;
} dit_config;

enum { DIT_ARCH_FLUX = 0, DIT_ARCH_SD3 = 1 };

typedef struct dit_ctx dit_ctx;

/* Device workspace bytes dit_create() needs for cfg at world size 1 (an upper
 * bound for any world size).  Returns 0 on an invalid cfg. */
size_t dit_workspace_bytes(const dit_config* cfg);

/* Create a context on CUDA device `device`, carving activations, the adapter
 * pool and the batch plan out of the caller-owned `workspace` (device,
 * >= dit_workspace_bytes(cfg) bytes, 256-B aligned).  *out is set on success.
 * Errors: DIT_EINVAL, DIT_ENOMEM, DIT_ECUDA. */
int dit_create(const dit_config* cfg, int device, void* workspace, size_t ws_bytes,
               dit_ctx** out);

void dit_destroy(dit_ctx* ctx);

/* Last error message of this context (or of the last failed dit_create when
 * ctx is NULL).  Never NULL. */
const char* dit_last_error(const dit_ctx* ctx);

/* ----------------------------------------------------------------- weights */
/* A named tensor handed across the boundary.  dtype: 0 = bf16 (the only one). */
typedef struct dit_tensor {
  const char* name;        /* e.g. "double.3.img.qkv.w" (synth.weight_manifest) */
  const void* ptr;         /* device pointer                                    */
  int32_t dtype;
  int32_t rank;            /* 1 or 2                                            */
  int64_t shape[4];
} dit_tensor;

/* load(): register the base weights.  Linear weights
 * are [out][in] row-major (K-major), biases [out]; names and shapes are those
 * of synth.weight_manifest(cfg).  BORROWED: must outlive the context and stay
 * unchanged.  May be called several times (later tensors replace earlier).
 * Errors: DIT_EINVAL (unknown name, wrong shape/dtype, duplicate in one call,
 * or an adapter is merged: lora_unmerge first). */
int dit_load_weights(dit_ctx* ctx, const dit_tensor* tensors, int n);

/* ------------------------------------------------------------------- LoRA */
/* add_patch(lora): copy adapter
 * `adapter_id` into the pool, enqueued on `stream` (a cudaStream_t).
 * tensors: "<module>.lora_A" [r][in] and "<module>.lora_B" [out][r] for every
 * adapted linear (synth.lora_targets: double qkv/proj/fc1/fc2 per stream,
 * single linear1/linear2), in device memory OR pinned host memory (copied with
 * cudaMemcpyDefault).  Missing modules are treated as zero (no delta).
 * Applied unmerged: y += scale * (x A^T) B^T (reading C9).
 * Asynchronous loading: `stream` may be a side
 * stream while steps run on another; every later dit_step that uses the adapter
 * waits for the copies on ITS OWN stream (an event, no host stall), so the
 * adapter can be registered the moment it arrives and used by the next step.
 * Caller buffers may be freed once `stream` has synchronised.
 * Errors: DIT_EEXIST, DIT_ERANK, DIT_ENOSPC, DIT_EINVAL. */
int lora_register(dit_ctx* ctx, int32_t adapter_id, int32_t rank, float scale,
                  const dit_tensor* tensors, int n, void* stream);

/* rm_patch: waits for the adapter's last use, frees the slot.
 * Errors: DIT_ENOENT. */
int lora_unregister(dit_ctx* ctx, int32_t adapter_id);

/* ---------------------------------------------------- merged LoRA (hot patch) */
/* Weight patching (adapters "patch the base model's weights
 * before inference, incurring no additional computational overhead"; hot-patch
 * at a step boundary once an asynchronously loaded adapter arrives,
 * PAPER.md:391-400).  lora_merge writes W' = bf16(W + scale * B A) of EVERY
 * adapted linear (same set as lora_register) for the registered adapter
 * `adapter_id` into `merged` and makes the ctx run those linears from W';
 * enqueued on `stream` (a cudaStream_t).  `merged`: caller-owned device memory,
 * >= dit_merge_bytes(cfg), 256-byte aligned, layout = the adapted linears in
 * pool order, each [out][in] bf16 at a 256-byte aligned offset; it must stay
 * alive until lora_unmerge.  The base weights are never written, so
 * lora_unmerge restores them exactly (a pointer switch).  `stream` may be a side
 * stream: the merge waits for the adapter's registration copies and for the last
 * step that read a previous merged copy, and every later dit_step waits for the
 * merge on its own stream (events, no host stall).  While an adapter is
 * merged the ctx is a patched replica specialised to it:
 * every request of a dit_step must name that adapter (else DIT_EADAPTER) and
 * no per-step LoRA work runs; it cannot be unregistered.
 * Errors: DIT_ENOENT (not registered), DIT_EEXIST (an adapter is already
 * merged), DIT_ENOMEM (buffer too small), DIT_EINVAL (NULL / misaligned),
 * DIT_ENOWEIGHTS, DIT_ECUDA.  Validation precedes any enqueue. */
size_t dit_merge_bytes(const dit_config* cfg);
int lora_merge(dit_ctx* ctx, int32_t adapter_id, void* merged, size_t bytes, void* stream);
/* In-place hot patch ("hot-patch the base model in GPU memory";
 * :1504-1509): W' = bf16(W + scale * B A) is written OVER the base weights of every
 * adapted linear -- no second copy.  For an exact restore the merge logs, into the
 * caller's device buffer `undo` (8-byte aligned, 8 bytes per entry), every element
 * whose original value the inverse bf16(W' - scale * B A) would not give back
 * (rounding W + d lost bits: W' in a higher binade than W, or a tie); lora_unmerge
 * then applies the inverse everywhere and rewrites the logged elements, so the
 * weights come back bit for bit.  The merge runs two passes on `stream`: a count
 * (the host waits for it: *undo_entries receives the entries needed), then, only
 * if entries * 8 <= undo_bytes, the patch (else DIT_ENOMEM and nothing is
 * written).  It waits for every dit_step enqueued before it (they read the base
 * weights); steps after it wait for it (events).  The borrowed base weights ARE
 * MODIFIED until lora_unmerge; dit_load_weights is refused meanwhile.  Otherwise as
 * lora_merge (a patched replica serving one adapter).  Errors: as lora_merge, plus
 * DIT_ENOMEM (undo log too small), DIT_EINVAL (max_rank not 64 or 128 after
 * padding / misaligned undo). */
int lora_merge_inplace(dit_ctx* ctx, int32_t adapter_id, void* undo, size_t undo_bytes,
                       uint64_t* undo_entries, void* stream);
/* Restore the base weights.  Waits (host) for the last enqueued dit_step that
 * read the merged weights, so `merged` may be freed once this returns; after an
 * in-place merge it also restores the weights (inverse + undo log, on the legacy
 * default stream, synchronised) before returning.
 * Errors: DIT_ENOENT (nothing merged), DIT_ECUDA. */
int lora_unmerge(dit_ctx* ctx);

/* -------------------------------------------------------------- ControlNet */
/* Deferred input "controlnet_inputs": register the
 * residual of request `slot` of the NEXT dit_step for block `block`:
 * block in [0, L_d) = double block `block`, [L_d, L_d + L_s) = single block
 * `block - L_d` (ControlNets feed "specific layers"; reading
 * C20).  After that block, h_img[slot] += cn_scale[slot] * scale * residual (for
 * a single block: the image rows of the joint sequence).  Up to CN_FANIN = 2
 * residuals may be registered per (slot, block) -- several ControlNets feeding
 * one block (fan-in); they are summed.
 * residual: device bf16 [Ni_local][D] row-major (this rank's image shard).
 * ready: a cudaEvent_t recorded by the producer, or NULL if already
 * resident.  The step does NOT wait at launch: the wait is enqueued right
 * before block `block`'s consuming kernel ("returns immediately if the data is
 * available, or blocks until the data arrives").
 * BORROWED and immutable until that dit_step completes.
 * Registrations apply to exactly one dit_step CALL and are cleared when it
 * returns, whatever its status (a failed step never leaves stale pointers).
 * Errors: DIT_EINVAL (slot >= B_max, block >= L_d + L_s, NULL or misaligned
 * residual), DIT_ENOSPC (fan-in limit reached for this slot and block). */
int controlnet_inject(dit_ctx* ctx, int32_t slot, int32_t block, const void* residual,
                      float scale, void* ready_event);

/* Drop every ControlNet registration made since the last dit_step (a scheduler
 * that cancels a request before stepping).  Errors: DIT_EINVAL (NULL ctx). */
int controlnet_clear(dit_ctx* ctx);

/* controlnet_inject with the readiness carried by a DEVICE FLAG instead of a
 * CUDA event -- the data engine's deferred fetch done in hardware
 * (SURVEY.md §8(f) f2): the producer (another stream, or
 * another GPU writing `residual` into this GPU's memory over NVLink) writes the
 * residual and then stores *flag = value >= expect with release semantics at
 * system scope; the consuming GEMM epilogue acquires *flag >= expect before it
 * reads the residual (no host synchronisation, no event).  flag: 4-byte aligned
 * device (or peer / host-mapped) memory, read with ld.acquire.sys.  A flag that
 * never reaches `expect` traps after a few seconds (sticky DIT_ECUDA) rather
 * than hanging.  The producer must not depend on this step.
 * Errors: as controlnet_inject, plus DIT_EINVAL (NULL / misaligned flag). */
int controlnet_inject_flag(dit_ctx* ctx, int32_t slot, int32_t block, const void* residual,
                           float scale, const uint32_t* flag, uint32_t expect);

/* --------------------------------------------- ControlNet producer side (f2) */
/* The data engine's push half: a
 * ControlNet executor on another GPU or in another process writes each residual
 * straight into the DiT's registered buffer and releases a ready flag, which the DiT's
 * consuming GEMM epilogue acquires (controlnet_inject_flag) -- deferred fetch with no
 * host round trip.  controlnet_push copies `bytes` (multiple of 16, 16-byte aligned)
 * from `src` to `dst` with a grid of CTAs (dst may be a peer GPU's memory mapped by
 * cudaDeviceEnablePeerAccess / dit_ipc_open: the stores travel over NVLink), then a
 * second kernel stores *flag = value with a system-scope release after the copy
 * (stream order + fence.sys).  Enqueued on `stream`; nothing is read back.
 * Errors: DIT_EINVAL (NULL / misaligned / bytes % 16), DIT_ECUDA. */
int controlnet_push(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value, void* stream);

/* Inter-process export / import of a device buffer (residuals and flags of another
 * executor).  A handle is DIT_IPC_HANDLE_BYTES opaque bytes: the CUDA IPC handle of the
 * allocation containing dev_ptr plus dev_ptr's offset inside it, so interior pointers of
 * a caching allocator work.  dit_ipc_open maps it into this process (*out = the same
 * byte the exporter named); dit_ipc_close unmaps.  The exporter must keep the
 * allocation alive while it is open elsewhere.  Errors: DIT_EINVAL, DIT_ECUDA. */
#define DIT_IPC_HANDLE_BYTES 72
int dit_ipc_export(const void* dev_ptr, void* handle_out);
int dit_ipc_open(const void* handle, void** out);
int dit_ipc_close(void* dev_ptr);

/* ------------------------------------------------------ sequence parallel */
/* Parallelism descriptor: this context is rank `rank` of
 * `world` GPUs running one dit_step together with Ulysses sequence
 * parallelism.  At world > 1 it also maps every peer's workspace (CUDA IPC handles
 * all-gathered over the new communicator) so the exchange is fused into the
 * epilogues (dit_sp_exchange); if any rank cannot map, all ranks use NCCL all-to-alls.  nccl_unique_id: 128-byte ncclUniqueId (host), identical on all
 * ranks (broadcast by the caller).  Collective: every rank must call it.
 * world == 1 disables communication.  Shard layout (bit-exact):
 * rank r owns, of every request, txt rows [r*Nt/P, (r+1)*Nt/P) and img rows
 * [r*Ni/P, (r+1)*Ni/P); latents / txt / residuals are passed pre-sharded.
 * Errors: DIT_EPARALLEL (world does not divide H), DIT_ENCCL, DIT_EINVAL. */
int sp_init(dit_ctx* ctx, int32_t world, int32_t rank, const void* nccl_unique_id);

/* Bring-your-own-transport variant of sp_init (no NCCL): every rank calls
 * dit_peer_handle (which also resets this context's arrival flags, so it must
 * precede any peer's first dit_step), the caller all-gathers the
 * DIT_PEER_HANDLE_BYTES-byte handles by any means (a serving control plane, a
 * gloo group, a file), and every rank then calls sp_init_peers with all of them
 * in rank order (host, world x DIT_PEER_HANDLE_BYTES).  The fused exchange
 * (dit_sp_exchange == 2) is then the only exchange: there is no all-to-all
 * fallback.  Works across processes on one GPU too (the tests' cross-process
 * check of the system-scope flag protocol).
 * Errors: DIT_EINVAL (world not in [2, 8], bad rank, NULL), DIT_EPARALLEL,
 * DIT_ECUDA (a peer's workspace cannot be mapped, or the configs differ). */
#define DIT_PEER_HANDLE_BYTES 80
int dit_peer_handle(dit_ctx* ctx, void* handle_out);
int sp_init_peers(dit_ctx* ctx, int32_t world, int32_t rank, const void* handles);

/* ------------------------------------------------------ latent parallelism */
/* Latent (CFG) parallelism (the conditional and unconditional
 * passes of classifier-free guidance on separate GPUs, with a scatter-gather of the
 * partial results at every denoising step).  This context becomes rank `rank` of
 * `world` = 2 GPUs: rank 0 computes every request's conditional pass, rank 1 its
 * unconditional pass; after the final layer the two ranks exchange their v
 * (ncclAllGather, B*Ni*C fp32 per rank) and BOTH apply the guided Euler update, so
 * latents_out is identical on both ranks.  Each rank passes the full latents and
 * its own branch's txt / pooled; batch.cfg_scale must be non-NULL.  Collective:
 * both ranks call it and then every dit_step together.  Exclusive with sp_init.
 * Errors: DIT_EPARALLEL (world != 2, or sp_init already active), DIT_ENCCL,
 * DIT_EINVAL. */
int lp_init(dit_ctx* ctx, int32_t world, int32_t rank, const void* nccl_unique_id);
/* lp_init also maps the peer's workspace through CUDA IPC (handles all-gathered
 * over the new communicator): the final GEMM's epilogue then stores this rank's v
 * straight into the peer's buffer as well and a device flag barrier replaces the
 * all-gather (dit_sp_exchange == 2; 1 = ncclAllGather, forced by DIT_SP_NCCL=1).
 * lp_init_peers is its bring-your-own-transport variant (see sp_init_peers):
 * handles = both ranks' dit_peer_handle outputs in rank order. */
int lp_init_peers(dit_ctx* ctx, int32_t world, int32_t rank, const void* handles);
/* Test analogue of lp_init over an in-process group (dit_local_group_create(2)). */
int lp_init_local(dit_ctx* ctx, void* group, int32_t rank);

/* -------------------------------------------------------------------- step */
typedef struct dit_batch {
  int32_t batch;              /* B (1 .. B_max)                                  */
  int32_t img_h, img_w;       /* packed latent grid; Ni = img_h * img_w (global) */
  int32_t txt_tokens;         /* Nt (global)                                     */
  const int32_t* adapter_id;  /* host [B]; -1 = base model                       */
  const float* sigma;         /* host [B]; this step's sigma per request         */
  const float* sigma_next;    /* host [B]                                        */
  const float* guidance;      /* host [B] (Flux-Dev distilled guidance, 3.5)     */
  const float* cn_scale;      /* host [B] ControlNet conditioning scale; NULL=1  */
  const float* latents_in;    /* device fp32 [B][Ni/P][C]                        */
  float* latents_out;         /* device fp32 [B][Ni/P][C]; must NOT alias input  */
  const void* txt;            /* device bf16 [B][Nt/P][Ct]                       */
  const void* pooled;         /* device bf16 [B][Cp]                             */
  float* v_out;               /* device fp32 [B][Ni/P][C] noise_pred; nullable   */
  /* Classifier-free guidance (reading C22).  NULL = one
   * pass per request.  Non-NULL: host [B] guidance scales g_b; every request runs a
   * conditional and an unconditional SEQUENCE and
   *   v_b = v_uncond + g_b (v_cond - v_uncond),  latents_out = latents_in + dsig v_b.
   * Without latent parallelism the step runs 2B sequences (2B <= B_max, else
   * DIT_EBATCH): txt is then [2B][Nt][Ct] and pooled [2B][Cp] -- the B conditional
   * prompts, then the B unconditional ones -- and ControlNet slot s < B feeds request
   * s's conditional pass, slot B + s its unconditional pass.  Under lp_init (one
   * branch per GPU) txt / pooled are [B] rows of THIS rank's branch (rank 0
   * conditional, rank 1 unconditional) and slots are request indices.  v_out, when
   * given, receives the guided v. */
  const float* cfg_scale;
  /* Ragged batch (mixed resolutions, reading C24).  NULL =
   * every request uses img_h x img_w.  Non-NULL: host [B][2], request b's own packed
   * grid (h_b, w_b) with h_b * w_b <= img_h * img_w; img_h x img_w is then the PADDED
   * slot size: latents_in / latents_out / v_out stay [B][img_h*img_w][C] and request b's
   * tokens are its first h_b * w_b rows (rows beyond are ignored on input and
   * unspecified on output); ControlNet residuals of request b are [h_b*w_b][D].  Each
   * request's result equals running it alone at its own grid (keys of the padding are
   * masked out of attention).  Sequence parallelism must be off (DIT_EPARALLEL). */
  const int32_t* img_hw;
} dit_batch;

/* execute() + denoise(): one flow-matching Euler step
 * latents_out = latents_in + (sigma_next - sigma) * v for every request,
 * asynchronously on `stream` (a cudaStream_t).  All pointers are borrowed.
 * Errors: DIT_EBATCH, DIT_ESHAPE (also: an SD3 token grid larger than
 * pos_embed_max), DIT_EADAPTER, DIT_EALIAS, DIT_EINVAL (also: lp_init active and
 * cfg_scale NULL), DIT_ENOWEIGHTS, DIT_ECUDA, DIT_ENCCL. */
int dit_step(dit_ctx* ctx, const dit_batch* batch, void* stream);

/* ------------------------------------------------------------- CUDA graphs */
/* dit_graph_create captures ONE dit_step on `batch` (shape, adapter ids, device
 * pointers, and the ControlNet registrations made before it -- slots, blocks,
 * ready events) on `stream` (a non-default cudaStream_t) into an instantiated CUDA
 * graph; nothing executes.  Every host->device upload of the step (plan tables,
 * per-step scalars, ControlNet tables) is a copy node reading the graph's own
 * pinned block.  dit_graph_launch replays it: it re-runs the step's host logic
 * on `batch` in staging mode (validation, sigma / sigma_next / guidance / CFG and
 * ControlNet scales, residual pointers -> the block; the registrations are then
 * cleared, as by dit_step), then cudaGraphLaunch -- one launch instead of ~450.
 * `batch` must match the captured one in shape, adapter ids and device pointers,
 * and the ControlNet registrations in (slot, block, event) (else DIT_EINVAL);
 * the host stays at most one replay ahead of the device.  Adapters must be
 * registered (or merged) before the capture; replays wait on their events.
 * Not capturable (DIT_EPARALLEL / DIT_EINVAL): in-process groups, the fused peer
 * exchanges (their epochs are per launch), device-flag ControlNet inputs.
 * A graph is bound to its ctx; destroy it before the ctx. */
typedef struct dit_graph dit_graph;
int dit_graph_create(dit_ctx* ctx, const dit_batch* batch, void* stream, dit_graph** out);
int dit_graph_launch(dit_graph* graph, const dit_batch* batch, void* stream);
void dit_graph_destroy(dit_graph* graph);

/* Algorithmic tensor FLOPs of one dit_step on `batch` (DESIGN.md §5 formula:
 * projections 2MNK, attention 4 N^2 D per request-block, LoRA 2r(in+out)). */
double dit_step_flops(const dit_ctx* ctx, const dit_batch* batch);

/* Number of kernels the last dit_step launched (for bench.py gpu_launches). */
int dit_last_launch_count(const dit_ctx* ctx);

/* Sequence-parallel exchange in use: 0 none (world 1), 1 NCCL all-to-all + gather/scatter
 * kernels, 2 fused -- the QKV and attention epilogues store straight into the owning rank's
 * buffers (peer-mapped over NVLink through CUDA IPC) behind device flag barriers (the
 * default when every rank can map every peer; DIT_SP_NCCL=1 forces 1).  Under latent
 * parallelism: 1 = ncclAllGather of v (or the in-process group), 2 = v stored into the
 * peer by the final GEMM's epilogue. */
int dit_sp_exchange(const dit_ctx* ctx);

/* ------------------------------------------------------ profiling exports */
/* Per-launch device timing for bench.py's roofline (CUDA events recorded on
 * the launch stream around every kernel while enabled).  kind: 0 tcgen05
 * GEMM (all projections, LoRA shrink/expand), 1 attention, 2 LN-modulate,
 * 3 modulation skinny GEMM, 4 other small kernels, 5 SP all-to-all (NCCL),
 * 6 SP layout gather/scatter kernels; GEMM sub-kinds (included in 0):
 * 10 embeddings, 11 double QKV, 12 double proj, 13 double fc1, 14 double fc2,
 * 15 single linear1, 16 single linear2, 17 final, 18 LoRA shrink.  dit_profile_read
 * synchronises on the recorded events and returns the summed device time,
 * the summed ALGORITHMIC flops and the number of launches of that kind since
 * the last dit_profile_reset. */
int dit_profile(dit_ctx* ctx, int enable);
int dit_profile_read(dit_ctx* ctx, int kind, double* total_ms, double* flops, int* launches);
int dit_profile_reset(dit_ctx* ctx);

/* ---------------------------------------------------- test-only exports */
/* Fill a device bf16 tensor of n elements with the synth counter generator
 * (synth/__init__.py docstring): w = bf16(offset + (2u-1)*scale). */
int dit_fill_synthetic(void* dst_bf16, int64_t n, uint64_t seed, uint64_t tensor_id,
                       float scale, float offset, void* stream);

/* In-process communicator for tests (one host thread per rank, all ranks'
 * contexts in this process): the SP all-to-all becomes event-ordered device
 * copies.  Lets the exact sequence-parallel kernels and layouts be exercised
 * on a single GPU.  sp_init_local is the test analogue of sp_init. */
void* dit_local_group_create(int32_t world);
void dit_local_group_destroy(void* group);
int sp_init_local(dit_ctx* ctx, void* group, int32_t rank);

/* Bench/test-only: one attention launch, q/k/v device bf16 [B][H][N][d]
 * head-major, O bf16 [B*N][H*d] (joint rows).  Asynchronous on stream. */
int dit_debug_attention(const void* q, const void* k, const void* v, int32_t B, int32_t H, int32_t N, int32_t d,
                        void* out, void* stream);

/* Bench/test-only: dit_debug_attention with the split tail chosen explicitly (split_tail = 1:
 * when the persistent grid's last round of work items is at most half full, each tail item's keys
 * are split into 2-4 parts whose partial O / max / sum a last part merges in part order --
 * deterministic, within fp32 rounding of the unsplit result; 0: never).  dit_step uses it when
 * the context was created with DIT_ATTN_SPLIT_TAIL=1 (opt-in: the tail items' rounding then
 * depends on the batch composition, so bitwise batch invariance no longer holds for them).
 * Asynchronous on stream. */
int dit_debug_attention_ex(const void* q, const void* k, const void* v, int32_t B, int32_t H, int32_t N, int32_t d,
                           void* out, int32_t split_tail, void* stream);

/* Bench/test-only: out = bf16(A W^T + bias) through the step's tcgen05 GEMM (A [M][K],
 * W [N][K], bias [N], out [M][N], all device bf16; K % 64 == 0).  Asynchronous on stream. */
int dit_debug_gemm(const void* A, const void* W, const void* bias, void* out, int32_t M, int32_t N, int32_t K,
                   void* stream);

/* Bench-only: h[M][N] (device fp32) += gate[N] (device fp32) * (A W^T + bias) through the step's
 * GEMM with its gated-residual epilogue (N % 32 == 0).  Asynchronous on stream. */
int dit_debug_gemm_resid(const void* A, const void* W, const void* bias, float* h, const float* gate, int32_t M,
                         int32_t N, int32_t K, void* stream);

/* Debug-only: record a clock64 timeline of CTA 0's first work item of the
 * tcgen05 attention kernel into buf (device int64 [20 events][64 kv tiles]);
 * NULL disables (the default). */
int dit_debug_attention_trace(void* buf);

/* Test-only stand-in for a remote ControlNet producer: after `delay_ns`, one CTA
 * copies `bytes` (multiple of 16, 16-byte aligned) from src to dst and then
 * publishes *flag = value (st.release.sys).  Enqueued on `stream`. */
int dit_debug_delayed_publish(void* dst, const void* src, size_t bytes, uint32_t* flag, uint32_t value,
                              uint64_t delay_ns, void* stream);

/* Test-only stand-in for a slow producer that occupies no SM: stalls `stream` for
 * delay_ns on the host (cudaLaunchHostFunc + nanosleep); later work on that stream
 * (a copy, an event record) starts after it. */
int dit_debug_host_delay(void* stream, uint64_t delay_ns);

/* ncclGetUniqueId for sp_init (rank 0 calls it, the caller broadcasts the 128 bytes). */
int dit_nccl_unique_id(void* out128);

/* Host copy of the sequence-parallel index maps the kernels use (bit-exact
 * layout tests, no GPU needed).  which: 0 shard map (local row -> global joint
 * row b*N+n), 1 QKV send layout, 2 gather (recv -> attention layout), 3 O send
 * rows, 4 O scatter rows (stream-split); fused exchange: 5 QKV peer stores
 * (dest * 3BHlN + attention-buffer index), 6 O peer stores (dest * 2^40 +
 * row * H + global head of the stream-split O buffer).  Writes up to cap int64 entries to
 * out; returns the number of entries, or -status. */
int64_t dit_sp_layout(int32_t which, int32_t world, int32_t rank, int32_t B, int32_t H, int32_t Nt, int32_t Ni,
                      int64_t* out, int64_t cap);

/* Integer plan artefacts of `batch` (host outputs; bit-exact tests):
 * row_adapter: int32 [rows] LoRA pool slot of each local row of the
 *   txt-stream GEMM followed by the img-stream GEMM (-1 = none), computed by the
 *   step's own planner without running a step; rows = S*(Nt/P) + S*(Ni/P), S =
 *   sequences (2B with CFG on one GPU).  Returns rows written, or -status. */
int dit_debug_row_adapter(dit_ctx* ctx, const dit_batch* batch, int32_t* out, int cap);
/* The integer tables the LAST dit_step uploaded for row space `which` (0 txt
 * stream GEMM rows, 1 img stream, 2 joint sequence of the single blocks), read
 * back from the device -- exactly what the GEMM / shrink kernels consumed: kind
 * 0 row -> adapter-pool slot int32 [M] (-1 none), 1 tile -> its distinct slots
 * sorted ascending [tiles_m][B_max] (256-row tiles; unused entries 0), 2 distinct
 * slots per tile [tiles_m], 3 the LoRA shrink work list of (tile, slot) pairs
 * [n_shrink][2] in tile order.  Returns entries written, or -status (-DIT_ENOENT
 * before the first dit_step).  Synchronous, test-only. */
int dit_debug_plan(dit_ctx* ctx, int32_t which, int32_t kind, int32_t* out, int cap);
/* shard_map: int32 [B*(Nt/P + Ni/P)]: global joint token index (txt first,
 * request-major: b*N + n) of every local row.  Returns rows, or -status. */
int dit_debug_shard_map(dit_ctx* ctx, const dit_batch* batch, int32_t* out, int cap);

#ifdef __cplusplus
}
#endif
#endif /* DIT_H_ */
