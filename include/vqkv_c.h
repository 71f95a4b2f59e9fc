/*
 * vqkv_c.h -- C-ABI of the B200-native VQKV hot path (libvqkv_b200.so).
 *
 * Plain pointers and sizes only; no torch, no Eigen, no exceptions cross this
 * boundary.  Every call returns an int status (VQKV_OK == 0) whose non-zero
 * values mirror the exception kinds of proj/core/include/vqkv/errors.hpp:12-49;
 * vqkv_last_error() returns the thread-local message.  The C++ mirror in
 * include/vqkv/ headers rethrows the matching vqkv:: exception.
 *
 * Each entry point replaces one reference interface (proj/core/...):
 *   vqkv_stack_create      <- load_stack + Codebook::refresh   (codebook.cpp:30-39, 277-316)
 *   vqkv_quantize_batch    <- quantize_batch                   (codebook.cpp:225-237)
 *   vqkv_reconstruct_block <- reconstruct_block                (codebook.cpp:239-250)
 *   vqkv_attend_decode     <- attend over CacheState segments  (attention.cpp:26-69,
 *                                                               kv_cache.cpp:143-189)
 *   vqkv_lse_combine       <- (new) merge of sequence-split partial attention
 *
 * Device pointers ("_dev") live on the stack's device; the work is enqueued
 * on `stream` (a cudaStream_t passed as void*, NULL = legacy default stream)
 * and is asynchronous.  Stacks are immutable after creation, so any number of
 * host threads / streams may use one stack concurrently (codebook.hpp:45-46).
 *
 * Batching: the reference API quantizes one (layer, head) stream per call; a
 * single stream cannot fill a B200, so the batched entry points take
 * n_streams independent streams of rows_per_stream rows each, laid out
 * contiguously.  Each stream's codes are a CodeMatrix payload
 * (codebook.cpp:74-151: LSB-first bit stream, ceil(log2 S_i) bits per stage,
 * rows back to back) of vqkv_payload_bytes(stack, rows_per_stream) bytes, and
 * the streams' payloads are concatenated.  The bytes are identical to
 * CodeMatrix::payload() of the reference.
 */
#ifndef VQKV_C_H
#define VQKV_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum vqkv_status {
    VQKV_OK = 0,
    VQKV_INVALID_INPUT = 1,   /* vqkv::InvalidInput  */
    VQKV_INVALID_STATE = 2,   /* vqkv::InvalidState  */
    VQKV_INVALID_CODE = 3,    /* vqkv::InvalidCode   */
    VQKV_FORMAT_ERROR = 4,    /* vqkv::FormatError   */
    VQKV_IO_ERROR = 5,        /* vqkv::IoError       */
    VQKV_CUDA_ERROR = 6,      /* CUDA runtime / launch failure */
    VQKV_UNSUPPORTED = 7      /* shape the device path does not implement */
};

enum vqkv_cache_kind { VQKV_KEY = 0, VQKV_VALUE = 1 };

typedef struct vqkv_stack_s* vqkv_stack_t;

const char* vqkv_last_error(void);
const char* vqkv_version(void);

/* ---------------------------------------------------------------------------
 * Codebook stacks.  entries: host fp32, stage-major concatenation of the
 * S_i x D raw entry matrices (row-major); projections: host fp32, N x D x D
 * (row-major), or NULL for identity.  Effective entries
 * (entries . projection^T) and their squared norms are computed ON THE
 * DEVICE with the reference's fp32 operation order (codebook.cpp:30-39), so
 * every kernel and the host see bit-identical codebooks.
 * ------------------------------------------------------------------------- */
int vqkv_stack_create(int device, int kind, uint32_t n_stages, const uint32_t* sizes, uint32_t dim,
                      const float* entries, const float* projections, vqkv_stack_t* out);
int vqkv_stack_destroy(vqkv_stack_t stack);
int vqkv_stack_describe(vqkv_stack_t stack, uint32_t* n_stages, uint32_t* dim, uint64_t* row_bits,
                        int* kind, int* device);
int vqkv_stack_stage_size(vqkv_stack_t stack, uint32_t stage, uint32_t* size);
/* download effective entries (S x D) and squared norms (S) of one stage to host */
int vqkv_stack_effective(vqkv_stack_t stack, uint32_t stage, float* effective_host, float* sqnorm_host);
/* device pointer of a stage's fp32 effective entries (read-only) */
int vqkv_stack_effective_dev(vqkv_stack_t stack, uint32_t stage, const float** effective_dev);
/* CodeMatrix payload size for `rows` rows: ceil(rows * row_bits / 8) */
uint64_t vqkv_payload_bytes(vqkv_stack_t stack, uint64_t rows);
/* Returns and clears the sticky device-side error of the stack (out-of-range
 * codes seen by a decode); VQKV_OK if none.  Synchronizes the device. */
int vqkv_stack_take_error(vqkv_stack_t stack);

/* ---------------------------------------------------------------------------
 * Encode: quantize_batch over n_streams x rows_per_stream rows of dim D
 * (xs_dev fp32 [n_streams][rows][D]).  Writes the concatenated payloads and
 * residual_norms_dev [n_streams][rows] (||x - reconstruct(codes)||, fp32).
 * search_block: the reference's nearest-search block (codebook.hpp:25,
 * default 4096); it never changes results but selects the reference's
 * dot-product order for length-1 blocks, which this path reproduces.
 * ------------------------------------------------------------------------- */
int vqkv_quantize_batch(vqkv_stack_t stack, const float* xs_dev, uint32_t n_streams,
                        uint64_t rows_per_stream, uint64_t search_block, uint8_t* payload_dev,
                        float* residual_norms_dev, void* stream);
/* As vqkv_quantize_batch, additionally writing the final residual vectors
 * (x - e_0[z_0] - e_1[z_1] - ..., in stage order, fp32 [n_streams][rows][D])
 * when residuals_dev is not NULL -- QuantizeResult::final_residual of
 * codebook.hpp:103-106. */
int vqkv_quantize_batch_ex(vqkv_stack_t stack, const float* xs_dev, uint32_t n_streams,
                           uint64_t rows_per_stream, uint64_t search_block, uint8_t* payload_dev,
                           float* residual_norms_dev, float* residuals_dev, void* stream);
/* nearest_entry over one stage for `rows` vectors (codebook.cpp:180-192):
 * index_dev[r] = argmin, distance_dev[r] = sqrt(max(0, score + ||x||^2)).
 * Non-finite inputs are the caller's to reject (the reference throws). */
int vqkv_nearest_batch(vqkv_stack_t stack, uint32_t stage, const float* xs_dev, uint64_t rows,
                       uint64_t search_block, uint32_t* index_dev, float* distance_dev, void* stream);
/* Same contract with HOST buffers: copies in, encodes, copies out (pinned
 * staging, chunked and overlapped).  Blocks until the results are on the host. */
int vqkv_quantize_batch_host(vqkv_stack_t stack, const float* xs_host, uint32_t n_streams,
                             uint64_t rows_per_stream, uint64_t search_block, uint8_t* payload_host,
                             float* residual_norms_host, void* stream);
/* The same pipeline without blocking the host: the results are on the host
 * once `stream` has completed (the host buffers must stay alive until then).
 * Consecutive calls (keys, then values) overlap their copies with each
 * other's encodes. */
int vqkv_quantize_batch_host_async(vqkv_stack_t stack, const float* xs_host, uint32_t n_streams,
                                   uint64_t rows_per_stream, uint64_t search_block, uint8_t* payload_host,
                                   float* residual_norms_host, void* stream);

/* ---------------------------------------------------------------------------
 * Decode: rows [begin, end) of each stream, out_dev fp32 [n_streams][end-begin][D].
 * Sums effective entries in stage order (codebook.cpp:208-223): bit-exact.
 * Out-of-range codes (possible only in foreign payloads) produce NaN rows and
 * set the stack's sticky error (see vqkv_stack_take_error).
 * ------------------------------------------------------------------------- */
int vqkv_reconstruct_block(vqkv_stack_t stack, const uint8_t* payload_dev, uint32_t n_streams,
                           uint64_t rows_per_stream, uint64_t begin, uint64_t end, float* out_dev,
                           void* stream);
/* the same with streams stride bytes apart (0 = dense: payload bytes of `rows`),
 * e.g. a device-resident cache's fixed-capacity payload buffers */
int vqkv_reconstruct_block_ex(vqkv_stack_t stack, const uint8_t* payload_dev, uint64_t stream_stride,
                              uint32_t n_streams, uint64_t rows, uint64_t begin, uint64_t end, float* out_dev,
                              void* stream);

/* ---------------------------------------------------------------------------
 * Decode-step attention over the three-segment cache of kv_cache.hpp:41-108,
 * for `n_pairs` (batch x kv-head) streams, each with `group` query heads (GQA).
 *   q_dev       fp32 [n_pairs][group][Dk]
 *   init/local  fp32 raw rows [n_pairs][n_init|n_local][Dk|Dv]
 *   kcodes/vcodes  CodeMatrix payloads [n_pairs][payload_bytes(n_comp)]
 *   out_dev     fp32 [n_pairs][group][Dv]  (softmax-normalised output)
 *   lse_dev     fp32 [n_pairs][group]     natural-log sum-exp of scale*logits
 *               (may be NULL)
 * Token order = init | compressed | local, as CacheState::view_block
 * (pending rows are passed as part of `local`).  scale <= 0 means 1/sqrt(Dk)
 * (attention.cpp:14-16).
 * ------------------------------------------------------------------------- */
typedef struct vqkv_attend_args {
    uint32_t n_pairs;
    uint32_t group;
    const float* q_dev;
    const float* init_k_dev;
    const float* init_v_dev;
    uint64_t n_init;
    const uint8_t* kcodes_dev;
    const uint8_t* vcodes_dev;
    uint64_t n_comp;
    const float* local_k_dev;
    const float* local_v_dev;
    uint64_t n_local;
    double scale;
    float* out_dev;
    float* lse_dev;
    /* per-pair strides of the segment buffers (0 = dense): rows between pairs
     * for init / local (a cache keeps them in fixed-capacity buffers), bytes
     * between pairs for the code payloads (capacity, >= payload bytes) */
    uint64_t init_stride;
    uint64_t local_stride;
    uint64_t kcodes_stride;
    uint64_t vcodes_stride;
    /* key-code layout: VQKV_KEYCODES_ROWS (0) = the CodeMatrix payload above;
     * VQKV_KEYCODES_GROUP_MAJOR (1) = the attention layout written by
     * vqkv_keycodes_to_gm, kcodes_cap tokens per group segment (kcodes_stride =
     * bytes between pairs, 0 = vqkv_keycodes_gm_bytes(key_stack, kcodes_cap)) */
    uint32_t kcodes_layout;
    uint64_t kcodes_cap;
} vqkv_attend_args;
#define VQKV_KEYCODES_ROWS 0
#define VQKV_KEYCODES_GROUP_MAJOR 1
int vqkv_attend_decode(vqkv_stack_t key_stack, vqkv_stack_t value_stack, const vqkv_attend_args* args,
                       void* stream);

/* Attention layout of key codes ("group-major records"; no reference counterpart: a
 * device-resident form of the key CodeMatrix rows laid out for the decode-attention kernel,
 * the same bytes per token at the paper geometry).  Per pair, per group g of 8 key stages:
 * an 80-bit record per token t holding eight 10-bit fields, field k = the code of stage
 * 8g + ((t & 7) ^ k) (0 past the last stage) -- the rotation makes the kernel's shared-memory
 * LUT reads conflict-free -- stored as cap u64 words (record bits 0-63) then cap u16 words
 * (bits 64-79).  Needs D = 128 and every key stage <= 1024 entries; cap must be a multiple of
 * 16.  vqkv_keycodes_gm_bytes returns 0 when unsupported.
 * vqkv_keycodes_to_gm writes rows [src_row, src_row + count) of each pair's payload
 * (payload_stride bytes apart) to records [dst_row, dst_row + count) of each pair's
 * buffer (gm_stride bytes apart, 0 = vqkv_keycodes_gm_bytes).  vqkv_keycodes_from_gm is the
 * inverse for records [0, count): it writes CodeMatrix payloads (codebook.cpp:96-120 bit layout,
 * payload_stride bytes apart, 0 = dense) of `count` rows. */
uint64_t vqkv_keycodes_gm_bytes(vqkv_stack_t key_stack, uint64_t cap);
/* 1 when vqkv_attend_decode accepts args with kcodes_layout = VQKV_KEYCODES_GROUP_MAJOR
 * (the LUT attention path covers them), else 0. */
int vqkv_attend_gm_supported(vqkv_stack_t key_stack, vqkv_stack_t value_stack, const vqkv_attend_args* args);
int vqkv_keycodes_to_gm(vqkv_stack_t key_stack, const uint8_t* payload_dev, uint64_t payload_stride, uint32_t n_pairs,
                        uint64_t src_row, uint64_t count, uint8_t* gm_dev, uint64_t cap, uint64_t gm_stride,
                        uint64_t dst_row, void* stream);
int vqkv_keycodes_from_gm(vqkv_stack_t key_stack, const uint8_t* gm_dev, uint64_t cap, uint64_t gm_stride,
                          uint32_t n_pairs, uint64_t count, uint8_t* payload_dev, uint64_t payload_stride,
                          void* stream);

/* CodeMatrix::append of whole packed blocks (codebook.cpp:96-120), batched over
 * streams: for each stream i, bits [0, src_bits) of src + i*src_stride are
 * written at bit dst_bits of dst + i*dst_stride (bits below dst_bits kept).
 * Used by a device-resident cache to append flushed rows at any bit offset. */
int vqkv_payload_append(uint8_t* dst_dev, uint64_t dst_stride, uint64_t dst_bits, const uint8_t* src_dev,
                        uint64_t src_stride, uint64_t src_bits, uint32_t n_streams, void* stream);

/* HOST-buffer variants (copy in, compute, copy out; synchronous), used by the
 * C++ mirror API (include/vqkv/ headers) whose signatures take host matrices. */
/* quantize_batch of `rows` host rows (one stream), optional final residuals */
int vqkv_quantize_rows_host(vqkv_stack_t stack, const float* xs_host, uint64_t rows, uint64_t search_block,
                            uint8_t* payload_host, float* residual_norms_host, float* residuals_host);
/* nearest_entry for one host vector against stage `stage` */
int vqkv_nearest_host(vqkv_stack_t stack, uint32_t stage, const float* x_host, uint64_t search_block,
                      uint32_t* index, float* distance);
int vqkv_reconstruct_block_host(vqkv_stack_t stack, const uint8_t* payload_host, uint64_t rows,
                                uint64_t begin, uint64_t end, float* out_host);
int vqkv_attend_decode_host(vqkv_stack_t key_stack, vqkv_stack_t value_stack,
                            const vqkv_attend_args* host_args);
/* attend_raw (attention.cpp:71-88): softmax(scale q K^T) V over `rows` raw host rows
 * keys [rows][dk], values [rows][dv], one query [dk] -> out [dv] (host), on `device`.
 * scale <= 0 means 1/sqrt(dk).  No codebooks involved. */
int vqkv_attend_raw_host(int device, const float* keys_host, const float* values_host, uint64_t rows, uint32_t dk,
                         uint32_t dv, const float* query_host, double scale, float* out_host);

/* Merge G partial attention results of a sequence split (one per shard):
 * o = sum_g exp(lse_g - LSE) o_g, LSE = log sum_g exp(lse_g).
 * parts_o_dev fp32 [n_parts][rows][dv], parts_lse_dev fp32 [n_parts][rows]. */
int vqkv_lse_combine(const float* parts_o_dev, const float* parts_lse_dev, uint32_t n_parts, uint64_t rows,
                     uint32_t dv, float* out_dev, float* out_lse_dev, void* stream);

/* Sequence-split decode attention (configs[4]), the one exchange step: every rank of the NCCL
 * communicator `nccl_comm` (an ncclComm_t) holds the partial result of its contiguous token shard for
 * the same rows (query heads), part_o_dev fp32 [rows][dv] and part_lse_dev fp32 [rows] (the lse output
 * of vqkv_attend_decode).  One ncclAllGather of both (grouped), then the vqkv_lse_combine merge on every
 * rank: out_dev [rows][dv], out_lse_dev [rows] (may be null).  gather_o_dev [world][rows][dv] and
 * gather_lse_dev [world][rows] are caller scratch, or null for stream-ordered allocations.  All work is
 * stream-ordered on `stream`; NCCL (libnccl.so.2) is loaded on first use. */
int vqkv_lse_allgather_combine(void* nccl_comm, const float* part_o_dev, const float* part_lse_dev, uint64_t rows,
                               uint32_t dv, float* gather_o_dev, float* gather_lse_dev, float* out_dev,
                               float* out_lse_dev, void* stream);
/* ncclCommInitAll(comms, ndev, devs): one communicator per listed device in this process (the
 * single-process 8-GPU layout); vqkv_nccl_comm_destroy releases one. */
int vqkv_nccl_comm_init_all(int ndev, const int* devs, void** comms);
int vqkv_nccl_comm_destroy(void* comm);

/* One mini-batch of the codebook trainer (trainer.cpp:22-86, accumulate_loss): rows x D fp32 on the device,
 * quantized with the reference's search order; the per-stage residual chain, loss terms and
 * straight-through gradients are computed on the GPU in the reference's fp32 operation order.
 * grad_proj_dev: fp32 [N][D][D] (null: loss only), the gradient of the projections summed over the batch
 * rows in order (trainer.cpp:62-67; the caller divides the step by rows, trainer.cpp:229-233).
 * sums_host: double [3 + N] = { sum ||r_N||^2, sum_i ||r_{i+1}||^2, sum_i commitment_i, then per stage i
 * sum ||r_{i+1}||^2 (holdout_stage_mse) }.  Synchronizes `stream`. */
int vqkv_train_batch(vqkv_stack_t stack, const float* batch_dev, uint64_t rows, float beta, float gamma,
                     int square_commitment, float* grad_proj_dev, double* sums_host, void* stream);
/* vqkv_train_batch with host buffers: batch_host [rows][D], grad_proj_host [N][D][D] (may be null). */
int vqkv_train_batch_host(vqkv_stack_t stack, const float* batch_host, uint64_t rows, float beta, float gamma,
                          int square_commitment, float* grad_proj_host, double* sums_host);

/* ---------------------------------------------------------------------------
 * Diagnostics / test hooks.
 * ------------------------------------------------------------------------- */
/* 0 = auto (tensor-core path for D == 128, exact SIMT otherwise),
 * 1 = force the exact SIMT path, 2 = force tensor-core path (fails if D != 128). */
int vqkv_set_encode_path(int path);
/* counters of the last tensor-core encode on this thread's stack:
 * [0] row-stages scored, [1] row-stages whose candidate window held >1 entry
 * (resolved by exact fp32 rescoring), [2] rows routed to the exact path
 * (non-finite input).  Synchronizes. */
int vqkv_encode_counters(vqkv_stack_t stack, uint64_t* counters3);
/* Diagnostics: with VQKV_DBG bit 1 set, the tensor-core encoder sums clock64
 * cycles per epilogue phase (lane 0 of every epilogue warp): [0] tile
 * prologue, [1] waiting for accumulators, [2] chunk max trees, [3] candidate
 * selection, [4] residual update + next A tile, [5] rescoring pass set-up,
 * [6] rescoring loads + dot products, [7] rescoring min-reduction, [8] code
 * store, then inside the update: [9] e_z loads issued + first residual TMEM
 * load, [10] wait for the e_z gather, [11] rest of the update, ([4] is the
 * final store-wait + arrive), [12] accumulator loads; [13] the number of
 * rescored (row, candidate) pairs; MMA-issuer thread totals: [14] waits for
 * a free accumulator, [15] MMA + commit issue, [16] waits for the chunk,
 * [17] waits for the A tile.  Synchronizes. */
int vqkv_encode_phase_clocks(vqkv_stack_t stack, uint64_t* out18);
/* number of kernel launches issued by the library since load (all threads) */
uint64_t vqkv_launch_count(void);
/* Kernel timing hooks: when enabled, the library records a CUDA event pair on
 * the launching stream around each hot kernel (names: "encode_tc",
 * "encode_exact", "pack", "reconstruct", "attend_lut_build", "attend", "attend_combine").
 * vqkv_profile_collect synchronizes on the recorded events, returns the busy
 * milliseconds of `name` (the length of the union of its launches' intervals:
 * the sum for launches on one stream; chunked encodes overlap on two streams)
 * and its launch count, and forgets them. */
int vqkv_profile_enable(int on);
int vqkv_profile_collect(const char* name, double* total_ms, uint64_t* launches);

/* ---------------------------------------------------------------------------
 * Reference fixtures (host): bit-identical restatements of the reference's
 * synthetic input generator and random codebook stacks, so inputs match the
 * reference's on the same seeds.
 * ------------------------------------------------------------------------- */
/* synthetic.cpp:40-63 generate(): kind 0 gaussian_mixture, 1 rope_rotated_keys;
 * out: host fp32 [count][dim] */
int vqkv_generate_synthetic(int kind, uint32_t dim, uint64_t count, uint32_t component_count,
                            uint64_t seed, double rope_base, float component_std, float mean_scale,
                            float* out_host);
/* test_util.hpp:30-50 random_stack(mt19937_64(seed), n, size, dim):
 * entries [n][size][dim], projections [n][dim][dim] (host fp32) */
int vqkv_random_stack(uint64_t seed, uint32_t n_stages, uint32_t size, uint32_t dim, float* entries_host,
                      float* projections_host);
/* FNV-1a-64 (codebook.cpp:326-336 stack_content_hash over the RSVQ bytes) */
uint64_t vqkv_fnv1a64(const uint8_t* data, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* VQKV_C_H */
