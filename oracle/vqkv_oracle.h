/*
 * vqkv_oracle.h -- C API of the CPU ORACLE (test infrastructure only).
 *
 * THIS IS A CHECKER, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product library (paper_2603_16435_b200/, libvqkv_b200.so) never links it.
 *
 * It is a plain-C++ restatement (no Eigen) of the reference's hot path:
 *   proj/core/src/codebook.cpp:30-250    refresh, CodeMatrix, nearest_scored,
 *                                        quantize, reconstruct, *_batch/_block
 *   proj/core/src/codebook.cpp:252-336   RSVQ container + FNV-1a hash
 *   proj/core/include/vqkv/bitpack.hpp   LSB-first bit stream
 *   proj/core/src/kv_cache.cpp:41-204    window policy, prefill, append, view
 *   proj/core/src/attention.cpp:14-88    attend / attend_raw
 *   proj/core/src/synthetic.cpp:26-63    synthetic generator
 *   proj/tests/test_util.hpp:15-60       random_stack / random_matrix
 * Parity pinning: see oracle/README.md (KATs from the reference tests).
 */
#ifndef VQKV_ORACLE_H
#define VQKV_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror vqkv/errors.hpp exception kinds */
enum {
    ORC_OK = 0,
    ORC_INVALID_INPUT = 1,
    ORC_INVALID_STATE = 2,
    ORC_INVALID_CODE = 3,
    ORC_FORMAT_ERROR = 4,
    ORC_IO_ERROR = 5,
    ORC_OTHER = 9
};

const char* orc_last_error(void);
uint64_t orc_last_error_offset(void);

/* ---- RNG (std::mt19937_64, libstdc++) -------------------------------- */
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng*);
uint64_t orc_rng_next(orc_rng*); /* rng() */
/* test_util.hpp:51-59 random_matrix: scale * N(0,1) row-major */
void orc_random_matrix(orc_rng*, int64_t rows, int64_t cols, float scale, float* out);

/* ---- stacks ------------------------------------------------------------ */
typedef struct orc_stack orc_stack;
/* test_util.hpp:30-50 */
orc_stack* orc_random_stack(orc_rng*, uint32_t n_stages, uint32_t size, int64_t dim, int kind);
/* raw entries + projections; refresh() computes effective + sqnorm.
   entries: concatenated stage-major [S_i x D]; projections [N x D x D]
   (projections may be NULL: identity, as test_util.hpp:15-28). */
orc_stack* orc_stack_new(uint32_t n_stages, const uint32_t* sizes, int64_t dim,
                         const float* entries, const float* projections, int kind);
void orc_stack_free(orc_stack*);
uint32_t orc_stack_num_stages(const orc_stack*);
int64_t orc_stack_dim(const orc_stack*);
uint32_t orc_stack_stage_size(const orc_stack*, uint32_t stage);
int orc_stack_kind(const orc_stack*);
void orc_stack_get_entries(const orc_stack*, uint32_t stage, float* out);
void orc_stack_get_projection(const orc_stack*, uint32_t stage, float* out);
void orc_stack_get_effective(const orc_stack*, uint32_t stage, float* out);
void orc_stack_get_sqnorm(const orc_stack*, uint32_t stage, float* out);
int orc_stack_save(const orc_stack*, const char* path);
/* serialize to memory: returns byte count; if buf!=NULL and cap large enough writes it */
uint64_t orc_stack_serialize(const orc_stack*, uint8_t* buf, uint64_t cap);
orc_stack* orc_stack_load(const char* path);
orc_stack* orc_stack_load_bytes(const uint8_t* buf, uint64_t n);
uint64_t orc_stack_hash(const orc_stack*);

/* ---- code matrix helpers --------------------------------------------------- */
unsigned orc_index_bit_width(uint32_t size);
uint64_t orc_row_bits(uint32_t n_stages, const uint32_t* sizes);
uint64_t orc_payload_bytes(uint32_t n_stages, const uint32_t* sizes, uint64_t rows);
/* CodeMatrix::append over `rows` rows of codes (u32 [rows x N]); validates */
int orc_codes_pack(uint32_t n_stages, const uint32_t* sizes, const uint32_t* codes, uint64_t rows,
                   uint8_t* payload);
int orc_codes_unpack(uint32_t n_stages, const uint32_t* sizes, const uint8_t* payload,
                     uint64_t rows, uint32_t* codes);

/* ---- quantizer (codebook.cpp:158-250) -------------------------------------- */
int orc_nearest_entry(const orc_stack*, uint32_t stage, const float* x, int64_t xdim,
                      uint64_t search_block, uint32_t* index, float* distance);
int orc_quantize(const orc_stack*, const float* x, int64_t xdim, uint64_t search_block,
                 uint32_t* codes, float* final_residual);
int orc_reconstruct(const orc_stack*, const uint32_t* codes, uint64_t n_codes, float* out);
/* quantize_batch: payload (CodeMatrix bytes) + residual norms.  Optional
   instrumentation (may be NULL): per (row, stage) best score, second-best
   score, ||r|| entering the stage (fp32), and per-stage max ||e||. */
int orc_quantize_batch(const orc_stack*, const float* xs, uint64_t rows, int64_t xdim,
                       uint64_t search_block, uint8_t* payload, float* residual_norms,
                       float* best, float* second, float* rnorm);
/* same as quantize_batch but over n_streams independent streams, one
   std::thread per stream up to `threads` (SPEC.md:270-272 independence). */
int orc_quantize_batch_mt(const orc_stack*, const float* xs, uint32_t n_streams,
                          uint64_t rows_per_stream, uint64_t search_block, uint8_t* payload,
                          float* residual_norms, int threads);
int orc_reconstruct_block(const orc_stack*, const uint8_t* payload, uint64_t rows,
                          uint64_t begin, uint64_t end, float* out);
void orc_stage_max_norm(const orc_stack*, float* out); /* per stage max ||e_i|| (fp32) */

/* ---- synthetic (synthetic.cpp:26-63) ----------------------------------- */
int orc_generate(int kind, int64_t dim, int64_t count, uint32_t component_count, uint64_t seed,
                 double rope_base, float component_std, float mean_scale, float* out);

/* ---- kv cache (kv_cache.cpp) + attention (attention.cpp) ---------------- */
typedef struct orc_cache orc_cache;
orc_cache* orc_cache_new(const orc_stack* keys, const orc_stack* values, uint64_t init_len,
                         uint64_t local_len, int eager);
void orc_cache_free(orc_cache*);
int orc_cache_prefill(orc_cache*, const float* keys, const float* values, int64_t rows,
                      int64_t kdim, int64_t vdim);
int orc_cache_append(orc_cache*, const float* key, int64_t kdim, const float* value, int64_t vdim);
/* counts[0..5] = init, compressed, pending, local, total, batched_compressions */
void orc_cache_counts(const orc_cache*, uint64_t* counts);
int orc_cache_view_block(const orc_cache*, uint64_t begin, uint64_t end, float* keys,
                         float* values, uint8_t* exact);
/* payload bytes / residual norms of the compressed segment */
void orc_cache_codes(const orc_cache*, int which, uint8_t* payload, float* norms);
/* MemoryReport: raw_bytes, payload_bits, overhead_bytes, ratio */
void orc_cache_memory_report(const orc_cache*, uint64_t* raw_bytes, uint64_t* payload_bits,
                             uint64_t* overhead_bytes, double* ratio);
int orc_attend(const orc_cache*, const float* q, int64_t qdim, uint64_t block_rows, double scale,
               float* out, uint64_t* peak_scalars, uint64_t* reconstructed_rows);
int orc_attend_raw(const float* keys, const float* values, int64_t rows, int64_t kdim,
                   int64_t vdim, const float* q, int64_t qdim, double scale, float* out);
/* attend() over explicit segments (no CacheState): init/local raw rows and a
   compressed CodeMatrix payload.  Used for large-context parity where the
   compressed segment is filled with synthetic codes. Also
   returns the natural-log LSE of scale*logits. */
int orc_attend_segments(const orc_stack* kst, const orc_stack* vst, const float* init_k,
                        const float* init_v, uint64_t n_init, const uint8_t* kpay,
                        const uint8_t* vpay, uint64_t n_comp, const float* local_k,
                        const float* local_v, uint64_t n_local, const float* q, double scale,
                        uint64_t block_rows, float* out, double* lse);

/* ---- trainer (proj/core/src/trainer.cpp:22-248) ---------------------------- */
/* accumulate_loss over one batch (trainer.cpp:36-86): sums[0..2] = sum over rows of ||r_N||^2,
   sum_i ||r_{i+1}||^2, sum_i commitment_i (before the division by the batch size), sums[3 + i] = sum of
   ||r_{i+1}||^2 per stage; grad (N x D x D, or NULL) = the projections' gradient summed over rows. */
int orc_train_batch(const orc_stack*, const float* batch, uint64_t rows, float beta, float gamma,
                    int square_commitment, float* grad, double* sums);
typedef struct {
    float learning_rate;
    uint64_t batch_size;
    uint64_t epochs;
    float beta, gamma;
    uint64_t seed;
    float init_scale;
    int square_commitment;
    float holdout_fraction;
} orc_train_config;
/* train() (trainer.cpp:166-248, train_entries = false): returns the trained stack; epoch_loss [epochs],
   stage_mse [N] (may be NULL). */
orc_stack* orc_train(const float* data, uint64_t count, int64_t dim, uint32_t n_stages, const uint32_t* sizes,
                     const orc_train_config* cfg, int kind, double* epoch_loss, double* stage_mse);

#ifdef __cplusplus
}
#endif
#endif
