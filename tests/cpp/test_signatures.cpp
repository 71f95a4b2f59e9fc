// Compile-only check of the drop-in surface: every entry point the reference's callers use
// (tools/vqkv.cpp:125-248, src/trainer.cpp:229, src/kv_cache.cpp:206-312) binds to a pointer of
// the reference's signature (proj/core/include/vqkv/*.hpp), with this build's matrix types
// standing in for Eigen::Ref<const MatrixF/VectorF>.  Built with -fsyntax-only by
// tests/test_abi_cpu.py; nothing here runs.
#include <string>
#include <type_traits>

#include "vqkv/attention.hpp"
#include "vqkv/codebook.hpp"
#include "vqkv/errors.hpp"
#include "vqkv/kv_cache.hpp"

namespace v = vqkv;

// codebook.hpp:98-138
[[maybe_unused]] static v::NearestResult (*p_nearest)(const v::Codebook&, const v::VectorF&, size_t) =
        &v::nearest_entry<v::VectorF>;
[[maybe_unused]] static v::QuantizeResult (*p_quantize)(const v::CodebookStack&, const v::VectorF&, size_t) =
        &v::quantize<v::VectorF>;
[[maybe_unused]] static v::VectorF (*p_reconstruct)(const v::CodebookStack&, const v::CodeVector&) = &v::reconstruct;
[[maybe_unused]] static v::QuantizeBatchResult (*p_qbatch)(const v::CodebookStack&, const v::MatrixF&, size_t) =
        &v::quantize_batch<v::MatrixF>;
[[maybe_unused]] static v::MatrixF (*p_rblock)(const v::CodebookStack&, const v::CodeMatrix&, size_t, size_t) =
        &v::reconstruct_block;
[[maybe_unused]] static v::CodebookStack (*p_load)(const std::string&) = &v::load_stack;
[[maybe_unused]] static void (*p_save)(const v::CodebookStack&, const std::string&) = &v::save_stack;
[[maybe_unused]] static uint64_t (*p_hash)(const v::CodebookStack&) = &v::stack_content_hash;

// attention.hpp:36-47
[[maybe_unused]] static v::VectorF (*p_attend)(const v::CacheState&, const v::VectorF&, const v::AttentionConfig&,
                                               v::AttendStats*) = &v::attend<v::VectorF>;
[[maybe_unused]] static v::VectorF (*p_attend_raw)(const v::MatrixF&, const v::MatrixF&, const v::VectorF&,
                                                   const v::AttentionConfig&) = &v::attend_raw<v::MatrixF, v::VectorF>;
[[maybe_unused]] static v::FidelityReport (*p_fidelity)(const v::CacheState&, const v::MatrixF&, const v::MatrixF&,
                                                        const v::MatrixF&, const v::AttentionConfig&) =
        &v::fidelity<v::MatrixF>;

// kv_cache.hpp:45-108
[[maybe_unused]] static void (v::CacheState::*p_prefill)(const v::MatrixF&, const v::MatrixF&) =
        &v::CacheState::prefill<v::MatrixF>;
[[maybe_unused]] static void (v::CacheState::*p_append)(const v::VectorF&, const v::VectorF&) =
        &v::CacheState::append_token<v::VectorF>;
[[maybe_unused]] static v::ViewBlock (v::CacheState::*p_view)(size_t, size_t) const = &v::CacheState::view_block;
[[maybe_unused]] static v::MemoryReport (v::CacheState::*p_mem)() const = &v::CacheState::memory_report;
[[maybe_unused]] static void (v::CacheState::*p_snap_save)(const std::string&) const = &v::CacheState::save_snapshot;
[[maybe_unused]] static v::CacheState (*p_snap_load)(const std::string&, const v::CodebookStack&,
                                                     const v::CodebookStack&) = &v::CacheState::load_snapshot;

// errors.hpp:12-49: the hierarchy the reference's callers catch and throw
static_assert(std::is_base_of_v<v::Error, v::InvalidInput> && std::is_base_of_v<v::Error, v::InvalidState> &&
              std::is_base_of_v<v::Error, v::InvalidCode> && std::is_base_of_v<v::Error, v::FormatError> &&
              std::is_base_of_v<v::Error, v::IoError> && std::is_base_of_v<v::Error, v::DivergedError>);
static_assert(std::is_constructible_v<v::DivergedError, const std::string&, size_t>);  // trainer.cpp:229
static_assert(std::is_constructible_v<v::FormatError, const std::string&, size_t>);
static_assert(std::is_same_v<decltype(v::DivergedError("", 0).epoch), size_t>);
static_assert(std::is_same_v<decltype(v::FormatError("", 0).byte_offset), size_t>);

// the reference CLI's bench sequence (tools/vqkv.cpp:180-248), call shapes only
[[maybe_unused]] static void bench_shape(const v::CodebookStack& ks, const v::CodebookStack& vs, const v::MatrixF& keys,
                                         const v::MatrixF& values, const v::MatrixF& queries, const v::VectorF& q0) {
    v::WindowPolicy policy{4, 1024, false};
    v::CacheState state(ks, vs, policy);
    state.prefill(keys, values);
    state.append_token(q0, q0);
    v::AttentionConfig attn;
    attn.block_rows = 128;
    v::FidelityReport fid = v::fidelity(state, keys, values, queries, attn);
    v::AttendStats stats;
    v::attend(state, q0, attn, &stats);
    (void)fid.output_max_abs_err;
    (void)stats.peak_reconstructed_scalars;
    state.save_snapshot("x.vqks");
    v::CacheState back = v::CacheState::load_snapshot("x.vqks", ks, vs);
    (void)back.memory_report().effective_ratio;
}
