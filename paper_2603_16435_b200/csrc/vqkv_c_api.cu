// vqkv_c_api.cu -- the C-ABI of libvqkv_b200.so (include/vqkv_c.h).
//
// Validation mirrors the reference's exception behaviour (errors.hpp:12-49,
// codebook.cpp:41-72 / 225-250, attention.cpp:20-35); CUDA work is enqueued
// on the caller's stream.
#include <vector>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "vqkv_internal.cuh"

namespace vqkv_dev {
std::atomic<uint64_t> g_launches{0};

namespace {
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
struct ProfRec {
    std::string name;
    cudaEvent_t a, b;
};
std::vector<ProfRec> g_prof_recs;
}  // namespace

bool prof_enabled() { return g_prof.load(std::memory_order_relaxed); }
void prof_record(const char* name, cudaEvent_t a, cudaEvent_t b) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_recs.push_back({name, a, b});
}
}  // namespace vqkv_dev

using namespace vqkv_dev;

namespace {

thread_local std::string t_err;
std::atomic<int> g_encode_path{0};

template <class F>
int guard(F&& f) {
    try {
        f();
        return VQKV_OK;
    } catch (const Err& e) {
        t_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        t_err = e.what();
        return VQKV_CUDA_ERROR;
    }
}

void need(bool ok, int code, const char* msg) {
    if (!ok) fail(code, msg);
}

void check_stack(vqkv_stack_t s) { need(s != nullptr, VQKV_INVALID_INPUT, "null stack"); }

// Streams per encode launch when a call is split into chunks: 32-160 MiB of input per chunk,
// picking the size whose tile count best fills whole rounds of the persistent grid (2 tiles
// per SM).  Consecutive chunks alternate between two compute streams, so the SMs a launch
// idles in its last round (uneven rescoring work per tile) are taken by the next chunk.
uint32_t encode_chunk_streams(const vqkv_stack_s& st, uint32_t n_streams, uint64_t rows) {
    if (const char* e = getenv("VQKV_CHUNK_STREAMS")) {  // dev override (A/B timing)
        const long v = strtol(e, nullptr, 10);
        if (v > 0) return uint32_t(std::min<long>(v, long(n_streams)));
    }
    const uint64_t per_stream_in = rows * st.dim * sizeof(float);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, st.device);
    const uint64_t slots = 2ull * uint64_t(sms), tiles_ps = (rows + 127) / 128;
    const uint64_t lo = std::max<uint64_t>(1, (32ull << 20) / per_stream_in);
    const uint64_t hi = std::max<uint64_t>(lo, (160ull << 20) / per_stream_in);
    uint32_t chunk = uint32_t(std::min<uint64_t>(n_streams, lo));
    double best_waste = 2.0;
    for (uint64_t c = lo; c <= std::min<uint64_t>(hi, n_streams); ++c) {
        const uint64_t t = c * tiles_ps, rounds = (t + slots - 1) / slots;
        const double waste = double(rounds * slots - t) / double(rounds * slots);
        if (waste < best_waste - 1e-3) {
            best_waste = waste;
            chunk = uint32_t(c);
        }
    }
    return chunk;
}

// The stack's copy streams and second compute stream, created on first use.  The copy streams are
// shared by every stack on a device (and live for the process), so host-buffer calls queued back to
// back (values behind keys, then the next step's keys) copy in call order at the link's full
// bandwidth: per-stack streams let the next call's prefetch halve the bandwidth of the inputs needed
// first.  (Each call stages all of its chunks, so an earlier call's copies never wait on its encodes.)
struct DevCopyStreams {
    cudaStream_t in = nullptr, out = nullptr;
};
std::mutex g_copy_mu;
DevCopyStreams g_copy[64];

void ensure_streams(vqkv_stack_s& st) {
    std::lock_guard<std::mutex> lk(st.mu);
    if (st.cp_in) return;
    {
        std::lock_guard<std::mutex> lk2(g_copy_mu);
        DevCopyStreams& d = g_copy[st.device & 63];
        if (!d.in) {
            VQKV_CUDA(cudaStreamCreateWithFlags(&d.in, cudaStreamNonBlocking));
            VQKV_CUDA(cudaStreamCreateWithFlags(&d.out, cudaStreamNonBlocking));
        }
        st.cp_in = d.in;
        st.cp_out = d.out;
    }
    VQKV_CUDA(cudaStreamCreateWithFlags(&st.cs_alt, cudaStreamNonBlocking));
}

// cs_alt starts after everything already queued on s (fork) / s continues after cs_alt (join)
void fork_alt(vqkv_stack_s& st, cudaStream_t s) {
    cudaEvent_t e;
    VQKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    VQKV_CUDA(cudaEventRecord(e, s));
    VQKV_CUDA(cudaStreamWaitEvent(st.cs_alt, e, 0));
    cudaEventDestroy(e);
}
void join_alt(vqkv_stack_s& st, cudaStream_t s) {
    cudaEvent_t e;
    VQKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    VQKV_CUDA(cudaEventRecord(e, st.cs_alt));
    VQKV_CUDA(cudaStreamWaitEvent(s, e, 0));
    cudaEventDestroy(e);
}

// quantize_batch on device buffers (used by the device and host entry points); split = chunk the
// streams over two compute streams (the host pipeline chunks itself and passes false)
void quantize_device(vqkv_stack_s& st, const float* xs, uint32_t n_streams, uint64_t rows, uint64_t sb,
                     uint8_t* payload, float* norms, float* residuals, cudaStream_t s, bool split = true) {
    const uint64_t total = uint64_t(n_streams) * rows;
    if (total == 0) return;
    const int path = g_encode_path.load();
    const bool tc = encode_tc_supported(st);
    if (path == 2 && !tc) fail(VQKV_UNSUPPORTED, "tensor-core encode path requires D == 128");
    if (tc && path != 1) {
        const uint32_t chunk = split ? encode_chunk_streams(st, n_streams, rows) : n_streams;
        if (chunk >= n_streams) {
            launch_encode_tc(st, xs, n_streams, rows, sb, payload, norms, residuals, s);
            return;
        }
        ensure_streams(st);
        fork_alt(st, s);
        const uint64_t pb = payload_bytes(st.row_bits, rows);
        uint32_t i = 0;
        for (uint32_t s0 = 0; s0 < n_streams; s0 += chunk, ++i) {
            const uint32_t ns = std::min<uint32_t>(chunk, n_streams - s0);
            launch_encode_tc(st, xs + uint64_t(s0) * rows * st.dim, ns, rows, sb, payload + uint64_t(s0) * pb,
                             norms + uint64_t(s0) * rows, residuals ? residuals + uint64_t(s0) * rows * st.dim : nullptr,
                             (i & 1) ? st.cs_alt : s);
        }
        join_alt(st, s);
        return;
    }
    uint16_t* codes = nullptr;
    VQKV_CUDA(cudaMallocAsync(&codes, sizeof(uint16_t) * total * st.n, s));
    launch_encode_exact(st, xs, total, sb, codes, norms, residuals, s);
    launch_pack_codes(codes, n_streams, rows, st.n, st, payload, s);
    VQKV_CUDA(cudaFreeAsync(codes, s));
}

// Carves the synchronous host entry points' device buffers out of the stack's grow-only scratch
// (no cudaMalloc/cudaFree per call; nothing to leak when a call throws).  Caller holds host_mu.
struct HostScratch {
    vqkv_stack_s& st;
    std::vector<uint64_t> sizes;
    explicit HostScratch(vqkv_stack_s& s) : st(s) {}
    // reserve `bytes` (+16 B of slack for whole-word reads), 256 B aligned; returns the offset
    uint64_t add(uint64_t bytes) {
        uint64_t off = 0;
        for (uint64_t b : sizes) off += b;
        sizes.push_back((bytes + 16 + 255) & ~uint64_t(255));
        return off;
    }
    uint8_t* commit() {
        uint64_t total = 0;
        for (uint64_t b : sizes) total += b;
        if (st.host_scratch_bytes < total) {
            if (st.host_scratch) VQKV_CUDA(cudaFree(st.host_scratch));
            st.host_scratch = nullptr;
            st.host_scratch_bytes = 0;
            VQKV_CUDA(cudaMalloc(&st.host_scratch, total));
            st.host_scratch_bytes = total;
        }
        return st.host_scratch;
    }
};

}  // namespace

extern "C" {

const char* vqkv_last_error(void) { return t_err.c_str(); }
const char* vqkv_version(void) { return "vqkv_b200 0.1 (sm_100a)"; }
uint64_t vqkv_launch_count(void) { return g_launches.load(); }

int vqkv_profile_enable(int on) {
    g_prof.store(on != 0);
    return VQKV_OK;
}

int vqkv_profile_collect(const char* name, double* total_ms, uint64_t* launches) {
    return guard([&] {
        need(name != nullptr, VQKV_INVALID_INPUT, "null name");
        std::lock_guard<std::mutex> lk(g_prof_mu);
        uint64_t n = 0;
        std::vector<ProfRec> keep, mine;
        for (auto& r : g_prof_recs) (r.name == name ? mine : keep).push_back(r);
        // busy time = length of the union of the launches' [start, end] intervals (launches on
        // two streams overlap; on one stream this is their sum), relative to the first start
        std::vector<std::pair<double, double>> iv;
        for (auto& r : mine) {
            VQKV_CUDA(cudaEventSynchronize(r.b));
            float t0 = 0.f, t1 = 0.f;
            VQKV_CUDA(cudaEventElapsedTime(&t0, mine[0].a, r.a));
            VQKV_CUDA(cudaEventElapsedTime(&t1, mine[0].a, r.b));
            iv.emplace_back(t0, t1);
            ++n;
        }
        for (auto& r : mine) {
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        std::sort(iv.begin(), iv.end());
        double ms = 0.0, lo = 0.0, hi = 0.0;
        bool open = false;
        for (const auto& x : iv) {
            if (open && x.first <= hi) {
                hi = std::max(hi, x.second);
            } else {
                if (open) ms += hi - lo;
                lo = x.first;
                hi = x.second;
                open = true;
            }
        }
        if (open) ms += hi - lo;
        g_prof_recs.swap(keep);
        if (total_ms) *total_ms = ms;
        if (launches) *launches = n;
    });
}

int vqkv_set_encode_path(int path) {
    return guard([&] {
        need(path >= 0 && path <= 2, VQKV_INVALID_INPUT, "encode path must be 0, 1 or 2");
        g_encode_path.store(path);
    });
}

int vqkv_stack_create(int device, int kind, uint32_t n_stages, const uint32_t* sizes, uint32_t dim,
                      const float* entries, const float* projections, vqkv_stack_t* out) {
    return guard([&] {
        need(out != nullptr, VQKV_INVALID_INPUT, "null output handle");
        *out = nullptr;
        need(kind == 0 || kind == 1, VQKV_INVALID_INPUT, "cache kind must be key (0) or value (1)");
        need(n_stages >= 1, VQKV_INVALID_INPUT, "stack must have at least one stage");  // codebook.cpp:63-65
        need(dim >= 1, VQKV_INVALID_INPUT, "codebook must have S >= 1 and D >= 1");
        need(sizes != nullptr && entries != nullptr, VQKV_INVALID_INPUT, "null sizes/entries");
        auto st = std::make_unique<vqkv_stack_s>();
        st->device = device;
        st->kind = kind;
        st->n = n_stages;
        st->dim = dim;
        uint64_t off = 0, off16 = 0, bit = 0;
        for (uint32_t s = 0; s < n_stages; ++s) {
            need(sizes[s] >= 1, VQKV_INVALID_INPUT, "codebook must have S >= 1 and D >= 1");
            need(sizes[s] <= 65536, VQKV_UNSUPPORTED, "codebook sizes above 65536 are not supported");
            StageInfo si{};
            si.size = sizes[s];
            si.bits = index_bit_width(sizes[s]);
            si.bit_off = uint32_t(bit);
            si.pad_size = (sizes[s] + 127u) / 128u * 128u;
            si.eff_off = off * dim;
            si.eff16_off = off16 * (uint64_t(dim) + 16);  // main K block + 16-wide ||e||^2 block
            si.pad_off = off16;
            bit += si.bits;
            off += sizes[s];
            off16 += si.pad_size;
            st->stages.push_back(si);
        }
        st->row_bits = bit;
        st->total_rows = off;
        st->total_pad_rows = off16;
        // codebook.cpp:48-50: non-finite entries/projections are rejected
        for (uint64_t i = 0; i < off * dim; ++i)
            need(std::isfinite(entries[i]), VQKV_INVALID_INPUT, "codebook contains non-finite values");
        if (projections)
            for (uint64_t i = 0; i < uint64_t(n_stages) * dim * dim; ++i)
                need(std::isfinite(projections[i]), VQKV_INVALID_INPUT, "codebook contains non-finite values");
        DeviceGuard g(device);
        {
            // the encoder's stream-ordered scratch (cudaMallocAsync) stays mapped
            // between calls instead of being unmapped at every synchronization
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        VQKV_CUDA(cudaMalloc(&st->d_stages, sizeof(StageInfo) * n_stages));
        VQKV_CUDA(cudaMemcpy(st->d_stages, st->stages.data(), sizeof(StageInfo) * n_stages, cudaMemcpyHostToDevice));
        VQKV_CUDA(cudaMalloc(&st->d_error, sizeof(int)));
        VQKV_CUDA(cudaMemset(st->d_error, 0, sizeof(int)));
        VQKV_CUDA(cudaMalloc(&st->d_counters, sizeof(unsigned long long) * 32));
        VQKV_CUDA(cudaMemset(st->d_counters, 0, sizeof(unsigned long long) * 32));
        stack_build_device(*st, entries, projections);
        *out = st.release();
    });
}

int vqkv_stack_destroy(vqkv_stack_t s) {
    return guard([&] {
        if (!s) return;
        DeviceGuard g(s->device);
        cudaDeviceSynchronize();
        cudaFree(s->d_stages);
        cudaFree(s->d_eff);
        cudaFree(s->d_raw);
        cudaFree(s->d_sqn);
        cudaFree(s->d_eff16);
        cudaFree(s->d_eff16lo);
        cudaFree(s->d_sqn_pad);
        cudaFree(s->d_error);
        cudaFree(s->d_counters);
        if (s->host_scratch) cudaFree(s->host_scratch);
        if (s->cs_alt) cudaStreamDestroy(s->cs_alt);
        if (s->cs_attn) cudaStreamDestroy(s->cs_attn);
        if (s->cs_attn_hi) cudaStreamDestroy(s->cs_attn_hi);
        for (auto& a : s->staging) {
            if (a.done) cudaEventSynchronize(a.done), cudaEventDestroy(a.done);
            if (a.base) cudaFree(a.base);
        }
        delete s;
    });
}

int vqkv_stack_describe(vqkv_stack_t s, uint32_t* n, uint32_t* dim, uint64_t* row_bits, int* kind, int* device) {
    return guard([&] {
        check_stack(s);
        if (n) *n = s->n;
        if (dim) *dim = s->dim;
        if (row_bits) *row_bits = s->row_bits;
        if (kind) *kind = s->kind;
        if (device) *device = s->device;
    });
}

int vqkv_stack_stage_size(vqkv_stack_t s, uint32_t stage, uint32_t* size) {
    return guard([&] {
        check_stack(s);
        need(stage < s->n, VQKV_INVALID_INPUT, "stage out of range");
        *size = s->stages[stage].size;
    });
}

int vqkv_stack_effective(vqkv_stack_t s, uint32_t stage, float* eff, float* sqn) {
    return guard([&] {
        check_stack(s);
        need(stage < s->n, VQKV_INVALID_INPUT, "stage out of range");
        DeviceGuard g(s->device);
        const StageInfo& si = s->stages[stage];
        if (eff)
            VQKV_CUDA(cudaMemcpy(eff, s->d_eff + si.eff_off, sizeof(float) * si.size * s->dim, cudaMemcpyDeviceToHost));
        if (sqn)
            VQKV_CUDA(cudaMemcpy(sqn, s->d_sqn + si.eff_off / s->dim, sizeof(float) * si.size, cudaMemcpyDeviceToHost));
    });
}

int vqkv_stack_effective_dev(vqkv_stack_t s, uint32_t stage, const float** p) {
    return guard([&] {
        check_stack(s);
        need(stage < s->n, VQKV_INVALID_INPUT, "stage out of range");
        *p = s->d_eff + s->stages[stage].eff_off;
    });
}

uint64_t vqkv_payload_bytes(vqkv_stack_t s, uint64_t rows) { return s ? payload_bytes(s->row_bits, rows) : 0; }

int vqkv_stack_take_error(vqkv_stack_t s) {
    int code = VQKV_OK;
    int st = guard([&] {
        check_stack(s);
        DeviceGuard g(s->device);
        VQKV_CUDA(cudaDeviceSynchronize());
        VQKV_CUDA(cudaMemcpy(&code, s->d_error, sizeof(int), cudaMemcpyDeviceToHost));
        VQKV_CUDA(cudaMemset(s->d_error, 0, sizeof(int)));
    });
    if (st != VQKV_OK) return st;
    if (code != VQKV_OK) t_err = "code index out of range for its stage (InvalidCode)";
    return code;
}

int vqkv_encode_counters(vqkv_stack_t s, uint64_t* c) {
    return guard([&] {
        check_stack(s);
        DeviceGuard g(s->device);
        VQKV_CUDA(cudaDeviceSynchronize());
        unsigned long long h[4];
        VQKV_CUDA(cudaMemcpy(h, s->d_counters, sizeof(h), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 3; ++i) c[i] = h[i];
    });
}

int vqkv_encode_phase_clocks(vqkv_stack_t s, uint64_t* c) {
    return guard([&] {
        check_stack(s);
        DeviceGuard g(s->device);
        VQKV_CUDA(cudaDeviceSynchronize());
        unsigned long long h[32];
        VQKV_CUDA(cudaMemcpy(h, s->d_counters, sizeof(h), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 13; ++i) c[i] = h[8 + i];
        c[13] = h[3];
        for (int i = 0; i < 4; ++i) c[14 + i] = h[21 + i];
    });
}

int vqkv_payload_append(uint8_t* dst, uint64_t dst_stride, uint64_t dst_bits, const uint8_t* src,
                        uint64_t src_stride, uint64_t src_bits, uint32_t n_streams, void* stream) {
    return guard([&] {
        if (src_bits == 0 || n_streams == 0) return;
        need(dst && src, VQKV_INVALID_INPUT, "null payload buffer");
        need(dst_stride * 8 >= dst_bits + src_bits, VQKV_INVALID_INPUT, "destination payload capacity exceeded");
        need(src_stride * 8 >= src_bits, VQKV_INVALID_INPUT, "source payload shorter than src_bits");
        launch_payload_append(dst, dst_stride, dst_bits, src, src_stride, src_bits, n_streams, as_stream(stream));
    });
}

int vqkv_quantize_batch(vqkv_stack_t s, const float* xs, uint32_t n_streams, uint64_t rows, uint64_t sb,
                        uint8_t* payload, float* norms, void* stream) {
    return vqkv_quantize_batch_ex(s, xs, n_streams, rows, sb, payload, norms, nullptr, stream);
}

int vqkv_nearest_batch(vqkv_stack_t s, uint32_t stage, const float* xs, uint64_t rows, uint64_t sb, uint32_t* idx,
                       float* dist, void* stream) {
    return guard([&] {
        check_stack(s);
        need(stage < s->n, VQKV_INVALID_INPUT, "stage out of range");
        need(sb >= 1, VQKV_INVALID_INPUT, "search_block must be >= 1");
        if (rows == 0) return;
        need(xs && idx && dist, VQKV_INVALID_INPUT, "null device buffer");
        DeviceGuard g(s->device);
        launch_nearest(*s, stage, xs, rows, sb, idx, dist, as_stream(stream));
    });
}

int vqkv_quantize_batch_ex(vqkv_stack_t s, const float* xs, uint32_t n_streams, uint64_t rows, uint64_t sb,
                           uint8_t* payload, float* norms, float* residuals, void* stream) {
    return guard([&] {
        check_stack(s);
        need(sb >= 1, VQKV_INVALID_INPUT, "search_block must be >= 1");
        const uint64_t total = uint64_t(n_streams) * rows;
        if (total == 0) return;  // codebook.cpp:227: empty batch is valid
        need(xs && norms && (payload || s->row_bits == 0), VQKV_INVALID_INPUT, "null device buffer");
        DeviceGuard g(s->device);
        quantize_device(*s, xs, n_streams, rows, sb, payload, norms, residuals, as_stream(stream));
    });
}

int vqkv_quantize_batch_host(vqkv_stack_t s, const float* xs, uint32_t n_streams, uint64_t rows, uint64_t sb,
                             uint8_t* payload, float* norms, void* stream) {
    const int st = vqkv_quantize_batch_host_async(s, xs, n_streams, rows, sb, payload, norms, stream);
    if (st != VQKV_OK) return st;
    return guard([&] {
        DeviceGuard g(s->device);
        VQKV_CUDA(cudaStreamSynchronize(as_stream(stream)));
    });
}

int vqkv_quantize_batch_host_async(vqkv_stack_t s, const float* xs, uint32_t n_streams, uint64_t rows, uint64_t sb,
                                   uint8_t* payload, float* norms, void* stream) {
    return guard([&] {
        check_stack(s);
        need(sb >= 1, VQKV_INVALID_INPUT, "search_block must be >= 1");
        const uint64_t total = uint64_t(n_streams) * rows;
        if (total == 0) return;
        need(xs && norms && (payload || s->row_bits == 0), VQKV_INVALID_INPUT, "null host buffer");
        DeviceGuard g(s->device);
        cudaStream_t cs = as_stream(stream);
        const uint64_t D = s->dim;
        const uint64_t pb = payload_bytes(s->row_bits, rows);
        // chunk over streams (encode_chunk_streams), staging sets so the copy engines overlap
        // the encoder (H2D i+1 | encode i | D2H i-1); staging comes from the stream-ordered pool
        // and nothing blocks the host, so consecutive calls (e.g. K then V) keep the copy engines busy
        const uint64_t per_stream_in = rows * D * sizeof(float);
        const uint32_t chunk = encode_chunk_streams(*s, n_streams, rows);
        ensure_streams(*s);
        cudaStream_t cp_in = s->cp_in, cp_out = s->cp_out;
        // chunk encodes alternate between the caller's stream and cs_alt: a persistent encode
        // launch idles SMs in its last round, and the next chunk's CTAs take them over
        cudaStream_t cst[2] = {cs, s->cs_alt};
        fork_alt(*s, cs);  // ordered after the caller's earlier work
        {  // the shared copy-in stream too: earlier work on `stream` may still be writing xs_host
            cudaEvent_t e;
            VQKV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            VQKV_CUDA(cudaEventRecord(e, cs));
            VQKV_CUDA(cudaStreamWaitEvent(cp_in, e, 0));
            cudaEventDestroy(e);
        }
        const uint32_t n_chunks = (n_streams + chunk - 1) / chunk;
        const uint64_t set_bytes = (per_stream_in + pb + sizeof(float) * rows) * chunk;
        // staging for every chunk (up to 16 GiB per arena): the shared copy-in stream then never waits
        // on this call's encodes, which would hold up the copies of the calls queued behind it
        const uint32_t nbuf = std::min<uint32_t>(n_chunks, std::max<uint32_t>(2, uint32_t((16ull << 30) / set_bytes)));
        std::vector<float*> dx(nbuf), dn(nbuf);
        std::vector<uint8_t*> dp(nbuf);
        std::vector<cudaEvent_t> in_ready(nbuf), done(nbuf), out_done(nbuf);
        cudaEvent_t last;
        // staging arena (see vqkv_stack_s::Staging): free once the call two before this one completed
        auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
        const uint64_t bx = al(per_stream_in * chunk), bp = al(std::max<uint64_t>(pb * chunk, 1)),
                       bn = al(sizeof(float) * rows * chunk);
        vqkv_stack_s::Staging* arena;
        {
            std::lock_guard<std::mutex> lk(s->mu);
            arena = &s->staging[s->staging_next];
            s->staging_next ^= 1u;
        }
        if (arena->done) VQKV_CUDA(cudaEventSynchronize(arena->done));
        else VQKV_CUDA(cudaEventCreateWithFlags(&arena->done, cudaEventDisableTiming));
        const uint64_t need = uint64_t(nbuf) * (bx + bp + bn);
        if (arena->bytes < need) {
            if (arena->base) VQKV_CUDA(cudaFree(arena->base));
            arena->base = nullptr;
            arena->bytes = 0;
            VQKV_CUDA(cudaMalloc(&arena->base, need));
            arena->bytes = need;
        }
        for (uint32_t b = 0; b < nbuf; ++b) {
            uint8_t* p0 = arena->base + uint64_t(b) * (bx + bp + bn);
            dx[b] = reinterpret_cast<float*>(p0);
            dp[b] = p0 + bx;
            dn[b] = reinterpret_cast<float*>(p0 + bx + bp);
            VQKV_CUDA(cudaEventCreateWithFlags(&in_ready[b], cudaEventDisableTiming));
            VQKV_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
            VQKV_CUDA(cudaEventCreateWithFlags(&out_done[b], cudaEventDisableTiming));
        }
        VQKV_CUDA(cudaEventCreateWithFlags(&last, cudaEventDisableTiming));
        uint32_t i = 0;
        for (uint32_t s0 = 0; s0 < n_streams; s0 += chunk, ++i) {
            const uint32_t b = i % nbuf;
            const uint32_t ns = std::min<uint32_t>(chunk, n_streams - s0);
            // a buffer's first use follows its allocation on cp_in; a reuse waits for its last copy-out
            // (never for other calls' copies queued on the shared copy-out stream)
            if (i >= nbuf) VQKV_CUDA(cudaStreamWaitEvent(cp_in, out_done[b], 0));
            VQKV_CUDA(cudaMemcpyAsync(dx[b], xs + uint64_t(s0) * rows * D, per_stream_in * ns, cudaMemcpyHostToDevice,
                                      cp_in));
            VQKV_CUDA(cudaEventRecord(in_ready[b], cp_in));
            cudaStream_t ce = cst[i & 1];
            VQKV_CUDA(cudaStreamWaitEvent(ce, in_ready[b], 0));
            quantize_device(*s, dx[b], ns, rows, sb, dp[b], dn[b], nullptr, ce, false);
            VQKV_CUDA(cudaEventRecord(done[b], ce));
            VQKV_CUDA(cudaStreamWaitEvent(cp_out, done[b], 0));
            VQKV_CUDA(cudaMemcpyAsync(payload + uint64_t(s0) * pb, dp[b], pb * ns, cudaMemcpyDeviceToHost, cp_out));
            VQKV_CUDA(cudaMemcpyAsync(norms + uint64_t(s0) * rows, dn[b], sizeof(float) * rows * ns,
                                      cudaMemcpyDeviceToHost, cp_out));
            VQKV_CUDA(cudaEventRecord(out_done[b], cp_out));
        }
        // the caller's stream completes only after the last copy-out; staging is
        // returned to the pool in stream order behind it
        VQKV_CUDA(cudaEventRecord(last, cp_out));  // after every chunk's copy-out, hence every encode
        VQKV_CUDA(cudaStreamWaitEvent(cs, last, 0));
        VQKV_CUDA(cudaEventRecord(arena->done, cs));  // after every copy-out: the arena is free again
        for (uint32_t b = 0; b < nbuf; ++b) {
            cudaEventDestroy(in_ready[b]);  // released once complete
            cudaEventDestroy(done[b]);
            cudaEventDestroy(out_done[b]);
        }
        cudaEventDestroy(last);
    });
}

int vqkv_reconstruct_block(vqkv_stack_t s, const uint8_t* payload, uint32_t n_streams, uint64_t rows, uint64_t begin,
                           uint64_t end, float* out, void* stream) {
    return vqkv_reconstruct_block_ex(s, payload, 0, n_streams, rows, begin, end, out, stream);
}

int vqkv_reconstruct_block_ex(vqkv_stack_t s, const uint8_t* payload, uint64_t stream_stride, uint32_t n_streams,
                              uint64_t rows, uint64_t begin, uint64_t end, float* out, void* stream) {
    return guard([&] {
        check_stack(s);
        // codebook.cpp:241-244
        if (begin > end || end > rows)
            fail(VQKV_INVALID_INPUT, "row range [" + std::to_string(begin) + ", " + std::to_string(end) +
                                         ") out of bounds for " + std::to_string(rows) + " rows");
        if (end == begin || n_streams == 0) return;
        need(payload && out, VQKV_INVALID_INPUT, "null device buffer");
        DeviceGuard g(s->device);
        need(stream_stride == 0 || stream_stride >= payload_bytes(s->row_bits, rows), VQKV_INVALID_INPUT,
             "payload stream stride shorter than the payload");
        launch_reconstruct(*s, payload, n_streams, rows, begin, end, out, as_stream(stream), stream_stride);
    });
}

int vqkv_attend_decode(vqkv_stack_t ks, vqkv_stack_t vs, const vqkv_attend_args* a, void* stream) {
    return guard([&] {
        check_stack(ks);
        check_stack(vs);
        need(a != nullptr, VQKV_INVALID_INPUT, "null args");
        need(ks->device == vs->device, VQKV_INVALID_INPUT, "key and value stacks live on different devices");
        if (a->n_pairs == 0 || a->group == 0) return;
        // attention.cpp:29-34
        need(a->n_init + a->n_comp + a->n_local >= 1, VQKV_INVALID_STATE, "cannot attend over an empty cache");
        need(a->q_dev && a->out_dev, VQKV_INVALID_INPUT, "null device buffer");
        need(a->n_init == 0 || (a->init_k_dev && a->init_v_dev), VQKV_INVALID_INPUT, "null init rows");
        need(a->n_local == 0 || (a->local_k_dev && a->local_v_dev), VQKV_INVALID_INPUT, "null local rows");
        need(a->n_comp == 0 || (a->kcodes_dev && a->vcodes_dev), VQKV_INVALID_INPUT, "null code payloads");
        need(a->kcodes_layout == VQKV_KEYCODES_ROWS || a->kcodes_layout == VQKV_KEYCODES_GROUP_MAJOR, VQKV_INVALID_INPUT,
             "unknown key-code layout");
        if (a->kcodes_layout == VQKV_KEYCODES_GROUP_MAJOR && a->n_comp > 0) {
            need(vqkv_dev::gm_supported(*ks) && vqkv_dev::attend_path() != 1 && vqkv_dev::attend_lut_supported(*ks, *vs, *a),
                 VQKV_INVALID_INPUT, "group-major key codes need the LUT attention path (D = 128, group 4, <= 1024 entries)");
            const uint64_t need_b = vqkv_dev::gm_pair_bytes(*ks, a->kcodes_cap);
            need(a->kcodes_cap % 16 == 0 && a->kcodes_cap >= a->n_comp, VQKV_INVALID_INPUT,
                 "kcodes_cap must be a multiple of 16 and >= n_comp");
            need(a->kcodes_stride == 0 || (a->kcodes_stride >= need_b && a->kcodes_stride % 16 == 0), VQKV_INVALID_INPUT,
                 "group-major kcodes_stride must be >= the buffer size and a multiple of 16");
            need(reinterpret_cast<uintptr_t>(a->kcodes_dev) % 16 == 0, VQKV_INVALID_INPUT,
                 "group-major key codes must be 16-byte aligned");
        }
        DeviceGuard g(ks->device);
        launch_attend(*ks, *vs, *a, as_stream(stream));
    });
}

uint64_t vqkv_keycodes_gm_bytes(vqkv_stack_t ks, uint64_t cap) {
    if (!ks || cap % 16 != 0 || !vqkv_dev::gm_supported(*ks)) return 0;
    return vqkv_dev::gm_pair_bytes(*ks, cap);
}

int vqkv_attend_gm_supported(vqkv_stack_t ks, vqkv_stack_t vs, const vqkv_attend_args* a) {
    if (!ks || !vs || !a) return 0;
    return (vqkv_dev::gm_supported(*ks) && vqkv_dev::attend_path() != 1 && vqkv_dev::attend_lut_supported(*ks, *vs, *a))
               ? 1
               : 0;
}

int vqkv_keycodes_to_gm(vqkv_stack_t ks, const uint8_t* payload, uint64_t payload_stride, uint32_t n_pairs,
                        uint64_t src_row, uint64_t count, uint8_t* gm, uint64_t cap, uint64_t gm_stride, uint64_t dst_row,
                        void* stream) {
    return guard([&] {
        check_stack(ks);
        need(vqkv_dev::gm_supported(*ks), VQKV_INVALID_INPUT, "stack has no group-major layout (D = 128, <= 1024 entries)");
        need(cap % 16 == 0 && dst_row + count <= cap, VQKV_INVALID_INPUT, "records out of the group-major capacity");
        const uint64_t gb = vqkv_dev::gm_pair_bytes(*ks, cap);
        need(gm_stride == 0 || gm_stride >= gb, VQKV_INVALID_INPUT, "gm_stride below the buffer size");
        const uint64_t pb = payload_bytes(ks->row_bits, src_row + count);
        need(payload_stride == 0 || payload_stride >= pb, VQKV_INVALID_INPUT, "payload_stride below the payload size");
        if (n_pairs == 0 || count == 0) return;
        need(payload && gm, VQKV_INVALID_INPUT, "null device buffer");
        DeviceGuard g(ks->device);
        vqkv_dev::launch_keycodes_to_gm(*ks, payload, payload_stride ? payload_stride : pb, n_pairs, src_row, count, gm, cap,
                                        gm_stride ? gm_stride : gb, dst_row, as_stream(stream));
    });
}

int vqkv_keycodes_from_gm(vqkv_stack_t ks, const uint8_t* gm, uint64_t cap, uint64_t gm_stride, uint32_t n_pairs,
                          uint64_t count, uint8_t* payload, uint64_t payload_stride, void* stream) {
    return guard([&] {
        check_stack(ks);
        need(vqkv_dev::gm_supported(*ks), VQKV_INVALID_INPUT, "stack has no group-major layout (D = 128, <= 1024 entries)");
        need(cap % 16 == 0 && count <= cap, VQKV_INVALID_INPUT, "records out of the group-major capacity");
        const uint64_t gb = vqkv_dev::gm_pair_bytes(*ks, cap), pb = payload_bytes(ks->row_bits, count);
        need(gm_stride == 0 || gm_stride >= gb, VQKV_INVALID_INPUT, "gm_stride below the buffer size");
        need(payload_stride == 0 || payload_stride >= pb, VQKV_INVALID_INPUT, "payload_stride below the payload size");
        if (n_pairs == 0 || count == 0) return;
        need(payload && gm, VQKV_INVALID_INPUT, "null device buffer");
        DeviceGuard g(ks->device);
        vqkv_dev::launch_keycodes_from_gm(*ks, gm, cap, gm_stride ? gm_stride : gb, n_pairs, count, payload,
                                          payload_stride ? payload_stride : pb, as_stream(stream));
    });
}

int vqkv_quantize_rows_host(vqkv_stack_t s, const float* xs, uint64_t rows, uint64_t sb, uint8_t* payload, float* norms,
                            float* residuals) {
    return guard([&] {
        check_stack(s);
        need(sb >= 1, VQKV_INVALID_INPUT, "search_block must be >= 1");
        if (rows == 0) return;
        DeviceGuard g(s->device);
        std::lock_guard<std::mutex> lk(s->host_mu);
        const uint64_t D = s->dim, pb = payload_bytes(s->row_bits, rows);
        HostScratch hs(*s);
        const uint64_t ox = hs.add(sizeof(float) * rows * D), on = hs.add(sizeof(float) * rows), op = hs.add(pb),
                       orr = residuals ? hs.add(sizeof(float) * rows * D) : 0;
        uint8_t* base = hs.commit();
        float* dx = reinterpret_cast<float*>(base + ox);
        float* dn = reinterpret_cast<float*>(base + on);
        uint8_t* dp = base + op;
        float* dr = residuals ? reinterpret_cast<float*>(base + orr) : nullptr;
        VQKV_CUDA(cudaMemcpy(dx, xs, sizeof(float) * rows * D, cudaMemcpyHostToDevice));
        quantize_device(*s, dx, 1, rows, sb, dp, dn, dr, nullptr);
        if (pb && payload) VQKV_CUDA(cudaMemcpy(payload, dp, pb, cudaMemcpyDeviceToHost));
        if (norms) VQKV_CUDA(cudaMemcpy(norms, dn, sizeof(float) * rows, cudaMemcpyDeviceToHost));
        if (residuals) VQKV_CUDA(cudaMemcpy(residuals, dr, sizeof(float) * rows * D, cudaMemcpyDeviceToHost));
    });
}

int vqkv_nearest_host(vqkv_stack_t s, uint32_t stage, const float* x, uint64_t sb, uint32_t* index, float* distance) {
    return guard([&] {
        check_stack(s);
        need(stage < s->n, VQKV_INVALID_INPUT, "stage out of range");
        need(sb >= 1, VQKV_INVALID_INPUT, "search_block must be >= 1");
        DeviceGuard g(s->device);
        std::lock_guard<std::mutex> lk(s->host_mu);
        HostScratch hs(*s);
        const uint64_t ox = hs.add(sizeof(float) * s->dim), oi = hs.add(sizeof(uint32_t)), od = hs.add(sizeof(float));
        uint8_t* base = hs.commit();
        float* dx = reinterpret_cast<float*>(base + ox);
        uint32_t* di = reinterpret_cast<uint32_t*>(base + oi);
        float* dd = reinterpret_cast<float*>(base + od);
        VQKV_CUDA(cudaMemcpy(dx, x, sizeof(float) * s->dim, cudaMemcpyHostToDevice));
        launch_nearest(*s, stage, dx, 1, sb, di, dd, nullptr);
        VQKV_CUDA(cudaMemcpy(index, di, sizeof(uint32_t), cudaMemcpyDeviceToHost));
        VQKV_CUDA(cudaMemcpy(distance, dd, sizeof(float), cudaMemcpyDeviceToHost));
    });
}

int vqkv_reconstruct_block_host(vqkv_stack_t s, const uint8_t* payload, uint64_t rows, uint64_t begin, uint64_t end,
                                float* out) {
    return guard([&] {
        check_stack(s);
        if (begin > end || end > rows)
            fail(VQKV_INVALID_INPUT, "row range [" + std::to_string(begin) + ", " + std::to_string(end) +
                                         ") out of bounds for " + std::to_string(rows) + " rows");
        if (end == begin) return;
        DeviceGuard g(s->device);
        std::lock_guard<std::mutex> lk(s->host_mu);
        const uint64_t pb = payload_bytes(s->row_bits, rows);
        HostScratch hs(*s);
        const uint64_t op = hs.add(pb), oo = hs.add(sizeof(float) * (end - begin) * s->dim);
        uint8_t* base = hs.commit();
        uint8_t* dp = base + op;
        float* dout = reinterpret_cast<float*>(base + oo);
        if (pb) VQKV_CUDA(cudaMemcpy(dp, payload, pb, cudaMemcpyHostToDevice));
        launch_reconstruct(*s, dp, 1, rows, begin, end, dout, nullptr);
        VQKV_CUDA(cudaMemcpy(out, dout, sizeof(float) * (end - begin) * s->dim, cudaMemcpyDeviceToHost));
        int code = 0;
        VQKV_CUDA(cudaMemcpy(&code, s->d_error, sizeof(int), cudaMemcpyDeviceToHost));
        VQKV_CUDA(cudaMemset(s->d_error, 0, sizeof(int)));
        if (code) fail(VQKV_INVALID_CODE, "code index out of range for its stage");
    });
}

int vqkv_attend_decode_host(vqkv_stack_t ks, vqkv_stack_t vs, const vqkv_attend_args* h) {
    return guard([&] {
        check_stack(ks);
        check_stack(vs);
        need(h != nullptr, VQKV_INVALID_INPUT, "null args");
        if (h->n_pairs == 0 || h->group == 0) return;
        need(h->n_init + h->n_comp + h->n_local >= 1, VQKV_INVALID_STATE, "cannot attend over an empty cache");
        need(ks->device == vs->device, VQKV_INVALID_INPUT, "key and value stacks live on different devices");
        need(h->init_stride == 0 && h->local_stride == 0 && h->kcodes_stride == 0 && h->vcodes_stride == 0,
             VQKV_INVALID_INPUT, "host attention buffers must be dense (strides 0)");
        need(h->kcodes_layout == VQKV_KEYCODES_ROWS, VQKV_INVALID_INPUT, "host attention takes CodeMatrix key rows");
        DeviceGuard g(ks->device);
        std::lock_guard<std::mutex> lk(ks->host_mu);
        const uint64_t P = h->n_pairs, G = h->group, Dk = ks->dim, Dv = vs->dim;
        struct Up {
            const void* src;
            uint64_t bytes, off;
        };
        HostScratch hs(*ks);
        auto plan = [&](const void* src, uint64_t bytes) { return Up{src, bytes, (src && bytes) ? hs.add(bytes) : 0}; };
        Up uq = plan(h->q_dev, sizeof(float) * P * G * Dk), uik = plan(h->init_k_dev, sizeof(float) * P * h->n_init * Dk),
           uiv = plan(h->init_v_dev, sizeof(float) * P * h->n_init * Dv),
           ulk = plan(h->local_k_dev, sizeof(float) * P * h->n_local * Dk),
           ulv = plan(h->local_v_dev, sizeof(float) * P * h->n_local * Dv),
           ukc = plan(h->kcodes_dev, P * payload_bytes(ks->row_bits, h->n_comp)),
           uvc = plan(h->vcodes_dev, P * payload_bytes(vs->row_bits, h->n_comp));
        const uint64_t oo = hs.add(sizeof(float) * P * G * Dv), ol = hs.add(sizeof(float) * P * G);
        uint8_t* base = hs.commit();
        auto up = [&](const Up& u) -> void* {
            if (!u.src || !u.bytes) return nullptr;
            VQKV_CUDA(cudaMemcpy(base + u.off, u.src, u.bytes, cudaMemcpyHostToDevice));
            return base + u.off;
        };
        vqkv_attend_args d = *h;
        d.q_dev = static_cast<const float*>(up(uq));
        d.init_k_dev = static_cast<const float*>(up(uik));
        d.init_v_dev = static_cast<const float*>(up(uiv));
        d.local_k_dev = static_cast<const float*>(up(ulk));
        d.local_v_dev = static_cast<const float*>(up(ulv));
        d.kcodes_dev = static_cast<const uint8_t*>(up(ukc));
        d.vcodes_dev = static_cast<const uint8_t*>(up(uvc));
        float* dout = reinterpret_cast<float*>(base + oo);
        float* dlse = reinterpret_cast<float*>(base + ol);
        d.out_dev = dout;
        d.lse_dev = h->lse_dev ? dlse : nullptr;
        need(d.q_dev != nullptr, VQKV_INVALID_INPUT, "null query");
        need(d.n_init == 0 || (d.init_k_dev && d.init_v_dev), VQKV_INVALID_INPUT, "null init rows");
        need(d.n_local == 0 || (d.local_k_dev && d.local_v_dev), VQKV_INVALID_INPUT, "null local rows");
        need(d.n_comp == 0 || (d.kcodes_dev && d.vcodes_dev), VQKV_INVALID_INPUT, "null code payloads");
        launch_attend(*ks, *vs, d, nullptr);
        VQKV_CUDA(cudaMemcpy(h->out_dev, dout, sizeof(float) * P * G * Dv, cudaMemcpyDeviceToHost));
        if (h->lse_dev) VQKV_CUDA(cudaMemcpy(h->lse_dev, dlse, sizeof(float) * P * G, cudaMemcpyDeviceToHost));
    });
}

int vqkv_attend_raw_host(int device, const float* keys, const float* values, uint64_t rows, uint32_t dk, uint32_t dv,
                         const float* query, double scale, float* out) {
    return guard([&] {
        // attention.cpp:73-78
        need(rows >= 1, VQKV_INVALID_INPUT, "keys and values must be nonempty and the same length");
        need(dk >= 1 && dv >= 1, VQKV_INVALID_INPUT, "query dimension does not match key dimension");
        need(keys && values && query && out, VQKV_INVALID_INPUT, "null host buffer");
        DeviceGuard g(device);
        struct Buf {  // RAII: freed on every path
            void* p = nullptr;
            ~Buf() {
                if (p) cudaFree(p);
            }
        } b;
        const uint64_t nk = rows * dk, nv = rows * dv;
        VQKV_CUDA(cudaMalloc(&b.p, sizeof(float) * (nk + nv + dk + dv)));
        float* d = static_cast<float*>(b.p);
        VQKV_CUDA(cudaMemcpy(d, keys, sizeof(float) * nk, cudaMemcpyHostToDevice));
        VQKV_CUDA(cudaMemcpy(d + nk, values, sizeof(float) * nv, cudaMemcpyHostToDevice));
        VQKV_CUDA(cudaMemcpy(d + nk + nv, query, sizeof(float) * dk, cudaMemcpyHostToDevice));
        launch_attend_raw(device, d, d + nk, rows, dk, dv, d + nk + nv, scale, d + nk + nv + dk, nullptr);
        VQKV_CUDA(cudaMemcpy(out, d + nk + nv + dk, sizeof(float) * dv, cudaMemcpyDeviceToHost));
    });
}

int vqkv_lse_combine(const float* o, const float* lse, uint32_t parts, uint64_t rows, uint32_t dv, float* out,
                     float* out_lse, void* stream) {
    return guard([&] {
        need(parts >= 1, VQKV_INVALID_INPUT, "need at least one partial result");
        if (rows == 0) return;
        need(o && lse && out, VQKV_INVALID_INPUT, "null device buffer");
        launch_lse_combine(o, lse, parts, rows, dv, out, out_lse, as_stream(stream));
    });
}

int vqkv_lse_allgather_combine(void* comm, const float* o, const float* lse, uint64_t rows, uint32_t dv, float* go,
                               float* gl, float* out, float* out_lse, void* stream) {
    return guard([&] {
        need(comm != nullptr, VQKV_INVALID_INPUT, "null NCCL communicator");
        if (rows == 0) return;
        need(o && lse && out, VQKV_INVALID_INPUT, "null device buffer");
        need(dv >= 1, VQKV_INVALID_INPUT, "dv must be >= 1");
        lse_allgather_combine(comm, o, lse, rows, dv, go, gl, out, out_lse, as_stream(stream));
    });
}

int vqkv_train_batch(vqkv_stack_t s, const float* batch, uint64_t rows, float beta, float gamma, int square_commitment,
                     float* grad_proj, double* sums, void* stream) {
    return guard([&] {
        check_stack(s);
        need(rows >= 1, VQKV_INVALID_INPUT, "loss needs a nonempty batch");
        need(batch && sums, VQKV_INVALID_INPUT, "null buffer");
        need(beta >= 0.f && gamma >= 0.f, VQKV_INVALID_INPUT, "beta and gamma must be nonnegative");
        DeviceGuard g(s->device);
        train_batch(*s, batch, rows, beta, gamma, square_commitment != 0, grad_proj, sums, as_stream(stream));
    });
}

int vqkv_train_batch_host(vqkv_stack_t s, const float* batch, uint64_t rows, float beta, float gamma,
                          int square_commitment, float* grad_proj, double* sums) {
    return guard([&] {
        check_stack(s);
        need(rows >= 1, VQKV_INVALID_INPUT, "loss needs a nonempty batch");
        need(batch && sums, VQKV_INVALID_INPUT, "null buffer");
        need(beta >= 0.f && gamma >= 0.f, VQKV_INVALID_INPUT, "beta and gamma must be nonnegative");
        DeviceGuard g(s->device);
        std::lock_guard<std::mutex> lk(s->host_mu);
        const uint64_t D = s->dim, gb = grad_proj ? sizeof(float) * uint64_t(s->n) * D * D : 0;
        HostScratch hs(*s);
        const uint64_t ob = hs.add(sizeof(float) * rows * D), og = hs.add(std::max<uint64_t>(gb, 1));
        uint8_t* base = hs.commit();
        float* db = reinterpret_cast<float*>(base + ob);
        float* dg = reinterpret_cast<float*>(base + og);
        VQKV_CUDA(cudaMemcpy(db, batch, sizeof(float) * rows * D, cudaMemcpyHostToDevice));
        train_batch(*s, db, rows, beta, gamma, square_commitment != 0, grad_proj ? dg : nullptr, sums, nullptr);
        if (grad_proj) VQKV_CUDA(cudaMemcpy(grad_proj, dg, gb, cudaMemcpyDeviceToHost));
    });
}

int vqkv_nccl_comm_init_all(int ndev, const int* devs, void** comms) {
    return guard([&] {
        need(ndev >= 1 && devs && comms, VQKV_INVALID_INPUT, "ndev >= 1 devices and a comms array required");
        nccl_comm_init_all(ndev, devs, comms);
    });
}

int vqkv_nccl_comm_destroy(void* comm) {
    return guard([&] {
        need(comm != nullptr, VQKV_INVALID_INPUT, "null NCCL communicator");
        nccl_comm_destroy(comm);
    });
}

}  // extern "C"
