// vqkv_cli.cpp -- the `vqkv` command-line front end on the B200 build: the reference's subcommands
// (proj/tools/vqkv.cpp: ratio, gen, train, compress, stats, bench) with the same options and the same
// key=value output lines, over the drop-in C++ API (include/vqkv/*.hpp -> libvqkv_b200.so): compress
// runs the GPU encoder, bench the GPU cache / attention / fidelity path, train the GPU trainer.
// Option parsing is a small hand-written --name value scanner (the reference uses CLI11).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "vqkv/attention.hpp"
#include "vqkv/kv_cache.hpp"
#include "vqkv/ratio.hpp"
#include "vqkv/synthetic.hpp"
#include "vqkv/trainer.hpp"

using namespace vqkv;

namespace {

// --name value / --flag scanner for one subcommand
struct Args {
    std::map<std::string, std::string> kv;
    std::map<std::string, bool> flags;
    Args(int argc, char** argv, const std::vector<std::string>& flag_names) {
        for (int i = 2; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw InvalidInput("unexpected argument '" + a + "'");
            bool is_flag = false;
            for (const auto& f : flag_names) is_flag |= (a == f);
            if (is_flag) {
                flags[a] = true;
                continue;
            }
            if (i + 1 >= argc) throw InvalidInput("option " + a + " needs a value");
            kv[a] = argv[++i];
        }
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    std::string str(const std::string& k, const std::string& def = "") const { return has(k) ? kv.at(k) : def; }
    std::string req(const std::string& k) const {
        if (!has(k)) throw InvalidInput(k + " is required");
        return kv.at(k);
    }
    uint64_t u(const std::string& k, uint64_t def) const { return has(k) ? std::stoull(kv.at(k)) : def; }
    double d(const std::string& k, double def) const { return has(k) ? std::stod(kv.at(k)) : def; }
    bool flag(const std::string& k) const { return flags.count(k) != 0; }
};

std::vector<uint32_t> parse_list(const std::string& spec, const char* what) {
    std::vector<uint32_t> v;
    std::stringstream ss(spec);
    std::string item;
    while (std::getline(ss, item, ',')) v.push_back(uint32_t(std::stoul(item)));
    if (v.empty()) throw InvalidInput(std::string(what) + " needs at least one value");
    return v;
}

SyntheticKind parse_kind(const std::string& name) {
    if (name == "gaussian_mixture") return SyntheticKind::gaussian_mixture;
    if (name == "rope_rotated_keys") return SyntheticKind::rope_rotated_keys;
    throw InvalidInput("unknown kind '" + name + "'");
}

// bench --spec "key=value,..." (vqkv.cpp:53-81)
SyntheticSpec parse_spec(const std::string& text) {
    SyntheticSpec spec;
    std::stringstream ss(text);
    std::string item;
    while (std::getline(ss, item, ',')) {
        const size_t eq = item.find('=');
        if (eq == std::string::npos) throw InvalidInput("bad --spec entry '" + item + "', expected key=value");
        const std::string key = item.substr(0, eq), value = item.substr(eq + 1);
        if (key == "kind") spec.kind = parse_kind(value);
        else if (key == "components") spec.component_count = uint32_t(std::stoul(value));
        else if (key == "seed") spec.seed = std::stoull(value);
        else if (key == "std") spec.component_std = std::stof(value);
        else if (key == "mean_scale") spec.mean_scale = std::stof(value);
        else if (key == "rope_base") spec.rope_base = std::stod(value);
        else throw InvalidInput("unknown --spec key '" + key + "'");
    }
    return spec;
}

void print_ratio(const RatioConfig& c, bool precise) {
    const double r = compression_ratio_percent(c);
    if (precise)
        std::printf("ratio nk=%u sk=%u nv=%u sv=%u dk=%u dv=%u percent=%.6f\n", c.n_key, c.s_key, c.n_value, c.s_value,
                    c.d_key, c.d_value, r);
    else
        std::printf("%.1f%%\n", r);
}

// rows [b, e) of a row-major matrix
MatrixF rows_of(const MatrixF& m, int64_t b, int64_t e) {
    MatrixF out(e - b, m.cols());
    std::copy(m.data() + b * m.cols(), m.data() + e * m.cols(), out.data());
    return out;
}
VectorF row_vec(const MatrixF& m, int64_t r) {
    VectorF v(m.cols());
    std::copy(m.data() + r * m.cols(), m.data() + (r + 1) * m.cols(), v.data());
    return v;
}

int cmd_ratio(const Args& a) {
    RatioConfig c;
    c.n_key = uint32_t(std::stoul(a.req("--nk")));
    c.s_key = uint32_t(std::stoul(a.req("--sk")));
    c.n_value = uint32_t(std::stoul(a.req("--nv")));
    c.s_value = uint32_t(std::stoul(a.req("--sv")));
    c.d_key = uint32_t(a.u("--dk", 128));
    c.d_value = uint32_t(a.u("--dv", 128));
    print_ratio(c, a.flag("--precise"));
    return 0;
}

int cmd_gen(const Args& a) {
    SyntheticSpec spec;
    spec.kind = parse_kind(a.str("--kind", "gaussian_mixture"));
    spec.dim = int64_t(a.u("--dim", uint64_t(spec.dim)));
    spec.count = int64_t(std::stoull(a.req("--count")));
    spec.component_count = uint32_t(a.u("--components", spec.component_count));
    spec.seed = a.u("--seed", spec.seed);
    spec.component_std = float(a.d("--std", spec.component_std));
    spec.mean_scale = float(a.d("--mean-scale", spec.mean_scale));
    spec.rope_base = a.d("--rope-base", spec.rope_base);
    const std::string out = a.req("--out");
    save_dataset(generate(spec), out);
    std::printf("gen kind=%s dim=%lld count=%lld out=%s\n",
                spec.kind == SyntheticKind::gaussian_mixture ? "gaussian_mixture" : "rope_rotated_keys",
                static_cast<long long>(spec.dim), static_cast<long long>(spec.count), out.c_str());
    return 0;
}

int cmd_train(const Args& a) {
    TrainConfig c;
    c.learning_rate = float(a.d("--lr", c.learning_rate));
    c.batch_size = size_t(a.u("--batch", c.batch_size));
    c.epochs = size_t(a.u("--epochs", c.epochs));
    c.beta = float(a.d("--beta", c.beta));
    c.gamma = float(a.d("--gamma", c.gamma));
    c.seed = a.u("--seed", c.seed);
    c.init_scale = float(a.d("--init-scale", c.init_scale));
    c.train_entries = a.flag("--train-entries");
    c.square_commitment = a.flag("--square-commitment");
    const std::string kind = a.str("--kind", "key");
    if (kind != "key" && kind != "value") throw InvalidInput("--kind must be key or value");
    const std::string out = a.req("--out");
    const VectorDataset data = load_dataset(a.req("--data"));
    TrainResult r = train(data, parse_list(a.req("--stages"), "--stages"), c,
                          kind == "key" ? CacheKind::key : CacheKind::value);
    save_stack(r.stack, out);
    for (size_t e = 0; e < r.report.per_epoch_loss.size(); ++e)
        std::printf("epoch index=%zu loss=%.8g\n", e + 1, r.report.per_epoch_loss[e]);
    for (size_t i = 0; i < r.report.per_stage_mse.size(); ++i)
        std::printf("stage index=%zu holdout_mse=%.8g\n", i + 1, r.report.per_stage_mse[i]);
    std::printf("train final_mse=%.8g stack=%s\n", r.report.final_mse, out.c_str());
    return 0;
}

// compress: VQCM file = "VQCM" + CodeMatrix::save (vqkv.cpp:125-146)
int cmd_compress(const Args& a) {
    const VectorDataset data = load_dataset(a.req("--data"));
    const CodebookStack stack = load_stack(a.req("--stack"));
    const std::string out_path = a.req("--out");
    if (data.dim() != stack.dim()) throw InvalidInput("dataset dimension does not match stack dimension");
    const QuantizeBatchResult r = quantize_batch(stack, data.payload);
    std::ofstream out(out_path, std::ios::binary);
    if (!out) throw IoError("cannot open " + out_path + " for writing");
    out.write("VQCM", 4);
    r.codes.save(out);
    if (!out) throw IoError("write failed for " + out_path);
    double mse = 0.0;
    for (int64_t i = 0; i < r.residual_norms.size(); ++i) mse += double(r.residual_norms[i]) * double(r.residual_norms[i]);
    mse /= double(r.residual_norms.size());
    std::printf("compress rows=%zu payload_bits=%zu mse=%.8g out=%s\n", r.codes.rows(), r.codes.payload_bits(), mse,
                out_path.c_str());
    return 0;
}

int cmd_stats(const Args& a) {
    if (a.has("--config")) {
        const std::vector<uint32_t> v = parse_list(a.str("--config"), "--config");
        if (v.size() != 4 && v.size() != 6) throw InvalidInput("--config expects nk,sk,nv,sv[,dk,dv]");
        RatioConfig c{v[0], v[1], v[2], v[3], v.size() == 6 ? v[4] : 128u, v.size() == 6 ? v[5] : 128u};
        print_ratio(c, a.flag("--precise"));
        return 0;
    }
    if (a.has("--snapshot")) {
        if (!a.has("--key-stack") || !a.has("--value-stack"))
            throw InvalidInput("--snapshot needs --key-stack and --value-stack");
        const CodebookStack ks = load_stack(a.str("--key-stack")), vs = load_stack(a.str("--value-stack"));
        const CacheState st = CacheState::load_snapshot(a.str("--snapshot"), ks, vs);
        const MemoryReport m = st.memory_report();
        std::printf("segments init=%zu compressed=%zu pending=%zu local=%zu total=%zu\n", st.init_rows(),
                    st.compressed_rows(), st.pending_rows(), st.local_rows(), st.total_len());
        std::printf("memory raw_bytes_equivalent=%zu compressed_payload_bits=%zu codebook_overhead_bytes=%zu "
                    "effective_ratio=%.6f\n",
                    m.raw_bytes_equivalent, m.compressed_payload_bits, m.codebook_overhead_bytes, m.effective_ratio);
        return 0;
    }
    throw InvalidInput("stats needs --config or --snapshot");
}

// prefill / decode simulation with memory checkpoints and a fidelity report (vqkv.cpp:180-248)
int cmd_bench(const Args& a) {
    const CodebookStack ks = load_stack(a.req("--key-stack")), vs = load_stack(a.req("--value-stack"));
    const size_t init_len = size_t(a.u("--linit", 4)), local_len = size_t(a.u("--llocal", 1024));
    const size_t tokens = size_t(std::stoull(a.req("--tokens")));
    size_t prefill_len = size_t(a.u("--prefill", 2048));
    const size_t n_queries = size_t(a.u("--queries", 64)), block_rows = size_t(a.u("--block-rows", 128));
    const size_t checkpoint_every = size_t(a.u("--checkpoint", 0));
    SyntheticSpec kspec = parse_spec(a.str("--spec", "kind=gaussian_mixture,components=32,seed=0"));
    kspec.dim = ks.dim();
    kspec.count = int64_t(tokens);
    SyntheticSpec vspec = kspec;
    vspec.kind = SyntheticKind::gaussian_mixture;
    vspec.dim = vs.dim();
    vspec.seed = kspec.seed + 1;
    const MatrixF keys = generate(kspec).payload, values = generate(vspec).payload;

    CacheState state(ks, vs, WindowPolicy{init_len, local_len, a.flag("--eager")});
    prefill_len = std::min(std::max<size_t>(prefill_len, 1), tokens);
    state.prefill(rows_of(keys, 0, int64_t(prefill_len)), rows_of(values, 0, int64_t(prefill_len)));
    auto checkpoint = [&]() {
        const MemoryReport m = state.memory_report();
        std::printf("checkpoint tokens=%zu init=%zu compressed=%zu pending=%zu local=%zu batched_compressions=%zu "
                    "raw_bytes_equivalent=%zu compressed_payload_bits=%zu codebook_overhead_bytes=%zu "
                    "effective_ratio=%.6f\n",
                    state.total_len(), state.init_rows(), state.compressed_rows(), state.pending_rows(),
                    state.local_rows(), state.batched_compressions(), m.raw_bytes_equivalent, m.compressed_payload_bits,
                    m.codebook_overhead_bytes, m.effective_ratio);
    };
    checkpoint();
    for (size_t t = prefill_len; t < tokens; ++t) {
        state.append_token(row_vec(keys, int64_t(t)), row_vec(values, int64_t(t)));
        if (checkpoint_every > 0 && (t + 1 - prefill_len) % checkpoint_every == 0) checkpoint();
    }
    checkpoint();

    std::mt19937_64 rng(kspec.seed ^ 0x9e3779b97f4a7c15ull);
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    MatrixF queries(int64_t(n_queries), ks.dim());
    for (int64_t i = 0; i < queries.size(); ++i) queries.data()[i] = gauss(rng);
    AttentionConfig attn;
    attn.block_rows = block_rows;
    const FidelityReport fid = fidelity(state, keys, values, queries, attn);
    AttendStats stats;
    attend(state, row_vec(queries, 0), attn, &stats);
    const size_t budget = block_rows * size_t(ks.dim() + vs.dim());
    std::printf("fidelity queries=%zu output_max_abs_err=%.8g output_mean_cosine=%.8f key_intermediate_mse=%.8g "
                "value_intermediate_mse=%.8g\n",
                n_queries, fid.output_max_abs_err, fid.output_mean_cosine, fid.key_intermediate_mse,
                fid.value_intermediate_mse);
    std::printf("working_set peak_reconstructed_scalars=%zu budget_scalars=%zu within_budget=%d\n",
                stats.peak_reconstructed_scalars, budget, stats.peak_reconstructed_scalars <= budget ? 1 : 0);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: vqkv {ratio|gen|train|compress|stats|bench} [--option value ...]\n");
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "ratio") return cmd_ratio(Args(argc, argv, {"--precise"}));
        if (cmd == "gen") return cmd_gen(Args(argc, argv, {}));
        if (cmd == "train") return cmd_train(Args(argc, argv, {"--train-entries", "--square-commitment"}));
        if (cmd == "compress") return cmd_compress(Args(argc, argv, {}));
        if (cmd == "stats") return cmd_stats(Args(argc, argv, {"--precise"}));
        if (cmd == "bench") return cmd_bench(Args(argc, argv, {"--eager"}));
        std::fprintf(stderr, "unknown subcommand '%s'\n", cmd.c_str());
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
