// vqkv/trainer.hpp -- drop-in for proj/core/include/vqkv/trainer.hpp (B200 build).
//
// train() keeps the reference's host loop (trainer.cpp:166-248: shuffling with std::mt19937_64,
// holdout split, mini-batches, SGD step, refresh) and runs every batch's forward pass, loss terms and
// straight-through gradients on the GPU (vqkv_train_batch_host, trainer.cu) in the reference's fp32
// operation order, so a training run reproduces the reference's stack bit for bit.
// train_entries (the ablation that also trains raw entries) is not implemented on the GPU: Unsupported.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "vqkv/codebook.hpp"
#include "vqkv/dataset.hpp"

namespace vqkv {

struct TrainConfig {
    float learning_rate = 0.001f;
    size_t batch_size = 65536;
    size_t epochs = 20;
    float beta = 0.25f;  // codebook-pull weight
    float gamma = 1.0f;  // commitment weight
    uint64_t seed = 0;
    float init_scale = 1.0f;
    bool train_entries = false;      // ablation (not on the GPU)
    bool square_commitment = false;  // square the commitment term
    float holdout_fraction = 0.01f;

    void validate() const {
        if (learning_rate <= 0.0f) throw InvalidInput("learning_rate must be positive");
        if (batch_size < 1) throw InvalidInput("batch_size must be >= 1");
        if (beta < 0.0f || gamma < 0.0f) throw InvalidInput("beta and gamma must be nonnegative");
        if (init_scale < 0.0f || !std::isfinite(init_scale))
            throw InvalidInput("init_scale must be a finite nonnegative value");
        if (holdout_fraction < 0.0f || holdout_fraction >= 1.0f) throw InvalidInput("holdout_fraction must be in [0, 1)");
    }
};

struct TrainReport {
    std::vector<double> per_epoch_loss;
    std::vector<double> per_stage_mse;  // held-out MSE of the reconstruction truncated to i + 1 stages
    double final_mse = 0.0;
};

struct LossTerms {
    double total = 0.0;
    double reconstruction = 0.0;
    double codebook_pull = 0.0;
    double commitment = 0.0;
};

struct TrainResult {
    CodebookStack stack;
    TrainReport report;
};

/// Gaussian entries scaled by init_scale, identity projections (trainer.cpp:125-148).
inline CodebookStack init_stack(int64_t dim, const std::vector<uint32_t>& stage_sizes, const TrainConfig& config,
                                CacheKind kind = CacheKind::key) {
    config.validate();
    if (dim < 1) throw InvalidInput("dimension must be >= 1");
    if (stage_sizes.empty()) throw InvalidInput("need at least one stage");
    for (uint32_t s : stage_sizes)
        if (s < 2) throw InvalidInput("every stage size must be >= 2");
    std::mt19937_64 rng(config.seed);
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    CodebookStack stack;
    stack.cache_kind = kind;
    stack.stages.resize(stage_sizes.size());
    for (size_t i = 0; i < stage_sizes.size(); ++i) {
        Codebook& cb = stack.stages[i];
        cb.entries.resize(stage_sizes[i], dim);
        for (int64_t j = 0; j < cb.entries.size(); ++j) cb.entries.data()[j] = config.init_scale * gauss(rng);
        cb.projection = MatrixF::Identity(dim, dim);
        cb.refresh();
    }
    return stack;
}

namespace detail {
// one batch on the GPU: sums [3 + N], optional gradients [N][D][D]
inline std::vector<double> train_batch(const CodebookStack& stack, const float* rows, size_t n_rows, float beta,
                                       float gamma, bool square_commitment, std::vector<float>* grad) {
    std::vector<double> sums(3 + stack.num_stages());
    if (grad) grad->assign(stack.num_stages() * size_t(stack.dim() * stack.dim()), 0.f);
    check(vqkv_train_batch_host(stack.device(), rows, n_rows, beta, gamma, square_commitment ? 1 : 0,
                                grad ? grad->data() : nullptr, sums.data()));
    return sums;
}
}  // namespace detail

/// Mean batch loss (trainer.cpp:150-160).
inline LossTerms loss(const CodebookStack& stack, const MatrixF& batch, float beta, float gamma,
                      bool square_commitment = false) {
    if (batch.rows() < 1) throw InvalidInput("loss needs a nonempty batch");
    if (batch.cols() != stack.dim()) throw InvalidInput("batch dimension does not match stack");
    const std::vector<double> s =
            detail::train_batch(stack, batch.data(), size_t(batch.rows()), beta, gamma, square_commitment, nullptr);
    LossTerms t;
    const double b = double(batch.rows());
    t.reconstruction = s[0] / b;
    t.codebook_pull = s[1] / b;
    t.commitment = s[2] / b;
    t.total = t.reconstruction + beta * t.codebook_pull + gamma * t.commitment;
    return t;
}

/// Mini-batch SGD with straight-through gradients through the argmin (trainer.cpp:166-248).
inline TrainResult train(const VectorDataset& dataset, const std::vector<uint32_t>& stage_sizes,
                         const TrainConfig& config, CacheKind kind = CacheKind::key) {
    dataset.validate();
    config.validate();
    if (config.train_entries) throw InvalidInput("train_entries is not supported: only the projections are trained (on the GPU)");
    const size_t count = size_t(dataset.count());
    const int64_t dim = dataset.dim();
    size_t batch = config.batch_size;
    if (count < 10 * batch) batch = std::min<size_t>(batch, 1024);  // desk-scale datasets

    std::mt19937_64 rng(config.seed);
    std::vector<size_t> order(count);
    std::iota(order.begin(), order.end(), size_t{0});
    std::shuffle(order.begin(), order.end(), rng);
    size_t n_holdout = 0;
    if (count >= 2) {
        n_holdout = std::max<size_t>(1, size_t(std::llround(double(count) * config.holdout_fraction)));
        n_holdout = std::min(n_holdout, count - 1);
    }
    std::vector<size_t> holdout(order.end() - ptrdiff_t(n_holdout), order.end());
    std::vector<size_t> train_rows(order.begin(), order.end() - ptrdiff_t(n_holdout));
    if (holdout.empty()) holdout = train_rows;  // single-vector dataset: evaluate in-sample

    TrainResult result;
    result.stack = init_stack(dim, stage_sizes, config, kind);
    CodebookStack& stack = result.stack;
    const size_t n_stages = stack.num_stages(), dd = size_t(dim * dim);
    std::vector<float> buf, grad;
    for (size_t epoch = 0; epoch < config.epochs; ++epoch) {
        std::shuffle(train_rows.begin(), train_rows.end(), rng);
        double epoch_loss = 0.0;
        size_t seen = 0;
        for (size_t begin = 0; begin < train_rows.size(); begin += batch) {
            const size_t len = std::min(batch, train_rows.size() - begin);
            buf.resize(len * size_t(dim));
            for (size_t i = 0; i < len; ++i)
                std::copy(dataset.payload.data() + train_rows[begin + i] * size_t(dim),
                          dataset.payload.data() + (train_rows[begin + i] + 1) * size_t(dim), buf.data() + i * size_t(dim));
            const std::vector<double> s =
                    detail::train_batch(stack, buf.data(), len, config.beta, config.gamma, config.square_commitment, &grad);
            const double b = double(len);
            const double total = s[0] / b + config.beta * (s[1] / b) + config.gamma * (s[2] / b);
            if (!std::isfinite(total)) throw DivergedError("training loss became non-finite", epoch + 1);
            const float step = config.learning_rate / float(len);
            for (size_t i = 0; i < n_stages; ++i) {
                float* p = stack.stages[i].projection.data();
                const float* g = grad.data() + i * dd;
                for (size_t k = 0; k < dd; ++k) p[k] = p[k] - step * g[k];
                stack.stages[i].refresh();
            }
            stack.device_.reset();  // the projections changed: the next batch uploads the new stack
            epoch_loss += total * b;
            seen += len;
        }
        result.report.per_epoch_loss.push_back(epoch_loss / double(seen));
    }
    // holdout_stage_mse (trainer.cpp:88-103)
    buf.resize(holdout.size() * size_t(dim));
    for (size_t i = 0; i < holdout.size(); ++i)
        std::copy(dataset.payload.data() + holdout[i] * size_t(dim), dataset.payload.data() + (holdout[i] + 1) * size_t(dim),
                  buf.data() + i * size_t(dim));
    const std::vector<double> s = detail::train_batch(stack, buf.data(), holdout.size(), 0.f, 0.f, false, nullptr);
    for (size_t i = 0; i < n_stages; ++i) result.report.per_stage_mse.push_back(s[3 + i] / double(holdout.size()));
    result.report.final_mse = result.report.per_stage_mse.back();
    return result;
}

}  // namespace vqkv
